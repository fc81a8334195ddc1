#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tc.py tests/test_gpu_ext.py tests/test_gpu_gpt2.py tests/test_gpu_dcgan.py -q -x --tb=short > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/q_c4.json 2> gpurun_out/q_c4.err
timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/q_c2.json 2> gpurun_out/q_c2.err
