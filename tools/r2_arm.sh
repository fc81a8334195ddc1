#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_coexec.py tests/test_gpu_spec.py tests/test_gpu_cancel.py tests/test_gpu_dcgan.py tests/test_gpu_resnet.py tests/test_gpu_music.py tests/test_gpu_dp.py "tests/test_gpu_contract.py::test_full_width_gradients[c2-bf16]" "tests/test_gpu_contract.py::test_full_width_gradients[c3-bf16]" "tests/test_gpu_contract.py::test_full_width_gradients[c3-fp32]" -q --tb=short > gpurun_out/arm_tests.log 2>&1; echo rc=$? >> gpurun_out/arm_tests.log
timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/arm_c2.json 2> gpurun_out/arm_c2.err
timeout 900 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/arm_c3.json 2> gpurun_out/arm_c3.err
