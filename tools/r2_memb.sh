#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_xformer.py tests/test_gpu_ext.py tests/test_gpu_gpt2.py tests/test_gpu_kernels.py "tests/test_gpu_contract.py::test_full_width_gradients[c4-bf16]" "tests/test_gpu_contract.py::test_full_width_gradients[c4-fp32]" "tests/test_gpu_opsweep.py" -q --tb=short > gpurun_out/memb_tests.log 2>&1; echo rc=$? >> gpurun_out/memb_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/memb_c4.json 2> gpurun_out/memb_c4.err
bash tools/r2_profiles.sh
