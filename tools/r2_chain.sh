#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_coexec.py tests/test_gpu_kernels.py tests/test_gpu_gpt2.py tests/test_gpu_dcgan.py tests/test_gpu_music.py tests/test_gpu_resnet.py "tests/test_gpu_contract.py::test_full_width_gradients[c4-bf16]" "tests/test_gpu_contract.py::test_full_width_gradients[c4-fp32]" "tests/test_gpu_contract.py::test_full_width_gradients[c2-fp32]" -q --tb=short > gpurun_out/chain_tests.log 2>&1; echo rc=$? >> gpurun_out/chain_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/chain_c4.json 2> gpurun_out/chain_c4.err
timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/chain_c2.json 2> gpurun_out/chain_c2.err
