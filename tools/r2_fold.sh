#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/contract.jsonl
CONTRACT_REPORT=gpurun_out/contract.jsonl timeout 900 python -m pytest tests/test_gpu_flash.py tests/test_gpu_gpt2.py "tests/test_gpu_contract.py::test_full_width_gradients[c4-bf16]" -q -x --tb=short -s > gpurun_out/fold_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fold_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/fold_bench.json 2> gpurun_out/fold_bench.err
