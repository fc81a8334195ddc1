#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/contract.jsonl
CONTRACT_REPORT=gpurun_out/contract.jsonl timeout 900 python -m pytest tests/test_gpu_flash.py "tests/test_gpu_contract.py::test_full_width_gradients[c4-bf16]" tests/test_gpu_gpt2.py -q --tb=short -s > gpurun_out/pytest_fa.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fa.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c4_fa.json 2> gpurun_out/bench_c4_fa.err
