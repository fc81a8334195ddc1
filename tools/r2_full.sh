#!/bin/bash
# full gpu suite with contract report, smoke, C4 bf16 + fp32 bench, C2 bench
mkdir -p gpurun_out
rm -f gpurun_out/contract.jsonl
CONTRACT_REPORT=gpurun_out/contract.jsonl timeout 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --precision fp32 --no-cpu-baseline > gpurun_out/bench_c4_fp32.json 2> gpurun_out/bench_c4_fp32.err
timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
