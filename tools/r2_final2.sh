#!/bin/bash
# round-2 closing run: full GPU suite with the contract report, smoke, every workload's bench
# line (C4 default with the CPU baseline), the C4 reference arm, forced-DP C4 with the fused
# gradient reduction
mkdir -p gpurun_out
rm -f gpurun_out/contract.jsonl
CONTRACT_REPORT=gpurun_out/contract.jsonl timeout 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_c4_ref.json 2> gpurun_out/final_c4_ref.err
timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
timeout 600 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err
timeout 900 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err
timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
COEX_NVLS=1 timeout 600 python bench.py --force-dp --no-cpu-baseline > gpurun_out/final_c4_fdp.json 2> gpurun_out/final_c4_fdp.err
