#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/contract.jsonl
CONTRACT_REPORT=gpurun_out/contract.jsonl timeout 1800 python -m pytest tests/test_gpu_xformer.py tests/test_gpu_gpt2.py tests/test_gpu_music.py tests/test_gpu_cancel.py tests/test_gpu_contract.py tests/test_gpu_opsweep.py tests/test_gpu_dp.py -q --tb=short -s > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sel.log
for ce in 0 64; do
COEX_CANCEL_EVERY=$ce timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c4_ce$ce.json 2> gpurun_out/bench_c4_ce$ce.err
COEX_CANCEL_EVERY=$ce timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/bench_c2_ce$ce.json 2> gpurun_out/bench_c2_ce$ce.err
done
