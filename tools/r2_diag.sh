#!/bin/bash
# diagnostics: C2 bf16 per-op sweep at full width, grad-probe per tensor, full gpu suite (no -x)
mkdir -p gpurun_out
timeout 600 python tools/op_sweep.py --workload c2 --precision bf16 --batch 8 --out gpurun_out/sweep_c2_bf16.json > gpurun_out/sweep_c2_bf16.txt 2>&1
timeout 600 python tools/contract_probe.py --case c2 --precision bf16 --mode imperative > gpurun_out/probe_c2_bf16_imp.txt 2>&1
rm -f gpurun_out/contract.jsonl
CONTRACT_REPORT=gpurun_out/contract.jsonl timeout 2400 python -m pytest tests -m gpu -q --tb=line > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_all.log
