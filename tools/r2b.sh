mkdir -p gpurun_out
rm -f gpurun_out/contract.jsonl
CONTRACT_REPORT=gpurun_out/contract.jsonl timeout 2400 python -m pytest tests/test_gpu_contract.py -q --tb=short > gpurun_out/contract.log 2>&1 || true
