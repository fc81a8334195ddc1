#!/bin/bash
# round-2 profile pass: flash kernel tests, smoke, flash timing + ncu, C4 GEMM shapes timing + ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_flash.py -q -s --tb=short > gpurun_out/p1_flash.log 2>&1; echo "rc=$?" >> gpurun_out/p1_flash.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/p1_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/p1_smoke.log
timeout 300 python tools/fa_bench.py > gpurun_out/p1_fa_bench.log 2>&1
timeout 300 python tools/ncu_ops.py c4_qkv c4_fc1 c4_fc2 c4_head c4_dhead c4_dw768 c4_dw3072 c4_dwte > gpurun_out/p1_gemm_shapes.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fa_ -c 4 -o gpurun_out/p1_fa -f python tools/fa_bench.py 96 1024 1 > gpurun_out/p1_ncu_fa.log 2>&1; echo "rc=$?" >> gpurun_out/p1_ncu_fa.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 2 -o gpurun_out/p1_gemm_fc1 -f python tools/ncu_ops.py c4_fc1 > gpurun_out/p1_ncu_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/p1_ncu_gemm.log
