#!/bin/bash
# GEMM issue-path check: tcgen05 GEMM tests, flash tests, C4 GEMM shapes, C4 bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_flash.py tests/test_gpu_ext.py -q -x --tb=short > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
timeout 300 python tools/ncu_ops.py c4_qkv c4_fc1 c4_fc2 c4_head c4_dhead c4_dw768 c4_dw3072 c4_dwte > gpurun_out/g_shapes.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
