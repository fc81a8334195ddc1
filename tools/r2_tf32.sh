#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_tc.py -q --tb=short > gpurun_out/tf32_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tf32_tests.log
PREC=fp32 timeout 300 python tools/ncu_ops.py c4_qkv c4_fc1 c4_fc2 gemm_8192 > gpurun_out/tf32_shapes.log 2>&1
