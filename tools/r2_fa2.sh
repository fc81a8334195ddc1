#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_flash.py -q -s --tb=short -k kernels > gpurun_out/fa2_test.log 2>&1; echo "rc=$?" >> gpurun_out/fa2_test.log
timeout 120 python tools/fa_bench.py > gpurun_out/fa2_bench.log 2>&1
timeout 300 python -m pytest tests/test_gpu_flash.py -q -s --tb=short -k gradients >> gpurun_out/fa2_test.log 2>&1; echo "rc=$?" >> gpurun_out/fa2_test.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fa_ -c 4 -o gpurun_out/fa2 -f python tools/fa_bench.py 96 1024 1 > gpurun_out/fa2_ncu.log 2>&1
