#!/bin/bash
mkdir -p gpurun_out
export COEX_CANCEL_EVERY=0
timeout 900 ncu --kernel-name regex:k_fa_ -c 4 --set full --import-source on -o gpurun_out/fa_full -f python tools/fa_probe.py > gpurun_out/ncu_fa.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_fa.log
