#!/bin/bash
# round-2 evidence (one GPU): C4 eager step-op launch list with DRAM bytes, full captures of the
# C4 GEMMs and flash-attention kernels, the in-graph device-stamp step profile
mkdir -p gpurun_out/r2prof
export STEP_OPS_REPS=1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2prof/c4_launches.csv python tools/step_ops.py --workload c4 --precision bf16 > gpurun_out/r2prof/c4_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc -s 2 -c 2 -o gpurun_out/r2prof/c4_gemm_fc2_head -f \
  python tools/ncu_ops.py c4_fc2 c4_head > gpurun_out/r2prof/c4_gemm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fa_ -c 5 -o gpurun_out/r2prof/c4_flash -f \
  python tools/fa_bench.py 96 1024 1 > gpurun_out/r2prof/c4_flash.log 2>&1
timeout 600 python tools/profile_step.py --workload c4 --precision bf16 --steps 6 > gpurun_out/r2prof/c4_step_profile.txt 2>&1
