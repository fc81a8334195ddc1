#!/bin/bash
# ncu evidence for the C2 step (run under gpurun, one GPU).  The pass graph's conditional
# bodies are invisible to ncu, so every op of one D+G step pair is re-launched eagerly
# (tools/step_ops.py, one repetition per launch) and captured:
#   1. launch list with per-launch durations            -> gpurun_out/c2_launches.csv
#   2. dram bytes of every tcgen05 GEMM launch           -> gpurun_out/c2_gemm_dram.csv
#   3. one full capture of the largest conv GEMM         -> gpurun_out/c2_gemm_full.ncu-rep
mkdir -p gpurun_out
export STEP_OPS_REPS=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv \
  python tools/step_ops.py > gpurun_out/c2_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:k_gemm_tc --csv --log-file gpurun_out/c2_gemm_dram.csv python tools/step_ops.py > gpurun_out/c2_gemm_dram.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc -c 2 -o gpurun_out/c2_gemm_full -f \
  python tools/ncu_ops.py conv_32x32x64 > gpurun_out/c2_gemm_full.log 2>&1
