#!/bin/bash
S="c4_qkv c4_fc1 c4_fc2 c4_head c4_dhead c4_dw768 c4_dw3072 c4_dwte"
for cfg in "" "COEX_DUO=0" "COEX_FORCE_BN=256" "COEX_FORCE_BN=128 COEX_DUO=0" "COEX_FORCE_BN=256 COEX_MAX_SPLIT=1"; do
  echo "== $cfg" >> gpurun_out/knobs.log
  env $cfg timeout 300 python tools/ncu_ops.py $S 2>&1 | sed 's/\[.*\]//' >> gpurun_out/knobs.log
done
