#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/ncu_ops.py c4_qkv c4_fc1 c4_fc2 c4_head c4_dhead c4_dw768 c4_dw3072 c4_dwte 2>&1 | sed 's/\[.*\]//' > gpurun_out/b2_shapes.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b2_c4.json 2> gpurun_out/b2_c4.err
timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/b2_c2.json 2> gpurun_out/b2_c2.err
COEX_DUO_PENALTY=1.0 COEX_BN256_BIAS=1.0 timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/b2_c2_old.json 2> gpurun_out/b2_c2_old.err
