#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_tc.py tests/test_gpu_ext.py tests/test_gpu_xformer.py tests/test_gpu_gpt2.py tests/test_gpu_dcgan.py tests/test_gpu_resnet.py tests/test_gpu_opsweep.py "tests/test_gpu_contract.py::test_full_width_gradients[c4-bf16]" "tests/test_gpu_contract.py::test_full_width_gradients[c2-bf16]" -q -x --tb=short > gpurun_out/tma_tests.log 2>&1; echo rc=$? >> gpurun_out/tma_tests.log
timeout 300 python tools/ncu_ops.py c4_qkv c4_fc1 c4_fc2 c4_head c4_dhead c4_dw768 c4_dw3072 c4_dwte conv_32x32x64 convt_16x16x128 2>&1 | sed 's/\[.*\]//' > gpurun_out/tma_shapes.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/tma_c4.json 2> gpurun_out/tma_c4.err
timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/tma_c2.json 2> gpurun_out/tma_c2.err
