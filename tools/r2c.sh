mkdir -p gpurun_out
for w in "c3 fp32 2" "c3 bf16 2" "c2 bf16 8" "c2 fp32 8" "c4 fp32 2" "c4 bf16 2"; do
  set -- $w
  timeout 900 python tools/op_sweep.py --workload $1 --precision $2 --batch $3 --out gpurun_out/sweep_$1_$2.json > gpurun_out/sweep_$1_$2.txt 2>&1
done
