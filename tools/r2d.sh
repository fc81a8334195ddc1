mkdir -p gpurun_out
( for w in "c3 fp32 imperative" "c3 fp32 coexec" "c2 bf16 imperative" "c2 bf16 coexec" "c4 fp32 coexec" "c4 bf16 imperative" "c5 fp32 coexec"; do
  set -- $w
  timeout 900 python tools/contract_probe.py --case $1 --precision $2 --mode $3 2>&1 | tail -4
done ) > gpurun_out/probe.txt 2>&1
timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_g.json 2> gpurun_out/bench_c4_g.err
