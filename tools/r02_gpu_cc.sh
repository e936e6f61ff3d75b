# candidate K1 grid: points per thread 16 / 32 / 64 (step time A/B)
set -x
O=gpurun_out/r02cc
mkdir -p $O
for per in 16 32 64 16 32 64; do
  OHX_K1LIST_PER=$per timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-dists --no-parity --no-e2e > $O/bench_$per.json 2>> $O/bench.err
  python3 -c "import json;d=json.loads(open('$O/bench_$per.json').read().strip().splitlines()[-1]);print($per, d['ms_per_step'], d['roofline']['kernels']['candidate_stage']['ms'])" >> $O/summary.txt
done
