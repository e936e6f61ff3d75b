# A/B of an environment switch on one box: bench.py device step, alternating
# runs.  usage: bash tools/ab_env.sh VAR VALUE_A VALUE_B ROUNDS OUTDIR
V=$1; A=$2; B=$3; R=${4:-3}; O=${5:-gpurun_out/ab}
mkdir -p $O
for r in $(seq 1 $R); do
  for val in $A $B; do
    env $V=$val timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-dists --no-parity --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']
print('$V=$val', round(d['ms_per_step'],4), {n: round(v['ms'],4) for n,v in k.items()})" >> $O/ab_$V.txt
  done
done
