set -x
O=gpurun_out/r02l
mkdir -p $O
for v in 0 1; do
OHX_D2H_REGISTER=$v OHX_TRACE=1 timeout 600 python tools/hull_output_probe.py --dist circle --n 1e8 --reps 2 > $O/probe_circle_reg$v.log 2>&1
done
timeout 900 python tools/h2d_probe.py 1e9 > $O/h2d.log 2>&1
