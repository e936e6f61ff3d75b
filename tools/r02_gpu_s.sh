# certification rate of the provisional region over 20 seeds per size:
# one whole-sample octagon (subs=1) vs intersections (subs=2, 4)
set -x
O=gpurun_out/r02s
mkdir -p $O
for s in 1 2 4; do
  OHX_SUBSAMPLES=$s timeout 900 python tools/subsample_seeds.py normal 1e9 20 >> $O/seeds.log 2>&1
done
for s in 1 2 4; do
  OHX_SUBSAMPLES=$s timeout 900 python tools/subsample_seeds.py normal 3e8 20 >> $O/seeds.log 2>&1
  OHX_SUBSAMPLES=$s timeout 900 python tools/subsample_seeds.py normal 1e8 20 >> $O/seeds.log 2>&1
  OHX_SUBSAMPLES=$s timeout 900 python tools/subsample_seeds.py square 1e8 10 >> $O/seeds.log 2>&1
done
