# provisional-region sample shape: one whole-sample octagon vs intersections
# of sub-sample octagons (candidates, certification, step time)
set -x
O=gpurun_out/r02r
mkdir -p $O
for cfg in "4 512" "2 512" "1 512" "1 256" "1 1024" "2 1024"; do
  set -- $cfg
  OHX_SUBSAMPLES=$1 OHX_SAMPLE_SEGS=$2 timeout 900 python tools/sample_config_sweep.py >> $O/sweep.log 2>&1
done
