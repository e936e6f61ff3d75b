# provisional-region sample size sweep (runs of 8192 points; 4 sub-samples), normal 1e9, 20 seeds
set -x
O=gpurun_out/r02ak
mkdir -p $O
for segs in 512 256 384 768 1024 512; do
  OHX_SAMPLE_SEGS=$segs timeout 300 python tools/subsample_seeds.py normal 1e9 20 >> $O/segs.log 2>&1
done
OHX_SAMPLE_SEGS=256 OHX_SAMPLE_RPB=1 timeout 300 python tools/subsample_seeds.py normal 1e9 20 >> $O/segs.log 2>&1
