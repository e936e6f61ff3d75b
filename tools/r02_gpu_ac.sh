# two sub-samples: certification rate over many seeds at the sizes it would
# be used for (n >= 2^26), and the small sizes it would not
set -x
O=gpurun_out/r02ac
mkdir -p $O
OHX_SUBSAMPLES=2 timeout 900 python tools/subsample_seeds.py normal 1e9 60 >> $O/seeds.log 2>&1
OHX_SUBSAMPLES=2 timeout 900 python tools/subsample_seeds.py normal 2e8 60 >> $O/seeds.log 2>&1
OHX_SUBSAMPLES=2 timeout 900 python tools/subsample_seeds.py normal 7e7 60 >> $O/seeds.log 2>&1
OHX_SUBSAMPLES=2 timeout 900 python tools/subsample_seeds.py square 1e8 20 >> $O/seeds.log 2>&1
OHX_SUBSAMPLES=2 timeout 900 python tools/subsample_seeds.py disk 1e8 5 >> $O/seeds.log 2>&1
OHX_SUBSAMPLES=4 timeout 900 python tools/subsample_seeds.py normal 1e9 60 >> $O/seeds.log 2>&1
