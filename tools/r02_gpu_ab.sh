# final full-size parity sweep over seeds on the round's code
set -x
O=gpurun_out/r02ab
mkdir -p $O
timeout 1500 python tools/sweep_full.py 10 normal:1e9,square:1e8 > $O/sweep_normal_square.log 2>&1
timeout 1500 python tools/sweep_full.py 5 circle:1e8 > $O/sweep_circle.log 2>&1
