# sample kernel zeroes the coverage counter; one-call stage folds; host
# sweep sort on range-normalised keys: bench (+distributions), traces, tests
set -x
O=gpurun_out/r02z
mkdir -p $O
timeout 1200 python bench.py --no-cpu --no-parity > $O/bench.json 2> $O/bench.err
OHX_TRACE=2 timeout 600 python tools/kernel_driver.py --dist square --n 1e8 --reps 5 --pipeline > $O/trace_square.log 2>&1
OHX_TRACE=2 timeout 600 python tools/kernel_driver.py --dist normal --n 1e9 --reps 5 --pipeline > $O/trace_normal.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
