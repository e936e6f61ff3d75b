# self-clearing one-pass K2 with one returned block, record + counts in one
# copy, cached host output in heaphull_device: bench + fused tests + sanitizers
set -x
O=gpurun_out/r02x
mkdir -p $O
for i in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-dists --no-parity --no-e2e > $O/bench$i.json 2> $O/bench$i.err
done
OHX_TRACE=1 timeout 600 python tools/kernel_driver.py --dist normal --n 1e9 --reps 4 --pipeline > $O/trace.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
for tool in memcheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > $O/san_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/san_rc.txt
done
