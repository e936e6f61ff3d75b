# device hull chains: tests, then the circle / disk hull stage split
set -x
O=gpurun_out/r02d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hullchain.py tests/test_mg.py -q -x > $O/pytest.log 2>&1
for dc in 1 0; do
  for dist in circle disk; do
    OHX_DEVICE_CHAIN=$dc OHX_TRACE=1 timeout 600 python tools/hull_output_probe.py --dist $dist --n 1e8 --reps 2 > $O/probe_${dist}_dc$dc.log 2>&1
  done
done
