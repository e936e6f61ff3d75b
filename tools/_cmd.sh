B="python bench.py --no-e2e --no-cpu --no-dists --no-parity --steps 20 --warmup 5"
for cfg in "OHX_KF_CAP_XY=0" "" "OHX_KF_CAP_XY=0" "" "OHX_KF_CAP_XY=4096"; do
  echo "== $cfg"; env $cfg $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['ms'],4) for k,v in r['kernels'].items()}, r.get('candidates'))"
done > gpurun_out/capxy_sweep.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_capxy.csv python bench.py --no-e2e --no-cpu --no-dists --no-parity --steps 2 --warmup 1 > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
