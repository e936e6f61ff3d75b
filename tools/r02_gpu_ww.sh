# round 2 session 3, final evidence: smoke, all GPU tests, both bench arms,
# launch lists (normal step, circle), sanitizers
set -x
O=gpurun_out/r02ww
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dists --no-parity --no-e2e > $O/ncu_bench.log 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launches.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_circle.csv python tools/kernel_driver.py --dist circle --n 1e8 --reps 2 --pipeline > $O/ncu_circle.log 2>&1
python tools/launch_summary.py $O/launches_circle.csv > $O/launches_circle.txt 2>&1
for tool in memcheck initcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > $O/san_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/san_rc.txt
done
