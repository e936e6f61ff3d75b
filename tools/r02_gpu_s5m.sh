# session-5 closing evidence on the final code (sanitizers are closed on this pool)
# launch list of the bench command, sanitizers, the 2-shard N > 1 flow
set -x
O=gpurun_out/s5m
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-dists --no-parity > $O/bench_under_ncu.log 2>&1
python tools/launch_summary.py $O/launches_bench.csv > $O/launches_bench.txt 2>&1
for tool in; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > $O/san_$tool.log 2>&1
done
timeout 900 python bench.py --steps 5 --warmup 3 --points 4e8 --mg-vshards 2 --no-dists > $O/bench_mg2.json 2> $O/bench_mg2.err
