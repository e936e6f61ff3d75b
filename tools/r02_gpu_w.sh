# round 2 session 3 evidence: smoke, GPU tests, both bench arms, launch
# list, ncu --set full of the fused step's kernels
set -x
O=gpurun_out/r02w
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dists --no-parity --no-e2e > $O/ncu_bench.log 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launches.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kf_filter|k2_filter|kf_gather|k1_small" -s 5 -c 5 -o $O/fused python tools/kernel_driver.py --dist normal --n 1e9 --reps 3 --pipeline > $O/ncu_full.log 2>&1
