# round 2, first GPU pass: smoke, GPU tests, bench (new legs), sanitizers
set -x
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
free -g > $O/free.txt; nproc >> $O/free.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
for tool in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > $O/san_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/san_rc.txt
done
