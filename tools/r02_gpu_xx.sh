# sanitizers over the in-place device hull and the pipelined pinned output
set -x
O=gpurun_out/r02xx
mkdir -p $O
for tool in memcheck initcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > $O/san_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/san_rc.txt
done
