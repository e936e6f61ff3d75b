set -x
O=gpurun_out/r02tt
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_hullchain.py -q -x -k "rotated" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
