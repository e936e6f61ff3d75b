set -x
O=gpurun_out/r02qq
mkdir -p $O
nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" > $O/pcie.txt 2>&1
timeout 600 python tools/h2d_streams_probe.py 1e9 > $O/h2d_streams.log 2>&1
