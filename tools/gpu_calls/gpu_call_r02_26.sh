mkdir -p gpurun_out
timeout 300 python tools/pcie_probe.py > gpurun_out/pcie.txt 2>&1
echo done
