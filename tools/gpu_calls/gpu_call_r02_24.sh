mkdir -p gpurun_out
./tools/_gsp > gpurun_out/gsp.txt 2>&1
echo done
