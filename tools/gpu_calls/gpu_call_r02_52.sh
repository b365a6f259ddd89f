mkdir -p gpurun_out
export FPBEM_M2L_Z=stream FPBEM_SERIAL=1
for q in 1 0; do for pr in 0 1 3 8; do
echo "quad $q probe $pr"; FPBEM_M2L_QUAD=$q FPBEM_MS_PROBE=$pr timeout 90 python tools/profile_matvec.py --config 3 --applies 50 2>&1 | tail -2 | head -1 | cut -c1-200
done; done
