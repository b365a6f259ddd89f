# A/B of the lattice DFT passes and the L2P (serial stage timing), DESIGN.md §3.1b
for c in 2 3 5; do
  echo "cfg$c dmma"; FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 20 2>&1 | grep near
  echo "cfg$c fma"; FPBEM_DFT=fma FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 20 2>&1 | grep near
done
echo "cfg5x64 dmma"; python tools/profile_matvec.py --config 5 --nrhs 64 --applies 5 2>&1 | grep near
FPBEM_SERIAL=1 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/ncu_cfg3d.csv python tools/profile_matvec.py --config 3 --applies 2 > /dev/null 2>&1
