# lattice DFT passes + M2L (serial stage timing)
for c in 2 3 5; do
  echo "cfg$c"; FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 30 2>&1 | grep near
done
echo "cfg5x64"; python tools/profile_matvec.py --config 5 --nrhs 64 --applies 5 2>&1 | grep near
