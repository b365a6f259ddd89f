# lattice near field: x+y plane kernel vs per-axis DFT passes (serial stage timing), two repetitions
for rep in 1 2; do
for c in 2 3 5; do
  echo "cfg$c xy"; FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 30 2>&1 | grep near
  echo "cfg$c axis"; FPBEM_NEAR_XY=0 FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 30 2>&1 | grep near
done
done
