# M2L stage A/B: per-axis DFT passes vs x+y plane kernels (serial stage timing), DESIGN.md §3.3
for c in 3 5; do
  for xy in 1 0 2; do echo "cfg$c xy$xy"; FPBEM_M2L_XY=$xy FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 30 2>&1 | grep near; done
done
