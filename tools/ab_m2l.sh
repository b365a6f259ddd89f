# M2L stage A/B: fields per CTA of the x+y plane kernels (serial stage timing), DESIGN.md §3.3
for c in 2 3; do
  for fb in 4 1 2 8; do echo "cfg$c fb$fb"; FPBEM_XY_FIELDS=$fb FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 30 2>&1 | grep near; done
done
