# per-mode product of the lattice near field (serial stage timing)
for c in 2 3 5; do
  echo "cfg$c"; FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 20 2>&1 | grep near
done
