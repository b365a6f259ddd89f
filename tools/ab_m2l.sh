# M2L stage A/B (serial stage timing): the flat Λ stream against the fused per-column z kernel,
# four against two modes per streamed block, and the stream's consumer warps
for c in 3 5; do
  for z in stream fused; do echo "cfg$c z=$z"; FPBEM_M2L_Z=$z FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 50 2>&1 | grep near; done
  echo "cfg$c two modes per block"; FPBEM_M2L_QUAD=0 FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 50 2>&1 | grep near
  for w in 11 9 7 5; do echo "cfg$c stream warps $w"; FPBEM_MS_WARPS=$w FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 50 2>&1 | grep near; done
done
