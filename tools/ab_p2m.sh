# P2M A/B at one right-hand side: FMA kernel vs the V0^T-resident DMMA GEMM (serial stage timing)
for c in 2 3 5; do
  for g in 1 2; do echo "cfg$c p2m$g"; FPBEM_P2M_GEMM=$g FPBEM_SERIAL=1 python tools/profile_matvec.py --config $c --applies 30 2>&1 | grep near; done
done
