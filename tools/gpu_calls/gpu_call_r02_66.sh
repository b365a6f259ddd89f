mkdir -p gpurun_out
CMD="python tools/profile_matvec.py --config 3 --applies 3"
timeout 300 $CMD > gpurun_out/plain_pm.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "far field (P2M + M2L)/" -s 6 -c 6 -o gpurun_out/far_chain_cfg3 $CMD > gpurun_out/ncu_far.log 2>&1
tail -3 gpurun_out/ncu_far.log; ls -la gpurun_out/far_chain_cfg3.ncu-rep
