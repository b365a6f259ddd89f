mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 300 python tools/debug_sim.py > gpurun_out/debug_sim.log 2>&1
FPBEM_SLAB_GRAPH=0 timeout 300 python tools/debug_sim.py > gpurun_out/debug_sim_nograph.log 2>&1
timeout 600 python tools/model_scaling.py --config 3 --no-gmres > gpurun_out/model_cfg3.jsonl 2> gpurun_out/model_cfg3.err
echo done
