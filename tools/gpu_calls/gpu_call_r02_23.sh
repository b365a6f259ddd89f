mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 300 python tools/debug_sim.py 3 > gpurun_out/debug_sim.log 2>&1
timeout 300 python tools/debug_sim.py 3 --stream > gpurun_out/debug_sim_stream.log 2>&1
FPBEM_SLAB_GRAPH=0 timeout 300 python tools/debug_sim.py 3 --stream > gpurun_out/debug_sim_nograph.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_near_lattice.py tests/test_gpu_parity.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_dft.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dft.log
timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_dft.json 2> gpurun_out/bench_dft.err
echo done
