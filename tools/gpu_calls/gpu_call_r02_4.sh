mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_near_lattice.py tests/test_gpu_parity.py tests/test_gpu_dist_gmres.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c.log
for nw in 8 10 20; do FPBEM_MMA_NW=$nw timeout 300 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_nw$nw.json 2> gpurun_out/bench_nw$nw.err; done
timeout 300 python tools/profile_gmres.py --config 3 --iters 100 > gpurun_out/prof_gmres2.txt 2>&1
echo done
