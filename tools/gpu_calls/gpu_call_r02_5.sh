mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 600 python -m pytest tests/test_gpu_near_lattice.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_d.log
for kc in 4 8 16; do for nw in 8 10; do FPBEM_MMA_KC=$kc FPBEM_MMA_NW=$nw timeout 300 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_kc${kc}_nw$nw.json 2> gpurun_out/bench_kc${kc}_nw$nw.err; done; done
echo done
