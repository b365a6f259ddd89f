mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_near_lattice.py tests/test_gpu_parity.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_e.log
for cw in 0 1; do FPBEM_CELLWISE=$cw timeout 300 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_cw$cw.json 2> gpurun_out/bench_cw$cw.err; done
echo done
