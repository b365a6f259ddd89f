mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_near_lattice.py tests/test_gpu_parity.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_g.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g.log
for f in 0 1; do FPBEM_FUSE_L2P=$f timeout 300 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_f$f.json 2> gpurun_out/bench_f$f.err; done
FPBEM_FUSE_L2P=1 timeout 300 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_f1b.json 2> gpurun_out/bench_f1b.err
echo done
