mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py tests/test_gpu_slabs.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_zmma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_zmma.log
timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_zmma.json 2> gpurun_out/bench_zmma.err
FPBEM_ZF_DFT=fma timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_zfma.json 2> gpurun_out/bench_zfma.err
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_c5_zmma.json 2> gpurun_out/bench_c5_zmma.err
FPBEM_ZF_DFT=fma timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_c5_zfma.json 2> gpurun_out/bench_c5_zfma.err
echo done
