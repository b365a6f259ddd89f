mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_near_lattice.py tests/test_gpu_parity.py -m gpu -q -x -rf -p no:cacheprovider -k "pipelined or full_size or fmm_matvec" > gpurun_out/pytest_pipe.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pipe.log
timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err
FPBEM_PIPE_H2D=0 timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_nopipe.json 2> gpurun_out/bench_nopipe.err
echo done
