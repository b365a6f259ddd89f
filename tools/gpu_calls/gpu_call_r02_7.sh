mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -rf -p no:cacheprovider -k "fmm_matvec or large_expansion or multi_rhs" > gpurun_out/pytest_f.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f.log
for cw in 0 1; do FPBEM_CELLWISE=$cw timeout 300 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_cw$cw.json 2> gpurun_out/bench_cw$cw.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cellwise|p2m|l2p" -c 12 --csv --log-file gpurun_out/launches_cw.csv python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/ncu_cw.log 2>&1
echo done
