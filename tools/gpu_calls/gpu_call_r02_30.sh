mkdir -p gpurun_out
for pr in 0 1 2; do FPBEM_ZF_PROBE=$pr timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 2 > gpurun_out/bench_probe$pr.json 2> gpurun_out/bench_probe$pr.err; done
for pr in 0 1 2; do FPBEM_ZF_PROBE=$pr timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 2 > gpurun_out/bench_c5_probe$pr.json 2> gpurun_out/bench_c5_probe$pr.err; done
echo done
