mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_xyt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_xyt.log
rm -f gpurun_out/xyt_summary.txt
for v in 1 0 1 0; do FPBEM_NEAR_XYT=$v timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 3 > gpurun_out/bench_xyt$v.json 2> gpurun_out/bench_xyt$v.err; python -c "
import json;d=json.load(open('gpurun_out/bench_xyt$v.json'))
print($v, round(d['ms_per_step'],4), 'near serial', round(d['stages_serial_ms']['near_gemm'],4), 'e2e %.4g' % d['e2e']['value'])" >> gpurun_out/xyt_summary.txt; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"xy_tile|dft_axis" -c 20 --csv --log-file gpurun_out/launches_xyt.csv python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/ncu_xyt.log 2>&1
echo done
