mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_epi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_epi.log
rm -f gpurun_out/epi_summary.txt
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 3 > gpurun_out/bench_epi.json 2> gpurun_out/bench_epi.err; python -c "
import json;d=json.load(open('gpurun_out/bench_epi.json'))
print(round(d['ms_per_step'],4), 'near serial', round(d['stages_serial_ms']['near_gemm'],4))" >> gpurun_out/epi_summary.txt; done
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 3 > gpurun_out/bench_c5_epi.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_c5_epi.json'))
print('c5', round(d['ms_per_step'],4))" >> gpurun_out/epi_summary.txt
echo done
