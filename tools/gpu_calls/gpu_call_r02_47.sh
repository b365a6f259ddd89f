mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_cw.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cw.log
rm -f gpurun_out/cw_summary.txt
for v in 0 1 0 1; do FPBEM_CELLWISE_V1=$v timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 3 > gpurun_out/bench_cw$v.json 2> gpurun_out/bench_cw$v.err; python -c "
import json;d=json.load(open('gpurun_out/bench_cw$v.json'))
print($v, round(d['ms_per_step'],4), 'p2m serial', round(d['stages_serial_ms']['p2m'],4))" >> gpurun_out/cw_summary.txt; done
FPBEM_CELLWISE_V1=0 timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 3 > gpurun_out/bench_c5_cw.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_c5_cw.json'))
print('c5', round(d['ms_per_step'],4), 'p2m serial', round(d['stages_serial_ms']['p2m'],4))" >> gpurun_out/cw_summary.txt
echo done
