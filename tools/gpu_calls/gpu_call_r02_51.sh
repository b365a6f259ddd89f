mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_zsym.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_zsym.log
rm -f gpurun_out/zsym_summary.txt
for v in 1 0 1 0; do FPBEM_ZF_ZSYM=$v timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 3 > gpurun_out/bench_zs$v.json 2> gpurun_out/bench_zs$v.err; python -c "
import json;d=json.load(open('gpurun_out/bench_zs$v.json'))
print($v, round(d['ms_per_step'],4), 'm2l serial', round(d['stages_serial_ms']['m2l'],4))" >> gpurun_out/zsym_summary.txt; done
for v in 1 0; do FPBEM_ZF_ZSYM=$v timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 3 > gpurun_out/bench_c5_zs$v.json 2> gpurun_out/bench_c5_zs$v.err; python -c "
import json;d=json.load(open('gpurun_out/bench_c5_zs$v.json'))
print('c5', $v, round(d['ms_per_step'],4), 'm2l serial', round(d['stages_serial_ms']['m2l'],4))" >> gpurun_out/zsym_summary.txt; done
echo done
