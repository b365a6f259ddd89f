mkdir -p gpurun_out
rm -f gpurun_out/cw_summary.txt
for v in 0 0; do FPBEM_CELLWISE_V1=$v timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 3 > gpurun_out/bench_cw$v.json 2> gpurun_out/bench_cw$v.err; python -c "
import json;d=json.load(open('gpurun_out/bench_cw$v.json'))
print($v, round(d['ms_per_step'],4), 'p2m serial', round(d['stages_serial_ms']['p2m'],4))" >> gpurun_out/cw_summary.txt; done
echo done
