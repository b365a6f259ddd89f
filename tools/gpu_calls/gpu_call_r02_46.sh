mkdir -p gpurun_out
rm -f gpurun_out/align_summary.txt
for w in 0 4 8 12 0 8; do FPBEM_ZF_ALIGN=$w timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 3 > gpurun_out/bench_al$w.json 2> gpurun_out/bench_al$w.err; python -c "
import json;d=json.load(open('gpurun_out/bench_al$w.json'))
print($w, round(d['ms_per_step'],4), 'm2l serial', round(d['stages_serial_ms']['m2l'],4))" >> gpurun_out/align_summary.txt; done
for w in 0 8; do FPBEM_ZF_ALIGN=$w timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 5 --trials 3 > gpurun_out/bench_c5_al$w.json 2> gpurun_out/bench_c5_al$w.err; python -c "
import json;d=json.load(open('gpurun_out/bench_c5_al$w.json'))
print('c5', $w, round(d['ms_per_step'],4), 'm2l serial', round(d['stages_serial_ms']['m2l'],4))" >> gpurun_out/align_summary.txt; done
FPBEM_ZF_ALIGN=8 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "circulant or full_size or fmm_matvec" -p no:cacheprovider > gpurun_out/pytest_align.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_align.log
echo done
