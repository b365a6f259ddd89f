mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py tests/test_gpu_cpp_driver.py tests/test_gpu_dist_gmres.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_tg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tg.log
timeout 900 python -m pytest tests/test_gpu_config_scale.py -m gpu -q -x -p no:cacheprovider -k "4-" > gpurun_out/pytest_tg_c4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tg_c4.log
rm -f gpurun_out/tg_summary.txt
for v in 1 0; do for c in 4 1; do FPBEM_NEAR_TGEMM=$v timeout 600 python bench.py --config $c --no-cpu-baseline --no-nosym --gmres-max-iter 300 --trials 3 > gpurun_out/bench_tg${v}_c$c.json 2> gpurun_out/bench_tg${v}_c$c.err; python -c "
import json;d=json.load(open('gpurun_out/bench_tg${v}_c$c.json'))
print('tgemm=$v cfg$c', round(d['ms_per_step'],4), 'gmres', d['gmres']['iterations'], round(d['gmres']['solve_s'],4), 'e2e %.4g' % d['e2e']['value'])" >> gpurun_out/tg_summary.txt; done; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"near_tgemm|near_gemm|near_reduce" -s 2 -c 4 --csv --log-file gpurun_out/ncu_tg_c4.csv python bench.py --config 4 --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/ncu_tg.log 2>&1
echo done
