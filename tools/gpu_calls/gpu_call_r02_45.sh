mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_near_lattice.py -m gpu -q -x -k "full_size or pipelined or orbits or tensor_core" -p no:cacheprovider > gpurun_out/pytest_xb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_xb.log
FPBEM_MMA_XBUF=1 timeout 600 python -m pytest tests/test_gpu_near_lattice.py -m gpu -q -x -k "full_size or pipelined or orbits or tensor_core" -p no:cacheprovider >> gpurun_out/pytest_xb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_xb.log
for xb in 2 1 2 1; do FPBEM_MMA_XBUF=$xb timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/bench_xb$xb.json 2> gpurun_out/bench_xb$xb.err; python -c "
import json;d=json.load(open('gpurun_out/bench_xb$xb.json'))
print($xb, round(d['ms_per_step'],4), round(d['stages_ms']['near_mode_product'],4))" >> gpurun_out/xb_summary.txt; done
FPBEM_MMA_XBUF=1 timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/bench_c5_xb1.json 2> gpurun_out/bench_c5_xb1.err
echo done
