mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s4b.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_s4b.log
tail -4 gpurun_out/pytest_gpu_s4b.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_s4b.json 2> gpurun_out/bench_s4b.err
python - <<P
import json
d=json.load(open("gpurun_out/bench_s4b.json"))
print(d["ms_per_step"], d["value"], d["e2e"]["value"], d["gmres"], d["roofline_m2l"])
P
