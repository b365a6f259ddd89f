mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_final.log
tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_final.log; tail -2 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench exit $?"
python - <<P
import json
d=json.load(open("gpurun_out/bench_final.json"))
print(d["ms_per_step"], d["value"], d["e2e"]["value"], d["gmres"]["solve_s"], d["roofline"]["frac"], d["roofline_m2l"]["frac_survey_definition"], d["gpu_launches"], d["clocks"])
P
