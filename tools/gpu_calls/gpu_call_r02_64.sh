mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_final.log
tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_final.log; tail -2 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench exit $?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference_final.json 2> gpurun_out/bench_reference_final.err; echo "ref exit $?"
rm -f gpurun_out/bench_per_config_final.jsonl
for c in 1 2 4 5; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-nosym >> gpurun_out/bench_per_config_final.jsonl 2> gpurun_out/bench_c$c.err; done
timeout 900 python tools/time_lockstep.py 5 64 > gpurun_out/lockstep_final.jsonl 2> gpurun_out/lockstep_final.err
python - <<P
import json
d=json.load(open("gpurun_out/bench_final.json"))
print(d["ms_per_step"], d["value"], d["e2e"]["value"], d["gmres"], d["roofline"]["frac"], d["roofline_m2l"]["frac_survey_definition"], d.get("no_symmetry"))
for l in open("gpurun_out/bench_per_config_final.jsonl"):
    d=json.loads(l); print(d["config"]["workload"][:30], d["ms_per_step"], d["value"], d["gmres"]["solve_s"], d["gmres"]["iterations"])
print(open("gpurun_out/lockstep_final.jsonl").read()[-600:])
P
