mkdir -p gpurun_out
timeout 2700 python tools/bench_configs.py --sweep --out gpurun_out/configs_r02_final.jsonl > gpurun_out/configs_r02_final.log 2>&1; echo "rc=$?" >> gpurun_out/configs_r02_final.log
tail -3 gpurun_out/configs_r02_final.log
python - <<P
import json
for l in open("gpurun_out/configs_r02_final.jsonl"):
    d=json.loads(l)
    print({k:d[k] for k in ("config","matvec_ms","matvec_rel_err","batched_nrhs","gmres","iterations","solve_s","total_solve_s","iterations_min_max","solution_rel_err","parity_solution_rel_err") if k in d})
P
