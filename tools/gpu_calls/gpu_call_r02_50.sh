mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "m2l_z_forms or flat_stream or fmm_matvec_matches" 2>&1 | tail -5
for mode in "fused 1" "stream 0" "stream 1"; do set -- $mode
  for cfg in 3 5; do
    FPBEM_M2L_Z=$1 FPBEM_M2L_QUAD=$2 timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-nosym > gpurun_out/bench_z_$1$2_$cfg.json 2> gpurun_out/bench_z_$1$2_$cfg.err
    python - <<P
import json
d=json.load(open("gpurun_out/bench_z_$1$2_$cfg.json"))
print("$1 quad$2 cfg$cfg", round(d["ms_per_step"],4), "serial m2l", round(d["stages_serial_ms"]["m2l"],4), "gmres", d["gmres"]["solve_s"], d["gmres"]["iterations"], d.get("roofline_m2l",{}).get("frac_survey_definition"))
P
  done
done
