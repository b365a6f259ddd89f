mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "m2l_z_forms or flat_stream or circulant_m2l" > gpurun_out/pytest_stream.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_stream.log
tail -5 gpurun_out/pytest_stream.log
for mode in fused stream; do
  for cfg in 3 5; do
    FPBEM_M2L_Z=$mode timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-nosym > gpurun_out/bench_z_${mode}_$cfg.json 2> gpurun_out/bench_z_${mode}_$cfg.err
    python - <<P
import json
d=json.load(open("gpurun_out/bench_z_${mode}_$cfg.json"))
print("$mode cfg$cfg", d["ms_per_step"], d["stages_serial_ms"], d["stages_ms"], d.get("roofline_m2l",{}).get("frac_survey_definition"))
P
  done
done
