mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s4.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_s4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_s4.log
timeout 900 python bench.py > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err
tail -3 gpurun_out/pytest_gpu_s4.log; tail -2 gpurun_out/smoke_s4.log; cat gpurun_out/bench_s4.json | cut -c1-600
