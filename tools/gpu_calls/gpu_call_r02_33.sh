mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1500 python -m pytest tests -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 900 python tools/model_rhs_shard.py > gpurun_out/model_cfg5_rhs.jsonl 2> gpurun_out/model_cfg5_rhs.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo done
