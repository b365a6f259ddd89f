mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python tools/bench_configs.py --configs 5 --out gpurun_out/configs_r02_c5.jsonl > gpurun_out/configs_r02_c5.log 2>&1; echo "rc=$?" >> gpurun_out/configs_r02_c5.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_gmres.csv python tools/profile_gmres.py --config 3 --iters 30 > gpurun_out/ncu_gmres.log 2>&1
timeout 300 python tools/profile_gmres.py --config 3 --iters 100 > gpurun_out/prof_gmres.txt 2>&1
echo done
