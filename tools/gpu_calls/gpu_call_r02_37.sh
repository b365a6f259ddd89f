mkdir -p gpurun_out
timeout 600 python tools/time_lockstep.py 5 64 --torch-stream > gpurun_out/lockstep64_ts.jsonl 2>&1
timeout 600 python tools/time_lockstep.py 5 64 --timed-applies > gpurun_out/lockstep64_ta.jsonl 2>&1
echo done
