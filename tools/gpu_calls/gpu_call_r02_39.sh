mkdir -p gpurun_out
timeout 600 python tools/time_lockstep.py 5 64 --oracle > gpurun_out/lockstep64_or.jsonl 2>&1
OMP_WAIT_POLICY=PASSIVE timeout 600 python tools/time_lockstep.py 5 64 --oracle > gpurun_out/lockstep64_or2.jsonl 2>&1
echo done
