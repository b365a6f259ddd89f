mkdir -p gpurun_out
timeout 600 python tools/time_lockstep.py 5 64 --host-apply > gpurun_out/lockstep64_ha.jsonl 2>&1
timeout 600 python tools/time_lockstep.py 5 64 --host-data > gpurun_out/lockstep64_hd.jsonl 2>&1
echo done
