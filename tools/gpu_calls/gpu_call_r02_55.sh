mkdir -p gpurun_out
rm -f gpurun_out/slabxy.txt
for xy in 1 0; do FPBEM_SLAB_XY=$xy timeout 900 python tools/model_scaling.py --config 3 --no-gmres > gpurun_out/model_xy$xy.jsonl 2>/dev/null; grep summary gpurun_out/model_xy$xy.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); s=d['summary']; print('xy=$xy', d['P'], round(s['max_rank_apply_ms'],4))" >> gpurun_out/slabxy.txt; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p2r0.csv python tools/model_scaling.py --config 3 --only 2,0 --no-gmres --steps 3 > gpurun_out/ncu_p2.log 2>&1
echo done
