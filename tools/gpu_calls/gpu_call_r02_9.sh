mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cellwise -c 2 -o gpurun_out/cw_cfg3 python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/ncu_cwfull.log 2>&1
echo done
