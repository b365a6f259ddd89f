mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python tools/model_rhs_shard.py > gpurun_out/model_cfg5_rhs.jsonl 2> gpurun_out/model_cfg5_rhs.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dft_axis_dmma_kernel|m2l_zpipe" -s 40 -c 3 -o gpurun_out/dft_cfg3 python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/ncu_dft.log 2>&1
echo done
