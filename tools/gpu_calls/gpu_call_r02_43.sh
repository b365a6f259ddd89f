mkdir -p gpurun_out
timeout 300 python tools/profile_gmres.py --config 3 --iters 100 > gpurun_out/prof_gmres_ab.txt 2>&1
FPBEM_MGS_FLAGBAR=1 timeout 300 python tools/profile_gmres.py --config 3 --iters 100 >> gpurun_out/prof_gmres_ab.txt 2>&1
timeout 300 python tools/profile_gmres.py --config 3 --iters 100 >> gpurun_out/prof_gmres_ab.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-nosym > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err
echo done
