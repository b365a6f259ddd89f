# fused MGS: elements per block before more SMs are used (GMRES per-iteration time, cfg2 N = 131072)
for pb in 1024 512 1024 512; do echo "per_block $pb"; FPBEM_MGS_PER_BLOCK=$pb python tools/profile_gmres.py --config 2 --iters 200; done
