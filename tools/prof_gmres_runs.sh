# GMRES per-iteration cost vs the matvec (tools/profile_gmres.py), DESIGN.md §7
python tools/profile_gmres.py --config 2 --iters 200
python tools/profile_gmres.py --config 3 --iters 100
python tools/profile_gmres.py --config 5 --nrhs 64 --iters 60
