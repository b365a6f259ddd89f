"""Benchmark of the periodic-FMBEM GMRES matvec hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3]

One step = one FMM operator product y = A x (near field + P2M + lattice M2L +
L2P) of a BASELINE.json configuration; the default is the largest single-GPU
single-RHS one, configs[2] = cfg3 (16^3 icosphere cells, 1,310,720 DOF,
k = 6.0). The operator is assembled once (offsets, U0, V0, M2L bank on the
host; near-field blocks on the device), and each timed batch covers exactly K
products on inputs resident in HBM (the near-field block spectrum, 1.2 GB on
cfg3, is far larger than the 126 MB L2, so every step streams it from HBM).
Timing follows the reference's protocol (src/scene.cpp:528-544): warm-up,
batches of >= 20 ms, best of 5 batches. `e2e` times the same product through
the C-ABI with pinned host buffers (host->device copy of x and device->host
copy of y inside every step), also best of 5 batches. A GMRES solve (tol 1e-6,
restart 50) is timed as the metric's second half.

--impl reference times the reference's CPU algorithm (the oracle port,
oracle/fpbem_oracle.cpp; the reference itself cannot be built here, see
DESIGN.md) on the host cores for the same workload.

With N > 1 (torchrun) the near-field (offset, target) pairs are split evenly
across the GPUs and the partial products are all-reduced over NCCL inside
every matvec: same total work, "scaling": "strong";
value = DOF / max-over-ranks time. --parallelism replicas runs independent
copies instead (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "FMBEM matvec DOF/s"
UNIT = "DOF/s"
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FP64_PEAK_FILE = ROOT / "profiles" / "r01_fp64_peak.json"
TRAFFIC_FILE = ROOT / "profiles" / "near_gemm_traffic.json"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def workload(cfg: int):
    from paper_2201_12050_b200 import Scene

    sc = Scene(cfg, 0)
    desc = {1: "cfg1: 8 spheres (icosphere s2, 320 tri) on a row, period 1.0, k=2.0",
            2: "cfg2: 4x32 closed cylinders (r 0.08, h 2.0, 1024 tri), lattice 0.22 m, k=2*pi*1000/343",
            3: "cfg3: 16^3 spheres (icosphere s2, 320 tri), period 0.5, k=6.0",
            4: "cfg4: 256 closed boxes 0.1x1.0x2.0 (3680 tri), period 1.05 m, 100 Hz",
            5: "cfg5: 32x32x4 spheres (320 tri), period 0.5, k=4.0"}[cfg]
    return sc, desc


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.sw_power_cap", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def fp64_peak():
    """FP64 tensor (DMMA) peak: MEASURED_PEAKS.json has none, so the repo's own
    microbenchmark (tools/fp64_peak.cu) result is used."""
    try:
        peaks = json.loads(PEAKS_FILE.read_text())
        if "fp64_tflops" in peaks:
            return float(peaks["fp64_tflops"]), "MEASURED_PEAKS.json fp64_tflops"
    except (OSError, ValueError):
        pass
    d = json.loads(FP64_PEAK_FILE.read_text())
    return float(d["dmma_tflops"]), "profiles/r01_fp64_peak.json (DMMA.8x8x4 microbenchmark, tools/fp64_peak.cu)"


def kernel_traffic(path):
    """DRAM bytes per launch of the dominant kernel from one committed
    `ncu --set full` capture (profiles/), or None."""
    try:
        return json.loads(path.read_text())
    except (OSError, ValueError):
        return None


def hbm_peak():
    """Measured HBM copy bandwidth (driver-written MEASURED_PEAKS.json), else the
    B200 profiling guide's fallback."""
    try:
        return float(json.loads(PEAKS_FILE.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    except (OSError, ValueError, KeyError):
        return 6500.0, "B200_PROFILING.md fallback"


class _WithNear:
    """FmmData-like view with host copies of the device-assembled near blocks."""

    def __init__(self, data, near_blocks):
        self._d = data
        self.near_blocks = near_blocks

    def __getattr__(self, name):
        return getattr(self._d, name)


def host_threads():
    """What the CPU legs ran on: nproc, OMP_NUM_THREADS and the threads OpenMP used."""
    import oracle as O

    return {"nproc": os.cpu_count(), "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
            "omp_threads": O.num_threads()}


def cpu_baseline(data, x, samples: int = 3):
    """Oracle (reference algorithm, OpenMP over target cells) on the host cores."""
    import oracle as O

    t0 = time.perf_counter()
    ora = O.OracleFmm(data)
    ora.matvec(x)  # warm-up (reference protocol: src/scene.cpp:529)
    best = float("inf")
    for _ in range(samples):
        t = time.perf_counter()
        ora.matvec(x)
        best = min(best, time.perf_counter() - t)
    th = host_threads()
    return {"value": data.N / best, "unit": UNIT, "cores": th["omp_threads"], "kind": "port", **th,
            "sample": f"{samples} single-RHS matvecs of the same operator after 1 warm-up, best of {samples} "
                      f"({best:.3f} s each; setup {time.perf_counter() - t0 - (samples + 1) * best:.1f} s)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O

    sc, desc = workload(args.config)
    t = time.perf_counter()
    data = sc.assemble_fmm(4)
    log(f"[ref] assembled {desc} in {time.perf_counter() - t:.1f} s")
    ora = O.OracleFmm(data)
    rng = np.random.default_rng(args.config)
    x = rng.uniform(-1, 1, data.N) + 1j * rng.uniform(-1, 1, data.N)
    for _ in range(args.warmup):
        ora.matvec(x)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        ora.matvec(x)
        times.append(time.perf_counter() - t)
    total = sum(times)
    value = data.N * args.steps / total
    th = host_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "complex128",
        "data": "synthetic (seeded U[-1,1] input; operator assembled from the config geometry)",
        "config": {"workload": desc, "n_dof_total": data.N, "nrhs": 1, "n_t": 4},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": th["omp_threads"], "kind": "port", **th,
                         "sample": "each step = one full single-RHS matvec of the workload on the host "
                                   "(oracle restatement of the reference; reference unbuildable here)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def timed_batches(fn, steps: int, trials: int, stream, barrier):
    """The reference's protocol (src/scene.cpp:528-544): `trials` batches of
    exactly `steps` products, each bracketed by a barrier and a device sync and
    timed with CUDA events on the launching stream; returns every batch's ms."""
    import torch

    out = []
    for _ in range(trials):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        out.append(e0.elapsed_time(e1))
    return out


def run_ours(args):
    import torch

    from paper_2201_12050_b200 import FmmOperators, gmres
    from paper_2201_12050_b200.fmm import gmres_distributed

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    sc, desc = workload(args.config)
    from paper_2201_12050_b200.fmm import assemble_near_gpu

    t = time.perf_counter()
    data = sc.assemble_fmm(4, skip_near_values=True)  # offsets, M2L bank, U0, V0 on the host
    t_host_asm = time.perf_counter() - t
    torch.cuda.synchronize(dev)
    t = time.perf_counter()
    near = assemble_near_gpu(sc, data, device=dev.index)  # near-field blocks on the GPU
    torch.cuda.synchronize(dev)
    t_dev_asm = time.perf_counter() - t
    t_asm = t_host_asm + t_dev_asm
    log(f"[rank {rank}] assembled {desc}: N={data.N} near={data.n_near} far={data.n_far} in {t_asm:.2f} s "
        f"(host {t_host_asm:.2f} s, device near blocks {t_dev_asm:.3f} s)")
    t = time.perf_counter()
    op = FmmOperators(data, device=dev.index, near_blocks=near)
    t_up = time.perf_counter() - t
    # a dedicated (non-default) stream shared by torch's events and the library's kernels
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    op.set_stream(stream.cuda_stream)
    comm = None
    slabs = False
    if world == 1 and args.slabs:  # the slab product with one rank (tests the N>1 code path on one GPU)
        op.set_slabs(None)
        slabs = True
    if world > 1 and args.parallelism in ("slabs", "pairs"):
        from paper_2201_12050_b200.fmm import Communicator

        comm = Communicator(dev.index)
        if args.parallelism == "slabs" and op.near_path()[0] == "lattice":
            # SURVEY §8e cfg3 row / north_star: whole cell planes per GPU, the lattice DFTs
            # below the slab axis on the rank's planes, one grouped NCCL all-to-all per
            # direction, the DFTs along the slab axis + the rank's share of the near-field
            # block spectrum and of Λ on its columns (strong scaling, no all-reduce of y)
            op.set_slabs(comm)
            slabs = True
        else:
            # direct near path: (offset, target) pairs split evenly across the GPUs,
            # partial products all-reduced over NCCL inside every matvec (strong scaling)
            op.set_comm(comm)

    rng = np.random.default_rng(args.config)  # the same input on every rank: the all-reduced product is A x
    xh = rng.uniform(-1, 1, data.N) + 1j * rng.uniform(-1, 1, data.N)
    x = torch.from_numpy(xh).to(dev)
    lo_r, hi_r = op.slab_rows() if slabs else (0, data.N)
    xs = x[lo_r:hi_r].contiguous()
    apply = (lambda: op.matvec_slab(xs)) if slabs else (lambda: op.matvec(x))
    warmup = max(3, args.warmup)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    from paper_2201_12050_b200 import _native

    lib = _native.cuda()
    sampler = ClockSampler(dev.index)
    with sampler:
        # ---- warm-up, then the device-resident timed batches
        for _ in range(warmup):
            apply()
        torch.cuda.synchronize(dev)
        time.sleep(0.25)  # let the sampler start
        launches0 = op.kernel_launches()
        trials_ms = timed_batches(apply, args.steps, args.trials, stream, barrier)
        launches = (op.kernel_launches() - launches0) // args.trials

        # ---- per-stage event timing (same stream); serial: the far field on the main stream
        op.enable_stage_timing(True)
        for _ in range(args.steps):
            apply()
        stages = op.stage_times()
        if not slabs:
            op.enable_stage_timing(True, serial=True)
            for _ in range(args.steps):
                apply()
        stages_serial = op.stage_times()
        op.enable_stage_timing(False)

        # ---- end-to-end through the C-ABI with pinned host buffers (this rank's rows)
        n_loc = hi_r - lo_r
        xp = torch.empty(n_loc, dtype=torch.complex128, pin_memory=True)
        xp.copy_(torch.from_numpy(xh[lo_r:hi_r]))
        yp = torch.empty(n_loc, dtype=torch.complex128, pin_memory=True)  # empty_like would not pin
        xpn, ypn = xp.numpy(), yp.numpy()

        def host_apply():
            if slabs:
                rc = lib.fpbem_cu_fmm_apply_slab(op.handle, xpn.ctypes.data, ypn.ctypes.data, 0)
            else:
                rc = lib.fpbem_cu_fmm_apply(op.handle, xpn.ctypes.data, ypn.ctypes.data, 1, 0)
            if rc:
                raise RuntimeError(lib.fpbem_cu_last_error().decode())

        host_apply()
        e2e_trials = []
        for _ in range(args.trials):
            barrier()
            t = time.perf_counter()
            for _ in range(args.steps):
                host_apply()
            e2e_trials.append(time.perf_counter() - t)
            barrier()

        # ---- GMRES solve (metric's second half); warm solve first (workspace allocation)
        b = torch.from_numpy(sc.rhs(0)).to(dev)
        solve = (lambda mi: gmres_distributed(op, b, tol=1e-6, restart=50, max_iter=mi)) if slabs else \
            (lambda mi: gmres(op, b, tol=1e-6, restart=50, max_iter=mi))
        solve(min(5, args.gmres_max_iter))
        torch.cuda.synchronize(dev)
        barrier()
        t = time.perf_counter()
        rep = solve(args.gmres_max_iter)
        torch.cuda.synchronize(dev)
        gmres_s = time.perf_counter() - t
    clocks = sampler.summary()

    # the same operator without the cell symmetries (a general mesh): the cost
    # model's path and its time per product
    nosym = None
    if world == 1 and not args.no_nosym:
        op2 = FmmOperators(data, device=dev.index, near_blocks=near, use_symmetries=False)
        op2.set_stream(stream.cuda_stream)
        for _ in range(warmup):
            op2.matvec(x)
        ms2 = min(timed_batches(lambda: op2.matvec(x), args.steps, args.trials, stream, barrier)) / args.steps
        p2 = op2.near_path()
        nosym = {"near_path": p2[0], "near_lattice": list(p2[1]), "ms_per_step": ms2, "value": data.N / (ms2 * 1e-3),
                 "note": "same operator, cell symmetries not used (one stored block per Fourier mode pair)"}
        op2.close()
        del op2

    # max over ranks
    ms = min(trials_ms)
    e2e_s = min(e2e_trials)
    vals = torch.tensor([ms, e2e_s, gmres_s], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
    ms, e2e_s, gmres_s = (float(v) for v in vals.cpu())

    path, lat_sizes, spec_bytes, modes_per_block, sym_mask, sym_dev = op.near_path()
    per = lambda st, k: st[k] / max(1, st["applies"])  # noqa: E731
    # roofline of the dominant kernel. Direct path: the near-field DMMA GEMM,
    # algorithmic flops per launch; lattice path: the per-mode block product, HBM-bound,
    # algorithmic bytes per launch = the stored block spectrum + x_hat read + y_hat written
    m = data.counts
    n_pairs = int(sum((m[0] - abs(int(o[0]))) * (m[1] - abs(int(o[1]))) * (m[2] - abs(int(o[2])))
                      for o in data.near_offsets))
    far_pairs = 0.0
    if comm is not None:  # rank 0's share of the near-field pairs (balanced against its far field)
        lo, hi, far_pairs = op.partition()
        n_pairs = hi - lo
    flops = 8.0 * data.n_dof ** 2 * float(n_pairs)
    gemm_ms = per(stages, "near_gemm")
    if path == "lattice":
        q_near = int(np.prod(lat_sizes))
        lo, hi, far_pairs = op.partition()  # stored blocks of this rank
        if slabs:  # this rank's stored blocks and the near-field modes of its columns
            si = op.slab_info()
            lo, hi, q_near = 0, si["near_blocks"], si["near_modes"]
        mode_bytes = 16.0 * data.n_dof ** 2 * (hi - lo) + 2 * 16.0 * data.n_dof * q_near
        mode_ms = per(stages, "near_mode_product")
        peak, peak_src = hbm_peak()
        traffic = kernel_traffic(ROOT / "profiles" / "near_mode_traffic.json")
        roofline = {"kernel": "near-field mode product", "bound": "hbm",
                    "achieved": mode_bytes / (mode_ms * 1e-3) / 1e9,
                    "peak": peak, "unit": "GB/s", "peak_source": peak_src, "algorithmic_bytes": mode_bytes,
                    "bytes_per_unit": f"16 n^2 per stored block ({hi - lo} blocks of n = {data.n_dof}) "
                                      f"+ 2 x 16 n per near-lattice mode ({q_near} modes)",
                    # a read-only stream can beat the read+write copy figure: also against the nominal HBM3e rate
                    "frac_of_nominal_7700": mode_bytes / (mode_ms * 1e-3) / 1e9 / 7700.0,
                    "launch_ms": mode_ms, "near_stage_ms": gemm_ms,
                    "near_stage_share_of_step": gemm_ms / per(stages, "total")}
    else:
        peak, peak_src = fp64_peak()
        traffic = kernel_traffic(TRAFFIC_FILE)
        roofline = {"kernel": "near_gemm_dmma_kernel", "bound": "tensor", "achieved": flops / (gemm_ms * 1e-3) / 1e12,
                    "peak": peak, "unit": "TFLOP/s", "peak_source": peak_src, "flops_per_launch": flops,
                    "launch_ms": gemm_ms,
                    "algorithmic_bytes": 16.0 * data.n_near * data.n_dof ** 2 + 2 * 16.0 * data.N}
    if slabs:  # the slab product's stage timing: [near_gemm] = the two exchanges, [total] = the product
        roofline.pop("near_stage_ms", None)
        roofline.pop("near_stage_share_of_step", None)
        roofline["exchange_ms"] = gemm_ms
        roofline["exchange_share_of_step"] = gemm_ms / per(stages, "total")
    roofline["frac"] = roofline["achieved"] / peak
    if traffic and traffic.get("config") != args.config:
        traffic = None  # the committed ncu capture is of another workload
    roofline["traffic"] = (traffic or {}).get("dram_bytes_per_launch")
    roofline["traffic_source"] = (traffic or {}).get("source")

    # M2L stage (pruned lattice DFTs + the Λ stream), timed alone (serial stage timing)
    fsz, paired = op.far_info()
    b = data.n_coef
    q = int(np.prod(fsz))
    n_cells = int(np.prod(data.counts))
    m2l_ms = per(stages_serial, "m2l") if not slabs else float("nan")
    lam_full = 16.0 * q * b * b
    parity = op.far_parity()
    # the flat Λ stream (single GPU, Lz > 1, <= 64 fields per mode) reads qz <= Lz/2 of half the columns
    # when the spectrum has both parities; the fused z kernel (FPBEM_M2L_Z=fused, slabs) half of Λ
    z_stream = (not slabs and fsz[2] > 1 and b <= 32 and b <= 64
                and os.environ.get("FPBEM_M2L_Z") != "fused")
    quad = z_stream and parity == 2 and os.environ.get("FPBEM_M2L_QUAD") != "0"
    lam_read = lam_full / 2 if paired else lam_full
    if quad:
        lam_read *= (fsz[2] // 2 + 1) / fsz[2]
    io = 2 * 16.0 * b * n_cells
    hbm, hbm_src = hbm_peak()
    m2l_roof = {"stage": ("M2L (x+y plane DFTs, z-DFT axis pass, flat Λ stream, inverse z pass, inverse x+y)"
                          if z_stream else "M2L (x+y plane DFTs, z-DFT/mode-product pipeline, inverse)"),
                "bound": "hbm",
                "launch_ms": m2l_ms, "peak": hbm, "unit": "GB/s", "peak_source": hbm_src,
                "lambda_paired": paired, "lambda_parity": parity, "z_form": "stream" if z_stream else "fused",
                "modes_per_streamed_block": 4 if quad else (2 if paired else 1), "fft_sizes": list(fsz),
                "compulsory_bytes": lam_read + io,
                "achieved": (lam_read + io) / (m2l_ms * 1e-3) / 1e9,
                "frac": (lam_read + io) / (m2l_ms * 1e-3) / 1e9 / hbm,
                "survey_bytes": lam_full + io,
                "frac_survey_definition": (lam_full + io) / (m2l_ms * 1e-3) / 1e9 / hbm,
                "note": "compulsory = the Λ blocks this apply reads (half of q b^2 when mirror-paired, qz <= Lz/2 "
                        "of those with the z-reflection parity) + moments in + locals out; survey = SURVEY §8d's "
                        "16 q b^2 + 2 x 16 b n_cells, the stream the reference's algorithm reads"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(_WithNear(data, near.cpu().numpy()), xh)

    strong = comm is not None
    if rank == 0:
        units = data.N if strong else world * data.N
        value = units * args.steps / (ms * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "complex128",
            "data": "synthetic (seeded U[-1,1] input; operator assembled from the config geometry)",
            "config": {
                "workload": desc, "n_dof_total": data.N, "n_dof_cell": data.n_dof, "lattice": list(data.counts),
                "near_offsets": data.n_near, "far_offsets": data.n_far, "n_t": 4, "nrhs": 1,
                "near_path": path, "near_lattice": list(lat_sizes), "near_modes_per_block": modes_per_block,
                "near_symmetries": [g for g in range(1, 8) if sym_mask >> g & 1], "near_symmetry_deviation": sym_dev,
                "parallelism": (f"slabs x{world}: whole cell planes per GPU along axis {si['axis']} (rank 0: "
                                f"{si['planes']} planes, {si['near_blocks']} stored near-field blocks, {si['far_modes']} "
                                "far modes); one grouped NCCL send/recv all-to-all per direction per product; "
                                "distributed GMRES on the slabs" if slabs else
                                f"near-field {'modes' if path == 'lattice' else 'pairs'} split over {world} GPUs "
                                f"(rank 0 {hi - lo if path == 'lattice' else n_pairs}, {far_pairs:.0f} fewer for its "
                                "far field) + NCCL all-reduce of y" if strong
                                else f"replicas x{world}" if world > 1 else "single GPU"),
                "l2": (f"inputs larger than L2: near-field block spectrum {spec_bytes / 1e9:.2f} GB streamed from HBM "
                       "every step" if path == "lattice" else
                       f"inputs larger than L2: near-field operator {16 * data.n_near * data.n_dof ** 2 / 1e9:.2f} GB "
                       "streamed from HBM every step"),
                "protocol": f"reference (src/scene.cpp:528-544): {warmup} warm-up products, {args.trials} batches "
                            f"of exactly {args.steps} products, best batch reported",
                "assembly_s": round(t_asm, 3), "assembly_host_s": round(t_host_asm, 3),
                "assembly_device_near_s": round(t_dev_asm, 3), "create_s": round(t_up, 3),
            },
            "trials_ms": trials_ms,
            "batch_ms": ms,
            "value_median": units * args.steps / (statistics.median(trials_ms) * 1e-3),
            "stages_ms": {k: (per(stages, k) if k != "applies" else v) for k, v in stages.items()},
            "stages_serial_ms": {k: (per(stages_serial, k) if k != "applies" else v)
                                 for k, v in stages_serial.items()},
            "roofline": roofline,
            "roofline_m2l": m2l_roof if not slabs else None,
            "e2e": {"value": units * args.steps / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": 16 * data.N, "d2h_bytes_per_step": 16 * data.N,
                    "trials_s": e2e_trials, "fraction_of_device_resident": (units * args.steps / e2e_s) / value},
            "gmres": {"solve_s": gmres_s, "iterations": rep.iterations, "converged": rep.converged,
                      "tol": 1e-6, "restart": 50, "max_iter": args.gmres_max_iter,
                      "final_estimate": rep.residual_history[-1] if rep.residual_history else None,
                      "ms_per_iteration": 1e3 * gmres_s / max(1, rep.iterations)},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if nosym is not None:
            line["no_symmetry"] = nosym
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if comm is not None:
        op.set_comm(None)
        comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--trials", type=int, default=5, help="timed batches of --steps products; best reported")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--gmres-max-iter", type=int, default=1000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nosym", action="store_true", help="skip the no-symmetry timing")
    ap.add_argument("--parallelism", choices=["slabs", "pairs", "replicas"], default="slabs",
                    help="N>1: cell slabs with NCCL all-to-all transposes (lattice near field; the direct path "
                         "falls back to pairs), near-field pairs (NCCL all-reduce of y) or independent replicas")
    ap.add_argument("--slabs", action="store_true", help="N=1: run the slab-distributed product with one rank")
    args = ap.parse_args()
    if args.impl == "reference":
        # bounded CPU sample: each step is a full CPU matvec
        args.steps = min(args.steps, 5)
        args.warmup = min(max(args.warmup, 1), 1)
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
