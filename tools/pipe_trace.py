"""Timeline of the pipelined host-pointer product (FPBEM_PIPE_TRACE=1 prints it per product on stderr).

    FPBEM_PIPE_TRACE=1 python tools/pipe_trace.py [config] [products]
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from bench import workload
    from paper_2201_12050_b200 import FmmOperators
    from paper_2201_12050_b200.fmm import assemble_near_gpu

    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    sc, _ = workload(cfg)
    data = sc.assemble_fmm(4, skip_near_values=True)
    near = assemble_near_gpu(sc, data, device=0)
    op = FmmOperators(data, device=0, near_blocks=near)
    rng = np.random.default_rng(cfg)
    x = torch.from_numpy(rng.uniform(-1, 1, data.N) + 1j * rng.uniform(-1, 1, data.N)).pin_memory()
    y = torch.empty_like(x).pin_memory()
    from paper_2201_12050_b200 import _native

    lib = _native.cuda()
    xn, yn = x.numpy(), y.numpy()

    def host_apply():  # the C-ABI call of bench.py's e2e leg
        if lib.fpbem_cu_fmm_apply(op.handle, xn.ctypes.data, yn.ctypes.data, 1, 0):
            raise RuntimeError(lib.fpbem_cu_last_error().decode())

    # the same pinned buffers through plain copies (what the PCIe link gives them)
    xd = torch.empty(data.N, dtype=torch.complex128, device="cuda")
    for name, fn in (("h2d", lambda: xd.copy_(x, non_blocking=True)), ("d2h", lambda: y.copy_(xd, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"plain {name} of the same buffers: {ms:.3f} ms = {16 * data.N / ms / 1e6:.1f} GB/s")
    for _ in range(3):
        host_apply()
    t = time.perf_counter()
    for _ in range(reps):
        host_apply()
    dt = (time.perf_counter() - t) / reps
    print(f"cfg{cfg}: {dt * 1e3:.3f} ms per host-pointer product, {data.N / dt:.3e} DOF/s")


if __name__ == "__main__":
    main()
