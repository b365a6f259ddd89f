"""Host<->device copy rates on the box (pinned, 21 MB = one cfg3 vector): H2D alone, D2H alone, both at once."""
import time

import torch


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def main():
    n = 1310720
    h_in = torch.empty(n, dtype=torch.complex128, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.complex128, pin_memory=True)
    d_a = torch.empty(n, dtype=torch.complex128, device="cuda")
    d_b = torch.empty(n, dtype=torch.complex128, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    mb = n * 16 / 1e6

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both)]:
        t = timed(fn)
        print(f"{name}: {t * 1e3:.3f} ms for {mb:.1f} MB each = {mb / t / 1e3:.1f} GB/s per direction", flush=True)


if __name__ == "__main__":
    main()
