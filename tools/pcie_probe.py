"""Pinned host <-> device copy times for the headline vector (2^20 complex128 = 16.8 MB) and its
pipeline parts: the floor of the host-buffer apply (bf_apply_host) next to the device time."""
import torch

n = 1 << 20
dev = torch.empty(n, dtype=torch.complex128, device="cuda")
dev2 = torch.empty(n, dtype=torch.complex128, device="cuda")
host = torch.empty(n, dtype=torch.complex128).pin_memory()
host2 = torch.empty(n, dtype=torch.complex128).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for frac in (1, 2, 8):
    m = n // frac
    h2d = timed(lambda: dev[:m].copy_(host[:m], non_blocking=True))
    d2h = timed(lambda: host2[:m].copy_(dev2[:m], non_blocking=True))
    print(f"1/{frac} of the vector ({m * 16 / 1e6:.1f} MB): H2D {h2d:.1f} us ({m * 16 / h2d / 1e3:.1f} GB/s), "
          f"D2H {d2h:.1f} us ({m * 16 / d2h / 1e3:.1f} GB/s)")


def both():
    with torch.cuda.stream(s1):
        dev.copy_(host, non_blocking=True)
    with torch.cuda.stream(s2):
        host2.copy_(dev2, non_blocking=True)


torch.cuda.synchronize()
import time
for _ in range(5):
    both()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    both()
torch.cuda.synchronize()
print(f"H2D + D2H of the whole vector on two streams: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us per pair")
