"""HBM rate against the read : write mix (torch elementwise kernels over 8.6 GB
fp64 arrays): the stencil kernels' ceilings depend on their mix, not only on
the copy bandwidth of MEASURED_PEAKS.json (1 : 1).

    python scripts/micro/rw_mix.py
"""
import torch

n = 1025 * 1023 * 1023
a = torch.randn(n, dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
c = torch.empty_like(a)


def timed(f, nbytes, name, reps=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name:28s} {ms:7.3f} ms  {nbytes / ms / 1e9:6.2f} TB/s", flush=True)


timed(lambda: a.sum(), 8 * n, "read only (sum)")
timed(lambda: b.fill_(1.0), 8 * n, "write only (fill)")
timed(lambda: b.copy_(a), 16 * n, "1 read : 1 write (copy)")
timed(lambda: torch.add(a, b, out=c), 24 * n, "2 reads : 1 write (add)")
