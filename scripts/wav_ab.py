"""A/B timing of the wavelet transform W / W^T at cfg 4 size (J = 10,
N_x = 1,046,529) and a digest of the results (the variants must agree bit
for bit).

    python scripts/wav_ab.py                 # top two stages fused (default)
    HWG_WAV_FUSE=0 python scripts/wav_ab.py  # one launch per stage
"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_08875_b200.device import GpuContext  # noqa: E402

J, K = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (10, 10)
ctx = GpuContext(2, J, K)
gen = torch.Generator(device="cuda").manual_seed(2)
X = torch.randn((ctx.n_t, ctx.n_x), dtype=torch.float64, device="cuda", generator=gen)
Y = torch.empty_like(X)
tag = os.environ.get("HWG_WAV_FUSE", "1")
for tr in (False, True):
    for _ in range(2):
        ctx.wavelet(X, Y, tr)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        ctx.wavelet(X, Y, tr)
    b.record()
    torch.cuda.synchronize()
    h = hashlib.sha1(Y.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"HWG_WAV_FUSE={tag} {'W^T' if tr else 'W  '} {a.elapsed_time(b) / 10:.3f} ms  {h}")
