"""One cfg-N PCG solve (setup + one warm solve + one profiled solve) for
ncu launch lists / traffic captures; prints nothing else of interest.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:mg2d_reg --csv --log-file out.csv python scripts/profile_solve.py 4
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2009_08875_b200 as hw  # noqa: E402
from paper_2009_08875_b200 import inputs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
d, J, K, dist, u0, n_t, n_x = bench.workload(cfg)
F = inputs.forcing(dist, n_t, n_x)
asm = hw.assemble_system(hw.ProblemData(D=bench.diffusion_of(cfg, d), c=0.0, u0=u0), J, K,
                         hw.SolveConfig(), forcing=F, host_rhs=False, domain=bench.domain_of(cfg))
del F
f = asm.rhs.f_hat.array
w = torch.empty_like(f)
stats, rc = asm.ctx.pcg(f, w, 0.0, 1e-6)
torch.cuda.synchronize()
print(f"cfg{cfg}: {stats['iterations']} iterations, rc {rc}", flush=True)
