"""A/B of the pipelined pack / Gram batches (cil_diag_pipeline) on the C2 workload: step time of
cil_features by CUDA events, counts compared."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import cilgen  # noqa: E402
import paper_2203_14742_b200 as cil  # noqa: E402
from paper_2203_14742_b200 import _capi  # noqa: E402

dev = torch.device("cuda")
grid, P, N, M = (2, 64, 64), 100, 500, 15
seed = cilgen.config_seed(2)
A = torch.empty((P, N) + grid, device=dev)
B = torch.empty((P, N) + grid, device=dev)
for p in range(P):
    cilgen.make_set(seed, 2 * p, N, grid, device=dev, out=A[p])
    cilgen.make_set(seed, 2 * p + 1, N, grid, device=dev, out=B[p])
R = torch.tensor([bench.pilot_radii(A[0, :64], B[0, :64], grid, M)], dtype=torch.float64, device=dev)
ws = cil.Workspace()
res = {}
for rnd in range(3):
    for on in (0, 1):
        _capi.lib.cil_diag_pipeline(on)
        for _ in range(3):
            c, _, st = cil.features(A, B, grid, cil.L2, R, ws=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            c, _, st = cil.features(A, B, grid, cil.L2, R, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(on, []).append(round(e0.elapsed_time(e1) / 10, 4))
        res[("c", on)] = c.clone()
_capi.lib.cil_diag_pipeline(1)
print("serial", res[0], "pipelined", res[1], "identical", torch.equal(res[("c", 0)], res[("c", 1)]),
      "status", int(st.max()))
