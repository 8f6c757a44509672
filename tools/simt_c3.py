"""The FP32 CUDA-core engine (engine=SIMT) at the C3 shape: all six measures and the max family
alone; per-class event times (tools/simt_var.sh-style variant timing)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import cilgen  # noqa: E402
import paper_2203_14742_b200 as cil  # noqa: E402
from paper_2203_14742_b200 import _capi  # noqa: E402

dev = torch.device("cuda")
grid, N, M = (2, 128, 128), 2000, 20
A = cilgen.make_set(cilgen.config_seed(3), 0, N, grid, device=dev)
B = cilgen.make_set(cilgen.config_seed(3), 1, N, grid, device=dev)
Rall = torch.tensor(bench.pilot_radii_all(A, B, grid, M, 0x3F), dtype=torch.float64, device=dev)
tag = sys.argv[1] if len(sys.argv) > 1 else "-"
for name, mask, rows in (("all six", 0x3F, list(range(6))), ("max family", 0x32, [1, 4, 5])):
    ws = cil.Workspace()
    R = Rall[rows]
    cil.features(A, B, grid, mask, R, ws=ws, engine=cil.ENGINE_SIMT)
    torch.cuda.synchronize()
    _capi.prof_enable(True)
    for _ in range(2):
        c, _, st = cil.features(A, B, grid, mask, R, ws=ws, engine=cil.ENGINE_SIMT)
    torch.cuda.synchronize()
    _capi.prof_enable(False)
    p = _capi.prof_read()
    print(tag, name, {k: round(v[0] / 2, 2) for k, v in p.items() if v[1]}, int(c.sum()) % 1000003, int(st[0]))
