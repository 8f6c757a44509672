"""A/B of the concurrent engines (cil_diag_concurrent_engines) at the C3 and a C5-shaped (N = 2000)
configuration, all six measures: step time by CUDA events on the caller's stream, counts compared."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import cilgen  # noqa: E402
import paper_2203_14742_b200 as cil  # noqa: E402
from paper_2203_14742_b200 import _capi  # noqa: E402

dev = torch.device("cuda")
for name, grid, seed in (("C3", (2, 128, 128), 3), ("C5-shape N=2000", (2, 256, 256), 5)):
    N, M = 2000, 20
    A = cilgen.make_set(cilgen.config_seed(seed), 0, N, grid, device=dev)
    B = cilgen.make_set(cilgen.config_seed(seed), 1, N, grid, device=dev)
    R = torch.tensor(bench.pilot_radii_all(A, B, grid, M, 0x3F), dtype=torch.float64, device=dev)
    ws = cil.Workspace()
    res = {}
    for on in (0, 1, 0, 1):
        _capi.lib.cil_diag_concurrent_engines(on)
        for _ in range(2):
            c, _, st = cil.features(A, B, grid, 0x3F, R, ws=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            c, _, st = cil.features(A, B, grid, 0x3F, R, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(on, []).append(e0.elapsed_time(e1) / 3)
        res.setdefault(("c", on), c.clone())
    _capi.lib.cil_diag_concurrent_engines(1)
    same = torch.equal(res[("c", 0)], res[("c", 1)])
    print(f"{name}: serial {res[0]} ms, concurrent {res[1]} ms, counts identical {same}, status {int(st[0])}")
    del A, B, ws
    torch.cuda.empty_cache()
