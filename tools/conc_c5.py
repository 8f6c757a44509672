"""Concurrent vs serial engines at a C5-shaped size (N = RKN, default 6000): step time and the
per-class event times (tools/conc_c5.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import cilgen  # noqa: E402
import paper_2203_14742_b200 as cil  # noqa: E402
from paper_2203_14742_b200 import _capi  # noqa: E402

dev = torch.device("cuda")
grid, N, M = (2, 256, 256), int(os.environ.get("RKN", "6000")), 20
A = cilgen.make_set(cilgen.config_seed(5), 0, N, grid, device=dev)
B = cilgen.make_set(cilgen.config_seed(5), 1, N, grid, device=dev)
R = torch.tensor(bench.pilot_radii_all(A, B, grid, M, 0x3F), dtype=torch.float64, device=dev)
ws = cil.Workspace()
for on in (0, 1, 0, 1):
    _capi.lib.cil_diag_concurrent_engines(on)
    cil.features(A, B, grid, 0x3F, R, ws=ws)
    torch.cuda.synchronize()
    _capi.prof_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cil.features(A, B, grid, 0x3F, R, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    _capi.prof_enable(False)
    p = _capi.prof_read()
    print("concurrent" if on else "serial    ", round(e0.elapsed_time(e1), 1), "ms",
          {k: round(v[0], 1) for k, v in p.items() if v[1]})
_capi.lib.cil_diag_concurrent_engines(1)
