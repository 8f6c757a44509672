"""Times the CUDA-core max family (k_simt, Linf + W1inf + W1infsum) at the C3 shape for one build of
libcil.so: python tools/simt_var.py TAG (used by tools/simt_var.sh; prints one line)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cilgen  # noqa: E402
import paper_2203_14742_b200 as cil  # noqa: E402
from paper_2203_14742_b200 import _capi  # noqa: E402

dev = torch.device("cuda")
grid, N, M = (2, 128, 128), 2000, 20
mask = cil.LINF | cil.W1INF | cil.W1INFSUM
A = cilgen.make_set(cilgen.config_seed(3), 0, N, grid, device=dev)
B = cilgen.make_set(cilgen.config_seed(3), 1, N, grid, device=dev)
rng, _ = cil.distance_range(A[:128], B[:128], grid + (0.0,), mask)
R, _ = cil.radii_from_range(rng, M)
R = R[0]
ws = cil.Workspace()
for _ in range(2):
    c, _, st = cil.features(A, B, grid + (0.0,), mask, R, ws=ws)
torch.cuda.synchronize()
_capi.prof_enable(True)
for _ in range(4):
    cil.features(A, B, grid + (0.0,), mask, R, ws=ws)
torch.cuda.synchronize()
_capi.prof_enable(False)
p = _capi.prof_read()["simt_tile"]
print(f"{sys.argv[1] if len(sys.argv) > 1 else '-':24s} simt_tile {p[0] / p[1]:.3f} ms  status {int(st[0])}  "
      f"counts {int(c.sum())}")
