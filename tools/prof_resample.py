"""Standalone timing of cil_resample_counts at the C6 shape (64 x 1000 x 1000 bins,
1000 replicates of 50 x 950 draws) — for ncu and quick A/B runs."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import cilgen  # noqa: E402
import paper_2203_14742_b200 as cil  # noqa: E402

P, N, n_rep, N_set, M = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 1000, 1000, 50, 13
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
bins = torch.randint(0, M + 1, (P, 1, N, N), dtype=torch.uint8, device=dev, generator=g)
draws = [cilgen.boot_draws_a2(3, p, n_rep, N, N_set) for p in range(P)]
I1 = torch.tensor(np.stack([d[0] for d in draws]), device=dev)
I2 = torch.tensor(np.stack([d[1] for d in draws]), device=dev)
for _ in range(3):
    cil.resample_counts(bins, I1, I2, M, want_counts=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
R = 10
for _ in range(R):
    cil.resample_counts(bins, I1, I2, M, want_counts=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
print(f"resample P={P}: {ms:.3f} ms/call, {P * n_rep * N_set * (N - N_set) / ms / 1e9:.1f} G lookups/s")
