"""The README usage example, runnable: python tools/readme_example.py (B200)."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2203_14742_b200 as cil
grid = (2, 64, 64, 0.0)                       # S species x H x W, h (0: 1/(W-1))
A = torch.randn(100, 500, 2, 64, 64, device="cuda")   # P = 100 set pairs, N = 500 patterns each
B = torch.randn(100, 500, 2, 64, 64, device="cuda")
rng, _ = cil.distance_range(A, B, grid, cil.L2)        # per-item (min, max) distance
radii, _ = cil.radii_from_range(rng, 15)               # power-law radii R_1 > ... > R_15
counts, y, status = cil.features(A, B, grid, cil.L2, radii)   # Eq. (1): y [P, 1, 15]
mu, Sigma = cil.stats(y.reshape(100, -1))              # mu_0, Sigma_0 over the 100 vectors
out, st = cil.loglik(mu, Sigma, y.reshape(100, -1), ridge=1e-6)  # (quad, logdet, loglik), Eq. (4)

torch.cuda.synchronize(); print(y.shape, out.shape, int(status.max()), int(st.max()), out[:2].tolist())
