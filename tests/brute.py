"""Independent NumPy brute force (tiny inputs only) — a second, differently-written
implementation of the paper's definitions used to pin the C oracle.

It shares nothing with oracle/cil_oracle.c: vectorised np.diff / broadcasting instead
of scalar loops.  Definitions: Eq. (1); Eqs. (5)-(10) PAPER.md:178-193
with the readings R1 (weight h^dim), R3 (forward difference, last node omitted),
R4 (species summed / maxed) of DESIGN.md.
"""
from __future__ import annotations

import numpy as np


def distances(A, B, grid):
    """d[6][N][Nt] for (L2, Linf, W12sum, W12, W1inf, W1infsum); grid[4] (optional) = species
    mask of the derivative terms (0 = all)."""
    S, H, W, h = grid[:4]
    gs = int(grid[4]) if len(grid) > 4 else 0
    if h <= 0:
        h = 1.0 / (W - 1) if W > 1 else 1.0
    dim = 2 if H > 1 else 1
    w = h ** dim
    A = np.asarray(A, np.float64).reshape(-1, S, H, W)
    B = np.asarray(B, np.float64).reshape(-1, S, H, W)
    U = A[:, None] - B[None, :]                      # [N, Nt, S, H, W]
    sel = [s for s in range(S) if gs == 0 or (gs >> s) & 1]
    DX = np.diff(U[:, :, sel], axis=-1) / h          # [.., W-1]  last node dropped
    DY = np.diff(U[:, :, sel], axis=-2) / h          # [.., H-1, W]
    red = lambda X, f: f(X.reshape(X.shape[0], X.shape[1], -1), axis=-1) if X.size else np.zeros(U.shape[:2])
    s0, sx, sy = red(U ** 2, np.sum), red(DX ** 2, np.sum), red(DY ** 2, np.sum)
    m0, mx, my = red(np.abs(U), np.max), red(np.abs(DX), np.max), red(np.abs(DY), np.max)
    a0, ax, ay = np.sqrt(w * s0), np.sqrt(w * sx), np.sqrt(w * sy)
    return np.stack([a0, m0, a0 + ax + ay, np.sqrt(a0 ** 2 + ax ** 2 + ay ** 2),
                     np.maximum(np.maximum(m0, mx), my), m0 + mx + my])


def counts(A, B, grid, mask, radii):
    d = distances(A, B, grid)
    sel = [q for q in range(6) if (mask >> q) & 1]
    radii = np.asarray(radii, np.float64).reshape(len(sel), -1)
    return np.stack([(d[q][None, :, :] < radii[i][:, None, None]).sum(axis=(1, 2))
                     for i, q in enumerate(sel)]).astype(np.int64)


def synth(pool, n_ens, N_set, N_tilde, data, k0, grid, mask, radii):
    """Alg. 3 written out with the brute-force counts; returns (Y, ytilde)."""
    N = N_set + N_tilde
    pool = np.asarray(pool)
    vecs = []
    for k in range(n_ens):
        for l in range(n_ens):
            s1 = pool[k * N:k * N + N_set]
            s2 = pool[l * N + N_set:(l + 1) * N]
            vecs.append((counts(s1, s2, grid, mask, radii) / (N_set * N_tilde)).ravel())
    s2 = pool[k0 * N + N_set:(k0 + 1) * N]
    yt = (counts(data, s2, grid, mask, radii) / (N_set * N_tilde)).ravel()
    return np.array(vecs), yt
