"""cilgen-v1 — seeded, index-addressable synthetic pattern generator (harness only).

This module feeds BOTH the CUDA path and the FP64 oracle; it holds none of the
method's arithmetic (no distances, no counts, no statistics).  It stands in for
the paper's PDE forward solvers, which are out of scope:
patterns with "about five 'wavelengths'" of spot/stripe
structure on a uniform grid x = i*h, h = 1/(W-1).

Recipe:
  F(x, y) = sqrt(2/J) * sum_{j<J} cos(k_j (x cos t_j + y sin t_j) + p_j),  J = 48
      t_j, p_j ~ U(0, 2pi),  k_j = 2 pi n_w U(0.9, 1.1),  n_w = 5 wavelengths
  g = tanh(2 (F - 0.5))                         (spots)
  v_s = off_s + a * amp_s * (g + 0.25 * F'_s)   (a ~ U(0.85, 1.15) per pattern;
                                                F'_s an independent field per species)
Profiles give (off, amp) per species, from the homogeneous steady states of the
paper's models (GM (2, 4) at theta_0 = (0.5, 1)).

Randomness is counter-based (splitmix64 of (seed, set_id, idx, counter)), so any
rank or test can generate any row with no communication and the same bits.
The separable form cos(a + b) = cos a cos b - sin a sin b turns each field into a
(H x 2J) @ (2J x W) product evaluated in float64, then rounded to float32.
"""
from __future__ import annotations

import math

import numpy as np
import torch

J = 48
VERSION = "cilgen-v1"

PROFILES = {
    # name: (offsets per species, amplitudes per species)
    "GM": ((2.0, 4.0), (1.0, 0.6)),
    "FHN": ((0.0, 0.0), (1.0, 1.0)),
    "BZ": ((4.5, 1.5467), (1.0, 0.5)),
}

_MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix(x: np.ndarray) -> np.ndarray:
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & _MASK64
    z = x
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _MASK64
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _MASK64
    return z ^ (z >> np.uint64(31))


def uniforms(seed: int, set_id: int, idx: np.ndarray, n_counters: int) -> np.ndarray:
    """U[0,1) doubles, shape [len(idx), n_counters]; a pure function of its arguments."""
    with np.errstate(over="ignore"):
        idx = np.asarray(idx, dtype=np.uint64).reshape(-1, 1)
        k = _splitmix(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))
        k = _splitmix(k ^ np.uint64(set_id & 0xFFFFFFFFFFFFFFFF))
        k = _splitmix(k ^ idx)
        c = np.arange(n_counters, dtype=np.uint64).reshape(1, -1)
        u = _splitmix(k + c * np.uint64(0xD1B54A32D192ED03))
    return (u >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def make_patterns(seed: int, set_id: int, idx, grid, profile: str = "GM", *,
                  n_w: float = 5.0, amp_scale: float = 1.0, device="cpu",
                  scaled: bool = False) -> torch.Tensor:
    """Patterns [n, S, H, W] float32 for pattern indices ``idx`` of set ``set_id``.

    grid = (S, H, W) or (S, H, W, h).  ``scaled`` applies the per-pattern,
    per-species min-max normalisation of PAPER.md:451-456.
    """
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    idx = np.arange(idx) if isinstance(idx, (int, np.integer)) else np.asarray(idx)
    idx = np.asarray(idx, dtype=np.int64).reshape(-1)
    n = idx.shape[0]
    off, amp = PROFILES[profile]
    if S > len(off):
        off = tuple(off) + tuple(off[-1] for _ in range(S - len(off)))
        amp = tuple(amp) + tuple(amp[-1] for _ in range(S - len(amp)))
    if n == 0:
        return torch.zeros((0, S, H, W), dtype=torch.float32, device=device)
    nf = 1 + S                       # main field + one secondary field per species
    U = uniforms(seed, set_id, idx, nf * 3 * J + 1)
    a = 0.85 + 0.30 * U[:, -1]                                   # amplitude jitter
    P = U[:, :-1].reshape(n, nf, 3, J)
    theta = 2 * math.pi * P[:, :, 0, :]
    phi = 2 * math.pi * P[:, :, 1, :]
    kk = 2 * math.pi * n_w * (0.9 + 0.2 * P[:, :, 2, :])
    dev = torch.device(device)
    t = lambda x: torch.as_tensor(x, dtype=torch.float64, device=dev)
    theta, phi, kk = t(theta), t(phi), t(kk)
    h = 1.0 / (W - 1) if W > 1 else 1.0
    xs = torch.arange(W, dtype=torch.float64, device=dev) * h       # column coordinate
    ys = torch.arange(H, dtype=torch.float64, device=dev) * h       # row coordinate
    kx = kk * torch.cos(theta)                                       # [n, nf, J]
    ky = kk * torch.sin(theta)
    ax = kx[..., None, :] * xs[:, None] + phi[..., None, :]          # [n, nf, W, J]
    by = ky[..., None, :] * ys[:, None]                              # [n, nf, H, J]
    Lm = torch.cat([torch.cos(by), -torch.sin(by)], dim=-1)          # [n, nf, H, 2J]
    Rm = torch.cat([torch.cos(ax), torch.sin(ax)], dim=-1)           # [n, nf, W, 2J]
    F = torch.matmul(Lm, Rm.transpose(-1, -2)) * math.sqrt(2.0 / J)  # [n, nf, H, W]
    g = torch.tanh(2.0 * (F[:, 0] - 0.5))
    out = torch.empty((n, S, H, W), dtype=torch.float64, device=dev)
    a_t = t(a)[:, None, None] * amp_scale
    for s in range(S):
        out[:, s] = off[s] + a_t * amp[s] * (g + 0.25 * F[:, 1 + s])
    if scaled:
        flat = out.reshape(n, S, -1)
        mn = flat.min(dim=-1, keepdim=True).values
        mx = flat.max(dim=-1, keepdim=True).values
        out = ((flat - mn) / (mx - mn)).reshape(n, S, H, W)
    return out.to(torch.float32)


def make_set(seed: int, set_id: int, n: int, grid, profile: str = "GM", device="cpu",
             chunk: int = 2048, out: torch.Tensor | None = None, row0: int = 0, **kw) -> torch.Tensor:
    """Rows [row0, row0 + n) of a set, generated in chunks (bounded temporaries)."""
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    if out is None:
        out = torch.empty((n, S, H, W), dtype=torch.float32, device=device)
    step = max(1, min(chunk, (1 << 25) // (3 * H * W)))
    for s0 in range(0, n, step):
        s1 = min(n, s0 + step)
        out[s0:s1] = make_patterns(seed, set_id, np.arange(row0 + s0, row0 + s1), grid, profile,
                                   device=device, **kw)
    return out


# Seeds per config: 22031474200 + config number.
def config_seed(config_number: int) -> int:
    return 22031474200 + int(config_number)


# --------------------------------------------------------------------------- bootstrap draws
# The random draws of the bootstrap estimators (Alg. A1 / A2) are inputs
# of both the library and the oracle (reading R14 of DESIGN.md): seeded, host-side, no
# method arithmetic.  Uniforms come from the same splitmix64 counters as the patterns.
def _draw_uniforms(seed: int, stream: int, shape) -> np.ndarray:
    n = int(np.prod(shape))
    u = uniforms(seed, 1_000_000 + stream, np.arange(1, dtype=np.int64), n)[0]
    return u.reshape(shape)


def boot_draws_a2(seed: int, stream: int, n_rep: int, N_syn: int, N_set: int):
    """Alg. A2 draws for one theta: I1 [n_rep][N_set] with replacement from the pool
    (step 2.1); I2 [n_rep][N_syn - N_set] with replacement from the patterns NOT drawn
    into s^1 of the same replicate (step 2.2, "the remaining patterns"); J [N_syn - N_set]
    a subset of the pool without replacement (step 4)."""
    Nt = N_syn - N_set
    u1 = _draw_uniforms(seed, 3 * stream, (n_rep, N_set))
    I1 = np.minimum((u1 * N_syn).astype(np.int64), N_syn - 1)
    drawn = np.zeros((n_rep, N_syn), dtype=bool)
    np.put_along_axis(drawn, I1, True, axis=1)
    rest = (~drawn).sum(axis=1)                                   # >= N_syn - N_set >= 1
    order = np.argsort(drawn, axis=1, kind="stable")              # undrawn indices first, increasing
    u2 = _draw_uniforms(seed, 3 * stream + 1, (n_rep, Nt))
    pos = np.minimum((u2 * rest[:, None]).astype(np.int64), rest[:, None] - 1)
    I2 = np.take_along_axis(order, pos, axis=1)
    u3 = _draw_uniforms(seed, 3 * stream + 2, (N_syn,))
    J = np.argsort(u3, kind="stable")[:Nt]
    return I1.astype(np.int32), I2.astype(np.int32), J.astype(np.int32)


def boot_draws_a1(seed: int, stream: int, n_rep: int, half: int):
    """Alg. A1 draws: I1, I2 [n_rep][half] with replacement from s~1 and s~2 (step 2.1)."""
    u1 = _draw_uniforms(seed, 3 * stream, (n_rep, half))
    u2 = _draw_uniforms(seed, 3 * stream + 1, (n_rep, half))
    I1 = np.minimum((u1 * half).astype(np.int64), half - 1)
    I2 = np.minimum((u2 * half).astype(np.int64), half - 1)
    return I1.astype(np.int32), I2.astype(np.int32)
