"""FP64 CPU oracle for the CIL hot path — ctypes wrapper around ``cil_oracle.c``.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
module.  The product package ``paper_2203_14742_b200`` never imports it, and it
imports nothing from the product package: the two share no code.

Every function follows the plain definition in arXiv 2203.14742:
Eq. (1), Eq. (2), Eq. (4) PAPER.md:144-148,
Eqs. (5)-(10) PAPER.md:178-193, Eqs. (11)-(13) and Alg. 3 PAPER.md:236-297.
Readings of the paper where it is silent: DESIGN.md "Readings" R1..R10.
Pins (what fixes this oracle to something other than itself): tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cil_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# measure bits (bit order = concatenation order)
L2, LINF, W12SUM, W12, W1INF, W1INFSUM = (1 << i for i in range(6))
MEASURE_NAMES = ["L2", "LINF", "W12SUM", "W12", "W1INF", "W1INFSUM"]
ITEM_OK, ITEM_NONFINITE, ITEM_NOTPD = 0, 1, 2

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no fast-math, no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm", "-lpthread"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, u32, f64 = ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_double
        lib.oracle_features.argtypes = [P, i64, i64, P, i64, i64, i32, i32, i32, f64, u32, u32, P, i32,
                                        f64, P, P, P, P, P, i32]
        lib.oracle_features.restype = i32
        lib.oracle_distance_matrix.argtypes = [P, i64, i64, P, i64, i64, i32, i32, i32, f64, u32, u32, P]
        lib.oracle_stats.argtypes = [P, i32, i32, P, P]
        lib.oracle_stats.restype = i32
        lib.oracle_loglik.argtypes = [P, P, P, i32, f64, P]
        lib.oracle_loglik.restype = i32
        lib.oracle_synth_loglik.argtypes = [P, i64, i32, i32, i32, P, i64, i32, i32, i32, i32, f64,
                                            u32, u32, P, i32, f64, P, P, i32]
        lib.oracle_synth_loglik.restype = i32
        lib.oracle_subnorms.argtypes = [P, P, P, P]
        lib.oracle_resample_features.argtypes = [P, i64, i64, P, i64, i64, i32, i32, i32, f64, u32, u32, P, i32, i32,
                                                 P, i64, P, i64, f64, P, P, P, P, i32]
        lib.oracle_resample_features.restype = i32
        lib.oracle_synth_boot.argtypes = [P, i64, i32, P, i64, i32, i32, P, P, P, i32, i32, i32, f64, u32, u32, P,
                                          i32, f64, P, P, i32]
        lib.oracle_synth_boot.restype = i32
        _lib = lib
    return _lib


def _f32(x):
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    return x


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def n_measures(mask: int) -> int:
    return bin(mask & 0x3F).count("1")


def _rows(X, K):
    X = _f32(X)
    n = X.shape[0] if X.ndim > 0 else 0
    X2 = X.reshape(n, -1) if n else X.reshape(0, K)
    assert X2.shape[1] == K, (X2.shape, K)
    return X2


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


def features(A, B, grid, mask, radii, band: float = 1e-6, nthreads: int | None = None):
    """Eq. (1)/(2): counts, band counts lo/hi, y and #ambiguous (pair, radius) cases.

    A: [N][S][H][W] (or [N][K]) float32, B: [Nt][...]; grid = (S, H, W, h);
    radii: [n_meas][M] strictly decreasing.  Returns dict of numpy arrays.
    """
    S, H, W, h = grid[:4]
    gs = int(grid[4]) if len(grid) > 4 else 0
    K = S * H * W
    A2, B2 = _rows(A, K), _rows(B, K)
    nq = n_measures(mask)
    radii = np.ascontiguousarray(np.asarray(radii, dtype=np.float64).reshape(nq, -1))
    M = radii.shape[1]
    cnt = np.zeros((nq, M), np.int64)
    lo = np.zeros_like(cnt)
    hi = np.zeros_like(cnt)
    y = np.zeros((nq, M), np.float64)
    amb = np.zeros(1, np.int64)
    st = _load().oracle_features(_ptr(A2), K, A2.shape[0], _ptr(B2), K, B2.shape[0], S, H, W,
                                 float(h), gs, mask, _ptr(radii), M, float(band), _ptr(cnt), _ptr(lo),
                                 _ptr(hi), _ptr(y), _ptr(amb), nthreads or default_threads())
    if st < 0:
        raise ValueError("oracle_features: invalid arguments")
    return {"counts": cnt, "lo": lo, "hi": hi, "y": y, "ambiguous": int(amb[0]), "status": st}


def distance_matrix(A, B, grid, mask):
    """All pairwise distances d[q][i][j] for the selected measures (tiny inputs)."""
    S, H, W, h = grid[:4]
    gs = int(grid[4]) if len(grid) > 4 else 0
    K = S * H * W
    A2, B2 = _rows(A, K), _rows(B, K)
    nq = n_measures(mask)
    D = np.zeros((nq, A2.shape[0], B2.shape[0]), np.float64)
    _load().oracle_distance_matrix(_ptr(A2), K, A2.shape[0], _ptr(B2), K, B2.shape[0], S, H, W,
                                   float(h), gs, mask, _ptr(D))
    return D


class _Grid(ctypes.Structure):
    _fields_ = [("S", ctypes.c_int), ("H", ctypes.c_int), ("W", ctypes.c_int), ("h", ctypes.c_double),
                ("gs", ctypes.c_uint)]


def subnorms(a, b, grid):
    """(s0, sx, sy, m0, mx, my) of u = a - b (sums of squares, derivative terms / h^2)."""
    S, H, W, h = grid[:4]
    gs = int(grid[4]) if len(grid) > 4 else 0
    a, b = _f32(a).ravel(), _f32(b).ravel()
    g = _Grid(S, H, W, float(h), gs)
    out = np.zeros(6, np.float64)
    _load().oracle_subnorms(_ptr(a), _ptr(b), ctypes.byref(g), _ptr(out))
    return out


def stats(Y):
    """mu, Sigma (two-pass, 1/(n-1)) of the n realisations Y[n][D]."""
    Y = np.ascontiguousarray(np.asarray(Y, np.float64))
    n, D = Y.shape
    mu = np.zeros(D)
    Sig = np.zeros((D, D))
    if _load().oracle_stats(_ptr(Y), n, D, _ptr(mu), _ptr(Sig)) != 0:
        raise ValueError("oracle_stats needs n >= 2")
    return mu, Sig


def loglik(mu, Sigma, y, ridge: float = 0.0):
    """(quad, logdet, loglik), status — Eq. (4)/(12) plus the Gaussian log-density [R8]."""
    mu = np.ascontiguousarray(np.asarray(mu, np.float64))
    Sigma = np.ascontiguousarray(np.asarray(Sigma, np.float64))
    y = np.ascontiguousarray(np.asarray(y, np.float64))
    out = np.zeros(3)
    st = _load().oracle_loglik(_ptr(mu), _ptr(Sigma), _ptr(y), mu.shape[0], float(ridge), _ptr(out))
    return out, st


def synth_loglik(pool, n_ens, N_set, N_tilde, data, k0, grid, mask, radii, ridge=0.0,
                 nthreads: int | None = None):
    """SCIL at one theta (Alg. 3): returns (out[3], status, Y[n_ens^2 + 1][D])."""
    S, H, W, h = grid[:4]
    gs = int(grid[4]) if len(grid) > 4 else 0
    K = S * H * W
    P2 = _rows(pool, K)
    D2 = _rows(data, K)
    assert P2.shape[0] >= n_ens * (N_set + N_tilde)
    assert D2.shape[0] == N_set
    nq = n_measures(mask)
    radii = np.ascontiguousarray(np.asarray(radii, np.float64).reshape(nq, -1))
    M = radii.shape[1]
    out = np.zeros(3)
    Y = np.zeros((n_ens * n_ens + 1, nq * M))
    st = _load().oracle_synth_loglik(_ptr(P2), K, n_ens, N_set, N_tilde, _ptr(D2), K, int(k0), S, H,
                                     W, float(h), gs, mask, _ptr(radii), M, float(ridge), _ptr(out),
                                     _ptr(Y), nthreads or default_threads())
    return out, st, Y


def resample_features(A, B, grid, mask, radii, I1, I2, band: float = 1e-6, nthreads: int | None = None):
    """Bootstrap step 2 (Alg. A1 / A2): for replicate k, s^1 = A[I1[k]], s^2 = B[I2[k]]
    constructed explicitly, then Eq. (1).  I1 [n_rep][n1], I2 [n_rep][n2] int.
    Returns dict counts / lo / hi [n_rep][nq][M], y [n_rep][nq*M], status."""
    S, H, W, h = grid[:4]
    gs = int(grid[4]) if len(grid) > 4 else 0
    K = S * H * W
    A2, B2 = _rows(A, K), _rows(B, K)
    nq = n_measures(mask)
    radii = np.ascontiguousarray(np.asarray(radii, dtype=np.float64).reshape(nq, -1))
    M = radii.shape[1]
    I1 = np.ascontiguousarray(np.asarray(I1, np.int32))
    I2 = np.ascontiguousarray(np.asarray(I2, np.int32))
    n_rep, n1, n2 = I1.shape[0], I1.shape[1], I2.shape[1]
    cnt = np.zeros((n_rep, nq, M), np.int64)
    lo = np.zeros_like(cnt)
    hi = np.zeros_like(cnt)
    y = np.zeros((n_rep, nq * M), np.float64)
    st = _load().oracle_resample_features(_ptr(A2), K, A2.shape[0], _ptr(B2), K, B2.shape[0], S, H, W, float(h),
                                          gs, mask, _ptr(radii), M, n_rep, _ptr(I1), n1, _ptr(I2), n2, float(band),
                                          _ptr(cnt), _ptr(lo), _ptr(hi), _ptr(y), nthreads or default_threads())
    if st < 0:
        raise ValueError("oracle_resample_features: invalid arguments or index out of range")
    return {"counts": cnt, "lo": lo, "hi": hi, "y": y, "status": st}


def synth_boot(pool, data, N_set, I1, I2, J, grid, mask, radii, ridge=0.0, nthreads: int | None = None):
    """SCIL with bootstrapping at one theta (Alg. A2): returns (out[3], status, Y[n_rep + 1][D])."""
    S, H, W, h = grid[:4]
    gs = int(grid[4]) if len(grid) > 4 else 0
    K = S * H * W
    P2 = _rows(pool, K)
    D2 = _rows(data, K)
    assert D2.shape[0] == N_set
    nq = n_measures(mask)
    radii = np.ascontiguousarray(np.asarray(radii, np.float64).reshape(nq, -1))
    M = radii.shape[1]
    I1 = np.ascontiguousarray(np.asarray(I1, np.int32))
    I2 = np.ascontiguousarray(np.asarray(I2, np.int32))
    J = np.ascontiguousarray(np.asarray(J, np.int32))
    n_rep = I1.shape[0]
    out = np.zeros(3)
    Y = np.zeros((n_rep + 1, nq * M))
    st = _load().oracle_synth_boot(_ptr(P2), K, P2.shape[0], _ptr(D2), K, N_set, n_rep, _ptr(I1), _ptr(I2),
                                   _ptr(J), S, H, W, float(h), gs, mask, _ptr(radii), M, float(ridge), _ptr(out),
                                   _ptr(Y), nthreads or default_threads())
    if st < 0:
        raise ValueError("oracle_synth_boot: invalid arguments or index out of range")
    return out, st, Y


def train_vectors(X, n_ens, grid, mask, radii, band: float = 1e-6, nthreads: int | None = None):
    """Alg. 1 / Alg. 2 steps 1-2: divide X into n_ens subsets of
    N = len(X) / n_ens rows (step 1); for every unordered pair k < l (lexicographic order,
    C(n_ens, 2) realisations) the correlation-integral vector of (s^k, s^l) by
    Eq. (1) (step 2).  Returns dict counts / lo / hi [n_pairs][nq][M], y [n_pairs][nq*M]."""
    S, H, W, h = grid[:4]
    gs = int(grid[4]) if len(grid) > 4 else 0
    K = S * H * W
    X2 = _rows(X, K)
    N = X2.shape[0] // n_ens
    out = {"counts": [], "lo": [], "hi": [], "y": []}
    for k in range(n_ens):
        for l in range(k + 1, n_ens):
            r = features(X2[k * N:(k + 1) * N], X2[l * N:(l + 1) * N], grid, mask, radii, band=band,
                         nthreads=nthreads)
            out["counts"].append(r["counts"])
            out["lo"].append(r["lo"])
            out["hi"].append(r["hi"])
            out["y"].append(r["y"].ravel())
    return {k: np.array(v) for k, v in out.items()}


def distance_range(A, B, grid, mask):
    """(min positive, max) distance of every selected measure over all pairs (
    a pattern against itself is excluded from the minimum, reading R16).  Tiny inputs."""
    D = distance_matrix(A, B, grid, mask)
    out = np.zeros((D.shape[0], 2))
    for q in range(D.shape[0]):
        d = D[q].ravel()
        pos = d[d > 0]
        out[q, 0] = pos.min() if pos.size else np.inf
        out[q, 1] = d.max()
    return out


def radii_from_range(rng, M, law: str = "power", margin: float = 1e-3):
    """R_0 = max (1 + margin), R_M = min (1 - margin) [R5]; power law
    R_m = R_0 b^-m with R_M / R_0 = b^-M, or linear R_m = R_0 - m h with h = (R_0 - R_M)/M,
    m = 1..M."""
    rng = np.asarray(rng, np.float64)
    out = np.zeros((rng.shape[0], M))
    for q in range(rng.shape[0]):
        R0, RM = rng[q, 1] * (1 + margin), rng[q, 0] * (1 - margin)
        for m in range(1, M + 1):
            if law == "power":
                b = (R0 / RM) ** (1.0 / M)
                out[q, m - 1] = R0 * b ** (-m)
            else:
                out[q, m - 1] = R0 - m * (R0 - RM) / M
    return out


def minmax_scale(X, grid):
    """Scaled patterns: per pattern and species
    (s - s_min) / (s_max - s_min) over the species' grid values, FP64 then FP32; a constant
    species maps to 0 (reading R17)."""
    S, H, W, _ = grid
    X = np.asarray(X, np.float32).reshape(-1, S, H * W).astype(np.float64)
    mn = X.min(axis=2, keepdims=True)
    mx = X.max(axis=2, keepdims=True)
    span = mx - mn
    Y = np.where(span > 0, (X - mn) / np.where(span > 0, span, 1.0), 0.0)
    return Y.astype(np.float32).reshape(-1, S, H, W)
