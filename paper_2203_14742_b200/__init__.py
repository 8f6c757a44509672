"""paper_2203_14742_b200 — B200-native hot path of the Correlation Integral
Likelihood (CIL / MCIL / SCIL) method of arXiv 2203.14742.

Python layer = argument marshalling over the C ABI of libcil.so (include/cil.h).
PyTorch supplies device memory and streams only.  Public calls (same names as the
C ABI, minus the prefix):

    features(A, B, grid, mask, radii)              -> counts, y, item_status   (Eq. (1)/(2))
    stats(Y)                                        -> mu, Sigma
    loglik(mu, Sigma, y_obs, ridge)                 -> out[P,3], item_status    (Eq. (4))
    synth_loglik(pools, n_ens, N_set, N_tilde, data, k0, grid, mask, radii)     (Alg. 3)
    bin_matrix(A, B, grid, mask, radii)             -> bins[P,n_meas,N,Nt] uint8 (bootstrap)
    resample_counts(bins, I1, I2, M)                -> counts, y               (Alg. A1/A2 step 2)
    synth_loglik_boot(pools, data, N_set, I1, I2, J, grid, mask, radii)         (Alg. A2)
    mcil_boot_stats(data, grid, mask, radii, I1, I2) -> mu_0, Sigma_0          (Alg. A1)
    train_vectors(X, n_ens, grid, mask, radii)      -> Y [P, C(n_ens,2), D]     (Alg. 1/2 steps 1-2)
    distance_range(A, B, grid, mask), radii_from_range(rng, M, law)
    minmax_scale(X, grid)                           -> scaled patterns
    gaussianity_chi2(Y)                             -> chi^2 statistic
    sharding.sharded_features / ring_features / gather_vectors                 (multi-GPU, §8(e))

Grid = (S, H, W[, h[, gs]]): gs = species mask of the derivative terms.

Measures (bit order = concatenation order): L2, LINF, W12SUM, W12,
W1INF, W1INFSUM (Eqs. (5)-(10)).
"""
from __future__ import annotations

import torch

from ._capi import CilError, Grid, check, lib  # noqa: F401  (fails loudly without libcil.so)

L2, LINF, W12SUM, W12, W1INF, W1INFSUM = (1 << i for i in range(6))
ALL = 0x3F
MEASURE_NAMES = ["L2", "LINF", "W12SUM", "W12", "W1INF", "W1INFSUM"]
ENGINE_AUTO, ENGINE_TC_3XBF16, ENGINE_TC_3XTF32, ENGINE_SIMT, ENGINE_TC_I8 = 0, 1, 2, 3, 4
ITEM_OK, ITEM_NONFINITE, ITEM_NOTPD, ITEM_BADRADII, ITEM_OVERFLOW, ITEM_BADINDEX = 0, 1, 2, 4, 8, 16

__all__ = ["features", "stats", "loglik", "synth_loglik", "features_workspace_size",
           "synth_workspace_size", "n_measures", "Workspace", "CilError", "bin_matrix", "resample_counts",
           "synth_loglik_boot", "mcil_boot_stats", "train_vectors", "gaussianity_chi2",
           "distance_range", "radii_from_range", "minmax_scale"]


def n_measures(mask: int) -> int:
    return bin(mask & ALL).count("1")


def _grid(grid) -> Grid:
    """(S, H, W[, h[, gs]]): gs = species mask of the derivative terms (0 = all)."""
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    h = float(grid[3]) if len(grid) > 3 else 0.0
    gs = int(grid[4]) if len(grid) > 4 else 0
    return Grid(S, H, W, h, gs)


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t) -> int | None:
    return t.data_ptr() if t is not None and t.numel() > 0 else None


class Workspace:
    """Grow-only device scratch buffer (the library never allocates)."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(device):
            self.buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        return self.buf


_default_ws = Workspace()


def features_workspace_size(P, N, Nt, grid, mask, M, engine=ENGINE_AUTO) -> int:
    return int(lib.cil_features_workspace_size(P, N, Nt, _grid(grid), mask, M, engine))


def synth_workspace_size(P, n_ens, N_set, N_tilde, grid, mask, M, engine=ENGINE_AUTO) -> int:
    return int(lib.cil_synth_workspace_size(P, n_ens, N_set, N_tilde, _grid(grid), mask, M, engine))


def _as_items(X, K):
    """[N,S,H,W] / [N,K] -> (P=1 view) or [P,N,S,H,W] / [P,N,K] -> P items."""
    if X.dim() in (2, 4):
        X = X.unsqueeze(0)
    P, N = X.shape[0], X.shape[1]
    if X.shape[2:].numel() != K:
        raise ValueError(f"pattern size != S*H*W = {K}")
    return X.reshape(P, N, K)


def features(A, B, grid, mask, radii, *, engine=ENGINE_AUTO, want_y=True, stream=None, ws: Workspace | None = None,
             counts=None, y=None, status=None):
    """Correlation-integral counts of one or P set pairs (Eq. (1)/(2)).

    A: [N,S,H,W] or [P,N,S,H,W] float32 CUDA; B likewise with Nt rows.
    radii: [n_meas, M] (shared) or [P, n_meas, M] float64 CUDA, strictly decreasing.
    Returns counts int64 [P,n_meas,M], y float64 [P,n_meas,M] (or None), item_status int32 [P].
    """
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    K = S * H * W
    A3, B3 = _as_items(A, K), _as_items(B, K)
    if A3.dtype != torch.float32 or B3.dtype != torch.float32:
        raise TypeError("patterns must be float32")
    if not (A3.is_cuda and B3.is_cuda and radii.is_cuda):
        raise TypeError("A, B and radii must be CUDA tensors")
    P, N, Nt = A3.shape[0], A3.shape[1], B3.shape[1]
    if B3.shape[0] != P:
        raise ValueError("A and B must have the same number of items")
    nq = n_measures(mask)
    radii = radii.to(torch.float64)
    if radii.dim() == 2:
        M, rstride = radii.shape[1], 0
    else:
        if radii.shape[0] != P:
            raise ValueError("radii must be [n_meas, M] or [P, n_meas, M]")
        M, rstride = radii.shape[2], radii.shape[1] * radii.shape[2]
    if radii.shape[-2] != nq:
        raise ValueError(f"radii rows {radii.shape[-2]} != n_measures(mask) = {nq}")
    radii = radii.contiguous()
    dev = A3.device
    if counts is None:
        counts = torch.empty((P, nq, M), dtype=torch.int64, device=dev)
    if want_y and y is None:
        y = torch.empty((P, nq, M), dtype=torch.float64, device=dev)
    if status is None:
        status = torch.empty((P,), dtype=torch.int32, device=dev)
    g = _grid(grid)
    nbytes = lib.cil_features_workspace_size(P, N, Nt, g, mask, M, engine)
    if nbytes == 0:
        raise CilError("cil_features_workspace_size: invalid arguments")
    wbuf = (ws or _default_ws).get(nbytes, dev)

    def stride_ld(X3):
        if X3.shape[1] == 0:
            return 0, K
        if X3.stride(2) != 1:
            raise ValueError("patterns must be contiguous along S*H*W")
        return X3.stride(0), X3.stride(1)

    sA, lda = stride_ld(A3)
    sB, ldb = stride_ld(B3)
    st = lib.cil_features(P, _ptr(A3), sA, lda, N, _ptr(B3), sB, ldb, Nt, g, mask, radii.data_ptr(), rstride, M,
                          counts.data_ptr(), y.data_ptr() if want_y else None, status.data_ptr(), engine,
                          wbuf.data_ptr(), wbuf.numel(), _stream(stream))
    check(st, "cil_features")
    return counts, (y if want_y else None), status


def recheck_count(P, N, Nt, grid, mask, M, engine=ENGINE_AUTO, ws: Workspace | None = None):
    """DIAGNOSTIC (synchronises): (listed, capacity) of the exact re-check list of the last features()
    call on the workspace `ws` (the default workspace if None)."""
    import ctypes
    w = (ws or _default_ws).buf
    listed, cap = ctypes.c_uint64(), ctypes.c_uint64()
    check(lib.cil_features_recheck_count(P, N, Nt, _grid(grid), mask, M, engine, w.data_ptr(), ctypes.byref(listed),
                                         ctypes.byref(cap)), "cil_features_recheck_count")
    return int(listed.value), int(cap.value)


def normalize(counts, npairs: float, *, stream=None):
    """y = counts / npairs on the device (cil_normalize; Eq. (1) normalisation)."""
    c = counts.contiguous()
    y = torch.empty(c.shape, dtype=torch.float64, device=c.device)
    check(lib.cil_normalize(c.numel(), c.data_ptr(), float(npairs), y.data_ptr(), _stream(stream)), "cil_normalize")
    return y


def stats(Y, *, stream=None):
    """mu [P,D], Sigma [P,D,D] of Y [P,n,D] (or [n,D]) — PAPER.md:111."""
    squeeze = Y.dim() == 2
    Y3 = (Y.unsqueeze(0) if squeeze else Y).to(torch.float64).contiguous()
    P, n, D = Y3.shape
    mu = torch.empty((P, D), dtype=torch.float64, device=Y3.device)
    Sig = torch.empty((P, D, D), dtype=torch.float64, device=Y3.device)
    check(lib.cil_stats(P, Y3.data_ptr(), n, D, mu.data_ptr(), Sig.data_ptr(), _stream(stream)), "cil_stats")
    return (mu[0], Sig[0]) if squeeze else (mu, Sig)


def loglik(mu, Sigma, y_obs, ridge: float = 0.0, *, stream=None):
    """Gaussian log-likelihood (Eq. (4)): out[P,3] = (quad, logdet, loglik), item_status [P].

    mu [D] or [P,D]; Sigma [D,D] or [P,D,D]; y_obs [D] or [P,D].
    """
    y2 = (y_obs.unsqueeze(0) if y_obs.dim() == 1 else y_obs).to(torch.float64).contiguous()
    P, D = y2.shape
    mu = mu.to(torch.float64).contiguous()
    Sigma = Sigma.to(torch.float64).contiguous()
    mu_stride = 0 if mu.dim() == 1 else D
    sig_stride = 0 if Sigma.dim() == 2 else D * D
    out = torch.empty((P, 3), dtype=torch.float64, device=y2.device)
    status = torch.empty((P,), dtype=torch.int32, device=y2.device)
    check(lib.cil_loglik(P, mu.data_ptr(), mu_stride, Sigma.data_ptr(), sig_stride, y2.data_ptr(), D, float(ridge),
                         out.data_ptr(), status.data_ptr(), _stream(stream)), "cil_loglik")
    return out, status


def synth_loglik(pools, n_ens, N_set, N_tilde, data, k0, grid, mask, radii, ridge: float = 0.0, *,
                 engine=ENGINE_AUTO, return_Y=False, stream=None, ws: Workspace | None = None, out=None,
                 status=None):
    """SCIL (Alg. 3) for P proposals.

    pools [P, N_syn, S,H,W] float32 (N_syn >= n_ens*(N_set+N_tilde)); data [N_set,S,H,W];
    k0 [P] int32; radii [P, n_meas, M] float64.  Returns out [P,3], item_status [P]
    (and Y [P, n_ens^2+1, D] if return_Y).
    """
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    K = S * H * W
    P = pools.shape[0]
    pools3 = pools.reshape(P, pools.shape[1], -1)
    data2 = data.reshape(data.shape[0], -1)
    if pools3.shape[-1] != K or data2.shape[-1] != K or data2.shape[0] != N_set:
        raise ValueError("pool / data shapes do not match grid and N_set")
    nq = n_measures(mask)
    radii = radii.to(torch.float64).contiguous()
    M = radii.shape[-1]
    if radii.shape != (P, nq, M):
        raise ValueError("radii must be [P, n_meas, M]")
    k0 = k0.to(torch.int32).contiguous()
    dev = pools.device
    if out is None:
        out = torch.empty((P, 3), dtype=torch.float64, device=dev)
    if status is None:
        status = torch.empty((P,), dtype=torch.int32, device=dev)
    Y = torch.empty((P, n_ens * n_ens + 1, nq * M), dtype=torch.float64, device=dev) if return_Y else None
    g = _grid(grid)
    nbytes = lib.cil_synth_workspace_size(P, n_ens, N_set, N_tilde, g, mask, M, engine)
    if nbytes == 0:
        raise CilError("cil_synth_workspace_size: invalid arguments")
    wbuf = (ws or _default_ws).get(nbytes, dev)
    st = lib.cil_synth_loglik(P, pools3.data_ptr(), pools3.stride(0), pools3.stride(1), n_ens, N_set, N_tilde,
                              data2.data_ptr(), data2.stride(0), k0.data_ptr(), g, mask, radii.data_ptr(), M,
                              float(ridge), out.data_ptr(), status.data_ptr(), Y.data_ptr() if return_Y else None,
                              engine, wbuf.data_ptr(), wbuf.numel(), _stream(stream))
    check(st, "cil_synth_loglik")
    return (out, status, Y) if return_Y else (out, status)


def _radii_arg(radii, P, nq):
    radii = radii.to(torch.float64).contiguous()
    if radii.dim() == 2:
        M, rstride = radii.shape[1], 0
    elif radii.dim() == 3 and radii.shape[0] == P:
        M, rstride = radii.shape[2], radii.shape[1] * radii.shape[2]
    else:
        raise ValueError("radii must be [n_meas, M] or [P, n_meas, M]")
    if radii.shape[-2] != nq:
        raise ValueError(f"radii rows {radii.shape[-2]} != n_measures(mask) = {nq}")
    return radii, M, rstride


def bin_matrix(A, B, grid, mask, radii, *, engine=ENGINE_AUTO, stream=None, ws: Workspace | None = None,
               bins=None, status=None):
    """Per-pair bin indices bins[p,q,i,j] = #{m : d_q(A_p,i, B_p,j) < R_p,q,m} (uint8), the
    first half of the bootstrap estimators (Alg. A1 / A2).

    A: [N,S,H,W] or [P,N,S,H,W] float32 CUDA (a 4-D A with 5-D B is shared by every item);
    B likewise.  radii [n_meas, M] or [P, n_meas, M].  Returns bins, item_status.
    """
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    K = S * H * W
    shareA = A.dim() in (2, 4) and B.dim() in (3, 5)
    A3, B3 = _as_items(A, K), _as_items(B, K)
    P = B3.shape[0] if shareA else A3.shape[0]
    if not shareA and B3.shape[0] != P:
        raise ValueError("A and B must have the same number of items")
    N, Nt = A3.shape[1], B3.shape[1]
    nq = n_measures(mask)
    radii, M, rstride = _radii_arg(radii, P, nq)
    dev = B3.device
    if bins is None:
        bins = torch.empty((P, nq, N, Nt), dtype=torch.uint8, device=dev)
    if status is None:
        status = torch.empty((P,), dtype=torch.int32, device=dev)
    g = _grid(grid)
    nbytes = lib.cil_bin_matrix_workspace_size(P, N, Nt, g, mask, M, engine)
    if nbytes == 0:
        raise CilError("cil_bin_matrix_workspace_size: invalid arguments or engine")
    wbuf = (ws or _default_ws).get(nbytes, dev)
    sA = 0 if shareA else A3.stride(0)
    st = lib.cil_bin_matrix(P, _ptr(A3), sA, A3.stride(1), N, _ptr(B3), B3.stride(0), B3.stride(1), Nt, g, mask,
                            radii.data_ptr(), rstride, M, bins.data_ptr(), status.data_ptr(), engine,
                            wbuf.data_ptr(), wbuf.numel(), _stream(stream))
    check(st, "cil_bin_matrix")
    return bins, status


def resample_counts(bins, I1, I2, M, *, want_counts=True, stream=None, status=None):
    """Correlation-integral vectors of resampled set pairs (Alg. A1 step 2 / Alg. A2 steps
    2.1-2.4) read off a bin matrix: bins [P, n_meas, N, Nt] uint8; I1 [P, n_rep, n1] and
    I2 [P, n_rep, n2] int32 draws (row / column indices, repetition allowed).
    Returns counts int64 [P, n_rep, n_meas, M] (or None), y float64 [P, n_rep, n_meas*M],
    item_status [P] (ITEM_BADINDEX for an index out of range)."""
    P, nq, N, Nt = bins.shape
    I1 = I1.to(torch.int32).contiguous()
    I2 = I2.to(torch.int32).contiguous()
    n_rep, n1, n2 = I1.shape[1], I1.shape[2], I2.shape[2]
    if I1.shape[0] != P or I2.shape[:2] != (P, n_rep):
        raise ValueError("I1 [P, n_rep, n1], I2 [P, n_rep, n2]")
    dev = bins.device
    counts = torch.empty((P, n_rep, nq, M), dtype=torch.int64, device=dev) if want_counts else None
    y = torch.empty((P, n_rep, nq * M), dtype=torch.float64, device=dev)
    if status is None:
        status = torch.zeros((P,), dtype=torch.int32, device=dev)
    st = lib.cil_resample_counts(P, bins.contiguous().data_ptr(), N, Nt, nq, M, n_rep, I1.data_ptr(), n1,
                                 I2.data_ptr(), n2, counts.data_ptr() if want_counts else None, y.data_ptr(), 0,
                                 status.data_ptr(), _stream(stream))
    check(st, "cil_resample_counts")
    return counts, y, status


def mcil_boot_stats(data, grid, mask, radii, I1, I2, *, engine=ENGINE_AUTO, stream=None):
    """MCIL with bootstrapping, Alg. A1: s~1 = first N_set/2 patterns of
    data, s~2 = the next N_set/2 (step 1); I1, I2 [n_rep, N_set/2] draws with replacement
    into s~1 and s~2 (step 2.1); y^k from the bin matrix (2.2-2.3); mu_0, Sigma_0 (step 3).
    Returns mu [D], Sigma [D, D], Y [n_rep, D], item_status."""
    D2 = data.reshape(data.shape[0], -1)
    h = D2.shape[0] // 2
    bins, st = bin_matrix(D2[:h].reshape((h,) + tuple(data.shape[1:])), D2[h:2 * h].reshape((h,) + tuple(data.shape[1:])),
                          grid, mask, radii, engine=engine, stream=stream)
    M = radii.shape[-1]
    _, Y, st = resample_counts(bins, I1.unsqueeze(0), I2.unsqueeze(0), M, want_counts=False, stream=stream,
                               status=st)
    mu, Sig = stats(Y[0], stream=stream)
    return mu, Sig, Y[0], st


def synth_loglik_boot(pools, data, N_set, I1, I2, J, grid, mask, radii, ridge: float = 0.0, *,
                      engine=ENGINE_AUTO, return_Y=False, stream=None, ws: Workspace | None = None, out=None,
                      status=None):
    """SCIL with bootstrapping, Alg. A2, for P proposals.

    pools [P, N_syn, S,H,W] float32; data [N_set, S,H,W]; I1 [P, n_rep, N_set],
    I2 [P, n_rep, N_syn - N_set], J [P, N_syn - N_set] int32 draws; radii [P, n_meas, M].
    Returns out [P,3] = (quad, logdet, loglik), item_status [P] (and Y [P, n_rep+1, D])."""
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    K = S * H * W
    P, N_syn = pools.shape[0], pools.shape[1]
    pools3 = pools.reshape(P, N_syn, -1)
    data2 = data.reshape(data.shape[0], -1)
    if pools3.shape[-1] != K or data2.shape[-1] != K or data2.shape[0] != N_set:
        raise ValueError("pool / data shapes do not match grid and N_set")
    nq = n_measures(mask)
    radii = radii.to(torch.float64).contiguous()
    M = radii.shape[-1]
    if radii.shape != (P, nq, M):
        raise ValueError("radii must be [P, n_meas, M]")
    I1 = I1.to(torch.int32).contiguous()
    I2 = I2.to(torch.int32).contiguous()
    J = J.to(torch.int32).contiguous()
    n_rep = I1.shape[1]
    Nt = N_syn - N_set
    if I1.shape != (P, n_rep, N_set) or I2.shape != (P, n_rep, Nt) or J.shape != (P, Nt):
        raise ValueError("I1 [P, n_rep, N_set], I2 [P, n_rep, N_syn-N_set], J [P, N_syn-N_set]")
    dev = pools.device
    if out is None:
        out = torch.empty((P, 3), dtype=torch.float64, device=dev)
    if status is None:
        status = torch.empty((P,), dtype=torch.int32, device=dev)
    Y = torch.empty((P, n_rep + 1, nq * M), dtype=torch.float64, device=dev) if return_Y else None
    g = _grid(grid)
    nbytes = lib.cil_synth_boot_workspace_size(P, N_syn, N_set, n_rep, g, mask, M, engine)
    if nbytes == 0:
        raise CilError("cil_synth_boot_workspace_size: invalid arguments or engine")
    wbuf = (ws or _default_ws).get(nbytes, dev)
    st = lib.cil_synth_loglik_boot(P, pools3.data_ptr(), pools3.stride(0), pools3.stride(1), N_syn,
                                   data2.data_ptr(), data2.stride(0), N_set, n_rep, I1.data_ptr(), I2.data_ptr(),
                                   J.data_ptr(), g, mask, radii.data_ptr(), M, float(ridge), out.data_ptr(),
                                   status.data_ptr(), Y.data_ptr() if return_Y else None, engine, wbuf.data_ptr(),
                                   wbuf.numel(), _stream(stream))
    check(st, "cil_synth_loglik_boot")
    return (out, status, Y) if return_Y else (out, status)


def diag_gram(A, B, grid, engine=ENGINE_TC_3XBF16, *, stream=None):
    """DIAGNOSTIC: per pair of one set pair, shape [N, Nt, 2] (no binning; not on the hot path):
    TC_I8 -> the engine's interval (lo, hi) of the unweighted L2 distance; TC_3XBF16 / TC_3XTF32 ->
    the FP32 d^2 and its statistical bound E."""
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    K = S * H * W
    A2, B2 = A.reshape(A.shape[0], -1).contiguous(), B.reshape(B.shape[0], -1).contiguous()
    N, Nt = A2.shape[0], B2.shape[0]
    g = _grid(grid)
    out = torch.empty((N, Nt, 2), dtype=torch.float32, device=A2.device)
    nbytes = lib.cil_features_workspace_size(1, N, Nt, g, L2, 1, engine) + 512
    wbuf = _default_ws.get(nbytes, A2.device)
    check(lib.cil_diag_gram(A2.data_ptr(), K, N, B2.data_ptr(), K, Nt, g, engine, out.data_ptr(),
                            wbuf.data_ptr(), wbuf.numel(), _stream(stream)), "cil_diag_gram")
    return out


def minmax_scale(X, grid, *, out=None, stream=None):
    """Scaled patterns: per pattern and species, (x - min) / (max - min)."""
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    K = S * H * W
    X2 = X.reshape(-1, K)
    if X2.stride(1) != 1:
        raise ValueError("patterns must be contiguous")
    Y = torch.empty_like(X2) if out is None else out.reshape(-1, K)
    check(lib.cil_minmax_scale(X2.shape[0], X2.data_ptr(), X2.stride(0), Y.data_ptr(), Y.stride(0), _grid(grid),
                               _stream(stream)), "cil_minmax_scale")
    return Y.reshape(X.shape)


def distance_range(A, B, grid, mask, *, stream=None, ws: Workspace | None = None, status=None):
    """[P, n_meas, 2] FP64: (min positive, max) distance over all pairs of each set pair
    (PAPER.md:109, 246).  A, B as in features (a 4-D A with 5-D B is shared)."""
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    K = S * H * W
    shareA = A.dim() in (2, 4) and B.dim() in (3, 5)
    A3, B3 = _as_items(A, K), _as_items(B, K)
    P = B3.shape[0] if shareA else A3.shape[0]
    N, Nt = A3.shape[1], B3.shape[1]
    nq = n_measures(mask)
    dev = B3.device
    rng = torch.empty((P, nq, 2), dtype=torch.float64, device=dev)
    if status is None:
        status = torch.empty((P,), dtype=torch.int32, device=dev)
    g = _grid(grid)
    nbytes = lib.cil_range_workspace_size(P, N, Nt, g, mask)
    if nbytes == 0:
        raise CilError("cil_range_workspace_size: invalid arguments")
    wbuf = (ws or _default_ws).get(nbytes, dev)
    check(lib.cil_distance_range(P, _ptr(A3), 0 if shareA else A3.stride(0), A3.stride(1), N, _ptr(B3), B3.stride(0),
                                 B3.stride(1), Nt, g, mask, rng.data_ptr(), status.data_ptr(), wbuf.data_ptr(),
                                 wbuf.numel(), _stream(stream)), "cil_distance_range")
    return rng, status


def radii_from_range(rng, M, law: str = "power", margin: float = 1e-3, *, stream=None, status=None):
    """Radii [P, n_meas, M] from a distance range: power law R_0 b^-m or linear
    R_0 - m h, R_0 = max (1 + margin), R_M = min (1 - margin)."""
    r = rng.to(torch.float64).contiguous()
    P, nq = r.shape[0], r.shape[1]
    radii = torch.empty((P, nq, M), dtype=torch.float64, device=r.device)
    if status is None:
        status = torch.zeros((P,), dtype=torch.int32, device=r.device)
    check(lib.cil_radii_from_range(P, nq, M, r.data_ptr(), {"power": 0, "linear": 1}[law], float(margin),
                                   radii.data_ptr(), status.data_ptr(), _stream(stream)), "cil_radii_from_range")
    return radii, status


def train_vectors(X, n_ens, grid, mask, radii, *, engine=ENGINE_AUTO, stream=None, ws: Workspace | None = None,
                  status=None):
    """Training vectors of Alg. 1 / Alg. 2: X [n_ens*N, S,H,W] or
    [P, n_ens*N, S,H,W] float32, divided into n_ens subsets of N rows; returns
    Y [P, n_ens(n_ens-1)/2, n_meas*M] for the subset pairs k < l (lexicographic) and item_status."""
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    K = S * H * W
    X3 = _as_items(X, K)
    P, rows = X3.shape[0], X3.shape[1]
    if rows % n_ens:
        raise ValueError("rows must be n_ens * N")
    N = rows // n_ens
    nq = n_measures(mask)
    radii, M, rstride = _radii_arg(radii, P, nq)
    dev = X3.device
    nv = n_ens * (n_ens - 1) // 2
    Y = torch.empty((P, nv, nq * M), dtype=torch.float64, device=dev)
    if status is None:
        status = torch.empty((P,), dtype=torch.int32, device=dev)
    g = _grid(grid)
    nbytes = lib.cil_train_workspace_size(P, n_ens, N, g, mask, M, engine)
    if nbytes == 0:
        raise CilError("cil_train_workspace_size: invalid arguments")
    wbuf = (ws or _default_ws).get(nbytes, dev)
    check(lib.cil_train_vectors(P, X3.data_ptr(), X3.stride(0), X3.stride(1), n_ens, N, g, mask, radii.data_ptr(),
                                rstride, M, Y.data_ptr(), status.data_ptr(), engine, wbuf.data_ptr(), wbuf.numel(),
                                _stream(stream)), "cil_train_vectors")
    return Y, status


def gaussianity_chi2(Y, *, bins: int = 10, ridge: float = 0.0, stream=None):
    """Numerical Gaussianity check of CIL vectors: the squared Mahalanobis
    distances d_k^2 = (y_k - mu)^T Sigma^-1 (y_k - mu) of the n vectors (cil_stats + cil_loglik) and
    Pearson's statistic over `bins` equiprobable chi^2_D bins (cil_gaussianity_pearson), all on the
    device.  Returns (statistic, degrees of freedom, d2 [n] on the device)."""
    Y2 = Y.to(torch.float64).contiguous()
    n, D = Y2.shape
    mu, Sig = stats(Y2, stream=stream)
    out, _ = loglik(mu, Sig, Y2, ridge, stream=stream)
    d2 = out[:, 0].contiguous()
    res = torch.empty(2, dtype=torch.float64, device=Y2.device)
    check(lib.cil_gaussianity_pearson(n, d2.data_ptr(), D, bins, res.data_ptr(), _stream(stream)),
          "cil_gaussianity_pearson")
    r = res.cpu()
    return float(r[0]), int(r[1]), d2


def diag_gram_family(A, B, grid, *, stream=None):
    """DIAGNOSTIC: the three-phase INT8 engine's intervals (lo, hi) for every pair of one set pair,
    shape [3, N, Nt, 2] for (L2/sqrt(w), W12^2/w, W12SUM/sqrt(w)).  Not on the hot path."""
    S, H, W = int(grid[0]), int(grid[1]), int(grid[2])
    K = S * H * W
    A2, B2 = A.reshape(A.shape[0], -1).contiguous(), B.reshape(B.shape[0], -1).contiguous()
    N, Nt = A2.shape[0], B2.shape[0]
    g = _grid(grid)
    out = torch.empty((3, N, Nt, 2), dtype=torch.float32, device=A2.device)
    nbytes = lib.cil_features_workspace_size(1, N, Nt, g, L2 | W12SUM | W12, 1, ENGINE_TC_I8) + 512
    wbuf = _default_ws.get(nbytes, A2.device)
    check(lib.cil_diag_gram_family(A2.data_ptr(), K, N, B2.data_ptr(), K, Nt, g, out.data_ptr(), wbuf.data_ptr(),
                                   wbuf.numel(), _stream(stream)), "cil_diag_gram_family")
    return out


def last_launch_count() -> int:
    """Kernel launches issued by the last library call on this thread."""
    return int(lib.cil_last_launch_count())
