"""GPU parity on seeded random shapes: the CUDA path (through the C ABI) against the FP64 oracle.

Each case draws (from a fixed seed) a grid S x H x W (1-D and 2-D, K a multiple of 4 as cil.h
requires), ragged N / Nt around the 128- and 256-row tile edges, P items, a measure mask, M radii
(1..64, i.e. every MAXM instantiation), a generator profile (GM, FHN, min-max scaled, PAPER.md:
451-456), shared or per-item radii, and an engine.  Counts must lie in the oracle's band
(strict <, Eq. (1); north-star band 1e-6) and y must equal counts / (N Nt)
exactly; SCIL (Alg. 3) must give every row of its count matrix Y within the
oracle's band, the log-likelihood within 1e-6 of the oracle's tail on that Y, and of the oracle's
whole Alg. 3 when the two Y agree; the bin matrix (Alg. A1 / A2) must give #{m : d < R_m} up to the
same band.  The point is the shapes nobody picked by hand: ragged tails in every dimension.
"""
import os

import numpy as np
import pytest
import torch

import cilgen

pytestmark = pytest.mark.gpu

BAND = 1e-6
ENGINES = ["SIMT", "TC_3XBF16", "TC_3XTF32", "TC_I8", "AUTO"]
PROFILES = ["GM", "FHN", "scaled"]
EDGE_ROWS = [1, 2, 31, 63, 64, 65, 127, 128, 129, 191, 255, 256, 257]


def _cases(start, n):
    """Case numbers of one fuzz family: start .. start + n - 1, plus (CIL_FUZZ_ROUNDS = R > 1, a
    longer soak run) R - 1 further blocks of fresh draws at k * 100000 + start, k = 1 .. R - 1."""
    rounds = max(1, int(os.environ.get("CIL_FUZZ_ROUNDS", "1")))
    return [k * 100000 + c for k in range(rounds) for c in range(start, start + n)]


@pytest.fixture(scope="module")
def cil():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2203_14742_b200 as cil
    return cil


def _draw_case(case):
    r = np.random.default_rng(20314742 + 1000 * case)
    while True:
        S = int(r.integers(1, 4))
        H = 1 if r.random() < 0.3 else int(r.integers(2, 40))
        W = int(r.integers(2, 72))
        if (S * H * W) % 4 == 0 and S * H * W <= 6000:
            break
    rows = lambda: int(r.choice(EDGE_ROWS)) if r.random() < 0.5 else int(r.integers(1, 300))
    N, Nt = rows(), rows()
    while N * Nt > 40000:                        # the oracle's budget per item
        N, Nt = max(1, N // 2), max(1, Nt // 2)
    P = int(r.integers(1, 4))
    mask = int(r.integers(1, 64))
    M = int(r.choice([1, 2, 7, 15, 16, 17, 31, 32, 33, 64]))
    profile = str(r.choice(PROFILES))
    per_item = bool(r.random() < 0.5) and P > 1
    engine = ENGINES[case % len(ENGINES)]
    lo_q, hi_q = float(r.uniform(0.0, 0.2)), float(r.uniform(0.8, 1.0))
    return dict(grid=(S, H, W, 0.0), N=N, Nt=Nt, P=P, mask=mask, M=M, profile=profile,
                per_item=per_item, engine=engine, lo_q=lo_q, hi_q=hi_q, seed=777 + case)


def _sets(c):
    prof = "GM" if c["profile"] == "scaled" else c["profile"]
    sc = c["profile"] == "scaled"
    A = torch.stack([cilgen.make_set(c["seed"], 2 * p, c["N"], c["grid"][:3], prof, scaled=sc)
                     for p in range(c["P"])])
    B = torch.stack([cilgen.make_set(c["seed"], 2 * p + 1, c["Nt"], c["grid"][:3], prof, scaled=sc)
                     for p in range(c["P"])])
    return A, B


def _radii(D, M, lo_q, hi_q):
    """Power-law radii R_0 b^-m over a quantile range of the distances."""
    out = []
    for q in range(D.shape[0]):
        d = D[q].ravel()
        R0 = max(np.quantile(d, hi_q) * 1.001, 1e-9)
        RM = min(max(np.quantile(d, lo_q) * 0.999, 1e-12), R0 * 0.5)
        out.append(R0 * (RM / R0) ** (np.arange(1, M + 1) / M))
    return np.array(out)


@pytest.mark.parametrize("case", _cases(0, 100))
def test_fuzz_features(cil, oracle_mod, case):
    O = oracle_mod
    c = _draw_case(case)
    grid, mask, M = c["grid"], c["mask"], c["M"]
    A, B = _sets(c)
    Ds = [O.distance_matrix(A[p].numpy(), B[p].numpy(), grid, mask) for p in range(c["P"])]
    if c["per_item"]:
        radii = np.stack([_radii(D, M, c["lo_q"], c["hi_q"]) for D in Ds])
    else:
        radii = _radii(Ds[0], M, c["lo_q"], c["hi_q"])
    dev = torch.device("cuda")
    counts, y, st = cil.features(A.to(dev), B.to(dev), grid, mask, torch.tensor(radii, device=dev),
                                 engine=getattr(cil, "ENGINE_" + c["engine"]))
    torch.cuda.synchronize()
    counts, y, st = counts.cpu().numpy(), y.cpu().numpy(), st.cpu().numpy()
    assert np.all(st == 0), (c, st.tolist())
    for p in range(c["P"]):
        R = radii[p] if c["per_item"] else radii
        ref = O.features(A[p].numpy(), B[p].numpy(), grid, mask, R, band=BAND)
        ok = np.all(ref["lo"] <= counts[p]) and np.all(counts[p] <= ref["hi"])
        assert ok, (c, p, counts[p].tolist(), ref["lo"].tolist(), ref["hi"].tolist())
        np.testing.assert_array_equal(y[p], counts[p] / float(c["N"] * c["Nt"]))


@pytest.mark.parametrize("case", _cases(100, 30))
def test_fuzz_bin_matrix(cil, oracle_mod, case):
    O = oracle_mod
    c = _draw_case(case)
    c["M"] = min(c["M"], 32)
    c["engine"] = ["SIMT", "TC_I8", "AUTO"][case % 3]          # cil.h: bins refuse the 3x engines
    grid, mask, M = c["grid"], c["mask"], c["M"]
    A, B = _sets(c)
    Ds = [O.distance_matrix(A[p].numpy(), B[p].numpy(), grid, mask) for p in range(c["P"])]
    radii = _radii(Ds[0], M, c["lo_q"], c["hi_q"])
    dev = torch.device("cuda")
    bins, st = cil.bin_matrix(A.to(dev), B.to(dev), grid, mask, torch.tensor(radii, device=dev),
                              engine=getattr(cil, "ENGINE_" + c["engine"]))
    torch.cuda.synchronize()
    bins, st = bins.cpu().numpy().astype(np.int64), st.cpu().numpy()
    assert np.all(st == 0), (c, st.tolist())
    for p in range(c["P"]):
        D = Ds[p]
        for q in range(D.shape[0]):
            lo = (D[q][..., None] < radii[q] * (1 - BAND)).sum(-1)
            hi = (D[q][..., None] < radii[q] * (1 + BAND)).sum(-1)
            g = bins[p, q]
            bad = (g < lo) | (g > hi)
            assert not bad.any(), (c, p, q, np.argwhere(bad)[:5].tolist())


@pytest.mark.parametrize("case", _cases(200, 24))
def test_fuzz_synth(cil, oracle_mod, case):
    O = oracle_mod
    c = _draw_case(case)
    r = np.random.default_rng(4242 + case)
    grid, mask = c["grid"], c["mask"]
    nq = O.n_measures(mask)
    P = c["P"]
    n_ens = int(r.integers(2, 6))
    N_set, Nt = int(r.integers(1, 40)), int(r.integers(1, 60))
    M = int(r.integers(1, min(64, 192 // nq) + 1))
    Nsyn = n_ens * (N_set + Nt) + int(r.integers(0, 5))
    prof = "GM" if c["profile"] == "scaled" else c["profile"]
    sc = c["profile"] == "scaled"
    pools = torch.stack([cilgen.make_set(c["seed"], 100 + p, Nsyn, grid[:3], prof, scaled=sc) for p in range(P)])
    data = cilgen.make_set(c["seed"], 999, N_set, grid[:3], prof, scaled=sc)
    k0 = r.integers(0, n_ens, size=P).astype(np.int32)
    radii = []
    for p in range(P):
        Dp = O.distance_matrix(pools[p].numpy(), pools[p].numpy(), grid, mask)
        Dp = np.where(Dp > 0, Dp, np.nan)
        radii.append(np.array([np.geomspace(np.nanquantile(d, 0.97), np.nanquantile(d, 0.05), M + 1)[:M]
                               if M > 1 else [np.nanquantile(d, 0.5)] for d in Dp]))
    radii = np.array(radii)
    dev = torch.device("cuda")
    out, st, Y = cil.synth_loglik(pools.to(dev), n_ens, N_set, Nt, data.to(dev), torch.tensor(k0, device=dev),
                                  grid, mask, torch.tensor(radii, device=dev), ridge=1e-3,
                                  engine=getattr(cil, "ENGINE_" + c["engine"]), return_Y=True)
    torch.cuda.synchronize()
    N = N_set + Nt
    for p in range(P):
        if not all(np.all(R > 0) and np.all(np.diff(R) < 0) for R in radii[p]):
            # a degenerate draw (e.g. min-max-scaled 2-node grids: every distance of a measure equal)
            # gives constant radii, which cil.h:23 rejects per item; the oracle takes them as given
            assert st[p].item() & cil.ITEM_BADRADII, (c, p, st[p].item())
            continue
        ref, rst, Yr = O.synth_loglik(pools[p].numpy(), n_ens, N_set, Nt, data.numpy(), int(k0[p]), grid, mask,
                                      radii[p], ridge=1e-3)
        Yg = Y[p].cpu().numpy()
        assert rst == st[p].item(), (c, p, rst, st[p].item())
        if not np.array_equal(Yg, Yr):
            # only pairs within the band of a radius may differ: each row of Y within its band counts
            pool = pools[p].numpy()
            for v in range(n_ens * n_ens + 1):
                k, l = divmod(v, n_ens)
                s1 = pool[k * N:k * N + N_set] if v < n_ens * n_ens else data.numpy()
                s2 = pool[(l if v < n_ens * n_ens else int(k0[p])) * N + N_set:][:Nt]
                b = O.features(s1, s2, grid, mask, radii[p], band=BAND)
                y = np.rint(Yg[v].reshape(nq, -1) * (N_set * Nt))
                assert np.all(b["lo"] <= y) and np.all(y <= b["hi"]), (c, p, v)
        # the tail (mu, Sigma, Cholesky log-density) on the GPU's own count matrix
        mu, Sig = O.stats(Yg[:-1])
        ref2, _ = O.loglik(mu, Sig, Yg[-1], ridge=1e-3)
        if rst == 0:
            np.testing.assert_allclose(out[p].cpu().numpy(), ref2, rtol=0, atol=1e-6, err_msg=str(c))
            if np.array_equal(Yg, Yr):
                np.testing.assert_allclose(out[p].cpu().numpy(), ref, rtol=0, atol=1e-6, err_msg=str(c))


@pytest.mark.parametrize("case", _cases(300, 16))
def test_fuzz_train_vectors(cil, oracle_mod, case):
    """Alg. 1 / Alg. 2 training vectors on random shapes: the k < l
    subset blocks of one panel, each within the oracle's band counts."""
    O = oracle_mod
    c = _draw_case(case)
    r = np.random.default_rng(5151 + case)
    grid, mask, M = c["grid"], c["mask"], c["M"]
    n_ens = int(r.integers(2, 7))
    N = int(r.integers(1, 80))
    X = torch.stack([cilgen.make_set(c["seed"], p, n_ens * N, grid[:3]) for p in range(c["P"])])
    D = O.distance_matrix(X[0].numpy(), X[0].numpy(), grid, mask)
    radii = _radii(D, M, c["lo_q"], c["hi_q"])
    dev = torch.device("cuda")
    Y, st = cil.train_vectors(X.to(dev), n_ens, grid, mask, torch.tensor(radii, device=dev),
                              engine=getattr(cil, "ENGINE_" + c["engine"]))
    torch.cuda.synchronize()
    assert np.all(st.cpu().numpy() == 0), c
    for p in range(c["P"]):
        ref = O.train_vectors(X[p].numpy(), n_ens, grid, mask, radii, band=BAND)
        got = np.rint(Y[p].cpu().numpy() * N * N).astype(np.int64).reshape(ref["lo"].shape)
        assert np.all(ref["lo"] <= got) and np.all(got <= ref["hi"]), (c, p, n_ens, N)


@pytest.mark.parametrize("case", _cases(400, 16))
def test_fuzz_distance_range_and_radii(cil, oracle_mod, case):
    """(min positive, max) distance per measure (reading R16) and the radii laws
    on random shapes, including sets that share rows (zero distances excluded from the minimum)."""
    O = oracle_mod
    c = _draw_case(case)
    grid, mask = c["grid"], c["mask"]
    A, B = _sets(c)
    B[:, : min(c["N"], c["Nt"]) // 2] = A[:, : min(c["N"], c["Nt"]) // 2]
    dev = torch.device("cuda")
    rng, st = cil.distance_range(A.to(dev), B.to(dev), grid, mask)
    law = ["power", "linear"][case % 2]
    radii, st1 = cil.radii_from_range(rng, c["M"], law)
    torch.cuda.synchronize()
    rng, radii = rng.cpu().numpy(), radii.cpu().numpy()
    for p in range(c["P"]):
        ref = O.distance_range(A[p].numpy(), B[p].numpy(), grid, mask)
        np.testing.assert_allclose(rng[p], ref, rtol=1e-6, atol=0, err_msg=str(c))
        if np.all(np.isfinite(ref)) and np.all(ref[:, 0] > 0):
            np.testing.assert_allclose(radii[p], O.radii_from_range(rng[p], c["M"], law), rtol=1e-12,
                                       err_msg=str(c))


@pytest.mark.parametrize("case", _cases(500, 12))
def test_fuzz_synth_boot(cil, oracle_mod, case):
    """Alg. A2 on random shapes and draws: replicate vectors within the band
    (resampled sets built explicitly by the oracle), the tail within 1e-6."""
    O = oracle_mod
    c = _draw_case(case)
    r = np.random.default_rng(6161 + case)
    grid, mask = c["grid"], c["mask"]
    nq = O.n_measures(mask)
    P = c["P"]
    N_set = int(r.integers(1, 30))
    N_syn = N_set + int(r.integers(1, 90))
    n_rep = int(r.integers(2, 40))
    M = int(r.integers(1, min(64, 192 // nq) + 1))
    pools = torch.stack([cilgen.make_set(c["seed"], 100 + p, N_syn, grid[:3]) for p in range(P)])
    data = cilgen.make_set(c["seed"], 999, N_set, grid[:3])
    radii, draws = [], []
    for p in range(P):
        D = O.distance_matrix(pools[p].numpy(), pools[p].numpy(), grid, mask)
        radii.append(_radii(D, M, c["lo_q"], c["hi_q"]))
        draws.append(cilgen.boot_draws_a2(c["seed"], p, n_rep, N_syn, N_set))
    radii = np.array(radii)
    I1, I2, J = (np.stack([d[i] for d in draws]) for i in range(3))
    dev = torch.device("cuda")
    engine = ["SIMT", "TC_I8", "AUTO"][case % 3]
    out, st, Y = cil.synth_loglik_boot(pools.to(dev), data.to(dev), N_set, torch.tensor(I1, device=dev),
                                       torch.tensor(I2, device=dev), torch.tensor(J, device=dev), grid, mask,
                                       torch.tensor(radii, device=dev), ridge=1e-3,
                                       engine=getattr(cil, "ENGINE_" + engine), return_Y=True)
    torch.cuda.synchronize()
    for p in range(P):
        ref, rst, Yr = O.synth_boot(pools[p].numpy(), data.numpy(), N_set, I1[p], I2[p], J[p], grid, mask,
                                    radii[p], ridge=1e-3)
        Yg = Y[p].cpu().numpy()
        rr = O.resample_features(pools[p].numpy(), pools[p].numpy(), grid, mask, radii[p], I1[p], I2[p], band=BAND)
        cnt = np.rint(Yg[:-1] * (N_set * (N_syn - N_set))).astype(np.int64).reshape(rr["lo"].shape)
        assert np.all(rr["lo"] <= cnt) and np.all(cnt <= rr["hi"]), (c, p)
        assert rst == st[p].item() or not np.array_equal(Yg, Yr), (c, p, rst, st[p].item())
        if st[p].item() == 0:
            mu, Sig = O.stats(Yg[:-1])
            o2, _ = O.loglik(mu, Sig, Yg[-1], ridge=1e-3)
            np.testing.assert_allclose(out[p].cpu().numpy(), o2, rtol=0, atol=1e-6, err_msg=str(c))
            if np.array_equal(Yg, Yr):
                np.testing.assert_allclose(out[p].cpu().numpy(), ref, rtol=0, atol=1e-6, err_msg=str(c))


@pytest.mark.parametrize("case", _cases(600, 10))
def test_fuzz_large_K(cil, oracle_mod, case):
    """Long patterns (K up to ~150 k: the INT8 engines' 65536-element chunks, ragged in K) with
    few rows, all six measures on some cases, against the oracle's band counts."""
    O = oracle_mod
    r = np.random.default_rng(7070 + case)
    while True:
        S, H, W = int(r.integers(1, 4)), int(r.integers(1, 300)), int(r.integers(2, 300))
        K = S * H * W
        if K % 4 == 0 and 20000 <= K <= 150000:
            break
    grid = (S, H, W, 0.0)
    N, Nt = int(r.integers(1, 140)), int(r.integers(1, 140))
    mask = 0x3F if case % 2 == 0 else int(r.integers(1, 64))
    M = int(r.choice([5, 16, 20, 33]))
    engine = ENGINES[case % len(ENGINES)]
    A = cilgen.make_set(case, 0, N, grid[:3], "FHN" if case % 3 == 0 else "GM")
    B = cilgen.make_set(case, 1, Nt, grid[:3], "FHN" if case % 3 == 0 else "GM")
    D = O.distance_matrix(A.numpy(), B.numpy(), grid, mask)
    radii = _radii(D, M, 0.05, 0.95)
    dev = torch.device("cuda")
    counts, y, st = cil.features(A.to(dev), B.to(dev), grid, mask, torch.tensor(radii, device=dev),
                                 engine=getattr(cil, "ENGINE_" + engine))
    torch.cuda.synchronize()
    assert int(st[0]) == 0, (grid, N, Nt, mask, M, engine)
    ref = O.features(A.numpy(), B.numpy(), grid, mask, radii, band=BAND)
    got = counts[0].cpu().numpy()
    assert np.all(ref["lo"] <= got) and np.all(got <= ref["hi"]), (grid, N, Nt, hex(mask), M, engine)
