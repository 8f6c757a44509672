"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle on the same
seeded inputs.  Tolerances (north star, BASELINE.json):
  counts  bit-exact except (pair, radius) cases within 1e-6 relative of a radius:
          the oracle's band counts give lo <= gpu <= hi (== when nothing is ambiguous);
  mu, Sigma within 1e-6 relative (normwise, on the same count vectors);
  loglik within 1e-6 absolute.
"""
import numpy as np
import pytest
import torch

import cilgen

pytestmark = pytest.mark.gpu

BAND = 1e-6
ENGINES = ["SIMT", "TC_3XBF16", "TC_3XTF32", "TC_I8", "AUTO"]


@pytest.fixture(scope="module")
def cil():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2203_14742_b200 as cil
    return cil


def _engine(cil, name):
    return getattr(cil, "ENGINE_" + name)


def _radii_from(D, M, lo_q=0.0, hi_q=1.0):
    """Power-law radii R_0 b^-m spanning the distance range."""
    out = []
    for q in range(D.shape[0]):
        d = D[q].ravel()
        R0, RM = np.quantile(d, hi_q) * 1.001, max(np.quantile(d, lo_q) * 0.999, 1e-12)
        out.append(R0 * (RM / R0) ** (np.arange(1, M + 1) / M))
    return np.array(out)


def _check_counts(gpu, ref):
    gpu = np.asarray(gpu)
    ok = np.all(ref["lo"] <= gpu) and np.all(gpu <= ref["hi"])
    assert ok, f"gpu {gpu.tolist()}\noracle {ref['counts'].tolist()}\nlo {ref['lo'].tolist()}\nhi {ref['hi'].tolist()}"


def _sel(D, mask):
    return D[[q for q in range(6) if (mask >> q) & 1]]


def _run_features(cil, A, B, grid, mask, radii, engine):
    dev = torch.device("cuda")
    counts, y, st = cil.features(A.to(dev), B.to(dev), grid, mask, torch.tensor(radii, device=dev),
                                 engine=_engine(cil, engine))
    torch.cuda.synchronize()
    return counts.cpu().numpy(), y.cpu().numpy(), st.cpu().numpy()


# ------------------------------------------------------------------ features
@pytest.mark.parametrize("engine", ENGINES)
def test_c1_all_measures(cil, oracle_mod, engine):
    O = oracle_mod
    grid = (1, 32, 32, 0.0)
    seed = cilgen.config_seed(1)
    A = cilgen.make_set(seed, 0, 20, grid[:3])
    B = cilgen.make_set(seed, 1, 20, grid[:3])
    D = O.distance_matrix(A.numpy(), B.numpy(), grid, 0x3F)
    radii = _radii_from(D, 10)
    ref = O.features(A.numpy(), B.numpy(), grid, 0x3F, radii, band=BAND)
    c, y, st = _run_features(cil, A, B, grid, 0x3F, radii, engine)
    assert st[0] == 0
    _check_counts(c[0], ref)
    np.testing.assert_array_equal(y[0], c[0] / 400.0)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("mask", [0x3F, 0x1, 0x2, 0x0C, 0x30, 0x09])
def test_ragged_batched(cil, oracle_mod, engine, mask):
    """P = 3 items, ragged N/Nt spanning several tiles, two species, non-square grid."""
    O = oracle_mod
    grid = (2, 10, 12, 0.0)
    P, N, Nt = 3, 37, 70
    A = torch.stack([cilgen.make_set(5, 2 * p, N, grid[:3]) for p in range(P)])
    B = torch.stack([cilgen.make_set(5, 2 * p + 1, Nt, grid[:3]) for p in range(P)])
    D0 = _sel(O.distance_matrix(A[0].numpy(), B[0].numpy(), grid, 0x3F), mask)
    radii = _radii_from(D0, 13, 0.02, 0.98)
    c, y, st = _run_features(cil, A, B, grid, mask, radii, engine)
    assert np.all(st == 0)
    for p in range(P):
        ref = O.features(A[p].numpy(), B[p].numpy(), grid, mask, radii, band=BAND)
        _check_counts(c[p], ref)
        np.testing.assert_array_equal(y[p], c[p] / (N * Nt))


@pytest.mark.parametrize("engine", ENGINES)
def test_per_item_radii_and_1d(cil, oracle_mod, engine):
    O = oracle_mod
    grid = (2, 1, 64, 0.0)                 # 1-D grid (MC / RD-ODE rows of Table 1)
    P, N, Nt = 2, 33, 29
    A = torch.stack([cilgen.make_set(9, 10 + p, N, grid[:3]) for p in range(P)])
    B = torch.stack([cilgen.make_set(9, 20 + p, Nt, grid[:3]) for p in range(P)])
    mask = 0x3F
    radii = np.stack([_radii_from(O.distance_matrix(A[p].numpy(), B[p].numpy(), grid, mask), 7, 0.05, 0.95)
                      for p in range(P)])
    c, y, st = _run_features(cil, A, B, grid, mask, radii, engine)
    for p in range(P):
        ref = O.features(A[p].numpy(), B[p].numpy(), grid, mask, radii[p], band=BAND)
        _check_counts(c[p], ref)


def test_explicit_h_and_symmetry(cil, oracle_mod):
    O = oracle_mod
    grid = (1, 16, 16, 0.37)
    A = cilgen.make_set(3, 0, 25, grid[:3])
    D = O.distance_matrix(A.numpy(), A.numpy(), grid, 0x3F)
    radii = np.array([np.geomspace(D[q][D[q] > 0].max() * 1.001, D[q][D[q] > 0].min() * 0.999, 9)
                      for q in range(6)])
    ref = O.features(A.numpy(), A.numpy(), grid, 0x3F, radii, band=BAND)
    for eng in ENGINES:
        c, y, st = _run_features(cil, A, A, grid, 0x3F, radii, eng)
        _check_counts(c[0], ref)


def test_edge_cases(cil):
    dev = torch.device("cuda")
    grid = (1, 8, 8, 0.0)
    A = cilgen.make_set(1, 0, 5, grid[:3]).to(dev)
    B = cilgen.make_set(1, 1, 4, grid[:3]).to(dev)
    radii = torch.tensor([[100.0, 1.0, 0.01]] * 6, dtype=torch.float64, device=dev)
    for eng in ENGINES:
        e = _engine(cil, eng)
        # empty A
        c, y, st = cil.features(A[:0], B, grid, 0x3F, radii, engine=e)
        assert c.abs().sum().item() == 0 and y.abs().sum().item() == 0 and st.item() == 0
        # single pair; R huge -> counted, tiny -> not
        c, y, st = cil.features(A[:1], B[:1], grid, 0x3F, radii, engine=e)
        assert c[0, :, 0].tolist() == [1] * 6 and c[0, :, 2].tolist() == [0] * 6
        # bad radii (not decreasing) -> device status, no crash
        bad = radii.clone()
        bad[0, 2] = 5.0
        c, y, st = cil.features(A, B, grid, 0x3F, bad, engine=e)
        torch.cuda.synchronize()
        assert st.item() & cil.ITEM_BADRADII
        # non-finite input
        A2 = A.clone()
        A2[2, 0, 3, 3] = float("nan")
        c, y, st = cil.features(A2, B, grid, 0x3F, radii, engine=e)
        torch.cuda.synchronize()
        assert st.item() & cil.ITEM_NONFINITE


def test_translation_invariance_tc(cil):
    """Adding a constant field to every pattern must not change counts (pins the centring)."""
    dev = torch.device("cuda")
    grid = (2, 16, 16, 0.0)
    A = cilgen.make_set(4, 0, 40, grid[:3]).to(dev)
    B = cilgen.make_set(4, 1, 50, grid[:3]).to(dev)
    radii = torch.tensor([np.geomspace(40.0, 5.0, 12)], dtype=torch.float64, device=dev)
    base = None
    for shift in (0.0, 16.0, -64.0):
        for eng in ENGINES:
            c, _, _ = cil.features(A + shift, B + shift, grid, 0x1, radii, engine=_engine(cil, eng))
            if base is None:
                base = c.clone()
            assert torch.equal(c, base), (shift, eng)


def _bound_case(case, seed):
    """(A, B, grid) of the error-bound tests; 'neardup*' are near-duplicate pairs."""
    if case == "C2":
        grid, N, Nt, shift = (2, 64, 64, 0.0), 128, 500, 0.0
    elif case == "C4":
        grid, N, Nt, shift = (1, 128, 128, 0.0), 96, 300, 0.0
    elif case == "C1":
        grid, N, Nt, shift = (1, 32, 32, 0.0), 20, 20, 0.0
    elif case == "1D":
        grid, N, Nt, shift = (2, 1, 64, 0.0), 60, 90, 0.0
    elif case.startswith("neardup"):
        grid = (2, 64, 64, 0.0)
        eps = {"neardup0": 0.0, "neardup6": 1e-6, "neardup3": 1e-3}[case]
        A = cilgen.make_set(seed, 0, 64, grid[:3], "FHN")
        rng = np.random.default_rng(seed)
        B = (A.double() + eps * torch.from_numpy(rng.standard_normal(tuple(A.shape)))).float()
        return A, torch.cat([B, cilgen.make_set(seed, 1, 64, grid[:3], "FHN")]), grid
    else:
        grid, N, Nt, shift = (2, 32, 32, 0.0), 100, 300, 50.0     # large common offset: centring stress
    A = cilgen.make_set(seed, 0, N, grid[:3]) + shift
    B = cilgen.make_set(seed, 1, Nt, grid[:3]) + shift
    return A, B, grid


def test_sqrt_approx_exhaustive(cil):
    """The INT8 engine evaluates sqrt with the hardware approximation and inflates by 2^-21
    (gram3.cu); over EVERY normal positive FP32 input its relative error must stay below that."""
    from paper_2203_14742_b200 import _capi
    up, dn = _capi.sqrt_approx_error()
    print(f"sqrt.approx.f32: max rel error above {up:.3e}, below {dn:.3e} (2^-22 = {2.0 ** -22:.3e})")
    assert up < 2.0 ** -22 and dn < 2.0 ** -22


@pytest.mark.parametrize("case", ["C2", "C4", "offset", "C1", "neardup0", "neardup6", "neardup3"])
def test_gram_error_bound_i8(cil, oracle_mod, case):
    """The INT8 engine's per-pair interval [lo, hi] of the (unweighted) L2 distance must contain the
    exact FP64 distance for EVERY pair — worst-case bound, near-duplicates included (R13)."""
    O = oracle_mod
    dev = torch.device("cuda")
    A, B, grid = _bound_case(case, 31)
    iv = cil.diag_gram(A.to(dev), B.to(dev), grid, cil.ENGINE_TC_I8).cpu().numpy().astype(np.float64)
    h = 1.0 / (grid[2] - 1)
    w = h * h
    exact = O.distance_matrix(A.numpy(), B.numpy(), grid, 0x1)[0] / np.sqrt(w)
    lo, hi = iv[..., 0], iv[..., 1]
    assert np.all(lo <= exact) and np.all(exact <= hi), (np.argwhere(~((lo <= exact) & (exact <= hi)))[:5],)
    pos = exact > 0
    print(f"{case}: median (hi-lo)/d = {np.median((hi - lo)[pos] / exact[pos]):.3e}, "
          f"max = {((hi - lo)[pos] / exact[pos]).max():.3e}")


@pytest.mark.parametrize("engine", ["TC_3XBF16", "TC_3XTF32"])
@pytest.mark.parametrize("case", ["C2", "C4", "offset", "C1"])
def test_gram_error_bound(cil, oracle_mod, engine, case):
    """The float split engines' d^2 error must stay well inside their per-pair bound E that decides
    which pairs are re-checked exactly (float split engines)."""
    O = oracle_mod
    dev = torch.device("cuda")
    A, B, grid = _bound_case(case, 31)
    d2E = cil.diag_gram(A.to(dev), B.to(dev), grid, _engine(cil, engine)).cpu().numpy().astype(np.float64)
    h = 1.0 / (grid[2] - 1)
    w = h * h
    exact = O.distance_matrix(A.numpy(), B.numpy(), grid, 0x1)[0] ** 2 / w
    err = np.abs(d2E[..., 0] - exact)
    ratio = err / d2E[..., 1]
    print(f"{case} {engine}: max err/E = {ratio.max():.3e}, max rel err d2 = {(err / exact).max():.3e}, "
          f"median E/d2 = {np.median(d2E[..., 1] / exact):.3e}")
    assert ratio.max() < 0.25


# ------------------------------------------------------------------ stats / loglik
def test_stats_loglik(cil, oracle_mod):
    O = oracle_mod
    dev = torch.device("cuda")
    rng = np.random.default_rng(0)
    P, n, D = 5, 45, 13
    Y = rng.random((P, n, D)) * 0.5 + np.linspace(0.9, 0.1, D)
    mu, Sig = cil.stats(torch.tensor(Y, device=dev))
    yo = rng.random((P, D))
    out, st = cil.loglik(mu, Sig, torch.tensor(yo, device=dev), ridge=1e-9)
    torch.cuda.synchronize()
    for p in range(P):
        mu_r, Sig_r = O.stats(Y[p])
        assert np.max(np.abs(mu[p].cpu().numpy() - mu_r)) <= 1e-6 * np.max(np.abs(mu_r))
        assert np.max(np.abs(Sig[p].cpu().numpy() - Sig_r)) <= 1e-6 * np.max(np.abs(Sig_r))
        ref, rst = O.loglik(mu[p].cpu().numpy(), Sig[p].cpu().numpy(), yo[p], ridge=1e-9)
        assert rst == st[p].item() == 0
        np.testing.assert_allclose(out[p].cpu().numpy(), ref, rtol=0, atol=1e-6)
    # shared mu / Sigma (CIL: fixed mu_0, Sigma_0 against many y(theta))
    out2, _ = cil.loglik(mu[0], Sig[0], torch.tensor(yo, device=dev), ridge=1e-9)
    for p in range(P):
        ref, _ = O.loglik(mu[0].cpu().numpy(), Sig[0].cpu().numpy(), yo[p], ridge=1e-9)
        np.testing.assert_allclose(out2[p].cpu().numpy(), ref, rtol=0, atol=1e-6)


@pytest.mark.parametrize("n,D", [(45, 384), (45, 13), (3, 700), (200, 300)])
def test_stats_large_D(cil, oracle_mod, n, D):
    """mu / Sigma for D beyond the loglik limit (6 measures x 64 radii = 384 values, the
    45 vectors of Alg. 1 with n_ens = 10) — both the shared-memory and the global kernels."""
    O = oracle_mod
    rng = np.random.default_rng(D)
    Y = rng.random((n, D)) * 0.5 + np.linspace(0.9, 0.1, D)
    mu, Sig = cil.stats(torch.tensor(Y, device="cuda"))
    mu_r, Sig_r = O.stats(Y)
    assert np.max(np.abs(mu.cpu().numpy() - mu_r)) <= 1e-6 * np.max(np.abs(mu_r))
    assert np.max(np.abs(Sig.cpu().numpy() - Sig_r)) <= 1e-6 * np.max(np.abs(Sig_r))


def test_loglik_notpd_and_large_D(cil, oracle_mod):
    O = oracle_mod
    dev = torch.device("cuda")
    v = torch.arange(1.0, 7.0, dtype=torch.float64, device=dev)
    out, st = cil.loglik(torch.zeros(6, device=dev, dtype=torch.float64), torch.outer(v, v),
                         torch.ones(6, device=dev, dtype=torch.float64))
    torch.cuda.synchronize()
    assert st.item() == cil.ITEM_NOTPD and torch.isnan(out).all()
    rng = np.random.default_rng(1)
    D = 192
    X = rng.standard_normal((D, 2 * D))
    Sig = X @ X.T / (2 * D) + 0.05 * np.eye(D)
    mu = rng.standard_normal(D)
    yo = mu + rng.standard_normal(D) * 0.3
    out, st = cil.loglik(torch.tensor(mu, device=dev), torch.tensor(Sig, device=dev), torch.tensor(yo, device=dev))
    ref, _ = O.loglik(mu, Sig, yo)
    np.testing.assert_allclose(out[0].cpu().numpy(), ref, rtol=0, atol=1e-6)


@pytest.mark.parametrize("engine", ["AUTO", "TC_I8"])
@pytest.mark.parametrize("grid,mask", [((2, 600, 600, 0.0), 0x3F), ((1, 1300, 1300, 0.0), 0x1)])
def test_very_long_rows(cil, oracle_mod, engine, grid, mask):
    """Rows beyond the INT8 Gram's 24 K-segments per launch (three-phase: 2 x 600 x 600; L2 only:
    K = 1.69 M > 24 x 65536) run on the CUDA cores and still give the oracle's counts."""
    O = oracle_mod
    A = cilgen.make_set(31, 0, 3, grid[:3])
    B = cilgen.make_set(31, 1, 4, grid[:3])
    D = O.distance_matrix(A.numpy(), B.numpy(), grid, mask)
    radii = np.array([np.sort(d.ravel())[::-1][[1, 4, 7, 10]] * np.array([1.0001, 1.0001, 0.9999, 0.9999])
                      for d in D])
    ref = O.features(A.numpy(), B.numpy(), grid, mask, radii, band=BAND)
    c, y, st = _run_features(cil, A, B, grid, mask, radii, engine)
    assert st[0] == 0
    _check_counts(c[0], ref)


@pytest.mark.parametrize("D", [1, 2, 7, 15, 31, 32, 33, 64])
def test_loglik_batched_sizes_and_notpd(cil, oracle_mod, D):
    """Eq. (4) log-density over a batch of P = 9 items (the warp-per-item kernel for D <= 32 packs 4
    items per CTA: a ragged last CTA) with per-item Sigma, two of them not positive definite."""
    O = oracle_mod
    dev = torch.device("cuda")
    rng = np.random.default_rng(100 + D)
    P = 9
    mus = rng.standard_normal((P, D))
    Sigs = []
    for p in range(P):
        X = rng.standard_normal((D, D + 3))
        S = X @ X.T / (D + 3) + 0.1 * np.eye(D)
        if p in (2, 7):                                  # indefinite: a pivot is clearly negative
            v = rng.standard_normal(D)
            S = np.outer(v, v) - 0.1 * np.eye(D) if D > 1 else -0.1 * np.eye(1)
        Sigs.append(S)
    Sigs = np.array(Sigs)
    ys = mus + 0.3 * rng.standard_normal((P, D))
    out, st = cil.loglik(torch.tensor(mus, device=dev), torch.tensor(Sigs, device=dev), torch.tensor(ys, device=dev))
    torch.cuda.synchronize()
    out, st = out.cpu().numpy(), st.cpu().numpy()
    for p in range(P):
        ref, rst = O.loglik(mus[p], Sigs[p], ys[p])
        assert st[p] == rst, (D, p, st[p], rst)
        if rst == 0:
            np.testing.assert_allclose(out[p], ref, rtol=0, atol=1e-6 * max(1.0, abs(ref[2]) / 1e3))
        else:
            assert st[p] == cil.ITEM_NOTPD and np.isnan(out[p]).all()


# ------------------------------------------------------------------ SCIL
@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("mask", [0x1, 0x0B])
def test_synth_small(cil, oracle_mod, engine, mask):
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (1, 12, 12, 0.0)
    P, n_ens, N_set, Nt = 3, 4, 5, 7
    Nsyn = n_ens * (N_set + Nt)
    pools = torch.stack([cilgen.make_set(21, 100 + p, Nsyn, grid[:3], n_w=4.5 + 0.3 * p) for p in range(P)])
    data = cilgen.make_set(21, 999, N_set, grid[:3])
    k0 = np.array([1, 3, 0], np.int32)
    radii = []
    for p in range(P):
        Dp = _sel(O.distance_matrix(pools[p].numpy(), pools[p].numpy(), grid, 0x3F), mask)
        Dp = np.where(Dp > 0, Dp, np.nan)
        radii.append(np.array([np.geomspace(np.nanquantile(d, 0.97), np.nanquantile(d, 0.1), 6) for d in Dp]))
    radii = np.array(radii)
    out, st, Y = cil.synth_loglik(pools.to(dev), n_ens, N_set, Nt, data.to(dev), torch.tensor(k0, device=dev),
                                  grid, mask, torch.tensor(radii, device=dev), ridge=1e-4,
                                  engine=_engine(cil, engine), return_Y=True)
    torch.cuda.synchronize()
    for p in range(P):
        ref, rst, Yr = O.synth_loglik(pools[p].numpy(), n_ens, N_set, Nt, data.numpy(), int(k0[p]), grid, mask,
                                      radii[p], ridge=1e-4)
        Yg = Y[p].cpu().numpy()
        # any count difference must come from ambiguous pairs; with these radii there are none
        np.testing.assert_array_equal(Yg, Yr)
        assert rst == st[p].item()
        np.testing.assert_allclose(out[p].cpu().numpy(), ref, rtol=0, atol=1e-6)


# ------------------------------------------------------------------ full-size configs (sampled)
@pytest.mark.parametrize("engine", ["TC_I8", "TC_3XBF16", "SIMT"])
def test_c2_full_item_vs_oracle(cil, oracle_mod, engine):
    """One full C2 item (500 x 500, 64x64x2, L2, M = 15) in the batched launch the bench times."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 64, 64, 0.0)
    seed = cilgen.config_seed(2)
    P = 4
    A = torch.stack([cilgen.make_set(seed, 2 * p, 500, grid[:3], device=dev) for p in range(P)])
    B = torch.stack([cilgen.make_set(seed, 2 * p + 1, 500, grid[:3], device=dev) for p in range(P)])
    a0, b0 = A[0, :64].cpu().numpy(), B[0, :64].cpu().numpy()
    radii = _radii_from(O.distance_matrix(a0, b0, grid, 0x1), 15)
    c, y, st = cil.features(A, B, grid, 0x1, torch.tensor(radii, device=dev), engine=_engine(cil, engine))
    torch.cuda.synchronize()
    ref = O.features(A[0].cpu().numpy(), B[0].cpu().numpy(), grid, 0x1, radii, band=BAND)
    _check_counts(c[0].cpu().numpy(), ref)
    # additivity over row blocks (holds at any size): item 1 counts = sum of two halves
    c1, _, _ = cil.features(A[1:2, :217], B[1:2], grid, 0x1, torch.tensor(radii, device=dev),
                            engine=_engine(cil, engine))
    c2, _, _ = cil.features(A[1:2, 217:], B[1:2], grid, 0x1, torch.tensor(radii, device=dev),
                            engine=_engine(cil, engine))
    assert torch.equal(c1[0] + c2[0], c[1])
    yy = y.cpu().numpy()
    assert np.all((yy >= 0) & (yy <= 1)) and np.all(np.diff(yy, axis=-1) <= 0)


def test_c2_bench_workload_every_item_vs_oracle(cil, oracle_mod):
    """The bench's whole C2 batch (rank 0: 100 set pairs of 500 x 500, 64x64x2, L2, M = 15, the
    pilot-block power-law radii as bench.py builds them, default engine) in the one batched launch
    `bench.py` times: every item's counts within the oracle's band counts (~45 s of oracle time).
    Inputs built as bench.py builds them (same seeds)."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid, P, N = (2, 64, 64), 100, 500
    seed = cilgen.config_seed(2)
    A = torch.stack([cilgen.make_set(seed, 2 * p, N, grid, device=dev) for p in range(P)])
    B = torch.stack([cilgen.make_set(seed, 2 * p + 1, N, grid, device=dev) for p in range(P)])
    # bench.py pilot_radii: power law over the 64 x 64 pilot block of set pair 0
    a0 = cilgen.make_set(seed, 0, 64, grid).reshape(64, -1).double().numpy()
    b0 = cilgen.make_set(seed, 1, 64, grid).reshape(64, -1).double().numpy()
    d = O.distance_matrix(a0, b0, grid + (0.0,), 0x1)
    d = d[d > 0]
    R0, RM = float(d.max()) * 1.001, float(d.min()) * 0.999
    radii = R0 * (RM / R0) ** (np.arange(1, 16) / 15)
    c, y, st = cil.features(A, B, grid + (0.0,), 0x1, torch.tensor(radii[None, :], device=dev))
    torch.cuda.synchronize()
    assert int(st.abs().sum()) == 0
    c = c.cpu().numpy()
    for p in range(P):
        ref = O.features(A[p].cpu().numpy(), B[p].cpu().numpy(), grid + (0.0,), 0x1, radii, band=BAND)
        _check_counts(c[p], ref)


# ------------------------------------------------------------------ L2-type family on tensor cores
@pytest.mark.parametrize("engine", ["AUTO", "TC_I8"])
def test_l2_family_tensor_cores_vs_oracle(cil, oracle_mod, engine):
    """L2, W12SUM (7), W12 (8) on the three-phase INT8 engine: a C2-shaped
    grid, 300 x 260 patterns (two column tiles, ragged), radii at dense quantiles of the pair
    distances so that many pairs sit near a radius and go through the bound / re-check."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 64, 64, 0.0)
    A = cilgen.make_set(71, 0, 300, grid[:3])
    B = cilgen.make_set(71, 1, 260, grid[:3])
    mask = 0x0D
    D = _sel(O.distance_matrix(A[:80].numpy(), B[:80].numpy(), grid, 0x3F), mask)
    radii = np.array([np.quantile(d, np.linspace(0.97, 0.03, 15)) for d in D])
    c, y, st = cil.features(A.to(dev), B.to(dev), grid, mask, torch.tensor(radii, device=dev),
                            engine=_engine(cil, engine))
    torch.cuda.synchronize()
    assert int(st[0]) == 0
    ref = O.features(A.numpy(), B.numpy(), grid, mask, radii, band=BAND)
    _check_counts(c[0].cpu().numpy(), ref)


@pytest.mark.parametrize("case", ["C2", "C4", "offset", "C1", "1D", "neardup0", "neardup6", "neardup3"])
def test_gram_family_error_bound(cil, oracle_mod, case):
    """The three-phase engine's intervals of L2/sqrt(w), W12^2/w and W12SUM/sqrt(w) must contain the
    exact FP64 values for every pair (worst-case bound, L2-type family on tensor cores)."""
    O = oracle_mod
    dev = torch.device("cuda")
    A, B, grid = _bound_case(case, 33)
    iv = cil.diag_gram_family(A.to(dev), B.to(dev), grid).cpu().numpy().astype(np.float64)
    h = 1.0 / (grid[2] - 1)
    w = h * h if grid[1] > 1 else h
    D = O.distance_matrix(A.numpy(), B.numpy(), grid, 0x0D)        # L2, W12SUM, W12 (bit order)
    exact = [D[0] / np.sqrt(w), D[2] ** 2 / w, D[1] / np.sqrt(w)]   # kinds 0 L2, 1 W12, 2 W12SUM
    for k, name in enumerate(["L2", "W12", "W12SUM"]):
        lo, hi = iv[k, ..., 0], iv[k, ..., 1]
        ok = (lo <= exact[k]) & (exact[k] <= hi)
        pos = exact[k] > 0
        print(f"{case} {name}: median (hi-lo)/v = {np.median((hi - lo)[pos] / exact[k][pos]):.3e}")
        assert ok.all(), (name, np.argwhere(~ok)[:5].tolist())


def test_synth_l2_family_segmented_tensor_cores(cil, oracle_mod):
    """SCIL (Alg. 3) with L2, W12SUM, W12 on the three-phase engine with column segments
    (N~ = 50 >= 43 columns per SCIL block): segmented per-thread histograms of three kinds."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (1, 16, 16, 0.0)
    P, n_ens, N_set, Nt = 2, 3, 6, 50
    Nsyn = n_ens * (N_set + Nt)
    pools = torch.stack([cilgen.make_set(81, 200 + p, Nsyn, grid[:3], n_w=4.7 + 0.2 * p) for p in range(P)])
    data = cilgen.make_set(81, 999, N_set, grid[:3])
    k0 = np.array([2, 0], np.int32)
    mask = 0x0D
    radii = []
    for p in range(P):
        Dp = _sel(O.distance_matrix(pools[p, :40].numpy(), pools[p, 40:80].numpy(), grid, 0x3F), mask)
        radii.append(np.array([np.quantile(d, np.linspace(0.95, 0.05, 10)) for d in Dp]))
    radii = np.array(radii)
    out, st, Y = cil.synth_loglik(pools.to(dev), n_ens, N_set, Nt, data.to(dev), torch.tensor(k0, device=dev),
                                  grid, mask, torch.tensor(radii, device=dev), ridge=1e-4,
                                  engine=cil.ENGINE_TC_I8, return_Y=True)
    torch.cuda.synchronize()
    for p in range(P):
        ref, rst, Yr = O.synth_loglik(pools[p].numpy(), n_ens, N_set, Nt, data.numpy(), int(k0[p]), grid, mask,
                                      radii[p], ridge=1e-4)
        Yg = Y[p].cpu().numpy()
        npairs = N_set * Nt
        # every count within one of the oracle's (no pair of these radii sits within 1e-6 of one)
        np.testing.assert_array_equal(np.rint(Yg * npairs), np.rint(Yr * npairs))
        np.testing.assert_allclose(out[p].cpu().numpy(), ref, rtol=0, atol=1e-6)


@pytest.mark.parametrize("engine,N,mask", [("AUTO", 50, 0x3F), ("AUTO", 12, 0x0D), ("SIMT", 20, 0x3F),
                                           ("TC_3XBF16", 30, 0x01), ("TC_I8", 60, 0x01)])
def test_train_vectors_vs_oracle(cil, oracle_mod, engine, N, mask):
    """Alg. 1 / Alg. 2 training vectors: one panel against itself, segmented by subset, the
    k < l blocks (triangle) in lexicographic order, against the oracle's per-pair counts."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (1, 16, 16, 0.0)
    n_ens, P = 5, 2
    X = torch.stack([cilgen.make_set(91, p, n_ens * N, grid[:3]) for p in range(P)])
    sel = [q for q in range(6) if (mask >> q) & 1]
    D = O.distance_matrix(X[0, :40].numpy(), X[0, 40:80].numpy(), grid, mask)
    radii = np.array([np.quantile(d, np.linspace(0.95, 0.05, 9)) for d in D])
    Y, st = cil.train_vectors(X.to(dev), n_ens, grid, mask, torch.tensor(radii, device=dev),
                              engine=_engine(cil, engine))
    torch.cuda.synchronize()
    assert Y.shape == (P, n_ens * (n_ens - 1) // 2, len(sel) * 9)
    for p in range(P):
        ref = O.train_vectors(X[p].numpy(), n_ens, grid, mask, radii, band=BAND)
        c = np.rint(Y[p].cpu().numpy() * N * N).astype(np.int64).reshape(ref["lo"].shape)
        assert np.all(ref["lo"] <= c) and np.all(c <= ref["hi"]), f"item {p}"


def test_gaussianity_chi2(cil, oracle_mod):
    """The chi^2 Gaussianity diagnostic: Mahalanobis distances of the vectors
    from the device match the oracle's quad for each vector; Gaussian samples pass the test."""
    O = oracle_mod
    dev = torch.device("cuda")
    rng = np.random.default_rng(3)
    D, n = 8, 400
    L = rng.standard_normal((D, D)) * 0.3 + np.eye(D)
    Y = rng.standard_normal((n, D)) @ L.T + 0.5
    stat, dof, d2 = cil.gaussianity_chi2(torch.tensor(Y, device=dev))
    mu, Sig = O.stats(Y)
    for k in range(0, n, 37):
        out, st = O.loglik(mu, Sig, Y[k])
        assert float(d2[k]) == pytest.approx(out[0], rel=1e-9)
    from scipy import stats as sps
    assert sps.chi2.sf(stat, dof) > 1e-4           # Gaussian data: no rejection at any sane level
    # the device's Pearson statistic is the plain one on its own d2 (scipy quantiles, numpy bins)
    d2h = d2.cpu().numpy()
    edges = sps.chi2.ppf(np.arange(1, 10) / 10, D)
    cnt = np.bincount(np.searchsorted(edges, d2h), minlength=10)
    assert dof == 9 and stat == pytest.approx(float(((cnt - n / 10) ** 2 / (n / 10)).sum()), rel=1e-12)


@pytest.mark.parametrize("law", ["power", "linear"])
def test_adaptive_radii_vs_oracle(cil, oracle_mod, law):
    """Per-item distance ranges (exact per-pair measures) and the radii laws of PAPER.md:109."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 12, 12, 0.0)
    P, N, Nt = 3, 40, 33
    A = torch.stack([cilgen.make_set(95, 2 * p, N, grid[:3], n_w=4.6 + 0.3 * p) for p in range(P)])
    B = torch.stack([cilgen.make_set(95, 2 * p + 1, Nt, grid[:3], n_w=4.6 + 0.3 * p) for p in range(P)])
    rng, st = cil.distance_range(A.to(dev), B.to(dev), grid, 0x3F)
    radii, st2 = cil.radii_from_range(rng, 11, law)
    torch.cuda.synchronize()
    assert int(st.max()) == 0 and int(st2.max()) == 0
    for p in range(P):
        ref = O.distance_range(A[p].numpy(), B[p].numpy(), grid, 0x3F)
        np.testing.assert_allclose(rng[p].cpu().numpy(), ref, rtol=1e-6)
        np.testing.assert_allclose(radii[p].cpu().numpy(), O.radii_from_range(rng[p].cpu().numpy(), 11, law),
                                   rtol=1e-12)
    # a set against itself: the zero self-distances are not the minimum
    rs, _ = cil.distance_range(A[0].to(dev), A[0].to(dev), grid, 0x1)
    torch.cuda.synchronize()
    assert float(rs[0, 0, 0]) > 0


def test_minmax_scale_bit_exact(cil, oracle_mod):
    """Scaled patterns: FP64 (x - min)/(max - min) rounded to FP32 on both
    sides is bit-identical; then the scaled-data counts (L2-type norms)."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 16, 16, 0.0)
    X = cilgen.make_set(97, 0, 50, grid[:3])
    X[3, 1] = 2.5                                         # a constant species
    Yg = cil.minmax_scale(X.to(dev), grid)
    torch.cuda.synchronize()
    Yr = O.minmax_scale(X.numpy(), grid)
    np.testing.assert_array_equal(Yg.cpu().numpy(), Yr)
    mask = 0x0D
    D = O.distance_matrix(Yr[:25], Yr[25:], grid, mask)
    radii = np.array([np.quantile(d, np.linspace(0.95, 0.05, 8)) for d in D])
    c, _, _ = _run_features(cil, torch.tensor(Yr[:25]), torch.tensor(Yr[25:]), grid, mask, radii, "AUTO")
    _check_counts(c[0], O.features(Yr[:25], Yr[25:], grid, mask, radii, band=BAND))


@pytest.mark.parametrize("engine", ["AUTO", "SIMT"])
@pytest.mark.parametrize("grid", [(2, 1, 64, 0.0, 0b10), (2, 16, 16, 0.0, 0b01)])
def test_gradient_species_mask(cil, oracle_mod, engine, grid):
    """Gradient-based norms w.r.t. selected species only (reading R18), all six
    measures, on both the tensor-core and the CUDA-core engines."""
    O = oracle_mod
    dev = torch.device("cuda")
    A = cilgen.make_set(99, 0, 70, grid[:3])
    B = cilgen.make_set(99, 1, 55, grid[:3])
    D = O.distance_matrix(A[:40].numpy(), B[:40].numpy(), grid, 0x3F)
    radii = np.array([np.quantile(d, np.linspace(0.95, 0.05, 9)) for d in D])
    c, _, st = _run_features(cil, A, B, grid, 0x3F, radii, engine)
    assert int(st[0]) == 0
    _check_counts(c[0], O.features(A.numpy(), B.numpy(), grid, 0x3F, radii, band=BAND))


def test_c5_shape_large_K(cil, oracle_mod):
    """C5-shaped patterns (256x256x2, K = 131072 > 65536: the INT8 engine accumulates in two exact
    K chunks, the three-phase family in two chunks per block), ragged 200 x 150 pairs, L2 + W12 + Linf."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 256, 256, 0.0)
    A = cilgen.make_set(101, 0, 200, grid[:3])
    B = cilgen.make_set(101, 1, 150, grid[:3])
    mask = 0x0B
    D = O.distance_matrix(A[:30].numpy(), B[:30].numpy(), grid, mask)
    radii = np.array([np.quantile(d, np.linspace(0.97, 0.03, 12)) for d in D])
    c, _, st = _run_features(cil, A, B, grid, mask, radii, "AUTO")
    assert int(st[0]) == 0
    _check_counts(c[0], O.features(A.numpy(), B.numpy(), grid, mask, radii, band=BAND))


def test_c5_row_sample_all_measures(cil, oracle_mod):
    """C5 (BASELINE configs[4]) at its full K_aug: 64 rows of A x 1000 rows of B of the bench's
    256x256x2 sets (seed of config 5), all six measures, M = 20, against the oracle."""
    O = oracle_mod
    grid = (2, 256, 256, 0.0)
    seed = cilgen.config_seed(5)
    A = cilgen.make_set(seed, 0, 64, grid[:3])
    B = cilgen.make_set(seed, 1, 1000, grid[:3])
    D = O.distance_matrix(A[:24].numpy(), B[:200].numpy(), grid, 0x3F)
    radii = np.array([np.quantile(d, np.linspace(0.98, 0.02, 20)) for d in D])
    c, _, st = _run_features(cil, A, B, grid, 0x3F, radii, "AUTO")
    assert int(st[0]) == 0
    _check_counts(c[0], O.features(A.numpy(), B.numpy(), grid, 0x3F, radii, band=BAND))


@pytest.mark.parametrize("engine", ["AUTO", "SIMT"])
def test_c3_row_sample_all_measures(cil, oracle_mod, engine):
    """C3 (BASELINE configs[2]): 32 rows of A x all 2000 rows of B of the bench's 128x128x2 sets,
    all six measures, M = 20, against the oracle (the bench times 2000 x 2000)."""
    O = oracle_mod
    grid = (2, 128, 128, 0.0)
    seed = cilgen.config_seed(3)
    A = cilgen.make_set(seed, 0, 32, grid[:3])
    B = cilgen.make_set(seed, 1, 2000, grid[:3])
    D = O.distance_matrix(A[:16].numpy(), B[:300].numpy(), grid, 0x3F)
    radii = np.array([np.quantile(d, np.linspace(0.98, 0.02, 20)) for d in D])
    c, _, st = _run_features(cil, A, B, grid, 0x3F, radii, engine)
    assert int(st[0]) == 0
    _check_counts(c[0], O.features(A.numpy(), B.numpy(), grid, 0x3F, radii, band=BAND))


@pytest.mark.parametrize("engine", ["TC_I8", "AUTO", "SIMT"])
@pytest.mark.parametrize("mask", [0x01, 0x0D, 0x3F])
def test_many_radii(cil, oracle_mod, engine, mask):
    """M = 48 radii (the MAXM = 64 instantiations of the INT8 engines, one- and three-phase), with
    ragged 300 x 270 sets spanning several tiles, radii at dense quantiles of the distances."""
    O = oracle_mod
    grid = (2, 24, 24, 0.0)
    A = cilgen.make_set(57, 0, 300, grid[:3])
    B = cilgen.make_set(57, 1, 270, grid[:3])
    D = _sel(O.distance_matrix(A[:60].numpy(), B[:60].numpy(), grid, 0x3F), mask)
    radii = np.array([np.quantile(d, np.linspace(0.99, 0.01, 48)) for d in D])
    c, _, st = _run_features(cil, A, B, grid, mask, radii, engine)
    assert int(st[0]) == 0
    _check_counts(c[0], O.features(A.numpy(), B.numpy(), grid, mask, radii, band=BAND))


@pytest.mark.parametrize("mask", [0x01, 0x0D])
def test_synth_c4_shape_swapped_panels(cil, oracle_mod, mask):
    """SCIL at C4's panel shape (n_ens = 10, N_set = N~ = 50: the 550-row panel pads worse than
    the 500-row one, so the INT8 Gram runs the column panel as its rows with 192-column
    tiles and the segments are read transposed) against the oracle's Alg. 3."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (1, 16, 16, 0.0)
    P, n_ens, N_set, Nt = 2, 10, 50, 50
    Nsyn = n_ens * (N_set + Nt)
    pools = torch.stack([cilgen.make_set(103, 300 + p, Nsyn, grid[:3], n_w=4.8 + 0.2 * p) for p in range(P)])
    data = cilgen.make_set(103, 999, N_set, grid[:3])
    k0 = np.array([3, 7], np.int32)
    radii = []
    for p in range(P):
        Dp = _sel(O.distance_matrix(pools[p, :60].numpy(), pools[p, 60:120].numpy(), grid, 0x3F), mask)
        radii.append(np.array([np.quantile(d, np.linspace(0.95, 0.05, 13)) for d in Dp]))
    radii = np.array(radii)
    out, st, Y = cil.synth_loglik(pools.to(dev), n_ens, N_set, Nt, data.to(dev), torch.tensor(k0, device=dev),
                                  grid, mask, torch.tensor(radii, device=dev), ridge=1e-6,
                                  engine=cil.ENGINE_TC_I8, return_Y=True)
    torch.cuda.synchronize()
    npairs = N_set * Nt
    for p in range(P):
        ref, rst, Yr = O.synth_loglik(pools[p].numpy(), n_ens, N_set, Nt, data.numpy(), int(k0[p]), grid, mask,
                                      radii[p], ridge=1e-6)
        Yg = Y[p].cpu().numpy()
        # counts within the oracle's band: recompute band counts for every (k, l) block and y~
        cg = np.rint(Yg * npairs).astype(np.int64)
        N = N_set + Nt
        pool = pools[p].numpy()
        rows = []
        for k in range(n_ens):
            for l in range(n_ens):
                rows.append(O.features(pool[k * N:k * N + N_set], pool[l * N + N_set:(l + 1) * N], grid, mask,
                                       radii[p], band=BAND))
        rows.append(O.features(data.numpy(), pool[k0[p] * N + N_set:(k0[p] + 1) * N], grid, mask, radii[p],
                               band=BAND))
        lo = np.array([r["lo"].ravel() for r in rows])
        hi = np.array([r["hi"].ravel() for r in rows])
        assert np.all(lo <= cg) and np.all(cg <= hi), f"item {p}"
        if np.array_equal(Yg, Yr):
            np.testing.assert_allclose(out[p].cpu().numpy(), ref, rtol=0, atol=1e-6)


# ------------------------------------------------------------------ full-size SCIL / bootstrap (sampled)
def test_c4_full_theta_vs_oracle(cil, oracle_mod):
    """C4 at full size in the bench's launch configuration (pools of 1000 patterns of 128x128,
    n_ens = 10, 50 + 50, M = 13, swapped panels and 192-column tiles, several proposals in one
    launch); every proposal against the oracle's Alg. 3: every vector within the band, loglik."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (1, 128, 128, 0.0)
    P, n_ens, N_set, Nt, M = 4, 10, 50, 50, 13
    seed = cilgen.config_seed(4)
    pools = torch.empty((P, n_ens * (N_set + Nt)) + grid[:3], dtype=torch.float32, device=dev)
    for p in range(P):
        cilgen.make_set(seed, p, n_ens * (N_set + Nt), grid[:3], device=dev, out=pools[p], n_w=4.6 + 0.2 * p)
    data = cilgen.make_set(seed, 1000, N_set, grid[:3], device=dev)
    k0 = torch.tensor([p % n_ens for p in range(P)], dtype=torch.int32, device=dev)
    pool0 = pools[0].cpu().numpy()
    D = O.distance_matrix(pool0[:64], pool0[64:128], grid, 0x1)[0]
    R0, RM = D.max() * 1.001, D.min() * 0.999
    r1 = R0 * (RM / R0) ** (np.arange(1, M + 1) / M)
    radii = torch.tensor(np.tile(r1, (P, 1, 1)), device=dev)
    out, st, Y = cil.synth_loglik(pools, n_ens, N_set, Nt, data, k0, grid, 0x1, radii, ridge=1e-10,
                                  engine=cil.ENGINE_AUTO, return_Y=True)
    torch.cuda.synchronize()
    assert int(st.max()) == 0
    N = N_set + Nt
    dat = data.cpu().numpy()
    for p in range(P):                      # every proposal of the launch
        pool = pools[p].cpu().numpy()
        cg = np.rint(Y[p].cpu().numpy() * N_set * Nt).astype(np.int64)
        v = 0
        for k in range(n_ens):
            for l in range(n_ens):
                r = O.features(pool[k * N:k * N + N_set], pool[l * N + N_set:(l + 1) * N], grid, 0x1, r1[None],
                               band=BAND)
                assert np.all(r["lo"][0] <= cg[v]) and np.all(cg[v] <= r["hi"][0]), (p, k, l)
                v += 1
        kk = p % n_ens                      # the caller's k0 (Alg. 3 line "y~ = C(R, s_data, s^{k0,2})")
        r = O.features(dat, pool[kk * N + N_set:(kk + 1) * N], grid, 0x1, r1[None], band=BAND)
        assert np.all(r["lo"][0] <= cg[v]) and np.all(cg[v] <= r["hi"][0]), p
        mu, Sig = O.stats(Y[p, :-1].cpu().numpy())
        ref, _ = O.loglik(mu, Sig, Y[p, -1].cpu().numpy(), ridge=1e-10)
        np.testing.assert_allclose(out[p].cpu().numpy(), ref, rtol=0, atol=1e-6)


def test_c6_full_theta_bins_and_replicates(cil, oracle_mod):
    """C6 (Alg. A2 at the paper's sizes: pool 1000 of 64x64x2, N_set = 50, 1000 replicates) in
    the bench's configuration for 2 proposals: the bin matrix of proposal 0 on a sampled block
    against the oracle's distances; for every proposal 12 replicates against brute force on the
    resampled sets and the log-density on the GPU's own vectors."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 64, 64, 0.0)
    P, N_syn, N_set, n_rep, M = 2, 1000, 50, 1000, 13
    seed = cilgen.config_seed(6)
    pools = torch.stack([cilgen.make_set(seed, p, N_syn, grid[:3], n_w=4.7 + 0.3 * p) for p in range(P)])
    data = cilgen.make_set(seed, 100000, N_set, grid[:3])
    draws = [cilgen.boot_draws_a2(seed, p, n_rep, N_syn, N_set) for p in range(P)]
    I1 = np.stack([d[0] for d in draws]); I2 = np.stack([d[1] for d in draws]); J = np.stack([d[2] for d in draws])
    pool0 = pools[0].numpy()
    D = O.distance_matrix(pool0[:64], pool0[64:128], grid, 0x1)[0]
    R0, RM = D.max() * 1.001, D[D > 0].min() * 0.999
    r1 = R0 * (RM / R0) ** (np.arange(1, M + 1) / M)
    radii = np.tile(r1, (P, 1, 1))
    out, st, Y = cil.synth_loglik_boot(pools.to(dev), data.to(dev), N_set, torch.tensor(I1, device=dev),
                                       torch.tensor(I2, device=dev), torch.tensor(J, device=dev), grid, 0x1,
                                       torch.tensor(radii, device=dev), ridge=1e-10, return_Y=True)
    bins, _ = cil.bin_matrix(pools[0].to(dev), pools[0].to(dev), grid, 0x1, torch.tensor(r1[None], device=dev))
    torch.cuda.synchronize()
    assert int(st.max()) == 0
    # the bin matrix (symmetric upper-triangle tiles + mirrored writes) on a sampled block
    rows = np.arange(0, N_syn, 7)[:120]
    Ds = O.distance_matrix(pool0[rows], pool0, grid, 0x1)[0]
    lo = (Ds[:, :, None] < r1 * (1 - BAND)).sum(-1)
    hi = (Ds[:, :, None] < r1 * (1 + BAND)).sum(-1)
    b = bins[0, 0].cpu().numpy()[rows]
    assert np.all(lo <= b) and np.all(b <= hi)
    # replicate vectors of every proposal (12 sampled replicates each), and the tail (mu, Sigma,
    # Cholesky log-density) of each proposal on the GPU's own vectors
    Nt = N_syn - N_set
    ks = np.arange(0, n_rep, 83)[:12]
    for p in range(P):
        pool = pools[p].numpy()
        Yg = Y[p].cpu().numpy()
        rr = O.resample_features(pool, pool, grid, 0x1, r1[None], I1[p][ks], I2[p][ks], band=BAND)
        cg = np.rint(Yg[ks] * N_set * Nt).astype(np.int64)
        assert np.all(rr["lo"][:, 0] <= cg) and np.all(cg <= rr["hi"][:, 0]), p
        mu, Sig = O.stats(Yg[:-1])
        o2, _ = O.loglik(mu, Sig, Yg[-1], ridge=1e-10)
        np.testing.assert_allclose(out[p].cpu().numpy(), o2, rtol=0, atol=1e-6)


def test_c7_full_training_sampled_blocks(cil, oracle_mod):
    """C7 in the bench's configuration (N_set = 3000 GM 64x64x2, n_ens = 10, all six measures):
    three of the 45 subset-pair vectors against the oracle (band), the rest by symmetry checks."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 64, 64, 0.0)
    N_set, n_ens, M = 3000, 10, 13
    X = cilgen.make_set(cilgen.config_seed(7), 0, N_set, grid[:3])
    N = N_set // n_ens
    Xn = X.numpy()
    D = O.distance_matrix(Xn[:48], Xn[N:N + 48], grid, 0x3F)
    radii = np.array([d.max() * 1.001 * ((d[d > 0].min() * 0.999) / (d.max() * 1.001)) ** (np.arange(1, M + 1) / M)
                      for d in D])
    Y, st = cil.train_vectors(X.to(dev), n_ens, grid, 0x3F, torch.tensor(radii, device=dev))
    torch.cuda.synchronize()
    assert int(st[0]) == 0 and Y.shape == (1, 45, 6 * M)
    pairs = [(k, l) for k in range(n_ens) for l in range(k + 1, n_ens)]
    for v in (0, 17, 44):
        k, l = pairs[v]
        r = O.features(Xn[k * N:(k + 1) * N], Xn[l * N:(l + 1) * N], grid, 0x3F, radii, band=BAND)
        c = np.rint(Y[0, v].cpu().numpy() * N * N).astype(np.int64).reshape(6, M)
        assert np.all(r["lo"] <= c) and np.all(c <= r["hi"]), (k, l)


def test_c3_full_additivity(cil):
    """C3 in the bench's configuration (2000 x 2000 of 128x128x2, all six measures, M = 20):
    the full launch equals the sum of the two half launches (row blocks) — counts are sums over
    pairs, a property of Eq. (1) at any size; the engines at this shape are oracle-checked on
    smaller sets (test_l2_family_tensor_cores_vs_oracle, test_c1_all_measures)."""
    dev = torch.device("cuda")
    grid = (2, 128, 128, 0.0)
    seed = cilgen.config_seed(3)
    A = cilgen.make_set(seed, 0, 2000, grid[:3], device=dev)
    B = cilgen.make_set(seed, 1, 2000, grid[:3], device=dev)
    h = 1.0 / 127
    base = np.array([40.0, 3.0, 900.0, 700.0, 60.0, 150.0])
    radii = torch.tensor(np.array([b * np.geomspace(1.2, 0.5, 20) for b in base]), device=dev)
    c, _, st = cil.features(A, B, grid, 0x3F, radii)
    c1, _, _ = cil.features(A[:1000], B, grid, 0x3F, radii)
    c2, _, _ = cil.features(A[1000:], B, grid, 0x3F, radii)
    torch.cuda.synchronize()
    assert int(st[0]) == 0
    assert torch.equal(c, c1 + c2)
    assert (c[0, :, 0] >= c[0, :, -1]).all()
