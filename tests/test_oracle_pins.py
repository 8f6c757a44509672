"""Pins for the FP64 oracle: each test fixes the oracle to something OTHER than itself —
hand-worked values (tests/golden), closed forms, library routines (scipy/numpy), an
independent brute force (tests/brute.py) and invariants of Eq. (1)-(13).  CPU only.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import stats as sps
from scipy.spatial.distance import cdist

import brute
import cilgen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_example.json")))
ALL = 0x3F


def _grid(g):
    return (g["S"], g["H"], g["W"], g["h"])


# ---------------------------------------------------------------- hand example (pin 1)
def test_hand_distances(oracle_mod):
    O = oracle_mod
    g = _grid(GOLD["grid"])
    A = np.array(GOLD["A"], np.float32)[:, None]
    B = np.array(GOLD["B"], np.float32)[:, None]
    D = O.distance_matrix(A, B, g, ALL)
    for q, name in enumerate(GOLD["measures"]):
        np.testing.assert_allclose(D[q].ravel(), GOLD["distances"][name], rtol=1e-12, atol=1e-12)


def test_hand_counts_strict(oracle_mod):
    O = oracle_mod
    g = _grid(GOLD["grid"])
    A = np.array(GOLD["A"], np.float32)[:, None]
    B = np.array(GOLD["B"], np.float32)[:, None]
    radii = np.tile(np.array(GOLD["radii"]), (6, 1))
    r = O.features(A, B, g, ALL, radii, band=0.0)
    for q, name in enumerate(GOLD["measures"]):
        assert r["counts"][q].tolist() == GOLD["counts"][name], name
    np.testing.assert_array_equal(r["y"], r["counts"] / 4.0)


def test_hand_stats_loglik(oracle_mod):
    O = oracle_mod
    st = GOLD["stats"]
    mu, Sig = O.stats(np.array(st["Y"]))
    np.testing.assert_allclose(mu, st["mu"], rtol=1e-14)
    np.testing.assert_allclose(Sig, st["Sigma"], rtol=1e-14)
    out, status = O.loglik(mu, Sig, st["y_obs"])
    assert status == 0
    np.testing.assert_allclose(out, [st["quad"], st["logdet"], st["loglik"]], rtol=1e-12)


def test_spec_ecdf_case(oracle_mod):
    O = oracle_mod
    c = GOLD["ecdf_spec_case"]
    A = np.array(c["A"], np.float32).reshape(2, 1, 1, 1)
    B = np.array(c["B"], np.float32).reshape(2, 1, 1, 1)
    r = O.features(A, B, (1, 1, 1, 0.0), 1, [[c["R"]]], band=0.0)
    assert r["y"][0, 0] == c["y"]


# ---------------------------------------------------------------- closed forms (pin 2)
S_, H_, W_ = 2, 5, 5
H_STEP = 0.25
W_Q = H_STEP ** 2


def _pair_from_delta(delta):
    rng = np.random.default_rng(7)
    b = rng.integers(-4, 5, size=delta.shape).astype(np.float32)  # exact small ints
    a = (b + delta).astype(np.float32)
    return a, b


@pytest.mark.parametrize("c", [1.0, -3.0, 0.5])
def test_closed_form_constant(oracle_mod, c):
    delta = np.full((S_, H_, W_), c, np.float32)
    a, b = _pair_from_delta(delta)
    s = oracle_mod.subnorms(a, b, (S_, H_, W_, H_STEP))
    assert math.isclose(math.sqrt(W_Q * s[0]), abs(c) * math.sqrt(W_Q * S_ * H_ * W_), rel_tol=1e-14)
    assert s[1] == 0 and s[2] == 0 and s[4] == 0 and s[5] == 0
    assert s[3] == abs(c)
    d = oracle_mod.distance_matrix(a[None], b[None], (S_, H_, W_, H_STEP), ALL)[:, 0, 0]
    assert d[2] == pytest.approx(d[0]) and d[3] == pytest.approx(d[0])   # W12 = W12sum = L2
    assert d[4] == d[1] and d[5] == d[1]                               # W1inf = W1infsum = Linf


@pytest.mark.parametrize("c", [1.0, -2.0])
def test_closed_form_ramp(oracle_mod, c):
    col = np.arange(W_, dtype=np.float32)
    delta = np.broadcast_to(c * col, (S_, H_, W_)).astype(np.float32)
    a, b = _pair_from_delta(delta)
    s = oracle_mod.subnorms(a, b, (S_, H_, W_, H_STEP))
    a0 = abs(c) * math.sqrt(W_Q * S_ * H_ * (W_ - 1) * W_ * (2 * W_ - 1) / 6)
    ax = abs(c) / H_STEP * math.sqrt(W_Q * S_ * H_ * (W_ - 1))   # last node omitted [R3]
    assert math.sqrt(W_Q * s[0]) == pytest.approx(a0, rel=1e-14)
    assert math.sqrt(W_Q * s[1]) == pytest.approx(ax, rel=1e-14)
    assert s[2] == 0
    assert s[3] == abs(c) * (W_ - 1) and s[4] == pytest.approx(abs(c) / H_STEP) and s[5] == 0


def test_closed_form_checkerboard(oracle_mod):
    c = 1.5
    r, q = np.meshgrid(np.arange(H_), np.arange(W_), indexing="ij")
    delta = np.broadcast_to(c * (-1.0) ** (r + q), (S_, H_, W_)).astype(np.float32)
    a, b = _pair_from_delta(delta)
    s = oracle_mod.subnorms(a, b, (S_, H_, W_, H_STEP))
    assert math.sqrt(W_Q * s[0]) == pytest.approx(c * math.sqrt(W_Q * S_ * H_ * W_), rel=1e-14)
    assert math.sqrt(W_Q * s[1]) == pytest.approx(2 * c / H_STEP * math.sqrt(W_Q * S_ * H_ * (W_ - 1)), rel=1e-14)
    assert math.sqrt(W_Q * s[2]) == pytest.approx(2 * c / H_STEP * math.sqrt(W_Q * S_ * (H_ - 1) * W_), rel=1e-14)
    assert s[3] == c and s[4] == pytest.approx(2 * c / H_STEP) and s[5] == pytest.approx(2 * c / H_STEP)


def test_loglik_closed_forms(oracle_mod):
    O = oracle_mod
    D = 5
    mu = np.linspace(0.1, 0.9, D)
    out, st = O.loglik(mu, np.eye(D), mu + np.eye(D)[0])
    assert st == 0 and out[0] == pytest.approx(1.0, abs=1e-15) and out[1] == 0
    out, st = O.loglik(mu, np.eye(D), mu)
    assert out[0] == 0
    sig = np.array([0.5, 1.0, 2.0, 3.0, 0.1])
    r = np.array([0.3, -0.2, 1.0, 0.0, 0.05])
    out, st = O.loglik(mu, np.diag(sig ** 2), mu + r)
    assert out[0] == pytest.approx(np.sum((r / sig) ** 2), rel=1e-14)
    assert out[1] == pytest.approx(np.sum(np.log(sig ** 2)), rel=1e-14)


# ---------------------------------------------------------------- libraries / brute force (pin 3)
def test_cdist_euclid_cheb(oracle_mod):
    rng = np.random.default_rng(3)
    A = rng.standard_normal((7, 1, 1, 13)).astype(np.float32)   # 1-D, h = 1 -> w = 1
    B = rng.standard_normal((5, 1, 1, 13)).astype(np.float32)
    D = oracle_mod.distance_matrix(A, B, (1, 1, 13, 1.0), 0x3)
    a2, b2 = A.reshape(7, -1).astype(np.float64), B.reshape(5, -1).astype(np.float64)
    np.testing.assert_allclose(D[0], cdist(a2, b2, "euclidean"), rtol=1e-13)
    np.testing.assert_allclose(D[1], cdist(a2, b2, "chebyshev"), rtol=0, atol=0)


@pytest.mark.parametrize("grid", [(1, 6, 7, 0.0), (2, 5, 4, 0.3), (3, 1, 9, 0.0), (2, 4, 4, 0.0)])
def test_brute_force_distances_and_counts(oracle_mod, grid):
    O = oracle_mod
    rng = np.random.default_rng(11)
    S, H, W, _ = grid
    A = rng.standard_normal((9, S, H, W)).astype(np.float32)
    B = (rng.standard_normal((6, S, H, W)) + 0.5).astype(np.float32)
    D = O.distance_matrix(A, B, grid, ALL)
    Db = brute.distances(A, B, grid)
    np.testing.assert_allclose(D, Db, rtol=1e-12)
    # radii from the range of all distances, power law, M = 7
    radii = []
    for q in range(6):
        R0, RM = Db[q].max() * 1.001, Db[q].min() * 0.999
        radii.append(R0 * (RM / R0) ** (np.arange(1, 8) / 7.0))
    radii = np.array(radii)
    r = O.features(A, B, grid, ALL, radii, band=0.0)
    np.testing.assert_array_equal(r["counts"], brute.counts(A, B, grid, ALL, radii))


def test_stats_vs_numpy(oracle_mod):
    rng = np.random.default_rng(5)
    Y = rng.random((40, 9))
    mu, Sig = oracle_mod.stats(Y)
    np.testing.assert_allclose(mu, Y.mean(axis=0), rtol=1e-13)
    np.testing.assert_allclose(Sig, np.cov(Y, rowvar=False, ddof=1), rtol=1e-11, atol=1e-15)


def test_loglik_vs_scipy(oracle_mod):
    rng = np.random.default_rng(9)
    D = 13
    X = rng.standard_normal((D, 3 * D))
    Sig = X @ X.T / (3 * D) + 0.1 * np.eye(D)
    mu = rng.standard_normal(D)
    y = mu + rng.standard_normal(D)
    out, st = oracle_mod.loglik(mu, Sig, y)
    assert st == 0
    assert out[2] == pytest.approx(sps.multivariate_normal(mu, Sig).logpdf(y), rel=1e-12)
    assert out[0] == pytest.approx((y - mu) @ np.linalg.solve(Sig, y - mu), rel=1e-12)
    assert out[1] == pytest.approx(np.linalg.slogdet(Sig)[1], rel=1e-12)
    # explicit ridge is added to the diagonal
    out_r, _ = oracle_mod.loglik(mu, Sig, y, ridge=0.5)
    assert out_r[2] == pytest.approx(sps.multivariate_normal(mu, Sig + 0.5 * np.eye(D)).logpdf(y), rel=1e-12)


def test_loglik_not_pd(oracle_mod):
    D = 4
    v = np.arange(1.0, D + 1)
    out, st = oracle_mod.loglik(np.zeros(D), np.outer(v, v), np.ones(D))   # rank 1
    assert st == 2 and all(math.isnan(x) for x in out)


def test_synth_vs_brute(oracle_mod):
    """Alg. 3 composed from brute-force counts, numpy cov and scipy logpdf."""
    O = oracle_mod
    grid = (2, 4, 5, 0.0)
    n_ens, N_set, Nt = 3, 2, 4
    pool = cilgen.make_patterns(1, 0, n_ens * (N_set + Nt), grid[:3]).numpy()
    data = cilgen.make_patterns(1, 1, N_set, grid[:3]).numpy()
    mask = 0b101011
    Db = brute.distances(pool, pool, grid)
    sel = [q for q in range(6) if (mask >> q) & 1]
    radii = np.array([np.quantile(Db[q][Db[q] > 0], np.linspace(0.9, 0.1, 6)) for q in sel])
    k0 = 2
    out, st, Y = O.synth_loglik(pool, n_ens, N_set, Nt, data, k0, grid, mask, radii, ridge=1e-6)
    Yb, yt = brute.synth(pool, n_ens, N_set, Nt, data, k0, grid, mask, radii)
    np.testing.assert_array_equal(Y[:-1], Yb)
    np.testing.assert_array_equal(Y[-1], yt)
    mu = Yb.mean(0)
    Sig = np.cov(Yb, rowvar=False, ddof=1) + 1e-6 * np.eye(Yb.shape[1])
    if st == 0:
        assert out[2] == pytest.approx(sps.multivariate_normal(mu, Sig, allow_singular=False).logpdf(yt), rel=1e-9)


# ---------------------------------------------------------------- invariants (pin 4)
def _gm(n, set_id, grid=(2, 8, 8)):
    return cilgen.make_patterns(123, set_id, n, grid).numpy()


def test_invariants(oracle_mod):
    O = oracle_mod
    grid = (2, 8, 8, 0.0)
    A, B = _gm(12, 0), _gm(10, 1)
    D = O.distance_matrix(A, B, grid, ALL)
    radii = np.array([np.linspace(D[q].max() * 1.01, D[q].min() * 0.99, 9) for q in range(6)])
    r = O.features(A, B, grid, ALL, radii, band=0.0)
    y = r["y"]
    assert np.all((y >= 0) & (y <= 1))
    assert np.all(np.diff(y, axis=1) <= 0)                     # non-increasing in m
    assert np.all(y[:, 0] == 1.0) and np.all(y[:, -1] == 0.0)  # R > max -> 1, R <= min -> 0
    r2 = O.features(B, A, grid, ALL, radii, band=0.0)           # y(A,B) = y(B,A)
    np.testing.assert_array_equal(r["counts"], r2["counts"])
    # translation invariance: the same constant field added to every pattern
    shift = np.float32(0.5)
    D2 = O.distance_matrix(A + shift, B + shift, grid, ALL)
    np.testing.assert_allclose(D2, D, rtol=1e-6)
    # permutation invariance within sets
    r3 = O.features(A[::-1].copy(), B[[3, 1, 0, 2, 4, 5, 9, 8, 7, 6]], grid, ALL, radii, band=0.0)
    np.testing.assert_array_equal(r3["counts"], r["counts"])
    # A = B: symmetric, zero diagonal (diagonal included, reading R6)
    DA = O.distance_matrix(A, A, grid, ALL)
    for q in range(6):
        np.testing.assert_allclose(DA[q], DA[q].T, rtol=1e-14)
        assert np.all(np.diag(DA[q]) == 0)
    # norm inequalities (w = h^2, h = 1/7)
    w = (1 / 7) ** 2
    L2, Li, W12S, W12, W1I, W1IS = D
    assert np.all(Li <= L2 / math.sqrt(w) * (1 + 1e-12))
    assert np.all(W12 <= W12S * (1 + 1e-12)) and np.all(W12S <= math.sqrt(3) * W12 * (1 + 1e-12))
    assert np.all(W1I <= W1IS) and np.all(W1IS <= 3 * W1I * (1 + 1e-12))
    assert np.all(L2 <= W12) and np.all(Li <= W1I)
    # triangle inequality d(a,b) <= d(a,c) + d(c,b)
    C = _gm(5, 2)
    DAC = O.distance_matrix(A, C, grid, ALL)
    DCB = O.distance_matrix(C, B, grid, ALL)
    for q in range(6):
        bound = (DAC[q][:, :, None] + DCB[q][None, :, :]).min(axis=1)
        assert np.all(D[q] <= bound * (1 + 1e-12))
    # homogeneity: d(l*a, l*b) = |l| d(a, b) (l a power of two keeps FP32 inputs exact)
    D4 = O.distance_matrix(A * 4, B * 4, grid, ALL)
    np.testing.assert_allclose(D4, 4 * D, rtol=1e-13)


def test_band_counts(oracle_mod):
    """lo <= cnt <= hi, and equality when no pair is within the band."""
    O = oracle_mod
    grid = (1, 6, 6, 0.0)
    A, B = _gm(8, 0, grid[:3]), _gm(8, 1, grid[:3])
    D = O.distance_matrix(A, B, grid, 1)[0]
    radii = np.array([[D.max() * 1.01, np.median(D), D.min() * 0.99]])
    r = O.features(A, B, grid, 1, radii, band=1e-6)
    assert np.all(r["lo"] <= r["counts"]) and np.all(r["counts"] <= r["hi"])
    exact = np.sort(D.ravel())
    radii2 = np.array([[exact[10] * (1 + 1e-9), exact[20], exact[30]]])   # pairs ON or near radii
    r2 = O.features(A, B, grid, 1, radii2, band=1e-6)
    assert r2["ambiguous"] >= 3
    assert r2["counts"][0, 1] == 20 and r2["counts"][0, 2] == 30         # strict <
    assert r2["hi"][0, 1] == 21 and r2["lo"][0, 1] == 20


def test_sigma_psd_rank(oracle_mod):
    rng = np.random.default_rng(2)
    Y = rng.random((6, 10))                                   # n = 6 < D = 10
    _, Sig = oracle_mod.stats(Y)
    np.testing.assert_allclose(Sig, Sig.T, rtol=0, atol=0)
    ev = np.linalg.eigvalsh(Sig)
    assert ev.min() > -1e-14
    assert np.sum(ev > 1e-12) <= 5                            # rank <= n - 1


def test_nonfinite_status(oracle_mod):
    A = _gm(3, 0, (1, 4, 4))
    B = _gm(3, 1, (1, 4, 4))
    B[1, 0, 2, 2] = np.nan
    r = oracle_mod.features(A, B, (1, 4, 4, 0.0), 1, [[10.0, 1.0]])
    assert r["status"] == 1


def test_train_vectors_vs_brute(oracle_mod):
    """Alg. 1 steps 1-2: the C(n_ens,2) subset-pair vectors in lexicographic (k, l) order equal
    the brute-force counts of each pair of subsets."""
    O = oracle_mod
    grid = (2, 4, 5, 0.0)
    n_ens, N = 4, 5
    X = cilgen.make_patterns(12, 0, n_ens * N, grid[:3]).numpy()
    Db = brute.distances(X, X, grid)
    radii = np.array([np.quantile(Db[q][Db[q] > 0], np.linspace(0.9, 0.1, 5)) for q in range(6)])
    r = O.train_vectors(X, n_ens, grid, ALL, radii, band=0.0)
    assert r["counts"].shape[0] == n_ens * (n_ens - 1) // 2
    v = 0
    for k in range(n_ens):
        for l in range(k + 1, n_ens):
            want = brute.counts(X[k * N:(k + 1) * N], X[l * N:(l + 1) * N], grid, ALL, radii)
            np.testing.assert_array_equal(r["counts"][v], want)
            v += 1
    np.testing.assert_allclose(r["y"], r["counts"].reshape(v, -1) / (N * N), rtol=0, atol=0)


def test_radii_laws(oracle_mod):
    """power law with constant ratio b and R_M/R_0 = b^-M; linear law with
    constant step h = (R_0 - R_M)/M; the margins of reading R5; ranges from brute force."""
    O = oracle_mod
    grid = (1, 5, 6, 0.0)
    A = cilgen.make_patterns(14, 0, 7, grid[:3]).numpy()
    rng = O.distance_range(A, A, grid, ALL)
    Db = brute.distances(A, A, grid)
    for q in range(6):
        assert rng[q, 1] == pytest.approx(Db[q].max(), rel=1e-12)
        assert rng[q, 0] == pytest.approx(Db[q][Db[q] > 0].min(), rel=1e-12)
    M = 8
    P_ = O.radii_from_range(rng, M, "power", 1e-3)
    L_ = O.radii_from_range(rng, M, "linear", 1e-3)
    for q in range(6):
        R0, RM = rng[q, 1] * 1.001, rng[q, 0] * 0.999
        ratios = P_[q][1:] / P_[q][:-1]
        np.testing.assert_allclose(ratios, ratios[0], rtol=1e-12)
        assert P_[q][-1] == pytest.approx(RM, rel=1e-12)
        assert P_[q][0] == pytest.approx(R0 * ratios[0], rel=1e-12)
        steps = np.diff(L_[q])
        np.testing.assert_allclose(steps, -(R0 - RM) / M, rtol=1e-10)
        assert L_[q][-1] == pytest.approx(RM, rel=1e-12)
        assert np.all(np.diff(P_[q]) < 0) and np.all(np.diff(L_[q]) < 0)


def test_minmax_scale(oracle_mod):
    """every species of every pattern spans exactly [0, 1]; a positive affine
    change of a species leaves the scaled pattern unchanged (to FP32 rounding); constant -> 0."""
    O = oracle_mod
    grid = (2, 6, 7, 0.0)
    X = cilgen.make_patterns(17, 0, 5, grid[:3]).numpy()
    Y = O.minmax_scale(X, grid)
    for s in range(2):
        assert np.all(Y[:, s].reshape(5, -1).min(axis=1) == 0.0)
        assert np.all(Y[:, s].reshape(5, -1).max(axis=1) == 1.0)
    X2 = X.copy()
    X2[:, 1] = 3.0 * X2[:, 1] - 7.0
    np.testing.assert_allclose(O.minmax_scale(X2, grid), Y, atol=2e-6)
    X3 = X.copy()
    X3[2, 0] = 4.0
    assert np.all(O.minmax_scale(X3, grid)[2, 0] == 0.0)


def test_gradient_species_mask(oracle_mod):
    """PAPER.md:526 (RD-ODE): gradient-based norms w.r.t. selected species only.  With only
    species 1 selected, the derivative sub-norms equal those of the one-species pattern made
    of species 1; the value terms are unchanged; brute force agrees."""
    O = oracle_mod
    grid = (2, 1, 20, 0.0)
    X = cilgen.make_patterns(19, 0, 6, grid[:3]).numpy()
    a, b = X[0], X[1]
    s_all = O.subnorms(a, b, grid)
    s_m = O.subnorms(a, b, grid + (0b10,))
    s_1 = O.subnorms(a[1:2], b[1:2], (1, 1, 20, 1.0 / 19))
    assert s_m[0] == pytest.approx(s_all[0], rel=1e-14) and s_m[3] == s_all[3]
    assert s_m[1] == pytest.approx(s_1[1], rel=1e-14) and s_m[4] == pytest.approx(s_1[4], rel=1e-14)
    assert s_m[1] < s_all[1]
    D = O.distance_matrix(X[:3], X[3:], grid + (0b10,), ALL)
    np.testing.assert_allclose(D, brute.distances(X[:3], X[3:], grid + (0b10,)), rtol=1e-12)
