"""Pins for the oracle's bootstrap estimators (Alg. A1 / A2): identity
draws reduce to Eq. (1) on the fixed sets; a single repeated pattern gives the closed form
n1*n2*[d(a,b) < R]; every replicate equals the independent NumPy brute force on the
explicitly resampled sets; Alg. A2 composed from brute-force counts, numpy cov and scipy
logpdf.  CPU only.
"""
import numpy as np
import pytest
from scipy import stats as sps

import brute
import cilgen

ALL = 0x3F


def _radii(D, sel, M=6):
    return np.array([np.quantile(D[q][D[q] > 0], np.linspace(0.9, 0.1, M)) for q in sel])


def test_identity_draws_equal_plain_counts(oracle_mod):
    O = oracle_mod
    grid = (2, 5, 6, 0.0)
    A = cilgen.make_patterns(3, 0, 7, grid[:3]).numpy()
    B = cilgen.make_patterns(3, 1, 5, grid[:3]).numpy()
    D = brute.distances(A, B, grid)
    radii = _radii(D, range(6))
    r = O.resample_features(A, B, grid, ALL, radii, np.arange(7)[None], np.arange(5)[None], band=0.0)
    plain = O.features(A, B, grid, ALL, radii, band=0.0)
    np.testing.assert_array_equal(r["counts"][0], plain["counts"])
    np.testing.assert_allclose(r["y"][0], plain["y"].ravel(), rtol=0, atol=0)


def test_repeated_single_pattern_closed_form(oracle_mod):
    """s1 = {a, a, ..., a} (n1 draws), s2 = {b, ..., b} (n2): counts = n1*n2*[d(a,b) < R_m]."""
    O = oracle_mod
    grid = (1, 6, 6, 0.0)
    A = cilgen.make_patterns(4, 0, 4, grid[:3]).numpy()
    B = cilgen.make_patterns(4, 1, 4, grid[:3]).numpy()
    D = brute.distances(A, B, grid)
    radii = _radii(D, range(6), M=5)
    a, b, n1, n2 = 2, 1, 3, 5
    r = O.resample_features(A, B, grid, ALL, radii, np.full((1, n1), a), np.full((1, n2), b), band=0.0)
    want = np.stack([n1 * n2 * (D[q, a, b] < radii[q]) for q in range(6)]).astype(np.int64)
    np.testing.assert_array_equal(r["counts"][0], want)
    np.testing.assert_allclose(r["y"][0], (want / (n1 * n2)).ravel(), rtol=0, atol=0)


@pytest.mark.parametrize("grid", [(2, 4, 5, 0.0), (1, 1, 12, 0.0)])
def test_resample_vs_brute(oracle_mod, grid):
    O = oracle_mod
    mask = ALL if grid[1] > 1 else 0b110011
    sel = [q for q in range(6) if (mask >> q) & 1]
    A = cilgen.make_patterns(5, 0, 9, grid[:3]).numpy()
    B = cilgen.make_patterns(5, 1, 8, grid[:3]).numpy()
    radii = _radii(brute.distances(A, B, grid), sel)
    I1, I2 = cilgen.boot_draws_a1(7, 0, 6, 8)
    I1 = I1 % 9
    r = O.resample_features(A, B, grid, mask, radii, I1, I2, band=0.0)
    for k in range(6):
        np.testing.assert_array_equal(r["counts"][k], brute.counts(A[I1[k]], B[I2[k]], grid, mask, radii))
    # with-repetition draws really repeat (so the test exercises multiplicities)
    assert any(len(set(I1[k])) < I1.shape[1] for k in range(6))


def test_bad_index_rejected(oracle_mod):
    O = oracle_mod
    grid = (1, 4, 4, 0.0)
    A = cilgen.make_patterns(1, 0, 3, grid[:3]).numpy()
    with pytest.raises(ValueError):
        O.resample_features(A, A, grid, 1, np.array([[2.0, 1.0]]), np.array([[0, 3]]), np.array([[0, 1]]))


def test_synth_boot_vs_brute(oracle_mod):
    """Alg. A2 composed from brute-force counts on the resampled sets, numpy mean / cov and
    scipy's multivariate normal logpdf."""
    O = oracle_mod
    grid = (2, 4, 5, 0.0)
    N_syn, N_set, n_rep = 14, 4, 9
    pool = cilgen.make_patterns(8, 0, N_syn, grid[:3]).numpy()
    data = cilgen.make_patterns(8, 1, N_set, grid[:3]).numpy()
    mask = 0b000011
    sel = [0, 1]
    radii = _radii(brute.distances(pool, pool, grid), sel, M=4)
    I1, I2, J = cilgen.boot_draws_a2(9, 0, n_rep, N_syn, N_set)
    for k in range(n_rep):                      # step 2.2 reading: s^2 avoids the patterns of s^1
        assert not set(I1[k]) & set(I2[k])
    assert len(set(J)) == N_syn - N_set
    out, st, Y = O.synth_boot(pool, data, N_set, I1, I2, J, grid, mask, radii, ridge=1e-6)
    Nt = N_syn - N_set
    Yb = np.array([(brute.counts(pool[I1[k]], pool[I2[k]], grid, mask, radii) / (N_set * Nt)).ravel()
                   for k in range(n_rep)])
    yt = (brute.counts(data, pool[J], grid, mask, radii) / (N_set * Nt)).ravel()
    np.testing.assert_array_equal(Y[:-1], Yb)
    np.testing.assert_array_equal(Y[-1], yt)
    mu = Yb.mean(0)
    Sig = np.cov(Yb, rowvar=False, ddof=1) + 1e-6 * np.eye(Yb.shape[1])
    assert st == 0
    assert out[2] == pytest.approx(sps.multivariate_normal(mu, Sig).logpdf(yt), rel=1e-9)


def test_a2_draw_recipe():
    """The harness draws: with replacement, s^2 from the complement of s^1, J a subset."""
    I1, I2, J = cilgen.boot_draws_a2(1, 3, 200, 60, 10)
    assert I1.shape == (200, 10) and I2.shape == (200, 50) and J.shape == (50,)
    assert I1.min() >= 0 and I1.max() < 60 and I2.min() >= 0 and I2.max() < 60
    assert all(not set(I1[k]) & set(I2[k]) for k in range(200))
    assert sum(len(set(I1[k])) < 10 for k in range(200)) > 100          # repetitions happen
    assert len(set(J.tolist())) == 50
    I1b, I2b, Jb = cilgen.boot_draws_a2(1, 3, 200, 60, 10)
    np.testing.assert_array_equal(I1, I1b)                                 # seeded, reproducible
