"""GPU parity of the bootstrap estimators (Alg. A1 / A2) through the C
ABI against the FP64 oracle on the same seeded inputs and draws.  Tolerances as in
test_gpu_parity: a pair's bin is exact unless its distance lies within 1e-6 relative of a
radius (then either neighbouring bin is correct); resampled counts within the oracle's
band counts lo <= gpu <= hi; mu / Sigma / loglik within 1e-6.
"""
import numpy as np
import pytest
import torch

import cilgen

pytestmark = pytest.mark.gpu

BAND = 1e-6


@pytest.fixture(scope="module")
def cil():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2203_14742_b200 as cil
    return cil


def _radii(D, M, lo=0.02, hi=0.98):
    out = []
    for d in D:
        d = d[d > 0].ravel()
        R0, RM = np.quantile(d, hi), np.quantile(d, lo)
        out.append(R0 * (RM / R0) ** (np.arange(0, M) / (M - 1)))
    return np.array(out)


def _bins_ok(bins, D, radii):
    """bins[q][i][j] == #{m : D < R} except within the 1e-6 band, where any bin between the
    band's two counts is correct."""
    lo = (D[:, :, :, None] < radii[:, None, None, :] * (1 - BAND)).sum(-1)
    hi = (D[:, :, :, None] < radii[:, None, None, :] * (1 + BAND)).sum(-1)
    ok = (lo <= bins) & (bins <= hi)
    assert ok.all(), f"{(~ok).sum()} bins outside the band; first at {np.argwhere(~ok)[0]}"
    return int((lo != hi).sum())


@pytest.mark.parametrize("engine", ["AUTO", "SIMT"])
def test_bin_matrix_all_measures(cil, oracle_mod, engine):
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 16, 16, 0.0)
    P, N, Nt = 2, 300, 277                       # several 256-row tiles and ragged tails
    A = torch.stack([cilgen.make_set(31, 2 * p, N, grid[:3]) for p in range(P)])
    B = torch.stack([cilgen.make_set(31, 2 * p + 1, Nt, grid[:3]) for p in range(P)])
    D0 = O.distance_matrix(A[0, :60].numpy(), B[0, :60].numpy(), grid, 0x3F)
    radii = _radii(D0, 9)
    bins, st = cil.bin_matrix(A.to(dev), B.to(dev), grid, 0x3F, torch.tensor(radii, device=dev),
                              engine=getattr(cil, "ENGINE_" + engine))
    torch.cuda.synchronize()
    assert int(st.max()) == 0
    for p in range(P):
        D = O.distance_matrix(A[p].numpy(), B[p].numpy(), grid, 0x3F)
        _bins_ok(bins[p].cpu().numpy(), D, radii)


def test_bin_matrix_c2_item_int8(cil, oracle_mod):
    """A full C2-shaped item (500 x 500, 64x64x2, L2) on the INT8 engine, per-item radii."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 64, 64, 0.0)
    seed = cilgen.config_seed(2)
    A = cilgen.make_set(seed, 0, 500, grid[:3])
    B = cilgen.make_set(seed, 1, 500, grid[:3])
    D = O.distance_matrix(A.numpy(), B.numpy(), grid, 0x1)
    radii = _radii(D, 13)
    bins, st = cil.bin_matrix(A.to(dev), B.to(dev), grid, 0x1, torch.tensor(radii, device=dev),
                              engine=cil.ENGINE_TC_I8)
    torch.cuda.synchronize()
    _bins_ok(bins[0].cpu().numpy(), D, radii)


def test_resample_counts_vs_oracle(cil, oracle_mod):
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (1, 12, 12, 0.0)
    N, Nt, n_rep = 40, 33, 25
    A = cilgen.make_set(41, 0, N, grid[:3])
    B = cilgen.make_set(41, 1, Nt, grid[:3])
    mask = 0b010011
    D = O.distance_matrix(A.numpy(), B.numpy(), grid, mask)
    radii = _radii(D, 7)
    I1, _ = cilgen.boot_draws_a1(42, 0, n_rep, N)
    _, I2 = cilgen.boot_draws_a1(42, 1, n_rep, Nt)
    I1 = I1[:, :17]                                  # n1 != N, n2 != Nt
    bins, st = cil.bin_matrix(A.to(dev), B.to(dev), grid, mask, torch.tensor(radii, device=dev))
    counts, y, st2 = cil.resample_counts(bins, torch.tensor(I1, device=dev)[None],
                                         torch.tensor(I2, device=dev)[None], radii.shape[1])
    torch.cuda.synchronize()
    assert int(st2.max()) == 0
    ref = O.resample_features(A.numpy(), B.numpy(), grid, mask, radii, I1, I2, band=BAND)
    c = counts[0].cpu().numpy()
    assert np.all(ref["lo"] <= c) and np.all(c <= ref["hi"])
    np.testing.assert_allclose(y[0].cpu().numpy(), c.reshape(n_rep, -1) / (I1.shape[1] * I2.shape[1]), rtol=0,
                               atol=0)


def test_resample_bad_index(cil):
    dev = torch.device("cuda")
    bins = torch.zeros((2, 1, 5, 6), dtype=torch.uint8, device=dev)
    I1 = torch.zeros((2, 3, 4), dtype=torch.int32, device=dev)
    I2 = torch.zeros((2, 3, 2), dtype=torch.int32, device=dev)
    I2[1, 2, 1] = 6                                   # out of range for item 1 only
    _, _, st = cil.resample_counts(bins, I1, I2, 4)
    torch.cuda.synchronize()
    assert st.tolist() == [0, cil.ITEM_BADINDEX]


@pytest.mark.parametrize("mask", [0b000001, 0b000011, 0b001101])   # 0b001101: the three-phase bins
def test_synth_boot_vs_oracle(cil, oracle_mod, mask):
    """Alg. A2 end to end (bins, resampling, mu/Sigma, y~, loglik) for 3 proposals."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 16, 16, 0.0)
    P, N_syn, N_set, n_rep = 3, 120, 10, 60
    pools = torch.stack([cilgen.make_set(51, 100 + p, N_syn, grid[:3], n_w=4.6 + 0.3 * p) for p in range(P)])
    data = cilgen.make_set(51, 999, N_set, grid[:3])
    sel = [q for q in range(6) if (mask >> q) & 1]
    radii, draws = [], []
    for p in range(P):
        D = O.distance_matrix(pools[p, :50].numpy(), pools[p, 50:100].numpy(), grid, mask)
        radii.append(_radii(D, 8))
        draws.append(cilgen.boot_draws_a2(52, p, n_rep, N_syn, N_set))
    radii = np.array(radii)
    I1 = np.stack([d[0] for d in draws])
    I2 = np.stack([d[1] for d in draws])
    J = np.stack([d[2] for d in draws])
    out, st, Y = cil.synth_loglik_boot(pools.to(dev), data.to(dev), N_set, torch.tensor(I1, device=dev),
                                       torch.tensor(I2, device=dev), torch.tensor(J, device=dev), grid, mask,
                                       torch.tensor(radii, device=dev), ridge=1e-5, return_Y=True)
    torch.cuda.synchronize()
    assert len(sel) * radii.shape[2] == Y.shape[2]
    for p in range(P):
        ref, rst, Yr = O.synth_boot(pools[p].numpy(), data.numpy(), N_set, I1[p], I2[p], J[p], grid, mask,
                                    radii[p], ridge=1e-5)
        Yg = Y[p].cpu().numpy()
        # the replicate vectors: a count may differ from the oracle's only for pairs in the band
        rr = O.resample_features(pools[p].numpy(), pools[p].numpy(), grid, mask, radii[p], I1[p], I2[p], band=BAND)
        npairs = N_set * (N_syn - N_set)
        c = np.rint(Yg[:-1] * npairs).astype(np.int64).reshape(rr["lo"].shape)
        assert np.all(rr["lo"] <= c) and np.all(c <= rr["hi"])
        if np.array_equal(Yg, Yr):
            assert rst == st[p].item()
            np.testing.assert_allclose(out[p].cpu().numpy(), ref, rtol=0, atol=1e-6)
        else:                                    # compare the tail on the GPU's own vectors
            mu, Sig = O.stats(Yg[:-1])
            o2, _ = O.loglik(mu, Sig, Yg[-1], ridge=1e-5)
            np.testing.assert_allclose(out[p].cpu().numpy(), o2, rtol=0, atol=1e-6)


def test_mcil_boot_stats(cil, oracle_mod):
    """Alg. A1: mu_0, Sigma_0 from bootstrap replicates of the two halves of s_data."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 16, 16, 0.0)
    N_set, n_rep = 50, 200
    data = cilgen.make_set(61, 0, N_set, grid[:3])
    h = N_set // 2
    D = O.distance_matrix(data[:h].numpy(), data[h:].numpy(), grid, 0x1)
    radii = _radii(D, 13)
    I1, I2 = cilgen.boot_draws_a1(62, 0, n_rep, h)
    mu, Sig, Y, st = cil.mcil_boot_stats(data.to(dev), grid, 0x1, torch.tensor(radii, device=dev),
                                         torch.tensor(I1, device=dev), torch.tensor(I2, device=dev))
    torch.cuda.synchronize()
    ref = O.resample_features(data[:h].numpy(), data[h:].numpy(), grid, 0x1, radii, I1, I2, band=BAND)
    c = np.rint(Y.cpu().numpy() * h * h).astype(np.int64).reshape(ref["lo"].shape)
    assert np.all(ref["lo"] <= c) and np.all(c <= ref["hi"])
    mu_r, Sig_r = O.stats(Y.cpu().numpy())
    np.testing.assert_allclose(mu.cpu().numpy(), mu_r, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(Sig.cpu().numpy(), Sig_r, rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("N_syn,N_set,n_rep,M,mask", [(300, 40, 150, 13, 0b000011), (257, 127, 9, 5, 0b000001),
                                                      (300, 40, 100, 9, 0b001101),
                                                      (1000, 50, 300, 13, 0b000001),
                                                      # K = 1700: the A row block does not fit in shared
                                                      # memory -> the streaming ring of the GEMM
                                                      (1700, 60, 40, 6, 0b000001),
                                                      # n1 = 128 > 127: the shared-atomic fallback
                                                      (300, 128, 20, 7, 0b000001),
                                                      # y~ edges: one data pattern; the 64-wide s_data
                                                      # tile full; one row past it (the wide layout)
                                                      (200, 1, 30, 5, 0b000001), (200, 64, 30, 5, 0b000001),
                                                      (200, 65, 30, 5, 0b000001)])
def test_synth_boot_tc_resample_bit_exact(cil, oracle_mod, N_syn, N_set, n_rep, M, mask):
    """The tensor-core resample inside Alg. A2 (one integer GEMM per measure: replicate row
    multiplicities x 0/1 threshold rows, then the column multiplicities in the epilogue) gives
    exactly the replicate vectors of the shared-atomic resample over the same bin matrix."""
    O = oracle_mod
    dev = torch.device("cuda")
    grid = (2, 16, 16, 0.0)
    P = 2
    pools = torch.stack([cilgen.make_set(71, 10 + p, N_syn, grid[:3], n_w=4.6 + 0.3 * p) for p in range(P)])
    data = cilgen.make_set(71, 99, N_set, grid[:3])
    radii, draws = [], []
    for p in range(P):
        D = O.distance_matrix(pools[p, :40].numpy(), pools[p, 40:80].numpy(), grid, mask)
        radii.append(_radii(D, M))
        draws.append(cilgen.boot_draws_a2(72, p, n_rep, N_syn, N_set))
    radii = torch.tensor(np.array(radii), device=dev)
    I1 = torch.tensor(np.stack([d[0] for d in draws]), device=dev)
    I2 = torch.tensor(np.stack([d[1] for d in draws]), device=dev)
    J = torch.tensor(np.stack([d[2] for d in draws]), device=dev)
    pd = pools.to(dev)
    _, st, Y = cil.synth_loglik_boot(pd, data.to(dev), N_set, I1, I2, J, grid, mask, radii, ridge=1e-5,
                                     return_Y=True)
    bins, bst = cil.bin_matrix(pd, pd, grid, mask, radii)
    _, y, rst = cil.resample_counts(bins, I1, I2, M, want_counts=False)
    torch.cuda.synchronize()
    assert st.tolist() == [0] * P and bst.tolist() == [0] * P and rst.tolist() == [0] * P
    assert torch.equal(Y[:, :n_rep], y)
    # y~ (Alg. A2 steps 4-5, computed from the pool's planes with the multiplicities of J) equals
    # the plain features of (s_data, pool[J]) — exact counts on both sides
    dd = data.to(dev)
    pj = torch.stack([pd[p][J[p].long()] for p in range(P)])
    _, yt, tst = cil.features(dd.unsqueeze(0).expand(P, *dd.shape).contiguous(), pj, grid, mask, radii)
    torch.cuda.synchronize()
    assert tst.tolist() == [0] * P
    assert torch.equal(Y[:, n_rep], yt.reshape(P, -1))


@pytest.mark.parametrize("engine_name", ["ENGINE_SIMT", "ENGINE_AUTO"])
def test_bin_matrix_symmetric_skip_equals_full(cil, engine_name):
    """A panel against itself (the pool x pool bin matrix) computes one triangle and mirrors it;
    the result equals the full computation on a separate copy of the panel, and is symmetric."""
    dev = torch.device("cuda")
    grid = (2, 16, 16, 0.0)
    P, N, M = 2, 333, 9
    mask = 0b111111
    engine = getattr(cil, engine_name)
    pools = torch.stack([cilgen.make_set(91, p, N, grid[:3]) for p in range(P)]).to(dev)
    from oracle import oracle as O
    D = O.distance_matrix(pools[0, :40].cpu().numpy(), pools[0, 40:80].cpu().numpy(), grid, mask)
    radii = torch.tensor(np.stack([_radii(D, M)] * P), device=dev)
    b_sym, s1 = cil.bin_matrix(pools, pools, grid, mask, radii, engine=engine)
    b_full, s2 = cil.bin_matrix(pools, pools.clone(), grid, mask, radii, engine=engine)
    torch.cuda.synchronize()
    assert s1.tolist() == [0] * P and s2.tolist() == [0] * P
    assert torch.equal(b_sym, b_sym.transpose(2, 3))
    assert torch.equal(b_sym, b_full)
