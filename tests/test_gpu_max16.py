"""GPU parity of the max family on the 15-bit fixed-point integer engine (max16.cu) and of the
row-bucketed re-check (recheck.cu) against the FP64 oracle.

max16.cu decides Linf, W1inf and W1infsum (Eqs. (6), (9), (10)) from quantised
operands with a rigorous interval and re-checks the pairs whose interval holds a radius, so its
counts must be the oracle's (strict <, Eq. (1)) up to the north-star band:
lo <= gpu <= hi.  The cases here stress what the quantisation depends on: a large common offset
(the per-item centre), very different scales per region, constant regions (scale 0), narrow
grids, ragged padding, 1-D grids, species masks, the mirrored bin matrix, and radii placed AT pair
distances so that many pairs take the re-check.
"""
import numpy as np
import pytest
import torch

import cilgen

pytestmark = pytest.mark.gpu

BAND = 1e-6
MAXF = 0x32          # LINF | W1INF | W1INFSUM


@pytest.fixture(scope="module")
def cil():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2203_14742_b200 as cil
    return cil


def _check(gpu, ref, what):
    gpu = np.asarray(gpu)
    ok = np.all(ref["lo"] <= gpu) and np.all(gpu <= ref["hi"])
    assert ok, (f"{what}\ngpu    {gpu.tolist()}\noracle {ref['counts'].tolist()}\n"
                f"lo     {ref['lo'].tolist()}\nhi     {ref['hi'].tolist()}")


def _radii_at_distances(D, M, every=3):
    """Radii equal to actual pair distances (every pair at such a distance is ambiguous for any
    engine and goes through the re-check), strictly decreasing."""
    out = []
    for d in D:
        u = np.unique(d[d > 0])[::-1]
        r = u[1:1 + every * M:every]
        if len(r) < M:
            r = np.geomspace(u[0] * 0.99, max(u[-1], 1e-12) * 1.01, M)
        out.append(r)
    return np.array(out)


def _features(cil, A, B, grid, mask, radii, engine="AUTO"):
    dev = torch.device("cuda")
    c, _, st = cil.features(A.to(dev), B.to(dev), grid, mask, torch.tensor(radii, device=dev),
                            engine=getattr(cil, "ENGINE_" + engine))
    torch.cuda.synchronize()
    return c[0].cpu().numpy(), int(st[0])


@pytest.mark.parametrize("engine", ["AUTO", "TC_I8"])
@pytest.mark.parametrize("offset,scale", [(1000.0, 1.0), (-3.5, 1e-3), (0.0, 1e4)])
def test_max16_offset_and_scale(cil, oracle_mod, engine, offset, scale):
    """A common offset far from zero (the centre c of each region) and extreme scales."""
    O = oracle_mod
    grid = (2, 24, 20, 0.0)
    A = cilgen.make_set(314, 0, 90, grid[:3]) * scale + offset
    B = cilgen.make_set(314, 1, 75, grid[:3]) * scale + offset
    for mask in (MAXF, 0x3F):
        D = O.distance_matrix(A[:30].numpy(), B[:30].numpy(), grid, mask)
        radii = _radii_at_distances(D, 10)
        c, st = _features(cil, A, B, grid, mask, radii, engine)
        assert st == 0
        _check(c, O.features(A.numpy(), B.numpy(), grid, mask, radii, band=BAND), f"{engine} {offset} {scale} {mask:#x}")


@pytest.mark.parametrize("grid", [(1, 12, 4, 0.0), (1, 1, 64, 0.0), (3, 7, 12, 0.0), (2, 1, 64, 0.0, 0b10),
                                  (2, 16, 16, 0.0, 0b01)])
def test_max16_grids_and_masks(cil, oracle_mod, grid):
    """Narrow grids (W = 4), 1-D grids, ragged padding (K_aug not a multiple of the 64-element
    chunk), species masks (R18)."""
    O = oracle_mod
    A = cilgen.make_set(2718, 0, 70, grid[:3])
    B = cilgen.make_set(2718, 1, 66, grid[:3])
    D = O.distance_matrix(A[:30].numpy(), B[:30].numpy(), grid, MAXF)
    radii = _radii_at_distances(D, 8)
    c, st = _features(cil, A, B, grid, MAXF, radii)
    assert st == 0
    _check(c, O.features(A.numpy(), B.numpy(), grid, MAXF, radii, band=BAND), f"grid {grid}")


def test_max16_constant_regions(cil, oracle_mod):
    """Patterns constant along x (D_x region all zero: scale 0) and an all-equal item (every
    distance 0)."""
    O = oracle_mod
    grid = (1, 12, 16, 0.0)
    rng = np.random.default_rng(5)
    col = rng.standard_normal((60, 1, 12, 1)).astype(np.float32)
    A = torch.from_numpy(np.repeat(col[:32], 16, axis=3))
    B = torch.from_numpy(np.repeat(col[28:], 16, axis=3))
    D = O.distance_matrix(A.numpy(), B.numpy(), grid, MAXF)
    radii = _radii_at_distances(D, 6)
    c, st = _features(cil, A, B, grid, MAXF, radii)
    assert st == 0
    _check(c, O.features(A.numpy(), B.numpy(), grid, MAXF, radii, band=BAND), "constant along x")
    Z = torch.full((20, 1, 12, 16), 0.75)
    c, st = _features(cil, Z, Z[:13].clone(), grid, MAXF, np.tile(np.geomspace(1.0, 0.01, 5), (3, 1)))
    assert st == 0 and (c == 20 * 13).all()     # d = 0 < every radius (strict <, Eq. (1))


def test_max16_bin_matrix_mirrored(cil, oracle_mod):
    """The bootstrap's bin matrix of a panel against itself (mirrored writes), max family."""
    O = oracle_mod
    grid = (2, 16, 16, 0.0)
    A = cilgen.make_set(77, 0, 90, grid[:3], "FHN")
    D = O.distance_matrix(A.numpy(), A.numpy(), grid, MAXF)
    radii = _radii_at_distances(D, 9, every=5)
    dev = torch.device("cuda")
    bins, st = cil.bin_matrix(A.to(dev), A.to(dev), grid, MAXF, torch.tensor(radii, device=dev),
                              engine=cil.ENGINE_AUTO)
    torch.cuda.synchronize()
    assert int(st[0]) == 0
    for q in range(3):
        lo = (D[q][..., None] < radii[q] * (1 - BAND)).sum(-1)
        hi = (D[q][..., None] < radii[q] * (1 + BAND)).sum(-1)
        g = bins[0, q].cpu().numpy().astype(np.int64)
        bad = (g < lo) | (g > hi)
        assert not bad.any(), (q, np.argwhere(bad)[:5].tolist())


@pytest.mark.parametrize("engine", ["AUTO", "SIMT", "TC_I8"])
@pytest.mark.parametrize("mode", ["features", "bins"])
def test_recheck_row_bucketed(cil, oracle_mod, engine, mode):
    """The row-bucketed re-check (forced for every list, cil_diag_recheck_sort_min(1)) gives the
    same results as the entry-by-entry pass, and the oracle's."""
    from paper_2203_14742_b200 import _capi
    O = oracle_mod
    grid = (2, 20, 20, 0.0)
    A = cilgen.make_set(4242, 0, 80, grid[:3])
    B = (A[:60].double() + 1e-6 * torch.randn(60, *grid[:3], dtype=torch.float64,
                                               generator=torch.Generator().manual_seed(9))).float()
    B = torch.cat([B, cilgen.make_set(4242, 1, 20, grid[:3])])
    D = O.distance_matrix(A.numpy(), B.numpy(), grid, 0x3F)
    radii = _radii_at_distances(D, 12)
    dev = torch.device("cuda")
    R = torch.tensor(radii, device=dev)
    e = getattr(cil, "ENGINE_" + engine)
    out = []
    for sort_min in (0, 1):
        _capi.lib.cil_diag_recheck_sort_min(sort_min)
        try:
            if mode == "features":
                c, _, st = cil.features(A.to(dev), B.to(dev), grid, 0x3F, R, engine=e)
                torch.cuda.synchronize()
                out.append(c[0].cpu().numpy())
            else:
                bins, st = cil.bin_matrix(A.to(dev), B.to(dev), grid, 0x3F, R, engine=e)
                torch.cuda.synchronize()
                out.append(bins[0].cpu().numpy())
        finally:
            _capi.lib.cil_diag_recheck_sort_min(0)
        assert int(st[0]) == 0
    assert np.array_equal(out[0], out[1]), engine
    if mode == "features":
        _check(out[1], O.features(A.numpy(), B.numpy(), grid, 0x3F, radii, band=BAND), engine)
    else:
        for q in range(6):
            lo = (D[q][..., None] < radii[q] * (1 - BAND)).sum(-1)
            hi = (D[q][..., None] < radii[q] * (1 + BAND)).sum(-1)
            g = out[1][q].astype(np.int64)
            assert ((g >= lo) & (g <= hi)).all(), (engine, q)


def test_recheck_huge_bucket(cil, oracle_mod):
    """One A row whose every partner sits at the same distance, with radii just above and below it
    (outside the oracle's 1e-6 band, inside the fixed-point engine's): > 1024 listed cases in one
    row bucket, so the row-bucketed re-check settles each entry by itself (no quadratic pairing);
    entry-by-entry and bucketed passes must give the oracle's counts."""
    from paper_2203_14742_b200 import _capi
    O = oracle_mod
    grid = (1, 16, 16, 0.0)
    rng = np.random.default_rng(11)
    a0 = (rng.integers(0, 1024, size=(1, 1, 16, 16)) / 1024.0).astype(np.float32)
    a1 = (rng.integers(0, 1024, size=(1, 1, 16, 16)) / 1024.0).astype(np.float32)
    A = torch.from_numpy(np.concatenate([a0, a1]))
    B = torch.from_numpy(np.repeat(a0 + np.float32(0.5), 1500, axis=0))      # exact: d(0, j) = 0.5 for all j
    radii = np.tile(np.array([0.5 * (1 + 1e-5), 0.5 * (1 - 1e-5), 0.01]), (3, 1))
    ref = O.features(A.numpy(), B.numpy(), grid, MAXF, radii, band=BAND)
    for sort_min in (0, 1):
        _capi.lib.cil_diag_recheck_sort_min(sort_min)
        try:
            c, st = _features(cil, A, B, grid, MAXF, radii)
            listed, _ = cil.recheck_count(1, 2, 1500, grid, MAXF, 3)
        finally:
            _capi.lib.cil_diag_recheck_sort_min(0)
        assert st == 0 and listed >= 3 * 1500, listed            # every (0, j) case of every measure
        _check(c, ref, f"sort_min {sort_min}")


@pytest.mark.parametrize("mode", ["features", "bins"])
def test_concurrent_engines_identical(cil, oracle_mod, mode):
    """The max family on the side stream concurrently with the three-phase tensor-core family gives
    the same counts / bins as the serial order (cil_diag_concurrent_engines), and the oracle's."""
    from paper_2203_14742_b200 import _capi
    O = oracle_mod
    grid = (2, 24, 24, 0.0)
    A = cilgen.make_set(8080, 0, 150, grid[:3])
    B = cilgen.make_set(8080, 1, 130, grid[:3])
    D = O.distance_matrix(A[:40].numpy(), B[:40].numpy(), grid, 0x3F)
    radii = _radii_at_distances(D, 10)
    dev = torch.device("cuda")
    R = torch.tensor(radii, device=dev)
    out = []
    for on in (0, 1):
        _capi.lib.cil_diag_concurrent_engines(on)
        try:
            if mode == "features":
                c, _, st = cil.features(A.to(dev), B.to(dev), grid, 0x3F, R)
            else:
                c, st = cil.bin_matrix(A.to(dev), B.to(dev), grid, 0x3F, R)
            torch.cuda.synchronize()
        finally:
            _capi.lib.cil_diag_concurrent_engines(1)
        assert int(st[0]) == 0
        out.append(c[0].cpu().numpy())
    assert np.array_equal(out[0], out[1])
    if mode == "features":
        _check(out[1], O.features(A.numpy(), B.numpy(), grid, 0x3F, radii, band=BAND), "concurrent")


def test_max16_per_item_scales(cil, oracle_mod):
    """Several items in one call, each with its own range (the quantisation scale and centre are per
    item and region): scales 1e-2, 1, 1e3 and offsets -50, 0, 7 in one batch, per-item radii."""
    O = oracle_mod
    grid = (2, 12, 16, 0.0)
    P, N, Nt, M = 3, 70, 55, 8
    scales, offs = (1e-2, 1.0, 1e3), (-50.0, 0.0, 7.0)
    A = torch.stack([cilgen.make_set(55, 2 * p, N, grid[:3]) * scales[p] + offs[p] for p in range(P)])
    B = torch.stack([cilgen.make_set(55, 2 * p + 1, Nt, grid[:3]) * scales[p] + offs[p] for p in range(P)])
    radii = []
    for p in range(P):
        D = O.distance_matrix(A[p, :30].numpy(), B[p, :30].numpy(), grid, 0x3F)
        radii.append(_radii_at_distances(D, M))
    radii = np.stack(radii)
    dev = torch.device("cuda")
    c, _, st = cil.features(A.to(dev), B.to(dev), grid, 0x3F, torch.tensor(radii, device=dev))
    torch.cuda.synchronize()
    assert (st.cpu().numpy() == 0).all()
    for p in range(P):
        _check(c[p].cpu().numpy(), O.features(A[p].numpy(), B[p].numpy(), grid, 0x3F, radii[p], band=BAND), f"item {p}")
