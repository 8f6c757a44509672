"""Small cases of every kernel family, for compute-sanitizer (one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py

C1 (all six measures, every engine), a small C3-shaped case (all six measures, several tiles, ragged),
a small C6-shaped SCIL-with-bootstrapping evaluation (bin matrix, row-dot resample, y~ leg), a small
SCIL (Alg. 3) evaluation with column segments, the Alg. 1 training vectors and the stats / loglik
tails.  Prints one line per case; exits non-zero on a library error.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cilgen  # noqa: E402
import paper_2203_14742_b200 as cil  # noqa: E402


def radii_for(A, B, grid, mask, M):
    rng, _ = cil.distance_range(A, B, grid, mask)
    r, _ = cil.radii_from_range(rng, M)
    return r[0]


def main():
    dev = torch.device("cuda")
    # C1: 20 x 20 of 32x32, every engine, all six measures
    g1 = (1, 32, 32, 0.0)
    A = cilgen.make_set(cilgen.config_seed(1), 0, 20, g1[:3], device=dev)
    B = cilgen.make_set(cilgen.config_seed(1), 1, 20, g1[:3], device=dev)
    R = radii_for(A, B, g1, cil.ALL, 10)
    for e in ("AUTO", "SIMT", "TC_I8", "TC_3XBF16", "TC_3XTF32"):
        c, y, st = cil.features(A, B, g1, cil.ALL, R, engine=getattr(cil, "ENGINE_" + e))
        torch.cuda.synchronize()
        print("C1", e, int(st[0]), c[0, :, 0].tolist())
    # small C3 shape: 2 x 32 x 32, 300 x 260, all six measures (three-phase INT8 + CUDA cores)
    g3 = (2, 32, 32, 0.0)
    A = cilgen.make_set(cilgen.config_seed(3), 0, 300, g3[:3], device=dev)
    B = cilgen.make_set(cilgen.config_seed(3), 1, 260, g3[:3], device=dev)
    R = radii_for(A[:64], B[:64], g3, cil.ALL, 20)
    c, y, st = cil.features(A, B, g3, cil.ALL, R)
    torch.cuda.synchronize()
    print("C3-small", int(st[0]), c[0, :, 10].tolist())
    from paper_2203_14742_b200 import _capi as _c
    _c.lib.cil_diag_recheck_sort_min(1)                   # the row-bucketed re-check on every list
    try:
        c2, y2, st2 = cil.features(A, B, g3, cil.ALL, R)
        bb, stb = cil.bin_matrix(A[:100], A[:100], g3, cil.ALL, R)
        torch.cuda.synchronize()
    finally:
        _c.lib.cil_diag_recheck_sort_min(0)
    print("C3-small bucketed", int(st2[0]), int(stb[0]), bool(torch.equal(c2, c)))
    # bin matrix (bootstrap) of the same sets, all measures
    bins, st = cil.bin_matrix(A[:100], B[:90], g3, cil.ALL, R)
    torch.cuda.synchronize()
    print("bins", int(st[0]), int(bins.sum()))
    # small C6: SCIL with bootstrapping, 3 proposals x pool 300 of 16x16x2, N_set 20, 64 replicates
    g6 = (2, 16, 16, 0.0)
    P, Nsyn, Nset, nrep = 3, 300, 20, 64
    pools = torch.stack([cilgen.make_set(cilgen.config_seed(6), 10 + p, Nsyn, g6[:3]) for p in range(P)]).to(dev)
    data = cilgen.make_set(cilgen.config_seed(6), 99, Nset, g6[:3], device=dev)
    d = [cilgen.boot_draws_a2(cilgen.config_seed(6), p, nrep, Nsyn, Nset) for p in range(P)]
    I1 = torch.tensor(np.stack([x[0] for x in d]), device=dev)
    I2 = torch.tensor(np.stack([x[1] for x in d]), device=dev)
    J = torch.tensor(np.stack([x[2] for x in d]), device=dev)
    Rb = radii_for(pools[0, :64], pools[0, 64:128], g6, cil.L2, 13)
    out, st = cil.synth_loglik_boot(pools, data, Nset, I1, I2, J, g6, cil.L2, Rb[None].repeat(P, 1, 1), ridge=1e-6)
    torch.cuda.synchronize()
    print("C6-small", st.tolist(), out[:, 2].tolist())
    # small SCIL (Alg. 3) with column segments: n_ens 4, 30 + 25 rows per subset
    g4 = (1, 16, 16, 0.0)
    n_ens, Ns, Nt = 4, 30, 25
    pools = torch.stack([cilgen.make_set(cilgen.config_seed(4), p, n_ens * (Ns + Nt), g4[:3]) for p in range(2)]).to(dev)
    data = cilgen.make_set(cilgen.config_seed(4), 500, Ns, g4[:3], device=dev)
    R4 = radii_for(pools[0, :60], pools[0, 60:120], g4, cil.L2 | cil.W12, 8)
    out, st = cil.synth_loglik(pools, n_ens, Ns, Nt, data, torch.tensor([1, 2], dtype=torch.int32, device=dev), g4,
                               cil.L2 | cil.W12, R4[None].repeat(2, 1, 1), ridge=1e-6)
    torch.cuda.synchronize()
    print("SCIL-small", st.tolist(), out[:, 2].tolist())
    # Alg. 1 training vectors (one panel against itself, k < l blocks)
    X = cilgen.make_set(cilgen.config_seed(7), 0, 5 * 40, g3[:3], device=dev)
    Y, st = cil.train_vectors(X, 5, g3, cil.ALL, R)
    torch.cuda.synchronize()
    print("train", int(st[0]), tuple(Y.shape))
    mu, Sig = cil.stats(Y[0])
    o, st = cil.loglik(mu, Sig, Y[0, :3], ridge=1e-9)
    torch.cuda.synchronize()
    print("stats/loglik", st.tolist())
    # K > 65536 (two exact int32 chunks per phase, the two-pass pack), all six measures
    g5 = (2, 256, 256, 0.0)
    A = cilgen.make_set(cilgen.config_seed(5), 0, 10, g5[:3], device=dev)
    B = cilgen.make_set(cilgen.config_seed(5), 1, 12, g5[:3], device=dev)
    R5 = radii_for(A, B, g5, cil.ALL, 6)
    for m in (cil.L2, cil.ALL):
        c, y, st = cil.features(A, B, g5, m, R5 if m == cil.ALL else R5[:1])
        torch.cuda.synchronize()
        print("C5-tiny", hex(m), int(st[0]), c[0, :, 3].tolist())
    # near-duplicates (every pair of (i, i) within 1e-6 of each other)
    Bn = (A.double() + 1e-6 * torch.randn(A.shape, device=dev, dtype=torch.float64)).float()
    c, y, st = cil.features(A, Bn, g5, cil.ALL, radii_for(A, Bn, g5, cil.ALL, 6))
    torch.cuda.synchronize()
    print("near-dup", int(st[0]), c[0, :, -1].tolist())
    from paper_2203_14742_b200 import _capi
    v = int(_capi.lib.cil_diag_bounds_violations())
    print("bounds violations:", v, "(-1 = not a bounds-checked build)")
    if v > 0:
        sys.exit(3)


if __name__ == "__main__":
    main()
