"""Multi-process sharding logic on CPU: world-size-2 gloo groups, the FP64 oracle as the
per-shard compute (the CUDA kernels need a GPU; here only the host-side partition and
the collective are under test)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_features(A, B, grid, mask, radii, want_y=False, **kw):
    from oracle import oracle as O
    r = O.features(A.numpy(), B.numpy(), grid, mask, radii.numpy(), band=0.0, nthreads=1)
    return torch.tensor(r["counts"][None]), None, torch.zeros(1, dtype=torch.int32)


def _normalize(counts, npairs):
    return counts.to(torch.float64) / npairs


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import cilgen
        from paper_2203_14742_b200 import sharding
        grid = (1, 6, 6, 0.0)
        N, Nt = 23, 9
        A = cilgen.make_set(77, 0, N, grid[:3])
        B = cilgen.make_set(77, 1, Nt, grid[:3])
        radii = torch.tensor([np.geomspace(3.0, 0.5, 6), np.geomspace(3.0, 0.3, 6)])
        lo, hi = sharding.row_range(N, world, rank)
        counts, y, st = sharding.sharded_features(A[lo:hi], B, grid, 0b11, radii, N,
                                                  features_fn=_oracle_features, normalize_fn=_normalize)
        # per-item sharding + all_gather of vectors
        Pl = 3
        y_local = torch.full((Pl, 4), float(rank)) + torch.arange(Pl * 4, dtype=torch.float64).view(Pl, 4)
        Y = sharding.gather_vectors(y_local)
        # item status words are OR-ed across ranks (rank r reports bit r of NONFINITE / NOTPD /
        # BADRADII / OVERFLOW: a MAX reduction would drop the lower bits)
        st_local = torch.tensor([1 << rank, 0, (1 << rank) | 16], dtype=torch.int32)
        st_or = sharding.or_status(st_local)
        q.put((rank, counts.numpy(), y.numpy(), Y.numpy(), (lo, hi), st_or.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_counts_equal_unsharded(oracle_mod, world):
    import cilgen
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    grid = (1, 6, 6, 0.0)
    A = cilgen.make_set(77, 0, 23, grid[:3]).numpy()
    B = cilgen.make_set(77, 1, 9, grid[:3]).numpy()
    radii = np.array([np.geomspace(3.0, 0.5, 6), np.geomspace(3.0, 0.3, 6)])
    full = oracle_mod.features(A, B, grid, 0b11, radii, band=0.0)
    ranges = [r[4] for r in res]
    want = sum(1 << r for r in range(world))
    for r in res:
        assert r[5].tolist() == [want, 0, want | 16]
    assert ranges[0][0] == 0 and ranges[-1][1] == 23
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    for rank, counts, y, Y, _, _ in res:
        np.testing.assert_array_equal(counts[0], full["counts"])          # identical on every rank
        np.testing.assert_array_equal(y[0], full["counts"] / (23 * 9))
        assert Y.shape == (world * 3, 4)
        for r in range(world):
            np.testing.assert_array_equal(Y[3 * r:3 * r + 3], r + np.arange(12).reshape(3, 4))


def test_row_range_partition():
    from paper_2203_14742_b200 import sharding
    for n in (0, 1, 7, 20000):
        for w in (1, 2, 3, 8):
            rs = [sharding.row_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1


def _ring_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import cilgen
        from paper_2203_14742_b200 import sharding
        grid = (1, 6, 6, 0.0)
        N, Nt = 17, 11
        A = cilgen.make_set(78, 0, N, grid[:3])
        B = cilgen.make_set(78, 1, Nt, grid[:3])
        radii = torch.tensor([np.geomspace(3.0, 0.5, 6), np.geomspace(3.0, 0.3, 6)])
        a0, a1 = sharding.row_range(N, world, rank)
        b0, b1 = sharding.row_range(Nt, world, rank)
        counts, y, st = sharding.ring_features(A[a0:a1], B[b0:b1].clone(), grid, 0b11, radii, N, Nt,
                                               features_fn=_oracle_features, normalize_fn=_normalize)
        q.put((rank, counts.numpy(), y.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ring_pass_counts_equal_unsharded(oracle_mod, world):
    """Both A and B sharded; B shards travel around the ring: the counts on
    every rank equal the unsharded oracle counts (uneven shards: 17 and 11 rows)."""
    import cilgen
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ring_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    grid = (1, 6, 6, 0.0)
    A = cilgen.make_set(78, 0, 17, grid[:3]).numpy()
    B = cilgen.make_set(78, 1, 11, grid[:3]).numpy()
    radii = np.array([np.geomspace(3.0, 0.5, 6), np.geomspace(3.0, 0.3, 6)])
    full = oracle_mod.features(A, B, grid, 0b11, radii, band=0.0)
    for rank, counts, y in res:
        np.testing.assert_array_equal(counts[0], full["counts"])
        np.testing.assert_array_equal(y[0], full["counts"] / (17 * 11))


def test_bench_rank_mismatch_fails_loudly():
    """bench.py --gpus N under a torchrun environment with another WORLD_SIZE must refuse to run
    (--gpus was silently ignored)."""
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--impl", "reference"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=2" in (r.stderr + r.stdout)


def test_bench_launches_ranks_reference_arm():
    """bench.py --gpus 2 without a torchrun environment re-launches itself as two ranks (torch.distributed.run
    on 127.0.0.1); on the reference arm rank 0 alone prints the JSON line and the other rank exits 0."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--steps", "1", "--warmup", "1"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
