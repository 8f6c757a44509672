"""Multi-GPU sharding of the CIL hot path; one process per GPU,
torch.distributed for the plumbing (NCCL over NVLink on B200).

Two partitions:
  * independent problems (set pairs of Alg. 1/2, proposals theta of Alg. 3): each rank
    owns a contiguous slice of items (`item_range`) — no data-path collective;
    `gather_vectors` all-gathers the per-item feature vectors when mu_0 / Sigma_0 over
    all items are needed (Alg. 1 step 3).
  * one large set pair (C5): rank r takes A rows [r N / G, (r+1) N / G) against all of B
    (`row_range`), runs cil_features on its shard, then one all_reduce(SUM) of the int64
    count vectors — the only exchange (<= n_meas * M * 8 bytes).  Integer sums are
    order-free, so counts are bit-identical for every G.
  * a pair too large for one GPU's memory ("ring-pass of B shards"): every
    rank holds one shard of A and one of B; in G steps the B shards travel around the ring
    (send to rank r+1, receive from r-1, double-buffered so the transfer of the next shard
    overlaps the counts of the current one), each rank counting its A shard against every
    B shard; then the same all_reduce(SUM).  No rank ever holds more than 2 B shards.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def row_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced block [lo, hi) of n rows for `rank` of `world`."""
    return (n * rank) // world, (n * (rank + 1)) // world


def item_range(p: int, world: int, rank: int) -> tuple[int, int]:
    return row_range(p, world, rank)


def or_status(status: torch.Tensor, *, group=None) -> torch.Tensor:
    """Bitwise OR of the per-item status words over the group (NCCL has no BOR reduction: the bits
    are split into 0/1 planes, all-reduced with MAX, and recombined)."""
    world, _ = _world(group)
    if world == 1:
        return status
    sh = torch.arange(8, device=status.device, dtype=status.dtype)
    planes = (status.unsqueeze(-1) >> sh) & 1
    dist.all_reduce(planes, op=dist.ReduceOp.MAX, group=group)
    return (planes << sh).sum(-1).to(status.dtype)


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def sharded_features(A_local, B, grid, mask, radii, N_total: int, *, group=None, features_fn=None,
                     normalize_fn=None, **kw):
    """Counts / y of ONE large set pair whose A rows are sharded across the group.

    A_local: this rank's rows of A ([n_r, S, H, W]); B: all of B ([Nt, S, H, W]) on every
    rank.  features_fn(A, B, grid, mask, radii, **kw) -> (counts [1,q,M] int64, y, status)
    defaults to the CUDA path (`paper_2203_14742_b200.features`); normalize_fn(counts,
    npairs) -> y defaults to `cil_normalize`.  Returns (counts, y, status) of the whole
    pair, identical on every rank.
    """
    if features_fn is None:
        from . import features as features_fn  # CUDA path
    counts, _, status = features_fn(A_local, B, grid, mask, radii, want_y=False, **kw)
    world, _ = _world(group)
    if world > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
        status = or_status(status, group=group)
    npairs = float(N_total) * float(B.shape[0])
    if normalize_fn is None:
        from . import normalize as normalize_fn
    y = normalize_fn(counts, npairs)
    return counts, y, status


def gather_vectors(y_local: torch.Tensor, *, group=None) -> torch.Tensor:
    """All-gather per-item feature vectors [P_local, D] -> [world * P_local, D] (equal P_local)."""
    world, _ = _world(group)
    if world == 1:
        return y_local
    out = torch.empty((world * y_local.shape[0],) + tuple(y_local.shape[1:]), dtype=y_local.dtype,
                      device=y_local.device)
    dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
    return out


def ring_features(A_local, B_local, grid, mask, radii, N_total: int, Nt_total: int, *, group=None,
                  features_fn=None, normalize_fn=None, **kw):
    """Counts / y of ONE set pair with both A and B row-sharded across the group (ring-pass).

    A_local: this rank's rows of A; B_local: this rank's rows of B, shard r = rows
    row_range(Nt_total, G, r) of B ([n, S, H, W] tensors on the compute device).
    features_fn / normalize_fn as in `sharded_features`.  Returns (counts, y, status) of the
    whole pair, identical on every rank."""
    if features_fn is None:
        from . import features as features_fn  # CUDA path
    world, rank = _world(group)
    sizes = [row_range(Nt_total, world, r)[1] - row_range(Nt_total, world, r)[0] for r in range(world)]
    if B_local.shape[0] != sizes[rank]:
        raise ValueError("B_local must be shard row_range(Nt_total, world, rank) of B")
    shape = (max(sizes),) + tuple(B_local.shape[1:])
    cur = torch.zeros(shape, dtype=B_local.dtype, device=B_local.device)
    nxt = torch.zeros_like(cur)
    cur[:sizes[rank]].copy_(B_local)
    counts = None
    status = None
    src = rank                                   # owner of the shard in `cur`
    for step in range(world):
        reqs = []
        if step + 1 < world:                     # start passing this shard on before counting it
            reqs.append(dist.isend(cur, (rank + 1) % world, group=group))
            reqs.append(dist.irecv(nxt, (rank - 1) % world, group=group))
        c, _, st = features_fn(A_local, cur[:sizes[src]], grid, mask, radii, want_y=False, **kw)
        counts = c if counts is None else counts + c
        status = st if status is None else torch.bitwise_or(status, st)
        for r in reqs:
            r.wait()
        cur, nxt = nxt, cur
        src = (src - 1) % world
    if world > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
        status = or_status(status, group=group)
    npairs = float(N_total) * float(Nt_total)
    if normalize_fn is None:
        from . import normalize as normalize_fn
    y = normalize_fn(counts, npairs)
    return counts, y, status
