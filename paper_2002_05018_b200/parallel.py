"""Multi-GPU plumbing of the hot path (one process per GPU, torch.distributed).

Subdomains are independent, so the Schur reduction shards across
ranks with no collective; the single exchange of the D3M path is gathering the
per-domain Schur blocks (K_D, g_d) so K can be assembled.
block_ldlt itself is an elimination-tree chain under natural order and runs
as replicas in this tier.
"""

from __future__ import annotations

import numpy as np


def shard(n_items: int, rank: int, world: int) -> list[int]:
    """Round-robin ownership of subdomains: item i belongs to rank i % world."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    return list(range(rank, n_items, world))


def exchange_reduced(local: dict, n_domains: int, group=None) -> list:
    """All-gather the (K_D, g_d) pairs each rank computed for its shard.

    ``local`` maps domain index -> (K_D, g_d) (numpy or DeviceArray).  Returns
    the full list in domain order on every rank.  Device blocks travel as
    flattened complex128 tensors (NCCL over NVLink on a GPU node, gloo on a
    CPU test host); the assembly order afterwards is the reference's
    (ascending domain), so the assembled K is identical on every rank and to
    a single-process run.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    device = "cuda" if backend == "nccl" else "cpu"
    # shapes first (small, object collective), then one flat payload per rank
    meta = {d: (tuple(np.shape(K)), tuple(np.shape(g))) for d, (K, g) in local.items()}
    metas = [None] * world
    dist.all_gather_object(metas, meta, group=group)
    def flat(x):
        if hasattr(x, "tensor"):
            return x.tensor.reshape(-1).to(device)
        return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.complex128)).reshape(-1)).to(device)
    mine = [flat(v) for d in sorted(local) for v in local[d]]
    payload = torch.cat(mine) if mine else torch.zeros(0, dtype=torch.complex128, device=device)
    sizes = [sum(int(np.prod(s)) for d in sorted(m) for s in m[d]) for m in metas]
    bufs = [torch.empty(max(sz, 1), dtype=torch.complex128, device=device) for sz in sizes]
    # gloo/nccl all_gather needs equal sizes: pad to the max
    mx = max(max(sizes), 1)
    padded = torch.zeros(mx, dtype=torch.complex128, device=device)
    padded[:payload.numel()] = payload
    gathered = [torch.empty(mx, dtype=torch.complex128, device=device) for _ in range(world)]
    dist.all_gather(gathered, padded, group=group)
    out = [None] * n_domains
    for r, m in enumerate(metas):
        o = 0
        for d in sorted(m):
            ks, gs = m[d]
            nk, ng = int(np.prod(ks)), int(np.prod(gs))
            K = gathered[r][o:o + nk].reshape(ks)
            g = gathered[r][o + nk:o + nk + ng].reshape(gs)
            o += nk + ng
            out[d] = (K, g) if device == "cuda" else (K.numpy(), g.numpy())
    del bufs
    if device == "cuda":
        from .device import DeviceArray
        out = [(DeviceArray(K.contiguous()), DeviceArray(g.contiguous())) for K, g in out]
    return out


def reduce_domains_distributed(systems, pivot_tol: float = 1e-12, group=None) -> list:
    """Each rank reduces its shard of ``systems`` on its GPU, then the Schur
    blocks are exchanged; every rank returns the full reduced list (factors
    stay cached on the owning rank's systems for recover_primal)."""
    import torch.distributed as dist

    from .subdomain import reduce_domains
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = shard(len(systems), rank, world)
    red = reduce_domains([systems[i] for i in mine], pivot_tol) if mine else []
    return exchange_reduced(dict(zip(mine, red)), len(systems), group)
