"""Multi-GPU plumbing of the hot path (one process per GPU, torch.distributed).

Subdomains are independent, so the Schur reduction and the
primal recovery shard across ranks with no collective inside them; the D3M
path has two exchanges:

* after the reduction, the per-domain Schur blocks (K_D, g_d) are gathered so
  every rank can assemble K (assemble_reduced, ascending domain order);
* after the recovery, the per-domain fields E_d are gathered so the duplicated
  interface dofs are averaged in the reference's order (subdomain.py:229-237).

Both exchanges move each domain's arrays once, and the ordered host/device
reductions afterwards are the single-process ones, so every rank's result is
bitwise equal to a single-process run.  block_ldlt itself is an
elimination-tree chain under natural order and runs as replicas in this tier
(DESIGN.md section 8).
"""

from __future__ import annotations

import numpy as np


def shard(n_items: int, rank: int, world: int) -> list[int]:
    """Round-robin ownership of subdomains: item i belongs to rank i % world."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    return list(range(rank, n_items, world))


def exchange_arrays(local: dict, n_items: int, group=None) -> list:
    """All-gather per-item tuples of complex128 arrays.

    ``local`` maps item index -> tuple of arrays (numpy, DeviceArray or torch)
    for the items this rank owns.  Returns the tuples of all items in item
    order on every rank: device tensors (DeviceArray) over NCCL, numpy arrays
    over gloo.  Shapes travel first (one object collective), then one padded
    flat payload per rank (all_gather needs equal sizes)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    device = "cuda" if backend == "nccl" else "cpu"
    meta = {d: tuple(tuple(np.shape(a)) for a in arrs) for d, arrs in local.items()}
    metas = [None] * world
    dist.all_gather_object(metas, meta, group=group)

    def flat(x):
        if hasattr(x, "tensor"):
            x = x.tensor
        if isinstance(x, torch.Tensor):
            return x.reshape(-1).to(device=device, dtype=torch.complex128)
        return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.complex128)).reshape(-1)).to(device)

    mine = [flat(a) for d in sorted(local) for a in local[d]]
    payload = torch.cat(mine) if mine else torch.zeros(0, dtype=torch.complex128, device=device)
    sizes = [sum(int(np.prod(s)) for d in m for s in m[d]) for m in metas]
    mx = max(max(sizes), 1)
    padded = torch.zeros(mx, dtype=torch.complex128, device=device)
    padded[:payload.numel()] = payload
    gathered = [torch.empty(mx, dtype=torch.complex128, device=device) for _ in range(world)]
    dist.all_gather(gathered, padded, group=group)
    out = [None] * n_items
    for r, m in enumerate(metas):
        o = 0
        for d in sorted(m):
            arrs = []
            for shp in m[d]:
                k = int(np.prod(shp))
                arrs.append(gathered[r][o:o + k].reshape(shp))
                o += k
            out[d] = tuple(arrs)
    if device == "cuda":
        from .device import DeviceArray
        return [tuple(DeviceArray(a.contiguous()) for a in t) for t in out]
    return [tuple(a.numpy() for a in t) for t in out]


def exchange_reduced(local: dict, n_domains: int, group=None) -> list:
    """All-gather the (K_D, g_d) pairs each rank computed for its shard;
    returns the full list in domain order on every rank."""
    return [tuple(t) for t in exchange_arrays(local, n_domains, group)]


def reduce_domains_distributed(systems, pivot_tol: float = 1e-12, group=None, keep: str = "factor",
                               reducer=None) -> list:
    """Each rank reduces its shard of ``systems`` (subdomain.reduce_domains on
    its GPU; ``reducer`` substitutes another function of the same signature,
    e.g. in host-only tests), then the Schur blocks are exchanged.  Every rank
    returns the full reduced list; the factors stay cached on the owning
    rank's systems for recover_primal_distributed."""
    import torch.distributed as dist

    if reducer is None:
        from .subdomain import reduce_domains as reducer
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = shard(len(systems), rank, world)
    red = reducer([systems[i] for i in mine], pivot_tol, keep=keep) if mine else []
    return exchange_reduced(dict(zip(mine, red)), len(systems), group)


def recover_primal_distributed(systems, lam, group=None, local_fields=None, average=None):
    """recover_primal (subdomain.py:217-237) with the domains sharded like
    reduce_domains_distributed: each rank forms E_d for the domains it
    reduced (their factors / X are cached there), the fields are gathered,
    and every rank averages them over the duplicated dofs in ascending domain
    order -- the single-process result, bitwise.  ``local_fields(systems,
    lam) -> [E_d]`` and ``average(systems, fields, one_d) -> E`` substitute
    the device stages (host-only tests)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = shard(len(systems), rank, world)
    if local_fields is None:
        local_fields = _device_fields
    if average is None:
        average = _device_average
    fields = local_fields([systems[i] for i in mine], lam) if mine else []
    allf = exchange_arrays({d: (e,) for d, e in zip(mine, fields)}, len(systems), group)
    one_d = all(np.ndim(v) == 1 for v in lam)
    return average(systems, [t[0] for t in allf], one_d)


def _device_fields(systems, lam):
    """E_d (n_d x r) of each of ``systems`` on this rank's GPU."""
    from .subdomain import _local_E
    ET, e_off, r, _ = _local_E(systems, lam)
    return [ET[:, o:o + s.n_dofs].t().contiguous() for s, o in zip(systems, e_off)]


def _device_average(systems, fields, one_d):
    """Ordered average of all domains' fields on this rank's GPU -> numpy
    (n_glob, or n_glob x r for multi-column loads)."""
    import torch

    from .device import to_device
    from .subdomain import _ordered_average
    dev = [to_device(e).reshape(s.n_dofs, -1) for s, e in zip(systems, fields)]
    r = int(dev[0].shape[1]) if dev else 1
    e_off = list(np.concatenate([[0], np.cumsum([s.n_dofs for s in systems])[:-1]]).astype(np.int64))
    ET = torch.cat([e.t() for e in dev], dim=1).contiguous()
    outT = _ordered_average(systems, ET, e_off, r)
    return (outT[0] if one_d else outT.t().contiguous()).cpu().numpy()
