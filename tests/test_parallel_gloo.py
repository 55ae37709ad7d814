"""Multi-process host logic on CPU (gloo, world size 2): subdomain sharding
and the Schur-block exchange reproduce the single-process assembly exactly."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from oracle import d3m_oracle as O
    from paper_2002_05018_b200 import parallel, workloads as wl
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    systems, part, _ = wl.synthetic_d3m((3, 2, 1), 8, 4, 11)
    mine = parallel.shard(len(systems), rank, world)
    local = {}
    for i in mine:
        s = systems[i]
        K_D, g_d, _ = O.reduce_domain(s.A, np.concatenate([c.D for c in s.couplings], axis=1), s.f)
        local[i] = (K_D, g_d)
    full = parallel.exchange_reduced(local, len(systems))
    sizes = [it.nodes.size for it in part.interfaces]
    blocks, g = O.assemble_reduced(full, [part.incident_interfaces(d) for d in range(part.n_domains)], sizes)
    out_q.put((rank, mine, {k: v.copy() for k, v in blocks.items()}, [x.copy() for x in g]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_round_robin():
    from paper_2002_05018_b200.parallel import shard
    assert shard(7, 0, 3) == [0, 3, 6] and shard(7, 2, 3) == [2, 5]
    assert sorted(sum((shard(10, r, 4) for r in range(4)), [])) == list(range(10))
    with pytest.raises(ValueError):
        shard(3, 2, 2)


def test_exchange_matches_single_process():
    import multiprocessing as mp
    from oracle import d3m_oracle as O
    from paper_2002_05018_b200 import workloads as wl
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    systems, part, _ = wl.synthetic_d3m((3, 2, 1), 8, 4, 11)
    red = []
    for s in systems:
        K_D, g_d, _ = O.reduce_domain(s.A, np.concatenate([c.D for c in s.couplings], axis=1), s.f)
        red.append((K_D, g_d))
    sizes = [it.nodes.size for it in part.interfaces]
    blocks, g = O.assemble_reduced(red, [part.incident_interfaces(d) for d in range(part.n_domains)], sizes)
    owned = sorted(sum((r[1] for r in res), []))
    assert owned == list(range(len(systems)))
    for rank, mine, b2, g2 in res:
        assert set(b2) == set(blocks)
        for k in blocks:
            assert np.array_equal(b2[k], blocks[k])
        for a, b in zip(g2, g):
            assert np.array_equal(a, b)
