"""Multi-process paths of the product (paper_2002_05018_b200.parallel).

CPU (gloo, world size 2): reduce_domains_distributed and
recover_primal_distributed run their real sharding and exchanges, with the
per-rank device stages substituted by the oracle (no GPU here); the
assembled K and the recovered field equal the single-process oracle run
bitwise.  GPU (-m gpu): two gloo ranks on cuda:0 run the whole product path
(GPU reduction of each rank's shard, exchange, assembly, block LDL^T replica,
solve, sharded recovery) and match the single-process product run bitwise.
The ranks' kernels never wait on each other (the collectives are gloo on
host tensors)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = ((3, 2, 1), 8, 4, 11)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_reducer(systems, pivot_tol, keep="factor"):
    from oracle import d3m_oracle as O
    out = []
    for s in systems:
        K_D, g_d, fac = O.reduce_domain(s.A, np.concatenate([c.D for c in s.couplings], axis=1), s.f)
        s.factor = fac
        out.append((K_D, g_d))
    return out


def _oracle_fields(systems, lam):
    out = []
    for s in systems:
        rhs = np.array(s.f, dtype=np.complex128)
        for c in s.couplings:
            if c.D.shape[1]:
                rhs = rhs - c.D @ np.asarray(lam[c.interface])
        out.append(s.factor.solve(rhs))
    return out


def _oracle_average(systems, fields, one_d):
    n_glob = 1 + max(int(np.max(s.dof_map)) for s in systems)
    acc = np.zeros(n_glob, dtype=np.complex128)
    cnt = np.zeros(n_glob)
    for s, e in zip(systems, fields):
        acc[s.dof_map] += np.asarray(e).reshape(-1)
        cnt[s.dof_map] += 1.0
    return acc / np.maximum(cnt, 1.0)


def _oracle_pipeline(systems, part, red):
    from oracle import d3m_oracle as O
    sizes = [it.nodes.size for it in part.interfaces]
    blocks, g = O.assemble_reduced(red, [part.incident_interfaces(d) for d in range(part.n_domains)], sizes)
    adj = O.clique_adjacency(len(sizes), blocks.keys())
    plan = O.symbolic_factor(adj, O.reorder(adj, sizes), sizes)
    lam = O.block_solve(O.block_ldlt(blocks, plan), g)
    return blocks, g, lam


def _cpu_worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from paper_2002_05018_b200 import parallel, workloads as wl
    from test_parallel_gloo import _oracle_average, _oracle_fields, _oracle_pipeline, _oracle_reducer
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    systems, part, _ = wl.synthetic_d3m(*CASE)
    red = parallel.reduce_domains_distributed(systems, reducer=_oracle_reducer)
    blocks, g, lam = _oracle_pipeline(systems, part, red)
    sol = parallel.recover_primal_distributed(systems, lam, local_fields=_oracle_fields, average=_oracle_average)
    mine = parallel.shard(len(systems), rank, world)
    owned_factors = [i for i, s in enumerate(systems) if s.factor is not None]
    out_q.put((rank, mine, owned_factors, {k: v.copy() for k, v in blocks.items()}, [x.copy() for x in g], sol))
    dist.barrier()
    dist.destroy_process_group()


def _run(target, world=2):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


def test_shard_round_robin():
    from paper_2002_05018_b200.parallel import shard
    assert shard(7, 0, 3) == [0, 3, 6] and shard(7, 2, 3) == [2, 5]
    assert sorted(sum((shard(10, r, 4) for r in range(4)), [])) == list(range(10))
    with pytest.raises(ValueError):
        shard(3, 2, 2)


def test_distributed_reduce_and_recover_match_single_process():
    from paper_2002_05018_b200 import workloads as wl
    res = _run(_cpu_worker)
    systems, part, _ = wl.synthetic_d3m(*CASE)
    red = _oracle_reducer(systems, 1e-12)
    blocks, g, lam = _oracle_pipeline(systems, part, red)
    sol = _oracle_average(systems, _oracle_fields(systems, lam), True)
    assert sorted(sum((r[1] for r in res), [])) == list(range(len(systems)))
    for rank, mine, owned, b2, g2, sol2 in res:
        assert owned == mine                      # factors stay on the owning rank
        assert set(b2) == set(blocks)
        for k in blocks:
            assert np.array_equal(b2[k], blocks[k])
        for a, b in zip(g2, g):
            assert np.array_equal(a, b)
        assert np.array_equal(sol2, sol)


def _gpu_worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import parallel, workloads as wl
    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    systems, part, _ = wl.synthetic_d3m((3, 3, 2), 14, 6, 5)
    red = parallel.reduce_domains_distributed(systems)
    R = d.assemble_reduced(red, part)
    gr = d.clique_graph(R.K)
    plan = d.symbolic_factor(gr, d.reorder(gr, R.K.sizes), R.K.sizes)
    F = d.block_ldlt(R.K, plan)
    lam = [np.asarray(v) for v in d.block_solve(F, R.g)]
    sol = parallel.recover_primal_distributed(systems, lam)
    out_q.put((rank, np.concatenate(lam), np.asarray(sol)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_distributed_product_path_on_gpu_matches_single_process(cuda):
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    systems, part, _ = wl.synthetic_d3m((3, 3, 2), 14, 6, 5)
    red = d.reduce_domains(systems)
    R = d.assemble_reduced(red, part)
    gr = d.clique_graph(R.K)
    plan = d.symbolic_factor(gr, d.reorder(gr, R.K.sizes), R.K.sizes)
    F = d.block_ldlt(R.K, plan)
    lam = d.block_solve(F, R.g)
    sol = np.asarray(d.recover_primal(systems, lam))
    lam = np.concatenate([np.asarray(v) for v in lam])
    for rank, lam2, sol2 in _run(_gpu_worker):
        assert np.array_equal(lam2, lam), rank
        assert np.array_equal(sol2, sol), rank
