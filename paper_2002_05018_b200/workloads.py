"""Seeded synthetic workloads of BASELINE.json (no datasets are involved).

* config 3 -- batched Schur complement: 64 subdomains, A_i = (M + M^T)/2 with
  M ~ CN(0, 1/n), diagonal offset U[-1,1] + jU[-0.1,0.1]; D_i n x m with one
  +-1 per column in a random distinct row (BASELINE.json configs[2]).
* config 4 -- blocked LDL^T of K alone: 4x4x4 subdomain grid, 144 interior
  faces of 256 unknowns in natural (ascending (dom_lo, dom_hi)) face order;
  block (f, g) stored iff the faces bound a common subdomain; entries
  CN(0, 1/256); diagonal blocks tril(G) + tril(G, -1)^T plus a real shift
  U[-2, 2] per diagonal entry (the pinned reading of "indefinite shift");
  16 RHS ~ CN(0, 1/256) (BASELINE.json configs[3]).
* a small synthetic D3M problem (random subdomain matrices coupled through
  face multipliers) for end-to-end pipeline tests.

CN(0, s2) means re, im ~ N(0, s2 / 2).  Draw order is part of the contract:
tests/golden fixtures generated from these functions pin it.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .blockmat import BlockSparseSym, from_blocks


def _cn(rng, shape, var):
    s = np.sqrt(var / 2.0)
    return rng.standard_normal(shape) * s + 1j * (rng.standard_normal(shape) * s)


# --------------------------------------------------------------------------
# domain grids and their faces
# --------------------------------------------------------------------------

def grid_faces(gx: int, gy: int, gz: int) -> list[tuple[int, int]]:
    """Interior faces (dom_lo, dom_hi), dom = ix + gx*(iy + gy*iz), sorted."""
    faces = []
    for iz in range(gz):
        for iy in range(gy):
            for ix in range(gx):
                d = ix + gx * (iy + gy * iz)
                if ix + 1 < gx:
                    faces.append((d, d + 1))
                if iy + 1 < gy:
                    faces.append((d, d + gx))
                if iz + 1 < gz:
                    faces.append((d, d + gx * gy))
    return sorted(faces)


@dataclass
class Interface:
    dom_lo: int
    dom_hi: int
    nodes: np.ndarray

    @property
    def n_nodes(self) -> int:
        return int(self.nodes.size)


@dataclass
class GridPartition:
    """Partition shim (mesh.py:Partition interface used by the hot path):
    ``interfaces[k].{dom_lo, dom_hi, nodes}`` and ``incident_interfaces(d)``."""
    n_domains: int
    interfaces: list = field(default_factory=list)

    def incident_interfaces(self, d: int) -> list[int]:
        return [k for k, it in enumerate(self.interfaces) if d in (it.dom_lo, it.dom_hi)]


def grid_partition(gx, gy, gz, face_dofs) -> GridPartition:
    faces = grid_faces(gx, gy, gz)
    itfs = [Interface(lo, hi, np.arange(k * face_dofs, (k + 1) * face_dofs, dtype=np.int64))
            for k, (lo, hi) in enumerate(faces)]
    return GridPartition(gx * gy * gz, itfs)


# --------------------------------------------------------------------------
# config 4
# --------------------------------------------------------------------------

def config4_matrix(seed: int = 4, grid=(4, 4, 4), n: int = 256) -> BlockSparseSym:
    faces = grid_faces(*grid)
    nf = len(faces)
    rng = np.random.default_rng(seed)
    var = 1.0 / n
    triples = []
    for f in range(nf):
        for g in range(f + 1):
            if f == g:
                G = _cn(rng, (n, n), var)
                Dg = np.tril(G) + np.tril(G, -1).T
                Dg[np.diag_indices(n)] += rng.uniform(-2.0, 2.0, n)
                triples.append((f, f, Dg))
            elif set(faces[f]) & set(faces[g]):
                triples.append((f, g, _cn(rng, (n, n), var)))
    return from_blocks(np.full(nf, n, dtype=np.int64), triples)


def config4_rhs(K: BlockSparseSym, nrhs: int = 16, seed: int = 44) -> list[np.ndarray]:
    rng = np.random.default_rng(seed)
    return [_cn(rng, (int(s), nrhs), 1.0 / 256.0) for s in K.sizes]


# --------------------------------------------------------------------------
# config 3
# --------------------------------------------------------------------------

def config3_domain(i: int, n: int = 2048, m: int = 384, seed: int = 3):
    """(A_i, D_i, f_i) of subdomain i, from its own seeded stream."""
    rng = np.random.default_rng([seed, i])
    M = _cn(rng, (n, n), 1.0 / n)
    A = (M + M.T) / 2.0
    A[np.diag_indices(n)] += rng.uniform(-1.0, 1.0, n) + 1j * rng.uniform(-0.1, 0.1, n)
    rows = rng.choice(n, m, replace=False)
    D = np.zeros((n, m), dtype=np.complex128)
    D[rows, np.arange(m)] = rng.choice(np.array([-1.0, 1.0]), m)
    f = np.zeros(n, dtype=np.complex128)
    return A, D, f


def config3_systems(count: int = 64, n: int = 2048, m: int = 384, seed: int = 3):
    from .subdomain import Coupling, SubdomainSystem
    out = []
    for i in range(count):
        A, D, f = config3_domain(i, n, m, seed)
        out.append(SubdomainSystem(i, A, f, np.arange(n, dtype=np.int64), [Coupling(0, D, 1)]))
    return out


# --------------------------------------------------------------------------
# small end-to-end D3M problem
# --------------------------------------------------------------------------

def synthetic_d3m(grid=(2, 2, 1), interior: int = 12, face_dofs: int = 5, seed: int = 0, shift: float = 4.0):
    """Subdomains with `interior` private dofs plus the dofs of their faces.
    A_d = random complex symmetric + shift*I (+ s*alpha on face dofs),
    coupling D = s * I on the face dofs (s = +1 on dom_lo, -1 on dom_hi).
    Returns (systems, partition, global A, global f) where the global
    monolithic system is the sum of the A_d restricted to shared dofs."""
    from .subdomain import Coupling, SubdomainSystem
    rng = np.random.default_rng(seed)
    part = grid_partition(*grid, face_dofs)
    nd = part.n_domains
    nf = len(part.interfaces)
    n_face_total = nf * face_dofs
    systems = []
    n_glob = n_face_total + nd * interior
    for d in range(nd):
        inc = part.incident_interfaces(d)
        gl = [np.arange(n_face_total + d * interior, n_face_total + (d + 1) * interior)]
        gl += [part.interfaces[k].nodes for k in inc]
        dof_map = np.concatenate(gl).astype(np.int64)
        n = dof_map.size
        G = _cn(rng, (n, n), 1.0)
        A = (G + G.T) / 2.0 + shift * np.eye(n)
        f = _cn(rng, (n,), 1.0)
        couplings = []
        o = interior
        for k in inc:
            s = 1 if part.interfaces[k].dom_lo == d else -1
            D = np.zeros((n, face_dofs), dtype=np.complex128)
            D[o:o + face_dofs, :] = s * np.eye(face_dofs)
            couplings.append(Coupling(k, D, s))
            o += face_dofs
        systems.append(SubdomainSystem(d, A, f, dof_map, couplings))
    return systems, part, n_glob


def rand_block_system(seed, max_blocks=8, max_size=8, density=0.4, shift=None):
    """Random well-conditioned block-sparse symmetric system with its dense
    scatter (the reference test generator's contract, conftest.py:26-60)."""
    rng = np.random.default_rng(seed)
    nb = int(rng.integers(1, max_blocks + 1))
    sizes = rng.integers(1, max_size + 1, size=nb)
    n = int(sizes.sum())
    G = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    S = (G + G.T) / 2.0
    S = S + (2.0 * n if shift is None else shift) * np.eye(n)
    off = np.concatenate([[0], np.cumsum(sizes)])
    keep = np.eye(nb, dtype=bool)
    for i in range(nb):
        for j in range(i):
            if rng.random() < density:
                keep[i, j] = keep[j, i] = True
    Sref = np.zeros_like(S)
    triples = []
    for i in range(nb):
        for j in range(nb):
            if keep[i, j]:
                blk = S[off[i]:off[i + 1], off[j]:off[j + 1]]
                Sref[off[i]:off[i + 1], off[j]:off[j + 1]] = blk
                if i >= j:
                    triples.append((i, j, blk))
    return from_blocks(sizes, triples), Sref
