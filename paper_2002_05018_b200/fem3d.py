"""3-D lowest-order Nedelec (Whitney edge element) front end for the FEM
configurations of BASELINE.json (configs 1, 2, 5) -- SURVEY.md 8(f1).

The reference ships only a 2-D scalar P1 analog (mesh.py, subdomain.py:124-163);
this module is its vector counterpart, built so the D3M hot path (reduce ->
assemble -> block LDL^T -> solve -> recover) can run on the paper's 3-D
problems.  It is host-side numpy (mesh generation and assembly are not on the
hot path).

Discretisation (mirrors the reference's scalar structure, time convention of
its `assemble_helmholtz`: A = S - k^2 M - jk B):
  * N^3 hexahedra on a cube of side L, each split into 6 tetrahedra sharing
    the cube's main diagonal (Kuhn split; conforming face diagonals);
  * unknowns: all mesh edges, oriented from lower to higher vertex index;
  * A = (1/mu_r) S - k^2 eps_r M - jk B,   S = curl-curl, M = mass,
    B = int_{outer boundary} (n x W_a).(n x W_b) dS  (first-order ABC);
  * f_a = - int_{outer boundary} W_a . U dS,  U = n x curl E_inc - jk n x (n x E_inc),
    E_inc = p exp(jk d.x), so the incident wave solves the free-space
    problem exactly (a built-in accuracy check);
  * eps_r = eps_sphere for tetrahedra whose centroid lies in the sphere.
Decomposition (mirrors partition_mesh / build_subdomain_systems):
  * domains by cell index, dom = ix + px (iy + py iz);
  * interface (lo, hi) = triangles shared by a tetrahedron of lo and one of
    hi; its dofs are the edges of those triangles (ascending edge id); the
    reference's cross-point drop rule (interface_lambda_nodes) is applied to
    edge ids;
  * A_d = domain part of A + s alpha M_Gamma per incident interface,
    D = s M_Gamma[:, kept], s = +1 on dom_lo, -1 on dom_hi, alpha = jk.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np

TWO_PI = 2.0 * math.pi

_LOCAL_EDGES = np.array([(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)], dtype=np.int64)
# 7-point degree-5 rule on the reference triangle (Dunavant): barycentrics, weights (sum 1)
_A1, _B1 = 0.0597158717, 0.4701420641
_A2, _B2 = 0.7974269853, 0.1012865073
_TRI_Q = np.array([[1 / 3, 1 / 3, 1 / 3], [_A1, _B1, _B1], [_B1, _A1, _B1], [_B1, _B1, _A1],
                   [_A2, _B2, _B2], [_B2, _A2, _B2], [_B2, _B2, _A2]])
_TRI_W = np.array([0.225, 0.1323941527, 0.1323941527, 0.1323941527,
                   0.1259391805, 0.1259391805, 0.1259391805])


@dataclass
class FemProblem:
    """Geometry, material and excitation of one FEM configuration."""
    cells: int                          # N hexahedra per axis
    side: float                         # cube side in wavelengths
    parts: tuple = (1, 1, 1)            # subdomains per axis
    sphere_radius: float = 0.0          # in wavelengths, centred; 0 = free space
    eps_sphere: float = 4.0
    polarisations: tuple = ((1.0, 0.0, 0.0),)
    directions: tuple = ((0.0, 0.0, 1.0),)
    wavelength: float = 1.0
    alpha: complex | None = None

    @property
    def k(self) -> float:
        return TWO_PI / self.wavelength

    def __post_init__(self):
        if self.alpha is None:
            self.alpha = 1j * self.k


def config1() -> FemProblem:
    """BASELINE configs[0]: free-space 0.5 lambda cube, 8^3 x 6 tets, 2x1x1."""
    return FemProblem(8, 0.5, (2, 1, 1))


def config2() -> FemProblem:
    """BASELINE configs[1]: 1 lambda cube, 16^3 x 6 tets, eps_r = 4 sphere of
    radius 0.25 lambda, 2x2x2 subdomains."""
    return FemProblem(16, 1.0, (2, 2, 2), sphere_radius=0.25)


def config5() -> FemProblem:
    """BASELINE configs[4]: 3 lambda cube, 48^3 x 6 tets, sphere 0.75 lambda,
    4x4x4 subdomains, 4 RHS (+-z incidence, x / y polarisation)."""
    return FemProblem(48, 3.0, (4, 4, 4), sphere_radius=0.75,
                      polarisations=((1, 0, 0), (0, 1, 0), (1, 0, 0), (0, 1, 0)),
                      directions=((0, 0, 1), (0, 0, 1), (0, 0, -1), (0, 0, -1)))


@dataclass
class Mesh3D:
    nodes: np.ndarray      # (V, 3)
    tets: np.ndarray       # (T, 4) vertex ids, increasing along the Kuhn path
    cell_of_tet: np.ndarray  # (T, 3) integer cell coordinates
    edges: np.ndarray      # (E, 2) vertex ids, e[0] < e[1]
    tet_edges: np.ndarray  # (T, 6) global edge ids (orientation sign is +1 by construction)
    n: int                 # cells per axis
    h: float

    @property
    def n_edges(self) -> int:
        return int(self.edges.shape[0])


def build_cube_mesh(cells: int, side: float) -> Mesh3D:
    N = cells
    h = side / N
    g = np.arange(N + 1)
    zz, yy, xx = np.meshgrid(g, g, g, indexing="ij")
    nodes = np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1).astype(np.float64) * h

    def vid(x, y, z):
        return x + (N + 1) * (y + (N + 1) * z)

    cz, cy, cx = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    cx, cy, cz = cx.ravel(), cy.ravel(), cz.ravel()
    tets, cells_of = [], []
    unit = np.eye(3, dtype=np.int64)
    for perm in itertools.permutations(range(3)):
        p0 = np.zeros(3, dtype=np.int64)
        p1 = unit[perm[0]]
        p2 = p1 + unit[perm[1]]
        p3 = p2 + unit[perm[2]]
        vs = [vid(cx + p[0], cy + p[1], cz + p[2]) for p in (p0, p1, p2, p3)]
        tets.append(np.stack(vs, axis=1))
        cells_of.append(np.stack([cx, cy, cz], axis=1))
    tets = np.concatenate(tets)
    cell_of = np.concatenate(cells_of)
    pairs = tets[:, _LOCAL_EDGES]                        # (T, 6, 2), increasing vertex ids
    flat = pairs.reshape(-1, 2)
    key = flat[:, 0] * nodes.shape[0] + flat[:, 1]
    uniq, inv = np.unique(key, return_inverse=True)
    edges = np.stack([uniq // nodes.shape[0], uniq % nodes.shape[0]], axis=1)
    return Mesh3D(nodes, tets, cell_of, edges, inv.reshape(-1, 6), N, h)


def _tet_geometry(nodes, tets):
    x = nodes[tets]                                        # (T, 4, 3)
    J = np.stack([x[:, 1] - x[:, 0], x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]], axis=2)  # columns
    det = np.linalg.det(J)
    Jinv = np.linalg.inv(J)                                # rows = grad xi_1..3
    g = np.empty((tets.shape[0], 4, 3))
    g[:, 1:] = Jinv
    g[:, 0] = -Jinv.sum(axis=1)
    return np.abs(det) / 6.0, g


def element_matrices(mesh: Mesh3D, mu_r: float = 1.0):
    """Curl-curl S_e and mass M_e (T, 6, 6) of the Whitney edge functions
    W_ij = l_i grad l_j - l_j grad l_i (curl W_ij = 2 grad l_i x grad l_j)."""
    vol, g = _tet_geometry(mesh.nodes, mesh.tets)
    i, j = _LOCAL_EDGES[:, 0], _LOCAL_EDGES[:, 1]
    curl = 2.0 * np.cross(g[:, i], g[:, j])                # (T, 6, 3)
    S = np.einsum("tad,tbd->tab", curl, curl) * (vol / mu_r)[:, None, None]
    gg = np.einsum("tpd,tqd->tpq", g, g)                   # grad l_p . grad l_q
    L = (np.ones((4, 4)) + np.eye(4)) / 20.0               # int l_p l_q / vol
    M = np.zeros_like(S)
    for a in range(6):
        ia, ja = _LOCAL_EDGES[a]
        for b in range(6):
            kb, lb = _LOCAL_EDGES[b]
            M[:, a, b] = (L[ia, kb] * gg[:, ja, lb] - L[ia, lb] * gg[:, ja, kb]
                          - L[ja, kb] * gg[:, ia, lb] + L[ja, lb] * gg[:, ia, kb])
    M *= vol[:, None, None]
    return S, M


def _faces(mesh: Mesh3D):
    """All tetrahedron faces: (T*4, 3) vertex ids (sorted), owner tet, local
    opposite vertex."""
    opp = np.array([0, 1, 2, 3])
    fl = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]])
    F = np.sort(mesh.tets[:, fl], axis=2).reshape(-1, 3)
    owner = np.repeat(np.arange(mesh.tets.shape[0]), 4)
    return F, owner, np.tile(opp, mesh.tets.shape[0])


def _face_edge_ids(mesh: Mesh3D, tri: np.ndarray) -> np.ndarray:
    V = mesh.nodes.shape[0]
    key = mesh.edges[:, 0] * V + mesh.edges[:, 1]
    pairs = np.stack([tri[:, [0, 0, 1]], tri[:, [1, 2, 2]]], axis=2)     # (F, 3, 2) sorted
    q = pairs[..., 0] * V + pairs[..., 1]
    return np.searchsorted(key, q)


def face_matrices(mesh: Mesh3D, tri: np.ndarray, normal_from: np.ndarray | None = None):
    """Tangential mass int_face W_a^t . W_b^t dS on triangles ``tri`` (F, 3)
    (edges (0,1),(0,2),(1,2) of the sorted triangle) -> (F, 3, 3), plus the
    face areas, unit normals and surface gradients."""
    x = mesh.nodes[tri]
    e1, e2 = x[:, 1] - x[:, 0], x[:, 2] - x[:, 0]
    cr = np.cross(e1, e2)
    area = 0.5 * np.linalg.norm(cr, axis=1)
    n = cr / (2.0 * area)[:, None]                      # right-handed w.r.t. (x0, x1, x2)
    # surface gradients of the 2-D barycentrics: grad l_p = (n x e_opp) / (2 area)
    ge = np.stack([x[:, 2] - x[:, 1], x[:, 0] - x[:, 2], x[:, 1] - x[:, 0]], axis=1)
    g = np.cross(n[:, None, :], ge) / (2.0 * area)[:, None, None]
    if normal_from is not None:                         # outward normal (away from the owner's interior)
        flip = np.einsum("fd,fd->f", n, x[:, 0] - normal_from) < 0
        n = n.copy()
        n[flip] *= -1.0
    E = np.array([(0, 1), (0, 2), (1, 2)])
    gg = np.einsum("fpd,fqd->fpq", g, g)
    L = (np.ones((3, 3)) + np.eye(3)) / 12.0
    M = np.zeros((tri.shape[0], 3, 3))
    for a in range(3):
        ia, ja = E[a]
        for b in range(3):
            kb, lb = E[b]
            M[:, a, b] = (L[ia, kb] * gg[:, ja, lb] - L[ia, lb] * gg[:, ja, kb]
                          - L[ja, kb] * gg[:, ia, lb] + L[ja, lb] * gg[:, ia, kb])
    return M * area[:, None, None], area, n, g


def _einc(prob: FemProblem, pts, p, d):
    ph = np.exp(1j * prob.k * (pts @ np.asarray(d, float)))
    E = np.asarray(p, float)[None, :] * ph[:, None]
    curlE = (1j * prob.k * np.cross(np.asarray(d, float), np.asarray(p, float)))[None, :] * ph[:, None]
    return E, curlE


@dataclass
class FemModel:
    prob: FemProblem
    mesh: Mesh3D
    eps_tet: np.ndarray
    Ae: np.ndarray                 # (T, 6, 6) complex element matrices
    bnd_tri: np.ndarray            # outer boundary triangles (B, 3)
    bnd_owner: np.ndarray          # owning tet
    bnd_edges: np.ndarray          # (B, 3) global edge ids
    bnd_B: np.ndarray              # (B, 3, 3) -jk * tangential mass
    f: np.ndarray                  # (E, nrhs) load
    dom_of_tet: np.ndarray
    n_domains: int
    interfaces: list = field(default_factory=list)
    itf_tri_edges: list = field(default_factory=list)  # per interface (F, 3) edge ids
    itf_M: list = field(default_factory=list)          # per interface (F, 3, 3) tangential mass

    def incident_interfaces(self, d: int) -> list[int]:
        return [i for i, it in enumerate(self.interfaces) if d in (it.dom_lo, it.dom_hi)]


def build_model(prob: FemProblem) -> FemModel:
    from .workloads import Interface
    mesh = build_cube_mesh(prob.cells, prob.side * prob.wavelength)
    S, M = element_matrices(mesh)
    c = mesh.nodes[mesh.tets].mean(axis=1)
    centre = np.full(3, 0.5 * prob.side * prob.wavelength)
    eps = np.where(np.linalg.norm(c - centre, axis=1) < prob.sphere_radius * prob.wavelength,
                   prob.eps_sphere, 1.0)
    k = prob.k
    Ae = S.astype(np.complex128) - (k * k) * eps[:, None, None] * M
    # outer boundary: faces used once
    F, owner, _ = _faces(mesh)
    V = mesh.nodes.shape[0]
    fkey = (F[:, 0] * V + F[:, 1]) * V + F[:, 2]
    uniq, first, counts = np.unique(fkey, return_index=True, return_counts=True)
    bsel = first[counts == 1]
    btri, bown = F[bsel], owner[bsel]
    Mb, area, nrm, gs = face_matrices(mesh, btri, normal_from=c[bown])
    bedges = _face_edge_ids(mesh, btri)
    Bb = (-1j * k) * Mb
    # load: f_a = - int W_a . U dS on every boundary face, 7-point rule
    nrhs = len(prob.polarisations)
    f = np.zeros((mesh.n_edges, nrhs), dtype=np.complex128)
    fface = np.zeros((btri.shape[0], 3, nrhs), dtype=np.complex128)   # per boundary face contributions
    x = mesh.nodes[btri]
    E3 = np.array([(0, 1), (0, 2), (1, 2)])
    for q, w in zip(_TRI_Q, _TRI_W):
        pts = q[0] * x[:, 0] + q[1] * x[:, 1] + q[2] * x[:, 2]
        Wq = np.stack([q[a] * gs[:, b] - q[b] * gs[:, a] for a, b in E3], axis=1)   # (F, 3, 3)
        for r, (p, dvec) in enumerate(zip(prob.polarisations, prob.directions)):
            Ei, cEi = _einc(prob, pts, p, dvec)
            U = np.cross(nrm, cEi) - 1j * k * np.cross(nrm, np.cross(nrm, Ei))
            val = -np.einsum("fad,fd->fa", Wq, U) * (w * area)[:, None]
            fface[:, :, r] += val
    for r in range(nrhs):
        np.add.at(f[:, r], bedges.ravel(), fface[:, :, r].ravel())
    # partition by cell
    px, py, pz = prob.parts
    N = prob.cells
    cc = mesh.cell_of_tet
    ix, iy, iz = cc[:, 0] * px // N, cc[:, 1] * py // N, cc[:, 2] * pz // N
    dom = ix + px * (iy + py * iz)
    # interfaces: interior faces whose two tets lie in different domains
    order = np.argsort(fkey, kind="stable")
    sk = fkey[order]
    pair = np.flatnonzero(sk[1:] == sk[:-1])
    fa, fb = order[pair], order[pair + 1]
    ta, tb = owner[fa], owner[fb]
    da, db = dom[ta], dom[tb]
    cross = da != db
    lo, hi = np.minimum(da, db)[cross], np.maximum(da, db)[cross]
    itri = F[fa[cross]]
    interfaces, itf_edges, itf_M = [], [], []
    for (dl, dh) in sorted(set(zip(lo.tolist(), hi.tolist()))):
        sel = (lo == dl) & (hi == dh)
        tri = itri[sel]
        te = _face_edge_ids(mesh, tri)
        Mi, _, _, _ = face_matrices(mesh, tri)
        interfaces.append(Interface(int(dl), int(dh), np.unique(te).astype(np.int64)))
        itf_edges.append(te)
        itf_M.append(Mi)
    model = FemModel(prob, mesh, eps, Ae, btri, bown, bedges, Bb, f, dom, px * py * pz, interfaces, itf_edges, itf_M)
    model.bnd_f = fface
    return model


def assemble_global(model: FemModel):
    """Monolithic sparse A (CSR) and load f, for verification (driver.run_verify)."""
    import scipy.sparse as sp
    mesh = model.mesh
    te = mesh.tet_edges
    rows = np.repeat(te, 6, axis=1).ravel()
    cols = np.tile(te, (1, 6)).ravel()
    be = model.bnd_edges
    brows = np.repeat(be, 3, axis=1).ravel()
    bcols = np.tile(be, (1, 3)).ravel()
    A = sp.coo_matrix((np.concatenate([model.Ae.ravel(), model.bnd_B.ravel()]),
                       (np.concatenate([rows, brows]), np.concatenate([cols, bcols]))),
                      shape=(mesh.n_edges, mesh.n_edges)).tocsr()
    return A, model.f


def subdomain_systems(model: FemModel, rhs: int | None = 0, sparse: bool = True):
    """Per-domain systems (subdomain.py:124-163 analog) for RHS column
    ``rhs`` (None: all of the problem's RHS columns, f_d of shape n x r);
    returns SubdomainSystem objects of the hot-path API.

    With ``sparse`` (default) A_d and the coupling blocks D are SparseBlock
    objects: the same additions as the dense assembly (np.add.at in element
    order, then the boundary terms, then A[rows, rows] += s*alpha*M_Gamma),
    performed on the compressed entry array, so ``np.asarray(A)`` equals the
    dense assembly bit for bit."""
    from .subdomain import Coupling, SparseBlock, SubdomainSystem, interface_lambda_nodes
    mesh = model.mesh
    kept = interface_lambda_nodes(model)
    systems = []
    for d in range(model.n_domains):
        tsel = np.flatnonzero(model.dom_of_tet == d)
        loc = np.unique(mesh.tet_edges[tsel])
        g2l = np.full(mesh.n_edges, -1, dtype=np.int64)
        g2l[loc] = np.arange(loc.size)
        n = loc.size
        le = g2l[mesh.tet_edges[tsel]]
        k_e = (np.repeat(le, 6, axis=1) * n + np.tile(le, (1, 6))).ravel()
        bsel = np.flatnonzero(model.dom_of_tet[model.bnd_owner] == d)
        k_b = np.zeros(0, np.int64)
        if bsel.size:
            lb = g2l[model.bnd_edges[bsel]]
            k_b = (np.repeat(lb, 3, axis=1) * n + np.tile(lb, (1, 3))).ravel()
        itfs = []
        for i_itf in model.incident_interfaces(d):
            itf = model.interfaces[i_itf]
            s = 1 if itf.dom_lo == d else -1
            nodes = itf.nodes
            pos = np.full(mesh.n_edges, -1, dtype=np.int64)
            pos[nodes] = np.arange(nodes.size)
            li = pos[model.itf_tri_edges[i_itf]]
            Mg = np.zeros((nodes.size, nodes.size))
            np.add.at(Mg, (np.repeat(li, 3, axis=1).ravel(), np.tile(li, (1, 3)).ravel()), model.itf_M[i_itf].ravel())
            itfs.append((i_itf, s, nodes, pos, Mg))
        if sparse:
            k_m = [(g2l[nodes][:, None] * n + g2l[nodes][None, :])[Mg != 0] for _, _, nodes, _, Mg in itfs]
            keys = np.unique(np.concatenate([k_e, k_b] + k_m))
            vals = np.zeros(keys.size, dtype=np.complex128)
            np.add.at(vals, np.searchsorted(keys, k_e), model.Ae[tsel].ravel())
            if bsel.size:
                np.add.at(vals, np.searchsorted(keys, k_b), model.bnd_B[bsel].ravel())
        else:
            A = np.zeros((n, n), dtype=np.complex128)
            np.add.at(A.reshape(-1), k_e, model.Ae[tsel].ravel())
            if bsel.size:
                np.add.at(A.reshape(-1), k_b, model.bnd_B[bsel].ravel())
        couplings = []
        for i_itf, s, nodes, pos, Mg in itfs:
            rows = g2l[nodes]
            blk = (s * model.prob.alpha) * Mg
            if sparse:
                kb = (rows[:, None] * n + rows[None, :]).ravel()
                p = np.minimum(np.searchsorted(keys, kb), keys.size - 1)
                hit = keys[p] == kb
                vals[p[hit]] += blk.ravel()[hit]
            else:
                A[np.ix_(rows, rows)] += blk
            cols = pos[kept[i_itf]]
            Dv = s * Mg[:, cols]
            if sparse:
                kd = (rows[:, None] * cols.size + np.arange(cols.size)[None, :]).ravel()
                o = np.argsort(kd, kind="stable")
                D = SparseBlock((n, cols.size), kd[o], Dv.ravel().astype(np.complex128)[o])
            else:
                D = np.zeros((n, cols.size), dtype=np.complex128)
                if cols.size:
                    D[rows[:, None], np.arange(cols.size)[None, :]] = Dv
            couplings.append(Coupling(i_itf, D, s))
        cols = list(range(model.bnd_f.shape[2])) if rhs is None else [rhs]
        fd = np.zeros((n, len(cols)), dtype=np.complex128)   # load of the domain's own boundary faces
        if bsel.size:
            for q, c in enumerate(cols):
                np.add.at(fd[:, q], g2l[model.bnd_edges[bsel]].ravel(), model.bnd_f[bsel, :, c].ravel())
        if rhs is not None:
            fd = fd[:, 0].copy()
        Ad = SparseBlock((n, n), keys, vals) if sparse else A
        systems.append(SubdomainSystem(d, Ad, fd, loc, couplings))
    return systems


def interpolate_einc(model: FemModel, rhs: int = 0) -> np.ndarray:
    """Edge dofs of the incident field (line integrals along each edge, 2-point
    Gauss): the discrete solution must approach this for free space."""
    mesh = model.mesh
    a, b = mesh.nodes[mesh.edges[:, 0]], mesh.nodes[mesh.edges[:, 1]]
    t = b - a
    out = np.zeros(mesh.n_edges, dtype=np.complex128)
    for s, w in ((0.5 - 0.5 / math.sqrt(3), 0.5), (0.5 + 0.5 / math.sqrt(3), 0.5)):
        E, _ = _einc(model.prob, a + s * t, model.prob.polarisations[rhs], model.prob.directions[rhs])
        out += w * np.einsum("ed,ed->e", E, t)
    return out


def solve_d3m(model: FemModel, rhs: int | None = 0, ordering: str = "builtin", timers: dict | None = None,
              keep: str = "auto", systems: list | None = None, margins: bool = False):
    """Full D3M pipeline of the hot path on the GPU (driver.run_pipeline:103-142
    analog): reduce -> assemble -> ordering / symbolic -> block LDL^T -> block
    solve -> recover, for RHS column ``rhs`` or, with rhs=None, all RHS
    columns at once (one factorisation, n x r solves).  Returns the global
    edge solution (host numpy, n_edges or n_edges x r) and fills ``timers``
    (seconds, wall clock with device synchronisation) when given.  ``keep``
    is passed to reduce_domains; prebuilt ``systems`` skip the front end.
    ``margins`` tracks the pivot-decision margins of every subdomain and
    diagonal-block factorisation (DenseFactor.margin, FactorStats)."""
    import time

    import torch

    from . import blockmat, factor, ordering as ordm, subdomain, symbolic

    def tick():
        torch.cuda.synchronize()
        return time.perf_counter()

    t = {}
    t0 = tick()
    if systems is None:
        systems = subdomain_systems(model, rhs)
    t1 = tick()
    red = subdomain.reduce_domains(systems, keep=keep, margins=margins)
    t2 = tick()
    R = subdomain.assemble_reduced(red, model)
    g = blockmat.clique_graph(R.K)
    order = ordm.reorder(g, R.K.sizes) if ordering == "builtin" else ordm.identity_ordering(R.K.nblocks)
    plan = symbolic.symbolic_factor(g, order, R.K.sizes)
    t3 = tick()
    F = factor.block_ldlt(R.K, plan, margins=margins)
    t4 = tick()
    lam = factor.block_solve(F, R.g)
    t5 = tick()
    sol = np.asarray(subdomain.recover_primal(systems, lam))
    t6 = tick()
    t.update(front_end=t1 - t0, reduce=t2 - t1, assemble_symbolic=t3 - t2, factor=t4 - t3, solve=t5 - t4,
             recover=t6 - t5, d3m_total=t6 - t1)
    if timers is not None:
        timers.update(t)
    return sol, systems, R, plan, F


def global_residual(model: FemModel, sol: np.ndarray, rhs: int | None = 0) -> float:
    """||A x - f||_inf / ||f||_inf of the monolithic system (subdomain.py:240-250);
    the max over columns for rhs=None."""
    A, f = assemble_global(model)
    fr = f if rhs is None else f[:, rhs]
    return float(np.abs(A @ sol - fr).max() / np.abs(fr).max())
