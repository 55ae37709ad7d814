"""Split upload of dense host subdomain matrices (subdomain._reduce_chunk):
the panel BK starts on the lower row blocks while the upper remainder, D and
F are still in flight, and the symmetry check / full scale run on an intact
device copy.  The results must be bitwise those of the one-pass path on
device-resident inputs, and the reference's errors (factor.py:94-103,
subdomain.py:174-175) must be raised unchanged."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _systems(B, n, m, seed, host="numpy"):
    import torch
    import paper_2002_05018_b200 as d
    rng = np.random.default_rng(seed)
    out = []
    for b in range(B):
        G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2 * n)
        A = (G + G.T) / 2
        A[np.diag_indices(n)] += rng.uniform(-1, 1, n) + 0.1j * rng.uniform(-1, 1, n)
        D = np.zeros((n, m), dtype=complex)
        D[rng.choice(n, m, replace=False), np.arange(m)] = rng.choice([-1.0, 1.0], m)
        f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        if host == "pinned":
            A = torch.from_numpy(A).pin_memory()
        out.append(d.SubdomainSystem(b, A, f, np.arange(n), [d.Coupling(0, D, 1)]))
    return out


def _device_copy(systems):
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200.device import DeviceArray, to_device
    return [d.SubdomainSystem(s.domain, DeviceArray(to_device(np.asarray(s.A))), s.f, s.dof_map,
                              [d.Coupling(c.interface, c.D, c.sign) for c in s.couplings]) for s in systems]


def _run(systems, keep):
    import paper_2002_05018_b200 as d
    red = d.reduce_domains(systems, keep=keep)
    return [(np.asarray(K), np.asarray(g), s.factor.perm, s.factor.tags) for (K, g), s in zip(red, systems)]


def test_split_upload_packed_factor_keeps_the_input_upper_triangle(cuda):
    """`packed` is the one-pass path's bit for bit: the factor below the
    diagonal and, above it, the input's entries (kernels.py:18, "only the
    lower triangle is read or written")."""
    import paper_2002_05018_b200 as d
    systems = _systems(3, 640, 40, 15)
    dev = _device_copy(systems)
    d.reduce_domains(systems, keep="factor")
    d.reduce_domains(dev, keep="factor")
    for s, s0 in zip(systems, dev):
        P, P0 = s.factor.packed.cpu().numpy(), s0.factor.packed.cpu().numpy()
        assert np.array_equal(P, P0)
        assert np.array_equal(np.triu(P, 1), np.triu(np.asarray(s.A), 1))


@pytest.mark.parametrize("host,keep", [("numpy", "factor"), ("pinned", "schur"), ("numpy", "solution")])
def test_split_upload_bitwise_equals_device_inputs(cuda, host, keep):
    systems = _systems(3, 640, 40, 11, host)
    got = _run(systems, keep)
    ref = _run(_device_copy(systems), keep)
    for (K, g, p, t), (K0, g0, p0, t0) in zip(got, ref):
        assert np.array_equal(p, p0) and np.array_equal(t, t0)
        assert np.array_equal(K, K0) and np.array_equal(g, g0)


def test_split_upload_inexact_symmetry_refactors_with_full_scale(cuda):
    """The largest entry sits in the upper triangle (asymmetry within the
    1e-12 tolerance): the lower-triangle scale differs from np.abs(A).max(),
    so the chunk is reduced again from the intact copy with the full scale."""
    systems = _systems(2, 600, 24, 12)
    A = systems[1].A
    A[3, 500] = 4.0 + 0.0j
    A[500, 3] = 4.0 * (1.0 - 2e-16)
    got = _run(systems, "factor")
    ref = _run(_device_copy(systems), "factor")
    for (K, g, p, t), (K0, g0, p0, t0) in zip(got, ref):
        assert np.array_equal(p, p0) and np.array_equal(t, t0)
        assert np.array_equal(K, K0) and np.array_equal(g, g0)


def test_split_upload_asymmetric_raises(cuda):
    systems = _systems(2, 600, 24, 13)
    systems[1].A[10, 400] += 1e-3
    with pytest.raises(ValueError, match="not symmetric"):
        _run(systems, "factor")


def test_split_upload_singular_names_domain(cuda):
    import paper_2002_05018_b200 as d
    systems = _systems(3, 576, 16, 14)
    systems[2] = d.SubdomainSystem(7, np.zeros((576, 576), dtype=complex), systems[2].f, systems[2].dof_map,
                                   systems[2].couplings)
    with pytest.raises(d.SingularDomainError, match="domain 7"):
        _run(systems, "factor")
