"""GPU parity: dense Bunch-Kaufman kernel and solves vs the oracle / the
reference goldens.  Pivots AND factor values must be bit-identical."""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from conftest import golden, permuted, rand_complex_symmetric, reconstruct

pytestmark = pytest.mark.gpu


def test_modulus_bit_exact_vs_host(cuda, oracle):
    """Device glibc-hypot and numpy-abs replicas vs host libm / numpy on
    random, wide-exponent and near-threshold pairs."""
    from paper_2002_05018_b200 import _lib
    from paper_2002_05018_b200.device import empty, stream_ptr, to_device
    rng = np.random.default_rng(0)
    N = 1 << 20
    parts = [rng.standard_normal(N) + 1j * rng.standard_normal(N)]
    e = rng.integers(-1070, 1020, N)
    parts.append(np.ldexp(rng.random(N), e) + 1j * np.ldexp(rng.random(N), e - rng.integers(0, 60, N)))
    x = rng.random(N)
    parts.append(x + 1j * x * (1 + (rng.random(N) - 0.5) * 1e-3))
    t = np.ldexp(1.0, -459) * (1 + rng.random(N))
    parts.append(t + 1j * t * rng.random(N))
    z = np.concatenate(parts)
    dz = to_device(z)
    h = cuda.empty(z.size, dtype=cuda.float64, device="cuda")
    a = cuda.empty(z.size, dtype=cuda.float64, device="cuda")
    _lib.call("d3m_modulus_probe", _lib.ptr(dz), _lib.ptr(h), _lib.ptr(a), z.size, stream_ptr())
    hh, ah = h.cpu().numpy(), a.cpu().numpy()
    assert np.array_equal(ah, np.abs(z)), "np.abs replica"
    ref = oracle.hypot_array(z.real, z.imag)       # host glibc libm hypot
    assert np.array_equal(hh, ref), "glibc hypot replica"


def _gpu_factor_matches(M, oracle, pivot_tol=1e-12):
    from paper_2002_05018_b200 import dense_ldlt_bk
    g = dense_ldlt_bk(M, pivot_tol)
    o = oracle.dense_ldlt_bk(M, pivot_tol)
    assert np.array_equal(g.perm, o.perm)
    assert np.array_equal(g.tags, o.tags)
    assert g.n_2x2 == o.n_2x2 and g.growth == o.growth
    packed = g.packed.cpu().numpy()
    assert np.array_equal(np.tril(packed).view(np.int64), np.tril(o.packed).view(np.int64))
    return g


def test_bk_bit_exact_vs_reference_goldens(cuda):
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from gen_golden_inputs import dense_suite
    from paper_2002_05018_b200 import dense_ldlt_bk
    g = golden("dense_bk.npz")
    offs = np.concatenate([[0], np.cumsum(g["sizes"])])
    for k, (name, M) in enumerate(dense_suite()):
        f = dense_ldlt_bk(M)
        assert np.array_equal(f.perm, g["perm"][offs[k]:offs[k + 1]]), name
        assert np.array_equal(f.tags, g["tags"][offs[k]:offs[k + 1]]), name
        assert f.n_2x2 == g["n2x2"][k] and f.growth == g["growth"][k], name
        W = np.tril(f.packed.cpu().numpy())
        assert hashlib.sha256(W.tobytes()).hexdigest() == g["digest"][k], name


@pytest.mark.parametrize("n", [1, 2, 3, 17, 64, 200, 256, 384, 513])
def test_bk_bit_exact_vs_oracle_sizes(cuda, oracle, n):
    M = rand_complex_symmetric(n, 1000 + n)
    M[np.diag_indices(n)] *= 0.05            # force 2x2 pivots and swaps
    _gpu_factor_matches(M, oracle)


def test_kats(cuda):
    from paper_2002_05018_b200 import dense_ldlt_bk
    f = dense_ldlt_bk(np.eye(4, dtype=complex))           # test_dense_factor.py:16-21
    assert np.array_equal(f.L, np.eye(4)) and np.array_equal(f.d, np.ones(4))
    assert np.array_equal(f.perm, np.arange(4)) and f.n_2x2 == 0
    M = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=complex)  # :24-31
    f = dense_ldlt_bk(M)
    assert f.n_2x2 == 1 and list(f.tags) == [2, 0]
    assert np.array_equal(f.L, np.eye(2)) and np.array_equal(f.dense_d(), M)


def test_reconstruction_and_growth(cuda):
    from paper_2002_05018_b200 import dense_ldlt_bk
    for seed in range(10):                                    # :34-50
        M = rand_complex_symmetric(12, seed)
        if seed % 2:
            M[0, 0] = M[3, 3] = 0
        f = dense_ldlt_bk(M)
        err = np.linalg.norm(permuted(M, f.perm) - reconstruct(f), "fro")
        assert err <= 1e-13 * np.linalg.norm(M, "fro")
        assert 1.0 <= f.growth <= 2.57


def test_errors(cuda):
    from paper_2002_05018_b200 import SingularBlockError, dense_ldlt_bk
    with pytest.raises(SingularBlockError, match="elimination step 0"):
        dense_ldlt_bk(np.zeros((3, 3), dtype=complex))
    M = rand_complex_symmetric(6, 5)
    M[:, 2] = 0
    M[2, :] = 0
    with pytest.raises(SingularBlockError):
        dense_ldlt_bk(M)
    D = np.diag([1.0, 1e-20]).astype(complex)               # :85-90
    with pytest.raises(SingularBlockError, match=r"threshold 1\.000e-12"):
        dense_ldlt_bk(D, pivot_tol=1e-12)
    assert dense_ldlt_bk(D, pivot_tol=1e-30).d[1] == 1e-20
    with pytest.raises(ValueError, match="not symmetric"):
        dense_ldlt_bk(np.array([[1.0, 2.0], [0.0, 1.0]], dtype=complex))
    with pytest.raises(ValueError):
        dense_ldlt_bk(np.ones((2, 3), dtype=complex))
    f = dense_ldlt_bk(np.zeros((0, 0), dtype=complex))
    assert f.n == 0 and f.solve(np.zeros((0, 2), dtype=complex)).shape == (0, 2)


def test_error_message_matches_oracle(cuda, oracle):
    from paper_2002_05018_b200 import SingularBlockError, dense_ldlt_bk
    M = rand_complex_symmetric(7, 3)
    M[:, 4] = 0
    M[4, :] = 0
    with pytest.raises(SingularBlockError) as eg:
        dense_ldlt_bk(M)
    with pytest.raises(oracle.OracleSingular) as eo:
        oracle.dense_ldlt_bk(M)
    assert str(eg.value) == str(eo.value)


def test_solve_vs_oracle(cuda, oracle):
    from paper_2002_05018_b200 import dense_ldlt_bk
    rng = np.random.default_rng(11)
    for n, m in [(24, 1), (18, 4), (100, 7), (256, 16), (300, 33)]:
        M = rand_complex_symmetric(n, n + m)
        M[np.diag_indices(n)] *= 0.1
        B = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))
        X = dense_ldlt_bk(M).solve(B)
        Xo = oracle.dense_ldlt_bk(M).solve(B)
        assert np.linalg.norm(X - Xo) <= 1e-11 * np.linalg.norm(Xo)
        assert np.linalg.norm(M @ X - B) <= 1e-9 * np.linalg.norm(B) * max(1.0, np.linalg.cond(M) * 1e-4)
    b = rng.standard_normal(24) + 1j * rng.standard_normal(24)
    M = rand_complex_symmetric(24, 11) + 24 * np.eye(24)
    x = dense_ldlt_bk(M).solve(b)
    assert x.shape == (24,)
    assert np.linalg.norm(M @ x - b) <= 1e-12 * np.linalg.norm(b)
    with pytest.raises(ValueError):
        dense_ldlt_bk(np.eye(3, dtype=complex)).solve(np.ones(4, dtype=complex))


def test_deterministic(cuda):
    from paper_2002_05018_b200 import dense_ldlt_bk
    M = rand_complex_symmetric(150, 9)
    a, b = dense_ldlt_bk(M), dense_ldlt_bk(M)
    assert np.array_equal(a.packed.cpu().numpy(), b.packed.cpu().numpy())
    B = np.ones((150, 3), dtype=complex)
    assert np.array_equal(a.solve(B), b.solve(B))


def test_bk_factor_binding_with_absolute_threshold(cuda, oracle):
    """The kernels.bk_factor(W, tol_abs) binding of INTEGRATION.md: check_sym
    bit 2 makes pivot_tol the absolute threshold, so a threshold placed
    exactly at a column maximum (where tol_abs / scale * scale could move by
    an ulp) decides like the reference: info and pivots equal the oracle's."""
    import torch
    from paper_2002_05018_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(77)
    n = 40
    G = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    M = (G + G.T) / 2
    M[20:, 20:] *= 1e-9                               # a numerically small trailing block
    W0 = np.ascontiguousarray(M)
    Wo = W0.copy()
    ref = oracle.bk_factor(Wo, 0.0)
    for tol_abs in (0.0, 1e-12, np.abs(Wo[25:, 25]).max(), 1e-7, 10.0):
        Wo = W0.copy()
        want = oracle.bk_factor(Wo, float(tol_abs))
        d = torch.from_numpy(W0.copy()).cuda()
        perm = torch.empty(n, dtype=torch.int64, device="cuda")
        tags = torch.empty(n, dtype=torch.int8, device="cuda")
        i32 = lambda: torch.empty(1, dtype=torch.int32, device="cuda")
        f64 = lambda: torch.empty(1, dtype=torch.float64, device="cuda")
        n2, info, gr, sc, asy = i32(), i32(), f64(), f64(), f64()
        P = _lib.ctypes.c_void_p
        rc = lib.d3m_bk_factor_batched(1, n, P(d.data_ptr()), n * n, n, float(tol_abs), 4, P(perm.data_ptr()),
                                       P(tags.data_ptr()), P(n2.data_ptr()), P(gr.data_ptr()), P(info.data_ptr()),
                                       P(sc.data_ptr()), P(asy.data_ptr()), None, None,
                                       P(torch.cuda.current_stream().cuda_stream))
        assert rc == 0
        assert int(info.item()) == want[4], tol_abs
        if want[4] < 0:
            assert np.array_equal(perm.cpu().numpy(), want[0]) and np.array_equal(tags.cpu().numpy(), want[1])
            assert np.array_equal(np.tril(d.cpu().numpy()), np.tril(Wo))
    assert ref[4] == -1
