"""The reference's PCG unit tests (proj/tests/test_pcg.cpp) re-expressed
against the standalone device PCG (`mo_pcg`, pcg.hpp:59-130): the session's
PCG kernels driven by a caller's operator.  The dense operator here is a
torch matmul on the device; the dense oracle of the random-SPD cases is
numpy (the reference uses Eigen's LDLT)."""
import ctypes
import os

import numpy as np
import pytest

from paper_1604_06525_b200 import pcg

pytestmark = pytest.mark.gpu


def _cudart():
    for name in ("libcudart.so", "libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    import torch
    return ctypes.CDLL(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart.so.12"))


def dense_apply(a):
    """y = A x on the device (test_pcg.cpp:16-21)."""
    import torch
    rt = _cudart()
    A = torch.as_tensor(np.asarray(a), device="cuda")
    n = A.shape[0]
    xb = torch.empty(n, dtype=A.dtype, device="cuda")
    nbytes = n * A.element_size()

    def f(x, y, _stream):
        torch.cuda.synchronize()
        assert rt.cudaMemcpy(ctypes.c_void_p(xb.data_ptr()), ctypes.c_void_p(x), ctypes.c_size_t(nbytes), 3) == 0
        yb = A @ xb
        torch.cuda.synchronize()
        assert rt.cudaMemcpy(ctypes.c_void_p(y), ctypes.c_void_p(yb.data_ptr()), ctypes.c_size_t(nbytes), 3) == 0
    return f


def test_two_variable_normal_system():
    """test_pcg.cpp:26-42"""
    a = np.array([[4.0, -2.0], [-2.0, 4.0]])
    d, out = pcg(dense_apply(a), [2.0, 0.0], [4.0, 4.0], max_iters=10, tol_rel=1e-12)
    assert out.iterations <= 2 and not out.indefinite and not out.nonfinite
    assert abs(d[0] - 2.0 / 3.0) <= 1e-14 * 2.0 / 3.0 and abs(d[1] - 1.0 / 3.0) <= 1e-14 / 3.0


def test_identity_converges_in_one_iteration():
    """test_pcg.cpp:44-55"""
    b = np.array([1.0, -2.0, 0.5, 3.0, -0.25])
    d, out = pcg(dense_apply(np.eye(5)), b, np.ones(5), max_iters=10, tol_rel=1e-10)
    assert out.iterations == 1
    np.testing.assert_array_equal(d, b)


def test_random_spd_reaches_dense_solution():
    """test_pcg.cpp:57-86 (numpy dense solve instead of Eigen's LDLT)"""
    rng = np.random.default_rng(555)
    for _ in range(6):
        n = 20
        g = rng.uniform(-1, 1, (n, n))
        a = g.T @ g + 0.5 * np.eye(n)
        b = rng.uniform(-1, 1, n)
        exact = np.linalg.solve(a, b)
        d, out = pcg(dense_apply(a), b, np.diag(a).copy(), max_iters=8 * n, tol_rel=1e-14)
        assert not out.indefinite
        assert np.max(np.abs(d - exact) / np.maximum(1.0, np.abs(exact))) < 1e-8


def test_no_preconditioner_ignores_m():
    """test_pcg.cpp:88-104"""
    a = np.array([[5.0, 1.0, 0.0], [1.0, 4.0, 1.0], [0.0, 1.0, 3.0]])
    d, out = pcg(dense_apply(a), [1.0, 2.0, 3.0], [1e30] * 3, max_iters=3, tol_rel=1e-14, use_preconditioner=False)
    assert not out.nonfinite
    np.testing.assert_allclose(d, np.linalg.solve(a, [1.0, 2.0, 3.0]), rtol=1e-9)


def test_excluded_entries_stay_plus_zero():
    """test_pcg.cpp:106-143: frozen index 2 keeps bitwise +0, the rest solve the submatrix"""
    a = np.array([[6.0, 1.0, 9.0, 0.5], [1.0, 5.0, 9.0, 1.0], [9.0, 9.0, 9.0, 9.0], [0.5, 1.0, 9.0, 4.0]])
    d, out = pcg(dense_apply(a), [1.0, -1.0, 123.0, 2.0], [6.0, 5.0, 1.0, 4.0], max_iters=8, tol_rel=1e-14,
                 excluded=[0, 0, 1, 0])
    assert not out.indefinite
    assert d[2] == 0.0 and not np.signbit(d[2])
    sub = np.array([[6.0, 1.0, 0.5], [1.0, 5.0, 1.0], [0.5, 1.0, 4.0]])
    np.testing.assert_allclose(d[[0, 1, 3]], np.linalg.solve(sub, [1.0, -1.0, 2.0]), rtol=1e-10)


def test_negative_definite_reports_indefinite():
    """test_pcg.cpp:145-155"""
    d, out = pcg(dense_apply(-np.eye(3)), [1.0, 1.0, 1.0], [1.0] * 3)
    assert out.indefinite and out.iterations == 0
    np.testing.assert_array_equal(d, np.zeros(3))


def test_zero_rhs_returns_immediately():
    """test_pcg.cpp:157-165"""
    d, out = pcg(dense_apply(np.eye(3)), [0.0] * 3, [1.0] * 3)
    assert out.iterations == 0
    np.testing.assert_array_equal(d, np.zeros(3))


def test_nonfinite_is_a_flag():
    """test_pcg.cpp:167-174"""
    _, out = pcg(dense_apply(np.eye(2)), [np.nan, 1.0], [1.0, 1.0])
    assert out.nonfinite


def test_iteration_cap_truncates_without_flags():
    """test_pcg.cpp:176-195"""
    rng = np.random.default_rng(99)
    n = 30
    g = rng.uniform(-1, 1, (n, n))
    a = g.T @ g + 0.1 * np.eye(n)
    _, out = pcg(dense_apply(a), np.ones(n), np.diag(a).copy(), max_iters=3, tol_rel=1e-16)
    assert out.iterations == 3 and not out.indefinite and not out.nonfinite


@pytest.mark.parametrize("n", [1, 7, 1000])
def test_float32_and_sizes(n):
    """Real = float (Solver<float>'s PCG) and vector tails of every length mod 4."""
    rng = np.random.default_rng(n)
    g = rng.uniform(-1, 1, (n, n))
    a = (g.T @ g + n * np.eye(n)).astype(np.float32)
    b = rng.uniform(-1, 1, n).astype(np.float32)
    d, out = pcg(dense_apply(a), b, np.diag(a).copy(), max_iters=4 * n + 10, tol_rel=1e-6)
    assert d.dtype == np.float32 and not out.indefinite and not out.nonfinite
    np.testing.assert_allclose(d, np.linalg.solve(a.astype(np.float64), b.astype(np.float64)), rtol=2e-3, atol=2e-4)
