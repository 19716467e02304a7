"""CPU: the engine's blocked Householder QR (nb=32, in-panel T) and implicit-Q
application, compiled for the host emulation, against LAPACK via numpy."""

import ctypes

import numpy as np
import pytest

from hostsim import build

P = ctypes.c_void_p


@pytest.fixture(scope="module")
def lib():
    return ctypes.CDLL(build())


@pytest.mark.parametrize("m,n,nc", [(5, 2, 2), (40, 10, 3), (100, 33, 5), (6, 1, 1), (20, 50, 4), (300, 70, 7),
                                    (65, 64, 20), (2100, 40, 3), (3000, 70, 5)])
def test_qr_and_apply(lib, m, n, nc):
    rs = np.random.RandomState(m * 7 + n)
    A0 = rs.randn(m, n)
    k = min(m, n)
    A = np.asfortranarray(A0.copy())
    Q = np.zeros((m, k), order="F")
    ws = np.zeros(64 << 20, np.uint8)
    assert lib.ttgbf_test_qr(A.ctypes.data_as(P), m, n, Q.ctypes.data_as(P), ws.ctypes.data_as(P),
                             ctypes.c_int64(ws.nbytes)) == 0
    R = np.triu(A[:k])
    Qn, Rn = np.linalg.qr(A0)
    assert np.abs(Q @ R - A0).max() <= 1e-13 * np.abs(A0).max() * max(m, n)
    assert np.abs(Q.T @ Q - np.eye(k)).max() <= 1e-13
    assert np.abs(R - Rn).max() <= 1e-12 * np.abs(Rn).max()      # same Householder sign convention
    C = rs.randn(k, nc)
    A = np.asfortranarray(A0.copy())
    X = np.zeros((m, nc), order="F")
    X[:k] = C
    assert lib.ttgbf_test_qr_apply(A.ctypes.data_as(P), m, n, X.ctypes.data_as(P), nc, ws.ctypes.data_as(P),
                                   ctypes.c_int64(ws.nbytes)) == 0
    assert np.abs(X - Qn @ C).max() <= 1e-12 * max(1.0, np.abs(C).max())
