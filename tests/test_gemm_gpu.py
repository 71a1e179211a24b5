"""The train step's dense-layer GEMMs (gemm_x3.cu: TMA-fed 3xTF32 tcgen05
kernels) against fp64 numpy on the feature-major layout: forward with fused
bias + relu, input gradient with the fused relu' mask, weight gradient with
the bias column. Gate: fp32-level relative error (3xTF32), including ragged
hit counts (tails of the 32-hit boxes and 256-hit tiles) and the head shapes
(2 and 3 outputs)."""
import ctypes as C

import numpy as np
import pytest

import paper_2205_07058_b200 as P

pytestmark = pytest.mark.gpu


def _lib():
    L = P.load_library()
    f = L.svlf_debug_gemm_x3
    f.argtypes = [C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int]
    f.restype = C.c_int
    return f


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _ld(n):
    if n == 154469:  # the C3 step's active hits in matrices of its real row stride
        return 262144
    return (n + 31) // 32 * 32 + 64


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("K", [134, 38, 128])
@pytest.mark.parametrize("n", [1, 1000, 77777, 154469])
def test_forward(K, n):
    import torch

    f = _lib()
    rng = np.random.default_rng(K + n)
    ld = _ld(n)
    W = rng.standard_normal((128, K)).astype(np.float32) / np.sqrt(K)
    b = rng.standard_normal(128).astype(np.float32) * 0.1
    X = rng.standard_normal((K, ld)).astype(np.float32)
    X[:, n:] = np.nan  # stale columns past n must not leak
    out = torch.full((128, ld), -7.0, device="cuda")
    dW_, db_, dX_ = _dev(W), _dev(b), _dev(X)  # keep the device copies alive across the call
    assert f(0, _p(dW_), 128, K, 0, _p(db_), _p(dX_), None, None, _p(out), None, n, ld, 3) == 0
    got = out.cpu().numpy()
    want = np.maximum(W.astype(np.float64) @ np.nan_to_num(X[:, :n].astype(np.float64)) + b[:, None], 0)
    assert _rel(got[:, :n], want) <= 2e-6
    tail = got[:, ((n + 31) // 32) * 32:]
    assert np.all(tail == -7.0)  # nothing written past the last 32-hit box (the box's tail is scratch)


@pytest.mark.parametrize("O,K,k0", [(128, 134, 6), (128, 38, 6), (128, 128, 0)])
@pytest.mark.parametrize("n", [5, 4097, 77777, 154469])
def test_input_gradient(O, K, k0, n):
    import torch

    f = _lib()
    rng = np.random.default_rng(O + K + n)
    ld = _ld(n)
    W = rng.standard_normal((O, K)).astype(np.float32) / np.sqrt(K)
    D = rng.standard_normal((O, ld)).astype(np.float32)
    D[:, n:] = np.nan
    mask = rng.standard_normal((K - k0, ld)).astype(np.float32)
    out = torch.full((K - k0, ld), -7.0, device="cuda")
    dW_, dD_, dm_ = _dev(W), _dev(D), _dev(mask)
    assert f(1, _p(dW_), O, K, k0, None, _p(dD_), None, _p(dm_), _p(out), None, n, ld, 3) == 0
    got = out.cpu().numpy()
    want = W[:, k0:].astype(np.float64).T @ D[:, :n].astype(np.float64)
    want[mask[:, :n] <= 0] = 0
    assert _rel(got[:, :n], want) <= 2e-6
    assert np.all(got[:, ((n + 31) // 32) * 32:] == -7.0)


@pytest.mark.parametrize("O,K", [(128, 134), (2, 128), (128, 38), (3, 128)])
@pytest.mark.parametrize("n", [1, 3000, 154469])
@pytest.mark.parametrize("products", [3, 1])
def test_weight_gradient(O, K, n, products):
    import torch

    f = _lib()
    rng = np.random.default_rng(O * K + n)
    ld = _ld(n)
    D = rng.standard_normal((O, ld)).astype(np.float32)
    X = rng.standard_normal((K, ld)).astype(np.float32)
    D[:, n:] = 1e30  # stale columns past n must be ignored
    X[:, n:] = 1e30
    dW = torch.zeros((O, K), device="cuda")
    db = torch.zeros(O, device="cuda")
    dD, dX = _dev(D), _dev(X)
    assert f(2, None, O, K, 0, None, _p(dD), _p(dX), None, _p(dW), _p(db), n, ld, products) == 0
    want = D[:, :n].astype(np.float64) @ X[:, :n].astype(np.float64).T
    wb = D[:, :n].astype(np.float64).sum(axis=1)
    # fp32 accumulation over n zero-mean products: the relative error grows like sqrt(n)
    tol = (2e-6 * max(1.0, np.sqrt(n / 1000))) if products == 3 else 2e-3
    assert _rel(dW.cpu().numpy(), want) <= tol
    assert _rel(db.cpu().numpy(), wb) <= tol
    # deterministic: a second run gives the same bits
    dW2 = torch.zeros_like(dW)
    db2 = torch.zeros_like(db)
    assert f(2, None, O, K, 0, None, _p(dD), _p(dX), None, _p(dW2), _p(db2), n, ld, products) == 0
    assert torch.equal(dW, dW2) and torch.equal(db, db2)
