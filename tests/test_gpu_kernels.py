"""GPU parity of the dense primitives: DMMA ZGEMM vs a torch complex128
matmul, and the pivoted batched inverse vs numpy (_linalg.py:19-52)."""

import ctypes

import numpy as np
import pytest
import torch

from paper_2508_19138_b200 import _lib

pytestmark = pytest.mark.gpu

OPS = {0: lambda x: x, 1: lambda x: x.transpose(-1, -2), 2: lambda x: x.conj(),
       3: lambda x: x.conj().transpose(-1, -2)}


def crand(shape, gen, dev):
    return torch.complex(torch.randn(shape, generator=gen, dtype=torch.float64),
                         torch.randn(shape, generator=gen, dtype=torch.float64)).to(dev)


@pytest.mark.parametrize("m,n,k", [(8, 8, 4), (5, 7, 3), (32, 32, 32), (64, 64, 64), (100, 37, 70),
                                   (256, 256, 256), (33, 65, 129), (1, 1, 1)])
@pytest.mark.parametrize("op_a,op_b", [(0, 0), (0, 3), (3, 0), (1, 2), (2, 1), (3, 3)])
@pytest.mark.parametrize("algo", [0, 2, 3])
def test_zgemm_matches_torch(cuda, m, n, k, op_a, op_b, algo):
    g = torch.Generator().manual_seed(m * 1000 + n * 10 + k + op_a * 7 + op_b)
    batch = 3
    a_shape = (batch, m, k) if op_a in (0, 2) else (batch, k, m)
    b_shape = (batch, k, n) if op_b in (0, 2) else (batch, n, k)
    a, b, c = crand(a_shape, g, cuda), crand(b_shape, g, cuda), crand((batch, m, n), g, cuda)
    d = torch.empty((batch, m, n), dtype=torch.complex128, device=cuda)
    alpha, beta = complex(0.7, -0.3), complex(-1.1, 0.4)
    lib = _lib.load()
    assert lib.negf_set_gemm_algo(algo) == 0
    rc = lib.negf_zgemm_batched(m, n, k, batch, alpha.real, alpha.imag,
                                a.data_ptr(), a[0].numel(), a.shape[-1], op_a,
                                b.data_ptr(), b[0].numel(), b.shape[-1], op_b,
                                beta.real, beta.imag, c.data_ptr(), m * n, n,
                                d.data_ptr(), m * n, n, _lib.stream_ptr())
    lib.negf_set_gemm_algo(2)
    assert rc == 0
    ref = alpha * (OPS[op_a](a) @ OPS[op_b](b)) + beta * c
    err = (d - ref).abs().max().item() / max(ref.abs().max().item(), 1e-300)
    assert err < 1e-13


@pytest.mark.parametrize("n", [1, 2, 5, 32, 63, 64, 96, 100, 128, 200, 256, 300, 333, 512])
@pytest.mark.parametrize("algo", [0, 2])
def test_zinv_matches_numpy(cuda, n, algo):
    rng = np.random.default_rng(n)
    batch = 4
    a = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    a[1] += 3 * np.eye(n)
    if n >= 4:  # force pivoting: zero leading element
        a[2, 0, 0] = 0.0
    s = torch.from_numpy(a).to(cuda)
    x = torch.empty_like(s)
    st = torch.zeros(batch, dtype=torch.int32, device=cuda)
    us = torch.zeros(batch, dtype=torch.float64, device=cuda)
    lib = _lib.load()
    nbytes = lib.negf_zinv_workspace_bytes(n, batch)
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=cuda)
    assert lib.negf_set_gemm_algo(algo) == 0
    rc = lib.negf_zinv_batched(n, batch, s.data_ptr(), x.data_ptr(), st.data_ptr(), us.data_ptr(),
                               ws.data_ptr(), nbytes, _lib.stream_ptr())
    lib.negf_set_gemm_algo(2)
    assert rc == 0
    torch.cuda.synchronize()
    assert st.cpu().numpy().tolist() == [0] * batch
    ref = np.linalg.inv(a)
    got = x.cpu().numpy()
    for b in range(batch):
        assert np.linalg.norm(got[b] - ref[b]) / np.linalg.norm(ref[b]) < 1e-11
    # pivot spread matches scipy's LU
    import scipy.linalg as sla
    for b in range(batch):
        lu, _ = sla.lu_factor(a[b])
        d = np.abs(np.diag(lu))
        assert us[b].item() == pytest.approx(d.max() / d.min(), rel=1e-8)


def test_zinv_flags_singular(cuda):
    n, batch = 80, 2
    a = np.random.default_rng(0).standard_normal((batch, n, n)).astype(complex)
    a[1, :, 5] = 0.0  # singular column
    for nn in (16, n):
        s = torch.from_numpy(a[:, :nn, :nn].copy()).to(cuda)
        x = torch.empty_like(s)
        st = torch.zeros(batch, dtype=torch.int32, device=cuda)
        lib = _lib.load()
        nbytes = lib.negf_zinv_workspace_bytes(nn, batch)
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=cuda)
        rc = lib.negf_zinv_batched(nn, batch, s.data_ptr(), x.data_ptr(), st.data_ptr(), None,
                                   ws.data_ptr(), nbytes, _lib.stream_ptr())
        assert rc == 0
        assert st.cpu().numpy().tolist() == [0, 1]


def _inv_check(cuda, a, tol=1e-11):
    batch, n = a.shape[0], a.shape[-1]
    s = torch.from_numpy(a.copy()).to(cuda)
    x = torch.empty_like(s)
    st = torch.zeros(batch, dtype=torch.int32, device=cuda)
    us = torch.zeros(batch, dtype=torch.float64, device=cuda)
    lib = _lib.load()
    nbytes = lib.negf_zinv_workspace_bytes(n, batch)
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=cuda)
    rc = lib.negf_zinv_batched(n, batch, s.data_ptr(), x.data_ptr(), st.data_ptr(), us.data_ptr(), ws.data_ptr(),
                               nbytes, _lib.stream_ptr())
    assert rc == 0
    torch.cuda.synchronize()
    assert st.cpu().numpy().tolist() == [0] * batch
    got = x.cpu().numpy()
    import scipy.linalg as sla
    for b in range(batch):
        lu, piv = sla.lu_factor(a[b])
        ref = sla.lu_solve((lu, piv), np.eye(n))
        assert np.linalg.norm(got[b] - ref) / np.linalg.norm(ref) < tol
        d = np.abs(np.diag(lu))
        # same pivot sequence as LAPACK zgetrf -> same |U_jj| range
        assert us[b].item() == pytest.approx(d.max() / d.min(), rel=1e-8)


@pytest.mark.parametrize("n", [513, 640, 1024, 1100, 2048, 2049, 3000, 4096])
def test_zinv_large_blocks_pivoted(cuda, n):
    """Blocks above the one-CTA register panel (512): cluster panel with the
    pivot search over the whole column (_linalg.py:30-52 semantics). Matrix 0
    is a general random matrix; matrix 1 is W-like and NOT accretive,
    M = I - V P with its leading half-block nearly singular, so the inverse
    needs row interchanges across the halves (the round-1 2x2 recursion
    without cross-half pivoting lost accuracy or failed here)."""
    rng = np.random.default_rng(n)
    batch = 2
    a = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    h = n // 2
    v = rng.standard_normal((n, n))
    v = 0.5 * (v + v.T) / np.sqrt(n)
    p = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    w = np.eye(n) - v @ p
    # leading h x h block of rank 2 (+1e-13 noise): singular without cross-half pivoting
    u1 = rng.standard_normal((h, 2)) + 1j * rng.standard_normal((h, 2))
    w[:h, :h] = u1 @ np.conj(u1.T) * 1e-3 + 1e-13 * rng.standard_normal((h, h))
    a[1] = w
    a[0, 0, 0] = 0.0
    _inv_check(cuda, a, tol=1e-10)


def test_zinv_large_blocks_accretive(cuda):
    """Carrier-like accretive matrix ((E + i eta) I - H) at 1024 orbitals."""
    n, batch = 1024, 3
    rng = np.random.default_rng(5)
    h = (rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))) / np.sqrt(n)
    h = 0.5 * (h + np.conj(np.swapaxes(h, -1, -2)))
    _inv_check(cuda, (0.3 + 0.05j) * np.eye(n) - h)


def test_zinv_large_flags_singular(cuda):
    n, batch = 700, 2
    a = np.random.default_rng(1).standard_normal((batch, n, n)).astype(complex)
    a[1, :, 600] = 0.0  # singular column in a late panel
    s = torch.from_numpy(a).to(cuda)
    x = torch.empty_like(s)
    st = torch.zeros(batch, dtype=torch.int32, device=cuda)
    lib = _lib.load()
    nbytes = lib.negf_zinv_workspace_bytes(n, batch)
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=cuda)
    rc = lib.negf_zinv_batched(n, batch, s.data_ptr(), x.data_ptr(), st.data_ptr(), None, ws.data_ptr(), nbytes,
                               _lib.stream_ptr())
    assert rc == 0
    assert st.cpu().numpy().tolist() == [0, 1]
