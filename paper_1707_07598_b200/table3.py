"""Materialized basis derivatives of the paper's Table 3 (basis.py:684-800).

``apply_Yk(basis, v, m)`` is d(S(m) v)/dm as an n x N_m CSR and
``apply_Xk(basis, w, m)`` is d(S(m)^T w)/dm as a k x N_m CSR, with the
reference's sparsity patterns (rows, column order, explicit zeros) and values.
Everything is computed on the GPU (msfv_yk_* / msfv_xk_* in include/msfv.h);
``*_dev`` return (indptr, indices, data, shape) as CUDA tensors, the
reference-named functions copy them into scipy.sparse.csr_matrix.
"""

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from .engine import phase, ptr, stream


def _sigma(basis):
    return basis.op.device_state(basis.engine)[2]


def _csr_host(indptr, indices, data, shape):
    """Device CSR -> scipy CSR.  The index and value arrays land in page-locked
    buffers from torch's caching host allocator (reused across calls: the
    copies run at link speed instead of faulting in fresh pageable pages,
    ~2 GB/s); the returned matrix's arrays keep their buffers alive."""
    ip = indptr.cpu().numpy()
    idx_t = np.int32 if (ip[-1] < 2 ** 31 and max(shape) < 2 ** 31) else np.int64
    hi = torch.empty(indices.shape, dtype=indices.dtype, pin_memory=True)
    hd = torch.empty(data.shape, dtype=data.dtype, pin_memory=True)
    hi.copy_(indices, non_blocking=True)
    hd.copy_(data, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return sp.csr_matrix((hd.numpy(), hi.numpy().astype(idx_t, copy=False), ip.astype(idx_t, copy=False)),
                         shape=shape)


def apply_Yk_dev(basis, v, m):
    """Device CSR of d(S v)/dm (basis.py:684-751)."""
    basis.check_model(m)
    eng = basis.engine
    L = eng.L
    b = (basis.partition.b1, basis.partition.b2, basis.partition.b3)
    ncb = b[0] * b[1] * b[2]
    words = (ncb + 31) // 32
    vv = eng.to_device(v).reshape(-1, 1)
    if vv.shape[0] != eng.k:
        raise ValueError(f"coefficient vector length {vv.shape[0]} != number of coarse columns {eng.k}")
    with phase("table3"):
        Sv = eng.prolong(basis.Sint, vv.contiguous())
        rhs = eng.empty(max(eng.nbl * eng.nI * ncb, 1))
        mask = torch.empty(eng.nbl * words, dtype=torch.int32, device=eng.device)
        _lib.check(L.msfv_yk_rhs(eng.plan, ptr(_sigma(basis)), ptr(Sv), ptr(rhs), ptr(mask), stream()), "yk_rhs")
        _lib.check(L.msfv_block_solve_compact(eng.plan, ptr(basis.factor), ptr(rhs), ptr(rhs), ncb, stream()),
                   "block_solve_compact")
        n = eng.Nn - 1
        counts = torch.empty(n, dtype=torch.int64, device=eng.device)
        _lib.check(L.msfv_yk_rowcount(eng.plan, ptr(mask), ptr(counts), stream()), "yk_rowcount")
        indptr = torch.zeros(n + 1, dtype=torch.int64, device=eng.device)
        torch.cumsum(counts, 0, out=indptr[1:])
        nnz = int(indptr[-1].item())
        indices = torch.empty(max(nnz, 1), dtype=torch.int32, device=eng.device)
        data = eng.empty(max(nnz, 1))
        _lib.check(L.msfv_yk_scatter(eng.plan, ptr(mask), ptr(rhs), ptr(indptr), ptr(indices), ptr(data), stream()),
                   "yk_scatter")
    return indptr, indices[:nnz], data[:nnz], (n, eng.Nm)


def apply_Xk_dev(basis, w, m):
    """Device CSR of d(S^T w)/dm (basis.py:754-800)."""
    basis.check_model(m)
    eng = basis.engine
    L = eng.L
    wv = eng.to_device(w).reshape(-1)
    if wv.shape[0] != eng.n:
        raise ValueError(f"field length {wv.shape[0]} != pinned dimension {eng.n}")
    with phase("table3"):
        F = eng.zeros(eng.Nn, 1)
        F[1:, 0] = wv
        z = eng.zeros(eng.Nn, 1)
        eng.interior_solve(basis.factor, F, z)                         # z = interior_solve(w)
        present = torch.empty(eng.nbl, dtype=torch.int32, device=eng.device)
        _lib.check(L.msfv_xk_present(eng.plan, ptr(z), ptr(present), stream()), "xk_present")
        counts = torch.empty(eng.k, dtype=torch.int64, device=eng.device)
        _lib.check(L.msfv_xk_rowcount(eng.plan, ptr(present), ptr(counts), stream()), "xk_rowcount")
        indptr = torch.zeros(eng.k + 1, dtype=torch.int64, device=eng.device)
        torch.cumsum(counts, 0, out=indptr[1:])
        nnz = int(indptr[-1].item())
        indices = torch.empty(max(nnz, 1), dtype=torch.int32, device=eng.device)
        data = eng.empty(max(nnz, 1))
        _lib.check(L.msfv_xk_values(eng.plan, ptr(_sigma(basis)), ptr(basis.Sint), ptr(z), ptr(present), ptr(indptr),
                                    ptr(indices), ptr(data), stream()), "xk_values")
    return indptr, indices[:nnz], data[:nnz], (eng.k, eng.Nm)


def apply_Yk(basis, v, m, workers=1):
    """d(S(m) v)/dm as a scipy CSR, n_pinned x n_cells (basis.py:684-751)."""
    return _csr_host(*apply_Yk_dev(basis, v, m))


def apply_Xk(basis, w, m, workers=1):
    """d(S(m)^T w)/dm as a scipy CSR, k x n_cells (basis.py:754-800)."""
    return _csr_host(*apply_Xk_dev(basis, w, m))
