"""Geometry-bound device engine: one msfv_plan per (mesh, partition) and thin
typed wrappers around every C-ABI entry point.

PyTorch provides device memory (caching allocator) and the stream; every
call enqueues on ``torch.cuda.current_stream()``.  No CPU fallback exists.
"""

import ctypes
import weakref

import numpy as np
import torch

from . import _lib

F64 = torch.float64


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


# torch.cuda.current_stream() walks several Python layers (device index, lazy
# init, availability checks: ~5 us); every kernel launch asks for the stream,
# so the raw getters are used when this torch build has them.
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_raw_device = getattr(torch._C, "_cuda_getDevice", None)


def stream():
    if _raw_stream is not None and _raw_device is not None:
        return ctypes.c_void_p(_raw_stream(_raw_device()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class PhaseTimer:
    """Optional CUDA-event bracketing of named phases on the current stream
    (used by bench.py for the per-kernel-class breakdown; off by default)."""

    enabled = False
    events = []

    @classmethod
    def start(cls):
        cls.enabled = True
        cls.events = []

    @classmethod
    def stop(cls):
        """Synchronize and return {phase: total ms}."""
        cls.enabled = False
        torch.cuda.synchronize()
        out = {}
        for name, a, b in cls.events:
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        cls.events = []
        return out


class phase:
    def __init__(self, name):
        self.name = name

    def __enter__(self):
        if PhaseTimer.enabled:
            self.a = torch.cuda.Event(enable_timing=True)
            self.a.record()

    def __exit__(self, *exc):
        if PhaseTimer.enabled:
            b = torch.cuda.Event(enable_timing=True)
            b.record()
            PhaseTimer.events.append((self.name, self.a, b))


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("the MSFV B200 path needs a CUDA device; there is no CPU fallback")


class Points:
    """A survey matrix (P or Q) uploaded for one engine (msfv_points)."""

    def __init__(self, engine, M):
        import scipy.sparse as sp
        M = sp.csc_matrix(M)
        M.sort_indices()
        self.ncol = M.shape[1]
        self.nnz = M.nnz
        h = ctypes.c_void_p()
        colptr = np.ascontiguousarray(M.indptr, dtype=np.int64)
        rows = np.ascontiguousarray(M.indices, dtype=np.int64)
        vals = np.ascontiguousarray(M.data, dtype=np.float64)
        L = _lib.load()
        _lib.check(L.msfv_points_create(engine.plan, self.nnz, self.ncol,
                                        colptr.ctypes.data_as(ctypes.c_void_p),
                                        rows.ctypes.data_as(ctypes.c_void_p),
                                        vals.ctypes.data_as(ctypes.c_void_p),
                                        ctypes.byref(h)), "points_create")
        self.handle = h
        self._fin = weakref.finalize(self, L.msfv_points_destroy, h)
        nib = ctypes.c_int64()
        _lib.check(L.msfv_points_interior_blocks(h, ctypes.byref(nib)), "points_interior_blocks")
        self.interior_blocks = int(nib.value)     # blocks with survey nodes in their interior


class Engine:
    def __init__(self, cells, h, blocks, reduced=False):
        """blocks=None: geometry-only plan (fine-mesh entry points only);
        reduced: reduced-dimension boundary conditions for the basis."""
        require_cuda()
        L = _lib.load()
        self.L = L
        plan = ctypes.c_void_p()
        if blocks is None:
            _lib.check(L.msfv_plan_create_mesh((ctypes.c_int32 * 3)(*cells), (ctypes.c_double * 3)(*h),
                                               ctypes.byref(plan)), "plan_create_mesh")
        else:
            _lib.check(L.msfv_plan_create((ctypes.c_int32 * 3)(*cells), (ctypes.c_double * 3)(*h),
                                          (ctypes.c_int32 * 3)(*blocks), ctypes.byref(plan)), "plan_create")
        self.plan = plan
        self._fin = weakref.finalize(self, L.msfv_plan_destroy, plan)
        self.reduced = bool(reduced)
        if reduced:
            _lib.check(L.msfv_plan_set_reduced(plan, 1), "plan_set_reduced")
        self._bound = None
        info = (ctypes.c_int64 * _lib.INFO_COUNT)()
        _lib.check(L.msfv_plan_info(plan, info, _lib.INFO_COUNT))
        self.info = list(info)
        self.cells, self.h = tuple(cells), tuple(h)
        self.blocks = None if blocks is None else tuple(blocks)
        self.Nn = info[_lib.INFO_NN]
        self.n = info[_lib.INFO_N]
        self.Nm = info[_lib.INFO_NCELLS]
        self.E = info[_lib.INFO_NEDGES]
        self.nbl = info[_lib.INFO_NBLOCKS]
        self.nI = info[_lib.INFO_NI]
        self.P1s = info[_lib.INFO_P1S]
        self.k = info[_lib.INFO_K]
        self.ak_doubles = info[_lib.INFO_AK_DOUBLES]
        self.NT, self.PT, self.TB = info[_lib.INFO_NT], info[_lib.INFO_PT], info[_lib.INFO_TB]
        self.factor_doubles = info[_lib.INFO_FACTOR_DOUBLES]
        self.scratch_doubles = info[_lib.INFO_SCRATCH_DOUBLES]
        # 1: register-window DMMA band (split build); 2: L2-resident DMMA band (larger blocks)
        self.local_solver = int(info[_lib.INFO_TC])
        self.tensor_core = self.local_solver == 1
        self.coarse_multifrontal = info[_lib.INFO_COARSE] == 2
        self.device = torch.device("cuda", torch.cuda.current_device())
        self._csc = None

    # ------------------------------------------------------------- buffers
    def zeros(self, *shape):
        return torch.zeros(shape, dtype=F64, device=self.device)

    def empty(self, *shape):
        return torch.empty(shape, dtype=F64, device=self.device)

    def flags(self):
        return torch.zeros(1, dtype=torch.int32, device=self.device)

    def to_device(self, a, n=None):
        """numpy / torch (host or device) -> contiguous float64 device tensor."""
        if isinstance(a, torch.Tensor):
            t = a
            if t.dtype != F64:
                t = t.to(F64)
            t = t.to(self.device, non_blocking=True)
        else:
            h = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            # a page-locked source (e.g. misfit_ssd's residual) copies asynchronously
            t = h.to(self.device, non_blocking=True)
        return t.contiguous()

    # ------------------------------------------------------------- kernels
    def operator(self, m):
        with phase("operator"):
            return self._operator(m)

    def _operator(self, m):
        sigma = self.empty(self.Nm)
        w = self.empty(self.E)
        fl = self.flags()
        _lib.check(self.L.msfv_operator(self.plan, ptr(m), ptr(sigma), ptr(w), ptr(fl), stream()), "operator")
        return sigma, w, fl

    def edge_average(self, sigma, dm):
        tmp = self.empty(self.Nm)
        c = self.empty(self.E)
        with phase("edge_average"):
            _lib.check(self.L.msfv_edge_average(self.plan, ptr(sigma), ptr(dm), ptr(tmp), ptr(c), stream()),
                       "edge_average")
        return c

    def basis(self, w, fl=None):
        with phase("basis"):
            return self._basis(w, fl)

    def _basis(self, w, fl=None):
        factor = self.empty(max(self.factor_doubles, 1))
        Sint = self.empty(max(self.nbl * 8 * self.nI, 1))
        Kloc = self.empty(self.nbl * 64)
        scratch = self.empty(max(self.scratch_doubles, 1))
        fl = fl if fl is not None else self.flags()
        _lib.check(self.L.msfv_basis_build(self.plan, ptr(w), ptr(factor), ptr(Sint), ptr(Kloc), ptr(scratch),
                                           ptr(fl), stream()), "basis_build")
        return factor, Sint, Kloc, fl

    def basis_forward(self, w, fl=None):
        """Split build, part 1: factors, Galerkin blocks, y = L^-1 R parked in Sint."""
        with phase("basis"):
            factor = self.empty(max(self.factor_doubles, 1))
            Sint = self.empty(max(self.nbl * 8 * self.nI, 1))
            Kloc = self.empty(self.nbl * 64)
            fl = fl if fl is not None else self.flags()
            _lib.check(self.L.msfv_basis_forward(self.plan, ptr(w), ptr(factor), ptr(Sint), ptr(Kloc), ptr(fl),
                                                 stream()), "basis_forward")
        return factor, Sint, Kloc, fl

    def build_pipelined(self, m_host, chunks=4):
        """Model upload in z-slabs on the copy stream with the operator and the
        forward basis build of each slab queued behind its copy (the upload
        of slab i + 1 overlaps the build of slab i).  Returns
        (m_dev, sigma, w, flags, factor, Sint, Kloc)."""
        n1, n2, n3 = self.cells
        b3 = self.blocks[2]
        nb3 = n3 // b3
        plane = n1 * n2
        # the copies go out first: everything else below is host work that
        # overlaps them
        m_dev = self.empty(self.Nm)
        cur, cp = torch.cuda.current_stream(), self.copy_stream
        chunks = max(1, min(chunks, nb3))
        bounds = [round(i * nb3 / chunks) for i in range(chunks + 1)]
        ready = torch.cuda.Event()
        ready.record(cur)                       # m_dev allocated on the current stream
        cp.wait_event(ready)
        evs = []
        with torch.cuda.stream(cp):
            for c in range(chunks):
                k0, kc1 = bounds[c] * b3, min(bounds[c + 1] * b3 + 1, n3)
                m_dev[k0 * plane:kc1 * plane].copy_(m_host[k0 * plane:kc1 * plane], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cp)
                evs.append(ev)
        m_dev.record_stream(cp)
        sigma, w, fl = self.empty(self.Nm), self.empty(self.E), self.flags()
        factor = self.empty(max(self.factor_doubles, 1))
        Sint = self.empty(max(self.nbl * 8 * self.nI, 1))
        Kloc = self.empty(self.nbl * 64)
        with phase("operator+basis (pipelined)"):
            for c in range(chunks):
                bk0, bk1 = bounds[c], bounds[c + 1]
                cur.wait_event(evs[c])
                _lib.check(self.L.msfv_operator_slab(self.plan, ptr(m_dev), ptr(sigma), ptr(w), ptr(fl), bk0 * b3,
                                                     bk1 * b3, stream()), "operator_slab")
                _lib.check(self.L.msfv_basis_forward_slab(self.plan, ptr(w), ptr(factor), ptr(Sint), ptr(Kloc),
                                                          ptr(fl), bk0, bk1, stream()), "basis_forward_slab")
        return m_dev, sigma, w, fl, factor, Sint, Kloc

    def basis_backward(self, factor, Sint):
        """Split build, part 2 (on the current stream): Sint = S_I."""
        _lib.check(self.L.msfv_basis_backward(self.plan, ptr(factor), ptr(Sint), stream()), "basis_backward")

    @property
    def side_stream(self):
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.device)
        return self._side

    def galerkin(self, Kloc, shift=0.0, out=None):
        Ak = out if out is not None else self.empty(self.ak_doubles)
        with phase("galerkin"):
            _lib.check(self.L.msfv_galerkin(self.plan, ptr(Kloc), float(shift), ptr(Ak), stream()), "galerkin")
        return Ak

    def coarse_dense(self, Kloc, shift=0.0):
        """Dense natural-order A_k (+ shift I) for the host-side A_k attribute."""
        out = self.empty(self.k, self.k)
        _lib.check(self.L.msfv_coarse_dense(self.plan, ptr(Kloc), float(shift), ptr(out), stream()), "coarse_dense")
        return out

    def coarse_trace(self, Ak):
        d = self.empty(self.k)
        _lib.check(self.L.msfv_coarse_diag(self.plan, ptr(Ak), ptr(d), stream()), "coarse_diag")
        return d

    def coarse_factor(self, Ak, fl):
        with phase("coarse_factor"):
            _lib.check(self.L.msfv_coarse_factor(self.plan, ptr(Ak), ptr(fl), stream()), "coarse_factor")

    def coarse_solve(self, Lk, X):
        """In place: X (k, nrhs) contiguous device tensor."""
        assert X.is_contiguous() and X.shape[0] == self.k
        with phase("coarse_solve"):
            scratch = self.empty(max(self.NT * self.TB * X.shape[1], 1))
            _lib.check(self.L.msfv_coarse_solve(self.plan, ptr(Lk), ptr(X), ptr(scratch), X.shape[1], stream()),
                       "coarse_solve")
        return X

    def receive(self, pts, Sint, Y=None, Xfield=None, nrhs=None):
        nrhs = nrhs if nrhs is not None else (Y.shape[1] if Y is not None else Xfield.shape[1])
        out = self.empty(pts.ncol, nrhs)
        with phase("survey_receive"):
            _lib.check(self.L.msfv_survey_receive(self.plan, pts.handle, ptr(Sint), ptr(Y), ptr(Xfield), nrhs,
                                                  ptr(out), stream()), "survey_receive")
        return out

    def restrict_points(self, pts, Sint, Z=None, nrhs=None):
        nrhs = nrhs if nrhs is not None else (Z.shape[1] if Z is not None else pts.ncol)
        out = self.empty(self.k, nrhs)
        with phase("survey_restrict"):
            _lib.check(self.L.msfv_survey_restrict(self.plan, pts.handle, ptr(Sint), ptr(Z), nrhs, ptr(out),
                                                   stream()), "survey_restrict")
        return out

    def scatter_points(self, pts, Z=None, nrhs=None, field=None):
        nrhs = nrhs if nrhs is not None else (Z.shape[1] if Z is not None else pts.ncol)
        f = field if field is not None else self.zeros(self.Nn, nrhs)
        with phase("survey_scatter"):
            _lib.check(self.L.msfv_survey_scatter(self.plan, pts.handle, ptr(Z), nrhs, ptr(f), stream()),
                       "survey_scatter")
        return f

    def prolong(self, Sint, Y):
        nrhs = Y.shape[1]
        out = self.empty(self.Nn, nrhs)
        with phase("prolong"):
            _lib.check(self.L.msfv_prolong(self.plan, ptr(Sint), ptr(Y), nrhs, ptr(out), stream()), "prolong")
        return out

    def residual(self, src, alpha, wt, X, beta, nrhs, out=None):
        o = out if out is not None else self.zeros(self.Nn, nrhs)
        with phase("residual"):
            _lib.check(self.L.msfv_residual(self.plan, ptr(src), float(alpha), ptr(wt), ptr(X), float(beta), nrhs,
                                            ptr(o), stream()), "residual")
        return o

    def interior_solve(self, factor, rhs, out=None):
        nrhs = rhs.shape[1]
        o = out if out is not None else rhs
        with phase("interior_solve"):
            _lib.check(self.L.msfv_interior_solve(self.plan, ptr(factor), ptr(rhs), ptr(o), nrhs, stream()),
                       "interior_solve")
        return o

    def restrict_op(self, Sint, w1, X1, w2, X2, nrhs, scale=1.0):
        part = self.empty(self.nbl * 8 * nrhs)
        out = self.empty(self.k, nrhs)
        with phase("restrict_op"):
            _lib.check(self.L.msfv_restrict_op(self.plan, ptr(Sint), ptr(w1), ptr(X1), ptr(w2), ptr(X2), nrhs,
                                               float(scale), ptr(part), ptr(out), stream()), "restrict_op")
        return out

    def cell_gradient(self, sigma, U, Z, Y, R):
        nrhs = U.shape[1]
        g = self.empty(self.Nm)
        xi = self.empty(self.E)
        with phase("cell_gradient"):
            _lib.check(self.L.msfv_cell_gradient(self.plan, ptr(sigma), ptr(U), ptr(Z), ptr(Y), ptr(R), nrhs,
                                                 ptr(xi), ptr(g), stream()), "cell_gradient")
        return g

    def interior_fields(self, pts, factor, Z=None, nrhs=None):
        """Compact blockdiag(A_II^-1) (M Z)_I on the point set's interior blocks
        (None when it has none)."""
        nrhs = nrhs if nrhs is not None else (Z.shape[1] if Z is not None else pts.ncol)
        if pts.interior_blocks == 0:
            return None
        rc = self.empty(pts.interior_blocks * self.nI * max(nrhs, 1))
        with phase("interior_solve"):
            _lib.check(self.L.msfv_points_interior_scatter(self.plan, pts.handle, ptr(Z), nrhs, ptr(rc), stream()),
                       "points_interior_scatter")
            _lib.check(self.L.msfv_points_interior_solve(self.plan, pts.handle, ptr(factor), ptr(rc), ptr(rc), nrhs,
                                                         stream()), "points_interior_solve")
        return rc

    def block_gradient(self, sigma, Sint, T, y, pz=None, Zc=None, pr=None, Rc=None):
        """Fused per-block rapply gradient; raises NotImplementedError when the
        block closure does not fit in shared memory."""
        nrhs = T.shape[1]
        g = self.empty(self.Nm)
        with phase("block_gradient"):
            _lib.check(self.L.msfv_block_gradient(self.plan, ptr(sigma), ptr(Sint), ptr(T), ptr(y), nrhs,
                                                  None if pz is None else pz.handle, ptr(Zc),
                                                  None if pr is None else pr.handle, ptr(Rc), ptr(g), stream()),
                       "block_gradient")
        return g

    def block_gradient_to_host(self, sigma, Sint, T, y, pz=None, Zc=None, pr=None, Rc=None, chunks=4):
        """block_gradient with the result copied to a page-locked host array
        slab by slab: the copy of slab i runs on a side stream while slab
        i + 1 is computed.  Returns the numpy view of the host buffer."""
        nrhs = T.shape[1]
        g = self.empty(self.Nm)
        host = torch.empty(self.Nm, dtype=F64, pin_memory=True)
        nb3 = self.cells[2] // self.blocks[2]
        cur = torch.cuda.current_stream()
        cp = self.copy_stream
        bounds = [round(i * nb3 / chunks) for i in range(chunks + 1)]
        per_slab = self.Nm // nb3
        with phase("block_gradient"):
            for c in range(chunks):
                b0, b1 = bounds[c], bounds[c + 1]
                if b1 <= b0:
                    continue
                _lib.check(self.L.msfv_block_gradient_slab(
                    self.plan, ptr(sigma), ptr(Sint), ptr(T), ptr(y), nrhs, None if pz is None else pz.handle,
                    ptr(Zc), None if pr is None else pr.handle, ptr(Rc), b0, b1, ptr(g), stream()),
                    "block_gradient_slab")
                ev = torch.cuda.Event()
                ev.record(cur)
                cp.wait_event(ev)
                with torch.cuda.stream(cp):
                    host[b0 * per_slab:b1 * per_slab].copy_(g[b0 * per_slab:b1 * per_slab], non_blocking=True)
        g.record_stream(cp)
        cp.synchronize()
        return host.numpy()

    @property
    def copy_stream(self):
        if getattr(self, "_copy", None) is None:
            self._copy = torch.cuda.Stream(device=self.device)
        return self._copy

    def jv_coarse_rhs(self, Sint, c, T, pr=None, Rc=None):
        """-EP^T((G U + G R) o c) on the coarse nodes (k x nrhs); raises
        NotImplementedError when the block closure does not fit in shared memory."""
        nrhs = T.shape[1]
        part = self.empty(self.nbl * 8 * max(nrhs, 1))
        out = self.empty(self.k, nrhs)
        with phase("jv_rhs"):
            _lib.check(self.L.msfv_jv_coarse_rhs(self.plan, ptr(Sint), ptr(c), ptr(T), nrhs,
                                                 None if pr is None else pr.handle, ptr(Rc), ptr(part), ptr(out),
                                                 stream()), "jv_coarse_rhs")
        return out

    # ------------------------------------------------ reduced boundary values
    def boundary_reduced(self, w, fl):
        """Skeleton values of the reduced boundary problems (box table)."""
        faces = self.empty(max(self.info[_lib.INFO_RED_FACE], 1))
        bx = self.empty(max(self.info[_lib.INFO_RED_BOX], 1))
        with phase("boundary_reduced"):
            _lib.check(self.L.msfv_boundary_reduced(self.plan, ptr(w), ptr(faces), ptr(bx), ptr(fl), stream()),
                       "boundary_reduced")
        return bx

    def bind_boundary(self, bx):
        """Bind the box table the following launches read (reduced plans)."""
        if self._bound is not bx:
            _lib.check(self.L.msfv_plan_bind_boundary(self.plan, ptr(bx)), "plan_bind_boundary")
            self._bound = bx

    # ------------------------------------------------------------ fine mesh
    def fine_apply(self, w, X, out=None):
        """A(w) X over all pinned nodes; X, out full node fields (Nn, nrhs)."""
        o = out if out is not None else self.empty(*X.shape)
        with phase("fine_apply"):
            _lib.check(self.L.msfv_fine_apply(self.plan, ptr(w), ptr(X), X.shape[1], ptr(o), stream()), "fine_apply")
        return o

    def full_gradient(self, sigma, U, V):
        """-sigma C^T sum_s (G U_s)(G V_s) (FullSensitivity.rapply)."""
        g = self.empty(self.Nm)
        xi = self.empty(self.E)
        with phase("full_gradient"):
            _lib.check(self.L.msfv_full_gradient(self.plan, ptr(sigma), ptr(U), ptr(V), U.shape[1], ptr(xi), ptr(g),
                                                 stream()), "full_gradient")
        return g

    # ------------------------------------------------- edge space (enriched)
    def edge_grad(self, X):
        """G_p X: (E, ncol) edge fields of the node fields X (Nn, ncol)."""
        X = X.contiguous()
        o = self.empty(self.E, X.shape[1])
        _lib.check(self.L.msfv_edge_grad(self.plan, ptr(X), X.shape[1], ptr(o), stream()), "edge_grad")
        return o

    def edge_div(self, F):
        """G_p^T F: node fields (Nn, ncol) of the edge fields F (E, ncol)."""
        F = F.contiguous()
        o = self.empty(self.Nn, F.shape[1])
        _lib.check(self.L.msfv_edge_div(self.plan, ptr(F), F.shape[1], ptr(o), stream()), "edge_div")
        return o

    def cell_gather(self, sigma, xi):
        """-sigma o (C^T xi) for one edge vector xi (E,)."""
        g = self.empty(self.Nm)
        _lib.check(self.L.msfv_cell_gather(self.plan, ptr(sigma), ptr(xi.contiguous()), ptr(g), stream()),
                   "cell_gather")
        return g

    def reg_apply(self, alpha, v, out=None):
        o = out if out is not None else self.empty(self.Nm)
        _lib.check(self.L.msfv_reg_apply(self.plan, float(alpha), ptr(v), ptr(o), stream()), "reg_apply")
        return o

    def reg_faces(self, d):
        o = self.empty(self.Nm)
        _lib.check(self.L.msfv_reg_faces(self.plan, ptr(d), ptr(o), stream()), "reg_faces")
        return o

    def basis_csc_box(self, Sint, src, bsrc, bx):
        vals = self.empty(src.numel())
        _lib.check(self.L.msfv_basis_csc_box(src.numel(), ptr(Sint), ptr(src), ptr(bsrc), ptr(bx), ptr(vals),
                                             stream()), "basis_csc_box")
        return vals

    def basis_csc(self, Sint, src, hatv):
        vals = self.empty(src.numel())
        _lib.check(self.L.msfv_basis_csc(src.numel(), ptr(Sint), ptr(src), ptr(hatv), ptr(vals), stream()),
                   "basis_csc")
        return vals


_ENGINES = {}


def engine_for_mesh(mesh):
    """Geometry-only engine of a mesh (fine-mesh entry points)."""
    key = ((mesh.n1, mesh.n2, mesh.n3), (float(mesh.h1), float(mesh.h2), float(mesh.h3)), None,
           torch.cuda.current_device() if torch.cuda.is_available() else -1)
    eng = _ENGINES.get(key)
    if eng is None:
        eng = Engine(*key[:3])
        _ENGINES[key] = eng
    return eng


def engine_for(partition, reduced=False):
    """The engine (plan) of a partition; ``reduced``: a separate plan whose
    basis uses the reduced-dimension boundary conditions (msfv_reduced.cu)."""
    m = partition.mesh
    key = ((m.n1, m.n2, m.n3), (float(m.h1), float(m.h2), float(m.h3)),
           (partition.b1, partition.b2, partition.b3), torch.cuda.current_device() if torch.cuda.is_available() else -1)
    if reduced:
        key = key + ("reduced",)
    eng = _ENGINES.get(key)
    if eng is None:
        eng = Engine(*key[:3], reduced=reduced)
        _ENGINES[key] = eng
    return eng
