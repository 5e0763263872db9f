"""Diffusion operator A(m) = G^T diag(C exp(m)) G with node 0 pinned.

Drop-in for the reference's operators.py.  ``assemble_operator`` keeps its
signature (operators.py:164-166) but evaluates sigma and the edge weights on
the GPU (K1); the scipy matrices ``G``, ``C`` and ``A`` are only materialised
on the host when a caller reads ``.grad`` / ``.cell_map`` / ``.A`` (they are
not on the hot path).
"""

import numpy as np
import scipy.sparse as sp

from .errors import InvalidModelError

PINNED_NODE = 0


def sigma_map(m):
    """Cell conductivities exp(m) (operators.py:23-28)."""
    m = np.asarray(m, dtype=float)
    if not np.all(np.isfinite(m)):
        raise InvalidModelError("model vector contains non-finite entries")
    return np.exp(m)


def sigma_deriv(m):
    """Diagonal of d sigma / d m (operators.py:31-33)."""
    return sigma_map(m)


def _axis_shapes(mesh):
    n1, n2, n3 = mesh.n1, mesh.n2, mesh.n3
    return ((n1, n2 + 1, n3 + 1), (n1 + 1, n2, n3 + 1), (n1 + 1, n2 + 1, n3))


def _axis_grid(shape):
    # i fastest, then j, then k (the reference's ravel(order="F"))
    k, j, i = np.meshgrid(np.arange(shape[2]), np.arange(shape[1]), np.arange(shape[0]), indexing="ij")
    return i.ravel(), j.ravel(), k.ravel()


def nodal_gradient(mesh):
    """Edge-by-node difference operator, entries +-1/h (operators.py:53-74)."""
    h = (mesh.h1, mesh.h2, mesh.h3)
    indptr, indices, data = [], [], []
    for ax, shape in enumerate(_axis_shapes(mesh)):
        i, j, k = _axis_grid(shape)
        a = mesh.node_index(i, j, k)
        step = np.zeros(3, dtype=np.int64)
        step[ax] = 1
        b = mesh.node_index(i + step[0], j + step[1], k + step[2])
        indices.append(np.column_stack([a, b]).ravel())
        inv = 1.0 / h[ax]
        data.append(np.tile([-inv, inv], a.size))
    idx = np.concatenate(indices)
    ne = idx.size // 2
    return sp.csr_matrix((np.concatenate(data), idx, np.arange(0, 2 * ne + 1, 2)),
                         shape=(ne, mesh.n_nodes))


def edge_cell_map(mesh):
    """Edge-by-cell averaging map, V/4 per touching cell (operators.py:77-109)."""
    nmax = (mesh.n1, mesh.n2, mesh.n3)
    quarter = 0.25 * mesh.cell_volume
    rows, cols, off = [], [], 0
    for ax, shape in enumerate(_axis_shapes(mesh)):
        ijk = _axis_grid(shape)
        r = off + np.arange(ijk[0].size)
        t1, t2 = [a for a in range(3) if a != ax]
        for d2 in (-1, 0):
            for d1 in (-1, 0):
                c = [x.copy() for x in ijk]
                c[t1] = c[t1] + d1
                c[t2] = c[t2] + d2
                ok = (c[t1] >= 0) & (c[t1] < nmax[t1]) & (c[t2] >= 0) & (c[t2] < nmax[t2])
                rows.append(r[ok])
                cols.append(mesh.cell_index(c[0][ok], c[1][ok], c[2][ok]))
        off += ijk[0].size
    rows = np.concatenate(rows)
    C = sp.coo_matrix((np.full(rows.size, quarter), (rows, np.concatenate(cols))),
                      shape=(off, mesh.n_cells))
    return C.tocsr()


class DiffusionOperator:
    """A(m) with the model's sigma and edge weights resident on the GPU.

    Attributes mirror operators.py:112-161; host copies are produced lazily.
    """

    def __init__(self, mesh, m, pieces=None, engine=None):
        if hasattr(m, "detach"):       # torch tensor (host or device)
            m_np = None
            if m.numel() != mesh.n_cells:
                raise ValueError(f"model length {m.numel()} != number of cells {mesh.n_cells}")
        else:
            m_np = np.asarray(m, dtype=float)
            if m_np.shape != (mesh.n_cells,):
                raise ValueError(f"model length {m_np.size} != number of cells {mesh.n_cells}")
        self.mesh = mesh
        self._pieces = pieces
        self.pinned_node = PINNED_NODE
        self._engine = engine
        self._m_host = m_np
        self._m_src = m
        self._dev = None            # (engine, m_dev, sigma_dev, w_dev)
        self._A = None

    # ---- device state (bound to a partition's engine on first use)
    def device_state(self, engine):
        if self._dev is not None and self._dev[0] is engine:
            return self._dev
        from .engine import require_cuda
        require_cuda()
        src = self._m_src if self._m_host is None else self._m_host
        m_dev = engine.to_device(src).reshape(-1)
        sigma, w, fl = engine.operator(m_dev)
        # status bits accumulate along the forward chain (operator, basis,
        # coarse factor) and are read once, when a result is handed back
        self.flags = fl
        self._dev = (engine, m_dev, sigma, w)
        return self._dev

    def bind(self, engine):
        self.device_state(engine)
        return self

    # ---- reference attributes
    @property
    def m(self):
        if self._m_host is None:
            self._m_host = self._m_src.detach().to("cpu", dtype=__import__("torch").float64).numpy().copy()
        return self._m_host

    @property
    def sigma(self):
        if self._dev is not None:
            return self._dev[2].cpu().numpy()
        return sigma_map(self.m)

    @property
    def edge_weights(self):
        if self._dev is not None:
            return self._dev[3].cpu().numpy()
        return self.cell_map @ self.sigma

    @property
    def pieces(self):
        if self._pieces is None:
            self._pieces = (nodal_gradient(self.mesh), edge_cell_map(self.mesh))
        return self._pieces

    @property
    def grad(self):
        return self.pieces[0]

    @property
    def cell_map(self):
        return self.pieces[1]

    @property
    def unpinned(self):
        G = self.grad
        return (G.T @ sp.diags(self.edge_weights) @ G).tocsr()

    @property
    def A(self):
        if self._A is None:
            Gp = self.grad[:, 1:]
            self._A = (Gp.T @ sp.diags(self.edge_weights) @ Gp).tocsr()
            self._A.sort_indices()
        return self._A

    @property
    def n(self):
        return self.mesh.n_nodes - 1

    def pad(self, u):
        u = np.asarray(u)
        return np.concatenate([np.zeros((1,) + u.shape[1:], dtype=u.dtype), u], axis=0)

    def unpad(self, u_full):
        return np.asarray(u_full)[1:]


def assemble_operator(mesh, m, pieces=None):
    """A(m) (operators.py:164-166).  sigma and the edge weights are evaluated on
    the device when a basis or forward call binds the operator to a partition;
    the finiteness / positivity checks of operators.py:26-27,128-129 run there
    too and raise InvalidModelError at the first result read back to the host
    (no host pass over m on the hot path)."""
    return DiffusionOperator(mesh, m, pieces=pieces)


def grad_A_u_full(mesh, m, u_full, pieces=None):
    """d(A(m) u)/dm for a fixed full-space field (operators.py:169-180); host, test helper."""
    u_full = np.asarray(u_full, dtype=float)
    if u_full.shape != (mesh.n_nodes,):
        raise ValueError(f"field length {u_full.size} != number of nodes {mesh.n_nodes}")
    G, C = pieces if pieces is not None else (nodal_gradient(mesh), edge_cell_map(mesh))
    return (G.T @ sp.diags(G @ u_full) @ C @ sp.diags(sigma_deriv(m))).tocsr()


def grad_A_u(mesh, m, u, pieces=None):
    u = np.asarray(u, dtype=float)
    if u.shape != (mesh.n_nodes - 1,):
        raise ValueError(f"field length {u.size} != pinned dimension {mesh.n_nodes - 1}")
    return grad_A_u_full(mesh, m, np.concatenate([[0.0], u]), pieces=pieces)[1:]
