"""Skeleton data of the reduced-dimension boundary conditions as a
differentiable map of the edge weights (extension N4; the
reference has only the model-independent hats, basis.py:84-116).

``SkeletonMap.values(w)`` returns the non-zero skeleton entries of the
prolongation, B(w), in the same formulas as msfv_reduced.cu (the forward
basis build) and oracle/msfv_reduced.py:

  * line nodes between two adjacent coarse nodes: the normalized cumulative
    resistance u(t) = sum_{s >= t} (1/w_s) / sum_s (1/w_s) for the lower end,
    1 - u(t) for the upper end;
  * interior nodes of a face patch between four coarse nodes: the 5-point
    problem of the patch's in-plane edges (conductance w_e / h_e^2) with the
    line solutions as Dirichlet data, one column per corner.

The map is small (O(skeleton) unknowns, batched 1D sums and (b-1)^2-unknown
patch solves), so its derivatives are taken by automatic differentiation of
these tensor formulas: ``vjp`` (d<B, Lambda>/dw, the gradient path) and
``jvp`` (dB for an edge-weight perturbation, the J v path).  The heavy parts
of the sensitivity (interior solves, stencils, coarse solves) stay in the
libmsfv kernels (reduced_sens.py).

Entries are addressed by (full node id, coarse column); node 0 is pinned and
never a line or patch-interior node.
"""

import numpy as np
import torch


def _edge_index(mesh, ax, i, j, k):
    """Reference edge order: x-, y-, z-edges, i fastest (operators.py:36-50)."""
    n1, n2, n3 = mesh.n1, mesh.n2, mesh.n3
    i, j, k = np.asarray(i), np.asarray(j), np.asarray(k)
    if ax == 0:
        return i + n1 * (j + (n2 + 1) * k)
    ex = n1 * (n2 + 1) * (n3 + 1)
    if ax == 1:
        return ex + i + (n1 + 1) * (j + n2 * k)
    ey = (n1 + 1) * n2 * (n3 + 1)
    return ex + ey + i + (n1 + 1) * (j + (n2 + 1) * k)


class SkeletonMap:
    """Index tables of the line segments and face patches of a partition."""

    _cache = {}

    @classmethod
    def get(cls, partition, device):
        mesh = partition.mesh
        # keyed by the geometry, not by id(partition): ids are reused after garbage collection
        key = (mesh.n1, mesh.n2, mesh.n3, float(mesh.h1), float(mesh.h2), float(mesh.h3), partition.b1, partition.b2,
               partition.b3, str(device))
        m = cls._cache.get(key)
        if m is None:
            m = cls._cache[key] = SkeletonMap(partition, device)
        return m

    def __init__(self, partition, device):
        mesh = partition.mesh
        b = (partition.b1, partition.b2, partition.b3)
        nb = tuple(partition.nb)
        h = (mesh.h1, mesh.h2, mesh.h3)
        self.device = device
        self.b, self.nb = b, nb
        dev = lambda a, dt=torch.int64: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=device)  # noqa: E731

        def col(ci, cj, ck):
            return np.asarray(ci) + (nb[0] + 1) * (np.asarray(cj) + (nb[1] + 1) * np.asarray(ck))

        # ---- line segments per axis
        self.lines = []
        seg_id = []                                     # [ax] -> array (nb0+1, nb1+1, nb2+1) of segment ids (-1: none)
        for ax in range(3):
            ext = [nb[0] + 1, nb[1] + 1, nb[2] + 1]
            ext[ax] = nb[ax]
            C = np.stack(np.meshgrid(np.arange(ext[0]), np.arange(ext[1]), np.arange(ext[2]), indexing="ij"),
                         axis=-1).reshape(-1, 3)
            ids = -np.ones((nb[0] + 1, nb[1] + 1, nb[2] + 1), dtype=np.int64)
            ids[C[:, 0], C[:, 1], C[:, 2]] = np.arange(len(C))
            seg_id.append(ids)
            p0 = C * np.array(b)
            s = np.arange(b[ax])
            P = np.repeat(p0[:, None, :], b[ax], axis=1)
            P[:, :, ax] += s[None, :]
            edges = _edge_index(mesh, ax, P[..., 0], P[..., 1], P[..., 2])            # (nseg, b)
            t = np.arange(1, b[ax])
            Pn = np.repeat(p0[:, None, :], max(b[ax] - 1, 0), axis=1)
            if b[ax] > 1:
                Pn[:, :, ax] += t[None, :]
            nodes = mesh.node_index(Pn[..., 0], Pn[..., 1], Pn[..., 2])               # (nseg, b-1) full node ids
            chi = C.copy()
            chi[:, ax] += 1
            cols = np.stack([col(C[:, 0], C[:, 1], C[:, 2]), col(chi[:, 0], chi[:, 1], chi[:, 2])], axis=1)
            self.lines.append(dict(ax=ax, b=b[ax], edges=dev(edges), nodes=dev(nodes), cols=dev(cols),
                                   nseg=len(C)))

        # ---- face patches per normal axis
        self.faces = []
        for ax in range(3):
            ua, va = [d for d in range(3) if d != ax]
            bu, bv = b[ua], b[va]
            if bu < 2 or bv < 2:
                self.faces.append(None)
                continue
            ext = [nb[0], nb[1], nb[2]]
            ext[ax] = nb[ax] + 1
            C = np.stack(np.meshgrid(np.arange(ext[0]), np.arange(ext[1]), np.arange(ext[2]), indexing="ij"),
                         axis=-1).reshape(-1, 3)
            npatch = len(C)
            base = C * np.array(b)
            ni = (bu - 1) * (bv - 1)
            idx = lambda u, v: (u - 1) + (bu - 1) * (v - 1)                            # noqa: E731
            # perimeter line nodes adjacent to interior nodes: 4 lines, local id and (segment, t, low/high corner)
            per = {}
            for v in range(1, bv):
                per[(0, v)] = len(per)
            for v in range(1, bv):
                per[(bu, v)] = len(per)
            for u in range(1, bu):
                per[(u, 0)] = len(per)
            for u in range(1, bu):
                per[(u, bv)] = len(per)
            nper = len(per)
            # local edges touching an interior node: (axis in patch, low point (u, v))
            e_ax, e_lo, e_a, e_b, e_pa, e_pb = [], [], [], [], [], []
            for v in range(1, bv):                       # u-edges (u, v)-(u+1, v), u = 0 .. bu-1
                for u in range(0, bu):
                    e_ax.append(0)
                    e_lo.append((u, v))
            for v in range(0, bv):                       # v-edges (u, v)-(u, v+1), u = 1 .. bu-1
                for u in range(1, bu):
                    e_ax.append(1)
                    e_lo.append((u, v))
            for eax, (u, v) in zip(e_ax, e_lo):
                pa, pb = (u, v), ((u + 1, v) if eax == 0 else (u, v + 1))
                ins = lambda p: 1 <= p[0] < bu and 1 <= p[1] < bv                      # noqa: E731
                e_a.append(idx(*pa) if ins(pa) else -1)
                e_b.append(idx(*pb) if ins(pb) else -1)
                e_pa.append(per.get(pa, -1) if not ins(pa) else -1)
                e_pb.append(per.get(pb, -1) if not ins(pb) else -1)
            e_ax, e_a, e_b, e_pa, e_pb = map(np.array, (e_ax, e_a, e_b, e_pa, e_pb))
            lo = np.array(e_lo)
            # global edge ids (npatch, nedge)
            Pe = np.repeat(base[:, None, :], len(lo), axis=1)
            Pe[:, :, ua] += lo[None, :, 0]
            Pe[:, :, va] += lo[None, :, 1]
            eglob = np.empty((npatch, len(lo)), dtype=np.int64)
            for a_loc, a_glob in ((0, ua), (1, va)):
                sel = e_ax == a_loc
                eglob[:, sel] = _edge_index(mesh, a_glob, Pe[:, sel, 0], Pe[:, sel, 1], Pe[:, sel, 2])
            ih2 = np.where(e_ax == 0, 1.0 / h[ua] ** 2, 1.0 / h[va] ** 2)
            # interior nodes (npatch, ni) and the 4 corner columns (c4 = 2 du + dv)
            uu, vv = np.meshgrid(np.arange(1, bu), np.arange(1, bv), indexing="ij")
            order = np.argsort(idx(uu, vv).ravel())
            uu, vv = uu.ravel()[order], vv.ravel()[order]
            Pn = np.repeat(base[:, None, :], ni, axis=1)
            Pn[:, :, ua] += uu[None, :]
            Pn[:, :, va] += vv[None, :]
            nodes = mesh.node_index(Pn[..., 0], Pn[..., 1], Pn[..., 2])
            cols = np.empty((npatch, 4), dtype=np.int64)
            for du in (0, 1):
                for dv in (0, 1):
                    cc = C.copy()
                    cc[:, ua] += du
                    cc[:, va] += dv
                    cols[:, 2 * du + dv] = col(cc[:, 0], cc[:, 1], cc[:, 2])
            # perimeter values from the line solutions: (line axis, segment id, t, c4 of low end, c4 of high end)
            p_ax = np.empty(nper, dtype=np.int64)
            p_t = np.empty(nper, dtype=np.int64)
            p_lo4 = np.empty(nper, dtype=np.int64)
            p_hi4 = np.empty(nper, dtype=np.int64)
            p_seg = np.empty((npatch, nper), dtype=np.int64)
            for (u, v), q in per.items():
                if u in (0, bu):                         # line along va at u = 0 / bu
                    du = 0 if u == 0 else 1
                    p_ax[q], p_t[q], p_lo4[q], p_hi4[q] = va, v, 2 * du + 0, 2 * du + 1
                    cc = C.copy()
                    cc[:, ua] += du
                else:                                    # line along ua at v = 0 / bv
                    dv = 0 if v == 0 else 1
                    p_ax[q], p_t[q], p_lo4[q], p_hi4[q] = ua, u, 0 + dv, 2 + dv
                    cc = C.copy()
                    cc[:, va] += dv
                p_seg[:, q] = seg_id[p_ax[q]][cc[:, 0], cc[:, 1], cc[:, 2]]
            assert (p_seg >= 0).all()
            # assembly plans: (target, flat positions, edge selection, sign), device tensors built once
            ia, ib = e_a >= 0, e_b >= 0
            plan = []
            for tgt, rows, cols_, ncol, sel, sign in (("A", e_a, e_a, ni, ia, 1.0), ("A", e_b, e_b, ni, ib, 1.0),
                                                      ("A", e_a, e_b, ni, ia & ib, -1.0),
                                                      ("A", e_b, e_a, ni, ia & ib, -1.0),
                                                      ("K", e_a, e_pb, nper, ia & (e_pb >= 0), 1.0),
                                                      ("K", e_b, e_pa, nper, ib & (e_pa >= 0), 1.0)):
                if sel.any():
                    plan.append((tgt, dev(rows[sel] * ncol + cols_[sel]), dev(np.flatnonzero(sel)), sign))
            # perimeter values: per line axis the perimeter slots it feeds
            pplan = []
            for a_line in (ua, va):
                q = np.flatnonzero(p_ax == a_line)
                pplan.append((a_line, dev(q), dev(p_seg[:, q]), dev(p_t[q]), dev(p_lo4[q]), dev(p_hi4[q])))
            self.faces.append(dict(ax=ax, ua=ua, va=va, ni=ni, nper=nper, npatch=npatch, eglob=dev(eglob),
                                   ih2=dev(ih2, torch.float64), plan=plan, pplan=pplan, nodes=dev(nodes),
                                   cols=dev(cols)))
        self._entries = None

    # ------------------------------------------------------------------ forward
    def _line_lo(self, w):
        """Per axis: u(t), t = 0 .. b (nseg, b + 1), the lower end's values."""
        out = []
        for L in self.lines:
            r = 1.0 / w[L["edges"]]                                                     # (nseg, b)
            tail = torch.flip(torch.cumsum(torch.flip(r, dims=[1]), dim=1), dims=[1])   # sum_{s >= t}
            lo = torch.cat([tail, torch.zeros_like(tail[:, :1])], dim=1) / r.sum(dim=1, keepdim=True)
            out.append(lo)
        return out

    def values(self, w):
        """Non-zero skeleton entries B(w) as one flat vector, ordered like ``entries()``."""
        los = self._line_lo(w)
        parts = []
        for L, lo in zip(self.lines, los):
            if L["b"] > 1:
                u = lo[:, 1:L["b"]]                                                     # (nseg, b-1)
                parts.append(torch.stack([u, 1.0 - u], dim=2).reshape(-1))
        for F in self.faces:
            if F is None:
                continue
            npatch, ni, nper = F["npatch"], F["ni"], F["nper"]
            k = w[F["eglob"]] * F["ih2"][None, :]                                       # (npatch, nedge)
            A = torch.zeros(npatch, ni * ni, dtype=w.dtype, device=w.device)
            K = torch.zeros(npatch, ni * nper, dtype=w.dtype, device=w.device)
            for tgt, flat, sel, sign in F["plan"]:
                (A if tgt == "A" else K).index_add_(1, flat, sign * k[:, sel])
            # perimeter values (npatch, nper, 4) from the line solutions
            V = torch.zeros(npatch, nper, 4, dtype=w.dtype, device=w.device)
            for a_line, q, seg, t, lo4, hi4 in F["pplan"]:
                lo = los[a_line][seg, t[None, :]]                                       # (npatch, nq)
                V[:, q, lo4] = lo
                V[:, q, hi4] = 1.0 - lo
            rhs = K.reshape(npatch, ni, nper) @ V
            sol = torch.linalg.solve(A.reshape(npatch, ni, ni), rhs)                    # (npatch, ni, 4)
            parts.append(sol.reshape(-1))
        return torch.cat(parts) if parts else torch.zeros(0, dtype=w.dtype, device=w.device)

    def entries(self):
        """(full node ids, coarse columns) of the entries, in the order of ``values``."""
        if self._entries is None:
            nodes, cols = [], []
            for L in self.lines:
                if L["b"] > 1:
                    n = L["nodes"][:, :, None].expand(-1, -1, 2)
                    c = L["cols"][:, None, :].expand(-1, L["b"] - 1, -1)
                    nodes.append(n.reshape(-1))
                    cols.append(c.reshape(-1))
            for F in self.faces:
                if F is None:
                    continue
                n = F["nodes"][:, :, None].expand(-1, -1, 4)
                c = F["cols"][:, None, :].expand(-1, F["ni"], -1)
                nodes.append(n.reshape(-1))
                cols.append(c.reshape(-1))
            z = torch.zeros(0, dtype=torch.int64, device=self.device)
            self._entries = (torch.cat(nodes) if nodes else z, torch.cat(cols) if cols else z)
        return self._entries

    # ------------------------------------------- structured entry contractions
    # The entries come in groups (a line segment: b-1 nodes x 2 columns; a face
    # patch: (bu-1)(bv-1) nodes x 4 columns), so products with node fields and
    # coefficient rows are small batched matrix products instead of per-entry
    # gathers of ns-wide rows.
    def _group_tables(self):
        if getattr(self, "_gt", None) is None:
            gt = []
            for L in self.lines:
                if L["b"] > 1:
                    gt.append((L["nodes"], L["cols"]))
            for F in self.faces:
                if F is not None:
                    gt.append((F["nodes"], F["cols"]))
            self._gt = gt
        return self._gt

    def contract(self, Fn, Fc):
        """e[g, i, c] = sum_s Fn[nodes[g, i], s] Fc[cols[g, c], s], flat in the order of ``values``."""
        return torch.cat([torch.bmm(Fn[n], Fc[c].transpose(1, 2)).reshape(-1) for n, c in self._group_tables()])

    def _split(self, v):
        out, o = [], 0
        for n, c in self._group_tables():
            m = n.numel() * c.shape[1]
            out.append(v[o:o + m].reshape(n.shape[0], n.shape[1], c.shape[1]))
            o += m
        return out

    def spread_nodes(self, v, Fc, n_nodes):
        """f[nodes[g, i], :] = sum_c v[g, i, c] Fc[cols[g, c], :]  (every node belongs to one group)."""
        f = torch.zeros(n_nodes, Fc.shape[1], dtype=Fc.dtype, device=Fc.device)
        for (n, c), vg in zip(self._group_tables(), self._split(v)):
            f[n.reshape(-1)] = torch.bmm(vg, Fc[c]).reshape(-1, Fc.shape[1])
        return f

    def spread_cols(self, v, Fn, n_cols):
        """out[col, :] = sum over groups and nodes of v[g, i, c] Fn[nodes[g, i], :] for cols[g, c] == col
        (fixed-order segment sums over the (group, column) products)."""
        parts, cols = [], []
        for (n, c), vg in zip(self._group_tables(), self._split(v)):
            parts.append(torch.bmm(vg.transpose(1, 2), Fn[n]).reshape(-1, Fn.shape[1]))
            cols.append(c.reshape(-1))
        data, cols = torch.cat(parts), torch.cat(cols)
        if getattr(self, "_cperm", None) is None or self._cperm[0] != n_cols:
            self._cperm = (n_cols, torch.argsort(cols, stable=True), torch.bincount(cols, minlength=n_cols))
        _, perm, cnt = self._cperm
        return torch.segment_reduce(data[perm].contiguous(), "sum", lengths=cnt, axis=0, initial=0.0)

    # ------------------------------------------------------------ derivatives
    def vjp(self, w, lam):
        """d<B(w), lam>/dw for entry weights ``lam`` (the gradient path)."""
        wr = w.detach().clone().requires_grad_(True)
        with torch.enable_grad():
            s = torch.dot(self.values(wr), lam.detach())
        (g,) = torch.autograd.grad(s, wr)
        return g

    def jvp(self, w, dw):
        """dB for the edge-weight perturbation ``dw`` (the J v path)."""
        _, out = torch.autograd.functional.jvp(self.values, (w.detach(),), (dw.detach(),))
        return out
