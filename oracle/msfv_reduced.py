"""CPU oracle for the reduced-dimension boundary conditions.

TEST INFRASTRUCTURE ONLY (imported by tests/, never by the product path).

The reference builds the Lagrange basis from trilinear hats on the skeleton
(generate_bc_lagrange, basis.py:84-116) and states "no reduced-dimension edge
problems", so there is no reference output for this extension
("parity unpinned"; validated by the reference's own basis properties:
partition of unity and sigma == 1 reproducing the hats, tests/test_reduced.py).
The classical MSFV localization (BASELINE.json north_star) replaces the hats by
reduced problems with the model's conductances along the skeleton:

  * line segments between adjacent coarse nodes (1D): -d/dx (k du/dx) = 0 with
    u = 1 at one end, 0 at the other; k the edge weights w = C sigma of the
    segment's edges: the discrete solution is the normalized cumulative
    resistance, u(t) = sum_{s >= t} (1/w_s) / sum_s (1/w_s) for the lower end;
  * face patches between four coarse nodes (2D): the 5-point problem of the
    patch's in-plane edges (conductance w_e / h_e^2) on its interior nodes,
    Dirichlet data on the patch perimeter from the line solutions (the coarse
    corner's own value 1, the other corners 0);
  * block interiors (3D): unchanged (the Lagrange local problems with these
    boundary values).

``reduced_values(part, w)`` returns the skeleton data as the n x k CSC matrix
the reference's BC generators return (pinned node 0 dropped), with the same
sparsity pattern as the hats; ``build_basis_reduced`` feeds it through the
oracle's cache/basis path (build_cache(values=...), basis.py:421-616).
"""

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import msfv_oracle as orc


def _edge_index(mesh, ax, i, j, k):
    """Reference edge order: x-edges, y-edges, z-edges, i fastest (operators.py:36-50)."""
    n1, n2, n3 = mesh.n1, mesh.n2, mesh.n3
    if ax == 0:
        return i + n1 * (j + (n2 + 1) * k)
    ex = n1 * (n2 + 1) * (n3 + 1)
    if ax == 1:
        return ex + i + (n1 + 1) * (j + n2 * k)
    ey = (n1 + 1) * n2 * (n3 + 1)
    return ex + ey + i + (n1 + 1) * (j + (n2 + 1) * k)


def reduced_values(part, w):
    mesh = part.mesh
    b = part.b
    nb = part.nb
    h = (mesh.h1, mesh.h2, mesh.h3)
    n = mesh.n_nodes - 1
    vals = {}                                  # (node, coarse column) -> value

    def coarse_col(ci, cj, ck):
        return ci + (nb[0] + 1) * (cj + (nb[1] + 1) * ck)

    def node(p):
        return mesh.node(int(p[0]), int(p[1]), int(p[2]))

    # coarse nodes themselves
    for ck in range(nb[2] + 1):
        for cj in range(nb[1] + 1):
            for ci in range(nb[0] + 1):
                vals[(node((ci * b[0], cj * b[1], ck * b[2])), coarse_col(ci, cj, ck))] = 1.0

    for ax in range(3):
        rng = [range(nb[0] + 1), range(nb[1] + 1), range(nb[2] + 1)]
        rng[ax] = range(nb[ax])
        for ck in rng[2]:
            for cj in rng[1]:
                for ci in rng[0]:
                    c = [ci, cj, ck]
                    p0 = [ci * b[0], cj * b[1], ck * b[2]]
                    r = np.empty(b[ax])
                    for s in range(b[ax]):
                        q = list(p0)
                        q[ax] += s
                        r[s] = 1.0 / w[_edge_index(mesh, ax, *q)]
                    R = r.sum()
                    lo = np.array([r[t:].sum() / R for t in range(b[ax] + 1)])
                    c_hi = list(c)
                    c_hi[ax] += 1
                    for t in range(1, b[ax]):
                        q = list(p0)
                        q[ax] += t
                        vals[(node(q), coarse_col(*c))] = lo[t]
                        vals[(node(q), coarse_col(*c_hi))] = r[:t].sum() / R

    # face patches
    for ax in range(3):
        ua, va = [d for d in range(3) if d != ax]
        bu, bv = b[ua], b[va]
        rng = [range(nb[0]), range(nb[1]), range(nb[2])]
        rng[ax] = range(nb[ax] + 1)
        for ck in rng[2]:
            for cj in rng[1]:
                for ci in rng[0]:
                    base = [ci * b[0], cj * b[1], ck * b[2]]
                    if bu < 2 or bv < 2:
                        continue
                    ni = (bu - 1) * (bv - 1)
                    A = np.zeros((ni, ni))
                    corners = []
                    for du in (0, 1):
                        for dv in (0, 1):
                            cc = [ci, cj, ck]
                            cc[ua] += du
                            cc[va] += dv
                            corners.append(tuple(cc))
                    rhs = np.zeros((ni, 4))
                    idx = lambda u, v: (u - 1) + (bu - 1) * (v - 1)    # noqa: E731
                    for v in range(1, bv):
                        for u in range(1, bu):
                            row = idx(u, v)
                            p = list(base)
                            p[ua] += u
                            p[va] += v
                            for d, (du, dv) in enumerate(((-1, 0), (1, 0), (0, -1), (0, 1))):
                                eax = ua if du else va
                                q = list(p)
                                q[ua] += du
                                q[va] += dv
                                lowp = list(p)
                                if du < 0 or dv < 0:
                                    lowp = q
                                k_e = w[_edge_index(mesh, eax, *lowp)] / h[eax] ** 2
                                A[row, row] += k_e
                                uu, vv = u + du, v + dv
                                if 1 <= uu < bu and 1 <= vv < bv:
                                    A[row, idx(uu, vv)] -= k_e
                                else:
                                    # perimeter node: a line node or a coarse node (values set above)
                                    for c4, corner in enumerate(corners):
                                        rhs[row, c4] += k_e * vals.get((node(q), coarse_col(*corner)), 0.0)
                    sol = sla.cho_solve(sla.cho_factor(A, lower=True), rhs)
                    for v in range(1, bv):
                        for u in range(1, bu):
                            p = list(base)
                            p[ua] += u
                            p[va] += v
                            for c4, corner in enumerate(corners):
                                vals[(node(p), coarse_col(*corner))] = sol[idx(u, v), c4]
    rows, cols, data = [], [], []
    for (nd, c), v in vals.items():
        if nd == 0 or v == 0.0:
            continue
        rows.append(nd - 1)
        cols.append(c)
        data.append(v)
    return sp.csc_matrix((data, (rows, cols)), shape=(n, part.n_coarse))


def build_basis_reduced(op, part):
    """Oracle basis with reduced-dimension boundary conditions at the operator's model."""
    values = reduced_values(part, op.w)
    cache = orc.build_cache(part, op.G, op.C, values=values)
    return orc.build_basis(op, part, cache)


def forward_reduced(op, survey, part):
    basis = build_basis_reduced(op, part)
    return orc.forward_reduced(op, survey, basis)
