"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference ships block/salt models and a top-surface survey
(models.py:9-83); BASELINE.json's 3D configs ask for smoothed Gaussian
random fields.  Recipe: standard normal on the (n3, n2, n1)
grid from ``default_rng(seed)``, ``gaussian_filter(mode="reflect")``,
rescaled to the requested std, flattened x-fastest.
"""

import numpy as np
import scipy.sparse as sp

from .forward import Survey


def gaussian_field(mesh, sigma_cells, std, seed):
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(seed)
    g = gaussian_filter(rng.standard_normal((mesh.n3, mesh.n2, mesh.n1)), sigma_cells, mode="reflect")
    g = std * (g - g.mean()) / g.std()
    return g.ravel()


def _surface_positions(count, n):
    """``count`` positions spread over the interior of [0, n] (models.py:46-51)."""
    if count < 1:
        raise ValueError("survey counts must be >= 1")
    return np.unique(np.round(np.linspace(0, n, count + 2))[1:-1].astype(int))


def build_survey(mesh, n_src=(3, 3), n_rec=(8, 8)):
    """Top-plane x-dipoles and point receivers, pinned ids (models.py:54-83)."""
    n = mesh.n_nodes - 1
    kt = mesh.n3
    sx = _surface_positions(n_src[0], mesh.n1 - 1)
    sy = _surface_positions(n_src[1], mesh.n2)
    J, I = np.meshgrid(sy, sx, indexing="ij")
    a = mesh.node_index(I.ravel(), J.ravel(), kt) - 1
    ns = a.size
    Q = sp.csc_matrix((np.tile([1.0, -1.0], ns), np.column_stack([a, a + 1]).ravel(),
                       np.arange(0, 2 * ns + 1, 2)), shape=(n, ns))
    rx = _surface_positions(n_rec[0], mesh.n1)
    ry = _surface_positions(n_rec[1], mesh.n2)
    J, I = np.meshgrid(ry, rx, indexing="ij")
    rec = mesh.node_index(I.ravel(), J.ravel(), kt) - 1
    P = sp.csc_matrix((np.ones(rec.size), rec, np.arange(rec.size + 1)), shape=(n, rec.size))
    return Survey(P=P, Q=Q)


# BASELINE.json configs 3-5 (3D).  Unit cube: h = 1/n.
CONFIGS = {
    3: dict(n=64, b=8, field=(4.0, 1.0), anomaly="cube", n_src=(2, 2), n_rec=(16, 16)),
    4: dict(n=128, b=8, field=(6.0, 1.5), anomaly=None, n_src=(4, 4), n_rec=(32, 32)),
    5: dict(n=256, b=8, field=(8.0, 1.0), anomaly="boxes", n_src=(8, 4), n_rec=(64, 64)),
}


def config_model(mesh, cfg, seed):
    m = gaussian_field(mesh, cfg["field"][0], cfg["field"][1], seed)
    n1, n2, n3 = mesh.n1, mesh.n2, mesh.n3
    ci, cj, ck = mesh.cell_triple(np.arange(mesh.n_cells))
    x, y, z = (ci + 0.5) / n1, (cj + 0.5) / n2, (ck + 0.5) / n3
    if cfg["anomaly"] == "cube":
        m = m + 2.0 * ((x >= 0.4) & (x <= 0.6) & (y >= 0.4) & (y <= 0.6) & (z >= 0.4) & (z <= 0.6))
    elif cfg["anomaly"] == "boxes":
        rng = np.random.default_rng(seed + 7)
        for _ in range(3):
            amp = rng.uniform(-2, 2)
            lo = rng.uniform(0, 0.8, 3)
            side = rng.uniform(0.1, 0.3, 3)
            hi = lo + side
            m = m + amp * ((x >= lo[0]) & (x <= hi[0]) & (y >= lo[1]) & (y <= hi[1])
                           & (z >= lo[2]) & (z <= hi[2]))
    return m


def config_problem(cfg_id, seed=0):
    """(mesh, partition, survey, m) for a BASELINE.json 3D config."""
    from .mesh import create_mesh, create_partition
    cfg = CONFIGS[cfg_id]
    n = cfg["n"]
    mesh = create_mesh(n, n, n, 1.0 / n, 1.0 / n, 1.0 / n)
    part = create_partition(mesh, cfg["b"], cfg["b"], cfg["b"])
    survey = build_survey(mesh, cfg["n_src"], cfg["n_rec"])
    return mesh, part, survey, config_model(mesh, cfg, seed)


def top_random_survey(mesh, n_rec, n_src, seed):
    """Seeded receivers and x-dipoles at random top-plane nodes (the layout of
    models.py:54-83 with random positions instead of a regular grid)."""
    rng = np.random.default_rng(seed)
    n = mesh.n_nodes - 1
    I, J = np.meshgrid(np.arange(mesh.n1 + 1), np.arange(mesh.n2 + 1), indexing="ij")
    top = np.sort(mesh.node_index(I.ravel(), J.ravel(), mesh.n3)) - 1
    rec = np.sort(rng.choice(top, size=n_rec, replace=False))
    P = sp.csc_matrix((np.ones(n_rec), (rec, np.arange(n_rec))), shape=(n, n_rec))
    i = rng.choice(mesh.n1, size=n_src, replace=n_src > mesh.n1)
    j = rng.integers(0, mesh.n2 + 1, size=n_src)
    a = mesh.node_index(i, j, mesh.n3) - 1
    Q = sp.csc_matrix((np.tile([1.0, -1.0], n_src), np.column_stack([a, a + 1]).ravel(),
                       np.arange(0, 2 * n_src + 1, 2)), shape=(n, n_src))
    return Survey(P=P, Q=Q)


def table3_problem(seed=0):
    """The paper's Table-3 geometry: 64 x 64 x 32 cells,
    16^3-cell coarse blocks, 72 sources and 3698 receivers (here on the top
    plane), m a smoothed Gaussian field (sigma 4 cells, std 1) from the seed.
    Returns (mesh, partition, survey, m)."""
    from .mesh import create_mesh, create_partition
    mesh = create_mesh(64, 64, 32, 1 / 64, 1 / 64, 1 / 64)
    part = create_partition(mesh, 16, 16, 16)
    survey = top_random_survey(mesh, 3698, 72, seed + 1)
    return mesh, part, survey, gaussian_field(mesh, 4.0, 1.0, seed)
