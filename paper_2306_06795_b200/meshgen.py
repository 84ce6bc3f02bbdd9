"""Input generator for BASELINE config 4: a Delaunay triangulation of a seeded
jittered grid on the unit square (interior points jittered uniformly by
+-jitter*h, boundary points fixed), positively oriented, every boundary edge
tagged DirichletZero, written in the reference mesh JSON schema
(mesh.hpp:81-83: {"vertices", "triangles", "boundary"}). This restates the
recipe of the reference's data/meshes/generate.py with the jitter and tags
BASELINE.json names; the mesh is then read by the reference's read_mesh.
"""
from __future__ import annotations

import json

import numpy as np


def splitmix64_unit(i: int, seed: int = 0x5EED) -> float:
    """u in [0, 1) from splitmix64(seed ^ i) (portable)."""
    m = (1 << 64) - 1
    z = ((seed ^ i) + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    z = z ^ (z >> 31)
    return (z >> 11) * 2.0 ** -53


def force_wavenumbers(seed: int = 2024):
    """k1, k2 ~ U[1, 4] for f = (sin(k1 x), cos(k2 y))."""
    return 1.0 + 3.0 * splitmix64_unit(0, seed), 1.0 + 3.0 * splitmix64_unit(1, seed)


def jittered_delaunay(n: int, seed: int = 7, jitter: float = 0.3) -> dict:
    from scipy.spatial import Delaunay

    rng = np.random.default_rng(seed)
    xs = np.linspace(0.0, 1.0, n + 1)
    gx, gy = np.meshgrid(xs, xs, indexing="ij")
    pts = np.stack([gx.ravel(), gy.ravel()], axis=1)
    h = 1.0 / n
    inner = ((pts[:, 0] > 1e-12) & (pts[:, 0] < 1 - 1e-12) &
             (pts[:, 1] > 1e-12) & (pts[:, 1] < 1 - 1e-12))
    pts[inner] += rng.uniform(-jitter * h, jitter * h, size=(int(inner.sum()), 2))
    tri = Delaunay(pts).simplices.astype(np.int64)
    a, b, c = pts[tri[:, 0]], pts[tri[:, 1]], pts[tri[:, 2]]
    area = 0.5 * ((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1]))
    if np.any(np.abs(area) < 1e-14):
        raise RuntimeError("degenerate triangle")
    neg = area < 0
    tri[neg] = tri[neg][:, [0, 2, 1]]
    e = np.concatenate([tri[:, [0, 1]], tri[:, [1, 2]], tri[:, [2, 0]]])
    e.sort(axis=1)
    uniq, cnt = np.unique(e, axis=0, return_counts=True)
    bnd = uniq[cnt == 1]
    return {"vertices": pts.tolist(), "triangles": tri.tolist(),
            "boundary": [[int(p), int(q), "DirichletZero"] for p, q in bnd]}


def write_mesh(path: str, n: int, seed: int = 7, jitter: float = 0.3) -> str:
    with open(path, "w") as f:
        json.dump(jittered_delaunay(n, seed, jitter), f, separators=(",", ":"))
    return path
