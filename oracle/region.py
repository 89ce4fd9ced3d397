"""TEST/BASELINE INFRASTRUCTURE ONLY — restatement of the reference's region (covering)
path, used by bench.py's CPU reference arm and cpu_baseline to time bounded samples of the
reference algorithm on the host cores.  Never imported by the shipped package.

Follows: partition.py:29-164 (covering, nearest-centre assignment, Voronoi-sort regions),
pipeline.py:62-98 (_region_task), delaunay.py:91-114, 205-227, 252-273 (cap Delaunay by
stereographic projection + SciPy/Qhull planar Delaunay, interior selection),
geometry.py:45-83 (tangent frame, stereographic projection).
"""

from __future__ import annotations

import numpy as np
from scipy.spatial import Delaunay

from .scvt_oracle import (RULES, Fans, build_fans, canonical_sort, cell_quadrature,
                          convex_hull_delaunay, geodesic_distance, normalize, sample_by_density,
                          subdivide)


def tangent_frame(contact):
    """geometry.py:53-66."""
    t = normalize(np.asarray(contact, dtype=float))
    seed = np.zeros(3)
    seed[np.argmin(np.abs(t))] = 1.0
    e1 = normalize(np.cross(t, seed))
    return t, e1, np.cross(t, e1)


def stereographic_project(z, t, e1, e2, eps=1e-9):
    """geometry.py:67-83."""
    denom = np.sum(t * (z + t), axis=-1)
    if np.any(denom <= eps):
        raise ValueError("antipode")
    s = 2.0 / denom
    x = s[..., None] * z + (s - 1.0)[..., None] * t
    return np.stack([np.sum((x - t) * e1, axis=-1), np.sum((x - t) * e2, axis=-1)], axis=-1)


def neighbor_lists(triangles, p):
    """partition.py:66-79 (one-level lists only)."""
    adj = [set() for _ in range(p)]
    for a, b, c in np.asarray(triangles):
        adj[a].update((b, c))
        adj[b].update((a, c))
        adj[c].update((a, b))
    return tuple(tuple(sorted(s)) for s in adj)


def bootstrap_covering(p, seed, density, movement_tol=1e-3, max_iterations=200):
    """partition.py:82-120: coarse density-matched CVT of p cells (Lloyd, 4-pt rule)."""
    centers = sample_by_density(density, p, seed)
    tri = convex_hull_delaunay(centers)
    for _ in range(max_iterations):
        f = build_fans(centers, tri)
        _, first, _ = cell_quadrature(centers, f, density, RULES["4pt"], p)
        new = normalize(first)
        movement = np.abs(new - centers).max()
        centers = new
        tri = convex_hull_delaunay(centers)
        if movement <= movement_tol:
            break
    return centers, neighbor_lists(tri, p)


def nearest_cell(points, centers, chunk=1 << 16):
    """partition.py:60-63 (chunked argmax of Z . centers^T)."""
    out = np.empty(len(points), dtype=np.int64)
    for s in range(0, len(points), chunk):
        out[s:s + chunk] = np.argmax(points[s:s + chunk] @ centers.T, axis=1)
    return out


def region_payload(points, geometric, centers, one_level, l):
    """pipeline.py:171-197 for region l."""
    region = np.asarray((l,) + one_level[l], dtype=int)
    members = np.flatnonzero(np.isin(geometric, region))
    owned = geometric[members] == l
    return {"coords": points[members], "ids": members, "owned": owned, "contact": centers[l],
            "centers": centers, "region": region}


def region_task(payload, density, rule="7pt", depth=3, chunk=16384):
    """pipeline.py:62-98: cap Delaunay -> interior selection -> owned fans -> quadrature.
    Returns (owned ids, mass, first, energy)."""
    coords, ids, owned = payload["coords"], payload["ids"], payload["owned"]
    t, e1, e2 = tangent_frame(payload["contact"])
    plane = stereographic_project(coords, t, e1, e2)
    dt = Delaunay(plane)
    tri = dt.simplices.astype(np.int64)
    v = coords[tri]
    det = np.einsum("ij,ij->i", v[:, 0], np.cross(v[:, 1], v[:, 2]))
    flip = det < 0
    tri[flip] = tri[flip][:, [0, 2, 1]]
    # spherical circumcircles avoiding the projection antipode (delaunay.py:150-169)
    v = coords[tri]
    n = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
    centers_t = n / np.linalg.norm(n, axis=1, keepdims=True)
    radii = geodesic_distance(centers_t, v[:, 0])
    wraps = geodesic_distance(centers_t, -t) < radii
    centers_t[wraps] = -centers_t[wraps]
    radii[wraps] = np.pi - radii[wraps]
    # select_region_triangles (delaunay.py:252-273)
    cen = payload["centers"]
    inside = np.zeros(len(cen), dtype=bool)
    inside[payload["region"]] = True
    d = np.arccos(np.clip(centers_t @ cen.T, -1.0, 1.0))
    keep = d[:, ~inside].min(axis=1) - d[:, inside].min(axis=1) >= 2.0 * radii
    tri = canonical_sort(tri[keep])
    f = build_fans(coords, tri)
    sel = owned[f.cells]
    f = Fans(f.verts[sel], f.cells[sel], f.edge_other[sel], f.signed_area[sel], f.obtuse_count)
    k = len(coords)
    mass = np.zeros(k)
    first = np.zeros((k, 3))
    energy = 0.0
    S = len(f.cells)
    for s in range(0, S, chunk):
        e = min(S, s + chunk)
        sub = subdivide(Fans(f.verts[s:e], f.cells[s:e], f.edge_other[s:e], f.signed_area[s:e],
                             0), depth)
        m, c, en = cell_quadrature(coords, sub, density, RULES[rule], k)
        mass += m
        first += c
        energy += en
    return ids[owned], mass[owned], first[owned], energy
