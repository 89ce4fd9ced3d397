"""Host-side geometry: seeded initial generators, quadrature rules and the composite node
table the quadrature kernel consumes.

Mirrors `scvtmesh/geometry.py` (reference file:line cited per function).  Nothing here is on
the per-iteration path: point generation runs once (host NumPy for PCG64 stream parity,
SURVEY.md §8(a) a1) and the node table is built once per device context.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.special import roots_jacobi, roots_legendre

EPS_PROJ = 1e-9    # geometry.py:19
EPS_AREA = 1e-14   # geometry.py:20


def normalize(v):
    """Scale vectors in the last axis to unit length (geometry.py:23-26)."""
    v = np.asarray(v, dtype=float)
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def geodesic_distance(a, b):
    """atan2(|a x b|, a.b) great-circle distance (geometry.py:29-40)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return np.arctan2(np.linalg.norm(np.cross(a, b), axis=-1), np.sum(a * b, axis=-1))


def random_sphere_points(k: int, seed: int) -> np.ndarray:
    """K normalised N(0, I3) points from default_rng(seed) (geometry.py:225-229)."""
    rng = np.random.default_rng(seed)
    return normalize(rng.standard_normal((k, 3)))


def icosahedron_vertices() -> np.ndarray:
    """The 12 unit icosahedron vertices (geometry.py:211-222)."""
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    raw = np.array([[-1, 0, phi], [1, 0, phi], [-1, 0, -phi], [1, 0, -phi],
                    [0, phi, 1], [0, phi, -1], [0, -phi, 1], [0, -phi, -1],
                    [phi, 1, 0], [phi, -1, 0], [-phi, 1, 0], [-phi, -1, 0]], dtype=float)
    return normalize(raw)


def _conical_product_rule(n: int):
    """Duffy / conical-product rule with n^2 positive nodes (geometry.py:142-160)."""
    xj, wj = roots_jacobi(n, 1.0, 0.0)
    xl, wl = roots_legendre(n)
    xi = 0.5 * (xj + 1.0)
    eta = 0.5 * (xl + 1.0)
    lam1 = np.repeat(xi, n)
    lam2 = np.tile(eta, n) * (1.0 - lam1)
    lam0 = 1.0 - lam1 - lam2
    weights = np.repeat(wj / 4.0, n) * np.tile(wl / 2.0, n)
    return np.stack([lam0, lam1, lam2], axis=-1), weights / weights.sum()


def _radon_seven_point():
    """Radon's degree-5 symmetric 7-node rule (DECISIONS.md D1; the reference has none)."""
    s15 = np.sqrt(15.0)
    a1 = (6.0 - s15) / 21.0
    a2 = (6.0 + s15) / 21.0
    bary = np.array([
        [1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0],
        [1.0 - 2.0 * a1, a1, a1], [a1, 1.0 - 2.0 * a1, a1], [a1, a1, 1.0 - 2.0 * a1],
        [1.0 - 2.0 * a2, a2, a2], [a2, 1.0 - 2.0 * a2, a2], [a2, a2, 1.0 - 2.0 * a2],
    ])
    w = np.array([9.0 / 40.0] + [(155.0 - s15) / 1200.0] * 3 + [(155.0 + s15) / 1200.0] * 3)
    return bary, w / w.sum()


@dataclass(frozen=True)
class QuadratureRule:
    """Barycentric nodes and unit-sum weights (geometry.py:163-185)."""

    name: str
    bary: np.ndarray
    weights: np.ndarray

    @classmethod
    def four_point(cls) -> "QuadratureRule":
        return cls("4pt", *_conical_product_rule(2))

    @classmethod
    def nine_point(cls) -> "QuadratureRule":
        return cls("9pt", *_conical_product_rule(3))

    @classmethod
    def seven_point(cls) -> "QuadratureRule":
        return cls("7pt", *_radon_seven_point())


FOUR_POINT = QuadratureRule.four_point()
NINE_POINT = QuadratureRule.nine_point()
SEVEN_POINT = QuadratureRule.seven_point()

QUADRATURE_RULES = {"4pt": FOUR_POINT, "9pt": NINE_POINT, "7pt": SEVEN_POINT}


def subdivision_leaves(depth: int) -> np.ndarray:
    """Barycentric vertices (4**depth, 3, 3) of the leaves of `subdivide_fans`
    (delaunay.py:383-407) relative to the parent sub-triangle, vertex order preserved
    (children (v0,m01,m02), (m01,v1,m12), (m02,m12,v2), (m01,m12,m02)) so asymmetric rules
    land on exactly the reference's node positions."""
    leaves = np.eye(3)[None, :, :]
    for _ in range(depth):
        v0, v1, v2 = leaves[:, 0], leaves[:, 1], leaves[:, 2]
        m01, m12, m02 = 0.5 * (v0 + v1), 0.5 * (v1 + v2), 0.5 * (v0 + v2)
        leaves = np.concatenate([
            np.stack([v0, m01, m02], axis=1),
            np.stack([m01, v1, m12], axis=1),
            np.stack([m02, m12, v2], axis=1),
            np.stack([m01, m12, m02], axis=1),
        ])
    return leaves


def composite_nodes(rule: QuadratureRule, depth: int):
    """(l1, l2, w) of every quadrature node of the depth-d subdivided sub-triangle:
    x = v0 + l1 (v1 - v0) + l2 (v2 - v0), weight w = w_q / 4**depth (the leaf's signed
    area is the parent's / 4**depth, delaunay.py:406)."""
    if depth < 0 or depth > 6:
        raise ValueError("subdivision depth must be in [0, 6]")
    leaves = subdivision_leaves(depth)                     # (L, 3 vertices, 3 bary)
    nodes = np.einsum("qv,lvj->lqj", rule.bary, leaves)   # (L, Q, 3)
    w = np.broadcast_to(rule.weights / float(4 ** depth), nodes.shape[:2])
    nodes = nodes.reshape(-1, 3)
    return (np.ascontiguousarray(nodes[:, 1]), np.ascontiguousarray(nodes[:, 2]),
            np.ascontiguousarray(w.reshape(-1)))
