"""NumPy/SciPy restatement of the reference SCVT evaluation + Lloyd-P-LBFGS (TEST ORACLE).

See oracle/__init__.py for the rules that govern this module.  Each function cites the
reference (`/root/reference/pkg/src/scvtmesh/<file>.py:<line>`) it restates.  Additions the
BASELINE requires and the reference lacks (7-point rule, depth-d subdivision inside the
evaluator, tanh^4 and two-centre densities) follow DECISIONS.md and are injected into the
live reference identically by tests/golden/make_golden.py.
"""

from __future__ import annotations

import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np
from scipy.spatial import ConvexHull, QhullError
from scipy.special import roots_jacobi, roots_legendre

# ----------------------------------------------------------------------------- errors
# errors.py:4-65 (names only; the oracle raises them, tests compare types by name)


class ScvtError(Exception):
    pass


class InsufficientPointsError(ScvtError):
    pass


class DegenerateTriangleError(ScvtError):
    pass


class CentroidAtOriginError(ScvtError):
    pass


class NonpositiveDiagonalError(ScvtError):
    pass


class NonDescentError(ScvtError):
    pass


class LineSearchFailure(ScvtError):
    pass


class PoleAmbiguityError(ScvtError):
    pass


# ----------------------------------------------------------------------------- geometry
EPS_CENTROID = 1e-12          # cvt_core.py:33
EPS_CURVATURE = 1e-14         # optimizer.py:32
WOLFE_C1 = 1e-4               # optimizer.py:33
WOLFE_C2 = 0.9                # optimizer.py:34
MAX_LINE_SEARCH_EVALS = 10    # optimizer.py:35
POLE_EPS = 1e-9               # density.py:22


def normalize(v):
    """geometry.py:23-26."""
    v = np.asarray(v, dtype=float)
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def geodesic_distance(a, b):
    """geometry.py:29-40 (atan2 form)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return np.arctan2(np.linalg.norm(np.cross(a, b), axis=-1), np.sum(a * b, axis=-1))


def planar_circumcenter_3d(a, b, c):
    """geometry.py:105-119 — in-plane circumcentre (the Voronoi vertex the fans use)."""
    a = np.asarray(a, dtype=float)
    ab = np.asarray(b, dtype=float) - a
    ac = np.asarray(c, dtype=float) - a
    n = np.cross(ab, ac)
    n2 = np.sum(n * n, axis=-1, keepdims=True)
    ab2 = np.sum(ab * ab, axis=-1, keepdims=True)
    ac2 = np.sum(ac * ac, axis=-1, keepdims=True)
    return a + (ac2 * np.cross(n, ab) + ab2 * np.cross(ac, n)) / (2.0 * n2)


def random_sphere_points(k: int, seed: int) -> np.ndarray:
    """geometry.py:225-229."""
    rng = np.random.default_rng(seed)
    return normalize(rng.standard_normal((k, 3)))


def icosahedron_vertices() -> np.ndarray:
    """geometry.py:211-222."""
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    raw = np.array([[-1, 0, phi], [1, 0, phi], [-1, 0, -phi], [1, 0, -phi],
                    [0, phi, 1], [0, phi, -1], [0, -phi, 1], [0, -phi, -1],
                    [phi, 1, 0], [phi, -1, 0], [-phi, 1, 0], [-phi, -1, 0]], dtype=float)
    return normalize(raw)


# ----------------------------------------------------------------------------- rules
@dataclass(frozen=True)
class Rule:
    """geometry.py:163-185 (QuadratureRule): barycentric nodes, unit-sum weights."""

    name: str
    bary: np.ndarray
    weights: np.ndarray


def conical_product_rule(n: int):
    """geometry.py:142-160 — n^2-node Duffy rule, weights normalised to sum 1."""
    xj, wj = roots_jacobi(n, 1.0, 0.0)
    xl, wl = roots_legendre(n)
    xi = 0.5 * (xj + 1.0)
    eta = 0.5 * (xl + 1.0)
    wxi = wj / 4.0
    weta = wl / 2.0
    lam1 = np.repeat(xi, n)
    lam2 = np.tile(eta, n) * (1.0 - lam1)
    lam0 = 1.0 - lam1 - lam2
    bary = np.stack([lam0, lam1, lam2], axis=-1)
    weights = np.repeat(wxi, n) * np.tile(weta, n)
    return bary, weights / weights.sum()


def radon7() -> Rule:
    """DECISIONS.md D1: Radon's degree-5, 7-node, all-positive symmetric rule (not in the
    reference, geometry.py:142-185 has 4pt/9pt only); weights normalised to sum 1."""
    s15 = np.sqrt(15.0)
    a1 = (6.0 - s15) / 21.0
    a2 = (6.0 + s15) / 21.0
    bary = np.array([
        [1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0],
        [1.0 - 2.0 * a1, a1, a1], [a1, 1.0 - 2.0 * a1, a1], [a1, a1, 1.0 - 2.0 * a1],
        [1.0 - 2.0 * a2, a2, a2], [a2, 1.0 - 2.0 * a2, a2], [a2, a2, 1.0 - 2.0 * a2],
    ])
    w = np.array([9.0 / 40.0] + [(155.0 - s15) / 1200.0] * 3 + [(155.0 + s15) / 1200.0] * 3)
    return Rule("7pt", bary, w / w.sum())


RULES = {
    "4pt": Rule("4pt", *conical_product_rule(2)),
    "9pt": Rule("9pt", *conical_product_rule(3)),
    "7pt": radon7(),
}


# ----------------------------------------------------------------------------- density
@dataclass(frozen=True)
class Density:
    """density.py:25-51 plus the BASELINE variants 'tanh4' / 'tanh4x2' (DECISIONS.md D3/D4).

    For 'tanh4x2' ``center`` is a (2, 3) array and d = min over centres."""

    variant: str
    gamma: float = 1.0
    beta: float = 0.0
    alpha: float = 1.0
    center: np.ndarray | None = None
    w_lon: float | None = None
    w_lat: float | None = None

    @property
    def max_value(self) -> float:
        """density.py:42-51; tanh4 variants: value at d = 0."""
        if self.variant in ("const", "x3"):
            return 1.0
        if self.variant in ("tanh4", "tanh4x2"):
            g = self.gamma
            return float((((1.0 - g) / 2.0) * (np.tanh(self.beta / self.alpha) + 1.0) + g) ** 4)
        return float(1.0 / (2.0 * (1.0 - self.gamma)) * (np.tanh(self.beta / self.alpha) + 1.0)
                     + self.gamma)


def latlon_point(lat_deg: float, lon_deg: float) -> np.ndarray:
    la, lo = np.deg2rad(lat_deg), np.deg2rad(lon_deg)
    return normalize(np.array([np.cos(la) * np.cos(lo), np.cos(la) * np.sin(lo), np.sin(la)]))


def density_for(name: str) -> Density:
    """density.py:54-79 presets + the BASELINE configs."""
    name = name.lower()
    if name in ("const", "constant", "uniform"):
        return Density("const")
    if name == "x3":
        return Density("x3", gamma=(1.0 / 3.0) ** 4)
    if name == "x16":
        return Density("x16", gamma=(1.0 / 16.0) ** 4, beta=np.pi / 6.0, alpha=0.3,
                       center=np.array([1.0, 0.0, 0.0]), w_lon=0.3, w_lat=1.2)
    if name == "x64":
        return Density("x64", gamma=(1.0 / 64.0) ** 4, beta=np.pi / 6.0, alpha=0.15,
                       center=normalize(np.array([0.0, -0.866, 0.5])))
    if name == "c3":
        return Density("tanh4", gamma=1.0 / 16.0, beta=np.pi / 6.0, alpha=0.20,
                       center=latlon_point(30, -90))
    if name == "c4":
        return Density("tanh4", gamma=1.0 / 8.0, beta=np.pi / 6.0, alpha=0.20,
                       center=latlon_point(30, -90))
    if name == "c5":
        return Density("tanh4x2", gamma=1.0 / 16.0, beta=np.pi / 8.0, alpha=0.15,
                       center=np.stack([latlon_point(30, -90), latlon_point(-20, 150)]))
    raise ValueError(f"unknown density {name!r}")


def _latlon(x):
    """density.py:82-90."""
    x = np.asarray(x, dtype=float)
    horiz = np.hypot(x[..., 0], x[..., 1])
    if np.any(horiz < POLE_EPS):
        raise PoleAmbiguityError("longitude undefined within 1e-9 of a pole")
    return np.arctan2(x[..., 2], horiz), np.arctan2(x[..., 1], x[..., 0])


def _from_latlon(lat, lon):
    """density.py:93-97."""
    return np.stack([np.cos(lat) * np.cos(lon), np.cos(lat) * np.sin(lon), np.sin(lat)], axis=-1)


def elliptical_distance(x, f: Density):
    """density.py:100-113."""
    lat_x, lon_x = _latlon(x)
    lat_c, lon_c = _latlon(f.center)
    x = np.asarray(x, dtype=float)
    x_ic = _from_latlon(lat_x, np.broadcast_to(lon_c, lat_x.shape))
    x_ci = _from_latlon(np.broadcast_to(lat_c, lat_x.shape), lon_x)
    d_lon = geodesic_distance(x, x_ic)
    d_lat = geodesic_distance(x, x_ci)
    return np.sqrt((d_lon / f.w_lon) ** 2 + (d_lat / f.w_lat) ** 2)


def eval_density(f: Density, x):
    """density.py:116-129 (+ tanh4 / tanh4x2, DECISIONS.md D3/D4).  Renormalises first, as
    the reference does (density.py:118)."""
    x = normalize(x)
    if f.variant == "const":
        return np.ones(x.shape[:-1]) if x.ndim > 1 else 1.0
    if f.variant == "x3":
        return (1.0 - f.gamma) * x[..., 2] ** 4 + f.gamma
    if f.variant in ("tanh4", "tanh4x2"):
        cs = np.atleast_2d(f.center)
        d = geodesic_distance(x, cs[0])
        for c in cs[1:]:
            d = np.minimum(d, geodesic_distance(x, c))
        g = f.gamma
        return (((1.0 - g) / 2.0) * (np.tanh((f.beta - d) / f.alpha) + 1.0) + g) ** 4
    if f.w_lon is not None:
        d = elliptical_distance(x, f)
    else:
        d = geodesic_distance(x, f.center)
    return (np.tanh((f.beta - d) / f.alpha) + 1.0) / (2.0 * (1.0 - f.gamma)) + f.gamma


def sample_by_density(f: Density, k: int, seed: int) -> np.ndarray:
    """density.py:132-152 — rejection sampling on the default_rng(seed) PCG64 stream."""
    if k < 1:
        raise ValueError("k must be >= 1")
    rng = np.random.default_rng(seed)
    rho_max = f.max_value
    out = np.empty((k, 3))
    have = 0
    while have < k:
        batch = max(4 * (k - have), 1024)
        pts = normalize(rng.standard_normal((batch, 3)))
        keep = rng.random(batch) * rho_max < eval_density(f, pts)
        pts = pts[keep]
        take = min(k - have, len(pts))
        out[have:have + take] = pts[:take]
        have += take
    return out


# ----------------------------------------------------------------------------- Delaunay
def canonical(triangles):
    """delaunay.py:133-141 — rotate each triple so the smallest ID leads."""
    t = np.asarray(triangles, dtype=np.int64)
    lead = np.argmin(t, axis=1)
    out = np.empty_like(t)
    for r in range(3):
        rows = lead == r
        out[rows] = np.roll(t[rows], -r, axis=1)
    return out


def canonical_sort(triangles):
    """delaunay.py:144-147 — canonical rotation + lexicographic sort."""
    tris = canonical(triangles)
    order = np.lexsort((tris[:, 2], tris[:, 1], tris[:, 0]))
    return tris[order]


def ccw_outward(triangles, pts):
    """delaunay.py:172-178."""
    v = pts[triangles]
    det = np.einsum("ij,ij->i", v[:, 0], np.cross(v[:, 1], v[:, 2]))
    flip = det < 0
    triangles = triangles.copy()
    triangles[flip] = triangles[flip][:, [0, 2, 1]]
    return triangles


def convex_hull_delaunay(points) -> np.ndarray:
    """delaunay.py:181-202 — canonical (T,3) int64 triangles of the hull (Qhull via SciPy)."""
    pts = np.asarray(points, dtype=float)
    if len(pts) < 4:
        raise InsufficientPointsError(f"need >= 4 points on the sphere, got {len(pts)}")
    try:
        hull = ConvexHull(pts)
    except QhullError as exc:
        raise InsufficientPointsError(f"degenerate global point set: {exc}") from exc
    if len(hull.vertices) != len(pts):
        raise InsufficientPointsError(f"{len(pts) - len(hull.vertices)} points inside the hull")
    return canonical_sort(ccw_outward(hull.simplices.astype(np.int64), pts))


def empty_circumcircle_violations(points, triangles, margin=1e-12) -> int:
    """delaunay.py:305-313 (brute force; small K only) with circumcentres from 150-169."""
    pts = np.asarray(points, dtype=float)
    v = pts[triangles]
    n = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
    centers = n / np.linalg.norm(n, axis=1, keepdims=True)
    radii = geodesic_distance(centers, v[:, 0])
    d = np.arccos(np.clip(centers @ pts.T, -1.0, 1.0))
    inside = d < radii[:, None] - margin
    for kk in range(3):
        inside[np.arange(len(triangles)), triangles[:, kk]] = False
    return int(inside.sum())


def triangle_edges(triangles) -> np.ndarray:
    """delaunay.py:72-78 — unique undirected edges, sorted pairs, lexicographic."""
    e = np.concatenate([triangles[:, [0, 1]], triangles[:, [1, 2]], triangles[:, [2, 0]]])
    e.sort(axis=1)
    return np.unique(e, axis=0)


# ----------------------------------------------------------------------------- fans
@dataclass
class Fans:
    """delaunay.py:316-334 (VoronoiFans)."""

    verts: np.ndarray
    cells: np.ndarray
    edge_other: np.ndarray
    signed_area: np.ndarray
    obtuse_count: int


def build_fans(points, triangles) -> Fans:
    """delaunay.py:337-380 — 6 flat sub-triangles per Delaunay triangle."""
    pts = np.asarray(points, dtype=float)
    t = triangles
    va, vb, vc = pts[t[:, 0]], pts[t[:, 1]], pts[t[:, 2]]
    oc = planar_circumcenter_3d(va, vb, vc)
    mab = 0.5 * (va + vb)
    mbc = 0.5 * (vb + vc)
    mca = 0.5 * (vc + va)
    n = np.cross(vb - va, vc - va)
    n = n / np.linalg.norm(n, axis=1, keepdims=True)
    outward = np.einsum("ij,ij->i", n, va + vb + vc) < 0
    n[outward] = -n[outward]
    v0 = np.stack([va, mab, vb, mbc, vc, mca], axis=1)
    v1 = np.stack([mab, vb, mbc, vc, mca, va], axis=1)
    v2 = np.broadcast_to(oc[:, None, :], v0.shape)
    cells = np.stack([t[:, 0], t[:, 1], t[:, 1], t[:, 2], t[:, 2], t[:, 0]], axis=1)
    edge_other = np.stack([t[:, 1], t[:, 0], t[:, 2], t[:, 1], t[:, 0], t[:, 2]], axis=1)
    cross = np.cross(v1 - v0, v2 - v0)
    signed = 0.5 * np.einsum("tsj,tj->ts", cross, n)
    obtuse = int(np.any(signed < 0, axis=1).sum())
    verts = np.stack([v0, v1, v2], axis=2).reshape(-1, 3, 3)
    return Fans(verts, cells.reshape(-1), edge_other.reshape(-1), signed.reshape(-1), obtuse)


def subdivide(f: Fans, depth: int) -> Fans:
    """delaunay.py:383-407 — 4**depth in-plane children, area/4 per level."""
    verts, cells, edge_other, signed = f.verts, f.cells, f.edge_other, f.signed_area
    for _ in range(depth):
        v0, v1, v2 = verts[:, 0], verts[:, 1], verts[:, 2]
        m01, m12, m02 = 0.5 * (v0 + v1), 0.5 * (v1 + v2), 0.5 * (v0 + v2)
        verts = np.concatenate([
            np.stack([v0, m01, m02], axis=1),
            np.stack([m01, v1, m12], axis=1),
            np.stack([m02, m12, v2], axis=1),
            np.stack([m01, m12, m02], axis=1),
        ])
        cells = np.tile(cells, 4)
        edge_other = np.tile(edge_other, 4)
        signed = np.tile(signed / 4.0, 4)
    return Fans(verts, cells, edge_other, signed, f.obtuse_count)


def cell_quadrature(points, f: Fans, density: Density, rule: Rule, k: int, measure="flat",
                    cell_energy=False):
    """cvt_core.py:55-117 (with_pairs=False) — (mass (k,), first (k,3), energy); with
    ``cell_energy`` also the per-cell energies (k,) whose sum is the energy (test helper)."""
    pts = np.asarray(points, dtype=float)
    mass = np.zeros(k)
    first = np.zeros((k, 3))
    if len(f.cells) == 0:
        return (mass, first, 0.0, np.zeros(k)) if cell_energy else (mass, first, 0.0)
    nodes = np.einsum("qv,svj->sqj", rule.bary, f.verts)
    radii = np.linalg.norm(nodes, axis=-1)
    nodes = nodes / radii[..., None]
    rho = eval_density(density, nodes)
    if measure == "sphere":
        nvec = np.cross(f.verts[:, 1] - f.verts[:, 0], f.verts[:, 2] - f.verts[:, 0])
        nn = np.linalg.norm(nvec, axis=1)
        nn[nn == 0.0] = 1.0
        plane_d = np.abs(np.einsum("sj,sj->s", nvec / nn[:, None], f.verts[:, 0]))
        rho = rho * (plane_d[:, None] / radii ** 3)
    elif measure != "flat":
        raise ValueError(f"unknown integration measure {measure!r}")
    w = rule.weights
    sub_mass = (rho @ w) * f.signed_area
    sub_first = np.einsum("sq,q,sqj->sj", rho, w, nodes) * f.signed_area[:, None]
    z_cell = pts[f.cells]
    diff = nodes - z_cell[:, None, :]
    sq = np.einsum("sqj,sqj->sq", diff, diff)
    sub_energy = ((rho * sq) @ w) * f.signed_area
    energy = float(np.sum(sub_energy))
    np.add.at(mass, f.cells, sub_mass)
    np.add.at(first, f.cells, sub_first)
    if cell_energy:
        ecell = np.zeros(k)
        np.add.at(ecell, f.cells, sub_energy)
        return mass, first, energy, ecell
    return mass, first, energy


def moments(points, triangles, density: Density, rule: Rule, depth: int = 0,
            measure="flat", chunk: int = 16384, select=None):
    """Fans -> (chunked) subdivision -> quadrature (pipeline.py:206-215 global path with the
    depth-d subdivision of DECISIONS.md D2).  ``select`` optionally restricts the sub-
    triangles to a boolean mask over fan rows (bench sampling only)."""
    pts = np.asarray(points, dtype=float)
    k = len(pts)
    f = build_fans(pts, triangles)
    if select is not None:
        f = Fans(f.verts[select], f.cells[select], f.edge_other[select], f.signed_area[select],
                 f.obtuse_count)
    mass = np.zeros(k)
    first = np.zeros((k, 3))
    energy = 0.0
    S = len(f.cells)
    step = chunk if depth > 0 else max(S, 1)
    for s in range(0, S, step):
        e = min(S, s + step)
        sub = Fans(f.verts[s:e], f.cells[s:e], f.edge_other[s:e], f.signed_area[s:e],
                   f.obtuse_count)
        sub = subdivide(sub, depth)
        m, c, en = cell_quadrature(pts, sub, density, rule, k, measure)
        mass += m
        first += c
        energy += en
    return mass, first, energy, f.obtuse_count


@dataclass
class EvalResult:
    """optimizer.py:66-76 (+ mass and triangles for parity checks)."""

    energy: float
    grad: np.ndarray
    grad_norm: float
    lloyd_diag: np.ndarray
    first: np.ndarray
    mass: np.ndarray = None
    triangles: np.ndarray = None
    migration: str = "in-place"


class Evaluator:
    """pipeline.py:101-286 global path (covering=None)."""

    def __init__(self, density: Density, rule: Rule | str, depth: int = 0, measure="flat"):
        self.density = density
        self.rule = RULES[rule] if isinstance(rule, str) else rule
        self.depth = depth
        self.measure = measure
        self.evaluations = 0
        self.fallbacks = 0

    def evaluate(self, points) -> EvalResult:
        """pipeline.py:261-279."""
        points = np.asarray(points, dtype=float)
        tri = convex_hull_delaunay(points)
        mass, first, energy, _ = moments(points, tri, self.density, self.rule, self.depth,
                                         self.measure)
        self.evaluations += 1
        cz = np.einsum("ij,ij->i", first, points)
        grad = 2.0 * cz[:, None] * points - 2.0 * first
        return EvalResult(energy=energy, grad=grad, grad_norm=float(np.linalg.norm(grad)),
                          lloyd_diag=2.0 * cz, first=first, mass=mass, triangles=tri)

    def redecompose(self, points):
        return None


# ----------------------------------------------------------------------------- optimizer
@dataclass
class StoppingCriteria:
    """optimizer.py:40-53."""

    max_iterations: int = 2000
    movement_tol: float = 5e-4
    grad_tol: float = 5e-4
    stall_tol: float = 1e-7


@dataclass
class IterationRecord:
    """optimizer.py:56-63."""

    n: int
    energy: float
    grad_norm: float
    step: float
    fevals: int | None
    time_ms: float


class CorrectionHistory:
    """optimizer.py:79-114."""

    def __init__(self, m: int = 7):
        self.m = m
        self._pairs = deque(maxlen=m)
        self.skipped = 0

    def __len__(self):
        return len(self._pairs)

    def __iter__(self):
        return iter(self._pairs)

    def push(self, s, y) -> bool:
        ys = float(y @ s)
        if ys <= EPS_CURVATURE * np.linalg.norm(s) * np.linalg.norm(y):
            self.skipped += 1
            return False
        self._pairs.append((s, y, 1.0 / ys))
        return True

    def clear(self):
        self._pairs.clear()

    def gamma(self) -> float:
        if not self._pairs:
            return 1.0
        s, y, _ = self._pairs[-1]
        return float((y @ s) / (y @ y))


class GammaIdentity:
    """optimizer.py:117-124."""

    def __init__(self, gamma):
        self.gamma = gamma

    def apply(self, q):
        return self.gamma * q


class LloydDiagonal:
    """optimizer.py:127-134."""

    def __init__(self, inverse_diag):
        self.inverse_diag = inverse_diag

    def apply(self, q):
        return (q.reshape(-1, 3) * self.inverse_diag[:, None]).ravel()


def two_loop_direction(g, hist: CorrectionHistory, h0):
    """optimizer.py:147-167."""
    q = g.copy()
    alphas = []
    for s, y, rho in reversed(list(hist)):
        a = rho * (s @ q)
        alphas.append(a)
        q -= a * y
    q = h0.apply(q)
    for (s, y, rho), a in zip(hist, reversed(alphas)):
        b = rho * (y @ q)
        q += s * (a - b)
    q = -q
    if q @ g >= 0.0:
        raise NonDescentError(f"direction has q.g = {q @ g:.3e} >= 0")
    return q


def wolfe_line_search(phi, f0, dphi0, c1=WOLFE_C1, c2=WOLFE_C2,
                      max_evals=MAX_LINE_SEARCH_EVALS, initial_step=1.0):
    """optimizer.py:170-237 — strong-Wolfe bracketing + quadratic zoom."""
    if dphi0 >= 0.0:
        raise NonDescentError(f"line search needs a descent direction, dphi0={dphi0:.3e}")
    evals = 0
    best = None

    def record(alpha, f, payload):
        nonlocal best
        if f < f0 and (best is None or f < best[0]):
            best = (f, alpha, payload)

    def exhausted_result():
        if best is None:
            raise LineSearchFailure(f"no decrease within {max_evals} evaluations")
        f, alpha, payload = best
        return alpha, f, payload, evals, True

    def zoom(lo, f_lo, d_lo, hi, f_hi):
        nonlocal evals
        while evals < max_evals:
            span = hi - lo
            denom = 2.0 * (f_hi - f_lo - d_lo * span)
            alpha = lo - d_lo * span * span / denom if denom != 0.0 else lo + 0.5 * span
            low, high = (lo, hi) if lo < hi else (hi, lo)
            margin = 0.1 * abs(span)
            if not (low + margin <= alpha <= high - margin):
                alpha = lo + 0.5 * span
            f, d, payload = phi(alpha)
            evals += 1
            record(alpha, f, payload)
            if f > f0 + c1 * alpha * dphi0 or f >= f_lo:
                hi, f_hi = alpha, f
            else:
                if abs(d) <= -c2 * dphi0:
                    return alpha, f, payload, evals, False
                if d * span >= 0.0:
                    hi, f_hi = lo, f_lo
                lo, f_lo, d_lo = alpha, f, d
        return exhausted_result()

    alpha_prev, f_prev, d_prev = 0.0, f0, dphi0
    alpha = initial_step
    first = True
    while evals < max_evals:
        f, d, payload = phi(alpha)
        evals += 1
        record(alpha, f, payload)
        if f > f0 + c1 * alpha * dphi0 or (not first and f >= f_prev):
            return zoom(alpha_prev, f_prev, d_prev, alpha, f)
        if abs(d) <= -c2 * dphi0:
            return alpha, f, payload, evals, False
        if d >= 0.0:
            return zoom(alpha, f, d, alpha_prev, f_prev)
        alpha_prev, f_prev, d_prev = alpha, f, d
        alpha *= 2.0
        first = False
    return exhausted_result()


def lloyd_step(points, first_moments):
    """optimizer.py:240-246."""
    norms = np.linalg.norm(first_moments, axis=1)
    if np.any(norms <= 1e-12):
        raise CentroidAtOriginError("first moment ~0")
    return first_moments / norms[:, None]


@dataclass
class MinimizeResult:
    """optimizer.py:249-257."""

    points: np.ndarray
    records: list
    reason: str
    fevals: int
    resets: int
    wall_time: float
    final: EvalResult = field(repr=False, default=None)


def _initial_inverse(method, hist, res):
    """optimizer.py:260-275 (lbfgs / lloyd-plbfgs)."""
    if method == "lbfgs":
        return GammaIdentity(hist.gamma())
    d = res.lloyd_diag
    if np.any(d <= 0.0):
        return GammaIdentity(hist.gamma())
    return LloydDiagonal(1.0 / d)


def minimize(points, method, evaluator, criteria=None, corrections=7, callback=None):
    """optimizer.py:278-391 (methods lloyd / lbfgs / lloyd-plbfgs)."""
    if method not in ("lloyd", "lbfgs", "lloyd-plbfgs"):
        raise ValueError(method)
    criteria = criteria or StoppingCriteria()
    z = normalize(np.array(points, dtype=float))
    k = len(z)
    t0 = time.perf_counter()
    res = evaluator.evaluate(z)
    fevals_total = 1
    hist = CorrectionHistory(corrections)
    records = []
    resets = 0
    reason = "max-iterations"
    for n in range(1, criteria.max_iterations + 1):
        t_iter = time.perf_counter()
        f_prev = res.energy
        if method == "lloyd":
            z_new = lloyd_step(z, res.first)
            res_new = evaluator.evaluate(z_new)
            fevals_total += 1
            fevals_iter = None
            alpha = 1.0
        else:
            h0 = _initial_inverse(method, hist, res)
            g = res.grad.ravel()
            try:
                q = two_loop_direction(g, hist, h0)
            except NonDescentError:
                hist.clear()
                resets += 1
                try:
                    q = two_loop_direction(g, hist, h0)
                except NonDescentError:
                    q = -hist.gamma() * g
            q3 = q.reshape(k, 3)
            q3 = q3 - np.einsum("ij,ij->i", q3, z)[:, None] * z

            def phi(alpha, z=z, q3=q3):
                v = z + alpha * q3
                norms = np.linalg.norm(v, axis=1)
                zt = v / norms[:, None]
                r = evaluator.evaluate(zt)
                d = float(np.einsum("ij,ij->i", r.grad, q3 / norms[:, None]).sum())
                return r.energy, d, (zt, r)

            dphi0 = float(np.einsum("ij,ij->", res.grad, q3))
            try:
                alpha, _, payload, evals, _ = wolfe_line_search(phi, res.energy, dphi0)
                z_new, res_new = payload
                fevals_iter = evals
            except (NonDescentError, LineSearchFailure):
                hist.clear()
                resets += 1
                z_new = lloyd_step(z, res.first)
                res_new = evaluator.evaluate(z_new)
                fevals_iter = 1
                alpha = 0.0
            fevals_total += fevals_iter
            s = (z_new - z).ravel()
            y = (res_new.grad - res.grad).ravel()
            hist.push(s, y)
        movement = float(np.abs(z_new - z).max())
        records.append(IterationRecord(n, res_new.energy, res_new.grad_norm, alpha, fevals_iter,
                                       (time.perf_counter() - t_iter) * 1e3))
        if callback is not None:
            callback(n, z_new, res_new)
        z, res = z_new, res_new
        if movement <= criteria.movement_tol:
            reason = "movement"
            break
        if abs(res.energy - f_prev) / abs(f_prev) < criteria.stall_tol:
            reason = "energy-stall"
            break
        if res.grad_norm / res.energy <= criteria.grad_tol:
            reason = "gradient"
            break
    return MinimizeResult(z, records, reason, fevals_total, resets, time.perf_counter() - t0, res)


# ----------------------------------------------------------------------------- FLOP model
def algorithmic_flops(n: int, q: int, depth: int, variant: str) -> float:
    """F_eval = T*6*4^d*(Q*f_node + f_leaf) + T*f_tri + N*f_gen."""
    f_node = 44 + {"const": 0, "x3": 4, "x64": 27, "x16": 27, "tanh4": 29, "tanh4x2": 48}.get(
        variant, 29)
    t = 2 * n - 4
    return float(t * 6 * 4 ** depth * (q * f_node + 16) + t * 200 + n * 15)
