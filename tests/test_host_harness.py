"""The cell builder and fan quadrature of csrc/scvt_device.cuh, compiled for the CPU by the
TEST-ONLY harness (tests/native/host_harness.cpp), against Qhull and the golden moments.

This exercises the exact device arithmetic (predicates, clipping, certificate, quadrature)
without a GPU; the GPU kernels (warp-cooperative builder, k_quad) are checked by
tests/test_gpu_parity.py on the B200."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from conftest import ROOT, rel

SRC = os.path.join(ROOT, "tests", "native", "host_harness.cpp")
SO = os.path.join(ROOT, "tests", "native", "libscvt_host_harness.so")
P = ctypes.POINTER
dp = lambda a: a.ctypes.data_as(P(ctypes.c_double))  # noqa: E731
ip = lambda a: a.ctypes.data_as(P(ctypes.c_int))  # noqa: E731


@pytest.fixture(scope="module")
def h():
    deps = [SRC, os.path.join(ROOT, "paper_1709_06924_b200", "csrc", "scvt_device.cuh")]
    if not os.path.exists(SO) or any(os.path.getmtime(d) > os.path.getmtime(SO) for d in deps):
        subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", SO, SRC], check=True)
    return ctypes.CDLL(SO)


def cells(h, z):
    z = np.ascontiguousarray(z, dtype=np.float64)
    n = len(z)
    nbr = np.zeros((n, 32), np.int32)
    deg = np.zeros(n, np.int32)
    st = np.zeros(4, np.int32)
    s = h.harness_cells(dp(z), n, ip(nbr), ip(deg), ip(st))
    return s, nbr, deg, st


def triangles(nbr, deg):
    out = []
    for i in range(len(deg)):
        r = nbr[i, :deg[i]]
        for t in range(len(r)):
            a, b = r[t], r[(t + 1) % len(r)]
            if i < a and i < b:
                out.append((i, a, b))
    t = np.array(out, np.int64)
    return t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))]


def consistent(nbr, deg):
    n = len(deg)
    for i in range(n):
        r = list(nbr[i, :deg[i]])
        for t in range(len(r)):
            a, b = r[t], r[(t + 1) % len(r)]
            ra = list(nbr[a, :deg[a]])
            if i not in ra or ra[ra.index(i) - 1] != b:
                return False
    return int(deg.sum()) == 6 * n - 12


@pytest.mark.parametrize("kind,n", [("uniform", 2562), ("uniform", 40962), ("c4", 2562),
                                    ("c4", 40962), ("c5", 40962), ("c3", 40962), ("c5", 10242)])
def test_cells_match_qhull(h, kind, n):
    z = O.random_sphere_points(n, 0) if kind == "uniform" else \
        O.sample_by_density(O.density_for(kind), n, 0)
    s, nbr, deg, st = cells(h, z)
    assert s == 0
    np.testing.assert_array_equal(triangles(nbr, deg), O.convex_hull_delaunay(z))


@pytest.mark.parametrize("name", ["tet", "ico", "rnd50", "rnd162"])
def test_small_sets(h, gold, name):
    g = gold("small_sets")
    s, nbr, deg, _ = cells(h, g[name + "_z"])
    assert s == 0
    np.testing.assert_array_equal(triangles(nbr, deg), g[name + "_triangles"])


def test_cocircular_cube_is_consistent(h):
    """Cube vertices: six exactly cocircular quads.  Symbolic perturbation must give one
    consistent triangulation (Qhull's choice may differ: flagged degeneracy)."""
    cube = O.normalize(np.array([[x, y, z] for x in (-1, 1) for y in (-1, 1) for z in (-1, 1)],
                                float))
    s, nbr, deg, st = cells(h, cube)
    assert s == 0 and consistent(nbr, deg)
    assert st[3] > 0   # tie-breaks were needed


def test_bisected_icosahedra(h):
    ico = O.icosahedron_vertices()
    z = ico
    for _ in range(3):
        e = O.triangle_edges(O.convex_hull_delaunay(z))
        z = np.vstack([z, O.normalize(z[e[:, 0]] + z[e[:, 1]])])
        s, nbr, deg, _ = cells(h, z)
        assert s == 0 and consistent(nbr, deg)
        np.testing.assert_array_equal(triangles(nbr, deg), O.convex_hull_delaunay(z))


@pytest.mark.parametrize("name", ["rnd5", "rnd6"])
def test_hemisphere_sets_detected(h, gold, name):
    """Hull misses the origin -> a Voronoi cell would span a hemisphere -> ST_UNBOUNDED."""
    s, _, _, _ = cells(h, gold("small_sets")[name + "_z"])
    assert s & 2


def test_duplicates_detected(h):
    z = O.random_sphere_points(300, 3)
    z[10] = z[20]
    s, _, _, _ = cells(h, z)
    assert s & 1


def test_insphere_predicate(h):
    o = np.array([1.0, 0, 0]); a = np.array([0, 1.0, 0]); b = np.array([0, 0, 1.0])
    am = ctypes.c_int(0)
    far = O.normalize(np.array([-1.0, -1.0, -1.0]))
    near = O.normalize(np.array([1.0, 1.0, 1.0]))
    assert h.harness_insphere(dp(o), dp(a), dp(b), dp(far), ctypes.byref(am)) == -1
    assert h.harness_insphere(dp(o), dp(a), dp(b), dp(near), ctypes.byref(am)) == 1
    assert am.value == 0


def _quad(h, z, nbr, deg, rule, depth, field, sphere=0):
    from paper_1709_06924_b200 import density as D, geometry as G

    l1, l2, w = G.composite_nodes(G.QUADRATURE_RULES[rule], depth)
    p = D.device_params(field)
    prm = np.zeros(15)
    prm[0:3] = [p["gamma"], p["beta"], p["alpha"]]
    prm[3:9] = p["center"]
    prm[9:11] = [p["w_lon"], p["w_lat"]]
    if field.variant == "x16":
        c = field.center
        lat, lon = np.arctan2(c[2], np.hypot(c[0], c[1])), np.arctan2(c[1], c[0])
        prm[11:15] = [lat, lon, np.cos(lat), np.sin(lat)]
    out = np.zeros((len(z), 5))
    ob = ctypes.c_int(0)
    h.harness_quad(dp(np.ascontiguousarray(z)), len(z), ip(nbr), ip(deg), dp(l1), dp(l2), dp(w),
                   len(w), p["density_kind"], dp(prm), sphere, dp(out), ctypes.byref(ob))
    return out, ob.value


@pytest.mark.parametrize("rule,depth", [("4pt", 0), ("9pt", 0), ("7pt", 1), ("7pt", 3)])
def test_quadrature_vs_golden(h, gold, rule, depth):
    from paper_1709_06924_b200 import density as D

    g = gold("c1_eval")
    z = g["z"]
    _, nbr, deg, _ = cells(h, z)
    out, ob = _quad(h, z, nbr, deg, rule, depth, D.density_preset("const"))
    p = f"{rule}_d{depth}_"
    assert rel(out[:, 0], g[p + "mass"]) <= 1e-13
    assert rel(out[:, 1:4], g[p + "first"]) <= 1e-13
    assert abs(out[:, 4].sum() - g[p + "energy"]) <= 1e-13 * g[p + "energy"]
    assert ob == int(g["obtuse_count"])


@pytest.mark.parametrize("cfg", ["x3", "x16", "x64", "c3", "c4", "c5"])
def test_density_kinds_vs_golden(h, gold, cfg):
    from paper_1709_06924_b200 import density as D

    g = gold("density_eval")
    z = g["uniform_z"]
    _, nbr, deg, _ = cells(h, z)
    out, _ = _quad(h, z, nbr, deg, "4pt", 0, D.density_preset(cfg))
    p = f"uniform_{cfg}_4pt_d0_"
    assert rel(out[:, 1:4], g[p + "first"]) <= 1e-13
    assert rel(out[:, 0], g[p + "mass"]) <= 1e-13


@pytest.mark.parametrize("cfg,which", [("const", "uniform"), ("c4", "uniform"), ("c5", "uniform"),
                                       ("c4", "sampled"), ("c5", "sampled")])
def test_sym7_fit_path_vs_golden(h, gold, cfg, which):
    """Leaf-grid 7-point placement + per-patch local fit of rho^(1/4) (the k_quad fast path)
    against the reference's 7pt/depth-3 moments."""
    from paper_1709_06924_b200 import density as D, geometry as G

    g = gold("c1_eval") if cfg == "const" else gold("density_eval")
    z = g["z"] if cfg == "const" else g[f"{which}_{cfg}_z" if which == "sampled" else "uniform_z"]
    pref = "7pt_d3_" if cfg == "const" else (f"sampled_{cfg}_7pt_d3_" if which == "sampled"
                                            else f"uniform_{cfg}_7pt_d3_")
    f = D.density_preset(cfg)
    _, nbr, deg, _ = cells(h, z)
    l1, l2, w = G.composite_nodes(G.QUADRATURE_RULES["7pt"], 3)
    p = D.device_params(f)
    prm = np.zeros(15)
    prm[0:3] = [p["gamma"], p["beta"], p["alpha"]]
    prm[3:9] = p["center"]
    if p["table"] is not None:
        co, wd = p["table"]
        co = np.ascontiguousarray(co)
        kind = 7 if f.variant == "tanh4x2" else 6
    else:
        co, wd, kind = np.zeros(1), 0.0, 0
    out = np.zeros((len(z), 5))
    h.harness_quad_sym7(dp(np.ascontiguousarray(z)), len(z), ip(nbr), ip(deg), dp(l1), dp(l2),
                        dp(w), dp(co), co.shape[1] if co.ndim == 3 else 0, ctypes.c_double(wd),
                        dp(prm), kind, dp(out))
    assert rel(out[:, 0], g[pref + "mass"]) <= 1e-13
    assert rel(out[:, 1:4], g[pref + "first"]) <= 1e-13
    assert abs(out[:, 4].sum() - g[pref + "energy"]) <= 1e-13 * g[pref + "energy"]


# ------------------------------------------------------------ exact predicate
def _frac_det(o, a, b, c):
    from fractions import Fraction as F

    o, a, b, c = ([F(float(v)) for v in p] for p in (o, a, b, c))
    u = [a[k] - o[k] for k in range(3)]
    v = [b[k] - o[k] for k in range(3)]
    w = [c[k] - o[k] for k in range(3)]
    return (u[0] * (v[1] * w[2] - v[2] * w[1]) + u[1] * (v[2] * w[0] - v[0] * w[2])
            + u[2] * (v[0] * w[1] - v[1] * w[0]))


def _frac_sign(x):
    return (x > 0) - (x < 0)


def _sos_truth(pts, idx):
    """Sign under the radial symbolic perturbation, in exact rationals: D, then the
    first-order terms of the points in increasing index order (origin: index < 0, fixed)."""
    from fractions import Fraction as F

    o, a, b, c = pts
    d = _frac_det(o, a, b, c)
    if d != 0:
        return _frac_sign(d), 1

    def det3(p, q, r):
        p, q, r = ([F(float(v)) for v in x] for x in (p, q, r))
        return (p[0] * (q[1] * r[2] - q[2] * r[1]) + p[1] * (q[2] * r[0] - q[0] * r[2])
                + p[2] * (q[0] * r[1] - q[1] * r[0]))

    t1, t2, t3, t4 = det3(a, b, c), det3(o, b, c), det3(a, o, c), det3(a, b, o)
    e = [-(t2 + t3 + t4), t1 - t3 - t4, t1 - t2 - t4, t1 - t2 - t3]
    for k in sorted((k for k in range(4) if idx[k] >= 0), key=lambda k: idx[k]):
        if e[k] != 0:
            return _frac_sign(e[k]), 2
    return 1, 2


def _orient(h, pts, idx, exact_only=False):
    tier = ctypes.c_int(-1)
    fn = h.harness_orient_exact if exact_only else h.harness_orient
    s = fn(*(dp(np.ascontiguousarray(p, dtype=float)) for p in pts), *idx, ctypes.byref(tier))
    return s, tier.value


def test_exact_orient_on_near_coplanar_quads(h):
    """Relative margins 1e-20 ... 1e-30 (a point lifted off the plane of three others by a few
    ulp of its coordinate, or less): the FP64 filter cannot decide; the exact tier must agree
    with rational arithmetic, sign for sign."""
    rng = np.random.default_rng(7)
    checked = 0
    for trial in range(400):
        zh = rng.uniform(-0.9, 0.9)
        r = np.sqrt(1 - zh * zh)
        ang = rng.uniform(0, 2 * np.pi, 4)
        pts = [np.array([r * np.cos(t), r * np.sin(t), zh]) for t in ang]
        k = rng.integers(0, 4)
        pts[k] = pts[k].copy()
        pts[k][2] = zh + rng.choice([-1, 1]) * rng.integers(0, 4) * np.spacing(zh) * 2.0 ** -rng.integers(0, 40)
        idx = [int(x) for x in rng.permutation(4)]
        truth, ttier = _sos_truth(pts, idx)
        s, tier = _orient(h, pts, idx)
        assert s == truth, (trial, pts, idx, s, truth)
        se, te = _orient(h, pts, idx, exact_only=True)
        assert se == truth and te == ttier
        checked += tier > 0
    assert checked > 300       # most cases reached the exact tiers


def test_sos_consistency_on_exactly_coplanar_quads(h):
    """Exact ties (four points on one circle of latitude: coplanar, D = 0 exactly): the
    symbolic perturbation decides, consistently with the rational first-order terms, and a
    quad seen from any rotation of its triangle gives the same answer."""
    rng = np.random.default_rng(11)
    for trial in range(200):
        zh = float(rng.choice([0.25, -0.5, 0.125, 0.75]))
        r = np.sqrt(1 - zh * zh)
        ang = np.sort(rng.uniform(0, 2 * np.pi, 4))
        pts = [np.array([r * np.cos(t), r * np.sin(t), zh]) for t in ang]
        assert _frac_det(*pts) == 0
        idx = [int(x) for x in rng.choice(1000, 4, replace=False)]
        truth, ttier = _sos_truth(pts, idx)
        s, tier = _orient(h, pts, idx)
        assert tier == 2 and s == truth and ttier == 2
        # cyclic relabelling of the triangle (o, a, b) -> (a, b, o) leaves D and the decision
        p2 = [pts[1], pts[2], pts[0], pts[3]]
        i2 = [idx[1], idx[2], idx[0], idx[3]]
        assert _orient(h, p2, i2)[0] == s


def test_orientation_against_the_origin_great_circle_tie(h):
    """o = the origin (index -1, never perturbed): three points on a great circle give
    D = 0 and every first-order term vanishes -> the documented +1."""
    pts = [np.zeros(3), np.array([1.0, 0, 0]), np.array([0, 1.0, 0]), np.array([-1.0, 0, 0])]
    s, tier = _orient(h, pts, [-1, 5, 6, 7])
    assert s == 1 and tier == 2


def test_fit_degree_classes_drop_only_noise_level_coefficients(h):
    """k_quad's per-patch fit degree (scvt_device.cuh local_fit_impl): a fit of class 2 (3)
    has had a6 (a5 and a6) set to exact zeros, which is allowed only when those Chebyshev
    coefficients are at the rounding floor of the table values (4e-15 relative); the classes
    must actually occur at a BASELINE-like patch size (the c4 density at N = 40,962: at full
    size 86 % of the sub-triangles are class 3), and the two-term 1/|x| series bound is the
    patch's 1 - |x|^2."""
    import paper_1709_06924_b200 as P
    from paper_1709_06924_b200 import density as D

    f = D.density_preset("c4")
    n = 40962
    z = np.ascontiguousarray(P.sample_by_density(f, n, 0))
    _, nbr, deg, _ = cells(h, z)
    p = D.device_params(f)
    prm = np.zeros(15)
    prm[0:3] = [p["gamma"], p["beta"], p["alpha"]]
    prm[3:9] = p["center"]
    co, wd = p["table"]
    co = np.ascontiguousarray(co)
    order = np.arange(n, dtype=np.int32)
    nsub = 2 * int(deg.sum())
    tail = np.zeros((nsub, 4))
    acc = np.zeros(nsub, np.int32)
    h.harness_fit_tails.restype = ctypes.c_longlong
    m = h.harness_fit_tails(dp(z), n, ip(order), ip(nbr), ip(deg), dp(co), co.shape[1],
                            ctypes.c_double(wd), dp(prm), 6, dp(tail), ip(acc))
    assert m == nsub
    assert set(np.unique(acc)) <= {0, 1, 2, 3}
    assert (acc > 0).mean() > 0.9                      # most patches are fitted
    assert (acc >= 2).mean() > 0.05                    # and the lower degrees do occur
    assert np.all(tail[acc >= 2, 0] <= 4e-15)          # |a6| at the noise floor
    assert np.all(tail[acc == 3, 1] <= 4e-15)          # |a5| + |a6| at the noise floor
    assert np.all(tail[acc == 1, 0] > 4e-15)           # full degree only where a6 matters
    assert np.all((tail[:, 3] > -1e-12) & (tail[:, 3] < 0.1))     # 1 - |x|^2 bound of the patch
