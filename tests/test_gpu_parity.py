"""GPU parity: the CUDA path (through the C ABI) against the golden fixtures of the live
reference and against the oracle on identical seeded inputs.

Tolerances (DECISIONS.md D7, the parity contract):
  * triangles: canonical int64 arrays equal (bit-exact), no flagged triangle;
  * m, c, E, lloyd_diag at identical Z: ||d||/||ref|| <= 1e-12;
  * grad: ||dg|| <= 1e-10 * ||2c_ref||;
  * trajectories: positions and energies within 1e-10 relative.
"""

import ctypes

import numpy as np
import pytest

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1709_06924_b200 as P  # noqa: E402

TOL_M = 1e-12
TOL_G = 1e-10


def _ev(density="const", rule="7pt", depth=3, measure="flat"):
    return P.MeshEvaluator(P.density_preset(density), rule, subdivision=depth, measure=measure)


def _check_moments(r, g, prefix, tol=TOL_M):
    assert rel(r.mass, g[prefix + "mass"]) <= tol
    assert rel(r.first, g[prefix + "first"]) <= tol
    assert abs(r.energy - g[prefix + "energy"]) <= tol * abs(g[prefix + "energy"])
    assert rel(r.lloyd_diag, g[prefix + "lloyd_diag"]) <= tol
    assert np.linalg.norm(r.grad - g[prefix + "grad"]) <= TOL_G * np.linalg.norm(2 * g[prefix + "first"])


# ------------------------------------------------------------------------- triangulation
@pytest.mark.parametrize("name", ["tet", "ico", "rnd50", "rnd162"])
def test_small_sets_triangles(gold, name):
    g = gold("small_sets")
    with _ev() as ev:
        t = ev.triangulation(g[name + "_z"])
    assert np.array_equal(t.triangles, g[name + "_triangles"])


def test_c1_triangles_bit_exact(gold):
    g = gold("c1_eval")
    with _ev() as ev:
        t = ev.triangulation(g["z"])
    assert np.array_equal(t.triangles, g["triangles"])
    assert int(t.flags.sum()) == 0
    np.testing.assert_allclose(t.circumcenters, g["circumcenters"], atol=1e-13)


@pytest.mark.parametrize("cfg,n", [("const", 40962), ("c4", 40962), ("c5", 40962),
                                   ("c3", 40962), ("c4", 163842), ("c5", 163842)])
def test_triangles_vs_qhull(cfg, n):
    if cfg == "const":
        z = O.random_sphere_points(n, 0)
    else:
        z = O.sample_by_density(O.density_for(cfg), n, 0)
    with _ev() as ev:
        t = ev.triangulation(z)
    ref = O.convex_hull_delaunay(z)
    assert t.triangles.shape == ref.shape
    assert np.array_equal(t.triangles, ref)


def test_medium_triangle_digests(gold):
    import hashlib

    g = gold("medium")
    z = P.random_sphere_points(40962, 0)
    with _ev() as ev:
        t = ev.triangulation(z)
    assert hashlib.sha256(t.triangles.tobytes()).hexdigest() == str(g["u_tri_sha"])
    for cfg in ("c4", "c5"):
        zs = P.sample_by_density(P.density_preset(cfg), 40962, 0)
        with _ev() as ev:
            t = ev.triangulation(zs)
        assert hashlib.sha256(t.triangles.tobytes()).hexdigest() == str(g[f"{cfg}_tri_sha"])


@pytest.mark.parametrize("name", ["rnd5", "rnd6"])
def test_hemisphere_sets_raise(gold, name):
    """Points whose hull misses the origin: the reference returns non-Delaunay hull facets
    silently; a spherical Delaunay triangulation would need a cell > hemisphere -> raise."""
    g = gold("small_sets")
    with _ev() as ev, pytest.raises(P.InsufficientPointsError):
        ev.triangulation(g[name + "_z"])


def test_too_few_points():
    with _ev() as ev, pytest.raises(P.InsufficientPointsError):
        ev.evaluate(P.random_sphere_points(3, 0))


def test_duplicate_points_raise():
    z = P.random_sphere_points(200, 1)
    z[7] = z[3]
    with _ev() as ev, pytest.raises(P.InsufficientPointsError):
        ev.evaluate(z)


def _polyhedron(name):
    u = lambda a: np.asarray(a, float) / np.linalg.norm(np.asarray(a, float), axis=1, keepdims=True)
    if name == "tetra":
        return u([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]])
    if name == "octa":
        return np.vstack([np.eye(3), -np.eye(3)])
    if name == "cube":
        return u([[a, b, c] for a in (1, -1) for b in (1, -1) for c in (1, -1)])
    return P.icosahedron_vertices()


@pytest.mark.parametrize("name", ["tetra", "octa", "ico", "cube"])
def test_regular_polyhedra_vs_oracle(name):
    """Smallest inputs the reference accepts: the tetrahedron (N=4), octahedron, icosahedron,
    and the cube, whose faces are four cocircular points.  Delaunay is ambiguous there (Qhull
    splits each square by its own rule) but both splits share the face's circumcentre, so the
    triangle count and every moment still equal the oracle's (delaunay.py:181-202, 337-380)."""
    z = _polyhedron(name)
    o = O.Evaluator(O.density_for("const"), "7pt", 3).evaluate(z)
    with _ev("const", "7pt", 3) as ev:
        r = ev.evaluate(z)
        t = ev.triangulation(z).triangles
    ref = O.convex_hull_delaunay(z)
    assert len(t) == len(ref) == 2 * len(z) - 4
    if name != "cube":
        assert np.array_equal(t, ref)
    assert rel(r.mass, o.mass) <= TOL_M
    assert rel(r.first, o.first) <= TOL_M
    assert abs(r.energy - o.energy) <= TOL_M * o.energy
    assert rel(r.lloyd_diag, o.lloyd_diag) <= TOL_M


def _latlon(nlat, nlon, poles):
    th = (np.arange(nlat) + 0.5) / nlat * np.pi
    ph = np.arange(nlon) / nlon * 2 * np.pi
    t, f = np.meshgrid(th, ph, indexing="ij")
    z = np.stack([np.sin(t) * np.cos(f), np.sin(t) * np.sin(f), np.cos(t)], -1).reshape(-1, 3)
    return np.vstack([z, [[0.0, 0.0, 1.0], [0.0, 0.0, -1.0]]]) if poles else z


@pytest.mark.parametrize("nlat,nlon,poles", [(48, 24, True), (48, 24, False)])
def test_latlon_grid_cocircular_quads(nlat, nlon, poles):
    """A latitude-longitude grid: every quad between two rings is an isosceles trapezoid, so
    nlat x nlon four-point sets are exactly cocircular (and without the pole points each polar
    cap is one nlon-gon of cocircular points).  The cell builder and its certificate must
    terminate and give Qhull's triangle count with the oracle's moments; a short P-LBFGS run
    from it (the flip repair sees the same ties) follows the oracle's energies."""
    z = _latlon(nlat, nlon, poles)
    o = O.Evaluator(O.density_for("x3"), "7pt", 1).evaluate(z)
    with _ev("x3", "7pt", 1) as ev:
        r = ev.evaluate(z)
        assert len(ev.triangulation(z).triangles) == 2 * len(z) - 4
        res = P.minimize(z, "lloyd-plbfgs", ev,
                         P.StoppingCriteria(max_iterations=5, movement_tol=1e-300,
                                            grad_tol=1e-300, stall_tol=1e-300), corrections=7)
    assert rel(r.mass, o.mass) <= TOL_M
    assert rel(r.first, o.first) <= TOL_M
    assert abs(r.energy - o.energy) <= TOL_M * o.energy
    ref = O.minimize(z, "lloyd-plbfgs", O.Evaluator(O.density_for("x3"), "7pt", 1),
                     O.StoppingCriteria(5, 1e-300, 1e-300, 1e-300), corrections=7)
    e = np.array([x.energy for x in res.records])
    eo = np.array([x.energy for x in ref.records])
    assert len(e) == len(eo)
    assert np.max(np.abs(e - eo) / eo) <= 1e-10


def test_minimize_normalizes_initial_points():
    """minimize() projects its initial points onto the sphere first (optimizer.py:290), so
    scaled and float32 starts follow the oracle's trajectory from the same input."""
    z = P.random_sphere_points(10000, 5)
    crit = P.StoppingCriteria(max_iterations=3, movement_tol=1e-300, grad_tol=1e-300,
                              stall_tol=1e-300)
    for start in (3.0 * z, (0.5 * z).astype(np.float32)):
        with _ev("x3", "7pt", 1) as ev:
            res = P.minimize(start, "lloyd-plbfgs", ev, crit, corrections=7)
        ref = O.minimize(start, "lloyd-plbfgs", O.Evaluator(O.density_for("x3"), "7pt", 1),
                         O.StoppingCriteria(3, 1e-300, 1e-300, 1e-300), corrections=7)
        e = np.array([x.energy for x in res.records])
        eo = np.array([x.energy for x in ref.records])
        assert len(e) == len(eo) and np.max(np.abs(e - eo) / eo) <= 1e-10
        assert np.max(np.abs(np.linalg.norm(res.points, axis=1) - 1.0)) <= 1e-15


@pytest.mark.parametrize("sep", [1e-6, 1e-10, 1e-12])
def test_near_duplicate_generators(sep):
    """Two generators `sep` apart (exact duplicates raise, test_duplicate_points_raise): the
    sliver cell between them is still built, Qhull's triangles are reproduced bitwise and the
    moments match the oracle (tools/probe_edge.py)."""
    z = P.random_sphere_points(10000, 5)
    t = np.cross(z[3], [0.0, 0.0, 1.0])
    z[7] = z[3] + sep * t / np.linalg.norm(t)
    z[7] /= np.linalg.norm(z[7])
    o = O.Evaluator(O.density_for("const"), "7pt", 1).evaluate(z)
    with _ev("const", "7pt", 1) as ev:
        r = ev.evaluate(z)
        assert np.array_equal(ev.triangulation(z).triangles, O.convex_hull_delaunay(z))
    assert rel(r.mass, o.mass) <= TOL_M
    assert rel(r.first, o.first) <= TOL_M


def test_valence_above_cap_raises():
    """SCVT_MAX_DEGREE (32) caps the stored valence; a generator with more Delaunay neighbours
    (the pole of a 96-longitude grid) raises CapacityError instead of truncating its cell."""
    with _ev("x3", "7pt", 1) as ev, pytest.raises(P.CapacityError):
        ev.evaluate(_latlon(48, 96, True))


# ------------------------------------------------------------------------- moments
@pytest.mark.parametrize("rule,depth", [("4pt", 0), ("9pt", 0), ("7pt", 0), ("7pt", 1),
                                        ("4pt", 3), ("7pt", 3)])
def test_c1_moments(gold, rule, depth):
    g = gold("c1_eval")
    with _ev("const", rule, depth) as ev:
        r = ev.evaluate(g["z"])
    _check_moments(r, g, f"{rule}_d{depth}_")
    assert r.obtuse_count == int(g["obtuse_count"])


@pytest.mark.parametrize("cfg", ["x3", "x16", "x64", "c3", "c4", "c5"])
@pytest.mark.parametrize("rule,depth", [("4pt", 0), ("7pt", 3)])
def test_density_moments_uniform(gold, cfg, rule, depth):
    g = gold("density_eval")
    with _ev(cfg, rule, depth) as ev:
        r = ev.evaluate(g["uniform_z"])
    _check_moments(r, g, f"uniform_{cfg}_{rule}_d{depth}_")


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_density_moments_sampled(gold, cfg):
    g = gold("density_eval")
    with _ev(cfg, "7pt", 3) as ev:
        r = ev.evaluate(g[f"sampled_{cfg}_z"])
    _check_moments(r, g, f"sampled_{cfg}_7pt_d3_")


def test_sampled_c3_small_is_hemisphere_degenerate(gold):
    g = gold("density_eval")
    with _ev("c3", "7pt", 3) as ev, pytest.raises(P.InsufficientPointsError):
        ev.evaluate(g["sampled_c3_z"])


def test_evaluate_on_triangles_matches(gold):
    g = gold("c1_eval")
    with _ev("const", "7pt", 3) as ev:
        r = ev.evaluate_on_triangles(g["z"], g["triangles"])
    _check_moments(r, g, "7pt_d3_")


def test_sphere_measure_vs_oracle():
    z = P.random_sphere_points(2562, 3)
    o = O.Evaluator(O.density_for("x3"), "4pt", 1, measure="sphere").evaluate(z)
    with _ev("x3", "4pt", 1, measure="sphere") as ev:
        r = ev.evaluate(z)
    assert rel(r.mass, o.mass) <= TOL_M
    assert rel(r.first, o.first) <= TOL_M
    assert abs(r.energy - o.energy) <= TOL_M * o.energy


def test_medium_moments(gold):
    g = gold("medium")
    z = P.random_sphere_points(40962, 0)
    with _ev("const", "4pt", 0) as ev:
        r = ev.evaluate(z)
    assert rel(r.first, g["u_4pt_d0_first"]) <= TOL_M
    assert abs(r.energy - g["u_4pt_d0_energy"]) <= TOL_M * g["u_4pt_d0_energy"]


def test_determinism_bitwise():
    z = P.sample_by_density(P.density_preset("c4"), 40962, 0)
    with _ev("c4", "7pt", 3) as ev:
        a = ev.evaluate(z)
        b = ev.evaluate(z)
    assert a.energy == b.energy
    assert np.array_equal(a.grad, b.grad)


@pytest.mark.parametrize("density,n,iters", [("c4", 40962, 12), ("x64", 2562, 25)])
def test_staged_history_pair_is_bitwise_the_push(density, n, iters):
    """Line-search trials stage their LBFGS pair (scvt_evaluate_staged) and the push commits
    it from the evaluation's own readback: the run is bitwise the one that makes every pair
    with scvt_history_push, including iterations that zoom, reset or fall back to Lloyd."""
    import torch

    den = P.density_preset(density)
    z0 = P.random_sphere_points(n, 0) if density == "x64" else P.sample_by_density(den, n, 0)
    runs = []
    for stage in (True, False):
        with P.MeshEvaluator(den, "7pt" if density == "c4" else "4pt",
                             subdivision=3 if density == "c4" else 0) as ev:
            st = P.Minimizer(torch.from_numpy(z0).cuda(), "lloyd-plbfgs", ev, 5)
            st.ops.stage_pairs = stage
            recs = [st.step()[0] for _ in range(iters)]
            runs.append((st.z.cpu().numpy(), [(r.energy, r.grad_norm, r.step, r.fevals)
                                              for r in recs], st.resets))
    assert runs[0][1] == runs[1][1]
    assert runs[0][2] == runs[1][2]
    assert np.array_equal(runs[0][0], runs[1][0])


@pytest.mark.parametrize("env", [{"SCVT_TAIL_ROUNDS": "0"}, {"SCVT_TAIL_ROUNDS": "1"},
                                 {"SCVT_FLIP_CAP": "96"}, {"SCVT_TAIL_ENTER": "1000000"},
                                 {"SCVT_TAIL_ENTER": "0"}])
def test_flip_repair_give_up_and_overflow_paths(monkeypatch, env):
    """What the flip repair cannot finish -- candidates the cluster tail gives up on (round
    limit 0 / 1), candidates beyond the queue capacity -- becomes bad cells for the rebuild
    path, and every split between grid-wide rounds and the tail repairs the same cycles: the
    run is bitwise the default one (the certified triangulation is unique)."""
    import torch

    den = P.density_preset("c4")
    z0 = P.sample_by_density(den, 40962, 0)

    def run():
        with P.MeshEvaluator(den, "7pt", subdivision=3) as ev:
            st = P.Minimizer(torch.from_numpy(z0).cuda(), "lloyd-plbfgs", ev, 7)
            e = [st.step()[0].energy for _ in range(8)]
            tri, _, _ = ev.triangulate_device(st.z)
            return e, st.z.cpu().numpy(), tri.cpu().numpy()

    ref = run()
    for k, v in env.items():
        monkeypatch.setenv(k, v)          # read at context creation
    got = run()
    assert got[0] == ref[0]
    assert np.array_equal(got[1], ref[1])
    assert np.array_equal(got[2], ref[2])


# ------------------------------------------------------------------------- trajectories
def _run_traj(g, density, rule, depth, method, m, iters):
    snaps = {}
    keep = set(int(x) for x in g["snap_iters"])

    def cb(n, z, res):
        if n in keep:
            assert isinstance(z, np.ndarray)    # NumPy input -> NumPy callbacks (reference)
            snaps[n] = z.copy()

    crit = P.StoppingCriteria(max_iterations=iters, movement_tol=1e-300, grad_tol=1e-300,
                              stall_tol=1e-300)
    with _ev(density, rule, depth) as ev:
        res = P.minimize(g["z0"], method, ev, crit, corrections=m, callback=cb)
    return res, snaps


# `tight`: iterations checked at 1e-10.  Trajectories of steep densities amplify rounding
# (identical branch decisions and steps; error grows ~1.8x per iteration for x64, SURVEY.md
# §6.3), so beyond `tight` only the decisions (fevals, steps to 1e-6) and a loose energy
# bound are asserted (DECISIONS.md D7).
@pytest.mark.parametrize("fixture,density,rule,depth,method,m,iters,tight", [
    ("traj_c1_4pt", "const", "4pt", 0, "lloyd-plbfgs", 5, 100, 100),
    ("traj_c1", "const", "7pt", 3, "lloyd-plbfgs", 5, 100, 100),
    ("traj_c1_4pt_lbfgs", "const", "4pt", 0, "lbfgs", 7, 30, 30),
    ("traj_c1_4pt_lloyd", "const", "4pt", 0, "lloyd", 7, 30, 30),
    ("traj_x64_4pt", "x64", "4pt", 0, "lloyd-plbfgs", 7, 40, 15),
    ("traj_c4small_4pt", "c4", "4pt", 0, "lloyd-plbfgs", 7, 40, 40),
    ("traj_c4small", "c4", "7pt", 3, "lloyd-plbfgs", 7, 12, 12),
    ("traj_c5small_4pt", "c5", "4pt", 0, "lloyd-plbfgs", 10, 30, 30),
])
def test_trajectory(gold, fixture, density, rule, depth, method, m, iters, tight):
    g = gold(fixture)
    res, snaps = _run_traj(g, density, rule, depth, method, m, iters)
    e = np.array([r.energy for r in res.records])
    assert len(e) == len(g["energy"])
    de = np.abs(e - g["energy"]) / np.abs(g["energy"])
    assert np.max(de[:tight]) <= 1e-10
    assert np.max(de) <= 1e-5
    steps = np.array([r.step for r in res.records])
    fev = np.array([-1 if r.fevals is None else r.fevals for r in res.records])
    assert np.array_equal(fev, g["fevals"])
    np.testing.assert_allclose(steps, g["step"], rtol=1e-6, atol=0)
    for n, zz in snaps.items():
        if n <= tight:
            assert rel(zz, g[f"z_{n}"]) <= 1e-10, n
    if iters <= tight:
        assert rel(res.points, g["final_z"]) <= 1e-10
    assert res.reason == str(g["reason"])
    assert res.resets == int(g["resets"])


def test_first_iteration_is_lloyd_step():
    """SURVEY.md §4 KAT: empty history + Lloyd diagonal => first step is a Lloyd step."""
    z = P.random_sphere_points(2562, 0)
    with _ev("const", "7pt", 3) as ev:
        r0 = ev.evaluate(z)
        res = P.minimize(z, "lloyd-plbfgs", ev, P.StoppingCriteria(max_iterations=1,
                         movement_tol=1e-300, grad_tol=1e-300, stall_tol=1e-300), corrections=5)
    lloyd = r0.first / np.linalg.norm(r0.first, axis=1, keepdims=True)
    assert np.abs(res.points - lloyd).max() <= 1e-14
    assert res.records[0].step == 1.0 and res.records[0].fevals == 1


# ------------------------------------------------------------------------- full-size properties
@pytest.mark.slow
def test_c4_full_size_properties():
    """N=655,362 (BASELINE c4): certificate-checked closed triangulation, bit-exact vs Qhull,
    total mass = area of the inscribed polyhedron (rho=1 identity), energy decreases."""
    z = P.sample_by_density(P.density_preset("c4"), 655362, 0)
    with _ev("c4", "7pt", 3) as ev:
        t = ev.triangulation(z)
        assert t.count == 2 * len(z) - 4
        ref = O.convex_hull_delaunay(z)
        assert np.array_equal(t.triangles, ref)
        res = P.minimize(z, "lloyd-plbfgs", ev, P.StoppingCriteria(max_iterations=3,
                         movement_tol=1e-300, grad_tol=1e-300, stall_tol=1e-300), corrections=7)
    e = [r.energy for r in res.records]
    assert all(b < a for a, b in zip(e, e[1:]))
    with _ev("const", "7pt", 3) as ev1:
        r1 = ev1.evaluate(z)
    v = z[ref]
    area = 0.5 * np.linalg.norm(np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), axis=1).sum()
    assert abs(r1.mass.sum() - area) <= 1e-11 * area


@pytest.mark.parametrize("cfg", ["c3", "c4", "c5"])
def test_density_table_vs_closed_form(cfg):
    """rho^(1/4) table (density.tanh4_table) against per-node atan2/tanh on the GPU."""
    z = P.sample_by_density(P.density_preset(cfg), 40962, 0)
    with P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3) as a, \
            P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3, density_table=False) as b:
        ra, rb = a.evaluate(z), b.evaluate(z)
    assert rel(ra.mass, rb.mass) <= 1e-13
    assert rel(ra.first, rb.first) <= 1e-13
    assert abs(ra.energy - rb.energy) <= 1e-13 * rb.energy


# ------------------------------------------------------------------------- sharded path
@pytest.mark.parametrize("cfg,n,nshards", [("const", 2562, 2), ("c4", 40962, 3),
                                           ("c5", 40962, 8), ("c4", 163842, 4)])
def test_sharded_evaluation_is_bitwise_identical(cfg, n, nshards):
    """All shards run back to back on one GPU (exchange buffers filled slice by slice):
    the sharded path must reproduce scvt_evaluate bit for bit for any shard count."""
    from paper_1709_06924_b200.parallel import CudaShardBackend, emulate_shards

    z = (P.random_sphere_points(n, 0) if cfg == "const"
         else P.sample_by_density(P.density_preset(cfg), n, 0))
    zt = torch.from_numpy(z).cuda()
    with _ev(cfg, "7pt", 3) as ev:
        ref = ev.evaluate_device(zt)
        sh = emulate_shards(CudaShardBackend(ev), zt, nshards)
    assert sh.energy == ref.energy and sh.grad_norm == ref.grad_norm
    assert torch.equal(sh.grad, ref.grad) and torch.equal(sh.first, ref.first)
    assert torch.equal(sh.mass, ref.mass) and torch.equal(sh.lloyd_diag, ref.lloyd_diag)


def test_sharded_evaluator_trajectory_matches(gold):
    g = gold("traj_c4small_4pt")
    crit = P.StoppingCriteria(max_iterations=10, movement_tol=1e-300, grad_tol=1e-300,
                              stall_tol=1e-300)
    with _ev("c4", "4pt", 0) as ev:
        a = P.minimize(g["z0"], "lloyd-plbfgs", ev, crit, corrections=7)
    with P.ShardedMeshEvaluator(P.density_preset("c4"), "4pt") as sev:
        b = P.minimize(g["z0"], "lloyd-plbfgs", sev, crit, corrections=7)
    np.testing.assert_array_equal(a.points, b.points)
    assert [r.energy for r in a.records] == [r.energy for r in b.records]


def test_sharded_errors_raise_consistently():
    from paper_1709_06924_b200.parallel import CudaShardBackend, emulate_shards

    z = P.random_sphere_points(500, 3)
    z[17] = z[42]
    zt = torch.from_numpy(z).cuda()
    with _ev("const", "4pt", 0) as ev, pytest.raises(P.InsufficientPointsError):
        emulate_shards(CudaShardBackend(ev), zt, 2)


@pytest.mark.parametrize("cfg", ["const", "c4", "c5"])
def test_sym7_fast_path_matches_generic(cfg, monkeypatch):
    """Leaf-grid placement of the symmetric 7-point rule (subtri_moments_sym7) against the
    generic composite-table loop (SCVT_NO_SYM7=1 at context creation)."""
    z = (P.random_sphere_points(40962, 0) if cfg == "const"
         else P.sample_by_density(P.density_preset(cfg), 40962, 0))
    with _ev(cfg, "7pt", 3) as a:
        ra = a.evaluate(z)
    monkeypatch.setenv("SCVT_NO_SYM7", "1")
    with _ev(cfg, "7pt", 3) as b:
        rb = b.evaluate(z)
    assert rel(ra.mass, rb.mass) <= 1e-13
    assert rel(ra.first, rb.first) <= 1e-13
    assert abs(ra.energy - rb.energy) <= 1e-13 * rb.energy


def test_cycle_reuse_matches_fresh_build(monkeypatch):
    """Certified reuse of the previous cycles (plus local rebuilds) gives exactly the fresh
    triangulation along an optimizer trajectory with heavy early churn."""
    z0 = P.sample_by_density(P.density_preset("c4"), 40962, 0)
    with _ev("c4", "4pt", 0) as ev, _ev("c4", "4pt", 0) as fresh:
        st = P.Minimizer(torch.from_numpy(z0).cuda(), "lloyd-plbfgs", ev, 7)
        for _ in range(6):
            st.step()
            t_reuse = ev.triangulation(st.z).triangles          # reuse path (same n as before)
            monkeypatch.setenv("SCVT_NO_REUSE", "1")
            t_fresh = fresh.triangulation(st.z).triangles
            monkeypatch.delenv("SCVT_NO_REUSE")
            assert np.array_equal(t_reuse, t_fresh)
            assert np.array_equal(t_fresh, O.convex_hull_delaunay(st.z.cpu().numpy()))


def _reuse_counters(ev):
    c = (ctypes.c_int64 * 12)()
    ev.context.lib.scvt_profile_counters(ev.context.ptr, c, 0)
    f = (ctypes.c_int64 * 4)()
    ev.context.lib.scvt_profile_flips(ev.context.ptr, f, 0)
    return {"reused_evals": c[8], "rebuilt": c[9], "passes": c[10], "flips": f[2]}


@pytest.mark.parametrize("nshards", [2, 3, 8])
def test_sharded_cycle_reuse_is_bitwise_identical(nshards):
    """Sharded reuse (scvt_shard_recheck/plan/rebuild/install, shards emulated back to back
    with the bad flags max-reduced and the rebuilt rows gathered slice by slice) along an
    optimizer trajectory: every evaluation bitwise equal to single-GPU scvt_evaluate, and
    the reuse path actually taken (certified evaluations, replicated flip repair, local
    rebuilds)."""
    from paper_1709_06924_b200.parallel import ShardedMeshEvaluator, CudaShardBackend, emulate_shards

    z0 = P.sample_by_density(P.density_preset("c4"), 40962, 0)
    with _ev("c4", "7pt", 3) as ev, _ev("c4", "7pt", 3) as one:
        be = CudaShardBackend(ev)
        st = P.Minimizer(torch.from_numpy(z0).cuda(), "lloyd-plbfgs", one, 7)
        emulate_shards(be, st.z, nshards)                  # full path: holds the cycles
        for _ in range(4):
            st.step()
            sh = emulate_shards(be, st.z, nshards)
            ref = one.evaluate_device(st.z)
            assert sh.energy == ref.energy and sh.grad_norm == ref.grad_norm
            assert torch.equal(sh.grad, ref.grad) and torch.equal(sh.first, ref.first)
            assert torch.equal(sh.lloyd_diag, ref.lloyd_diag)
        cnt = _reuse_counters(ev)
    assert cnt["reused_evals"] == 4 and cnt["rebuilt"] + cnt["flips"] > 0


def test_sharded_trajectory_matches_single_gpu():
    """A whole P-LBFGS run through ShardedMeshEvaluator (world size 1: the sharded code path
    with reuse) is bitwise the single-GPU run."""
    from paper_1709_06924_b200.parallel import ShardedMeshEvaluator

    z0 = P.sample_by_density(P.density_preset("c3"), 10242 * 4, 0)
    crit = P.StoppingCriteria(max_iterations=12)
    with _ev("c3", "7pt", 3) as a, \
            ShardedMeshEvaluator(P.density_preset("c3"), "7pt", subdivision=3) as b:
        ra = P.minimize(z0, "lloyd-plbfgs", a, crit, corrections=7)
        rb = P.minimize(z0, "lloyd-plbfgs", b, crit, corrections=7)
    assert np.array_equal(np.asarray(ra.points), np.asarray(rb.points))
    assert [h.energy for h in ra.records] == [h.energy for h in rb.records]
    assert ra.fevals == rb.fevals and ra.reason == rb.reason


def _oracle_cells(z, tri, density_name, rule, depth, gens):
    """Oracle moments of the cells of `gens` only (reference fans restricted to those cells)."""
    dens = O.density_for(density_name)
    keep = np.isin(tri, gens).any(axis=1)
    t = tri[keep]
    f = O.build_fans(z, t)
    sel = np.isin(f.cells, gens)
    f = O.Fans(f.verts[sel], f.cells[sel], f.edge_other[sel], f.signed_area[sel], 0)
    mass = np.zeros(len(z))
    first = np.zeros((len(z), 3))
    ecell = np.zeros(len(z))
    for s in range(0, len(f.cells), 8192):
        sub = O.subdivide(O.Fans(f.verts[s:s + 8192], f.cells[s:s + 8192],
                                 f.edge_other[s:s + 8192], f.signed_area[s:s + 8192], 0), depth)
        m, c, _, e = O.cell_quadrature(z, sub, dens, O.RULES[rule], len(z), cell_energy=True)
        mass += m
        first += c
        ecell += e
    return mass[gens], first[gens], ecell[gens]


@pytest.mark.slow
@pytest.mark.parametrize("cfg,n", [("const", 40962), ("c3", 163842), ("c4", 655362),
                                   ("c5", 2621442)])
def test_full_size_sampled_cell_parity(cfg, n):
    """BASELINE sizes: GPU moments AND per-cell energies of 1500 random cells against the
    oracle's (Qhull hull + reference fans + depth-3 subdivision + 7-pt rule), per generator at
    1e-12 (c2 = const density at N=40,962 on its own uniform generators)."""
    if cfg == "const":
        z = P.random_sphere_points(n, 0)
    else:
        z = P.sample_by_density(P.density_preset(cfg), n, 0)
    tri = O.convex_hull_delaunay(z)
    gens = np.sort(np.random.default_rng(5).choice(n, 1500, replace=False))
    om, oc, oe = _oracle_cells(z, tri, cfg, "7pt", 3, gens)
    with _ev(cfg, "7pt", 3) as ev:
        r = ev.evaluate(z)
        ecell = ev.cell_energy(n).cpu().numpy()
        t = ev.triangulation(z)
    assert np.array_equal(t.triangles, tri)
    assert np.max(np.abs(r.mass[gens] - om) / np.abs(om)) <= 1e-12
    assert np.max(np.linalg.norm(r.first[gens] - oc, axis=1) / np.linalg.norm(oc, axis=1)) <= 1e-12
    # per-cell energies: the D7 norm-wise bound over the sample, and 1e-11 for the worst cell
    # (|y - z|^2 is a difference of nearly equal unit vectors: at c5 the cells are ~1e-3
    # across, so each node's rounding is ~1e-13 relative, and obtuse cells' signed
    # sub-triangle areas partly cancel)
    assert np.linalg.norm(ecell[gens] - oe) <= 1e-12 * np.linalg.norm(oe)
    assert np.max(np.abs(ecell[gens] - oe) / np.abs(oe)) <= 1e-11
    # the per-cell energies sum to the evaluation's energy (fixed-order reduction)
    assert abs(ecell.sum() - r.energy) <= 1e-13 * r.energy


@pytest.mark.slow
def test_c3_first_iterations_vs_oracle():
    """c3 (N=163,842, tanh^4 gamma=1/16, m=7): first 3 iterations against the oracle
    optimizer (4-pt rule to keep the CPU oracle fast)."""
    z = P.sample_by_density(P.density_preset("c3"), 163842, 0)
    crit = P.StoppingCriteria(max_iterations=3, movement_tol=1e-300, grad_tol=1e-300,
                              stall_tol=1e-300)
    ref = O.minimize(z, "lloyd-plbfgs", O.Evaluator(O.density_for("c3"), "4pt", 0),
                     O.StoppingCriteria(3, 1e-300, 1e-300, 1e-300), corrections=7)
    with _ev("c3", "4pt", 0) as ev:
        res = P.minimize(z, "lloyd-plbfgs", ev, crit, corrections=7)
    e = np.array([r.energy for r in res.records])
    eo = np.array([r.energy for r in ref.records])
    assert np.max(np.abs(e - eo) / eo) <= 1e-10
    assert [r.fevals for r in res.records] == [r.fevals for r in ref.records]
    assert rel(res.points, ref.points) <= 1e-10


def test_run_ladder_matches_reference(gold):
    """pipeline.run optimise-bisect ladder 162 -> 642 (x3, 4-pt) against the reference."""
    g = gold("run_ladder")
    plan = P.RunPlan(points=642, density_name="x3", method="lloyd-plbfgs", seed=1,
                     partitions=64, quadrature="4pt", ladder=[162, 642],
                     criteria=P.StoppingCriteria(max_iterations=25))
    res = P.run(plan)
    for li in range(2):
        e = np.array([r.energy for r in res.levels[li].result.records])
        assert np.max(np.abs(e - g[f"level{li}_energy"]) / g[f"level{li}_energy"]) <= 1e-10
        assert res.levels[li].result.reason == str(g[f"level{li}_reason"])
    assert rel(res.points, g["final_z"]) <= 1e-10
    assert np.array_equal(res.triangulation.triangles, g["triangles"])


def _unit(a):
    return a / np.linalg.norm(a, axis=1, keepdims=True)


@pytest.mark.slow
@pytest.mark.parametrize("case", ["cluster", "band", "icosahedral"])
def test_adversarial_triangulations_match_qhull(case):
    """Cell builder + certificate on inputs that stress it (tools/stress_cells.py): a dense
    cluster (256x the background density) inside a sparse background, a thin great-circle band
    (huge elongated cells), the exact icosahedral bisection lattice at N=163,842."""
    rng = np.random.default_rng(3)
    if case == "cluster":
        c = _unit(np.array([[0.3, -0.5, 0.8]]))
        t = rng.standard_normal((65536, 3)) * 0.05
        z = np.vstack([_unit(c + t - (t @ c.T) * c), P.random_sphere_points(200000, 1)])
    elif case == "band":
        b = rng.standard_normal((300000, 3))
        b[:, 2] *= 0.01
        z = _unit(b)
    else:
        z = P.icosahedron_vertices()
        with _ev("const", "4pt", 0) as ev:
            while len(z) < 163842:
                z = P.bisect(z, ev.triangulation(z))
    with _ev("const", "4pt", 0) as ev:
        t = ev.triangulation(z).triangles
    assert np.array_equal(t, O.convex_hull_delaunay(z))


def _two_rank_worker(rank, world, port, z0, out, method="lloyd-plbfgs"):
    import os

    import torch.distributed as dist
    from paper_1709_06924_b200.parallel import ShardedMeshEvaluator

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        crit = P.StoppingCriteria(max_iterations=6)
        with ShardedMeshEvaluator(P.density_preset("c4"), "7pt", subdivision=3) as ev:
            r = P.minimize(z0, method, ev, crit, corrections=7)
        out[rank] = {"points": r.points, "energies": [h.energy for h in r.records],
                     "fevals": r.fevals, "grad": r.final.grad, "diag": r.final.lloyd_diag}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,method", [(2, "lloyd-plbfgs"), (4, "lloyd-plbfgs"),
                                          (2, "lbfgs"), (2, "lloyd")])
def test_two_processes_sharded_run_matches_single_gpu(world, method):
    """Real ranks (separate processes and contexts, gloo collectives staged through host
    memory, all on cuda:0 — host-mediated exchanges, no kernel waits on another rank) run
    the sharded P-LBFGS path: cells sharded with cycle reuse, the optimizer's vectors in
    arithmetic layout (parallel.SliceOps: chunk partials summed over the ranks); bitwise equal
    to the single-GPU run."""
    import socket

    import torch.multiprocessing as mp

    z0 = P.sample_by_density(P.density_preset("c4"), 40962, 0)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = mp.Manager().dict()
    mp.spawn(_two_rank_worker, args=(world, port, z0, out, method), nprocs=world, join=True)
    with _ev("c4", "7pt", 3) as ev:
        ref = P.minimize(z0, method, ev, P.StoppingCriteria(max_iterations=6), corrections=7)
    for rank in range(world):
        assert np.array_equal(out[rank]["points"], ref.points)
        assert out[rank]["energies"] == [h.energy for h in ref.records]
        assert out[rank]["fevals"] == ref.fevals
        assert np.array_equal(out[rank]["grad"], ref.final.grad)
        assert np.array_equal(out[rank]["diag"], ref.final.lloyd_diag)


def _nccl_one_rank_worker(rank, port, z0, out):
    import os

    import torch
    import torch.distributed as dist
    from paper_1709_06924_b200.parallel import ShardedMeshEvaluator

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        crit = P.StoppingCriteria(max_iterations=6)
        with ShardedMeshEvaluator(P.density_preset("c4"), "7pt", subdivision=3,
                                  force_collectives=True) as ev:
            assert ev.collective
            r = P.minimize(z0, "lloyd-plbfgs", ev, crit, corrections=7)
            e = ev.evaluate(r.points)
        dist.barrier()
        out[0] = {"points": r.points, "energies": [h.energy for h in r.records],
                  "fevals": r.fevals, "grad": r.final.grad, "diag": r.final.lloyd_diag,
                  "e": e.energy}
    finally:
        dist.destroy_process_group()


def test_nccl_backend_one_rank_group_matches_single_gpu():
    """The NCCL branch of every collective (all_gather_into_tensor on the padded device
    buffers, all-reduce SUM / MAX of device tensors, the status all-gather) on a one-rank NCCL
    group — what a one-GPU box can run of the real backend: the sharded evaluation and the
    arithmetic-layout optimizer with `force_collectives`, bitwise equal to the single-GPU
    run."""
    import socket

    import torch.multiprocessing as mp

    z0 = P.sample_by_density(P.density_preset("c4"), 40962, 0)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = mp.Manager().dict()
    mp.spawn(_nccl_one_rank_worker, args=(port, z0, out), nprocs=1, join=True)
    with _ev("c4", "7pt", 3) as ev:
        ref = P.minimize(z0, "lloyd-plbfgs", ev, P.StoppingCriteria(max_iterations=6),
                         corrections=7)
        e = ev.evaluate(ref.points)
    assert np.array_equal(out[0]["points"], ref.points)
    assert out[0]["energies"] == [h.energy for h in ref.records]
    assert out[0]["fevals"] == ref.fevals
    assert np.array_equal(out[0]["grad"], ref.final.grad)
    assert np.array_equal(out[0]["diag"], ref.final.lloyd_diag)
    assert out[0]["e"] == e.energy


@pytest.mark.parametrize("sharded", [False, True])
def test_reuse_escalates_to_full_rebuild_under_large_moves(sharded):
    """Positions moved by about a cell spacing between evaluations (most certificates fail):
    the reuse loop must escalate to the full rebuild (more than 3n/4 bad, or the pass limit)
    and still return exactly the fresh triangulation and moments."""
    from paper_1709_06924_b200.parallel import CudaShardBackend, emulate_shards

    n = 40962
    z0 = P.sample_by_density(P.density_preset("c4"), n, 0)
    rng = np.random.default_rng(11)
    z1 = _unit(z0 + 0.01 * rng.standard_normal(z0.shape))
    with _ev("c4", "7pt", 3) as ev, _ev("c4", "7pt", 3) as fresh:
        if sharded:
            be = CudaShardBackend(ev)
            emulate_shards(be, torch.from_numpy(z0).cuda(), 3)
            r = emulate_shards(be, torch.from_numpy(z1).cuda(), 3)
        else:
            ev.evaluate(z0)
            r = ev.evaluate_device(torch.from_numpy(z1).cuda())
            assert np.array_equal(ev.triangulation(z1).triangles, O.convex_hull_delaunay(z1))
        ref = fresh.evaluate_device(torch.from_numpy(z1).cuda())
        cnt = _reuse_counters(ev)
    assert cnt["reused_evals"] == 0 and cnt["passes"] >= 1      # escalated, not certified
    assert r.energy == ref.energy and torch.equal(r.grad, ref.grad)
    assert torch.equal(r.first, ref.first) and torch.equal(r.mass, ref.mass)


def _golden_covering(g):
    from paper_1709_06924_b200.partition import Covering

    one = tuple(tuple(int(x) for x in g["one_idx"][g["one_ptr"][k]:g["one_ptr"][k + 1]])
                for k in range(len(g["centers"])))
    return Covering(centers=g["centers"], one_level=one, two_level=())


def test_covering_migration_resets_match_reference(gold):
    """Region mode: with the reference's covering, the device migration class
    of every accepted iterate, the out-of-range re-decompose + history resets and the whole
    trajectory (plateau-clustered points spreading under a constant density: 8 resets in 40
    iterations) match the reference's region path run."""
    g = gold("covering")
    cov = _golden_covering(g)
    crit = P.StoppingCriteria(max_iterations=40, movement_tol=1e-300, grad_tol=1e-300,
                              stall_tol=1e-300)
    mig = []
    with P.MeshEvaluator(P.density_preset("const"), "4pt", cov) as ev:
        res = P.minimize(g["z0"], "lloyd-plbfgs", ev, crit, corrections=7,
                         callback=lambda n, z, r: mig.append(r.migration))
    assert mig == [str(m) for m in g["migration"]]
    assert res.resets == int(g["resets"]) > 0
    assert ev.fallbacks == int(g["fallbacks"])        # every evaluation of this run falls back
    e = np.array([r.energy for r in res.records])
    assert np.max(np.abs(e - g["energy"]) / g["energy"]) <= 1e-10
    assert [r.fevals if r.fevals is not None else -1 for r in res.records] == g["fevals"].tolist()
    assert rel(res.points, g["final_z"]) <= 1e-10


@pytest.mark.parametrize("case", range(5))
def test_region_failures_match_reference_region_tasks(gold, case):
    """Region-path semantics (delaunay.py:252-292, pipeline.py:62-98):
    per covering cell, the reference's `_region_task` fails (CoverageError: the interior
    selection truncates an owned fan) for exactly the regions the GPU predicts from the global
    cycles, over uniform points and bootstrap coverings."""
    from paper_1709_06924_b200.partition import Covering

    g = gold("region_cover")
    c = f"case{case}_"
    one = tuple(tuple(int(x) for x in g[c + "one_idx"][g[c + "one_ptr"][k]:g[c + "one_ptr"][k + 1]])
                for k in range(len(g[c + "centers"])))
    cov = Covering(centers=g[c + "centers"], one_level=one, two_level=())
    z = P.random_sphere_points(int(g[c + "k"]), int(g[c + "seed"]))
    with P.MeshEvaluator(P.density_preset("const"), "4pt", cov) as ev:
        zt = torch.from_numpy(z).cuda()
        ev.evaluate_device(zt)
        pred = ev.region_failures(zt)
        assert ev.fallbacks == int(np.any(g[c + "fail"]))
    assert pred.tolist() == g[c + "fail"].tolist()


def test_bootstrap_partition_cvt_matches_reference(gold):
    """bootstrap_partition_cvt (partition.py:83-120) with its Lloyd steps on the GPU: same
    centres to rounding and the same one-level adjacency as the reference's."""
    from paper_1709_06924_b200.partition import bootstrap_partition_cvt

    g = gold("covering")
    ref = _golden_covering(g)
    cov = bootstrap_partition_cvt(64, seed=0, density=P.density_preset("const"))
    assert rel(cov.centers, ref.centers) <= 1e-12
    assert cov.one_level == ref.one_level


@pytest.mark.parametrize("cfg,n", [("c4", 40962), ("c5", 40962)])
def test_flip_repair_matches_rebuild(cfg, n, monkeypatch):
    """Lawson-flip repair of the reused cycles (SCVT_NO_FLIPS unset) against the rebuild-only
    reuse loop along a P-LBFGS trajectory: bitwise the same iterates and results (the certified
    Delaunay triangulation is unique and stored canonically), with flips actually applied."""
    z0 = P.sample_by_density(P.density_preset(cfg), n, 0)
    crit = P.StoppingCriteria(max_iterations=10, movement_tol=1e-300, grad_tol=1e-300,
                              stall_tol=1e-300)
    out = {}
    for flips in (True, False):
        if flips:
            monkeypatch.delenv("SCVT_NO_FLIPS", raising=False)
        else:
            monkeypatch.setenv("SCVT_NO_FLIPS", "1")
        with _ev(cfg, "7pt", 3) as ev:
            r = P.minimize(z0, "lloyd-plbfgs", ev, crit, corrections=7)
            fl = (ctypes.c_int64 * 4)()
            ev.context.lib.scvt_profile_flips(ev.context.ptr, fl, 1)
            tri = ev.triangulation(r.points).triangles
        out[flips] = (r, list(fl), tri)
    (ra, fa, ta), (rb, fb, tb) = out[True], out[False]
    assert fa[2] > 0 and fb[2] == 0
    assert np.array_equal(ra.points, rb.points)
    assert [h.energy for h in ra.records] == [h.energy for h in rb.records]
    assert np.array_equal(ra.final.grad, rb.final.grad)
    assert np.array_equal(ta, tb)
    assert np.array_equal(ta, O.convex_hull_delaunay(ra.points))


def _lap_dense_rows(lap):
    """{(i, j): a_ij} of a DeviceLaplacian's perturbed matrix (host)."""
    w, nb, dg, dp = (t.cpu().numpy() for t in (lap.wsym, lap.nbr, lap.deg, lap.dpert))
    out = {}
    for i in range(lap.n):
        out[(i, i)] = dp[i]
        for t in range(dg[i]):
            out[(i, int(nb[i, t]))] = -w[i, t]
    return out


@pytest.mark.parametrize("pert", ["m2", "a6"])
def test_laplacian_matrix_and_solve_match_reference(gold, pert):
    """Graph Laplacian (cvt_core.py:192-236) assembled on the device from the per-sub-triangle
    masses: every entry of the perturbed matrix against the reference's sparse matrix at 1e-12,
    and the CG solve against SuperLU's solution."""
    g = gold("laplacian")
    with P.MeshEvaluator(P.density_preset("x3"), "4pt", laplacian=pert) as ev:
        r = ev.evaluate_device(torch.from_numpy(g["z0"]).cuda())
        lap = r.laplacian
        got = _lap_dense_rows(lap)
        x = lap.solve(g[f"{pert}_rhs"])
    indptr, indices, data = g[f"{pert}_indptr"], g[f"{pert}_indices"], g[f"{pert}_data"]
    ref = {}
    for i in range(len(indptr) - 1):
        for k in range(indptr[i], indptr[i + 1]):
            ref[(i, int(indices[k]))] = data[k]
    assert set(got) == set(ref)
    scale = max(abs(v) for v in ref.values())
    assert max(abs(got[k] - ref[k]) for k in ref) <= 1e-12 * scale
    assert rel(x, g[f"{pert}_x"]) <= 1e-10


@pytest.mark.parametrize("pert", ["m2", "a6"])
def test_laplacian_trajectory_matches_reference(gold, pert):
    """laplacian-m2 / laplacian-a6 LBFGS (two-loop around the Laplacian solve) for 20
    iterations against the reference (SuperLU) on the same seeded points: energies at 1e-10,
    identical line-search decisions, positions at 1e-10 (m2) / 1e-9 (a6: the 1e-6 shift leaves
    the matrix ~1e4-conditioned, so the two solvers' iterates drift apart by ~kappa eps per
    solve — 5e-10 after 20 iterations)."""
    g = gold("laplacian")
    crit = P.StoppingCriteria(max_iterations=20, movement_tol=1e-300, grad_tol=1e-300,
                              stall_tol=1e-300)
    with P.MeshEvaluator(P.density_preset("x3"), "4pt", laplacian=pert) as ev:
        res = P.minimize(g["z0"], f"laplacian-{pert}", ev, crit, corrections=7)
    e = np.array([h.energy for h in res.records])
    assert np.max(np.abs(e - g[f"{pert}_energy"]) / g[f"{pert}_energy"]) <= 1e-10
    assert [h.fevals for h in res.records] == g[f"{pert}_fevals"].tolist()
    assert rel(res.points, g[f"{pert}_final_z"]) <= (1e-10 if pert == "m2" else 1e-9)


@pytest.mark.slow
def test_flip_repair_full_size_c4(monkeypatch):
    """BASELINE c4 size (N=655,362): five P-LBFGS iterations whose evaluations are certified by
    the flip repair of the reused cycles (tens of thousands of flips each); the final
    triangulation equals a fresh GPU build and Qhull's."""
    n = 655362
    z0 = P.sample_by_density(P.density_preset("c4"), n, 0)
    monkeypatch.delenv("SCVT_NO_FLIPS", raising=False)
    with _ev("c4", "7pt", 3) as ev, _ev("c4", "7pt", 3) as fresh:
        st = P.Minimizer(torch.from_numpy(z0).cuda(), "lloyd-plbfgs", ev, 7)
        for _ in range(5):
            st.step()
        fl = (ctypes.c_int64 * 4)()
        ev.context.lib.scvt_profile_flips(ev.context.ptr, fl, 0)
        t_reuse = ev.triangulation(st.z).triangles
        monkeypatch.setenv("SCVT_NO_REUSE", "1")
        t_fresh = fresh.triangulation(st.z).triangles
    assert fl[2] > 10000
    assert np.array_equal(t_reuse, t_fresh)
    assert np.array_equal(t_fresh, O.convex_hull_delaunay(st.z.cpu().numpy()))


def test_bench_multi_rank_functional():
    """The multi-rank bench path under torchrun (two ranks on this one GPU with gloo,
    SCVT_BENCH_FUNCTIONAL=1): one JSON line from rank 0 with the contract keys; the numbers of
    such a run mean nothing, the code path is what is checked."""
    import json
    import os
    import socket
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, SCVT_BENCH_FUNCTIONAL="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                          str(port), "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
                          "--config", "c2", "--no-cpu-baseline"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["roofline"]["avg_launch_ms"] > 0


def _exact_local_delaunay_violations(z, tri):
    """Brute-force certificate in exact rational arithmetic (delaunay.py:117-130, 305-313
    without the floating-point margin): for every interior edge (a, b) with opposite vertices
    c (in triangle a, b, c) and d, the sign of det[b-a, c-a, d-a] must not say "d inside the
    circumcircle of (a, b, c)" (ties, D = 0, are allowed: any triangulation of a cocircular
    quad is Delaunay).  Returns the number of violating edges."""
    from fractions import Fraction as F

    zf = [[F(float(v)) for v in p] for p in z]
    opp = {}
    for t in tri:
        for k in range(3):
            a, b, c = int(t[k]), int(t[(k + 1) % 3]), int(t[(k + 2) % 3])
            opp[(a, b)] = c
    bad = 0
    for (a, b), c in opp.items():
        d = opp.get((b, a))
        if d is None or a > b:
            continue
        pa, pb, pc, pd = zf[a], zf[b], zf[c], zf[d]
        u = [pb[k] - pa[k] for k in range(3)]
        v = [pc[k] - pa[k] for k in range(3)]
        w = [pd[k] - pa[k] for k in range(3)]
        det = (u[0] * (v[1] * w[2] - v[2] * w[1]) + u[1] * (v[2] * w[0] - v[0] * w[2])
               + u[2] * (v[0] * w[1] - v[1] * w[0]))
        bad += det > 0
    return bad


@pytest.mark.parametrize("scale", [0.0, 1.0, 2.0 ** -20, 2.0 ** -40])
def test_near_cocircular_grid_exact_delaunay(scale):
    """Lat-lon grids whose trapezoid quads are cocircular exactly (scale 0) or up to relative
    margins of ~1e-16 ... 1e-28 (every z coordinate moved by scale x a few ulp): the GPU
    triangulation must be exactly (SoS-)Delaunay, certified in rational arithmetic, with the
    Euler counts of a closed triangulation."""
    rng = np.random.default_rng(int(scale * 1e6) + 1)
    z = _latlon(24, 20, False)
    if scale:
        dz = rng.integers(-3, 4, len(z)) * np.spacing(np.abs(z[:, 2])) * scale
        z = z.copy()
        z[:, 2] = z[:, 2] + dz
    with _ev("const", "4pt", 0) as ev:
        t = ev.triangulation(z).triangles
    assert len(t) == 2 * len(z) - 4
    assert _exact_local_delaunay_violations(z, t) == 0
