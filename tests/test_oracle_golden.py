"""Pin the oracle (oracle/) to golden vectors produced by the LIVE reference
(tests/golden/make_golden.py).  CPU only; sized to run in about a minute."""

import hashlib

import numpy as np
import pytest

import oracle as O
from conftest import rel


def test_rules_match_reference(gold):
    g = gold("rules")
    for k in ("4pt", "9pt", "7pt"):
        np.testing.assert_array_equal(O.RULES[k].bary, g[f"{k}_bary"])
        np.testing.assert_array_equal(O.RULES[k].weights, g[f"{k}_weights"])


def test_c1_triangles_bitexact(gold):
    g = gold("c1_eval")
    z = O.random_sphere_points(2562, 0)
    np.testing.assert_array_equal(z, g["z"])
    np.testing.assert_array_equal(O.convex_hull_delaunay(z), g["triangles"])


@pytest.mark.parametrize("rule,depth", [("4pt", 0), ("9pt", 0), ("7pt", 0), ("7pt", 1)])
def test_c1_moments(gold, rule, depth):
    g = gold("c1_eval")
    r = O.Evaluator(O.density_for("const"), rule, depth).evaluate(g["z"])
    p = f"{rule}_d{depth}_"
    np.testing.assert_array_equal(r.first, g[p + "first"])
    np.testing.assert_array_equal(r.mass, g[p + "mass"])
    assert r.energy == g[p + "energy"]
    np.testing.assert_array_equal(r.grad, g[p + "grad"])


def test_c1_moments_subdiv3(gold):
    g = gold("c1_eval")
    r = O.Evaluator(O.density_for("const"), "7pt", 3).evaluate(g["z"])
    assert rel(r.first, g["7pt_d3_first"]) <= 1e-15
    assert abs(r.energy - g["7pt_d3_energy"]) <= 1e-15 * g["7pt_d3_energy"]


@pytest.mark.parametrize("name", ["tet", "ico", "rnd5", "rnd6", "rnd50", "rnd162"])
def test_small_sets(gold, name):
    g = gold("small_sets")
    z = g[name + "_z"]
    np.testing.assert_array_equal(O.convex_hull_delaunay(z), g[name + "_triangles"])
    r = O.Evaluator(O.density_for("const"), "4pt", 0).evaluate(z)
    np.testing.assert_array_equal(r.first, g[name + "_4pt_d0_first"])


@pytest.mark.parametrize("cfg", ["x3", "x16", "x64", "c3", "c4", "c5"])
def test_density_moments_4pt(gold, cfg):
    g = gold("density_eval")
    r = O.Evaluator(O.density_for(cfg), "4pt", 0).evaluate(g["uniform_z"])
    p = f"uniform_{cfg}_4pt_d0_"
    assert rel(r.first, g[p + "first"]) <= 1e-15
    assert rel(r.mass, g[p + "mass"]) <= 1e-15
    assert abs(r.energy - g[p + "energy"]) <= 1e-15 * abs(g[p + "energy"])


@pytest.mark.parametrize("cfg", ["c3", "c4", "c5"])
def test_sampled_sets(gold, cfg):
    g = gold("density_eval")
    f = O.density_for(cfg)
    z = O.sample_by_density(f, 2562, 0)
    np.testing.assert_array_equal(z, g[f"sampled_{cfg}_z"])
    assert f.max_value == float(g[f"sampled_{cfg}_rho_max"])
    np.testing.assert_array_equal(O.eval_density(f, z), g[f"sampled_{cfg}_rho"])
    np.testing.assert_array_equal(O.convex_hull_delaunay(z), g[f"sampled_{cfg}_triangles"])


def test_sampled_c4_subdiv3_moments(gold):
    g = gold("density_eval")
    r = O.Evaluator(O.density_for("c4"), "7pt", 3).evaluate(g["sampled_c4_z"])
    p = "sampled_c4_7pt_d3_"
    assert rel(r.first, g[p + "first"]) <= 1e-14
    assert abs(r.energy - g[p + "energy"]) <= 1e-14 * abs(g[p + "energy"])


@pytest.mark.parametrize("cfg,n", [("c3", 163842), ("c4", 655362)])
def test_sampler_stream_parity(gold, cfg, n):
    g = gold("sampler")
    z = O.sample_by_density(O.density_for(cfg), n, 0)
    np.testing.assert_array_equal(z[:64], g[f"{cfg}_head"])
    np.testing.assert_array_equal(z[-64:], g[f"{cfg}_tail"])
    assert hashlib.sha256(z.tobytes()).hexdigest() == str(g[f"{cfg}_sha"])


def test_medium_digests(gold):
    g = gold("medium")
    z = O.random_sphere_points(40962, 0)
    t = O.convex_hull_delaunay(z)
    assert hashlib.sha256(t.tobytes()).hexdigest() == str(g["u_tri_sha"])
    r = O.Evaluator(O.density_for("const"), "4pt", 0).evaluate(z)
    assert rel(r.first, g["u_4pt_d0_first"]) <= 1e-15


def _traj(g, density, rule, depth, method, m, iters):
    crit = O.StoppingCriteria(max_iterations=iters, movement_tol=1e-300, grad_tol=1e-300,
                              stall_tol=1e-300)
    return O.minimize(g["z0"], method, O.Evaluator(O.density_for(density), rule, depth), crit,
                      corrections=m)


@pytest.mark.parametrize("fixture,density,method,m,iters", [
    ("traj_c1_4pt", "const", "lloyd-plbfgs", 5, 100),
    ("traj_c1_4pt_lbfgs", "const", "lbfgs", 7, 30),
    ("traj_c1_4pt_lloyd", "const", "lloyd", 7, 30),
    ("traj_x64_4pt", "x64", "lloyd-plbfgs", 7, 40),
    ("traj_c4small_4pt", "c4", "lloyd-plbfgs", 7, 40),
    ("traj_c3small_4pt", "c3", "lloyd-plbfgs", 7, 40),
    ("traj_c5small_4pt", "c5", "lloyd-plbfgs", 10, 30),
])
def test_trajectory_state_machine(gold, fixture, density, method, m, iters):
    """The oracle's optimizer reproduces the reference trajectory bit-for-bit, including the
    nonpositive-diagonal, line-search-failure and Lloyd-fallback branches."""
    g = gold(fixture)
    res = _traj(g, density, "4pt", 0, method, m, iters)
    np.testing.assert_array_equal([r.energy for r in res.records], g["energy"])
    np.testing.assert_array_equal([-1 if r.fevals is None else r.fevals for r in res.records],
                                  g["fevals"])
    np.testing.assert_array_equal(res.points, g["final_z"])
    assert res.resets == int(g["resets"])
    assert res.reason == str(g["reason"])


def test_trajectory_c1_subdiv3_first_iterations(gold):
    g = gold("traj_c1")
    res = _traj(g, "const", "7pt", 3, "lloyd-plbfgs", 5, 2)
    e = np.array([r.energy for r in res.records])
    assert np.max(np.abs(e - g["energy"][:2]) / g["energy"][:2]) <= 1e-14
    assert rel(res.points, g["z_2"]) <= 1e-14


def test_flop_model_matches_survey():
    """SURVEY.md §8(d) table values."""
    assert abs(O.algorithmic_flops(2562, 7, 3, "const") - 6.38e8) / 6.38e8 < 0.01
    assert abs(O.algorithmic_flops(655362, 7, 3, "tanh4") - 2.65e11) / 2.65e11 < 0.01
