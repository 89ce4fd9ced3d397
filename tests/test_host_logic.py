"""Host-side logic of the package (no GPU): rules and composite node tables, density table,
sampling, scalar line search, stopping rules, ladders, config plumbing."""

import numpy as np
import pytest

import oracle as O
import paper_1709_06924_b200 as P
from paper_1709_06924_b200 import density as D
from paper_1709_06924_b200 import geometry as G
from paper_1709_06924_b200.optimizer import wolfe_line_search


def test_rules_equal_oracle():
    for k in ("4pt", "9pt", "7pt"):
        np.testing.assert_array_equal(G.QUADRATURE_RULES[k].bary, O.RULES[k].bary)
        np.testing.assert_array_equal(G.QUADRATURE_RULES[k].weights, O.RULES[k].weights)


@pytest.mark.parametrize("rule", ["4pt", "9pt", "7pt"])
@pytest.mark.parametrize("depth", [0, 1, 2, 3])
def test_composite_weights(rule, depth):
    l1, l2, w = G.composite_nodes(G.QUADRATURE_RULES[rule], depth)
    assert len(w) == 4 ** depth * len(G.QUADRATURE_RULES[rule].weights)
    assert abs(w.sum() - 1.0) < 1e-14
    assert np.all((l1 >= 0) & (l2 >= 0) & (l1 + l2 <= 1))


def test_composite_depth0_is_rule():
    r = G.QUADRATURE_RULES["9pt"]
    l1, l2, w = G.composite_nodes(r, 0)
    np.testing.assert_array_equal(l1, r.bary[:, 1])
    np.testing.assert_array_equal(l2, r.bary[:, 2])
    np.testing.assert_array_equal(w, r.weights)


@pytest.mark.parametrize("rule,deg", [("4pt", 3), ("9pt", 5), ("7pt", 5)])
def test_composite_exactness(rule, deg):
    """Subdivided rules stay exact for total degree <= rule degree on the reference triangle
    (integral of x^a y^b = a! b! / (a+b+2)!, area-normalised by 2)."""
    from math import factorial

    l1, l2, w = G.composite_nodes(G.QUADRATURE_RULES[rule], 2)
    for a in range(deg + 1):
        for b in range(deg + 1 - a):
            exact = 2.0 * factorial(a) * factorial(b) / factorial(a + b + 2)
            assert abs(np.sum(w * l1 ** a * l2 ** b) - exact) < 1e-14


def test_composite_nodes_match_reference_subdivision():
    """Node positions of the composite table == rule applied to the leaves of
    subdivide_fans (delaunay.py:383-407) incl. leaf vertex order (asymmetric 4pt rule)."""
    rng = np.random.default_rng(0)
    v = rng.standard_normal((1, 3, 3))
    fans = O.Fans(v, np.zeros(1, np.int64), np.zeros(1, np.int64), np.ones(1), 0)
    sub = O.subdivide(fans, 3)
    rule = O.RULES["4pt"]
    ref = np.einsum("qv,svj->sqj", rule.bary, sub.verts).reshape(-1, 3)
    l1, l2, _ = G.composite_nodes(G.QUADRATURE_RULES["4pt"], 3)
    v0, v1, v2 = v[0]
    mine = v0 + l1[:, None] * (v1 - v0) + l2[:, None] * (v2 - v0)
    d = np.abs(np.sort(ref, axis=0) - np.sort(mine, axis=0)).max()
    assert d < 1e-14


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_tanh4_table_accuracy(name):
    """rho^(1/4) table vs the closed form (both branches, random points): <= 3e-15 relative."""
    f = D.density_preset(name)
    coef, w = D.tanh4_table(f)
    rng = np.random.default_rng(1)
    y = D.normalize(rng.standard_normal((200000, 3)))
    u = np.zeros(len(y))
    for c in np.atleast_2d(f.center):
        x0 = np.linalg.norm(y - c, axis=1)
        x1 = np.linalg.norm(y + c, axis=1)
        uc = np.where(x0 ** 2 <= 2, D.eval_tanh4_table(coef[0], w, x0),
                      D.eval_tanh4_table(coef[1], w, x1))
        u = np.maximum(u, uc)
    ref = D.eval_density(f, y) ** 0.25
    assert np.max(np.abs(u - ref) / ref) <= 3e-15


@pytest.mark.parametrize("name", ["const", "x3", "x16", "x64", "c3", "c4", "c5"])
def test_density_host_eval_equals_oracle(name):
    z = P.random_sphere_points(5000, 2)
    np.testing.assert_array_equal(np.broadcast_to(D.eval_density(D.density_preset(name), z), 5000),
                                  np.broadcast_to(O.eval_density(O.density_for(name), z), 5000))
    assert D.density_preset(name).max_value == O.density_for(name).max_value


def test_sampler_matches_oracle():
    for name in ("c4", "c5"):
        np.testing.assert_array_equal(P.sample_by_density(D.density_preset(name), 3000, 0),
                                      O.sample_by_density(O.density_for(name), 3000, 0))


def test_density_kinds():
    assert D.density_preset("const").kind == 0
    assert D.density_preset("x16").kind == 2
    assert D.density_preset("x64").kind == 3
    assert D.density_preset("c4").kind == 4
    assert D.density_preset("c5").kind == 5
    p = D.device_params(D.density_preset("c5"))
    assert p["table"] is not None and p["center"][3:].any()


def _quadratic_phi(a, b, c):
    return lambda alpha: (a * alpha ** 2 + b * alpha + c, 2 * a * alpha + b, alpha)


@pytest.mark.parametrize("a,b", [(1.0, -1.0), (0.05, -1.0), (10.0, -1.0), (1e-4, -1e-3)])
def test_line_search_equals_oracle(a, b):
    phi = _quadratic_phi(a, b, 3.0)
    mine = wolfe_line_search(phi, 3.0, b)
    ref = O.wolfe_line_search(phi, 3.0, b)
    assert mine == ref


def test_line_search_failure_and_nondescent():
    with pytest.raises(P.LineSearchFailure):
        wolfe_line_search(lambda al: (10.0 + al, 1.0, al), 1.0, -1.0)
    with pytest.raises(P.NonDescentError):
        wolfe_line_search(lambda al: (al, 1.0, al), 0.0, 0.5)


def test_stopping_criteria_validation():
    with pytest.raises(ValueError):
        P.StoppingCriteria(movement_tol=0.0)
    with pytest.raises(ValueError):
        P.StoppingCriteria(max_iterations=0)


def test_bisection_ladder_and_bisect():
    assert P.bisection_ladder(655362, floor=2562) == [2562, 10242, 40962, 163842, 655362]
    ico = P.icosahedron_vertices()
    t = O.convex_hull_delaunay(ico)
    tri = P.SphericalTriangulation(t, np.zeros((len(t), 3)), np.zeros(len(t)))
    z = P.bisect(ico, tri)
    assert len(z) == 42 and np.allclose(np.linalg.norm(z, axis=1), 1.0)


def test_same_public_names_as_reference():
    ref = ["DensityField", "density_preset", "QuadratureRule", "QUADRATURE_RULES",
           "StoppingCriteria", "minimize", "MeshEvaluator", "bisect", "bisection_ladder"]
    for name in ref:
        assert hasattr(P, name), name


def test_unknown_perturbation_and_measure_rejected():
    """The graph Laplacian perturbations of cvt_core.py:206-214 are "a6" and "m2"; anything else
    raises like the reference's ValueError; the sharded evaluator keeps it single-GPU."""
    ev = P.MeshEvaluator(P.density_preset("const"), "4pt", laplacian="a6")
    assert ev.laplacian == "a6"
    with pytest.raises(ValueError):
        P.MeshEvaluator(P.density_preset("const"), "4pt", laplacian="b7")
    with pytest.raises(ValueError):
        P.MeshEvaluator(P.density_preset("const"), "4pt", measure="bogus")
    with pytest.raises(P.ConfigError):
        P.ShardedMeshEvaluator(P.density_preset("const"), "4pt", laplacian="m2")
    from paper_1709_06924_b200.optimizer import METHODS

    assert set(METHODS) == {"lloyd", "lbfgs", "lloyd-plbfgs", "laplacian-a6", "laplacian-m2"}


def test_runplan_validation():
    with pytest.raises(P.ConfigError):
        P.RunPlan(points=642, ladder=[160, 642])
    with pytest.raises(P.ConfigError):
        P.RunPlan(points=3)
    with pytest.raises(P.ConfigError):
        P.RunPlan(points=642, quadrature="5pt")
    p = P.RunPlan(points=642, density_name="x64")
    assert p.quadrature == "9pt" and p.ladder == [642]


def test_covering_host_helpers_match_reference_golden():
    """partition.py host forms: the adjacency bitmap handed to scvt_migration encodes exactly
    the one-level lists, and detect_migration / assign_points classify like the reference."""
    import numpy as np

    from conftest import golden
    from paper_1709_06924_b200.partition import (Covering, PointAssignment, assign_points,
                                                 detect_migration)

    g = golden("covering")
    one = tuple(tuple(int(x) for x in g["one_idx"][g["one_ptr"][k]:g["one_ptr"][k + 1]])
                for k in range(len(g["centers"])))
    cov = Covering(centers=g["centers"], one_level=one, two_level=())
    bits = cov.adjacency_bitmap()
    for a in range(cov.cell_count):
        got = [b for b in range(cov.cell_count) if (bits[a, b >> 5] >> (b & 31)) & 1]
        assert tuple(got) == one[a]
    a0 = assign_points(g["z0"], cov)
    assert detect_migration(a0, cov) == "in-place"
    far = PointAssignment(arithmetic=a0.arithmetic, geometric=a0.arithmetic.copy())
    far.geometric[0] = next(c for c in range(cov.cell_count) if c != far.arithmetic[0]
                            and c not in one[far.arithmetic[0]])
    assert detect_migration(far, cov) == "out-of-range"
    near = PointAssignment(arithmetic=a0.arithmetic, geometric=a0.arithmetic.copy())
    near.geometric[0] = one[near.arithmetic[0]][0]
    assert detect_migration(near, cov) == "neighbor-move"


def test_neighbor_lists_reproduce_reference_covering():
    """partition.neighbor_lists (partition.py:67-80) on the Delaunay triangles of the golden
    covering's centres gives the reference's one-level lists exactly; every two-level list
    holds its own cell and is closed over one more hop."""
    from conftest import golden
    from paper_1709_06924_b200.partition import neighbor_lists

    g = golden("covering")
    p = len(g["centers"])
    one, two = neighbor_lists(O.convex_hull_delaunay(g["centers"]), p)
    ref = tuple(tuple(int(x) for x in g["one_idx"][g["one_ptr"][k]:g["one_ptr"][k + 1]])
                for k in range(p))
    assert one == ref
    for l in range(p):
        assert l in two[l]
        assert set(two[l]) == {l}.union(one[l], *(one[m] for m in one[l]))


class _FakeOps:
    """Host stand-in for the device optimizer algebra (Minimizer control-flow tests)."""

    speculate = True

    def __init__(self, qg, dphi0):
        self.qg, self.dphi0 = qg, dphi0
        self.cleared = 0

    def vec3(self, z):
        return z.new_zeros(z.shape)

    positions = vec3

    def scalars(self, z):
        return z.new_ones(z.shape[0])

    def normalize(self, z):
        z /= z.norm(dim=1, keepdim=True)

    def history_clear(self):
        self.cleared += 1

    def gamma(self):
        return 1.0

    def direction_tangent_async(self, g, diag, gamma, z, q3):
        q3.copy_(-g)

    def direction_result(self):
        return self.qg, self.dphi0

    def trial(self, z, q3, alpha, zt, norms):
        zt.copy_(z + alpha * q3)

    def lloyd(self, first, z_out):
        z_out.copy_(first / first.norm(dim=1, keepdim=True))

    def push(self, z_old, z_new, g_old, g_new):
        return True, float((z_new - z_old).abs().max())


class _FakeEvaluator:
    """Evaluations succeed except at the speculative alpha = 1 trial point."""

    def __init__(self, ops):
        self.ops = ops
        self.evaluations = 0
        self.trial_calls = 0

    def _as_device(self, points):
        import torch

        return torch.as_tensor(np.asarray(points, dtype=float)), True

    def _ensure_ctx(self, n, m=None):
        return None

    def optimizer_ops(self, ctx, n):
        return self.ops

    def redecompose(self, points):
        return None

    def evaluate_device(self, z, q3=None, norms=None):
        from paper_1709_06924_b200.errors import CapacityError
        from paper_1709_06924_b200.pipeline import EvalResult

        if q3 is not None:
            self.trial_calls += 1
            raise CapacityError("trial point out of capacity")
        self.evaluations += 1
        return EvalResult(energy=1.0, grad=0.1 * z, grad_norm=1.0, lloyd_diag=z.new_ones(len(z)),
                          first=z.clone(), min_diag=1.0)


def test_failed_speculative_trial_discarded_on_lloyd_fallback():
    """q.g < 0 but g.q3 >= 0 -- the reference's line search raises NonDescentError
    before evaluating anything and takes the Lloyd fallback (optimizer.py:333-349), so an
    error raised by the speculative alpha = 1 trial must be discarded, not re-raised."""
    from paper_1709_06924_b200.optimizer import Minimizer

    ops = _FakeOps(qg=-1.0, dphi0=0.5)
    ev = _FakeEvaluator(ops)
    st = Minimizer(P.random_sphere_points(12, 0), "lloyd-plbfgs", ev, 5)
    rec, _, _, _ = st.step()
    assert ev.trial_calls == 1 and rec.step == 0.0 and rec.fevals == 1
    assert st.resets == 1 and ev.evaluations == 2       # initial + Lloyd step, trial uncounted


def test_failed_speculative_trial_reraised_when_the_reference_evaluates_it():
    """q.g < 0 and g.q3 < 0: the reference evaluates the alpha = 1 trial first, so its error
    propagates."""
    from paper_1709_06924_b200.errors import CapacityError
    from paper_1709_06924_b200.optimizer import Minimizer

    ev = _FakeEvaluator(_FakeOps(qg=-1.0, dphi0=-0.5))
    st = Minimizer(P.random_sphere_points(12, 0), "lloyd-plbfgs", ev, 5)
    with pytest.raises(CapacityError):
        st.step()
