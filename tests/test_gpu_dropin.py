"""Drop-in behaviour at the reference's boundary:

* the reference-style optimizer (the oracle's restatement of
  optimizer.py:278-391, duck-typed) driving the GPU evaluator through NumPy;
* the reverse: this package's `minimize` accepting a foreign evaluator of the reference
  protocol (`HostEvaluatorAdapter`), here the oracle's, against the live-reference golden;
* NumPy callbacks for NumPy input (optimizer.py:364-365);
* x16 near a pole raises PoleAmbiguityError on the device, as density.py:82-90 does;
* a measure="sphere" trajectory (cvt_core.py:84-90) against the oracle's.
"""

import numpy as np
import pytest

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1709_06924_b200 as P  # noqa: E402

CRIT = dict(movement_tol=1e-300, grad_tol=1e-300, stall_tol=1e-300)


class GpuMeshEvaluator:
    """The reference-side shim of INTEGRATION.md §2 (NumPy in, NumPy out)."""

    def __init__(self, density_name, rule, subdivision=0, measure="flat"):
        self._ev = P.MeshEvaluator(P.density_preset(density_name), rule, subdivision=subdivision,
                                   measure=measure)
        self.evaluations = 0

    def evaluate(self, points):
        r = self._ev.evaluate(np.asarray(points, dtype=float))
        self.evaluations += 1
        return O.EvalResult(energy=r.energy, grad=r.grad, grad_norm=r.grad_norm,
                            lloyd_diag=r.lloyd_diag, first=r.first, mass=r.mass)

    def redecompose(self, points):
        return None

    def close(self):
        self._ev.close()


def test_reference_optimizer_drives_gpu_evaluator(gold):
    g = gold("traj_c1_4pt")
    ev = GpuMeshEvaluator("const", "4pt")
    try:
        res = O.minimize(g["z0"], "lloyd-plbfgs", ev, O.StoppingCriteria(30, 1e-300, 1e-300, 1e-300),
                         corrections=5)
    finally:
        ev.close()
    e = np.array([r.energy for r in res.records])
    assert np.max(np.abs(e - g["energy"][:30]) / g["energy"][:30]) <= 1e-10
    assert [r.fevals for r in res.records] == g["fevals"][:30].tolist()
    with P.MeshEvaluator(P.density_preset("const"), "4pt") as gpu:
        mine = P.minimize(g["z0"], "lloyd-plbfgs", gpu,
                          P.StoppingCriteria(max_iterations=30, **CRIT), corrections=5)
    assert rel(res.points, mine.points) <= 1e-10


def test_minimize_accepts_a_reference_protocol_evaluator(gold):
    g = gold("traj_c1_4pt")
    snaps = {}

    def cb(n, z, r):
        assert isinstance(z, np.ndarray) and isinstance(r.grad, np.ndarray)
        if n in (1, 2, 5, 10, 20):
            snaps[n] = z.copy()

    ev = O.Evaluator(O.density_for("const"), "4pt", 0)
    res = P.minimize(g["z0"], "lloyd-plbfgs", ev, P.StoppingCriteria(max_iterations=20, **CRIT),
                     corrections=5, callback=cb)
    e = np.array([r.energy for r in res.records])
    assert np.max(np.abs(e - g["energy"][:20]) / g["energy"][:20]) <= 1e-10
    assert [r.fevals for r in res.records] == g["fevals"][:20].tolist()
    assert ev.evaluations == res.fevals          # no speculative trial reaches the evaluator
    for n, z in snaps.items():
        assert rel(z, g[f"z_{n}"]) <= 1e-10, n


def test_x16_pole_raises_like_the_reference():
    """A quadrature node at a pole: the reference's x16 density raises (density.py:82-90,
    elliptical_distance); so must the device.  A vertex rule (nodes at the fan sub-triangle
    vertices, one of which is the generator) puts a node exactly on a generator at the pole."""
    bary, w = np.eye(3), np.full(3, 1.0 / 3.0)
    z = np.vstack([P.random_sphere_points(640, 3), [[0.0, 0.0, 1.0]]])
    with pytest.raises(O.PoleAmbiguityError):
        O.Evaluator(O.density_for("x16"), O.Rule("vertex3", bary, w), 0).evaluate(z)
    with P.MeshEvaluator(P.density_preset("x16"), P.QuadratureRule("vertex3", bary, w)) as ev:
        with pytest.raises(P.PoleAmbiguityError):
            ev.evaluate(z)
    # away from the poles the same rule evaluates like the oracle
    z2 = P.random_sphere_points(641, 3)
    with P.MeshEvaluator(P.density_preset("x16"), P.QuadratureRule("vertex3", bary, w)) as ev:
        r = ev.evaluate(z2)
    o = O.Evaluator(O.density_for("x16"), O.Rule("vertex3", bary, w), 0).evaluate(z2)
    assert abs(r.energy - o.energy) <= 1e-12 * o.energy
    assert rel(r.first, o.first) <= 1e-12


def test_sphere_measure_trajectory_vs_oracle():
    z0 = P.random_sphere_points(2562, 0)
    it = 20
    ref = O.minimize(z0, "lloyd-plbfgs", O.Evaluator(O.density_for("x3"), "4pt", 0, "sphere"),
                     O.StoppingCriteria(it, 1e-300, 1e-300, 1e-300), corrections=7)
    with P.MeshEvaluator(P.density_preset("x3"), "4pt", measure="sphere") as ev:
        res = P.minimize(z0, "lloyd-plbfgs", ev, P.StoppingCriteria(max_iterations=it, **CRIT),
                         corrections=7)
    e = np.array([r.energy for r in res.records])
    eo = np.array([r.energy for r in ref.records])
    assert np.max(np.abs(e - eo) / eo) <= 1e-10
    assert [r.fevals for r in res.records] == [r.fevals for r in ref.records]
    assert rel(res.points, ref.points) <= 1e-10
