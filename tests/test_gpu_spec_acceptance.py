"""SPEC.md acceptance criteria and the reference's in-package test oracles
(SURVEY.md §4), run through the GPU path.  The reference ships no tests; these are the
known-answer checks its SPEC states, with the deviations written next to each check:

  AC1/AC2  iteration ratios LBFGS / Lloyd-P-LBFGS (X16 >= 1.5, X64 >= 2), final X64 energy
           within 5 % of Table 1.  Monte Carlo starts are uniform
           (`random_sphere_points`): rho-sampled x16/x64 starts at K = 2562 leave an open
           hemisphere empty (DECISIONS.md D12).  Stopping criteria = the paper's
           = the reference defaults (optimizer.py:40-53).
  AC3      X3 final energies of every method within 5 % of the Table 1 band.
  AC4      tangential gradient vs central differences (h = 1e-6) at K = 50: the gradient
           formula is the derivative of the energy for the exact spherical measure
           (cvt_core.py:67-72, measure="sphere") on a converged quadrature (7-pt rule on
           depth-3 fans): 1e-5 for const/x3; x16/x64 have kinked densities (|lat|, |lon|,
           geodesic distance to the centre) whose quadrature error floors the difference
           (the reference itself: 1.1e-4 / 4.1e-4 on one K = 50 start, unchanged at depths
           4-5; up to 4.3e-3 / 1.2e-2 over the 20 starts here, relative to |g_i|), bounded at
           5e-2 -- the SPEC's 1e-5 holds for the smooth densities only.
  AC5      Lloyd step == normalize(z - g / lloyd_diag) (the Eq. (5) form) to 1e-12, and the
           energy non-increasing under Lloyd steps.
  AC6      the GPU two-loop recursion vs the dense product-form BFGS matrix, and the secant
           equation H y_k = s_k for the newest pair.
  AC7      brute-force empty-circumcircle oracle (delaunay.py:305-313) on GPU triangulations at
           K = 162, 642, 2562 from the bisection ladder, Euler counts T = 2K - 4.
  AC8      rho = 1 total mass error vs 4 pi shrinks by 3.5-4.5x per bisection level.
  AC9      sharded evaluation bitwise identical for 1, 2, 4, 8 shards at K = 10242, X3.
  AC11     converged X3 equator/pole spacing ratio in [2.5, 3.6].
  AC12     X64: Laplacian(m2) needs fewer iterations than Lloyd-P-LBFGS (soft: 2 of 3 starts).
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1709_06924_b200 as P  # noqa: E402
from paper_1709_06924_b200.pipeline import default_quadrature  # noqa: E402


def _converge(dname, method, seed, k=2562, max_it=2000):
    dens = P.density_preset(dname)
    lap = {"laplacian-m2": "m2", "laplacian-a6": "a6"}.get(method)
    with P.MeshEvaluator(dens, default_quadrature(dname), laplacian=lap) as ev:
        return P.minimize(P.random_sphere_points(k, seed), method, ev,
                          P.StoppingCriteria(max_iterations=max_it))


@pytest.mark.parametrize("dname,ratio", [("x16", 1.5), ("x64", 2.0)])
def test_ac1_ac2_lloyd_preconditioning_speeds_up_lbfgs(dname, ratio):
    ok = 0
    for seed in (0, 1, 2):
        a = _converge(dname, "lloyd-plbfgs", seed)
        b = _converge(dname, "lbfgs", seed)
        ok += len(b.records) / len(a.records) >= ratio
        if dname == "x64":    # Table 1 X64 Lloyd P-LBFGS F = 1.04699e-04
            assert abs(a.final.energy - 1.04699e-4) <= 0.05 * 1.04699e-4
    assert ok >= 2


def test_ac3_x3_final_energies_in_table1_band():
    for m in ("lloyd", "lbfgs", "lloyd-plbfgs", "laplacian-m2", "laplacian-a6"):
        f = _converge("x3", m, 0).final.energy
        assert 0.95 * 1.325e-3 <= f <= 1.05 * 1.327e-3, (m, f)


@pytest.mark.parametrize("dname,tol", [("const", 1e-5), ("x3", 1e-5), ("x16", 5e-2),
                                       ("x64", 5e-2)])
def test_ac4_gradient_matches_central_differences(dname, tol):
    h = 1e-6
    with P.MeshEvaluator(P.density_preset(dname), "7pt", subdivision=3, measure="sphere") as ev:
        worst = 0.0
        for cfg in range(20):
            z = P.random_sphere_points(50, 100 + cfg)
            g = ev.evaluate(z).grad
            rng = np.random.default_rng(cfg)
            for i in rng.choice(50, 5, replace=False):
                t1 = np.cross(z[i], rng.standard_normal(3))
                t1 /= np.linalg.norm(t1)
                for t in (t1, np.cross(z[i], t1)):
                    zp, zm = z.copy(), z.copy()
                    zp[i] = P.normalize(z[i] + h * t)
                    zm[i] = P.normalize(z[i] - h * t)
                    fd = (ev.evaluate(zp).energy - ev.evaluate(zm).energy) / (2 * h)
                    worst = max(worst, abs(fd - g[i] @ t) / np.linalg.norm(g[i]))
    assert worst < tol, worst


def test_ac5_lloyd_identity_and_monotone_energy():
    with P.MeshEvaluator(P.density_preset("x3"), "4pt") as ev:
        for cfg in range(100):
            z = P.random_sphere_points(162, 1000 + cfg)
            r = ev.evaluate(z)
            lloyd = r.first / np.linalg.norm(r.first, axis=1, keepdims=True)
            eq5 = P.normalize(z - r.grad / r.lloyd_diag[:, None])
            assert np.max(np.abs(lloyd - eq5)) <= 1e-12
        z = P.random_sphere_points(642, 7)
        res = P.minimize(z, "lloyd", ev, P.StoppingCriteria(max_iterations=30, movement_tol=1e-300,
                                                            grad_tol=1e-300, stall_tol=1e-300))
        e = [ev.evaluate(z).energy] + [r.energy for r in res.records]
        assert all(b <= a + 1e-10 * a for a, b in zip(e, e[1:]))


def _dense_bfgs(pairs, h0):
    """The product form H = V^T H V + rho s s^T over the pairs, oldest first."""
    h = np.diag(h0)
    for s, y in pairs:
        rho = 1.0 / (y @ s)
        v = np.eye(len(s)) - rho * np.outer(y, s)
        h = v.T @ h @ v + rho * np.outer(s, s)
    return h


@pytest.mark.parametrize("k,m", [(8, 3), (12, 7), (20, 7)])
def test_ac6_two_loop_matches_dense_product_form(k, m):
    from paper_1709_06924_b200 import optimizer as OPT

    rng = np.random.default_rng(k * 31 + m)
    n3 = 3 * k
    with P.MeshEvaluator(P.density_preset("const"), "4pt") as ev:
        ctx = ev._ensure_ctx(k, m)
        ops = OPT._DeviceOps(ctx, k)
        ops.history_clear()
        dev = torch.device("cuda", ctx.device)
        pairs = []
        zo = torch.zeros((k, 3), dtype=torch.float64, device=dev)
        go = torch.zeros((k, 3), dtype=torch.float64, device=dev)
        a = rng.standard_normal((n3, n3))
        spd = a @ a.T + n3 * np.eye(n3)              # y = A s keeps y.s > 0
        for _ in range(m + 2):                       # overflow the ring of m pairs
            s = rng.standard_normal(n3)
            y = spd @ s
            zn = zo + torch.as_tensor(s.reshape(k, 3), device=dev)
            gn = go + torch.as_tensor(y.reshape(k, 3), device=dev)
            pushed, _ = ops.push(zo, zn, go, gn)
            assert pushed
            pairs.append((s, y))
            zo, go = zn, gn
        pairs = pairs[-m:]
        diag = rng.uniform(0.5, 2.0, k)
        h = _dense_bfgs(pairs, np.repeat(1.0 / diag, 3))
        g = rng.standard_normal(n3)
        gt = torch.as_tensor(g.reshape(k, 3), device=dev)
        q = torch.empty_like(gt)
        qg = ops.direction(gt, torch.as_tensor(diag, device=dev), 0.0, q)
        qn = q.cpu().numpy().ravel()
        assert np.linalg.norm(qn - (-h @ g)) <= 1e-12 * np.linalg.norm(h @ g)
        assert abs(qg - qn @ g) <= 1e-12 * abs(qg)
        # secant equation for the newest pair: H y_k = s_k
        s_k, y_k = pairs[-1]
        ops.direction(torch.as_tensor(y_k.reshape(k, 3), device=dev),
                      torch.as_tensor(diag, device=dev), 0.0, q)
        assert np.linalg.norm(-q.cpu().numpy().ravel() - s_k) <= 1e-10 * np.linalg.norm(s_k)


def _ladder_sets():
    z = P.icosahedron_vertices()
    out = {}
    with P.MeshEvaluator(P.density_preset("const"), "4pt") as ev:
        while len(z) < 2562:
            z = P.pipeline.bisect(z, ev.triangulation(z))
            out[len(z)] = z
    return out


def test_ac7_empty_circumcircles_and_euler_counts():
    sets = _ladder_sets()
    rng = np.random.default_rng(0)
    with P.MeshEvaluator(P.density_preset("const"), "4pt") as ev:
        for k in (162, 642, 2562):
            for z in (sets[k], P.normalize(sets[k] + 1e-3 * rng.standard_normal(sets[k].shape)),
                      P.random_sphere_points(k, k)):
                t = ev.triangulation(z).triangles
                assert len(t) == 2 * k - 4
                e = np.sort(np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]]), axis=1)
                assert len(np.unique(e, axis=0)) == 3 * k - 6
                assert O.empty_circumcircle_violations(z, t) == 0


def test_ac8_mass_convergence_rate():
    sets = _ladder_sets()
    err = []
    with P.MeshEvaluator(P.density_preset("const"), "4pt") as ev:
        for k in (162, 642, 2562):
            err.append(4.0 * np.pi - ev.evaluate(sets[k]).mass.sum())
    assert all(e > 0 for e in err)
    for a, b in zip(err, err[1:]):
        assert 3.5 <= a / b <= 4.5, (a, b)


def test_ac9_sharded_evaluation_bitwise_for_1_2_4_8():
    from paper_1709_06924_b200.parallel import CudaShardBackend, emulate_shards

    zt = torch.from_numpy(P.sample_by_density(P.density_preset("x3"), 10242, 0)).cuda()
    with P.MeshEvaluator(P.density_preset("x3"), "4pt") as ev:
        ref = ev.evaluate_device(zt)
        for ns in (1, 2, 4, 8):
            sh = emulate_shards(CudaShardBackend(ev), zt, ns)
            assert sh.energy == ref.energy and sh.grad_norm == ref.grad_norm
            assert torch.equal(sh.grad, ref.grad) and torch.equal(sh.first, ref.first)


def test_ac11_x3_spacing_ratio():
    r = _converge("x3", "lloyd-plbfgs", 0, max_it=3000)
    with P.MeshEvaluator(P.density_preset("x3"), "4pt") as ev:
        e = ev.triangulation(r.points).edges()
    z = r.points
    ln = np.linalg.norm(z[e[:, 0]] - z[e[:, 1]], axis=1)
    lat = np.abs(P.normalize(z[e[:, 0]] + z[e[:, 1]])[:, 2])
    ratio = ln[lat < np.sin(np.deg2rad(10))].mean() / ln[lat > np.cos(np.deg2rad(10))].mean()
    assert 2.5 <= ratio <= 3.6, ratio


def test_ac12_laplacian_m2_fewer_iterations_on_x64():
    fewer = 0
    for seed in (0, 1, 2):
        a = _converge("x64", "lloyd-plbfgs", seed)
        b = _converge("x64", "laplacian-m2", seed)
        fewer += len(b.records) < len(a.records)
    assert fewer >= 2
