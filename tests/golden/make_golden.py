"""Generate golden fixtures by running the LIVE reference (`scvtmesh`, pure Python).

Run in the build container only (it needs /root/reference, which does not exist on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [--only NAME ...] [--skip-slow]

The reference has no 7-point rule, never calls `subdivide_fans` from its evaluator and has
no tanh^4 / two-centre density.  They are injected WITHOUT editing
the reference, exactly as DECISIONS.md fixes them:

* 7-point rule: a `QuadratureRule("7pt", bary, weights)` instance (Radon degree-5 rule);
  `cell_quadrature` only reads `.bary`/`.weights` (cvt_core.py:80, 93).
* depth-d subdivision: `scvtmesh.pipeline.cell_quadrature` is wrapped so each chunk of fans
  goes through `delaunay.subdivide_fans(chunk, d)` first (delaunay.py:383-407), outputs summed.
* tanh^4 densities: `scvtmesh.cvt_core.eval_density` and `scvtmesh.density.eval_density` are
  replaced by a function that handles variants "tanh4"/"tanh4x2" and delegates otherwise;
  `max_value` comes from a DensityField subclass (density.py:42-51 is what the sampler reads).

Everything written here is small (.npz) and committed; the oracle (`oracle/`) and the CUDA
path are both checked against these files.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import scvtmesh  # noqa: E402
from scvtmesh import cvt_core, delaunay, density as dmod, geometry, optimizer, pipeline  # noqa: E402

# --------------------------------------------------------------------------- injections
A1 = (6.0 - np.sqrt(15.0)) / 21.0
A2 = (6.0 + np.sqrt(15.0)) / 21.0
W0 = 9.0 / 40.0
W1 = (155.0 - np.sqrt(15.0)) / 1200.0
W2 = (155.0 + np.sqrt(15.0)) / 1200.0


def radon7():
    bary = np.array([
        [1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0],
        [1.0 - 2.0 * A1, A1, A1], [A1, 1.0 - 2.0 * A1, A1], [A1, A1, 1.0 - 2.0 * A1],
        [1.0 - 2.0 * A2, A2, A2], [A2, 1.0 - 2.0 * A2, A2], [A2, A2, 1.0 - 2.0 * A2],
    ])
    w = np.array([W0, W1, W1, W1, W2, W2, W2])
    return geometry.QuadratureRule("7pt", bary, w / w.sum())


RULES = {"4pt": geometry.FOUR_POINT, "9pt": geometry.NINE_POINT, "7pt": radon7()}

_ORIG_CQ = cvt_core.cell_quadrature
_DEPTH = {"d": 0}
CHUNK = 16384


def _cq_subdivided(points, fans, density, rule, k, with_pairs=False, measure="flat"):
    d = _DEPTH["d"]
    if d == 0:
        return _ORIG_CQ(points, fans, density, rule, k, with_pairs=with_pairs, measure=measure)
    mass = np.zeros(k)
    first = np.zeros((k, 3))
    energy = 0.0
    S = len(fans.cells)
    for s in range(0, S, CHUNK):
        e = min(S, s + CHUNK)
        sub = delaunay.VoronoiFans(fans.verts[s:e], fans.cells[s:e], fans.edge_other[s:e],
                                   fans.signed_area[s:e], fans.obtuse_count)
        sub = delaunay.subdivide_fans(sub, d)
        m, c, en, _, _ = _ORIG_CQ(points, sub, density, rule, k, measure=measure)
        mass += m
        first += c
        energy += en
    return mass, first, energy, None, None


pipeline.cell_quadrature = _cq_subdivided


@dataclass(frozen=True)
class Tanh4Field(dmod.DensityField):
    """variant 'tanh4' (one centre) or 'tanh4x2' (center is (2,3)); d = geodesic, min over centres."""

    @property
    def max_value(self) -> float:
        return float((((1.0 - self.gamma) / 2.0) * (np.tanh(self.beta / self.alpha) + 1.0)
                      + self.gamma) ** 4)


_ORIG_EVAL = dmod.eval_density


def _eval_density(field, x):
    if field.variant in ("tanh4", "tanh4x2"):
        x = geometry.normalize(x)
        cs = np.atleast_2d(field.center)
        d = geometry.geodesic_distance(x, cs[0])
        for c in cs[1:]:
            d = np.minimum(d, geometry.geodesic_distance(x, c))
        g = field.gamma
        return (((1.0 - g) / 2.0) * (np.tanh((field.beta - d) / field.alpha) + 1.0) + g) ** 4
    return _ORIG_EVAL(field, x)


cvt_core.eval_density = _eval_density
dmod.eval_density = _eval_density


def latlon(lat_deg, lon_deg):
    la, lo = np.deg2rad(lat_deg), np.deg2rad(lon_deg)
    return geometry.normalize(np.array([np.cos(la) * np.cos(lo), np.cos(la) * np.sin(lo), np.sin(la)]))


def field_for(cfg: str):
    if cfg == "const":
        return dmod.density_preset("const")
    if cfg in ("x3", "x16", "x64"):
        return dmod.density_preset(cfg)
    if cfg == "c3":
        return Tanh4Field("tanh4", gamma=1.0 / 16.0, beta=np.pi / 6.0, alpha=0.20, center=latlon(30, -90))
    if cfg == "c4":
        return Tanh4Field("tanh4", gamma=1.0 / 8.0, beta=np.pi / 6.0, alpha=0.20, center=latlon(30, -90))
    if cfg == "c5":
        return Tanh4Field("tanh4x2", gamma=1.0 / 16.0, beta=np.pi / 8.0, alpha=0.15,
                          center=np.stack([latlon(30, -90), latlon(-20, 150)]))
    raise ValueError(cfg)


def evaluator(cfg, rule, depth):
    _DEPTH["d"] = depth
    return pipeline.MeshEvaluator(field_for(cfg), RULES[rule])


def eval_dict(z, cfg, rule, depth, prefix):
    ev = evaluator(cfg, rule, depth)
    r = ev.evaluate(z)
    mass, first, energy, _, _ = _cq_subdivided(
        z, delaunay.build_voronoi_geometry(z, delaunay.convex_hull_delaunay(z)),
        field_for(cfg), RULES[rule], len(z))
    return {
        f"{prefix}mass": mass, f"{prefix}first": r.first, f"{prefix}energy": np.float64(r.energy),
        f"{prefix}grad": r.grad, f"{prefix}grad_norm": np.float64(r.grad_norm),
        f"{prefix}lloyd_diag": r.lloyd_diag,
    }


def tri_digest(t):
    return hashlib.sha256(np.ascontiguousarray(t, dtype=np.int64).tobytes()).hexdigest()


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)", flush=True)


# --------------------------------------------------------------------------- cases
def case_rules():
    """Rule tables and KATs that are independent of point sets."""
    out = {}
    for k, r in RULES.items():
        out[f"{k}_bary"] = r.bary
        out[f"{k}_weights"] = r.weights
    save("rules", **out)


def case_c1_eval():
    z = geometry.random_sphere_points(2562, 0)
    tri = delaunay.convex_hull_delaunay(z)
    fans = delaunay.build_voronoi_geometry(z, tri)
    out = {"z": z, "triangles": tri.triangles, "circumcenters": tri.circumcenters,
           "circumradii": tri.circumradii, "obtuse_count": np.int64(fans.obtuse_count)}
    for rule, depth in (("4pt", 0), ("9pt", 0), ("7pt", 0), ("7pt", 1), ("4pt", 3), ("7pt", 3)):
        out.update(eval_dict(z, "const", rule, depth, f"{rule}_d{depth}_"))
    save("c1_eval", **out)


def case_density_eval():
    """Variable densities on small point sets (uniform and rho-sampled), 7pt_d3 and 4pt_d0."""
    out = {}
    zu = geometry.random_sphere_points(2562, 0)
    out["uniform_z"] = zu
    for cfg in ("x3", "x16", "x64", "c3", "c4", "c5"):
        out.update(eval_dict(zu, cfg, "4pt", 0, f"uniform_{cfg}_4pt_d0_"))
        out.update(eval_dict(zu, cfg, "7pt", 3, f"uniform_{cfg}_7pt_d3_"))
    for cfg in ("c3", "c4", "c5"):
        f = field_for(cfg)
        zs = dmod.sample_by_density(f, 2562, 0)
        out[f"sampled_{cfg}_z"] = zs
        out[f"sampled_{cfg}_rho_max"] = np.float64(f.max_value)
        out[f"sampled_{cfg}_rho"] = _eval_density(f, zs)
        tri = delaunay.convex_hull_delaunay(zs)
        out[f"sampled_{cfg}_triangles"] = tri.triangles
        out.update(eval_dict(zs, cfg, "7pt", 3, f"sampled_{cfg}_7pt_d3_"))
    save("density_eval", **out)


def case_sampler():
    """sample_by_density stream parity at the config sizes (digest + head only)."""
    out = {}
    for cfg, n in (("c3", 163842), ("c4", 655362), ("c5", 2621442)):
        f = field_for(cfg)
        z = dmod.sample_by_density(f, n, 0)
        out[f"{cfg}_head"] = z[:64]
        out[f"{cfg}_tail"] = z[-64:]
        out[f"{cfg}_sum"] = z.sum(axis=0)
        out[f"{cfg}_sha"] = np.array(hashlib.sha256(z.tobytes()).hexdigest())
    for n in (40962, 655362):
        z = geometry.random_sphere_points(n, 0)
        out[f"uniform{n}_sha"] = np.array(hashlib.sha256(z.tobytes()).hexdigest())
    save("sampler", **out)


def case_medium():
    """N=40,962 uniform, 4pt_d0 (cheap): triangle digest + full moments; and the c4
    sampler at N=40,962 (rho-sampled, extreme non-uniformity) triangle digest + 4pt moments."""
    out = {}
    z = geometry.random_sphere_points(40962, 0)
    tri = delaunay.convex_hull_delaunay(z)
    out["u_tri_sha"] = np.array(tri_digest(tri.triangles))
    out["u_tri_count"] = np.int64(tri.count)
    out["u_triangles_head"] = tri.triangles[:256]
    out.update(eval_dict(z, "const", "4pt", 0, "u_4pt_d0_"))
    for cfg in ("c4", "c3"):
        f = field_for(cfg)
        zs = dmod.sample_by_density(f, 40962, 0)
        tri = delaunay.convex_hull_delaunay(zs)
        out[f"{cfg}_tri_sha"] = np.array(tri_digest(tri.triangles))
        out[f"{cfg}_tri_count"] = np.int64(tri.count)
        out.update(eval_dict(zs, cfg, "4pt", 0, f"{cfg}_4pt_d0_"))
    save("medium", **out)


def case_small_sets():
    out = {}
    tet = geometry.normalize(np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1.0]]))
    ico = geometry.icosahedron_vertices()
    rnd = {n: geometry.random_sphere_points(n, 7) for n in (5, 6, 50, 162)}
    sets = {"tet": tet, "ico": ico, **{f"rnd{n}": v for n, v in rnd.items()}}
    for name, z in sets.items():
        tri = delaunay.convex_hull_delaunay(z)
        out[f"{name}_z"] = z
        out[f"{name}_triangles"] = tri.triangles
        out.update(eval_dict(z, "const", "4pt", 0, f"{name}_4pt_d0_"))
        out.update(eval_dict(z, "const", "7pt", 3, f"{name}_7pt_d3_"))
    save("small_sets", **out)


def _traj(z0, cfg, rule, depth, method, m, iters, keep, tol=1e-300):
    ev = evaluator(cfg, rule, depth)
    crit = optimizer.StoppingCriteria(max_iterations=iters, movement_tol=tol, grad_tol=tol,
                                      stall_tol=tol)
    snaps = {}

    def cb(n, z, res):
        if n in keep:
            snaps[n] = z.copy()

    t0 = time.perf_counter()
    res = optimizer.minimize(z0, method, ev, crit, corrections=m, callback=cb)
    print(f"  traj {cfg} {rule}_d{depth} {method} m={m}: {len(res.records)} it, "
          f"{res.fevals} fevals, reason={res.reason}, resets={res.resets}, "
          f"{time.perf_counter() - t0:.1f}s", flush=True)
    out = {
        "z0": z0,
        "energy": np.array([r.energy for r in res.records]),
        "grad_norm": np.array([r.grad_norm for r in res.records]),
        "step": np.array([r.step for r in res.records]),
        "fevals": np.array([-1 if r.fevals is None else r.fevals for r in res.records]),
        "final_z": res.points, "final_grad": res.final.grad, "final_first": res.final.first,
        "reason": np.array(res.reason), "resets": np.int64(res.resets),
        "fevals_total": np.int64(res.fevals),
        "snap_iters": np.array(sorted(snaps)),
    }
    for n, zz in snaps.items():
        out[f"z_{n}"] = zz
    return out


def case_traj_fast():
    z0 = geometry.random_sphere_points(2562, 0)
    save("traj_c1_4pt", **_traj(z0, "const", "4pt", 0, "lloyd-plbfgs", 5, 100, {1, 2, 5, 10, 20, 50}))
    save("traj_c1_4pt_lbfgs", **_traj(z0, "const", "4pt", 0, "lbfgs", 7, 30, {1, 2, 10}))
    save("traj_c1_4pt_lloyd", **_traj(z0, "const", "4pt", 0, "lloyd", 7, 30, {1, 2, 10}))
    z1 = dmod.sample_by_density(field_for("c4"), 2562, 0)
    save("traj_c4small_4pt", **_traj(z1, "c4", "4pt", 0, "lloyd-plbfgs", 7, 40, {1, 2, 5, 10, 20}))
    z2 = dmod.sample_by_density(field_for("c3"), 2562, 0)
    save("traj_c3small_4pt", **_traj(z2, "c3", "4pt", 0, "lloyd-plbfgs", 7, 40, {1, 2, 5, 10, 20}))


def case_traj_slow():
    z0 = geometry.random_sphere_points(2562, 0)
    save("traj_c1", **_traj(z0, "const", "7pt", 3, "lloyd-plbfgs", 5, 100,
                            {1, 2, 3, 5, 10, 20, 50}))
    z1 = dmod.sample_by_density(field_for("c4"), 2562, 0)
    save("traj_c4small", **_traj(z1, "c4", "7pt", 3, "lloyd-plbfgs", 7, 12, {1, 2, 3, 5}))


def case_traj_fallback():
    """Trajectories whose line searches zoom / exhaust / fall back (non-degenerate sets:
    the hull contains the origin, so the hull IS the spherical Delaunay triangulation)."""
    z0 = geometry.random_sphere_points(2562, 0)
    save("traj_x64_4pt", **_traj(z0, "x64", "4pt", 0, "lloyd-plbfgs", 7, 40, {1, 2, 5, 10, 20}))
    z1 = dmod.sample_by_density(field_for("c5"), 10242, 0)
    save("traj_c5small_4pt", **_traj(z1, "c5", "4pt", 0, "lloyd-plbfgs", 10, 30, {1, 2, 5, 10}))


def case_medium_slim():
    """Slim replacement for `medium` (keeps fixtures small)."""
    out = {}
    z = geometry.random_sphere_points(40962, 0)
    tri = delaunay.convex_hull_delaunay(z)
    out["u_tri_sha"] = np.array(tri_digest(tri.triangles))
    out["u_tri_count"] = np.int64(tri.count)
    d = eval_dict(z, "const", "4pt", 0, "u_4pt_d0_")
    out["u_4pt_d0_first"] = d["u_4pt_d0_first"]
    out["u_4pt_d0_energy"] = d["u_4pt_d0_energy"]
    for cfg in ("c4", "c5"):
        f = field_for(cfg)
        zs = dmod.sample_by_density(f, 40962, 0)
        tri = delaunay.convex_hull_delaunay(zs)
        out[f"{cfg}_tri_sha"] = np.array(tri_digest(tri.triangles))
        out[f"{cfg}_tri_count"] = np.int64(tri.count)
        d = eval_dict(zs, cfg, "4pt", 0, "x_")
        out[f"{cfg}_4pt_d0_energy"] = d["x_energy"]
        out[f"{cfg}_4pt_d0_first_sum"] = d["x_first"].sum(axis=0)
        out[f"{cfg}_4pt_d0_first_head"] = d["x_first"][:512]
    save("medium", **out)


def case_run_ladder():
    """pipeline.run: optimise-bisect ladder 162 -> 642 (x3 density, 4-pt rule, global path:
    partitions=64 keeps K < 16 p so no covering is used)."""
    _DEPTH["d"] = 0
    plan = pipeline.RunPlan(points=642, density_name="x3", method="lloyd-plbfgs", seed=1,
                            partitions=64, quadrature="4pt", ladder=[162, 642],
                            criteria=optimizer.StoppingCriteria(max_iterations=25))
    res = pipeline.run(plan)
    out = {"final_z": res.points, "triangles": res.triangulation.triangles}
    for li, lv in enumerate(res.levels):
        out[f"level{li}_energy"] = np.array([r.energy for r in lv.result.records])
        out[f"level{li}_points"] = lv.result.points
        out[f"level{li}_reason"] = np.array(lv.result.reason)
    save("run_ladder", **out)


def case_covering():
    """Region mode: a coarse covering (bootstrap_partition_cvt) and a P-LBFGS run through the
    reference's region path, whose migration class triggers re-decompose + history resets
    (optimizer.py:377-381)."""
    from scvtmesh import partition

    _DEPTH["d"] = 0
    # points clustered on the c4 plateau, optimised for a constant density: they spread over
    # the sphere, so some leave the neighbourhood of their frozen cell (out-of-range)
    z0 = dmod.sample_by_density(field_for("c4"), 2562, 3)
    cov = partition.bootstrap_partition_cvt(64, seed=0, density=field_for("const"))
    ev = pipeline.MeshEvaluator(field_for("const"), geometry.QUADRATURE_RULES["4pt"], cov,
                                workers=1, backend="thread")
    # per evaluation (line-search trials included): did the region path fall back?
    fb_seq = []
    orig_eval = ev.evaluate

    def evaluate(points):
        before = ev.fallbacks
        r = orig_eval(points)
        fb_seq.append(ev.fallbacks - before)
        return r

    ev.evaluate = evaluate
    crit = optimizer.StoppingCriteria(max_iterations=40, movement_tol=1e-300, grad_tol=1e-300,
                                      stall_tol=1e-300)
    mig = []
    res = optimizer.minimize(z0, "lloyd-plbfgs", ev, crit, corrections=7,
                             callback=lambda n, z, r: mig.append(r.migration))
    ev.close()
    print(f"  covering run: {len(res.records)} it, resets={res.resets}, fallbacks={ev.fallbacks}, "
          f"migration counts {dict((m, mig.count(m)) for m in set(mig))}", flush=True)
    one_ptr = np.cumsum([0] + [len(t) for t in cov.one_level])
    one_idx = np.concatenate([np.asarray(t, dtype=np.int64) for t in cov.one_level])
    save("covering", centers=cov.centers, one_ptr=one_ptr, one_idx=one_idx, z0=z0,
         energy=np.array([r.energy for r in res.records]),
         fevals=np.array([-1 if r.fevals is None else r.fevals for r in res.records]),
         migration=np.array(mig), resets=np.int64(res.resets), final_z=res.points,
         reason=np.array(res.reason), fallbacks=np.int64(ev.fallbacks),
         fallback_seq=np.array(fb_seq, dtype=np.int64))


def case_region_cover():
    """Region path (pipeline.py:62-98, 171-242): which Voronoi-sort regions of a covering the
    reference's `_region_task` fails for (CoverageError 1, AntipodeError 2,
    InsufficientPointsError 4, CollinearInputError 8), uniform points over bootstrap
    coverings; the GPU predicts the same per-region outcome from the global cycles."""
    import warnings

    from scvtmesh import errors, partition

    warnings.simplefilter("ignore")
    _DEPTH["d"] = 0
    codes = {errors.CoverageError: 1, errors.AntipodeError: 2,
             errors.InsufficientPointsError: 4, errors.CollinearInputError: 8}
    out = {}
    for ci, (k, p, seed) in enumerate([(2562, 64, 5), (1282, 32, 5), (5122, 64, 5),
                                        (10242, 64, 5), (642, 64, 2)]):
        z0 = geometry.random_sphere_points(k, seed)
        cov = partition.bootstrap_partition_cvt(p, seed=0, density=field_for("const"))
        ev = pipeline.MeshEvaluator(field_for("const"), geometry.QUADRATURE_RULES["4pt"], cov,
                                    workers=1, backend="thread")
        assign = ev._assign(z0)
        res = np.zeros(p, dtype=np.int64)
        for l in range(p):
            owned = np.flatnonzero(assign.geometric == l)
            if len(owned) == 0:
                continue
            try:
                pl = next(x for x in ev._payloads(z0, assign, False)
                          if np.array_equal(x["contact"], cov.centers[l]))
                pipeline._region_task(pl)
            except tuple(codes) as exc:
                res[l] = codes[type(exc)]
        ev.close()
        one_ptr = np.cumsum([0] + [len(t) for t in cov.one_level])
        one_idx = np.concatenate([np.asarray(t, dtype=np.int64) for t in cov.one_level])
        out.update({f"case{ci}_k": np.int64(k), f"case{ci}_seed": np.int64(seed),
                    f"case{ci}_centers": cov.centers, f"case{ci}_one_ptr": one_ptr,
                    f"case{ci}_one_idx": one_idx, f"case{ci}_fail": res})
        print(f"  region cover k={k} p={p}: failing regions {np.flatnonzero(res).tolist()} "
              f"codes {res[res > 0].tolist()}", flush=True)
    save("region_cover", **out)


def case_laplacian():
    """Graph-Laplacian preconditioned LBFGS (laplacian-m2 and laplacian-a6, cvt_core.py:192-240
    with SuperLU): x3 density, 4-pt rule, N=2562, 20 iterations each; plus one assembled matrix
    and a solve for the matrix/solve parity tests."""
    from scvtmesh import cvt_core as cc

    _DEPTH["d"] = 0
    z0 = geometry.random_sphere_points(2562, 0)
    out = {"z0": z0}
    for pert in ("m2", "a6"):
        ev = pipeline.MeshEvaluator(field_for("x3"), RULES["4pt"], laplacian=pert)
        crit = optimizer.StoppingCriteria(max_iterations=20, movement_tol=1e-300, grad_tol=1e-300,
                                          stall_tol=1e-300)
        res = optimizer.minimize(z0, f"laplacian-{pert}", ev, crit, corrections=7)
        print(f"  laplacian-{pert}: {len(res.records)} it, {res.fevals} fevals, "
              f"resets={res.resets}, reason={res.reason}", flush=True)
        out[f"{pert}_energy"] = np.array([r.energy for r in res.records])
        out[f"{pert}_fevals"] = np.array([-1 if r.fevals is None else r.fevals for r in res.records])
        out[f"{pert}_final_z"] = res.points
        r0 = ev.evaluate(z0)
        lap = r0.laplacian
        m = lap.perturbed.tocsr()
        out[f"{pert}_indptr"], out[f"{pert}_indices"], out[f"{pert}_data"] = m.indptr, m.indices, m.data
        rhs = np.random.default_rng(1).standard_normal((2562, 3))
        out[f"{pert}_rhs"], out[f"{pert}_x"] = rhs, lap.solve(rhs)
        ev.close()
    save("laplacian", **out)


CASES = {
    "rules": case_rules, "c1_eval": case_c1_eval, "density_eval": case_density_eval,
    "sampler": case_sampler, "medium": case_medium, "small_sets": case_small_sets,
    "traj_fast": case_traj_fast, "traj_slow": case_traj_slow,
    "traj_fallback": case_traj_fallback, "medium_slim": case_medium_slim,
    "run_ladder": case_run_ladder, "covering": case_covering, "laplacian": case_laplacian,
    "region_cover": case_region_cover,
}

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--skip-slow", action="store_true")
    a = ap.parse_args()
    names = a.only or [n for n in CASES if n != "medium" and not (a.skip_slow and n == "traj_slow")]
    print("scvtmesh", scvtmesh.__version__, "numpy", np.__version__, flush=True)
    for n in names:
        t0 = time.perf_counter()
        CASES[n]()
        print(f"[{n}] {time.perf_counter() - t0:.1f}s", flush=True)
