"""Full-size BASELINE goldens from the LIVE reference (c2-c5 at their own N), VERDICT r1 item 1.

Run in the build container only (needs /root/reference; hours of CPU):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_fullsize.py --cfg c2 [--workers 8]

Same injections as `make_golden.py` (7-point Radon rule, depth-3 subdivision inside the
evaluator, tanh^4 / two-centre densities; DECISIONS.md D1-D4), imported from there.  The only
difference is speed: the subdivided `cell_quadrature` wrapper farms contiguous blocks of
16,384-sub-triangle chunks out to a fork pool (the fans are inherited copy-on-write) and sums
the blocks' outputs in block order.  Every leaf is integrated by the reference's own
`cell_quadrature` (cvt_core.py:55-117) exactly as in the serial wrapper; only the grouping of
the final sum differs (rounding level, far inside DECISIONS.md D7).  The evaluator is the
reference's global path (`MeshEvaluator`, pipeline.py:206-215, 261-279) driven by the
reference's unmodified `optimizer.minimize` (optimizer.py:278-391).

Fixtures are compact (a 2048-row deterministic sample of every per-generator array plus
aggregate sums), so they can be committed:

* `full_<cfg>.npz`: evaluation 0 at z0 (energy, grad_norm, sums, sampled mass/first/grad/
  lloyd_diag rows, triangle digest and count), then per iteration energy/grad_norm/step/
  fevals, the energy of EVERY evaluation (line-search trials included), sampled rows of the
  iterate at the snapshot iterations, and aggregate sums of every snapshot.
"""

from __future__ import annotations

import argparse
import hashlib
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as MG  # noqa: E402  (installs the injections)
from scvtmesh import delaunay, density as dmod, geometry, optimizer, pipeline  # noqa: E402

SAMPLE = 2048
CFG = {
    # name: (N, density cfg, corrections, iterations, snapshot iterations)
    "c2": (40962, "const", 7, 100, (1, 2, 3, 5, 10, 20, 50, 100)),
    "c3": (163842, "c3", 7, 3, (1, 2, 3)),
    "c4": (655362, "c4", 7, 3, (1, 2, 3)),
    "c5": (2621442, "c5", 10, 3, (1, 2, 3)),
}

_W = {"fans": None, "z": None, "field": None, "k": 0}
WORKERS = 8


def sample_ids(n):
    """Deterministic sorted sample of generator ids (the GPU tests use the same call)."""
    return np.sort(np.random.default_rng(12345).choice(n, size=min(SAMPLE, n), replace=False))


def _block(args):
    lo, hi = args
    fans, z, k = _W["fans"], _W["z"], _W["k"]
    mass = np.zeros(k)
    first = np.zeros((k, 3))
    energy = 0.0
    for s in range(lo, hi, MG.CHUNK):
        e = min(hi, s + MG.CHUNK)
        sub = delaunay.VoronoiFans(fans.verts[s:e], fans.cells[s:e], fans.edge_other[s:e],
                                   fans.signed_area[s:e], fans.obtuse_count)
        sub = delaunay.subdivide_fans(sub, MG._DEPTH["d"])
        m, c, en, _, _ = MG._ORIG_CQ(z, sub, _W["field"], MG.RULES["7pt"], k)
        mass += m
        first += c
        energy += en
    ids = np.unique(fans.cells[lo:hi])
    return ids, mass[ids], first[ids], energy


def _cq_parallel(points, fans, density, rule, k, with_pairs=False, measure="flat"):
    assert not with_pairs and measure == "flat" and rule is MG.RULES["7pt"]
    S = len(fans.cells)
    nblk = max(1, min(8 * WORKERS, S // MG.CHUNK))
    per = -(-S // nblk)
    per = -(-per // MG.CHUNK) * MG.CHUNK
    blocks = [(s, min(S, s + per)) for s in range(0, S, per)]
    _W.update(fans=fans, z=np.asarray(points, dtype=float), field=density, k=k)
    with mp.get_context("fork").Pool(WORKERS) as pool:
        parts = pool.map(_block, blocks, chunksize=1)
    mass = np.zeros(k)
    first = np.zeros((k, 3))
    energy = 0.0
    for ids, m, c, en in parts:
        mass[ids] += m
        first[ids] += c
        energy += en
    _W.update(fans=None, z=None)
    return mass, first, energy, None, None


class RecordingEvaluator(pipeline.MeshEvaluator):
    """The reference's global-path evaluator, recording every evaluation's energy."""

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        self.log = []
        self.first_result = None
        self.first_tri = None

    def _global_result(self, points, want_triangles):
        out = super()._global_result(points, True)
        if self.first_tri is None:
            self.first_tri = out[4].triangles.copy()
        return out

    def evaluate(self, points):
        t0 = time.perf_counter()
        r = super().evaluate(points)
        self.log.append(r.energy)
        if self.first_result is None:
            self.first_result = r
        print(f"    eval {len(self.log)}: E={r.energy:.17e} |g|={r.grad_norm:.6e} "
              f"{time.perf_counter() - t0:.1f}s", flush=True)
        return r


def run(cfg, out_dir):
    n, dcfg, m, iters, snaps = CFG[cfg]
    if dcfg == "const":
        z0 = geometry.random_sphere_points(n, 0)
    else:
        z0 = dmod.sample_by_density(MG.field_for(dcfg), n, 0)
    ids = sample_ids(n)
    MG._DEPTH["d"] = 3
    pipeline.cell_quadrature = _cq_parallel
    ev = RecordingEvaluator(MG.field_for(dcfg), MG.RULES["7pt"])
    crit = optimizer.StoppingCriteria(max_iterations=iters, movement_tol=1e-300,
                                      grad_tol=1e-300, stall_tol=1e-300)
    kept = {}

    def cb(it, z, res):
        if it in snaps:
            kept[it] = (z.copy(), res)
        print(f"  iter {it}: E={res.energy:.17e}", flush=True)

    t0 = time.perf_counter()
    res = optimizer.minimize(z0, "lloyd-plbfgs", ev, crit, corrections=m, callback=cb)
    wall = time.perf_counter() - t0
    r0 = ev.first_result
    out = {
        "n": np.int64(n), "density": np.array(dcfg), "corrections": np.int64(m),
        "sample_ids": ids, "z0_sample": z0[ids], "z0_sum": z0.sum(axis=0),
        "z0_sha": np.array(hashlib.sha256(np.ascontiguousarray(z0).tobytes()).hexdigest()),
        "tri_sha": np.array(MG.tri_digest(ev.first_tri)), "tri_count": np.int64(len(ev.first_tri)),
        "e0_energy": np.float64(r0.energy), "e0_grad_norm": np.float64(r0.grad_norm),
        "e0_first_sum": r0.first.sum(axis=0), "e0_first_sq": np.float64((r0.first ** 2).sum()),
        "e0_diag_sum": np.float64(r0.lloyd_diag.sum()),
        "e0_first": r0.first[ids], "e0_grad": r0.grad[ids], "e0_lloyd_diag": r0.lloyd_diag[ids],
        "energy": np.array([r.energy for r in res.records]),
        "grad_norm": np.array([r.grad_norm for r in res.records]),
        "step": np.array([r.step for r in res.records]),
        "fevals": np.array([-1 if r.fevals is None else r.fevals for r in res.records]),
        "eval_energy": np.array(ev.log), "reason": np.array(res.reason),
        "resets": np.int64(res.resets), "fevals_total": np.int64(res.fevals),
        "snap_iters": np.array(sorted(kept)), "wall_s": np.float64(wall),
    }
    for it, (z, r) in kept.items():
        out[f"z_{it}"] = z[ids]
        out[f"z_{it}_sum"] = z.sum(axis=0)
        out[f"g_{it}"] = r.grad[ids]
        out[f"first_{it}_sum"] = r.first.sum(axis=0)
    path = os.path.join(out_dir, f"full_{cfg}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB) in {wall:.0f}s; "
          f"{len(res.records)} it, {res.fevals} fevals, reason={res.reason}", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", nargs="+", required=True)
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=HERE)
    ap.add_argument("--iters", type=int, default=None, help="override (smoke runs)")
    a = ap.parse_args()
    WORKERS = a.workers
    for c in a.cfg:
        if a.iters is not None:
            n, d, mm, _, sn = CFG[c]
            CFG[c] = (n, d, mm, a.iters, tuple(s for s in sn if s <= a.iters))
        run(c, a.out)
