"""Per-rank time estimate of the multi-GPU path at W GPUs, on one GPU.

The W shards of every evaluation run back to back (emulate_shards); every backend call is
timed with CUDA events and attributed to its shard; per evaluation the estimate takes, per
phase, the slowest shard (plan and install are replicated).  The arithmetic-layout work of one
rank (parallel.SliceOps: two-loop, trial points, history push, and the sliced finish) is timed
on a shadow context that follows the real trajectory with rank 0's slice and no exchange.
Communication is not included (volumes printed).  Usage: CFG N W ITERS"""
import collections
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402
from paper_1709_06924_b200 import parallel as PL  # noqa: E402

cfg, n, W, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
z0 = torch.from_numpy(P.sample_by_density(P.density_preset(cfg), n, 0)).cuda()
LOG = []   # (phase, shard, e0, e1)


def timed(phase, shard, fn, *a):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = fn(*a)
    e1.record()
    LOG.append((phase, shard, e0, e1))
    return r


class Timed(PL.CudaShardBackend):
    shadow = None

    def cells(self, z, s, ns, buf):
        return timed("cells", s, super().cells, z, s, ns, buf)

    def moments(self, z, s, ns, cyc, res):
        return timed("moments", s, super().moments, z, s, ns, cyc, res)

    def recheck(self, z, s, ns, rnd, bad):
        return timed(f"recheck{rnd}", s, super().recheck, z, s, ns, rnd, bad)

    def rebuild(self, n_, s, ns, cap, rows):
        return timed("rebuild", s, super().rebuild, n_, s, ns, cap, rows)

    def flip_detect(self, z, s, ns):
        return timed("flip_detect", s, super().flip_detect, z, s, ns)

    def flip_rounds(self, z, ns, cand, cap, counts):
        return timed("flip_rounds", -1, super().flip_rounds, z, ns, cand, cap, counts)

    def plan(self, n_, ns, bad):
        return timed("plan", -1, super().plan, n_, ns, bad)

    def install(self, n_, rows, nr):
        return timed("install", -1, super().install, n_, rows, nr)

    def finish(self, z, ns, res, q3=None, norms=None):
        r = super().finish(z, ns, res) if q3 is None else super().finish(z, ns, res, q3, norms)
        if self.shadow is not None:        # this rank's sliced finish on the same exchange rows
            sh = self.shadow
            q3s = None if q3 is None else q3[sh.lo:sh.hi].contiguous()
            ns_ = None if norms is None else norms[sh.lo:sh.hi].contiguous()
            timed("finish_slice", 0, sh.backend.finish_slice, z, ns, res, 0, W, sh.red,
                  lambda t: None, q3s, ns_)
        return r


class Ev(P.MeshEvaluator):
    def evaluate_device(self, z, q3=None, norms=None):
        r = PL.emulate_shards(self.backend, z, W, q3, norms)
        self.evaluations += 1
        return r


with Ev(P.density_preset(cfg), "7pt", subdivision=3) as ev, \
        P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3) as shadow_ev:
    ev.backend = Timed(ev)
    st = P.Minimizer(z0, "lloyd-plbfgs", ev, 7)
    sctx = shadow_ev._ensure_ctx(n, 7)
    ops = PL.SliceOps(sctx, n, 0, W, reduce_sum=lambda t: None, gather=lambda full: full)
    ops.backend = PL.CudaShardBackend(shadow_ev)
    lo, hi = ops.lo, ops.hi
    for it in range(3 + iters):
        if it == 3:
            torch.cuda.synchronize()
            LOG.clear()
            ev.backend.shadow = ops
            e_it0 = torch.cuda.Event(enable_timing=True)
            e_it0.record()
        z, res = st.z, st.res
        rec, _, z_new, res_new = st.step()
        if it >= 3:                                  # rank 0's arithmetic-layout algebra
            g_s, d_s = res.grad[lo:hi].contiguous(), res.lloyd_diag[lo:hi].contiguous()
            q3 = ops.vec3(z)
            gamma = ops.gamma()
            timed("algebra", 0, ops.direction_tangent, g_s, d_s, gamma, z, q3)
            for _ in range(rec.fevals or 1):
                zt = ops.positions(z)
                timed("algebra", 0, ops.trial, z, q3, 0.5, zt, ops.scalars(z))
            timed("algebra", 0, ops.push, z, z_new, g_s, res_new.grad[lo:hi].contiguous())
    e_it1 = torch.cuda.Event(enable_timing=True)
    e_it1.record()
    torch.cuda.synchronize()
    total = e_it0.elapsed_time(e_it1) / iters
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for ph, s, a, b in LOG:
        per[ph][s] += a.elapsed_time(b)
    est = 0.0
    for ph, d in per.items():
        worst = max(d.values()) / iters
        est += worst
        print(f"  {ph:12s} slowest shard {worst:7.3f} ms/iter  (all shards {sum(d.values()) / iters:7.3f})"
              + (f"  per shard {[round(v / iters, 3) for k, v in sorted(d.items())]}" if ph == "moments" else ""))
    print(f"W={W}: emulation (all shards + shadow) {total:.2f} ms/iter; per-rank device time "
          f"{est:.2f} ms/iter (+ host round trips and communication)")
    print(f"per evaluation exchange volumes: positions {24 * n / 1e6:.1f} MB all-gather, bad flags "
          f"{4 * n / 1e6:.1f} MB all-reduce, results {8 * 8 * n / 1e6:.1f} MB all-gather, "
          f"rebuilt cycles 136 B per rebuilt cell, chunk partials <= {8 * 176 * 1184 / 1e6:.1f} MB")
