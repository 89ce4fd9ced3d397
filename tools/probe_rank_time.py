"""Per-rank time estimate of the sharded path at W GPUs on one GPU: the W shards of every
evaluation run back to back (emulate_shards); every backend call is timed with CUDA events
and attributed to its shard; per evaluation the estimate is sum over phases of the slowest
shard's time + the replicated calls (plan, install, finish), and per iteration + the LBFGS
algebra (replicated).  Communication is not included (volumes printed)."""
import collections
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402
from paper_1709_06924_b200 import parallel as PL  # noqa: E402

cfg, n, W, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
z0 = torch.from_numpy(P.sample_by_density(P.density_preset(cfg), n, 0)).cuda()


class Timed(PL.CudaShardBackend):
    def __init__(self, ev):
        super().__init__(ev)
        self.log = []          # (phase, shard, ms)

    def _t(self, phase, shard, fn, *a):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn(*a)
        e1.record()
        self.log.append((phase, shard, e0, e1))
        return r

    def cells(self, z, s, ns, buf):
        return self._t("cells", s, super().cells, z, s, ns, buf)

    def moments(self, z, s, ns, cyc, res):
        return self._t("moments", s, super().moments, z, s, ns, cyc, res)

    def recheck(self, z, s, ns, rnd, bad):
        return self._t(f"recheck{rnd}", s, super().recheck, z, s, ns, rnd, bad)

    def rebuild(self, n_, s, ns, cap, rows):
        return self._t("rebuild", s, super().rebuild, n_, s, ns, cap, rows)

    def plan(self, n_, ns, bad):
        return self._t("plan", -1, super().plan, n_, ns, bad)

    def install(self, n_, rows, nr):
        return self._t("install", -1, super().install, n_, rows, nr)

    def finish(self, z, ns, res, q3=None, norms=None):
        if q3 is None:
            return self._t("finish", -1, super().finish, z, ns, res)
        return self._t("finish", -1, super().finish, z, ns, res, q3, norms)


class Ev(P.MeshEvaluator):
    def evaluate_device(self, z, q3=None, norms=None):
        r = PL.emulate_shards(self.backend, z, W, q3, norms)
        self.evaluations += 1
        return r


with Ev(P.density_preset(cfg), "7pt", subdivision=3) as ev:
    ev.backend = Timed(ev)
    st = P.Minimizer(z0, "lloyd-plbfgs", ev, 7)
    for _ in range(3):
        st.step()
    torch.cuda.synchronize()
    ev.backend.log.clear()
    t0 = time.perf_counter()
    e_it0, e_it1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_it0.record()
    for _ in range(iters):
        st.step()
    e_it1.record()
    torch.cuda.synchronize()
    total = e_it0.elapsed_time(e_it1) / iters
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for ph, s, a, b in ev.backend.log:
        per[ph][s] += a.elapsed_time(b)
    in_backend = sum(sum(d.values()) for d in per.values()) / iters
    est = 0.0
    for ph, d in per.items():
        worst = max(d.values()) / iters
        est += worst
        print(f"  {ph:9s} slowest shard {worst:7.3f} ms/iter  (all shards {sum(d.values()) / iters:7.3f})"
              + (f"  per shard {[round(v / iters, 3) for k, v in sorted(d.items())]}" if ph == "moments" else ""))
    other = total - in_backend          # LBFGS algebra, trial points, host: replicated
    print(f"W={W}: one-GPU emulation {total:.2f} ms/iter; estimated per-rank {est + other:.2f} "
          f"ms/iter (+ communication) = {total / (est + other):.2f}x of the emulated work")
    n_ = n
    print(f"per evaluation exchange volumes: bad flags {4 * n_ / 1e6:.1f} MB all-reduce, "
          f"results {8 * 8 * n_ / 1e6:.1f} MB all-gather, rebuilt cycles 136 B per rebuilt cell")
