"""Per-iteration time and reuse statistics over a window of a run: step ms (CUDA events),
evaluations, certified-by-reuse evaluations, certificate passes and rebuilt cells.
    python tools/probe_iter_stats.py CFG FIRST LAST"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

cfg, first, last = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
RUNS = {"c3": (163842, 7), "c4": (655362, 7), "c5": (2621442, 10)}
n, m = RUNS[cfg]
den = P.density_preset(cfg)
z0 = P.sample_by_density(den, n, 0)
with P.MeshEvaluator(den, "7pt", subdivision=3) as ev:
    st = P.Minimizer(torch.from_numpy(z0).cuda(), "lloyd-plbfgs", ev, m)
    lib, ctx = ev.context.lib, ev.context.ptr
    c = (ctypes.c_int64 * 12)()
    for it in range(1, last + 1):
        if it >= first:
            lib.scvt_profile_counters(ctx, c, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0 = st.fevals
            e0.record()
        rec = st.step()[0]
        if it >= first:
            e1.record()
            torch.cuda.synchronize()
            lib.scvt_profile_counters(ctx, c, 0)
            print(f"it {it}: {e0.elapsed_time(e1):7.2f} ms  evals {st.fevals - f0}  certified {c[8]}  "
                  f"passes {c[10]}  rebuilt {c[9]}  step {rec.step:g}")
