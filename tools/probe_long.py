"""Per-window statistics over a long run: iteration time, cells/quad time per evaluation, flip
rounds and flips per repair, repairs that fell back to rebuilds.  Usage: CFG ITERS WINDOW"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

cfg, iters, win = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
RUNS = {"c3": (163842, 7), "c4": (655362, 7), "c5": (2621442, 10)}
n, m = RUNS[cfg]
den = P.density_preset(cfg)
z0 = P.sample_by_density(den, n, 0)
with P.MeshEvaluator(den, "7pt", subdivision=3) as ev:
    st = P.Minimizer(torch.from_numpy(z0).cuda(), "lloyd-plbfgs", ev, m)
    lib = ev.context.lib
    ptr = ev.context.ptr
    lib.scvt_profile_enable(ptr, 1)
    for w0 in range(0, iters, win):
        ms = (ctypes.c_double * 3)(); cnt = (ctypes.c_int64 * 3)()
        lib.scvt_profile_read(ptr, ms, cnt, 1)
        f = (ctypes.c_int64 * 4)(); lib.scvt_profile_flips(ptr, f, 1)
        c = (ctypes.c_int64 * 12)(); lib.scvt_profile_counters(ptr, c, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(win):
            st.step()
        e1.record(); torch.cuda.synchronize()
        lib.scvt_profile_read(ptr, ms, cnt, 0)
        lib.scvt_profile_flips(ptr, f, 0)
        lib.scvt_profile_counters(ptr, c, 0)
        print(f"iters {w0 + 1}-{w0 + win}: {e0.elapsed_time(e1) / win:.2f} ms/iter, cells "
              f"{ms[0] / max(cnt[0], 1):.2f} ms/eval, quad {ms[1] / max(cnt[1], 1):.2f}, "
              f"rounds/repair {f[1] / max(f[0], 1):.1f}, flips/repair {f[2] / max(f[0], 1):.0f}, "
              f"open {f[3]}/{f[0]}, rebuilt cells {c[9]}", flush=True)
