"""Cell-builder time per evaluation along the bench trajectory, with/without cycle reuse."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402
from paper_1709_06924_b200 import _lib  # noqa: E402

lib = _lib.load()
cfg, n = sys.argv[1], int(sys.argv[2])
z = P.sample_by_density(P.density_preset(cfg), n, 0) if cfg != "const" else P.random_sphere_points(n, 0)
with P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3) as ev:
    st = P.Minimizer(torch.from_numpy(z).cuda(), "lloyd-plbfgs", ev, 7)
    lib.scvt_profile_enable(ev.context.ptr, 1)
    for it in range(1, 1 + (int(sys.argv[3]) if len(sys.argv) > 3 else 12)):
        c = (ctypes.c_int64 * 12)()
        lib.scvt_profile_counters(ev.context.ptr, c, 1)
        fl = (ctypes.c_int64 * 4)()
        lib.scvt_profile_flips(ev.context.ptr, fl, 1)
        ms = (ctypes.c_double * 3)(); cnt = (ctypes.c_int64 * 3)()
        lib.scvt_profile_read(ev.context.ptr, ms, cnt, 1)
        st.step()
        torch.cuda.synchronize()
        lib.scvt_profile_counters(ev.context.ptr, c, 0)
        lib.scvt_profile_read(ev.context.ptr, ms, cnt, 0)
        lib.scvt_profile_flips(ev.context.ptr, fl, 0)
        print(f"iter {it}: evals {cnt[2]} cells_ms/eval {ms[0]/max(cnt[0],1):.2f} quad_ms/eval "
              f"{ms[1]/max(cnt[1],1):.2f} eval_ms {ms[2]/max(cnt[2],1):.2f} reused {c[8]} cert_passes {c[10]} "
              f"flips {fl[2]} in {fl[1]} rounds (open {fl[3]}) rebuilt cells {c[9]} max_sweep_batches {c[6]} max_clips {c[7]} max_scanned {c[11] & ((1 << 40) - 1)} max_passes {c[11] >> 40}", flush=True)
