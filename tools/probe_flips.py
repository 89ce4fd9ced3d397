"""Flip-repair statistics along a trajectory: evaluations, rounds, flips, fallbacks to the
rebuild path (scvt_profile_flips) and the cells time per evaluation.
    python tools/probe_flips.py CFG N ITERS"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402
from paper_1709_06924_b200 import _lib  # noqa: E402

cfg, n, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
den = P.density_preset(cfg)
z0 = P.random_sphere_points(n, 0) if cfg == "const" else P.sample_by_density(den, n, 0)
lib = _lib.load()
with P.MeshEvaluator(den, "7pt", subdivision=3) as ev:
    st = P.Minimizer(torch.from_numpy(z0).cuda(), "lloyd-plbfgs", ev, 7)
    for _ in range(3):
        st.step()
    ctx = ev.context
    f = (ctypes.c_int64 * 4)()
    lib.scvt_profile_flips(ctx.ptr, f, 1)
    lib.scvt_profile_enable(ctx.ptr, 1)
    ms = (ctypes.c_double * 3)()
    cnt = (ctypes.c_int64 * 3)()
    lib.scvt_profile_read(ctx.ptr, ms, cnt, 1)
    for _ in range(iters):
        st.step()
    torch.cuda.synchronize()
    lib.scvt_profile_flips(ctx.ptr, f, 1)
    lib.scvt_profile_read(ctx.ptr, ms, cnt, 1)
print(f"{cfg} N={n}: {f[0]} repairs, {f[1] / max(f[0], 1):.2f} rounds/repair, "
      f"{f[2] / max(f[0], 1):.0f} flips/repair, {f[3]} left open; cells "
      f"{ms[0] / max(cnt[0], 1):.3f} ms/eval; E={st.res.energy!r}")
