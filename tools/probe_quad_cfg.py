"""k_quad and evaluation time for one config with the library named by SCVT_B200_LIB:
python tools/probe_quad_cfg.py CFG N [reps]  (scvt_profile counters, CUDA events)."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402
from paper_1709_06924_b200 import _lib  # noqa: E402

cfg, n = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
lib = _lib.load()
den = P.density_preset(cfg)
z = P.random_sphere_points(n, 0) if cfg == "const" else P.sample_by_density(den, n, 0)
zt = torch.from_numpy(z).cuda()
with P.MeshEvaluator(den, "7pt", subdivision=3) as ev:
    r0 = ev.evaluate_device(zt)
    lib.scvt_profile_enable(ev.context.ptr, 1)
    ms = (ctypes.c_double * 3)()
    cnt = (ctypes.c_int64 * 3)()
    lib.scvt_profile_read(ev.context.ptr, ms, cnt, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = ev.evaluate_device(zt)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps * 1e3
    lib.scvt_profile_read(ev.context.ptr, ms, cnt, 1)
print(f"{os.path.basename(os.environ.get('SCVT_B200_LIB', 'default'))} {cfg} N={n} "
      f"quad_ms={ms[1] / max(cnt[1], 1):.3f} cells_ms={ms[0] / max(cnt[0], 1):.3f} "
      f"eval_wall_ms={wall:.3f} E={r.energy!r} E0={r0.energy!r}")
