"""Cell-builder work counters per configuration."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402
from paper_1709_06924_b200 import _lib  # noqa: E402

os.environ.setdefault("SCVT_NO_REUSE", "1")   # time full builds
lib = _lib.load()
for cfg, n in [("const", 40962), ("const", 655362), ("c4", 655362)]:
    z = P.random_sphere_points(n, 0) if cfg == "const" else P.sample_by_density(P.density_preset(cfg), n, 0)
    zt = torch.from_numpy(z).cuda()
    with P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3) as ev:
        ev.evaluate_device(zt)
        ctx = ev.context
        lib.scvt_profile_enable(ctx.ptr, 1)
        c = (ctypes.c_int64 * 12)()
        lib.scvt_profile_counters(ctx.ptr, c, 1)
        ev.evaluate_device(zt)
        torch.cuda.synchronize()
        lib.scvt_profile_counters(ctx.ptr, c, 1)
        ms = (ctypes.c_double * 3)()
        cnt = (ctypes.c_int64 * 3)()
        lib.scvt_profile_read(ctx.ptr, ms, cnt, 1)
    cells = max(c[0], 1)
    print(f"{cfg} n={n}: cells_ms={ms[0]:.2f} per cell: passes {c[1]/cells:.2f} scanned {c[2]/cells:.1f} "
          f"cands {c[3]/cells:.1f} clips {c[4]/cells:.1f} rounds {c[5]/cells:.2f} max_sweep_batches {c[6]} max_clips {c[7]}", flush=True)
