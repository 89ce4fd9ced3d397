"""Why cells fail the reuse certificate along a trajectory (probe build with -DSCVT_PROBE_FLIPS):
per iteration the directed edges failing the in-circle test, triangles no longer facing
outward, and cycle inconsistencies.  Usage: SCVT_B200_LIB=tmpvar/lib_probe_flips.so CFG N ITERS"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402
from paper_1709_06924_b200 import _lib  # noqa: E402

lib = _lib.load()
lib.scvt_probe_flips.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
cfg, n, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
z = P.sample_by_density(P.density_preset(cfg), n, 0)
out = (ctypes.c_ulonglong * 3)()
with P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3) as ev:
    st = P.Minimizer(torch.from_numpy(z).cuda(), "lloyd-plbfgs", ev, 7)
    lib.scvt_probe_flips(out)
    for it in range(1, iters + 1):
        st.step()
        torch.cuda.synchronize()
        lib.scvt_probe_flips(out)
        print(f"iter {it}: incircle {out[0]} orientation {out[1]} inconsistent {out[2]}", flush=True)
