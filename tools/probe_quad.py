import ctypes, sys, torch
sys.path.insert(0, ".")
import paper_1709_06924_b200 as P
from paper_1709_06924_b200 import _lib
lib = _lib.load()
z = P.sample_by_density(P.density_preset("c4"), 655362, 0)
zt = torch.from_numpy(z).cuda()
with P.MeshEvaluator(P.density_preset("c4"), "7pt", subdivision=3) as ev:
    ev.evaluate_device(zt)
    lib.scvt_profile_enable(ev.context.ptr, 1)
    ms = (ctypes.c_double * 3)(); cnt = (ctypes.c_int64 * 3)()
    lib.scvt_profile_read(ev.context.ptr, ms, cnt, 1)
    for _ in range(3): ev.evaluate_device(zt)
    torch.cuda.synchronize(); lib.scvt_profile_read(ev.context.ptr, ms, cnt, 1)
print("quad_ms", ms[1] / cnt[1])
