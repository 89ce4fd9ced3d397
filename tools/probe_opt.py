"""Host-side time per optimizer operation (each C call ends in a sync or is stream-ordered)."""
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402
from paper_1709_06924_b200 import optimizer as OPT  # noqa: E402

acc = defaultdict(float)
cnt = defaultdict(int)
for name in ("gamma", "direction", "direction_tangent", "tangent", "trial", "dirderiv", "minimum", "push", "lloyd"):
    f = getattr(OPT._DeviceOps, name)

    def wrap(self, *a, _f=f, _n=name):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = _f(self, *a)
        torch.cuda.synchronize()
        acc[_n] += time.perf_counter() - t
        cnt[_n] += 1
        return r
    setattr(OPT._DeviceOps, name, wrap)
ev_f = P.MeshEvaluator.evaluate_device


def ev_wrap(self, z, *a):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = ev_f(self, z, *a)
    torch.cuda.synchronize()
    acc["evaluate"] += time.perf_counter() - t
    cnt["evaluate"] += 1
    return r


P.MeshEvaluator.evaluate_device = ev_wrap
z = P.sample_by_density(P.density_preset("c4"), 655362, 0)
with P.MeshEvaluator(P.density_preset("c4"), "7pt", subdivision=3) as ev:
    st = P.Minimizer(torch.from_numpy(z).cuda(), "lloyd-plbfgs", ev, 7)
    for _ in range(4):
        st.step()
    acc.clear(); cnt.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        st.step()
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
for k in sorted(acc, key=lambda k: -acc[k]):
    print(f"{k:10s} calls/iter {cnt[k]/10:4.1f}  ms/iter {1e3*acc[k]/10:7.3f}")
print(f"total ms/iter {1e3*tot/10:.3f}  unaccounted {1e3*(tot-sum(acc.values()))/10:.3f}")
