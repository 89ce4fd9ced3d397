"""GPU idle time per optimizer iteration: kernel timeline of a few steps via torch.profiler
(CUPTI), gaps between consecutive kernels summed and attributed to the preceding kernel."""
import collections
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

cfg, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
dens = {"c1": "const", "c2": "const"}.get(cfg, cfg)
z0 = torch.from_numpy(P.random_sphere_points(n, 0) if dens == "const"
                      else P.sample_by_density(P.density_preset(dens), n, 0)).cuda()
with P.MeshEvaluator(P.density_preset(dens), "7pt", subdivision=3) as ev:
    st = P.Minimizer(z0, "lloyd-plbfgs", ev, 7)
    for _ in range(4):
        st.step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            st.step()
        torch.cuda.synchronize()
ev_list = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev_list.sort(key=lambda e: e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in ev_list)
span = ev_list[-1].time_range.end - ev_list[0].time_range.start
gaps = collections.Counter()
for a, b in zip(ev_list, ev_list[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 0:
        gaps[a.name[:50]] += g
print(f"steps {steps}: span {span / steps / 1e3:.3f} ms/step, busy {busy / steps / 1e3:.3f}, "
      f"idle {(span - busy) / steps / 1e3:.3f} ms/step, kernels/step {len(ev_list) / steps:.0f}")
for k, v in gaps.most_common(15):
    print(f"  gap after {k:50s} {v / steps:8.1f} us/step")
busy_k = collections.Counter()
for e in ev_list:
    busy_k[e.name[:50]] += e.time_range.end - e.time_range.start
for k, v in busy_k.most_common(25):
    print(f"  busy {k:50s} {v / steps:8.1f} us/step")
