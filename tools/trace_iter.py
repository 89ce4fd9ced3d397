"""Per-iteration timeline of the optimizer loop (torch.profiler / CUPTI): wall time per
iteration, GPU-busy time, idle gaps, kernel launches and host syncs, top kernels.

    python tools/trace_iter.py CFG [WARM] [ITERS]      (CFG: c1..c5; defaults 5 warm-up, 10)
Writes gpurun_out/trace_<cfg>.json (chrome trace) when run under gpurun."""
import collections
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_06924_b200 as P  # noqa: E402

CFG = {"c1": (2562, "const", 5), "c2": (40962, "const", 7), "c3": (163842, "c3", 7),
       "c4": (655362, "c4", 7), "c5": (2621442, "c5", 10)}
cfg = sys.argv[1]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 5
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
n, dname, m = CFG[cfg]
dens = P.density_preset(dname)
z0 = P.sample_by_density(dens, n, 0)
ev = P.MeshEvaluator(dens, "7pt", subdivision=3)
st = P.Minimizer(torch.from_numpy(z0).cuda(), "lloyd-plbfgs", ev, m)
for _ in range(warm):
    st.step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

fev0 = st.fevals
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    for _ in range(iters):
        st.step()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
evs = prof.events()
kern = [e for e in evs if e.device_type == torch.autograd.DeviceType.CUDA]
busy = 0.0
ivs = sorted((e.time_range.start, e.time_range.end) for e in kern)
cur_s, cur_e = None, None
for s_, e_ in ivs:
    if cur_e is None or s_ > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s_, e_
    else:
        cur_e = max(cur_e, e_)
if cur_e is not None:
    busy += cur_e - cur_s
by = collections.defaultdict(lambda: [0, 0.0])
for e in kern:
    by[e.name][0] += 1
    by[e.name][1] += e.time_range.elapsed_us()
syncs = sum(1 for e in evs if "Synchronize" in e.name)
launches = sum(1 for e in evs if e.name in ("cudaLaunchKernel", "cuLaunchKernel", "cudaLaunchKernelExC"))
memcpy = sum(1 for e in evs if "Memcpy" in e.name and e.device_type != torch.autograd.DeviceType.CUDA)
print(f"{cfg}: N={n} {iters} iterations, {(st.fevals - fev0) / iters:.2f} evals/iter: "
      f"wall {wall / iters * 1e3:.3f} ms/iter, GPU busy {busy / iters / 1e3:.3f} ms/iter "
      f"({busy / (wall * 1e6):.0%}), launches {launches / iters:.1f}/iter, "
      f"syncs {syncs / iters:.1f}/iter, memcpy calls {memcpy / iters:.1f}/iter")
for name, (c, us) in sorted(by.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {us / iters:9.1f} us/iter  {c / iters:5.1f}x  {name[:110]}")
api = collections.defaultdict(lambda: [0, 0.0])
for e in evs:
    if e.device_type != torch.autograd.DeviceType.CUDA and e.name.startswith("cuda"):
        api[e.name][0] += 1
        api[e.name][1] += e.time_range.elapsed_us()
print("  host CUDA API:")
for name, (c, us) in sorted(api.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {us / iters:9.1f} us/iter  {c / iters:5.1f}x  {name}")
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(f"gpurun_out/trace_{cfg}.json")
