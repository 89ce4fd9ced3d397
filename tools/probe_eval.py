"""Quick timing probe: one evaluation / triangulation at a few sizes (CUDA events)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts)


for cfg, n in [("const", 2562), ("const", 40962), ("c4", 163842), ("c4", 655362)]:
    t0 = time.time()
    z = P.random_sphere_points(n, 0) if cfg == "const" else P.sample_by_density(P.density_preset(cfg), n, 0)
    zt = torch.from_numpy(z).cuda()
    with P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3) as ev:
        tt = timed(lambda: ev.triangulate_device(zt))
        te = timed(lambda: ev.evaluate_device(zt))
        _, _, st = ev.triangulate_device(zt)
    print(f"{cfg} n={n}: triangulate {tt:.3f} ms, evaluate {te:.3f} ms, stats {st}, setup {time.time()-t0:.1f}s", flush=True)
