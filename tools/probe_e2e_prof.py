"""cProfile of one cold 1-iteration minimize() at c4 (after the API warm-up), to find the
fixed part of the e2e wall time."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1709_06924_b200 as P  # noqa: E402

dev = torch.device("cuda:0")
density = P.density_preset("c4")
z0 = P.sample_by_density(density, 655362, 0)
bench._e2e(P, density, z0, 7, 2, dev, 1)          # warm-up everything once
host = torch.from_numpy(z0).pin_memory()
crit = P.StoppingCriteria(max_iterations=1, movement_tol=1e-300, grad_tol=1e-300, stall_tol=1e-300)
with P.MeshEvaluator(density, "7pt", subdivision=3) as ev:
    ev._ensure_ctx(len(z0), 7)
    torch.cuda.synchronize()
    zdev = host.to(dev, non_blocking=True)
    t0 = time.perf_counter()
    r0 = ev.evaluate_device(zdev.clone())
    torch.cuda.synchronize()
    print(f"cold evaluate_device {1e3 * (time.perf_counter() - t0):.2f} ms")
    t0 = time.perf_counter()
    r0 = ev.evaluate_device(zdev.clone())
    torch.cuda.synchronize()
    print(f"same points again (reuse) {1e3 * (time.perf_counter() - t0):.2f} ms")
with P.MeshEvaluator(density, "7pt", subdivision=3) as ev:
    ev._ensure_ctx(len(z0), 7)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    zdev = host.to(dev, non_blocking=True)
    res = P.minimize(zdev, "lloyd-plbfgs", ev, crit, corrections=7)
    torch.cuda.synchronize()
    pr.disable()
    print(f"minimize 1 iteration {1e3 * (time.perf_counter() - t0):.2f} ms, fevals {res.fevals}")
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
