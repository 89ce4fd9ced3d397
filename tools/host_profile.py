"""Host-side profile of optimizer iterations (cProfile, cumulative) at a small config, where
the step is host-bound.    python tools/host_profile.py CFG N ITERS"""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

cfg, n, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
den = P.density_preset(cfg)
z0 = P.random_sphere_points(n, 0) if cfg == "const" else P.sample_by_density(den, n, 0)
with P.MeshEvaluator(den, "7pt", subdivision=3) as ev:
    st = P.Minimizer(torch.from_numpy(z0).cuda(), "lloyd-plbfgs", ev, 7)
    for _ in range(5):
        st.step()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(iters):
        st.step()
    pr.disable()
    torch.cuda.synchronize()
ps = pstats.Stats(pr)
ps.sort_stats("cumulative").print_stats(28)
