"""Host-side profile (cProfile) of optimizer iterations: where the Python/ctypes time goes
between GPU launches.  Usage: CFG N STEPS"""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

cfg, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
dens = {"c1": "const", "c2": "const"}.get(cfg, cfg)
z0 = torch.from_numpy(P.random_sphere_points(n, 0) if dens == "const"
                      else P.sample_by_density(P.density_preset(dens), n, 0)).cuda()
with P.MeshEvaluator(P.density_preset(dens), "7pt", subdivision=3) as ev:
    st = P.Minimizer(z0, "lloyd-plbfgs", ev, 7)
    for _ in range(5):
        st.step()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(steps):
        st.step()
    torch.cuda.synchronize()
    pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
