"""cProfile of the host side of the optimizer loop at a small (launch/host-bound) size."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

n, iters = int(sys.argv[1]), int(sys.argv[2])
z0 = torch.from_numpy(P.random_sphere_points(n, 0)).cuda()
with P.MeshEvaluator(P.density_preset("const"), "7pt", subdivision=3) as ev:
    st = P.Minimizer(z0, "lloyd-plbfgs", ev, 5)
    for _ in range(5):
        st.step()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(iters):
        st.step()
    torch.cuda.synchronize()
    pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
