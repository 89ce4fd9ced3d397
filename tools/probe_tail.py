"""Cell-builder tail along the bench trajectory: per iteration, a fresh triangulation's stats
(max candidate passes, sweep cells) and its time, next to the reuse path's time."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

cfg, n, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
z = P.sample_by_density(P.density_preset(cfg), n, 0)
with P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3) as ev, \
        P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3) as ev2:
    st = P.Minimizer(torch.from_numpy(z).cuda(), "lloyd-plbfgs", ev, 7)
    for it in range(iters):
        st.step()
        x = st.z.clone()
        for rep in range(2):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            tri, flags, stats = ev2.triangulate_device(x)
            torch.cuda.synchronize(); t1 = time.perf_counter()
        print(it, f"{(t1 - t0) * 1e3:.2f} ms", stats, flush=True)
