"""Per-iteration time of the sharded evaluator (world size 1 = the sharded code path with no
communication) against the single-GPU evaluator along the bench trajectory."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402
from paper_1709_06924_b200.parallel import ShardedMeshEvaluator  # noqa: E402

cfg, n, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
z0 = torch.from_numpy(P.sample_by_density(P.density_preset(cfg), n, 0)).cuda()
for name, cls in [("single", P.MeshEvaluator), ("sharded", ShardedMeshEvaluator)]:
    with cls(P.density_preset(cfg), "7pt", subdivision=3) as ev:
        st = P.Minimizer(z0, "lloyd-plbfgs", ev, 7)
        for _ in range(3):
            st.step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(iters):
            st.step()
        torch.cuda.synchronize()
        print(name, f"{(time.perf_counter() - t0) / iters * 1e3:.2f} ms/iter", flush=True)
