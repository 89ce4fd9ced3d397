"""Triangle churn between consecutive optimizer iterates (bench trajectory)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

cfg, n = sys.argv[1], int(sys.argv[2])
z = P.sample_by_density(P.density_preset(cfg), n, 0) if cfg != "const" else P.random_sphere_points(n, 0)
with P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3) as ev:
    st = P.Minimizer(torch.from_numpy(z).cuda(), "lloyd-plbfgs", ev, 7)
    prev = None
    for it in range(1, 13):
        st.step()
        tri, _, _ = ev.triangulate_device(st.z)
        t = tri.cpu().numpy()
        key = (t[:, 0] * n + t[:, 1]) * n + t[:, 2]
        if prev is not None:
            changed = len(np.setdiff1d(key, prev, assume_unique=True))
            verts = np.unique(t[~np.isin(key, prev)].ravel())
            print(f"iter {it}: triangles changed {changed} ({100 * changed / len(key):.2f}%), "
                  f"generators touched {len(verts)} ({100 * len(verts) / n:.2f}%)", flush=True)
        prev = key
