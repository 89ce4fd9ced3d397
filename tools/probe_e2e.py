"""Split the e2e wall time of bench.py's public-API leg into a fixed part and a per-iteration
part: minimize() at several iteration counts, linear fit."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1709_06924_b200 as P  # noqa: E402

dev = torch.device("cuda:0")
density = P.density_preset("c4")
n = 655362
z0 = P.sample_by_density(density, n, 0)
rows = []
for steps in (1, 2, 5, 10, 20, 40):
    v = bench._e2e(P, density, z0, 7, steps, dev, 1)["value"]
    wall = steps * n / v
    rows.append((steps, wall))
    print(f"steps {steps:3d}  wall {wall * 1e3:8.2f} ms  per-iter {wall / steps * 1e3:6.2f} ms", flush=True)
s, w = np.array(rows).T
k, c = np.polyfit(s[2:], w[2:], 1)
print(f"fit (steps>=5): {k * 1e3:.3f} ms/iteration + {c * 1e3:.2f} ms fixed")
