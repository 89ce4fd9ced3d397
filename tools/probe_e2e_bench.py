import sys, json
sys.path.insert(0, ".")
import torch
import bench
import paper_1709_06924_b200 as P
density = P.density_preset("c4")
z0 = P.sample_by_density(density, 655362, 0)
dev = torch.device("cuda", 0)
for k in range(3):
    r = bench._e2e(P, density, z0, 7, 20, dev, 1)
    print("with callback", f"{r['value']:.3e}", flush=True)
