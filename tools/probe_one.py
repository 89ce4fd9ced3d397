"""Probe one configuration: python tools/probe_one.py CFG N [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

cfg, n = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
z = P.random_sphere_points(n, 0) if cfg == "const" else P.sample_by_density(P.density_preset(cfg), n, 0)
zt = torch.from_numpy(z).cuda()
with P.MeshEvaluator(P.density_preset(cfg), "7pt", subdivision=3) as ev:
    for _ in range(reps):
        r = ev.evaluate_device(zt)
    torch.cuda.synchronize()
print("E", r.energy)
