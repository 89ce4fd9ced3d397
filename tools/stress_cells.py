"""Adversarial inputs for the cell builder + certificate, checked against Qhull (oracle):
steep density, a dense cluster in a sparse background, a jittered icosahedral lattice (near
cocircular everywhere), a great-circle band.  Prints triangles-equal / flagged / timing."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_1709_06924_b200 as P  # noqa: E402


def normalize(a):
    return a / np.linalg.norm(a, axis=1, keepdims=True)


def cases():
    rng = np.random.default_rng(3)
    yield "x64 655k", P.sample_by_density(P.density_preset("x64"), 655362, 0)
    c = normalize(np.array([[0.3, -0.5, 0.8]]))
    t = rng.standard_normal((65536, 3)) * 0.05
    clus = normalize(c + t - (t @ c.T) * c)
    yield "cluster 65k in 0.05 rad + 200k background", np.vstack([clus, P.random_sphere_points(200000, 1)])
    z = P.icosahedron_vertices()
    with P.MeshEvaluator(P.density_preset("const"), "4pt") as ev:
        while len(z) < 655362:
            z = P.bisect(z, ev.triangulation(z))
    yield "icosahedral 655k exact (cocircular ties)", z
    yield "icosahedral 655k jittered 1e-9", normalize(z + 1e-9 * rng.standard_normal(z.shape))
    band = rng.standard_normal((300000, 3))
    band[:, 2] *= 0.01
    yield "great-circle band 300k", normalize(band)


for name, z in cases():
    zt = torch.from_numpy(np.ascontiguousarray(z)).cuda()
    with P.MeshEvaluator(P.density_preset("const"), "7pt", subdivision=3) as ev:
        try:
            torch.cuda.synchronize(); t0 = time.perf_counter()
            tri, flags, stats = ev.triangulate_device(zt)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
            t_gpu = ev.triangulation(zt).triangles
        except Exception as exc:            # noqa: BLE001
            print(f"{name}: GPU raised {type(exc).__name__}: {exc}", flush=True)
            continue
    t0 = time.perf_counter()
    try:
        ref = O.convex_hull_delaunay(z)
        eq = np.array_equal(t_gpu, ref)
    except Exception as exc:                # noqa: BLE001
        eq = f"qhull raised {type(exc).__name__}"
    print(f"{name}: n={len(z)} equal_to_qhull={eq} flagged={stats['flagged']} "
          f"tie_breaks={stats['tie_breaks']} max_passes={stats['max_passes']} "
          f"sweep_cells={stats['sweep_cells']} gpu {dt * 1e3:.1f} ms (qhull {time.perf_counter() - t0:.1f} s)",
          flush=True)
