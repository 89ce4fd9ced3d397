"""Per-iteration host wall time of a public minimize() call from the initial point (the bench's
e2e leg without callbacks): the initial evaluation, then each iteration's time_ms and the
reuse statistics.   python tools/probe_e2e_iters.py [ITERS]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
den = P.density_preset("c4")
n = 655362
z0 = P.sample_by_density(den, n, 0)
host = torch.from_numpy(z0).pin_memory()
for rep in range(2):
    with P.MeshEvaluator(den, "7pt", subdivision=3) as ev:
        ev._ensure_ctx(n, 7)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        zd = host.to("cuda", non_blocking=True)
        st = P.Minimizer(zd, "lloyd-plbfgs", ev, 7)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ts = []
        for _ in range(iters):
            a = time.perf_counter()
            rec = st.step()[0]
            ts.append((time.perf_counter() - a) * 1e3)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        r = P.optimizer._to_host(st.ops.full(st.res), st.z)
        t3 = time.perf_counter()
    if rep:
        print(f"H2D + initial evaluation {1e3 * (t1 - t0):.2f} ms; {iters} iterations "
              f"{1e3 * (t2 - t1):.2f} ms; final copy to host {1e3 * (t3 - t2):.2f} ms")
        print("per iteration ms:", " ".join(f"{t:.2f}" for t in ts))
