"""Where the end-to-end minimize() time goes at c4: init evaluation, iterations, result
conversion, with and without the per-iteration position callback."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402

cfg, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
density = P.density_preset(cfg)
z0 = P.sample_by_density(density, n, 0)
host = torch.from_numpy(z0).pin_memory()
crit = P.StoppingCriteria(max_iterations=steps, movement_tol=1e-300, grad_tol=1e-300,
                          stall_tol=1e-300)
with P.MeshEvaluator(density, "7pt", subdivision=3) as ev:
    ev._ensure_ctx(n, 7)
    for label in ["minimize", "minimize(again)", "minimize(3)", "minimize(4)"]:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = P.minimize(host.cuda(non_blocking=True), "lloyd-plbfgs", ev, crit, corrections=7)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        per = [r.time_ms for r in res.records]
        print(f"{label}: wall {1e3 * (t1 - t0):.1f} ms for {steps} its -> "
              f"{steps * n / (t1 - t0):.3e} gen-upd/s; iteration sum {sum(per):.1f} ms; "
              f"first 4 {[round(p, 1) for p in per[:4]]} last {per[-1]:.1f}", flush=True)
    zt = torch.from_numpy(z0).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = P.Minimizer(zt, "lloyd-plbfgs", ev, 7)
    torch.cuda.synchronize()
    print(f"Minimizer init (normalize + first evaluation): {1e3 * (time.perf_counter() - t0):.1f} ms")

    # pieces of minimize(): init, loop, result conversion
    from paper_1709_06924_b200.optimizer import _to_host  # noqa: E402
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    zin = host.cuda(non_blocking=True)
    st = P.Minimizer(zin, "lloyd-plbfgs", ev, 7)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(steps):
        st.step()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    pts = st.z.cpu().numpy()
    t3 = time.perf_counter()
    fin = _to_host(st.res)  # noqa: F841
    t4 = time.perf_counter()
    print(f"init {1e3 * (t1 - t0):.1f} ms, loop {1e3 * (t2 - t1):.1f} ms, points D2H "
          f"{1e3 * (t3 - t2):.1f} ms, final D2H {1e3 * (t4 - t3):.1f} ms")
