import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1709_06924_b200 as P  # noqa: E402
g = np.load("tests/golden/traj_x64_4pt.npz")
crit = P.StoppingCriteria(max_iterations=40, movement_tol=1e-300, grad_tol=1e-300, stall_tol=1e-300)
with P.MeshEvaluator(P.density_preset("x64"), "4pt") as ev:
    res = P.minimize(g["z0"], "lloyd-plbfgs", ev, crit, corrections=7)
e = np.array([r.energy for r in res.records]); fe = [r.fevals for r in res.records]
st = np.array([r.step for r in res.records])
for k in range(len(e)):
    print(k + 1, f"{abs(e[k]-g['energy'][k])/g['energy'][k]:.2e}", fe[k], g["fevals"][k], f"{st[k]:.6g} {g['step'][k]:.6g}")
