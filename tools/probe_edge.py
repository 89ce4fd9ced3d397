"""Edge-input probe: near-duplicate generators at shrinking separations, non-unit and float32
inputs, vs the oracle (moments) and Qhull (triangles)."""
import numpy as np
import oracle as O
import paper_1709_06924_b200 as P


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


base = P.random_sphere_points(10000, 5)
for sep in (1e-4, 1e-6, 1e-8, 1e-10, 1e-12):
    z = base.copy()
    t = np.cross(z[3], [0.0, 0.0, 1.0]); t /= np.linalg.norm(t)
    z[7] = z[3] + sep * t
    z[7] /= np.linalg.norm(z[7])
    try:
        o = O.Evaluator(O.density_for("const"), "7pt", 1).evaluate(z)
        oq = O.convex_hull_delaunay(z)
    except Exception as e:
        print(sep, "oracle", type(e).__name__, e); continue
    try:
        with P.MeshEvaluator(P.density_preset("const"), "7pt", subdivision=1) as ev:
            r = ev.evaluate(z)
            tq = ev.triangulation(z).triangles
        print(sep, "mass", rel(r.mass, o.mass), "first", rel(r.first, o.first),
              "tri_equal", np.array_equal(tq, oq), "mass37", o.mass[3], o.mass[7])
    except Exception as e:
        print(sep, "gpu", type(e).__name__, e)

z = base * 3.0
with P.MeshEvaluator(P.density_preset("const"), "7pt", subdivision=1) as ev:
    try:
        r = ev.evaluate(z); print("non-unit ok", r.energy)
    except Exception as e:
        print("non-unit", type(e).__name__, e)
    try:
        r2 = ev.evaluate(base.astype(np.float32)); print("f32 ok", r2.energy)
    except Exception as e:
        print("f32", type(e).__name__, e)
try:
    print("oracle non-unit", O.Evaluator(O.density_for("const"), "7pt", 1).evaluate(z).energy)
except Exception as e:
    print("oracle non-unit", type(e).__name__, e)
