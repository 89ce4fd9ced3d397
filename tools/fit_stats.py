"""Host statistics of the k_quad fast-path decisions per fan sub-triangle (TEST-ONLY harness
tests/native/host_harness.cpp compiled for the CPU): fit accepted, 1/|x| series eligible,
two-centre dominance.  Triangulation from the harness cell builder."""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_06924_b200 import density as D  # noqa: E402
import paper_1709_06924_b200 as P  # noqa: E402

SRC = os.path.join(ROOT, "tests", "native", "host_harness.cpp")
SO = os.path.join(ROOT, "tests", "native", "libscvt_host_harness.so")
subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", SO, SRC], check=True)
h = ctypes.CDLL(SO)
Pp = ctypes.POINTER
dp = lambda a: a.ctypes.data_as(Pp(ctypes.c_double))  # noqa: E731
ip = lambda a: a.ctypes.data_as(Pp(ctypes.c_int))  # noqa: E731

for cfg, n in [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[1:]]:
    f = D.density_preset(cfg)
    z = np.ascontiguousarray(P.sample_by_density(f, n, 0))
    nbr = np.zeros((n, 32), np.int32)
    deg = np.zeros(n, np.int32)
    st = np.zeros(4, np.int32)
    h.harness_cells(dp(z), n, ip(nbr), ip(deg), ip(st))
    p = D.device_params(f)
    prm = np.zeros(15)
    prm[0:3] = [p["gamma"], p["beta"], p["alpha"]]
    prm[3:9] = p["center"]
    co, wd = p["table"]
    co = np.ascontiguousarray(co)
    kind = 7 if f.variant == "tanh4x2" else 6
    c = np.zeros(4, np.int64)
    h.harness_fit_stats(dp(z), n, ip(nbr), ip(deg), dp(co), co.shape[1] if co.ndim == 3 else len(co) // 2 // 7,
                        ctypes.c_double(wd), dp(prm), kind, c.ctypes.data_as(Pp(ctypes.c_longlong)))
    print(f"{cfg} n={n}: sub-triangles {c[1]}, fitted {c[0] / c[1]:.4f}, series {c[2] / c[1]:.4f}, "
          f"dominated {c[3] / c[1]:.4f}", flush=True)
