"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the SCVT energy/gradient + LBFGS hot path.

This package is a NumPy/SciPy restatement of the reference `scvtmesh` 0.1.0 path
(`/root/reference/pkg/src/scvtmesh`), every function citing the reference file:line it
follows.  It is the *checker*: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it.  The shipped package
`paper_1709_06924_b200` never imports it and fails loudly when its CUDA library is missing.

Parity pin: the oracle is checked against golden vectors produced by running the LIVE
reference in the build container (`tests/golden/make_golden.py`, fixtures in
`tests/golden/*.npz`; test `tests/test_oracle_golden.py`).  The triangulation goes through
the same third-party code as the reference: Qhull via `scipy.spatial.ConvexHull`
(SciPy 1.18.1, vendored qhull_r 8.0.2 "2020.2.r 2020/08/31").
"""

from .scvt_oracle import *  # noqa: F401,F403
