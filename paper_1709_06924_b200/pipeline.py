"""GPU `MeshEvaluator` — drop-in for `scvtmesh.pipeline.MeshEvaluator` (pipeline.py:101-286).

One evaluation = spherical Delaunay by per-generator Voronoi-cell clipping on a cube-map
bucket grid + Voronoi fans + depth-d subdivided quadrature of rho + gradient epilogue, all in
sm_100a kernels behind the C ABI (include/scvt_b200.h).  The reference's worker pool and
covering (pipeline.py:131-242) have no analogue here: one GPU evaluates every cell in one
pass (multi-GPU sharding lives in `parallel.py`).  Returned arrays are NumPy when the input
is NumPy (drop-in) and CUDA tensors when the input is a CUDA tensor (zero-copy, used by
`optimizer.minimize`).
"""

from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass

import numpy as np

from . import _lib
from .density import DensityField, device_params
from .errors import ConfigError
from .geometry import EPS_PROJ, QUADRATURE_RULES, QuadratureRule, composite_nodes, normalize

logger = logging.getLogger(__name__)


def _torch():
    import torch

    return torch


def to_numpy(*tensors):
    """Device tensors -> NumPy arrays through pinned host tensors (torch's caching host
    allocator: full PCIe rate, no per-call page-locking after the first), one sync.  Each
    array keeps its pinned tensor alive."""
    torch = _torch()
    outs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in tensors]
    devices = {t.device for t in tensors if t.is_cuda}
    for o, t in zip(outs, tensors):
        with torch.cuda.device(t.device):      # the copy is ordered on the tensor's stream
            o.copy_(t, non_blocking=True)
    for d in devices:                          # wait for every copy before handing out arrays
        torch.cuda.current_stream(d).synchronize()
    return [o.numpy() for o in outs]


@dataclass
class EvalResult:
    """optimizer.py:66-76 (+ mass).  Arrays are NumPy or CUDA tensors (see module doc)."""

    energy: float
    grad: object
    grad_norm: float
    lloyd_diag: object
    first: object
    migration: str = "in-place"
    laplacian: object = None
    mass: object = None
    obtuse_count: int = 0
    min_diag: float = float("nan")      # min lloyd_diag (cvt_core.py:184 test), device path
    dirderiv: float = float("nan")      # sum g.(q3/|v|) when evaluated as a line-search trial
    staged: bool = False                # the evaluation staged its LBFGS pair (evaluate_device)


class DeviceLaplacian:
    """LaplacianPreconditioner (cvt_core.py:192-236) on the device: density-weighted graph
    Laplacian over the Delaunay adjacency of one evaluation (weights and sparsity copied at
    assembly, C ABI `scvt_laplacian`), perturbed as ``a6`` (+1e-6 I) or ``m2`` (diagonal
    x 1.01); `solve` runs conjugate gradients on the three coordinate columns
    (`scvt_laplacian_solve`) where the reference factors with SuperLU."""

    TOL = 1e-14
    MAX_ITER = 50000

    def __init__(self, ctx, n: int, perturbation: str, device):
        torch = _torch()
        if perturbation not in ("a6", "m2"):
            raise ValueError(f"unknown perturbation {perturbation!r}")
        self.ctx, self.n, self.perturbation = ctx, n, perturbation
        self.wsym = torch.empty((n, _lib.MAX_DEGREE), dtype=torch.float64, device=device)
        self.diag = torch.empty(n, dtype=torch.float64, device=device)
        self.nbr = torch.empty((n, _lib.MAX_DEGREE), dtype=torch.int32, device=device)
        self.deg = torch.empty(n, dtype=torch.int32, device=device)
        ctx.call("scvt_laplacian", n, _lib.dptr(self.wsym), _lib.dptr(self.diag),
                 _lib.dptr(self.nbr), _lib.dptr(self.deg), what="laplacian")
        self.dpert = self.diag + 1e-6 if perturbation == "a6" else self.diag * (1.0 + 1e-2)
        self.iterations = 0

    def solve(self, rhs):
        """Solve A_pert x = rhs for an (n, 3) device tensor (or NumPy array)."""
        torch = _torch()
        host = not isinstance(rhs, torch.Tensor)
        b = torch.as_tensor(np.asarray(rhs, dtype=np.float64) if host else rhs,
                            device=self.wsym.device).reshape(self.n, 3).contiguous()
        x = torch.empty_like(b)
        it = ctypes.c_int32()
        self.ctx.call("scvt_laplacian_solve", self.n, _lib.dptr(self.nbr), _lib.dptr(self.deg),
                      _lib.dptr(self.wsym), _lib.dptr(self.dpert), _lib.dptr(b), _lib.dptr(x),
                      self.TOL, self.MAX_ITER, ctypes.byref(it), what="laplacian solve")
        self.iterations += it.value
        return to_numpy(x)[0] if host else x


@dataclass(frozen=True)
class SphericalTriangulation:
    """delaunay.py:50-78: canonical triangles (+ circumcircles) and per-triangle flags
    (1 = an edge failed the in-circle floating-point filter: cocircular candidate)."""

    triangles: np.ndarray
    circumcenters: np.ndarray
    circumradii: np.ndarray
    flags: np.ndarray | None = None

    @property
    def count(self) -> int:
        return len(self.triangles)

    def edges(self) -> np.ndarray:
        e = np.concatenate([self.triangles[:, [0, 1]], self.triangles[:, [1, 2]],
                            self.triangles[:, [2, 0]]])
        e.sort(axis=1)
        return np.unique(e, axis=0)


class _Context:
    """Owns one `scvt_ctx` (device workspace sized for n_max, LBFGS ring of m pairs)."""

    def __init__(self, device: int, n_max: int, cfg):
        self.lib = _lib.load()
        self.ptr = ctypes.c_void_p()
        rc = self.lib.scvt_create(ctypes.byref(self.ptr), device, n_max, ctypes.byref(cfg))
        if rc:
            msg = self.lib.scvt_last_error(self.ptr).decode() if self.ptr else ""
            self.lib.scvt_destroy(self.ptr)
            self.ptr = None
            _lib.check(rc, None, f"scvt_create: {msg}")
        self.n_max = n_max
        self.device = device
        self._stream = None
        torch = _torch()
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        self._current_stream = ((lambda: raw(device)) if raw is not None else
                                (lambda: torch.cuda.current_stream(device).cuda_stream))

    def call(self, name: str, *args, what: str | None = None):
        s = self._current_stream()          # calls are ordered on the caller's current stream
        if s != self._stream:
            self.lib.scvt_set_stream(self.ptr, ctypes.c_void_p(s))
            self._stream = s
        rc = getattr(self.lib, name)(self.ptr, *args)
        if rc:
            _lib.check(rc, self.ptr, what or name)

    def launches(self) -> int:
        return int(self.lib.scvt_launch_count(self.ptr))

    def close(self):
        if self.ptr:
            self.lib.scvt_destroy(self.ptr)
            self.ptr = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class MeshEvaluator:
    """Energy / gradient evaluator on one B200 (pipeline.py:101-286 protocol).

    Extra keywords ``subdivision`` (depth d of `subdivide_fans`, delaunay.py:383-407, applied
    to every fan sub-triangle; DECISIONS.md D2), ``device`` and ``density_table`` (tanh^4
    densities: evaluate rho through the piecewise polynomial of `density.tanh4_table`
    instead of atan2/tanh per node; both agree to ~1e-15).  ``workers``/``backend`` are accepted
    for signature compatibility.  The moments always come from the global path, which the
    reference's region path reproduces bitwise; a ``covering``
    (`partition.Covering`) adds the reference's per-evaluation migration class
    (`EvalResult.migration`, computed on the device), which drives the optimizer's
    re-decompose-and-reset rule (optimizer.py:377-381).  The graph Laplacian preconditioner
    (cvt_core.py:192-240) is assembled on the device when ``laplacian`` is "a6" or "m2"
    (`DeviceLaplacian`, `EvalResult.laplacian`)."""

    def __init__(self, density: DensityField, rule: QuadratureRule | str, covering=None,
                 workers: int = 1, backend: str = "process", laplacian: str | None = None,
                 measure: str = "flat", eps_proj: float = EPS_PROJ, *, subdivision: int = 0,
                 device: int | None = None, density_table: bool = True):
        if laplacian not in (None, "a6", "m2"):
            raise ValueError(f"unknown perturbation {laplacian!r}")
        if measure not in ("flat", "sphere"):
            raise ValueError(f"unknown integration measure {measure!r}")
        self.density = density
        self.rule = QUADRATURE_RULES[rule] if isinstance(rule, str) else rule
        self.covering = covering
        self.workers = max(1, workers)
        self.backend = backend
        self.laplacian = laplacian
        self.measure = measure
        self.eps_proj = eps_proj
        self.subdivision = int(subdivision)
        self.device = device
        self.density_table = bool(density_table)
        self.fallbacks = 0
        self.evaluations = 0
        self._l1, self._l2, self._w = composite_nodes(self.rule, self.subdivision)
        self._ctx: _Context | None = None
        self._m = 7
        self._arith = None      # frozen covering cells (device int32), see _migration
        self._cov_dev = None

    # -- context ----------------------------------------------------------------------
    def _device_index(self) -> int:
        torch = _torch()
        if self.device is not None:
            return int(self.device)
        if not torch.cuda.is_available():
            from .errors import DeviceError

            raise DeviceError("no CUDA device: the SCVT hot path runs only on the GPU")
        return torch.cuda.current_device()

    def _ensure_ctx(self, n: int, m: int | None = None) -> _Context:
        m = self._m if m is None else int(m)
        if self._ctx is not None and self._ctx.n_max >= n and self._m == m:
            return self._ctx
        if self._ctx is not None:
            self._ctx.close()
        cfg, keep = _lib.make_config(device_params(self.density), self.measure, self._l1,
                                     self._l2, self._w, m, self.density_table)
        self._ctx = _Context(self._device_index(), max(n, 4), cfg)
        del keep
        self._m = m
        return self._ctx

    @property
    def context(self) -> _Context | None:
        return self._ctx

    def close(self):
        if self._ctx is not None:
            self._ctx.close()
            self._ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def redecompose(self, points):
        """Refresh the frozen (arithmetic) cells from the current geometry (pipeline.py:
        157-162); nothing to do without a covering."""
        if self.covering is None:
            return None
        z, _ = self._as_device(points)
        self._migration(z, fresh=True)
        return None

    def _migration(self, z, fresh: bool = False) -> str:
        """The reference's per-evaluation migration class (pipeline.py:244-259 with
        partition.py:123-164) on the device: nearest covering centre of every point against
        the cells frozen at the first evaluation / last `redecompose`."""
        if self.covering is None:
            return "in-place"
        torch = _torch()
        from .partition import MIGRATION_CLASSES

        n = z.shape[0]
        if self._cov_dev is None:
            cov = self.covering
            self._cov_dev = (torch.as_tensor(np.ascontiguousarray(cov.centers, dtype=np.float64),
                                             device=z.device),
                             torch.as_tensor(cov.adjacency_bitmap().view(np.int32),
                                             device=z.device).contiguous(),
                             int(cov.cell_count))
        if self._arith is None or self._arith.shape[0] != n:
            self._arith = torch.empty(n, dtype=torch.int32, device=z.device)
            fresh = True
        centers, adj, p = self._cov_dev
        cls = ctypes.c_int32()
        self._ensure_ctx(n).call("scvt_migration", _lib.dptr(z), n, _lib.dptr(centers), p,
                                 _lib.dptr(adj), _lib.dptr(self._arith), int(fresh),
                                 ctypes.byref(cls), what="migration")
        return MIGRATION_CLASSES[cls.value]

    _FALLBACK_REASONS = {1: "truncated Voronoi fans (CoverageError)",
                         2: "point near the projection antipode (AntipodeError)",
                         4: "region with fewer than 3 members (InsufficientPointsError)"}

    def region_failures(self, z) -> np.ndarray:
        """Per covering cell, the reason bits (1 CoverageError, 2 AntipodeError,
        4 InsufficientPointsError) for which the reference's region task of that cell would
        fail at these (just evaluated) points; 0 where it succeeds or has no owned point."""
        centers, adj, p = self._cov_dev
        f = ctypes.c_int32()
        per = (ctypes.c_int32 * p)()
        self._ctx.call("scvt_region_cover", _lib.dptr(z), z.shape[0], _lib.dptr(centers), p,
                       _lib.dptr(adj), float(self.eps_proj), ctypes.byref(f), per,
                       what="region_cover")
        return np.frombuffer(per, dtype=np.int32).copy()

    def _region_fallback(self, z):
        """With a covering: whether the reference's region path would have failed for these
        points and fallen back to the global path (pipeline.py:244-259), which counts the
        evaluation in `fallbacks`; the moments are the global path's either way."""
        self._last_fallback = 0
        if self.covering is None:
            return
        f = ctypes.c_int32(int(np.bitwise_or.reduce(self.region_failures(z))))
        if f.value:
            self.fallbacks += 1
            self._last_fallback = 1
            why = "; ".join(v for k, v in self._FALLBACK_REASONS.items() if f.value & k)
            logger.warning("region path failed (%s); global fallback", why)

    def discard_evaluation(self):
        """Forget the last evaluation (a speculative line-search trial the reference never
        evaluates): its evaluation and fallback counts."""
        self.evaluations -= 1
        self.fallbacks -= getattr(self, "_last_fallback", 0)
        self._last_fallback = 0

    def optimizer_ops(self, ctx, n: int):
        """The optimizer's vector algebra for this evaluator's layout (one GPU: all rows)."""
        from .optimizer import _DeviceOps

        return _DeviceOps(ctx, n)

    # -- evaluation -------------------------------------------------------------------
    def _as_device(self, points):
        torch = _torch()
        if isinstance(points, torch.Tensor) and points.is_cuda:
            z = points
            if z.dtype != torch.float64:
                z = z.to(torch.float64)
            return z.contiguous(), False
        arr = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
        if arr.ndim != 2 or arr.shape[1] != 3:
            raise ValueError("points must be (K, 3)")
        return torch.from_numpy(arr).to(f"cuda:{self._device_index()}"), True

    def evaluate_device(self, z, q3=None, norms=None, pair=None) -> EvalResult:
        """Device-resident evaluation: ``z`` is a contiguous float64 CUDA tensor (K, 3).
        With ``q3``/``norms`` (a line-search trial z = v/|v|, v = z0 + alpha q3) the result also
        carries the directional derivative sum g.(q3/|v|) (optimizer.py:330).  ``pair`` =
        (z_old, g_old): also stage the LBFGS correction pair this point would push
        (`scvt_evaluate_staged`), so the optimizer's push costs no further host round trip."""
        torch = _torch()
        n = z.shape[0]
        ctx = self._ensure_ctx(n)
        grad = torch.empty_like(z)
        first = torch.empty_like(z)
        mass = torch.empty(n, dtype=torch.float64, device=z.device)
        diag = torch.empty(n, dtype=torch.float64, device=z.device)
        sc = (ctypes.c_double * 5)()
        if pair is not None:
            ctx.call("scvt_evaluate_staged", _lib.dptr(z), n, _lib.dptr(grad), _lib.dptr(first),
                     _lib.dptr(mass), _lib.dptr(diag), _lib.dptr(q3), _lib.dptr(norms),
                     _lib.dptr(pair[0]), _lib.dptr(pair[1]), sc, what="evaluate")
        else:
            ctx.call("scvt_evaluate_ex", _lib.dptr(z), n, _lib.dptr(grad), _lib.dptr(first),
                     _lib.dptr(mass), _lib.dptr(diag), _lib.dptr(q3), _lib.dptr(norms), sc,
                     what="evaluate")
        self.evaluations += 1
        migration = self._migration(z)
        self._region_fallback(z)
        return EvalResult(energy=float(sc[0]), grad=grad, grad_norm=float(sc[1]),
                          lloyd_diag=diag, first=first, mass=mass, obtuse_count=int(sc[2]),
                          min_diag=float(sc[3]),
                          dirderiv=float(sc[4]) if q3 is not None else float("nan"),
                          migration=migration, staged=pair is not None,
                          laplacian=(DeviceLaplacian(ctx, n, self.laplacian, z.device)
                                     if self.laplacian is not None else None))

    def evaluate(self, points) -> EvalResult:
        """pipeline.py:261-279.  NumPy in -> NumPy out; CUDA tensor in -> tensors out."""
        z, host = self._as_device(points)
        r = self.evaluate_device(z)
        if host:
            r.grad, r.first, r.mass, r.lloyd_diag = to_numpy(r.grad, r.first, r.mass,
                                                             r.lloyd_diag)
        return r

    def cell_energy(self, n: int):
        """Per-cell energies of the last evaluation (device tensor, n doubles)."""
        torch = _torch()
        ctx = self._ensure_ctx(n)
        out = torch.empty(n, dtype=torch.float64, device=f"cuda:{ctx.device}")
        ctx.call("scvt_cell_energy", n, _lib.dptr(out), what="cell_energy")
        return out

    def evaluate_on_triangles(self, points, triangles) -> EvalResult:
        """Moments over a caller-supplied canonical triangulation (parity tests)."""
        torch = _torch()
        z, host = self._as_device(points)
        n = z.shape[0]
        ctx = self._ensure_ctx(n)
        tri = torch.as_tensor(np.ascontiguousarray(triangles, dtype=np.int64), device=z.device)
        grad = torch.empty_like(z)
        first = torch.empty_like(z)
        mass = torch.empty(n, dtype=torch.float64, device=z.device)
        diag = torch.empty(n, dtype=torch.float64, device=z.device)
        sc = (ctypes.c_double * 3)()
        ctx.call("scvt_evaluate_on_triangles", _lib.dptr(z), n, _lib.dptr(tri), tri.shape[0],
                 _lib.dptr(grad), _lib.dptr(first), _lib.dptr(mass), _lib.dptr(diag), sc,
                 what="evaluate_on_triangles")
        r = EvalResult(energy=float(sc[0]), grad=grad, grad_norm=float(sc[1]), lloyd_diag=diag,
                       first=first, mass=mass, obtuse_count=int(sc[2]))
        if host:
            r.grad, r.first, r.mass, r.lloyd_diag = to_numpy(r.grad, r.first, r.mass,
                                                             r.lloyd_diag)
        return r

    def triangulate_device(self, z):
        """Canonical (2K-4, 3) int64 triangles + flags on the device, plus stats dict."""
        torch = _torch()
        n = z.shape[0]
        ctx = self._ensure_ctx(n)
        t = max(2 * n - 4, 1)
        tri = torch.empty((t, 3), dtype=torch.int64, device=z.device)
        flags = torch.empty(t, dtype=torch.uint8, device=z.device)
        st = (ctypes.c_int64 * 8)()
        ctx.call("scvt_triangulate", _lib.dptr(z), n, _lib.dptr(tri), _lib.dptr(flags), st,
                 what="triangulate")
        stats = {"triangles": int(st[0]), "flagged": int(st[1]), "max_valence": int(st[2]),
                 "ambiguous_edges": int(st[3]), "tie_breaks": int(st[4]),
                 "max_passes": int(st[5]), "sweep_cells": int(st[6]),
                 "sweep_batches": int(st[7])}
        return tri, flags, stats

    def triangulation(self, points) -> SphericalTriangulation:
        """Global Delaunay triangulation at ``points`` (pipeline.py:281-286), canonical order
        (delaunay.py:133-147).  Circumcircles follow delaunay.py:150-169 (host, output only)."""
        z, _ = self._as_device(points)
        tri, flags, _ = self.triangulate_device(z)
        tri = tri.cpu().numpy()
        pts = z.cpu().numpy()
        v = pts[tri]
        nrm = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
        centers = nrm / np.linalg.norm(nrm, axis=1, keepdims=True)
        radii = np.arctan2(np.linalg.norm(np.cross(centers, v[:, 0]), axis=-1),
                           np.sum(centers * v[:, 0], axis=-1))
        return SphericalTriangulation(tri, centers, radii, flags.cpu().numpy())


def parallel_iteration(points, covering, density, rule, workers=1, backend="thread",
                       measure="flat", subdivision=0):
    """pipeline.py:289-295: one pass -> (F, grad, Lloyd diagonal, migration status)."""
    with MeshEvaluator(density, rule, covering, workers=workers, backend=backend,
                       measure=measure, subdivision=subdivision) as ev:
        res = ev.evaluate(points)
    return res.energy, res.grad, res.lloyd_diag, res.migration


def bisect(points, tri: SphericalTriangulation) -> np.ndarray:
    """Edge-midpoint refinement K -> 4K - 6 (pipeline.py:298-303)."""
    points = np.asarray(points, dtype=float)
    edges = tri.edges()
    mids = normalize(points[edges[:, 0]] + points[edges[:, 1]])
    return np.vstack([points, mids])


def bisection_ladder(target: int, floor: int = 200) -> list[int]:
    """pipeline.py:306-315."""
    ladder = [target]
    while ladder[0] > floor and (ladder[0] + 6) % 4 == 0:
        ladder.insert(0, (ladder[0] + 6) // 4)
    return ladder


# ---------------------------------------------------------------------- ladder driver (§8(f)1)
def default_quadrature(density_name: str) -> str:
    """pipeline.py:56-59."""
    return "9pt" if density_name == "x64" else "4pt"


def default_partitions(k: int) -> int:
    """pipeline.py:48-53 (kept for API parity; the GPU always runs the global path)."""
    return max(8, min(64, k // 160))


@dataclass
class RunPlan:
    """pipeline.py:318-363, plus ``subdivision`` (depth-d fans, DECISIONS.md D2) and the
    BASELINE densities/rules (`density_preset` c3/c4/c5, "7pt")."""

    points: int
    density_name: str = "const"
    method: str = "lloyd-plbfgs"
    seed: int = 1
    workers: int = 1
    backend: str = "process"
    partitions: int | None = None
    quadrature: str | None = None
    ladder: list | None = None
    criteria: object = None
    intermediate_movement_tol: float = 1e-3
    measure: str = "flat"
    density_overrides: dict = None
    eps_proj: float = EPS_PROJ
    subdivision: int = 0
    corrections: int = 7

    def __post_init__(self):
        from .errors import ConfigError
        from .optimizer import StoppingCriteria

        if self.criteria is None:
            self.criteria = StoppingCriteria()
        if self.density_overrides is None:
            self.density_overrides = {}
        if self.points < 4:
            raise ConfigError("need at least 4 generators")
        if self.ladder is None:
            self.ladder = [self.points]
        if self.ladder[-1] != self.points:
            raise ConfigError(
                f"ladder must end at the target point count {self.points}, got {self.ladder}")
        for a, b in zip(self.ladder, self.ladder[1:]):
            if b != 4 * a - 6:
                raise ConfigError(f"ladder step {a} -> {b} violates the bisection arithmetic "
                                  f"(expect {4 * a - 6})")
        if self.quadrature is None:
            self.quadrature = default_quadrature(self.density_name)
        if self.quadrature not in QUADRATURE_RULES:
            raise ConfigError(f"unknown quadrature {self.quadrature!r}")

    def density(self) -> DensityField:
        from .density import density_preset

        d = density_preset(self.density_name)
        if self.density_overrides:
            d = d.with_overrides(**self.density_overrides)
        return d

    def rule(self) -> QuadratureRule:
        return QUADRATURE_RULES[self.quadrature]


@dataclass
class LevelResult:
    k: int
    result: object
    wall_time: float


@dataclass
class RunResult:
    plan: RunPlan
    points: np.ndarray
    triangulation: SphericalTriangulation
    levels: list
    covering: object
    wall_time: float

    @property
    def final(self):
        return self.levels[-1].result.final


def _covering_for(plan: RunPlan, k: int, density: DensityField):
    """pipeline.py:387-393: the level's covering when it is thick enough to decompose."""
    from .partition import bootstrap_partition_cvt

    p = plan.partitions if plan.partitions is not None else default_partitions(k)
    if k < 16 * p:
        logger.info("level K=%d below 16 x %d partitions; using the global path", k, p)
        return None
    return bootstrap_partition_cvt(p, seed=plan.seed, density=density)


def run(plan: RunPlan, initial_points=None, progress=None) -> RunResult:
    """Optimise-bisect ladder (pipeline.py:396-455) on the GPU: every level is minimised by
    the GPU optimizer, triangulated on the GPU, and bisected (K -> 4K - 6) to seed the next."""
    import time
    from dataclasses import replace

    from .density import sample_by_density
    from .errors import ConfigError, ScvtError
    from .optimizer import minimize

    t0 = time.perf_counter()
    density = plan.density()
    rule = plan.rule()
    if initial_points is not None:
        z = normalize(np.asarray(initial_points, dtype=float))
        if len(z) != plan.ladder[0]:
            raise ConfigError(f"initial points ({len(z)}) do not match the first ladder level "
                              f"({plan.ladder[0]})")
    else:
        z = sample_by_density(density, plan.ladder[0], plan.seed)
    laplacian = {"laplacian-a6": "a6", "laplacian-m2": "m2"}.get(plan.method)
    levels = []
    tri = None
    covering = None
    for li, k in enumerate(plan.ladder):
        last = li == len(plan.ladder) - 1
        criteria = plan.criteria if last else replace(
            plan.criteria, movement_tol=plan.intermediate_movement_tol)
        covering = _covering_for(plan, k, density)
        t_level = time.perf_counter()
        with MeshEvaluator(density, rule, covering, workers=plan.workers, backend=plan.backend,
                           laplacian=laplacian,
                           measure=plan.measure, eps_proj=plan.eps_proj,
                           subdivision=plan.subdivision) as ev:
            result = minimize(z, plan.method, ev, criteria, corrections=plan.corrections,
                              callback=progress)
            z = result.points
            tri = ev.triangulation(z)
        levels.append(LevelResult(k=k, result=result, wall_time=time.perf_counter() - t_level))
        logger.info("level K=%d: %d iterations, F=%.6e, |grad|=%.3e (%s)", k,
                    len(result.records), result.final.energy, result.final.grad_norm,
                    result.reason)
        if not last:
            z = bisect(z, tri)
            if len(z) != plan.ladder[li + 1]:
                raise ScvtError(f"bisection produced {len(z)} points; ladder expected "
                                f"{plan.ladder[li + 1]}")
    return RunResult(plan=plan, points=z, triangulation=tri, levels=levels, covering=covering,
                     wall_time=time.perf_counter() - t0)
