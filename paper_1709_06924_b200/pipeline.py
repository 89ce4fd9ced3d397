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

    def call(self, name: str, *args, what: str | None = None):
        torch = _torch()
        self.lib.scvt_set_stream(self.ptr, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
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
    instead of atan2/tanh per node; both agree to ~1e-15).  ``covering``/``workers``/
    ``backend`` are accepted for signature compatibility; the GPU path is always the
    covering-free global path, which the reference's region path reproduces bitwise
    (SURVEY.md §6.3).  ``laplacian`` (SuperLU graph Laplacian, cvt_core.py:192-240) is out of
    scope and raises."""

    def __init__(self, density: DensityField, rule: QuadratureRule | str, covering=None,
                 workers: int = 1, backend: str = "process", laplacian: str | None = None,
                 measure: str = "flat", eps_proj: float = EPS_PROJ, *, subdivision: int = 0,
                 device: int | None = None, density_table: bool = True):
        if laplacian is not None:
            raise ConfigError("the Laplacian preconditioner is outside this hot path")
        if measure not in ("flat", "sphere"):
            raise ValueError(f"unknown integration measure {measure!r}")
        self.density = density
        self.rule = QUADRATURE_RULES[rule] if isinstance(rule, str) else rule
        self.covering = covering
        self.workers = max(1, workers)
        self.backend = backend
        self.laplacian = None
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
        """No decomposition state on the global GPU path (pipeline.py:157-162)."""
        return None

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

    def evaluate_device(self, z) -> EvalResult:
        """Device-resident evaluation: ``z`` is a contiguous float64 CUDA tensor (K, 3)."""
        torch = _torch()
        n = z.shape[0]
        ctx = self._ensure_ctx(n)
        grad = torch.empty_like(z)
        first = torch.empty_like(z)
        mass = torch.empty(n, dtype=torch.float64, device=z.device)
        diag = torch.empty(n, dtype=torch.float64, device=z.device)
        sc = (ctypes.c_double * 3)()
        ctx.call("scvt_evaluate", _lib.dptr(z), n, _lib.dptr(grad), _lib.dptr(first),
                 _lib.dptr(mass), _lib.dptr(diag), sc, what="evaluate")
        self.evaluations += 1
        return EvalResult(energy=float(sc[0]), grad=grad, grad_norm=float(sc[1]),
                          lloyd_diag=diag, first=first, mass=mass, obtuse_count=int(sc[2]))

    def evaluate(self, points) -> EvalResult:
        """pipeline.py:261-279.  NumPy in -> NumPy out; CUDA tensor in -> tensors out."""
        z, host = self._as_device(points)
        r = self.evaluate_device(z)
        if host:
            r.grad = r.grad.cpu().numpy()
            r.first = r.first.cpu().numpy()
            r.mass = r.mass.cpu().numpy()
            r.lloyd_diag = r.lloyd_diag.cpu().numpy()
        return r

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
            r.grad, r.first = r.grad.cpu().numpy(), r.first.cpu().numpy()
            r.mass, r.lloyd_diag = r.mass.cpu().numpy(), r.lloyd_diag.cpu().numpy()
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
