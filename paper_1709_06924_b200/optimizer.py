"""Lloyd / LBFGS / Lloyd-preconditioned LBFGS driver (drop-in for `scvtmesh.optimizer`).

The control flow — two-loop with fallbacks, tangent projection, strong-Wolfe bracketing and
zoom, Lloyd fallback, curvature-guarded history, stopping rules — is the reference's
(optimizer.py:147-391) line for line, because its branch decisions define parity.  Every
vector lives on the GPU: the evaluator's kernels produce energy/gradient, and the LBFGS
vector algebra (two-loop dots/axpys, projection, trial points, directional derivatives,
history pushes) runs as FP64 kernels of the same library (include/scvt_b200.h).  The host
only sees the scalars the branch decisions need.
"""

from __future__ import annotations

import ctypes
import logging
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import (
    CentroidAtOriginError,
    ConfigError,
    LineSearchFailure,
    NonDescentError,
)
from .pipeline import EvalResult, MeshEvaluator, to_numpy

logger = logging.getLogger(__name__)

EPS_CURVATURE = 1e-14        # optimizer.py:32 (enforced inside scvt_history_push)
WOLFE_C1 = 1e-4              # optimizer.py:33
WOLFE_C2 = 0.9               # optimizer.py:34
MAX_LINE_SEARCH_EVALS = 10   # optimizer.py:35

METHODS = ("lloyd", "lbfgs", "lloyd-plbfgs", "laplacian-a6", "laplacian-m2")


@dataclass
class StoppingCriteria:
    """optimizer.py:40-53."""

    max_iterations: int = 2000
    movement_tol: float = 5e-4
    grad_tol: float = 5e-4
    stall_tol: float = 1e-7

    def __post_init__(self):
        if min(self.movement_tol, self.grad_tol, self.stall_tol) <= 0:
            raise ValueError("stopping tolerances must be positive")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")


@dataclass
class IterationRecord:
    """optimizer.py:56-63."""

    n: int
    energy: float
    grad_norm: float
    step: float
    fevals: int | None
    time_ms: float


@dataclass
class MinimizeResult:
    """optimizer.py:249-257 (``points`` and ``final`` arrays are NumPy)."""

    points: np.ndarray
    records: list
    reason: str
    fevals: int
    resets: int
    wall_time: float
    final: EvalResult = field(repr=False, default=None)


def wolfe_line_search(phi, f0: float, dphi0: float, c1: float = WOLFE_C1, c2: float = WOLFE_C2,
                      max_evals: int = MAX_LINE_SEARCH_EVALS, initial_step: float = 1.0,
                      first=None):
    """Strong-Wolfe bracketing + quadratic zoom (optimizer.py:170-237), scalar logic only.
    ``first``: phi(initial_step) already evaluated (speculatively, while the direction's scalars
    were in flight), used as the first trial."""
    if dphi0 >= 0.0:
        raise NonDescentError(f"line search needs a descent direction, dphi0={dphi0:.3e}")
    evals = 0
    best = None

    def record(alpha, f, payload):
        nonlocal best
        if f < f0 and (best is None or f < best[0]):
            best = (f, alpha, payload)

    def exhausted_result():
        if best is None:
            raise LineSearchFailure(f"no decrease within {max_evals} evaluations")
        f, alpha, payload = best
        return alpha, f, payload, evals, True

    def zoom(lo, f_lo, d_lo, hi, f_hi):
        nonlocal evals
        while evals < max_evals:
            span = hi - lo
            denom = 2.0 * (f_hi - f_lo - d_lo * span)
            alpha = lo - d_lo * span * span / denom if denom != 0.0 else lo + 0.5 * span
            low, high = (lo, hi) if lo < hi else (hi, lo)
            margin = 0.1 * abs(span)
            if not (low + margin <= alpha <= high - margin):
                alpha = lo + 0.5 * span
            f, d, payload = phi(alpha)
            evals += 1
            record(alpha, f, payload)
            if f > f0 + c1 * alpha * dphi0 or f >= f_lo:
                hi, f_hi = alpha, f
            else:
                if abs(d) <= -c2 * dphi0:
                    return alpha, f, payload, evals, False
                if d * span >= 0.0:
                    hi, f_hi = lo, f_lo
                lo, f_lo, d_lo = alpha, f, d
        return exhausted_result()

    alpha_prev, f_prev, d_prev = 0.0, f0, dphi0
    alpha = initial_step
    pre = first
    first = True
    while evals < max_evals:
        if pre is not None:
            (f, d, payload), pre = pre, None
        else:
            f, d, payload = phi(alpha)
        evals += 1
        record(alpha, f, payload)
        if f > f0 + c1 * alpha * dphi0 or (not first and f >= f_prev):
            return zoom(alpha_prev, f_prev, d_prev, alpha, f)
        if abs(d) <= -c2 * dphi0:
            return alpha, f, payload, evals, False
        if d >= 0.0:
            return zoom(alpha, f, d, alpha_prev, f_prev)
        alpha_prev, f_prev, d_prev = alpha, f, d
        alpha *= 2.0
        first = False
    return exhausted_result()


class _DeviceOps:
    """Thin wrappers over the optimizer entry points of the C ABI (one GPU: every vector holds
    all n rows).  `parallel.SliceOps` is the arithmetic-layout counterpart of one rank."""

    def __init__(self, ctx, n: int):
        self.ctx = ctx
        self.n = n

    # -- layout: one GPU holds every row
    def vec3(self, z):
        """An (owned rows, 3) work vector (q, q3)."""
        return z.new_empty(z.shape)

    def positions(self, z):
        """A full (n, 3) position buffer that trial / Lloyd points are written into."""
        return z.new_empty(z.shape)

    def scalars(self, z):
        """An (owned rows,) work vector (trial norms)."""
        return z.new_empty(z.shape[0])

    def full(self, res: EvalResult) -> EvalResult:
        """The result with every row (the owned rows are all of them here)."""
        return res

    def history_clear(self):
        self.ctx.call("scvt_history_clear")

    def gamma(self) -> float:
        g = ctypes.c_double()
        self.ctx.call("scvt_history_gamma", ctypes.byref(g))
        return g.value

    def direction(self, g, diag, gamma, q) -> float:
        qg = ctypes.c_double()
        self.ctx.call("scvt_lbfgs_direction", _lib.dptr(g), _lib.dptr(diag), float(gamma), self.n,
                      _lib.dptr(q), ctypes.byref(qg))
        return qg.value

    speculate = True     # the first line-search trial may be enqueued before the direction's
                         # scalars are read (one host round trip less per iteration)

    def direction_tangent_async(self, g, diag, gamma, z, q3):
        self.ctx.call("scvt_lbfgs_direction_tangent_async", _lib.dptr(g), _lib.dptr(diag),
                      float(gamma), _lib.dptr(z), self.n, _lib.dptr(q3))

    def direction_result(self):
        out = (ctypes.c_double * 2)()
        self.ctx.call("scvt_direction_result", out)
        return out[0], out[1]

    def direction_tangent(self, g, diag, gamma, z, q3):
        out = (ctypes.c_double * 2)()
        self.ctx.call("scvt_lbfgs_direction_tangent", _lib.dptr(g), _lib.dptr(diag),
                      float(gamma), _lib.dptr(z), self.n, _lib.dptr(q3), out)
        return out[0], out[1]

    def direction_general(self, g, h0, z, q, q3):
        """two_loop_direction with a general initial inverse (optimizer.py:147-167; h0 =
        LaplacianInverse, 137-144) + the tangent projection: returns (q.g, g.q3)."""
        self.ctx.call("scvt_twoloop_backward", _lib.dptr(g), self.n, _lib.dptr(q))
        r = h0.solve(q)
        qg = ctypes.c_double()
        self.ctx.call("scvt_twoloop_forward", _lib.dptr(r), _lib.dptr(g), self.n,
                      ctypes.byref(qg))
        q.copy_(r)
        return qg.value, self.tangent(q, z, g, q3)

    def tangent(self, q, z, g, q3) -> float:
        d = ctypes.c_double()
        self.ctx.call("scvt_tangent_project", _lib.dptr(q), _lib.dptr(z), _lib.dptr(g), self.n,
                      _lib.dptr(q3), ctypes.byref(d))
        return d.value

    def trial(self, z, q3, alpha, zt, norms):
        self.ctx.call("scvt_trial_point", _lib.dptr(z), _lib.dptr(q3), float(alpha), self.n,
                      _lib.dptr(zt), _lib.dptr(norms))

    def dirderiv(self, g, q3, norms) -> float:
        d = ctypes.c_double()
        self.ctx.call("scvt_directional_derivative", _lib.dptr(g), _lib.dptr(q3),
                      _lib.dptr(norms), self.n, ctypes.byref(d))
        return d.value

    def lloyd(self, first, z_out):
        self.ctx.call("scvt_lloyd_step", _lib.dptr(first), self.n, _lib.dptr(z_out),
                      what="lloyd_step")

    def minimum(self, v) -> float:
        m = ctypes.c_double()
        self.ctx.call("scvt_min", _lib.dptr(v), v.numel(), ctypes.byref(m))
        return m.value

    def scale(self, a, x, y):
        self.ctx.call("scvt_scale", float(a), _lib.dptr(x), x.numel(), _lib.dptr(y))

    stage_pairs = True   # line-search trials stage their correction pair (one host round trip
                         # per iteration instead of two)

    def push(self, z_old, z_new, g_old, g_new, staged=False):
        pushed = ctypes.c_int32()
        mv = ctypes.c_double()
        if staged:    # the pair was reduced with z_new's evaluation (scvt_evaluate_staged)
            self.ctx.call("scvt_history_commit_staged", _lib.dptr(z_new), _lib.dptr(g_new),
                          self.n, ctypes.byref(pushed), ctypes.byref(mv))
        else:
            self.ctx.call("scvt_history_push", _lib.dptr(z_old), _lib.dptr(z_new),
                          _lib.dptr(g_old), _lib.dptr(g_new), self.n, ctypes.byref(pushed),
                          ctypes.byref(mv))
        return bool(pushed.value), mv.value

    def max_abs_diff(self, a, b) -> float:
        m = ctypes.c_double()
        self.ctx.call("scvt_max_abs_diff", _lib.dptr(a), _lib.dptr(b), a.numel(), ctypes.byref(m))
        return m.value

    def normalize(self, z):
        self.ctx.call("scvt_normalize_rows", _lib.dptr(z), self.n)


def _to_host(res: EvalResult, z=None):
    """NumPy copy of a device result (and of the positions `z`), one pinned transfer."""
    ts = [res.grad, res.lloyd_diag, res.first] + ([res.mass] if res.mass is not None else [])
    arr = to_numpy(*ts, *([z] if z is not None else []))
    mass = arr[3] if res.mass is not None else None
    out = EvalResult(energy=res.energy, grad=arr[0], grad_norm=res.grad_norm,
                     lloyd_diag=arr[1], first=arr[2], migration=res.migration, mass=mass,
                     obtuse_count=res.obtuse_count, laplacian=res.laplacian)
    return (out, arr[-1]) if z is not None else out


class _HostLaplacian:
    """A reference-style preconditioner (``solve`` on NumPy (K, 3) arrays) seen from the
    device optimizer (LaplacianInverse, optimizer.py:137-144)."""

    def __init__(self, inner, device):
        self.inner, self.device = inner, device

    def solve(self, q):
        import torch

        x = np.asarray(self.inner.solve(to_numpy(q.reshape(-1, 3))[0]), dtype=np.float64)
        return torch.as_tensor(x.reshape(q.shape), device=self.device)


class HostEvaluatorAdapter:
    """Any evaluator of the reference's duck-typed protocol (``evaluate(points) -> EvalResult``
    with NumPy arrays, optional ``redecompose(points)``; optimizer.py:278-293) behind the
    device interface `Minimizer` drives, so `minimize` accepts it exactly like the reference's
    `minimize` does.  The optimizer algebra (two-loop, projection, trial points, history) still
    runs on the GPU; every evaluation crosses to the host and back.  No speculative trial:
    the wrapped evaluator sees exactly the reference's sequence of evaluations."""

    def __init__(self, inner, device: int | None = None):
        import torch

        from .density import density_preset

        if not callable(getattr(inner, "evaluate", None)):
            raise TypeError("evaluator must provide evaluate(points) -> EvalResult")
        self.inner = inner
        dev = torch.cuda.current_device() if device is None else int(device)
        # the algebra's context: any configuration works, the quadrature tables are unused
        self._algebra = MeshEvaluator(density_preset("const"), "4pt", device=dev)
        self.device = dev

    @property
    def evaluations(self):
        return getattr(self.inner, "evaluations", 0)

    @evaluations.setter
    def evaluations(self, v):
        if hasattr(self.inner, "evaluations"):
            self.inner.evaluations = v

    @property
    def context(self):
        return self._algebra.context

    def _as_device(self, points):
        return self._algebra._as_device(points)

    def _ensure_ctx(self, n, m=None):
        return self._algebra._ensure_ctx(n, m)

    def optimizer_ops(self, ctx, n):
        ops = _DeviceOps(ctx, n)
        ops.speculate = False
        ops.stage_pairs = False
        return ops

    def redecompose(self, points):
        fn = getattr(self.inner, "redecompose", None)
        if fn is not None:
            fn(to_numpy(points)[0] if not isinstance(points, np.ndarray) else points)

    def evaluate_device(self, z, q3=None, norms=None) -> EvalResult:
        import torch

        r = self.inner.evaluate(to_numpy(z)[0])
        dev = z.device

        def put(a):
            return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)

        grad, diag, first = put(r.grad), put(r.lloyd_diag), put(r.first)
        mass = getattr(r, "mass", None)
        dirderiv = float("nan")
        if q3 is not None:                         # phi's derivative (optimizer.py:330)
            qh, nh = to_numpy(q3, norms)
            dirderiv = float(np.einsum("ij,ij->i", np.asarray(r.grad), qh / nh[:, None]).sum())
        lap = getattr(r, "laplacian", None)
        return EvalResult(energy=float(r.energy), grad=grad, grad_norm=float(r.grad_norm),
                          lloyd_diag=diag, first=first,
                          mass=put(mass) if mass is not None else None,
                          migration=getattr(r, "migration", "in-place"),
                          laplacian=_HostLaplacian(lap, dev) if lap is not None else None,
                          min_diag=float(np.min(r.lloyd_diag)), dirderiv=dirderiv)

    def close(self):
        self._algebra.close()


class Minimizer:
    """The state of one `minimize` run, advanced one iteration at a time.

    `minimize` is `Minimizer(...)` + `step()` until a stopping rule fires; the benchmark
    drives `step()` directly so warm-up and timed iterations continue one trajectory."""

    def __init__(self, points, method: str, evaluator: MeshEvaluator, corrections: int = 7):
        import torch

        if method not in METHODS:
            raise ValueError(f"unknown method {method!r}; expected one of {METHODS}")
        if not hasattr(evaluator, "optimizer_ops"):      # reference-protocol evaluator
            evaluator = HostEvaluatorAdapter(evaluator)
        self.torch = torch
        self.method = method
        self.evaluator = evaluator
        z, _ = evaluator._as_device(points)
        self.z = z.clone()
        self.k = self.z.shape[0]
        self.ctx = evaluator._ensure_ctx(self.k, corrections)
        self.ops = evaluator.optimizer_ops(self.ctx, self.k)
        self.ops.normalize(self.z)                               # optimizer.py:290
        self.res = evaluator.evaluate_device(self.z)             # optimizer.py:293
        self.fevals = 1
        self.ops.history_clear()                                 # CorrectionHistory(m)
        self.resets = 0
        self.n = 0
        self.q = self.ops.vec3(self.z)
        self.q3 = self.ops.vec3(self.z)
        self._last_eval = None
        import inspect

        try:    # an evaluator (or subclass) whose evaluate_device takes no `pair` never stages
            self._ev_stages = "pair" in inspect.signature(evaluator.evaluate_device).parameters
        except (TypeError, ValueError):
            self._ev_stages = False

    def step(self):
        """One iteration (optimizer.py:300-366).  Returns (record, movement, z_new, res_new)
        and advances the state; the caller applies the stopping rules."""
        ops, ev, z, res = self.ops, self.evaluator, self.z, self.res
        self.n += 1
        n = self.n
        t_iter = time.perf_counter()
        if self.method == "lloyd":
            z_new = ops.positions(z)
            ops.lloyd(res.first, z_new)                          # optimizer.py:304
            res_new = ev.evaluate_device(z_new)
            self.fevals += 1
            fevals_iter = None
            alpha = 1.0
            movement = ops.max_abs_diff(z_new, z)
        else:
            # _initial_inverse (optimizer.py:260-275)
            diag = None
            gamma = ops.gamma()
            if self.method == "lloyd-plbfgs":
                if res.min_diag <= 0.0:                          # lloyd_preconditioner raises
                    logger.warning("nonpositive Lloyd diagonal; falling back to gamma identity")
                else:
                    diag = res.lloyd_diag
            q, q3 = self.q, self.q3
            if self.method.startswith("laplacian"):                # _initial_inverse
                if res.laplacian is None:
                    raise ValueError("evaluator did not supply a Laplacian factorization")

                def direction():
                    return ops.direction_general(res.grad, res.laplacian, z, q, q3)
            else:
                def direction():   # two_loop_direction + projection, fused on the device
                    return ops.direction_tangent(res.grad, diag, gamma, z, q3)
            # optimizer.py:147-167, 312-333
            first = None
            # trials stage the correction pair they would push (z, g are this iteration's)
            stage = getattr(ops, "stage_pairs", False) and self._ev_stages

            def trial_eval(zt, q3, norms):
                r = (ev.evaluate_device(zt, q3, norms, pair=(z, res.grad)) if stage
                     else ev.evaluate_device(zt, q3, norms))
                self._last_eval = r
                return r

            if getattr(ops, "speculate", False) and not self.method.startswith("laplacian"):
                # the direction and the alpha = 1 trial (always the line search's first) are
                # enqueued back to back; the direction's scalars are read after the trial's
                # evaluation.  A non-descent direction discards the trial (and any error it
                # raised), exactly as if it had never been evaluated.
                ops.direction_tangent_async(res.grad, diag, gamma, z, q3)
                zt, norms = ops.positions(z), ops.scalars(z)
                ops.trial(z, q3, 1.0, zt, norms)
                err = r1 = None
                try:
                    r1 = trial_eval(zt, q3, norms)
                except Exception as exc:  # noqa: BLE001 - re-raised below unless discarded
                    err = exc
                qg, dphi0 = ops.direction_result()
                if qg < 0.0 and dphi0 < 0.0:
                    if err is not None:     # the reference evaluates this very trial first
                        raise err
                    first = (r1.energy, r1.dirderiv, (zt, r1))
                elif r1 is not None:
                    # history reset (q.g >= 0) or Lloyd fallback (g.q3 >= 0, wolfe_line_search
                    # raises before any evaluation): the trial never happened in the reference
                    ev.discard_evaluation()
            else:
                qg, dphi0 = direction()
            if qg >= 0.0:
                logger.warning("non-descent direction at iteration %d; history reset", n)
                ops.history_clear()
                self.resets += 1
                qg, dphi0 = direction()
                if qg >= 0.0:
                    ops.scale(-ops.gamma(), res.grad, q)          # q = -hist.gamma() * g
                    dphi0 = ops.tangent(q, z, res.grad, q3)

            def phi(alpha, z=z, q3=q3):
                zt = ops.positions(z)
                norms = ops.scalars(z)
                ops.trial(z, q3, alpha, zt, norms)
                r = trial_eval(zt, q3, norms)                    # derivative fused in
                return r.energy, r.dirderiv, (zt, r)

            try:
                alpha, _, payload, evals, exhausted = wolfe_line_search(phi, res.energy, dphi0,
                                                                        first=first)
                z_new, res_new = payload
                fevals_iter = evals
                if exhausted:
                    logger.debug("line search exhausted at iteration %d", n)
            except (NonDescentError, LineSearchFailure) as exc:
                logger.warning("line search failed at iteration %d (%s); Lloyd fallback", n, exc)
                ops.history_clear()
                self.resets += 1
                z_new = ops.positions(z)
                ops.lloyd(res.first, z_new)
                res_new = ev.evaluate_device(z_new)
                self._last_eval = res_new
                fevals_iter = 1
                alpha = 0.0
            self.fevals += fevals_iter
            # optimizer.py:351-355; the pair staged by res_new's own evaluation is still the
            # context's staged one only if that evaluation was the last (a zoom may end on an
            # earlier trial): the commit checks the buffers and the general push is the fallback
            done = False
            if getattr(res_new, "staged", False) and self._last_eval is res_new:
                try:
                    _, movement = ops.push(z, z_new, res.grad, res_new.grad, staged=True)
                    done = True
                except ConfigError:     # the library holds no pair for these buffers
                    logger.debug("staged pair unavailable at iteration %d; regular push", n)
            if not done:
                _, movement = ops.push(z, z_new, res.grad, res_new.grad)
        rec = IterationRecord(n=n, energy=res_new.energy, grad_norm=res_new.grad_norm, step=alpha,
                              fevals=fevals_iter, time_ms=(time.perf_counter() - t_iter) * 1e3)
        self.z, self.res = z_new, res_new
        return rec, movement, z_new, res_new


def minimize(points, method: str, evaluator: MeshEvaluator, criteria: StoppingCriteria | None = None,
             corrections: int = 7, callback=None) -> MinimizeResult:
    """Drive one of the iteration methods to a stopping criterion (optimizer.py:278-391).

    ``points``: (K, 3) NumPy array or CUDA tensor.  ``evaluator``: this package's
    `MeshEvaluator` / `ShardedMeshEvaluator`, or any object with the reference's duck-typed
    ``evaluate``/``redecompose`` protocol (`HostEvaluatorAdapter`).  ``callback(n, z_new,
    res_new)`` receives NumPy arrays with every row when ``points`` is NumPy (as in the
    reference), and zero-copy CUDA tensors when ``points`` is a CUDA tensor (under a multi-GPU
    `ShardedMeshEvaluator` the vectors of res_new then hold the rank's arithmetic slice,
    `parallel.SliceOps`).  Returns NumPy ``points`` and ``final`` (all rows)."""
    criteria = criteria or StoppingCriteria()
    t0 = time.perf_counter()
    st = Minimizer(points, method, evaluator, corrections)
    host_input = not (isinstance(points, st.torch.Tensor) and points.is_cuda)
    records: list[IterationRecord] = []
    reason = "max-iterations"
    for _ in range(criteria.max_iterations):
        f_prev = st.res.energy
        rec, movement, z_new, res_new = st.step()
        records.append(rec)
        if callback is not None:
            if host_input:       # the reference hands NumPy arrays to callbacks
                res_h, z_h = _to_host(st.ops.full(res_new), z_new)
                callback(rec.n, z_h, res_h)
            else:
                callback(rec.n, z_new, res_new)
        res = st.res
        if movement <= criteria.movement_tol:                   # optimizer.py:368-376
            reason = "movement"
            break
        if abs(res.energy - f_prev) / abs(f_prev) < criteria.stall_tol:
            reason = "energy-stall"
            break
        if res.grad_norm / res.energy <= criteria.grad_tol:
            reason = "gradient"
            break
        if res.migration == "out-of-range":                     # optimizer.py:377-381
            logger.info("point migrated out of range at iteration %d; decomposition reset",
                        rec.n)
            evaluator.redecompose(st.z)
            st.ops.history_clear()
            st.resets += 1
    st.torch.cuda.current_stream(st.z.device).synchronize()
    wall = time.perf_counter() - t0
    final, points = _to_host(st.ops.full(st.res), st.z)
    return MinimizeResult(points=points, records=records, reason=reason,
                          fevals=st.fevals, resets=st.resets, wall_time=wall, final=final)


def lloyd_step(points, first_moments) -> np.ndarray:
    """optimizer.py:240-246 (host convenience for NumPy callers)."""
    first_moments = np.asarray(first_moments, dtype=float)
    norms = np.linalg.norm(first_moments, axis=1)
    if np.any(norms <= 1e-12):
        bad = np.flatnonzero(norms <= 1e-12)
        raise CentroidAtOriginError(f"first moment ~0 for cells {bad[:8].tolist()}")
    return first_moments / norms[:, None]
