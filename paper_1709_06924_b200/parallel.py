"""Multi-GPU evaluation: one process per GPU, generators sharded, NCCL for the exchanges.

The reference parallelises one evaluation over an overlapping domain decomposition on a worker
pool (pipeline.py:62-98, 171-242; paper §3.2).  Here each rank owns an equal share of the
generators in cube-map bucket order (a space-filling order, DECISIONS.md D5) and the only
exchanges are two all-gathers per evaluation:

  1. cells      every rank builds the grid (replicated, cheap) and the Voronoi cells of its
                generators; the packed cycles are all-gathered so each rank can certify its
                cells against their neighbours' cycles (the "halo" is implicit);
  2. moments    each rank integrates the fans of its generators; the per-generator results are
                all-gathered, scattered to id order and reduced by the same fixed-shape kernel
                on every rank.

From the second evaluation on, the previous cycles are reused exactly as on one GPU: each
rank runs the flip-mode certificate of its own cells, the non-Delaunay edges are all-gathered
and every rank applies the same (deterministic) flip rounds to its replica of the cycles;
cells the flips cannot repair go through the rounds: each rank certifies its owned cells at the new
positions, the bad flags are all-reduced (max), every rank derives the same bad set and
re-check list, rebuilds its own bad cells, and only those cycles are all-gathered; up to
four rounds, then the full path above.

Positions are replicated; the optimizer's vectors are in arithmetic layout (`SliceOps`): rank r
owns a contiguous range of whole chunks of the generator ids (include/scvt_b200.h,
SCVT_CHUNKS) and holds only those rows of the gradient, first moments, Lloyd diagonal, search
direction and LBFGS history.  Every dot product is reduced per chunk, the partial buffers are
summed over the ranks by one all-reduce per phase (each entry has a single non-zero
contributor, so the sum is exact), and every rank reduces the chunk partials in the same fixed
order: all ranks see the same scalars, run the identical control flow, and the run is bitwise
the single-GPU run for any rank count.  New positions are computed per slice and
all-gathered.  Errors are agreed on by an all-reduce of the status word before anyone raises,
so no rank is left in a collective.

`ShardedMeshEvaluator` is backend-agnostic: `CudaShardBackend` drives the C ABI; the CPU test
suite plugs a NumPy backend into the same orchestration under gloo (tests/test_parallel_gloo.py).
"""

from __future__ import annotations

import ctypes

from . import _lib
from .pipeline import EvalResult, MeshEvaluator

CYC_ROW = 34   # {id, valence, 32 neighbour ids} int32
RES_ROW = 8    # {id, m, cx, cy, cz, E, obtuse, 0} float64


def shard_rows(n: int, nshards: int) -> int:
    """Rows per shard (include/scvt_b200.h scvt_shard_rows)."""
    return (n + nshards - 1) // nshards


def shard_range(n: int, shard: int, nshards: int):
    """Owned slots [lo, hi) of the bucket order."""
    cap = shard_rows(n, nshards)
    lo = min(n, shard * cap)
    return lo, min(n, lo + cap)


class CudaShardBackend:
    """The three shard entry points of the C ABI on one device context."""

    def __init__(self, evaluator: MeshEvaluator):
        self.ev = evaluator

    def cells(self, z, shard, nshards, cyc_send):
        ctx = self.ev._ensure_ctx(z.shape[0])
        ctx.call("scvt_shard_cells", _lib.dptr(z), z.shape[0], shard, nshards,
                 _lib.dptr(cyc_send), what="shard_cells")

    def moments(self, z, shard, nshards, cyc_all, res_send):
        """The shard's moments into res_send; returns its status word: an int, or (certified
        held cycles, no host read) a 1-element int32 device tensor."""
        ctx = self.ev._ensure_ctx(z.shape[0])
        if cyc_all is None:
            import torch

            st_dev = torch.empty(1, dtype=torch.int32, device=z.device)
            ctx.call("scvt_shard_moments_async", _lib.dptr(z), z.shape[0], shard, nshards,
                     _lib.dptr(res_send), _lib.dptr(st_dev), what="shard_moments")
            return st_dev
        st = ctypes.c_int32(0)
        ctx.call("scvt_shard_moments", _lib.dptr(z), z.shape[0], shard, nshards,
                 _lib.dptr(cyc_all) if cyc_all is not None else None, _lib.dptr(res_send),
                 ctypes.byref(st), what="shard_moments")
        return int(st.value)

    # ---- cycle reuse (include/scvt_b200.h: scvt_shard_recheck / plan / rebuild / install)
    def recheck(self, z, shard, nshards, rnd, bad) -> bool:
        ctx = self.ev._ensure_ctx(z.shape[0])
        ready = ctypes.c_int32(0)
        ctx.call("scvt_shard_recheck", _lib.dptr(z), z.shape[0], shard, nshards, rnd,
                 _lib.dptr(bad), ctypes.byref(ready), what="shard_recheck")
        return bool(ready.value)

    def flip_detect(self, z, shard, nshards):
        """Flip-mode certificate of the owned cells: ((cap, 4) int32 candidates, (count, bad))."""
        import torch

        n = z.shape[0]
        ctx = self.ev._ensure_ctx(n)
        cap = 4 * shard_rows(n, nshards) + 64
        cand = torch.empty((cap, 4), dtype=torch.int32, device=z.device)
        cnt = (ctypes.c_int32 * 2)()
        ctx.call("scvt_shard_flip_detect", _lib.dptr(z), n, shard, nshards, _lib.dptr(cand), cap,
                 cnt, what="shard_flip_detect")
        return cand, (int(cnt[0]), int(cnt[1]))

    def flip_rounds(self, z, nshards, cand_all, cap, counts) -> int:
        ctx = self.ev._ensure_ctx(z.shape[0])
        c = (ctypes.c_int64 * nshards)(*counts)
        nb = ctypes.c_int32(0)
        ctx.call("scvt_shard_flip_rounds", _lib.dptr(z), z.shape[0], nshards, _lib.dptr(cand_all),
                 cap, c, ctypes.byref(nb), what="shard_flip_rounds")
        return int(nb.value)

    def flip(self, z) -> int:
        """Flip repair of the held cycles, replicated on every rank (no exchange)."""
        ctx = self.ev._ensure_ctx(z.shape[0])
        nb = ctypes.c_int32(0)
        ctx.call("scvt_shard_flip", _lib.dptr(z), z.shape[0], ctypes.byref(nb),
                 what="shard_flip")
        return int(nb.value)

    def plan(self, n, nshards, bad_all):
        ctx = self.ev._ensure_ctx(n)
        counts = (ctypes.c_int64 * (nshards + 1))()
        ctx.call("scvt_shard_plan", n, nshards, _lib.dptr(bad_all), counts, what="shard_plan")
        return [int(c) for c in counts]

    def rebuild(self, n, shard, nshards, cap, rows_send):
        ctx = self.ev._ensure_ctx(n)
        ctx.call("scvt_shard_rebuild", n, shard, nshards, cap, _lib.dptr(rows_send),
                 what="shard_rebuild")

    def install(self, n, rows, nrows):
        ctx = self.ev._ensure_ctx(n)
        ctx.call("scvt_shard_install", n, _lib.dptr(rows), nrows, what="shard_install")

    def bad_buffer(self, n, device):
        import torch

        return torch.empty(n, dtype=torch.int32, device=device)

    def raise_status(self, status: int):
        ctx = self.ev._ensure_ctx(1)
        rc = ctx.lib.scvt_shard_status(ctx.ptr, int(status))
        _lib.check(rc, ctx.ptr, "evaluate (sharded)")

    def finish(self, z, nshards, res_all, q3=None, norms=None) -> EvalResult:
        import torch

        n = z.shape[0]
        ctx = self.ev._ensure_ctx(n)
        grad = torch.empty_like(z)
        first = torch.empty_like(z)
        mass = torch.empty(n, dtype=torch.float64, device=z.device)
        diag = torch.empty(n, dtype=torch.float64, device=z.device)
        sc = (ctypes.c_double * 5)()
        ctx.call("scvt_shard_finish_ex", _lib.dptr(z), n, nshards, _lib.dptr(res_all),
                 _lib.dptr(grad), _lib.dptr(first), _lib.dptr(mass), _lib.dptr(diag),
                 _lib.dptr(q3), _lib.dptr(norms), sc, what="shard_finish")
        return EvalResult(energy=float(sc[0]), grad=grad, grad_norm=float(sc[1]),
                          lloyd_diag=diag, first=first, mass=mass, obtuse_count=int(sc[2]),
                          min_diag=float(sc[3]),
                          dirderiv=float(sc[4]) if q3 is not None else float("nan"))

    def finish_slice(self, z, nshards, res_all, rank, world, red, reduce_sum, q3=None,
                     norms=None) -> EvalResult:
        """Arithmetic-layout finish: the rank's rows of every output, the evaluation scalars
        reduced over the chunks of all ranks (include/scvt_b200.h scvt_slice_finish)."""
        n = z.shape[0]
        lo, hi = slice_range(n, rank, world)
        ctx = self.ev._ensure_ctx(n)
        grad = z.new_empty((hi - lo, 3))
        first = z.new_empty((hi - lo, 3))
        mass = z.new_empty(hi - lo)
        diag = z.new_empty(hi - lo)
        ctx.call("scvt_slice_finish", _lib.dptr(z), n, nshards, _lib.dptr(res_all), rank, world,
                 _lib.dptr(grad), _lib.dptr(first), _lib.dptr(mass), _lib.dptr(diag),
                 _lib.dptr(q3), _lib.dptr(norms), _lib.dptr(red), what="slice_finish")
        reduce_sum(red[:5 * CHUNKS])
        sc = (ctypes.c_double * 5)()
        ctx.call("scvt_slice_scalars", _lib.dptr(red), sc, what="evaluate (sharded)")
        return EvalResult(energy=float(sc[0]), grad=grad, grad_norm=float(sc[1]),
                          lloyd_diag=diag, first=first, mass=mass, obtuse_count=int(sc[2]),
                          min_diag=float(sc[3]),
                          dirderiv=float(sc[4]) if q3 is not None else float("nan"))

    def buffers(self, n, nshards, device):
        import torch

        r = shard_rows(n, nshards)
        return (torch.empty((r, CYC_ROW), dtype=torch.int32, device=device),
                torch.empty((nshards * r, CYC_ROW), dtype=torch.int32, device=device),
                torch.empty((r, RES_ROW), dtype=torch.float64, device=device),
                torch.empty((nshards * r, RES_ROW), dtype=torch.float64, device=device))


CHUNKS = 1184         # include/scvt_b200.h SCVT_CHUNKS
MAX_RED_VALS = 176    # partial values per phase (Gram pass with m <= 16)


def slice_range(n: int, rank: int, world: int):
    """Owned generator ids [lo, hi) of the arithmetic layout (include/scvt_b200.h
    scvt_slice_range): whole chunks [rank C/W, (rank+1) C/W) of ceil(n/C) ids."""
    if world < 1 or CHUNKS % world:
        raise ValueError(f"the world size must divide {CHUNKS}, got {world}")
    ch = max(1, -(-n // CHUNKS))
    nc = CHUNKS // world
    return min(n, rank * nc * ch), min(n, (rank + 1) * nc * ch)


def slice_pad(n: int, world: int) -> int:
    """Rows per rank in a gathered buffer: the slices laid end to end, the last one padded."""
    return (CHUNKS // world) * max(1, -(-n // CHUNKS))


def _padded_view(t, rows: int):
    """The (rows, ...) tensor over the whole storage of a [:n] view made by `_padded`."""
    import torch

    full = torch.empty(0, dtype=t.dtype, device=t.device)
    return full.set_(t.untyped_storage(), 0, (rows,) + tuple(t.shape[1:]))


def _padded(n: int, world: int, cols, like):
    """A [:n] view of a (world * pad, cols) buffer: the layout the slice all-gather fills."""
    import torch

    shape = (world * slice_pad(n, world),) + ((cols,) if cols else ())
    return torch.empty(shape, dtype=like.dtype, device=like.device)[:n]


def _gather_slices(full, rank: int, world: int, group):
    """All-gather the owned block of every rank into `full` (a [:n] view from `_padded`)."""
    n = full.shape[0]
    pad = slice_pad(n, world)
    buf = _padded_view(full, world * pad)
    _all_gather(buf, buf[rank * pad:(rank + 1) * pad].clone(), group)
    return full


def _all_reduce_sum(t, group):
    import torch.distributed as dist

    if dist.get_backend(group) != "nccl" and t.device.type != "cpu":
        h = t.cpu()                          # gloo: staged through host memory
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
        return t
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class SliceOps:
    """The optimizer's vector algebra on one rank of the arithmetic layout (include/scvt_b200.h
    "arithmetic-layout slices"): the same methods as `optimizer._DeviceOps`, each a chunked
    C call, one all-reduce SUM of the chunk partials, and the fixed-order finish.  Positions
    stay replicated; trial and Lloyd points are computed on the owned rows and all-gathered."""

    def __init__(self, ctx, n: int, rank: int, world: int, group=None, reduce_sum=None,
                 gather=None):
        import torch

        self.ctx, self.n, self.rank, self.world, self.group = ctx, n, rank, world, group
        self.lo, self.hi = slice_range(n, rank, world)
        self.len = self.hi - self.lo
        self.red = torch.zeros(MAX_RED_VALS * CHUNKS, dtype=torch.float64,
                               device=f"cuda:{ctx.device}")
        self._reduce_sum = reduce_sum or (lambda t: _all_reduce_sum(t, group))
        self._gather = gather or (lambda full: _gather_slices(full, rank, world, group))

    def _sum(self, nval: int):
        if nval:
            self._reduce_sum(self.red[:nval * CHUNKS])

    def _rows(self, t):
        return t[self.lo:self.hi]

    # -- layout
    def vec3(self, z):
        return z.new_empty((self.len, 3))

    def scalars(self, z):
        return z.new_empty(self.len)

    def positions(self, z):
        return _padded(self.n, self.world, 3, z)

    def full(self, res: EvalResult) -> EvalResult:
        def g(t, cols):
            out = _padded(self.n, self.world, cols, t)
            out[self.lo:self.hi] = t
            return self._gather(out)

        return EvalResult(energy=res.energy, grad=g(res.grad, 3), grad_norm=res.grad_norm,
                          lloyd_diag=g(res.lloyd_diag, 0), first=g(res.first, 3),
                          migration=res.migration, mass=g(res.mass, 0),
                          obtuse_count=res.obtuse_count, min_diag=res.min_diag,
                          dirderiv=res.dirderiv)

    # -- history
    def history_clear(self):
        self.ctx.call("scvt_history_clear")

    def gamma(self) -> float:
        g = ctypes.c_double()
        self.ctx.call("scvt_history_gamma", ctypes.byref(g))
        return g.value

    def push(self, z_old, z_new, g_old, g_new):
        nval = ctypes.c_int32()
        red = _lib.dptr(self.red)
        self.ctx.call("scvt_slice_history_pair", _lib.dptr(self._rows(z_old)),
                      _lib.dptr(self._rows(z_new)), _lib.dptr(g_old), _lib.dptr(g_new), self.n,
                      self.rank, self.world, red, ctypes.byref(nval))
        self._sum(nval.value)
        pushed = ctypes.c_int32()
        mv = ctypes.c_double()
        self.ctx.call("scvt_slice_history_commit", red, self.n, self.rank, self.world,
                      ctypes.byref(pushed), ctypes.byref(mv))
        return bool(pushed.value), mv.value

    # -- directions
    def _reduce(self, nval: int):
        out = (ctypes.c_double * nval)()
        self.ctx.call("scvt_reduce_chunks", _lib.dptr(self.red), nval, None, out)
        return list(out)

    def direction_tangent(self, g, diag, gamma, z, q3):
        nval = ctypes.c_int32()
        red = _lib.dptr(self.red)
        self.ctx.call("scvt_slice_gram", _lib.dptr(g), _lib.dptr(diag), float(gamma), self.n,
                      self.rank, self.world, red, ctypes.byref(nval))
        self._sum(nval.value)
        self.ctx.call("scvt_slice_combine", _lib.dptr(g), _lib.dptr(diag), float(gamma),
                      _lib.dptr(self._rows(z)), self.n, self.rank, self.world, red,
                      _lib.dptr(q3), red)
        self._sum(2)
        qg, dphi0 = self._reduce(2)
        return qg, dphi0

    def scale(self, a, x, y):
        self.ctx.call("scvt_scale", float(a), _lib.dptr(x), x.numel(), _lib.dptr(y))

    def tangent(self, q, z, g, q3) -> float:
        self.ctx.call("scvt_slice_tangent", _lib.dptr(q), _lib.dptr(self._rows(z)), _lib.dptr(g),
                      self.n, self.rank, self.world, _lib.dptr(q3), _lib.dptr(self.red))
        self._sum(1)
        return self._reduce(1)[0]

    # -- new positions (owned rows, then all-gathered)
    def trial(self, z, q3, alpha, zt, norms):
        self.ctx.call("scvt_trial_point", _lib.dptr(self._rows(z)), _lib.dptr(q3), float(alpha),
                      self.len, _lib.dptr(self._rows(zt)), _lib.dptr(norms))
        self._gather(zt)

    def lloyd(self, first, z_out):
        import torch

        from .errors import CentroidAtOriginError

        bad = torch.zeros(CHUNKS, dtype=torch.float64, device=z_out.device)
        try:
            self.ctx.call("scvt_lloyd_step", _lib.dptr(first), self.len,
                          _lib.dptr(self._rows(z_out)), what="lloyd_step")
        except CentroidAtOriginError:
            bad[self.rank] = 1.0
        self._reduce_sum(bad)                        # everyone raises, or no one
        if float(bad.sum()) > 0.0:
            raise CentroidAtOriginError("a first moment is ~0 (Lloyd step)")
        self._gather(z_out)

    # -- replicated positions: computed identically on every rank
    def max_abs_diff(self, a, b) -> float:
        m = ctypes.c_double()
        self.ctx.call("scvt_max_abs_diff", _lib.dptr(a), _lib.dptr(b), a.numel(), ctypes.byref(m))
        return m.value

    def normalize(self, z):
        self.ctx.call("scvt_normalize_rows", _lib.dptr(z), self.n)


def _all_gather(out, inp, group):
    import torch.distributed as dist

    if out.numel() != dist.get_world_size(group) * inp.numel():
        raise ValueError(f"all-gather of {tuple(inp.shape)} into {tuple(out.shape)} for "
                         f"{dist.get_world_size(group)} ranks")
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
        return
    # gloo (CPU tests; CUDA tensors staged through host memory): the same collective on the
    # same shapes, so the CPU tests exercise exactly the NCCL call
    host = out.device.type != "cpu"
    src = (inp.cpu() if host else inp).contiguous()
    dst = out.cpu() if host or not out.is_contiguous() else out
    dist.all_gather_into_tensor(dst, src, group=group)
    if dst is not out:
        out.copy_(dst)


REUSE_ROUNDS = 4   # certificate passes before a full rebuild (same as the single-GPU loop)


def _flip_sharded(backend, z, shards, nshards, gather_counts, gather_cand):
    """Flip repair with the certificate pass sharded (include/scvt_b200.h
    scvt_shard_flip_detect / _rounds): each shard queues the non-Delaunay edges of its cells,
    the candidate lists are all-gathered, and every rank runs the same flip rounds on the
    concatenation.  True: certified; False: take the rebuild rounds; None: no held cycles."""
    import torch

    cands, counts = [], []
    for s in shards:
        cand, cnt = backend.flip_detect(z, s, nshards)
        cands.append(cand)
        counts.append(torch.tensor(cnt, dtype=torch.int64, device=cand.device))
    allc = gather_counts(counts).cpu().reshape(nshards, 2)
    if bool((allc[:, 0] < 0).any()):
        return None
    if int(allc[:, 1].sum()) > 0 or int(allc[:, 0].max()) > cands[0].shape[0]:
        return False                        # orientation/consistency failures or overflow
    cap = int(allc[:, 0].max())
    cand_all = gather_cand([c[:cap] for c in cands], cap) if cap else None
    return backend.flip_rounds(z, nshards, cand_all, cap, allc[:, 0].tolist()) == 0


def _reuse_cycles(backend, z, shards, nshards, bad, cyc_send, cyc_all, reduce_bad, gather_rows,
                  gather_counts=None, gather_cand=None):
    """The single-GPU reuse loop split at its exchanges (include/scvt_b200.h).  `shards` are
    the shards this process runs (one under torch.distributed, all when emulating);
    `reduce_bad(bad_of_each_shard) -> bad_all`, `gather_rows(rows_of_each_shard, cap)`,
    `gather_counts(counts_of_each_shard)` and `gather_cand(candidates_of_each_shard, cap)`
    are the collectives.  True when the held cycles were certified for z."""
    n = z.shape[0]
    if not hasattr(backend, "recheck"):
        return False
    if hasattr(backend, "flip_detect") and gather_counts is not None:
        if _flip_sharded(backend, z, shards, nshards, gather_counts, gather_cand):
            return True                               # repaired by flips, identically everywhere
    elif hasattr(backend, "flip") and backend.flip(z) == 0:
        return True
    for rnd in range(REUSE_ROUNDS):
        local = []
        for s in shards:
            if not backend.recheck(z, s, nshards, rnd, bad):
                return False                          # no previous cycles: identical on all ranks
            local.append(bad.clone() if len(shards) > 1 else bad)
        bad_all = reduce_bad(local)
        counts = backend.plan(n, nshards, bad_all)
        nbad = counts[nshards]
        if nbad == 0:
            return True
        if nbad > (3 * n) // 4 or rnd == REUSE_ROUNDS - 1:
            return False                              # churn too large: full rebuild
        cap = max(counts[:nshards])
        rows = []
        for s in shards:
            backend.rebuild(n, s, nshards, cap, cyc_send)
            rows.append(cyc_send[:cap].clone() if len(shards) > 1 else cyc_send[:cap])
        gather_rows(rows, cap)
        backend.install(n, cyc_all, nshards * cap)
    return False


def _all_reduce_max(t, group):
    import torch.distributed as dist

    if dist.get_backend(group) != "nccl" and t.device.type != "cpu":
        h = t.cpu()                          # gloo: staged through host memory
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        t.copy_(h)
        return t
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def sharded_evaluate(backend, z, rank: int, world: int, group=None, comm_device=None,
                     q3=None, norms=None, finish=None):
    """One evaluation on rank `rank` of `world` (collectives through torch.distributed).
    `finish(res_all)`, when given, replaces the replicated finish (arithmetic layout)."""
    import torch

    n = z.shape[0]
    dev = comm_device or z.device
    cyc_send, cyc_all, res_send, res_all = backend.buffers(n, world, dev)
    reused = False
    if hasattr(backend, "recheck"):
        bad = backend.bad_buffer(n, dev)

        def gather_rows(rows, cap):
            _all_gather(cyc_all[:world * cap], rows[0], group)

        def gather_counts(local):
            out = torch.empty(world * local[0].numel(), dtype=local[0].dtype,
                              device=local[0].device)
            _all_gather(out, local[0], group)
            return out

        def gather_cand(local, cap):
            out = torch.empty((world * cap, 4), dtype=local[0].dtype, device=local[0].device)
            _all_gather(out, local[0].contiguous(), group)
            return out

        reused = _reuse_cycles(backend, z, [rank], world, bad, cyc_send, cyc_all,
                               lambda local: _all_reduce_max(local[0], group), gather_rows,
                               gather_counts, gather_cand)
    if reused:
        status = backend.moments(z, rank, world, None, res_send)
    else:
        backend.cells(z, rank, world, cyc_send)
        _all_gather(cyc_all, cyc_send, group)
        status = backend.moments(z, rank, world, cyc_all, res_send)
    st = (status.to(cyc_send.device) if isinstance(status, torch.Tensor) else
          torch.tensor([status], dtype=torch.int32, device=cyc_send.device))
    st_all = torch.empty(world, dtype=torch.int32, device=cyc_send.device)
    _all_gather(st_all, st, group)                            # everyone raises, or no one
    status = 0
    for w in st_all.tolist():      # status words are bit sets: OR them, as one GPU does
        status |= int(w)
    if status:
        backend.raise_status(status)
    _all_gather(res_all, res_send, group)
    if finish is not None:
        return finish(res_all)
    if q3 is None:
        return backend.finish(z, world, res_all)
    return backend.finish(z, world, res_all, q3, norms)


def emulate_shards(backend, z, nshards: int, q3=None, norms=None):
    """All shards of one evaluation run back to back in one process (no collectives): the
    exchange buffers are filled slice by slice.  Used to test the sharded path on one GPU."""
    n = z.shape[0]
    cyc_send, cyc_all, res_send, res_all = backend.buffers(n, nshards, z.device)
    r = shard_rows(n, nshards)
    reused = False
    if hasattr(backend, "recheck"):
        bad = backend.bad_buffer(n, z.device)

        def reduce_bad(local):
            out = local[0]
            for b in local[1:]:
                out = out.maximum(b)
            return out

        def gather_rows(rows, cap):
            for s, rw in enumerate(rows):
                cyc_all[s * cap:(s + 1) * cap] = rw

        import torch

        reused = _reuse_cycles(backend, z, list(range(nshards)), nshards, bad, cyc_send,
                               cyc_all, reduce_bad, gather_rows, lambda local: torch.cat(local),
                               lambda local, cap: torch.cat(local))
    if not reused:
        for s in range(nshards):
            backend.cells(z, s, nshards, cyc_send)
            cyc_all[s * r:(s + 1) * r] = cyc_send
    status = 0
    words = []
    for s in range(nshards):
        words.append(backend.moments(z, s, nshards, None if reused else cyc_all, res_send))
        res_all[s * r:(s + 1) * r] = res_send
    for w in words:                 # device status words are read after every shard ran
        status |= int(w.item()) if hasattr(w, "item") else int(w)
    if status:
        backend.raise_status(status)
    if q3 is None:
        return backend.finish(z, nshards, res_all)
    return backend.finish(z, nshards, res_all, q3, norms)


class ShardedMeshEvaluator(MeshEvaluator):
    """`MeshEvaluator` whose evaluations are sharded over the ranks of a process group
    (one GPU per rank, backend NCCL).  With world size 1 it runs the same sharded code path
    with no communication."""

    def __init__(self, *args, group=None, backend=None, force_collectives=False, **kwargs):
        super().__init__(*args, **kwargs)
        import torch.distributed as dist

        from .errors import ConfigError

        if self.laplacian is not None:
            raise ConfigError("the graph Laplacian preconditioner runs on one GPU")

        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        self.backend = backend or CudaShardBackend(self)
        # force_collectives: a one-rank group still goes through every collective call (the
        # NCCL code path on a one-GPU box: tests/test_gpu_parity.py)
        self.collective = self.world > 1 or (force_collectives and dist.is_initialized())
        self._red = None

    def optimizer_ops(self, ctx, n: int):
        """One GPU: the all-rows algebra; several: this rank's arithmetic slice."""
        if not self.collective:
            ops = super().optimizer_ops(ctx, n)
            ops.stage_pairs = False      # the sharded evaluation has no staged-pair variant
            return ops
        return SliceOps(ctx, n, self.rank, self.world, self.group)

    def _sum(self, t):
        return _all_reduce_sum(t, self.group)

    def evaluate_device(self, z, q3=None, norms=None) -> EvalResult:
        """World size 1: all rows.  Several ranks: the vectors of the result hold this rank's
        arithmetic slice (`slice_range`); the scalars are global."""
        if not self.collective:
            r = emulate_shards(self.backend, z, 1, q3, norms)
        else:
            import torch

            if self._red is None:
                self._red = torch.zeros(MAX_RED_VALS * CHUNKS, dtype=torch.float64,
                                        device=z.device)
            r = sharded_evaluate(
                self.backend, z, self.rank, self.world, self.group, q3=q3, norms=norms,
                finish=lambda res_all: self.backend.finish_slice(
                    z, self.world, res_all, self.rank, self.world, self._red, self._sum, q3,
                    norms))
        r.migration = self._migration(z)
        self._region_fallback(z)      # replicated: every rank holds every certified cycle
        self.evaluations += 1
        return r

    def evaluate(self, points) -> EvalResult:
        """pipeline.py:261-279 with every row on every rank."""
        from .pipeline import to_numpy

        z, host = self._as_device(points)
        r = self.evaluate_device(z)
        if self.collective:
            r = SliceOps(self._ensure_ctx(z.shape[0]), z.shape[0], self.rank, self.world,
                         self.group).full(r)
        if host:
            r.grad, r.first, r.mass, r.lloyd_diag = to_numpy(r.grad, r.first, r.mass,
                                                             r.lloyd_diag)
        return r


__all__ = ["ShardedMeshEvaluator", "CudaShardBackend", "SliceOps", "sharded_evaluate",
           "emulate_shards", "shard_rows", "shard_range", "slice_range"]
