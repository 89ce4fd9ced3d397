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
rank certifies its owned cells at the new positions, the bad flags are all-reduced (max),
every rank derives the same bad set and re-check list, rebuilds its own bad cells, and only
those cycles are all-gathered; up to four rounds, then the full path above.

Positions and LBFGS state are replicated, so every rank runs the identical optimizer control
flow, and the outputs are bitwise identical to the single-GPU `scvt_evaluate` for any rank
count (tests/test_gpu_parity.py emulates 2/3/8 shards on one GPU).  Errors are agreed on by an
all-reduce of the status word before anyone raises, so no rank is left in a collective.

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

    def moments(self, z, shard, nshards, cyc_all, res_send) -> int:
        ctx = self.ev._ensure_ctx(z.shape[0])
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

    def buffers(self, n, nshards, device):
        import torch

        r = shard_rows(n, nshards)
        return (torch.empty((r, CYC_ROW), dtype=torch.int32, device=device),
                torch.empty((nshards * r, CYC_ROW), dtype=torch.int32, device=device),
                torch.empty((r, RES_ROW), dtype=torch.float64, device=device),
                torch.empty((nshards * r, RES_ROW), dtype=torch.float64, device=device))


def _all_gather(out, inp, group):
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
        return
    # gloo (CPU tests; CUDA tensors staged through host memory): list form
    host = out.device.type != "cpu"
    src = inp.cpu() if host else inp
    dst = out.cpu() if host else out
    r = src.shape[0]
    parts = [dst[k * r:(k + 1) * r] for k in range(dst.shape[0] // r)]
    dist.all_gather(parts, src, group=group)
    if host:
        out.copy_(dst)


REUSE_ROUNDS = 4   # certificate passes before a full rebuild (same as the single-GPU loop)


def _reuse_cycles(backend, z, shards, nshards, bad, cyc_send, cyc_all, reduce_bad, gather_rows):
    """The single-GPU reuse loop split at its exchanges (include/scvt_b200.h).  `shards` are
    the shards this process runs (one under torch.distributed, all when emulating);
    `reduce_bad(bad_of_each_shard) -> bad_all` and `gather_rows(rows_of_each_shard, cap)`
    are the two collectives.  True when the held cycles were certified for z."""
    n = z.shape[0]
    if not hasattr(backend, "recheck"):
        return False
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
                     q3=None, norms=None):
    """One evaluation on rank `rank` of `world` (collectives through torch.distributed)."""
    import torch

    n = z.shape[0]
    dev = comm_device or z.device
    cyc_send, cyc_all, res_send, res_all = backend.buffers(n, world, dev)
    reused = False
    if hasattr(backend, "recheck"):
        bad = backend.bad_buffer(n, dev)

        def gather_rows(rows, cap):
            _all_gather(cyc_all[:world * cap], rows[0], group)

        reused = _reuse_cycles(backend, z, [rank], world, bad, cyc_send, cyc_all,
                               lambda local: _all_reduce_max(local[0], group), gather_rows)
    if reused:
        status = backend.moments(z, rank, world, None, res_send)
    else:
        backend.cells(z, rank, world, cyc_send)
        _all_gather(cyc_all, cyc_send, group)
        status = backend.moments(z, rank, world, cyc_all, res_send)
    st = torch.tensor([status], dtype=torch.int32, device=cyc_send.device)
    _all_reduce_max(st, group)                                # everyone raises, or no one
    if int(st.item()):
        backend.raise_status(int(st.item()))
    _all_gather(res_all, res_send, group)
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

        reused = _reuse_cycles(backend, z, list(range(nshards)), nshards, bad, cyc_send,
                               cyc_all, reduce_bad, gather_rows)
    if not reused:
        for s in range(nshards):
            backend.cells(z, s, nshards, cyc_send)
            cyc_all[s * r:(s + 1) * r] = cyc_send
    worst = 0
    for s in range(nshards):
        worst = max(worst, backend.moments(z, s, nshards, None if reused else cyc_all, res_send))
        res_all[s * r:(s + 1) * r] = res_send
    if worst:
        backend.raise_status(worst)
    if q3 is None:
        return backend.finish(z, nshards, res_all)
    return backend.finish(z, nshards, res_all, q3, norms)


class ShardedMeshEvaluator(MeshEvaluator):
    """`MeshEvaluator` whose evaluations are sharded over the ranks of a process group
    (one GPU per rank, backend NCCL).  With world size 1 it runs the same sharded code path
    with no communication."""

    def __init__(self, *args, group=None, backend=None, **kwargs):
        super().__init__(*args, **kwargs)
        import torch.distributed as dist

        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        self.backend = backend or CudaShardBackend(self)

    def evaluate_device(self, z, q3=None, norms=None) -> EvalResult:
        if self.world == 1:
            r = emulate_shards(self.backend, z, 1, q3, norms)
        else:
            r = sharded_evaluate(self.backend, z, self.rank, self.world, self.group, q3=q3,
                                 norms=norms)
        self.evaluations += 1
        return r


__all__ = ["ShardedMeshEvaluator", "CudaShardBackend", "sharded_evaluate", "emulate_shards",
           "shard_rows", "shard_range"]
