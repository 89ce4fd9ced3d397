"""The multi-GPU orchestration (paper_1709_06924_b200/parallel.py) under gloo with world
size 2 on CPU.  The CUDA backend cannot run here, so a NumPy stand-in backend (oracle
arithmetic, same exchange-row formats) is plugged into the SAME `sharded_evaluate`: shard
ranges, packing, both all-gathers, the status agreement and the final scatter/reduction are
what is under test.  The CUDA backend's bitwise equivalence across shard counts is checked on
the B200 (tests/test_gpu_parity.py::test_sharded_evaluation_is_bitwise_identical)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1709_06924_b200.parallel import CYC_ROW, RES_ROW, shard_range, shard_rows, sharded_evaluate


def _true_cycles(z):
    """Delaunay cycles of every generator (Qhull via the oracle), CCW from the min id."""
    n = len(z)
    nxt = [dict() for _ in range(n)]
    for a, b, c in O.convex_hull_delaunay(z):
        nxt[a][b] = c
        nxt[b][c] = a
        nxt[c][a] = b
    out = []
    for i in range(n):
        start = min(nxt[i])
        cyc, cur = [], start
        while True:
            cyc.append(cur)
            cur = nxt[i][cur]
            if cur == start:
                break
        out.append(cyc)
    return out


class NumpyShardBackend:
    def __init__(self, density="const", rule="4pt", fail_on=None):
        self.density = O.density_for(density)
        self.rule = O.RULES[rule]
        self.fail_on = fail_on
        self.held = None          # cycles of the last evaluation (all generators)
        self.rounds = []          # bad-set sizes of the reuse rounds (test introspection)

    # ---- cycle reuse, same protocol as CudaShardBackend (certificate stand-in: the held
    # cycle differs from the Delaunay cycle at the new positions)
    def bad_buffer(self, n, device):
        return torch.zeros(n, dtype=torch.int32)

    def recheck(self, z, shard, nshards, rnd, bad):
        zz = z.numpy()
        n = len(zz)
        if rnd == 0:
            if self.held is None or len(self.held) != n:
                return False
            self.truth = _true_cycles(zz)
        lo, hi = shard_range(n, shard, nshards)
        bad.zero_()
        for i in range(lo, hi):
            if rnd > 0 and not self.recheck_set[i]:
                continue
            if self.held[i] != self.truth[i]:
                bad[i] = 1
                bad[self.held[i]] = 1
        return True

    def plan(self, n, nshards, bad_all):
        b = np.nonzero(bad_all.numpy())[0]
        self.bad_set = b
        rs = np.zeros(n, dtype=bool)
        rs[b] = True
        for i in b:
            rs[self.held[i]] = True
        self.recheck_set = rs
        self.rounds.append(len(b))
        cap = shard_rows(n, nshards)
        return [int(np.sum((b >= s * cap) & (b < (s + 1) * cap))) for s in range(nshards)] + [len(b)]

    def rebuild(self, n, shard, nshards, cap, rows_send):
        lo, hi = shard_range(n, shard, nshards)
        rows_send[:cap].fill_(-1)
        for q, i in enumerate(i for i in self.bad_set if lo <= i < hi):
            cyc = self.truth[i]
            rows_send[q, 0] = int(i)
            rows_send[q, 1] = len(cyc)
            rows_send[q, 2:2 + len(cyc)] = torch.tensor(cyc, dtype=torch.int32)

    def install(self, n, rows, nrows):
        for r in rows[:nrows].numpy():
            if r[0] >= 0:
                self.held[r[0]] = [int(v) for v in r[2:2 + r[1]]]

    def buffers(self, n, nshards, device):
        r = shard_rows(n, nshards)
        return (torch.zeros((r, CYC_ROW), dtype=torch.int32),
                torch.zeros((nshards * r, CYC_ROW), dtype=torch.int32),
                torch.zeros((r, RES_ROW), dtype=torch.float64),
                torch.zeros((nshards * r, RES_ROW), dtype=torch.float64))

    def cells(self, z, shard, nshards, cyc_send):
        z = z.numpy()
        n = len(z)
        tri = O.convex_hull_delaunay(z)
        nxt = [dict() for _ in range(n)]
        for a, b, c in tri:
            nxt[a][b] = c
            nxt[b][c] = a
            nxt[c][a] = b
        lo, hi = shard_range(n, shard, nshards)
        cyc_send.fill_(-1)
        for q, i in enumerate(range(lo, hi)):
            start = min(nxt[i])
            cyc, cur = [], start
            while True:
                cyc.append(cur)
                cur = nxt[i][cur]
                if cur == start:
                    break
            cyc_send[q, 0] = i
            cyc_send[q, 1] = len(cyc)
            cyc_send[q, 2:2 + len(cyc)] = torch.tensor(cyc, dtype=torch.int32)

    def moments(self, z, shard, nshards, cyc_all, res_send):
        zz = z.numpy()
        n = len(zz)
        if cyc_all is None:                                 # cycles certified by reuse
            rows = np.full((n, CYC_ROW), -1, dtype=np.int64)
            for i, cyc in enumerate(self.held):
                rows[i, 0], rows[i, 1] = i, len(cyc)
                rows[i, 2:2 + len(cyc)] = cyc
        else:
            rows = cyc_all.numpy()
            rows = rows[rows[:, 0] >= 0]
            ids = np.sort(rows[:, 0])
            if not np.array_equal(ids, np.arange(n)):
                return 1 << 4                               # ST_INCONSISTENT
            self.held = [None] * n
            for r in rows:
                self.held[r[0]] = [int(v) for v in r[2:2 + r[1]]]
        tris = []
        for r in rows:
            i, d = r[0], r[1]
            for t in range(d):
                a, b = r[2 + t], r[2 + (t + 1) % d]
                if i < a and i < b:
                    tris.append((i, a, b))
        tri = O.canonical_sort(np.array(tris))
        f = O.build_fans(zz, tri)
        nodes = np.einsum("qv,svj->sqj", self.rule.bary, f.verts)
        nodes = nodes / np.linalg.norm(nodes, axis=-1, keepdims=True)
        rho = O.eval_density(self.density, nodes)
        w = self.rule.weights
        sub_m = (rho @ w) * f.signed_area
        sub_c = np.einsum("sq,q,sqj->sj", rho, w, nodes) * f.signed_area[:, None]
        diff = nodes - zz[f.cells][:, None, :]
        sub_e = ((rho * np.einsum("sqj,sqj->sq", diff, diff)) @ w) * f.signed_area
        m = np.zeros(n); c = np.zeros((n, 3)); e = np.zeros(n)
        np.add.at(m, f.cells, sub_m); np.add.at(c, f.cells, sub_c); np.add.at(e, f.cells, sub_e)
        lo, hi = shard_range(n, shard, nshards)
        res_send.fill_(0.0)
        res_send[:, 0] = -1.0
        for q, i in enumerate(range(lo, hi)):
            res_send[q, :6] = torch.tensor([i, m[i], c[i, 0], c[i, 1], c[i, 2], e[i]])
        if self.fail_on is not None and shard == self.fail_on:
            return 1 << 0                                   # ST_DUPLICATE on one rank only
        return 0

    def raise_status(self, status):
        raise RuntimeError(f"status {status}")

    def finish(self, z, nshards, res_all):
        zz = z.numpy()
        n = len(zz)
        rows = res_all.numpy()
        rows = rows[rows[:, 0] >= 0]
        order = rows[:, 0].astype(np.int64)
        first = np.zeros((n, 3)); e = np.zeros(n); m = np.zeros(n)
        first[order] = rows[:, 2:5]; e[order] = rows[:, 5]; m[order] = rows[:, 1]
        cz = np.einsum("ij,ij->i", first, zz)
        grad = 2.0 * cz[:, None] * zz - 2.0 * first
        return {"energy": float(e.sum()), "first": first, "grad": grad, "mass": m,
                "covered": len(order)}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _moved(z0, scale=0.001, seed=9):
    rng = np.random.default_rng(seed)
    z = z0 + scale * rng.standard_normal(z0.shape)
    return z / np.linalg.norm(z, axis=1, keepdims=True)


def _worker(rank, world, port, fail_on, out, second):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z0 = O.random_sphere_points(1202, 5)
        be = NumpyShardBackend(fail_on=fail_on)
        try:
            r = sharded_evaluate(be, torch.from_numpy(z0), rank, world)
            if second:        # same backend, moved points: the reuse rounds
                r = sharded_evaluate(be, torch.from_numpy(_moved(z0)), rank, world)
            out[rank] = {"energy": r["energy"], "first": r["first"], "covered": r["covered"],
                         "rounds": list(be.rounds)}
        except RuntimeError as exc:
            out[rank] = {"error": str(exc)}
    finally:
        dist.destroy_process_group()


def _run(world, fail_on=None, second=False):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), fail_on, out, second), nprocs=world, join=True)
    return dict(out)


def test_gloo_two_ranks_match_single_process():
    out = _run(2)
    z = O.random_sphere_points(1202, 5)
    ref = O.Evaluator(O.density_for("const"), "4pt", 0).evaluate(z)
    for rank in (0, 1):
        assert out[rank]["covered"] == 1202
        np.testing.assert_allclose(out[rank]["first"], ref.first, rtol=0, atol=1e-15)
        assert abs(out[rank]["energy"] - ref.energy) <= 1e-14 * ref.energy
    np.testing.assert_array_equal(out[0]["first"], out[1]["first"])
    assert out[0]["energy"] == out[1]["energy"]


def test_gloo_error_on_one_rank_raises_on_all():
    out = _run(2, fail_on=1)
    assert "error" in out[0] and "error" in out[1]


def test_gloo_cycle_reuse_rounds():
    """Second evaluation at moved points: the reuse protocol (per-shard certificate, max
    all-reduce of the bad flags, identical plan on both ranks, rebuilt rows all-gathered)
    must end with the Delaunay cycles of the new positions on both ranks."""
    out = _run(2, second=True)
    z = _moved(O.random_sphere_points(1202, 5))
    ref = O.Evaluator(O.density_for("const"), "4pt", 0).evaluate(z)
    assert out[0]["rounds"] == out[1]["rounds"]
    assert out[0]["rounds"][0] > 0 and out[0]["rounds"][-1] == 0   # some churn, then certified
    for rank in (0, 1):
        assert out[rank]["covered"] == 1202
        np.testing.assert_allclose(out[rank]["first"], ref.first, rtol=0, atol=1e-15)
        assert abs(out[rank]["energy"] - ref.energy) <= 1e-14 * ref.energy
    np.testing.assert_array_equal(out[0]["first"], out[1]["first"])


# ---- arithmetic layout (parallel.SliceOps): partition, exact chunk-partial exchange, gathers
def _chunk_dots(a, b, n, lo, hi, world):
    """NumPy stand-in of a chunked dot-product phase (include/scvt_b200.h slices): per chunk
    partials of the owned rows, zeros elsewhere."""
    from paper_1709_06924_b200.parallel import CHUNKS

    ch = max(1, -(-n // CHUNKS))
    red = np.zeros(CHUNKS)
    for c in range(CHUNKS):
        c0, c1 = max(lo, c * ch), min(hi, (c + 1) * ch)
        if c0 < c1:
            red[c] = float(np.sum(a[c0:c1] * b[c0:c1]))
    return red


def _slice_worker(rank, world, port, out):
    from paper_1709_06924_b200.parallel import (_all_reduce_sum, _gather_slices, _padded,
                                                slice_range)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 40962
        rng = np.random.default_rng(3)
        a, b = rng.standard_normal(n), rng.standard_normal(n)
        lo, hi = slice_range(n, rank, world)
        red = torch.from_numpy(_chunk_dots(a, b, n, lo, hi, world))
        _all_reduce_sum(red, None)
        z = torch.from_numpy(rng.standard_normal((n, 3)))
        full = _padded(n, world, 3, z)
        full[lo:hi] = z[lo:hi]                     # only the owned rows are valid locally
        _gather_slices(full, rank, world, None)
        out[rank] = {"red": red.numpy().copy(), "lohi": (lo, hi), "full": full.numpy().copy(),
                     "z": z.numpy()}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_arithmetic_slices(world):
    """Rank slices tile [0, n) with whole chunks; the all-reduced chunk partials equal the
    single-process partials bitwise (one non-zero contributor per entry); the padded
    all-gather reassembles the owned rows of every rank."""
    from paper_1709_06924_b200.parallel import CHUNKS, slice_range

    for n in (4, 2562, 40962, 655362, 2621442):
        for w in (1, 2, 4, 8):
            bounds = [slice_range(n, r, w) for r in range(w)]
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            assert all(bounds[r][1] == bounds[r + 1][0] for r in range(w - 1))
    with pytest.raises(ValueError):
        slice_range(100, 0, 3)                    # 3 does not divide the chunk count
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_slice_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    n = 40962
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    ref = _chunk_dots(a, b, n, 0, n, 1)
    for r in range(world):
        assert np.array_equal(out[r]["red"], ref)
        assert np.array_equal(out[r]["full"], out[r]["z"])
    assert len(ref) == CHUNKS


# ---- sharded flip repair protocol (parallel._flip_sharded): counts and candidates gathered
class _FlipMock:
    """Stand-in for the flip entry points: shard s queues s + 1 candidate rows {s, k, 0, 0};
    the rounds record what they were given."""

    def __init__(self, bad_on=None):
        self.bad_on = bad_on
        self.seen = None

    def flip_detect(self, z, shard, nshards):
        cap = 8
        cand = torch.zeros((cap, 4), dtype=torch.int32)
        for k in range(shard + 1):
            cand[k] = torch.tensor([shard, k, 0, 0], dtype=torch.int32)
        return cand, (shard + 1, 1 if shard == self.bad_on else 0)

    def flip_rounds(self, z, nshards, cand_all, cap, counts):
        self.seen = [cand_all[r * cap:r * cap + counts[r]].tolist() for r in range(nshards)]
        return 0


def _flip_worker(rank, world, port, bad_on, out):
    from paper_1709_06924_b200.parallel import _all_gather, _flip_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        be = _FlipMock(bad_on)

        def gather_counts(local):
            o = torch.empty(world * local[0].numel(), dtype=local[0].dtype)
            _all_gather(o, local[0], None)
            return o

        def gather_cand(local, cap):
            o = torch.empty((world * cap, 4), dtype=local[0].dtype)
            _all_gather(o, local[0].contiguous(), None)
            return o

        ok = _flip_sharded(be, torch.zeros((10, 3)), [rank], world, gather_counts, gather_cand)
        out[rank] = {"ok": ok, "seen": be.seen}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bad_on", [None, 1])
def test_gloo_sharded_flip_protocol(bad_on):
    """Every rank gets every shard's flip candidates in rank order (padded all-gather, counts
    first); a bad cell on any rank sends all of them to the rebuild rounds."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_flip_worker, args=(2, _free_port(), bad_on, out), nprocs=2, join=True)
    for r in (0, 1):
        if bad_on is None:
            assert out[r]["ok"] is True
            assert out[r]["seen"] == [[[0, 0, 0, 0]], [[1, 0, 0, 0], [1, 1, 0, 0]]]
        else:
            assert out[r]["ok"] is False and out[r]["seen"] is None
