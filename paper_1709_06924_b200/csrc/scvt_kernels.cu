// scvt_kernels.cu — sm_100a kernels + C ABI (include/scvt_b200.h) of the SCVT hot path.
//
// Pipeline of one evaluation (MeshEvaluator.evaluate, pipeline.py:261-279):
//   k_bucket_keys -> CUB radix sort -> k_bucket_start -> k_gather_sorted   (cube-map grid)
//   k_cells        per-generator Voronoi cell by half-plane clipping with a security-radius
//                  certificate  (replaces Qhull, delaunay.py:181-202)
//   k_verify       cycle consistency + local-Delaunay filter on every edge
//   CUB scan -> k_fill_incidences   (one incidence per (generator, incident triangle))
//   k_quad         fan sub-triangles + subdivided quadrature + density, FP64
//                  (delaunay.py:337-407, cvt_core.py:55-117, density.py:116-129)
//   k_gather       per-generator moments -> gradient epilogue (pipeline.py:265-279)
//   k_reduce_*     deterministic fixed-shape reductions (energy, |g|^2, obtuse count)
// plus the LBFGS vector kernels (optimizer.py:79-167, 322-355).
//
// All reductions use a fixed grid shape so results are bitwise reproducible run to run.

#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "scvt_device.cuh"
#include "scvt_cells_warp.cuh"
#include "../../include/scvt_b200.h"

using namespace scvt;

namespace {

constexpr int RED_BLOCKS = 296;      // 2 x 148 SMs: fixed reduction shape
// The optimizer's reductions run over a fixed partition of the generator ids into CHUNKS
// chunks of ceil(n / CHUNKS) ids (include/scvt_b200.h, SCVT_CHUNKS): one block per chunk, one
// partial per chunk and value, then a fixed-order pass over the CHUNKS partials.  A rank of an
// arithmetic-layout run owns a contiguous range of whole chunks, so the same partials come out
// whatever the rank count.
constexpr int CHUNKS = SCVT_CHUNKS;
constexpr int MAX_RED_VALS = 176;    // >= 2K + K(K+1)/2 + 1 for K <= 16
constexpr int RED_THREADS = 256;
constexpr int VEC_THREADS = 256;
#ifndef QUAD_THREADS_DEF
#define QUAD_THREADS_DEF 128
#endif
constexpr int QUAD_THREADS = QUAD_THREADS_DEF;   // k_quad block size
#ifndef QUAD_MINB
#define QUAD_MINB 5      // k_quad fast path: CTAs per SM the register budget must allow
#endif
#ifndef QUAD_MINB2
#define QUAD_MINB2 4     // two-centre fast path
#endif
constexpr int CELL_THREADS = 64;
constexpr int PART_ROW = 10;         // per-incidence partials: [half][m, cx, cy, cz, E]
constexpr int MAX_SLOTS = 64;        // partial-sum slots
constexpr int MAX_SHARDS = 256;      // sharded evaluation: ranks per evaluation

// ------------------------------------------------------------------ grid kernels
__global__ void k_bucket_keys(const double* __restrict__ z, int n, int G,
                              uint32_t* __restrict__ keys, int* __restrict__ vals) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = bucket_key(load3(z, i), G);
    vals[i] = i;
}

// start[b] = first sorted slot with key >= b: slot p fills the buckets (key[p-1], key[p]]
__global__ void k_bucket_start(const uint32_t* __restrict__ skeys, int n, int nb,
                               int* __restrict__ start) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > n) return;
    int lo = p == 0 ? 0 : (int)skeys[p - 1] + 1;
    int hi = p == n ? nb : (int)skeys[p];
    for (int b = lo; b <= hi; ++b) start[b] = p;
}

__global__ void k_gather_sorted(const double* __restrict__ z, const int* __restrict__ ids, int n,
                                double* __restrict__ zs) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int i = ids[p];
    double4 v = make_double4(z[3 * (int64_t)i], z[3 * (int64_t)i + 1], z[3 * (int64_t)i + 2], 0.0);
    reinterpret_cast<double4*>(zs)[p] = v;
}

// Fast path: one warp per generator (bucket order), polygon in registers.
__global__ void __launch_bounds__(CELL_WARPS * 32, 4)
k_cells_warp(GridView g, int p_lo, int p_hi, const int* __restrict__ list,
             const int* __restrict__ list_n, int* __restrict__ nbr, int* __restrict__ deg,
             int* __restrict__ status, int* __restrict__ stats,
             unsigned long long* __restrict__ diag, int* __restrict__ queue = nullptr) {
    __shared__ double s_c2[CELL_WARPS][WCAND];
    __shared__ int s_j[CELL_WARPS][WCAND];
    __shared__ int s_p[CELL_WARPS][WCAND];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // a host-sized grid runs one trip; a fixed (resident) grid serves a list whose length
    // only the device knows by pulling cells from an atomic queue (dynamic balance: cell
    // costs vary by orders of magnitude)
    auto next = [&](int64_t cur) -> int64_t {
        if (!queue) return cur < 0 ? (int64_t)blockIdx.x * CELL_WARPS + w
                                   : cur + (int64_t)gridDim.x * CELL_WARPS;
        int t = 0;
        if (lane == 0) t = atomicAdd(queue, 1);
        return __shfl_sync(0xffffffffu, t, 0);
    };
    for (int64_t idx = next(-1);; idx = next(idx)) {
    int64_t p;
    if (list) {                 // rebuild of a compacted list of sorted slots
        if (idx >= *list_n) return;
        p = list[idx];
    } else {
        p = p_lo + idx;
        if (p >= p_hi) return;   // warp-uniform
    }
    const int i = g.ids[p];
    const double* q = g.zs + 4 * p;
    V3 zi = v3(q[0], q[1], q[2]);
    CellStats cs;
    int d = build_cell_warp(g, i, zi, lane, s_c2[w], s_j[w], s_p[w], nbr + (int64_t)i * MAXDEG, &cs);
    if (lane == 0) {
        if (d == -ST_POLY_OVERFLOW) {
            deg[i] = -1;                         // single-thread fallback below
            atomicAdd(&stats[5], 1);
        } else if (d < 0) {
            atomicOr(status, -d);
            deg[i] = 0;
        } else {
            deg[i] = d;
            atomicMax(&stats[0], d);
        }
        if (cs.rounds > 1) atomicAdd(&stats[1], 1);
        atomicMax(&stats[2], cs.passes);
        if (cs.tie_breaks) atomicAdd(&stats[4], cs.tie_breaks);
        if (cs.sweep_visits) {
            atomicAdd(&stats[6], 1);
            atomicAdd(&stats[7], cs.sweep_visits >> 5);
        }
        if (diag) {
            atomicAdd(&diag[0], 1ull);
            atomicAdd(&diag[1], (unsigned long long)cs.passes);
            atomicAdd(&diag[2], (unsigned long long)cs.scanned);
            atomicAdd(&diag[3], (unsigned long long)cs.cands);
            atomicAdd(&diag[4], (unsigned long long)cs.clips);
            atomicAdd(&diag[5], (unsigned long long)cs.rounds);
            atomicMax(&diag[6], (unsigned long long)(cs.sweep_visits >> 5));
            atomicMax(&diag[7], (unsigned long long)cs.clips);
            atomicMax(&diag[8], (unsigned long long)cs.scanned);
            atomicMax(&diag[9], (unsigned long long)cs.passes);
        }
    }
    __syncwarp();
    }
}

// Fallback: one thread per generator the warp builder handed back (deg == -1).
__global__ void __launch_bounds__(CELL_THREADS)
k_cells(GridView g, int p_lo, int p_hi, const int* __restrict__ list,
        const int* __restrict__ list_n, int* __restrict__ nbr, int* __restrict__ deg,
        int* __restrict__ status, int* __restrict__ stats) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x;; idx += gridDim.x * blockDim.x) {
    int p;
    if (list) {
        if (idx >= *list_n) return;
        p = list[idx];
    } else {
        p = p_lo + idx;
        if (p >= p_hi) return;
    }
    int i = g.ids[p];
    if (deg[i] != -1) continue;
    V3 zi = v3(g.zs[4 * (int64_t)p], g.zs[4 * (int64_t)p + 1], g.zs[4 * (int64_t)p + 2]);
    Poly P, T;
    CellStats cs;
    int d = build_cell(g, i, zi, nbr + (int64_t)i * MAXDEG, &cs, P, T);
    if (d < 0) {
        atomicOr(status, -d);
        deg[i] = 0;
    } else {
        deg[i] = d;
        atomicMax(&stats[0], d);
    }
    if (cs.tie_breaks) atomicAdd(&stats[4], cs.tie_breaks);
    }
}

__device__ __forceinline__ int find_in_cycle(const int* __restrict__ row, int d, int x) {
    for (int k = 0; k < d; ++k)
        if (row[k] == x) return k;
    return -1;
}

// Certificate of a set of cycles at positions z, per edge (i, n_t) with triangles
// (i, n_t, n_{t+1}) and (i, n_{t-1}, n_t): (1) consistency — the triangle appears in n_t's
// cycle as (n_t, n_{t+1}, i); (2) positive orientation det[z_i, z_a, z_b] > 0; (3) local
// Delaunay — orient(z_i, z_a, z_b, z_c) < 0 decided by the robust predicate (FP64 filter ->
// double-double -> SoS).  Consistent + positively oriented + locally Delaunay everywhere
// means the cycles are THE (SoS-)Delaunay triangulation, however they were produced.
// mode 0: failures set status bits (certificate of a fresh build);
// mode 1: failures mark the cells of the offending triangle/quad in bad[] (reuse check).
__device__ __forceinline__ void mark_bad(int mode, int* status, int bit, int* bad, int* nbad,
                                         int i, int a, int b, int c) {
    if (mode == 0) { atomicOr(status, bit); return; }
    const int v[4] = {i, a, b, c};
    for (int k = 0; k < 4; ++k)
        if (v[k] >= 0 && atomicExch(&bad[v[k]], 1) == 0) atomicAdd(nbad, 1);
}

#ifdef SCVT_PROBE_FLIPS
__device__ unsigned long long g_probe[4];
#endif

// mode 2 (flip repair): an edge failing only the in-circle test is not marked bad but queued
// once (from its lower-id end) as a flip candidate {i, a, b, c}: triangles (i, a, b) and
// (i, c, a) -> (i, c, b) and (c, a, b).  Orientation and consistency failures mark bad as in
// mode 1.  list_ids: `list` holds generator ids instead of sorted slots.
#ifndef VERIFY_LANES_DEF
#define VERIFY_LANES_DEF 4
#endif
constexpr int VERIFY_LANES = VERIFY_LANES_DEF;   // threads per cell in k_verify

struct FlipQueue {
    int4* cand;
    int* ncand;
    int cap;
};

// Block-local staging of detected flip candidates: same-address global atomics serialise at
// ~4 ns each (20k candidates queued one atomicAdd at a time were most of the detection pass),
// so a block collects its candidates in shared memory and reserves their slots in the global
// queue with ONE atomicAdd when it flushes.
constexpr int SINK_CAP = 512;
struct CandSink {
    int4* q;      // shared [SINK_CAP]
    int* n;       // shared counter
};

__device__ __forceinline__ void queue_overflow(const int4 c, int* bad, int* nbad) {
    const int vv[4] = {c.x, c.y, c.z, c.w};     // cannot hold it: those cells are rebuilt
    for (int q = 0; q < 4; ++q)
        if (atomicExch(&bad[vv[q]], 1) == 0) atomicAdd(nbad, 1);
}

__device__ __forceinline__ void sink_push(const CandSink& sk, const FlipQueue& fq, const int4 c,
                                          int* bad, int* nbad) {
    const int k = atomicAdd(sk.n, 1);
    if (k < SINK_CAP) { sk.q[k] = c; return; }
    const int g = atomicAdd(fq.ncand, 1);       // staging full: straight to the global queue
    if (g < fq.cap) fq.cand[g] = c;
    else queue_overflow(c, bad, nbad);
}

// all threads of the block: move the staged candidates to the global queue (one atomicAdd)
__device__ __forceinline__ void sink_flush(const CandSink& sk, const FlipQueue& fq, int* bad,
                                           int* nbad) {
    __shared__ int s_base;
    __syncthreads();
    const int m = min(*sk.n, SINK_CAP);
    if (threadIdx.x == 0 && m > 0) s_base = atomicAdd(fq.ncand, m);
    __syncthreads();
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
        const int g = s_base + k;
        if (g < fq.cap) fq.cand[g] = sk.q[k];
        else queue_overflow(sk.q[k], bad, nbad);
    }
    __syncthreads();
    if (threadIdx.x == 0) *sk.n = 0;
    __syncthreads();
}

// Arguments of one certificate pass (k_verify, and the fused flip-round kernel).
struct VerifyArgs {
    const double* z;
    const int* ids;
    int p_lo, p_hi;
    const int* list;
    const int* list_n;
    const int* nbr;
    const int* deg;
    uint8_t* amb;
    int* status;
    int* stats;
    int mode;
    int* bad;
    int* nbad;
    FlipQueue fq;
    int list_ids;
    int list_len;       // >= 0: the list's length (entries < 0 are holes); < 0: read *list_n
};

// loads of the cycles: through the read-only path when an earlier launch wrote them (RO), plain
// L2 loads inside the kernel that rewrites them between its own rounds (k_flip_tail)
template <bool RO>
__device__ __forceinline__ int ldc(const int* p) {
    if (RO) return __ldg(p);
    return __ldcg(p);
}

// one (cell, lane) work item of the certificate; true once past the end of the work.
// Mode 2 runs on cycles that were certified at the previous positions and since then changed
// only by flips, which keep them combinatorially consistent (k_flip_apply checks the quad
// before it rewrites the four rows): the consistency lookup in the neighbour's row is skipped,
// every edge is tested once (from its lower-id end, which also queues the candidate) and every
// triangle's orientation once (from its minimum vertex).  The ambiguity flags feed only
// scvt_triangulate, which always runs a fresh mode-0 pass: modes 1-2 do not write them.
template <bool RO>
__device__ __forceinline__ bool verify_item(const VerifyArgs& v, int64_t gidx, const CandSink& sk) {
    const int idx = (int)(gidx / VERIFY_LANES), lane = (int)(gidx % VERIFY_LANES);
    int p, i;
    if (v.list) {               // re-certification of a compacted list of sorted slots
        if (idx >= (v.list_len >= 0 ? v.list_len : ldc<RO>(v.list_n))) return true;
        if (v.list_ids) {
            i = ldc<RO>(v.list + idx);
            if (i < 0) return false;                       // hole of a touched-cell list
        } else {
            p = ldc<RO>(v.list + idx);
            if (p < v.p_lo || p >= v.p_hi) return false;   // sharded re-check: owned slots only
            i = __ldg(v.ids + p);
        }
    } else {
        p = v.p_lo + idx;
        if (p >= v.p_hi) return true;
        i = __ldg(v.ids + p);
    }
    const int mode = v.mode;
    const int d = ldc<RO>(v.deg + i);
    const int* row = v.nbr + (int64_t)i * MAXDEG;
    if (d < 3 || d > MAXDEG) {
        if (lane == 0)
            mark_bad(mode > 1 ? 1 : mode, v.status, ST_INCONSISTENT, v.bad, v.nbad, i, -1, -1, -1);
        return false;
    }
    const double* z = v.z;
    V3 zi = load3(z, i);
    if (mode == 2) {
        for (int t = lane; t < d; t += VERIFY_LANES) {
            const int a = ldc<RO>(row + t);
            if (a < i) continue;            // the edge and its triangles belong to lower ids
            const int b = ldc<RO>(row + (t + 1 == d ? 0 : t + 1)),
                      c = ldc<RO>(row + (t == 0 ? d - 1 : t - 1));
            const V3 za = load3(z, a), zb = load3(z, b), zc = load3(z, c);
            int tier;
            if (i < b && orient_robust(v3(0, 0, 0), zi, za, zb, -1, i, a, b, &tier) <= 0) {
                mark_bad(1, v.status, ST_NOT_DELAUNAY, v.bad, v.nbad, i, a, b, -1);
#ifdef SCVT_PROBE_FLIPS
                atomicAdd(&g_probe[1], 1);
#endif
            }
            if (orient_robust(zi, za, zb, zc, i, a, b, c, &tier) > 0) {
#ifdef SCVT_PROBE_FLIPS
                atomicAdd(&g_probe[0], 1);
#endif
                // edges at cells already bound for the rebuild path (a triangle there faces
                // inward: the mesh folded, which no flip repairs) are not queued
                int* bad = v.bad;
                if (!(__ldcg(bad + i) | __ldcg(bad + a) | __ldcg(bad + b) | __ldcg(bad + c)))
                    sink_push(sk, v.fq, make_int4(i, a, b, c), bad, v.nbad);
            }
        }
        return false;
    }
    int namb = 0;
    for (int t = lane; t < d; t += VERIFY_LANES) {
        int a = ldc<RO>(row + t), b = ldc<RO>(row + (t + 1 == d ? 0 : t + 1)),
            c = ldc<RO>(row + (t == 0 ? d - 1 : t - 1));
        int da = ldc<RO>(v.deg + a);
        const int* ra = v.nbr + (int64_t)a * MAXDEG;
        int q = -1;
        if (da >= 3 && da <= MAXDEG)
            for (int k = 0; k < da; ++k)
                if (ldc<RO>(ra + k) == i) { q = k; break; }
        bool ok = q >= 0 && ldc<RO>(ra + (q == 0 ? da - 1 : q - 1)) == b;
        if (!ok) mark_bad(mode, v.status, ST_INCONSISTENT, v.bad, v.nbad, i, a, b, -1);
        V3 za = load3(z, a), zb = load3(z, b), zc = load3(z, c);
        if (mode >= 1) {   // reused cycles: the triangle must still face outward
            int tier;
            if (orient_robust(v3(0, 0, 0), zi, za, zb, -1, i, a, b, &tier) <= 0)
                mark_bad(mode, v.status, ST_NOT_DELAUNAY, v.bad, v.nbad, i, a, b, -1);
        }
        int tier;
        int sgn = orient_robust(zi, za, zb, zc, i, a, b, c, &tier);
        if (mode == 0) {
            v.amb[(int64_t)i * MAXDEG + t] = tier > 0 ? 1 : 0;
            namb += tier > 0;
        }
        if (sgn > 0) mark_bad(mode, v.status, ST_NOT_DELAUNAY, v.bad, v.nbad, i, a, b, c);
    }
    if (namb) atomicAdd(&v.stats[3], namb);
    return false;
}

__global__ void k_verify(const double* __restrict__ z, const int* __restrict__ ids, int p_lo,
                         int p_hi, const int* __restrict__ list, const int* __restrict__ list_n,
                         const int* __restrict__ nbr, const int* __restrict__ deg,
                         uint8_t* __restrict__ amb, int* __restrict__ status,
                         int* __restrict__ stats, int mode, int* __restrict__ bad,
                         int* __restrict__ nbad, FlipQueue fq = FlipQueue{nullptr, nullptr, 0},
                         int list_ids = 0) {
    // VERIFY_LANES threads per cell, each taking every VERIFY_LANES-th edge of its cycle: the
    // dependent neighbour-row lookups of different edges run in parallel instead of in one
    // thread's loop (the pass is memory-latency bound)
    const VerifyArgs v{z, ids, p_lo, p_hi, list, list_n, nbr, deg, amb, status, stats, mode,
                       bad, nbad, fq, list_ids, -1};
    __shared__ int4 s_q[SINK_CAP];
    __shared__ int s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const CandSink sk{s_q, &s_n};
    for (int64_t gidx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;;
         gidx += (int64_t)gridDim.x * blockDim.x)
        if (verify_item<true>(v, gidx, sk)) break;
    if (mode == 2) sink_flush(sk, fq, bad, nbad);
}

// ------------------------------------------------------------------ flip repair
// Lawson flips of the reused cycles (the north star's "repaired by edge flips"): every flip
// candidate of the detection pass takes a 64-bit ticket {i, a} on its four vertices (atomicMin);
// the candidates that hold all four tickets form an independent set and flip their edge in the
// cycles of i, a, b, c (canonical rotation: minimum id first).  The four vertices of every
// candidate, flipped or not, are re-certified by the next detection pass (the only edges whose
// status a flip changes are the quad's, whose ends are all among them).  Anything unexpected
// (degree limits, inconsistent neighbourhoods) marks the four cells bad for the rebuild path.
//
// A round is lock -> apply -> finish.  The first rounds (tens of thousands of candidates) run
// as three grid-wide launches each; once the queue is short the remaining rounds run inside
// ONE thread block (k_flip_tail: block barriers between the phases, no launches, no host
// reads), which also turns whatever is left after its round limit into bad cells.  The host
// never reads a counter between rounds: it sizes the number of grid-wide rounds from the queue
// lengths the previous evaluation reported (read back with that evaluation's scalars).
__device__ __forceinline__ unsigned long long flip_key(const int4& c) {
    return ((unsigned long long)(unsigned)c.x << 32) | (unsigned)c.y;
}

constexpr unsigned FULL_MASK = 0xffffffffu;

__device__ __forceinline__ void lock_item(const int4 c, unsigned long long* __restrict__ lock) {
    const unsigned long long key = flip_key(c);
    atomicMin(&lock[c.x], key); atomicMin(&lock[c.y], key);
    atomicMin(&lock[c.z], key); atomicMin(&lock[c.w], key);
}

// store the cyclic sequence y (one entry per lane, d entries) rotated so its minimum comes first
__device__ __forceinline__ void cyc_store_warp(int* __restrict__ row, int* __restrict__ degp,
                                               int y, int d, int lane) {
    const int mn = __reduce_min_sync(FULL_MASK, lane < d ? y : 0x7fffffff);
    const int pos = __ffs(__ballot_sync(FULL_MASK, lane < d && y == mn)) - 1;
    int src = lane + pos;
    if (src >= d) src -= d;
    const int out = __shfl_sync(FULL_MASK, y, src & 31);
    if (lane < d) row[lane] = out;
    if (lane == 0) *degp = d;
}

// One candidate (queue slot k) handled by one warp: lane k holds entry k of each of the four
// cycles, so the four rows are four coalesced loads issued together, positions are ballots and
// the rewritten rows are shuffles (one thread walking the rows serially took ~20 dependent
// loads per flip).  The cycles are read through L2 (__ldcg): k_flip_tail rewrites them between
// its rounds.  The touched-cell list has four fixed slots per candidate, next[4k .. 4k+3]: a
// vertex this candidate is the first to touch, or -1 (a hole) -- no list counter to contend
// for.  Returns 1 when the flip was made.
__device__ __forceinline__ int flip_warp(const int4 c, int k, int lane,
                                         const unsigned long long* __restrict__ lock,
                                         int* __restrict__ nbr, int* __restrict__ deg,
                                         int* __restrict__ dflag, int* __restrict__ next,
                                         int* __restrict__ bad, int* __restrict__ nbad) {
    const int vq = lane == 0 ? c.x : lane == 1 ? c.y : lane == 2 ? c.z : c.w;
    if (lane < 4) next[4 * (int64_t)k + lane] = atomicExch(&dflag[vq], 1) == 0 ? vq : -1;
    const unsigned long long key = flip_key(c);
    const bool mine = lane >= 4 || __ldcg(lock + vq) == key;
    if (!__all_sync(FULL_MASK, mine)) return 0;        // a conflicting flip won this round
    const int i = c.x, a = c.y, b = c.z, cc = c.w;
    const int dq = lane < 4 ? __ldcg(deg + vq) : 0;
    const int di = __shfl_sync(FULL_MASK, dq, 0), da = __shfl_sync(FULL_MASK, dq, 1),
              db = __shfl_sync(FULL_MASK, dq, 2), dc = __shfl_sync(FULL_MASK, dq, 3);
    int* ri = nbr + (int64_t)i * MAXDEG;
    int* ra = nbr + (int64_t)a * MAXDEG;
    int* rb = nbr + (int64_t)b * MAXDEG;
    int* rc = nbr + (int64_t)cc * MAXDEG;
    bool ok = di > 3 && di <= MAXDEG && da > 3 && da <= MAXDEG && db >= 3 && db < MAXDEG &&
              dc >= 3 && dc < MAXDEG && b != cc;
    if (ok) {
        const int xi = lane < di ? __ldcg(ri + lane) : -1;
        const int xa = lane < da ? __ldcg(ra + lane) : -1;
        const int xb = lane < db ? __ldcg(rb + lane) : -1;
        const int xc = lane < dc ? __ldcg(rc + lane) : -1;
        const int ti = __ffs(__ballot_sync(FULL_MASK, xi == a)) - 1;
        const int ta = __ffs(__ballot_sync(FULL_MASK, xa == i)) - 1;
        const int tb = __ffs(__ballot_sync(FULL_MASK, xb == i)) - 1;
        const int tc = __ffs(__ballot_sync(FULL_MASK, xc == a)) - 1;
        const unsigned bc_edge = __ballot_sync(FULL_MASK, xb == cc) | __ballot_sync(FULL_MASK, xc == b);
        ok = ti >= 0 && ta >= 0 && tb >= 0 && tc >= 0 && bc_edge == 0;     // b-c not an edge
        if (ok) {
            const int i_nx = __shfl_sync(FULL_MASK, xi, (ti + 1) % di);
            const int i_pv = __shfl_sync(FULL_MASK, xi, (ti + di - 1) % di);
            const int a_pv = __shfl_sync(FULL_MASK, xa, (ta + da - 1) % da);
            const int a_nx = __shfl_sync(FULL_MASK, xa, (ta + 1) % da);
            const int b_nx = __shfl_sync(FULL_MASK, xb, (tb + 1) % db);
            const int c_nx = __shfl_sync(FULL_MASK, xc, (tc + 1) % dc);
            ok = i_nx == b && i_pv == cc &&       // i: c, a, b
                 a_pv == b && a_nx == cc &&       // a: b, i, c
                 b_nx == a &&                     // b: i, a
                 c_nx == i;                       // c: a, i
        }
        if (ok) {
            // i: drop a;  a: drop i
            const int yi = __shfl_sync(FULL_MASK, xi, (lane + (lane >= ti ? 1 : 0)) & 31);
            const int ya = __shfl_sync(FULL_MASK, xa, (lane + (lane >= ta ? 1 : 0)) & 31);
            // b: i, c, a;  c: a, b, i
            const int sb = __shfl_sync(FULL_MASK, xb, (lane + 31) & 31);
            const int sc = __shfl_sync(FULL_MASK, xc, (lane + 31) & 31);
            const int yb = lane <= tb ? xb : (lane == tb + 1 ? cc : sb);
            const int yc = lane <= tc ? xc : (lane == tc + 1 ? b : sc);
            cyc_store_warp(ri, deg + i, yi, di - 1, lane);
            cyc_store_warp(ra, deg + a, ya, da - 1, lane);
            cyc_store_warp(rb, deg + b, yb, db + 1, lane);
            cyc_store_warp(rc, deg + cc, yc, dc + 1, lane);
            return 1;
        }
    }
    if (lane < 4 && atomicExch(&bad[vq], 1) == 0) atomicAdd(nbad, 1);
    return 0;
}

// Flip round, launch 1 of 3: tickets of the current queue; resets the counter the round
// fills next (the next queue of launch 3) and records the queue length for the host's sizing
// of the next evaluation's rounds.
__global__ void k_round_lock(const int4* __restrict__ cand, const int* __restrict__ ncand,
                             int cap, unsigned long long* __restrict__ lock,
                             int* __restrict__ next_n, int* __restrict__ hist) {
    const int nc = min(*ncand, cap);   // entries past the queue capacity were never stored
    if (blockIdx.x == 0 && threadIdx.x == 0) { *next_n = 0; *hist = nc; }
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += gridDim.x * blockDim.x)
        lock_item(cand[k], lock);
}

// launch 2 of 3: a warp per candidate; the flips are counted per block (one atomicAdd each)
constexpr int APPLY_THREADS = 256;
__global__ void __launch_bounds__(APPLY_THREADS)
k_flip_apply(const int4* __restrict__ cand, const int* __restrict__ ncand, int cap,
             const unsigned long long* __restrict__ lock, int* __restrict__ nbr,
             int* __restrict__ deg, int* __restrict__ dflag, int* __restrict__ next,
             int* __restrict__ bad, int* __restrict__ nbad, int* __restrict__ nflips) {
    __shared__ int s_flips;
    if (threadIdx.x == 0) s_flips = 0;
    __syncthreads();
    const int nc = min(*ncand, cap);
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    int mine = 0;
    for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nc; k += nwarps)
        mine += flip_warp(cand[k], k, lane, lock, nbr, deg, dflag, next, bad, nbad);
    if (lane == 0 && mine) atomicAdd(&s_flips, mine);
    __syncthreads();
    if (threadIdx.x == 0 && s_flips) atomicAdd(nflips, s_flips);
}

// one item of a round's last phase: release the tickets of the current queue, clear the
// touched-cell flags, and re-certify the touched cells (flip mode) into the next queue --
// three independent index ranges (the touched list has 4 nc slots, holes included)
template <bool RO>
__device__ __forceinline__ void finish_item(int64_t g, const int4* __restrict__ cand, int nc,
                                            unsigned long long* __restrict__ lock,
                                            int* __restrict__ flag, const VerifyArgs& v,
                                            const CandSink& sk) {
    if (g < nc) {
        const int4 c = RO ? cand[g] : __ldcg(cand + g);
        lock[c.x] = ~0ull; lock[c.y] = ~0ull; lock[c.z] = ~0ull; lock[c.w] = ~0ull;
    } else if (g < 5 * (int64_t)nc) {
        const int i = ldc<RO>(v.list + (g - nc));
        if (i >= 0) flag[i] = 0;
    } else {
        verify_item<RO>(v, g - 5 * (int64_t)nc, sk);
    }
}

// launch 3 of 3
__global__ void k_round_finish(const int4* __restrict__ cand, const int* __restrict__ ncand,
                               int cap, unsigned long long* __restrict__ lock,
                               int* __restrict__ flag, VerifyArgs v) {
    __shared__ int4 s_q[SINK_CAP];
    __shared__ int s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const CandSink sk{s_q, &s_n};
    const int nc = min(*ncand, cap);
    v.list_len = 4 * nc;
    const int64_t total = (5 + 4 * VERIFY_LANES) * (int64_t)nc;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x)
        finish_item<true>(g, cand, nc, lock, flag, v, sk);
    sink_flush(sk, v.fq, v.bad, v.nbad);
}

// The remaining rounds in one thread-block cluster (TAIL_CTAS SMs, hardware cluster barrier
// between the phases; all mutable data is read through L2 and fenced before each barrier).
// cnt: [0] [1] queue lengths, [4] flips, [5] rounds run here, [6] queue length on entry,
// [7] candidates given up.  Stops when the queue is empty, after TAIL_MAX_ROUNDS, or after
// TAIL_STUCK rounds in a row without a flip (the open candidates keep losing their tickets
// to rejected ones: rebuild path).
constexpr int TAIL_THREADS = 512;
constexpr int TAIL_CTAS = 8;
constexpr int TAIL_MAX_ROUNDS = 40;
constexpr int TAIL_STUCK = 3;

__device__ __forceinline__ void cluster_barrier() {
    __threadfence();
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __cluster_dims__(TAIL_CTAS, 1, 1) __launch_bounds__(TAIL_THREADS)
k_flip_tail(int4* __restrict__ cand0, int4* __restrict__ cand1, int* __restrict__ cnt, int cur,
            int cap, unsigned long long* __restrict__ lock, int* __restrict__ nbr,
            int* __restrict__ deg, int* __restrict__ fflag, int* __restrict__ list0,
            int* __restrict__ list1, VerifyArgs v, int max_rounds) {
    __shared__ int4 s_q[SINK_CAP];
    __shared__ int s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const CandSink sk{s_q, &s_n};
    const int nthreads = TAIL_CTAS * TAIL_THREADS;
    const int tid = blockIdx.x * TAIL_THREADS + threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int rounds = 0, stuck = 0;
    const int entry = min(__ldcg(cnt + cur), cap);
    for (;;) {
        const int nc = min(__ldcg(cnt + cur), cap);
        if (nc == 0 || rounds >= max_rounds || stuck >= TAIL_STUCK) break;
        const int nxt = 1 - cur;
        const int4* cq = cur ? cand1 : cand0;
        int4* nq = cur ? cand0 : cand1;
        int* nlist = nxt ? list1 : list0;
        const int flips0 = __ldcg(cnt + 4);
        cluster_barrier();                // everyone has read the counters of this round
        if (tid == 0) atomicExch(cnt + nxt, 0);
        for (int k = tid; k < nc; k += nthreads) lock_item(__ldcg(cq + k), lock);
        cluster_barrier();
        int mine = 0;
        for (int k = warp; k < nc; k += nthreads / 32)
            mine += flip_warp(__ldcg(cq + k), k, lane, lock, nbr, deg, fflag, nlist, v.bad, v.nbad);
        if (lane == 0 && mine) atomicAdd(cnt + 4, mine);
        cluster_barrier();
        VerifyArgs w = v;
        w.list = nlist; w.list_len = 4 * nc; w.fq = FlipQueue{nq, cnt + nxt, cap};
        const int64_t total = (5 + 4 * VERIFY_LANES) * (int64_t)nc;
        for (int64_t g = tid; g < total; g += nthreads)
            finish_item<false>(g, cq, nc, lock, fflag, w, sk);
        sink_flush(sk, w.fq, v.bad, v.nbad);
        cluster_barrier();
        stuck = __ldcg(cnt + 4) == flips0 ? stuck + 1 : 0;
        ++rounds;
        cur = nxt;
    }
    // whatever is still queued goes to the rebuild path
    const int nc = min(__ldcg(cnt + cur), cap);
    const int4* cq = cur ? cand1 : cand0;
    for (int k = tid; k < nc; k += nthreads) queue_overflow(__ldcg(cq + k), v.bad, v.nbad);
    if (tid == 0) { cnt[5] = rounds; cnt[6] = entry; cnt[7] = nc; }
}

__global__ void k_flag_slots(int n, const int* __restrict__ ids, const int* __restrict__ bad,
                             uint8_t* __restrict__ flags) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) flags[p] = bad[ids[p]] ? 1 : 0;
}

// Cells whose certificate verdict can change once the listed cells are rebuilt: the listed
// cells and their current (pre-rebuild) neighbours.  A cell that passed lists only neighbours
// that list it back, so a passing cell outside this set reads no rebuilt cycle.
__global__ void k_mark_recheck(const int* __restrict__ list, const int* __restrict__ list_n,
                               const int* __restrict__ ids, const int* __restrict__ nbr,
                               const int* __restrict__ deg, int* __restrict__ recheck) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < *list_n; idx += gridDim.x * blockDim.x) {
        const int i = ids[list[idx]];
        recheck[i] = 1;
        const int d = deg[i];
        if (d < 3 || d > MAXDEG) continue;
        const int* row = nbr + (int64_t)i * MAXDEG;
        for (int t = 0; t < d; ++t) recheck[row[t]] = 1;
    }
}

// incidence CSR in bucket (spatial) order: sorted slot p -> generator ids[p]
__global__ void k_deg_sorted(int p_lo, int cnt, const int* __restrict__ ids,
                             const int* __restrict__ deg, int* __restrict__ degs) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q > cnt) return;
    degs[q] = q == cnt ? 0 : deg[ids[p_lo + q]];
}

__global__ void k_fill_incidences(int p_lo, int cnt, const int* __restrict__ ids,
                                  const int* __restrict__ deg, const int* inc_start,
                                  int* __restrict__ inc_base, int* __restrict__ inc_gen, int cap,
                                  const int* __restrict__ skip, int* __restrict__ total) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    // skip (the bad count of a flip repair still in flight) != 0: the cycles are not certified,
    // so the incidence total is poisoned and k_quad / k_gather integrate nothing (their Euler
    // check); the host sees the count with the evaluation's scalars and resumes the rebuild
    if (q == 0 && skip && *skip) *total = -1;
    if (q >= cnt) return;
    int i = ids[p_lo + q];
    int s = inc_start[q], d = deg[i];
    inc_base[i] = s;
    for (int t = 0; t < d; ++t)
        if (s + t < cap) inc_gen[s + t] = i;
}

__global__ void k_iota(int n, int* __restrict__ ids) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) ids[p] = p;
}

// ------------------------------------------------------------------ quadrature
struct QuadArgs {
    const double* z;
    const int* nbr;
    const int* deg;
    const int* inc_start;   // [cnt+1] over the owned sorted slots (total at [cnt])
    const int* inc_base;    // [n] by generator id
    const int* inc_gen;
    int n;
    int cnt;                // owned sorted slots
    int n_inc;            // expected incidences 6n - 12 (n_inc_dev: an upper bound, see k_quad)
    int n_inc_dev;        // 1: the incidence count is inc_start[cnt] on the device (shards, fast path)
    const DensityParams* dpg;   // device copy of dp (tab set): what out-of-line paths read
    const double* nodes;  // device [3][nq]: l1, l2, w
    const double* table;  // device rho^(1/4) table (tanh4 kinds) or null
    int nq;
    DensityParams dp;
    double* part;         // [n_inc][PART_ROW]: per incidence, sub-triangle 0 then 1 (split mode)
    uint8_t* obtuse;      // [n_inc]
    int* status;
    int* defer_list;      // [2 n_inc] fan sub-triangles left to k_quad_table (thread ids of k_quad)
    int* defer_cnt;       // their count (zeroed before k_quad)
};

// SPLIT: one thread per fan sub-triangle instead of per incidence (twice the work units, a
// finer last wave, shorter per-thread chains); the two halves land in part[0..5) and
// part[5..10) and the gathers add them in a fixed order.
// DEFER (table kinds on the split fast path): a sub-triangle whose density fit was rejected is
// not swept here -- one such lane would hold its whole warp through the per-node table sweep
// (2.6x a fitted sweep) after the fitted one -- but queued for k_quad_table, which sweeps the
// rejected patches of the whole launch in full warps.  The result of a sub-triangle is the
// same bits whichever kernel computes it.
template <int KIND, bool SPHERE, bool SYM7, bool SPLIT = false, bool DEVCOUNT = false,
          bool DEFER = false>
__global__ void __launch_bounds__(QUAD_THREADS, SYM7 ? (KIND == DEN_TANH4X2_TAB ? QUAD_MINB2 : QUAD_MINB) : 1)
k_quad(QuadArgs a) {
    extern __shared__ double s_nodes[];
    // the symmetric 7-node fast path reads only the first leaf's 7 nodes of each column: a
    // compact [3][7] copy (keeps shared memory for more resident CTAs)
    const int nq_s = (SYM7 && !SPHERE && SPLIT) ? 7 : a.nq;
    for (int q = threadIdx.x; q < 3 * nq_s; q += blockDim.x)
        s_nodes[q] = a.nodes[(q / nq_s) * a.nq + q % nq_s];
    // the density table (28 KB) is read through the read-only cache, where it stays resident
    // (staging it in shared memory per CTA cost 1.4-2.7 % of k_quad, c4, c3, c5); a.dp.tab
    // points at it (set on the host: the kernel never takes the address of its parameters,
    // which would copy them to the stack of every thread)
    __syncthreads();
    const int t_id = blockIdx.x * blockDim.x + threadIdx.x;
    const int u = SPLIT ? t_id >> 1 : t_id;
    const int half = SPLIT ? t_id & 1 : 0;
    if (u >= a.n_inc) return;
    if (DEVCOUNT) {
        // shards: only the device knows the shard's incidence count; n_inc bounds it (the
        // grid's size).  A separate instantiation: this handful of instructions changes the
        // register allocation of the whole kernel (240 B of spills instead of 20)
        const int total = a.inc_start[a.cnt];
        if (total > a.n_inc) {
            if (u == 0) atomicOr(a.status, ST_EULER);
            return;
        }
        if (u >= total) return;
    } else if (a.inc_start[a.cnt] != a.n_inc) {   // not a closed triangulation: nothing to integrate
        if (u == 0) atomicOr(a.status, ST_EULER);
        return;
    }
    int i = a.inc_gen[u];
    int t = u - a.inc_base[i];
    int d = a.deg[i];
    const int* row = a.nbr + (int64_t)i * MAXDEG;
    int j = row[t], k = row[t + 1 == d ? 0 : t + 1];
    V3 vi = load3(a.z, i), vj = load3(a.z, j), vk = load3(a.z, k);
    double acc[5] = {0, 0, 0, 0, 0};
    int pole = 0;
    const double* l1 = s_nodes;
    const double* l2 = s_nodes + nq_s;
    const double* w = s_nodes + 2 * nq_s;
    if (SYM7 && !SPHERE && SPLIT) {
        // phase 1 -> shared slot -> phase 2 (scvt_device.cuh sym7_prologue / sym7_sweep):
        // only this thread's half of the fan is built, and nothing but the slot (sub-triangle,
        // generator, fits) is live across the node loop
        constexpr int NF = KIND == DEN_TANH4X2_TAB ? 2 : 1;
        __shared__ LocalFit s_fit[QUAD_THREADS][NF];
        __shared__ SubTri s_sub[QUAD_THREADS];
        __shared__ double s_z[QUAD_THREADS][3];
        int obt, degen;
        const SubTri st0 = fan_sub(vi, vj, vk, i, j, k, half, &obt, &degen);
        if (degen) atomicOr(a.status, ST_DEGENERATE_TRI);
        if (half == 0) a.obtuse[u] = (obt && i < j && i < k) ? 1 : 0;
        const DensityParams& dp = *a.dpg;
        const int mode = sym7_prologue<KIND>(dp, st0, s_fit[threadIdx.x]);
        if (DEFER && (mode & 3) == SWEEP_TABLE) {
            // one atomicAdd per warp; the queue's order does not matter (every entry writes
            // its own partial row)
            const unsigned m = __activemask();
            const int lane = threadIdx.x & 31;
            const int leader = __ffs(m) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(a.defer_cnt, __popc(m));
            base = __shfl_sync(m, base, leader);
            a.defer_list[base + __popc(m & ((1u << lane) - 1u))] = t_id;
            return;
        }
        s_sub[threadIdx.x] = st0;
        s_z[threadIdx.x][0] = vi.x; s_z[threadIdx.x][1] = vi.y; s_z[threadIdx.x][2] = vi.z;
        asm volatile("" ::: "memory");    // the sweep reads its inputs back from the slot
        const SubTri st = s_sub[threadIdx.x];
        const V3 zc = v3(s_z[threadIdx.x][0], s_z[threadIdx.x][1], s_z[threadIdx.x][2]);
        sym7_sweep<KIND, 8, DEFER>(mode, st, zc, l1, l2, w, dp, s_fit[threadIdx.x], acc, &pole);
        if (pole) atomicOr(a.status, ST_POLE);
        double* out = a.part + (int64_t)u * PART_ROW + (half ? 5 : 0);
#pragma unroll
        for (int c = 0; c < 5; ++c) out[c] = acc[c];
        return;
    }
    FanPair f = fan_pair(vi, vj, vk, i, j, k);
    if (f.degenerate) atomicOr(a.status, ST_DEGENERATE_TRI);
    {   // both halves in this thread, stored separately (per-sub-triangle masses feed
        // the graph Laplacian; the gathers add the halves: the same sums as before)
        subtri_moments<KIND, SPHERE>(f.s[0], vi, l1, l2, w, a.nq, a.dp, acc, &pole);
        double acc1[5] = {0, 0, 0, 0, 0};
        subtri_moments<KIND, SPHERE>(f.s[1], vi, l1, l2, w, a.nq, a.dp, acc1, &pole);
        double* out1 = a.part + (int64_t)u * PART_ROW + 5;
#pragma unroll
        for (int c = 0; c < 5; ++c) out1[c] = acc1[c];
    }
    if (pole) atomicOr(a.status, ST_POLE);
    // incidence-major: [u][half][m, cx, cy, cz, E] (80 B per incidence, one contiguous run
    // of 80 * valence bytes per generator for the gathers)
    double* out = a.part + (int64_t)u * PART_ROW + (SPLIT && half ? 5 : 0);
#pragma unroll
    for (int c = 0; c < 5; ++c) out[c] = acc[c];
    if (!SPLIT || half == 0) a.obtuse[u] = (f.obtuse && i < j && i < k) ? 1 : 0;
}

// The sub-triangles k_quad<..., DEFER> queued (rejected fits): per-node table evaluation of
// the density on the same leaf grid, every lane of a warp on the same sweep.  Grid-stride over
// the queue (its length is known on the device only).
constexpr int QTAB_THREADS = 64;
#ifndef QTAB_MINB
#define QTAB_MINB 8      // resident CTAs per SM the register budget must allow (one wave for the queue)
#endif
template <int KIND>
__global__ void __launch_bounds__(QTAB_THREADS, QTAB_MINB) k_quad_table(QuadArgs a) {
    __shared__ double s_nodes[21];
    for (int q = threadIdx.x; q < 21; q += blockDim.x)
        s_nodes[q] = a.nodes[(q / 7) * a.nq + q % 7];
    __syncthreads();
    const double* l1 = s_nodes;
    const double* l2 = s_nodes + 7;
    const double* w = s_nodes + 14;
    const int total = *a.defer_cnt;
    const DensityParams& dp = *a.dpg;
    // four lanes per queued sub-triangle (up / down leaves x even / odd leaf rows: 20, 16, 16
    // and 12 of the 64 leaves), summed in a fixed order by two shuffles: the sweep of one
    // sub-triangle is ~30k dependent-ish FP64 instructions, and a short queue (a shard's, or
    // c3's) is latency-, not throughput-bound
    const int lane = threadIdx.x & 31, part = lane & 3;
    const int per_pass = gridDim.x * (blockDim.x >> 2);
    for (int e0 = blockIdx.x * (blockDim.x >> 2) + ((threadIdx.x >> 5) << 3); e0 < total;
         e0 += per_pass) {           // e0: the warp's first entry (8 entries per warp)
        const int idx = e0 + (lane >> 2);
        const bool live = idx < total;
        double acc[5] = {0, 0, 0, 0, 0};
        int u = 0, half = 0, pole = 0;
        if (live) {
            const int t_id = a.defer_list[idx];
            u = t_id >> 1; half = t_id & 1;
            const int i = a.inc_gen[u];
            const int t = u - a.inc_base[i];
            const int d = a.deg[i];
            const int* row = a.nbr + (int64_t)i * MAXDEG;
            const int j = row[t], k = row[t + 1 == d ? 0 : t + 1];
            const V3 vi = load3(a.z, i), vj = load3(a.z, j), vk = load3(a.z, k);
            int obt, degen;
            const SubTri st = fan_sub(vi, vj, vk, i, j, k, half, &obt, &degen);
            sym7_table_sweep<KIND, 8>(st, vi, l1, l2, w, dp, acc, &pole, part, 4);
            if (pole) atomicOr(a.status, ST_POLE);
        }
#pragma unroll
        for (int c = 0; c < 5; ++c) {
            acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 1);
            acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 2);
        }
        if (live && part == 0) {
            double* out = a.part + (int64_t)u * PART_ROW + (half ? 5 : 0);
#pragma unroll
            for (int c = 0; c < 5; ++c) out[c] = acc[c];
        }
    }
}

// gradient epilogue (pipeline.py:265-279): g = 2(c.z)z - 2c, diag = 2 c.z
__device__ __forceinline__ void epilogue(const double* __restrict__ z, int i, double cx, double cy,
                                         double cz, double* __restrict__ grad,
                                         double* __restrict__ diag, double* __restrict__ g2) {
    V3 zi = load3(z, i);
    double czd = cx * zi.x + cy * zi.y + cz * zi.z;
    double gx = 2.0 * czd * zi.x - 2.0 * cx;
    double gy = 2.0 * czd * zi.y - 2.0 * cy;
    double gz = 2.0 * czd * zi.z - 2.0 * cz;
    grad[3 * (int64_t)i] = gx; grad[3 * (int64_t)i + 1] = gy; grad[3 * (int64_t)i + 2] = gz;
    diag[i] = 2.0 * czd;
    g2[i] = gx * gx + gy * gy + gz * gz;
}

// per generator (id order: coalesced outputs): fixed-order sum over its incidences — one
// contiguous run of 80 * valence bytes of the incidence-major partials — then the gradient
// epilogue.
__device__ __forceinline__ void incidence_sums(const double* __restrict__ part, int u0, int u1,
                                               int split, double* v5) {
#pragma unroll
    for (int c = 0; c < 5; ++c) v5[c] = 0.0;
    for (int u = u0; u < u1; ++u) {
        const double2* r = reinterpret_cast<const double2*>(part + (int64_t)u * PART_ROW);
        const double2 a0 = r[0], a1 = r[1], a2 = r[2], a3 = r[3], a4 = r[4];
        const double h0[5] = {a0.x, a0.y, a1.x, a1.y, a2.x};
        const double h1[5] = {a2.y, a3.x, a3.y, a4.x, a4.y};
        if (split) {
#pragma unroll
            for (int c = 0; c < 5; ++c) v5[c] += h0[c] + h1[c];
        } else {
#pragma unroll
            for (int c = 0; c < 5; ++c) v5[c] += h0[c];
        }
    }
}

__global__ void k_gather(const double* __restrict__ z, int n, int cnt,
                         const int* __restrict__ inc_start,
                         const int* __restrict__ inc_base, const int* __restrict__ deg,
                         const double* __restrict__ part, const uint8_t* __restrict__ obtuse,
                         int64_t n_inc, double* __restrict__ grad, double* __restrict__ first,
                         double* __restrict__ mass, double* __restrict__ diag,
                         double* __restrict__ e_gen, double* __restrict__ g2_gen,
                         double* __restrict__ ob_gen, int split) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v5[5] = {0, 0, 0, 0, 0}, ob = 0;
    if (inc_start[cnt] == n_inc) {
        const int u0 = inc_base[i], u1 = u0 + deg[i];
        incidence_sums(part, u0, u1, split, v5);
        for (int u = u0; u < u1; ++u) ob += obtuse[u];
    }
    const double m = v5[0], cx = v5[1], cy = v5[2], cz = v5[3], e = v5[4];
    epilogue(z, i, cx, cy, cz, grad, diag, g2_gen);
    first[3 * (int64_t)i] = cx; first[3 * (int64_t)i + 1] = cy; first[3 * (int64_t)i + 2] = cz;
    if (mass) mass[i] = m;
    e_gen[i] = e;
    ob_gen[i] = ob;
}

// ------------------------------------------------------------------ shard exchange rows
constexpr int CYC_ROW = 2 + MAXDEG;   // [id, deg, nbr...] int32
constexpr int RES_ROW = 8;            // [id, m, cx, cy, cz, E, obtuse, 0] f64

__global__ void k_pack_cycles(const int* __restrict__ ids, int p_lo, int cnt, int cap,
                              const int* __restrict__ nbr, const int* __restrict__ deg,
                              int* __restrict__ out) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= cap) return;
    int* row = out + (int64_t)q * CYC_ROW;
    if (q >= cnt) { row[0] = -1; row[1] = 0; return; }
    int i = ids[p_lo + q];
    int d = deg[i];
    row[0] = i;
    row[1] = d;
    for (int t = 0; t < MAXDEG; ++t) row[2 + t] = t < d ? nbr[(int64_t)i * MAXDEG + t] : -1;
}

__global__ void k_unpack_cycles(const int* __restrict__ rows, int nrows, int n,
                                int* __restrict__ nbr, int* __restrict__ deg,
                                int* __restrict__ degsum, int* __restrict__ status) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const int* row = rows + (int64_t)r * CYC_ROW;
    int i = row[0];
    if (i < 0) return;
    if (i >= n) { atomicOr(status, ST_INCONSISTENT); return; }
    int d = row[1];
    deg[i] = d;
    for (int t = 0; t < d && t < MAXDEG; ++t) nbr[(int64_t)i * MAXDEG + t] = row[2 + t];
    atomicAdd(degsum, d);
}

// rebuilt cells of a slot list packed as exchange rows (cap rows, padding id = -1)
__global__ void k_pack_list(const int* __restrict__ list, const int* __restrict__ cnt_dev,
                            int cap, const int* __restrict__ ids, const int* __restrict__ nbr,
                            const int* __restrict__ deg, int* __restrict__ out) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= cap) return;
    int* row = out + (int64_t)q * CYC_ROW;
    if (q >= *cnt_dev) { row[0] = -1; row[1] = 0; return; }
    int i = ids[list[q]];
    int d = deg[i];
    row[0] = i;
    row[1] = d;
    for (int t = 0; t < MAXDEG; ++t) row[2 + t] = t < d ? nbr[(int64_t)i * MAXDEG + t] : -1;
}

__global__ void k_set_int(int* p, int v) { *p = v; }

// per-shard counts of an ascending slot list (shard s owns slots [s*cap, (s+1)*cap)):
// counts[s] = lower_bound((s+1)*cap) - lower_bound(s*cap); counts[nshards] = total
__global__ void k_shard_counts(const int* __restrict__ list, const int* __restrict__ list_n,
                               int nshards, int64_t cap, int* __restrict__ counts) {
    __shared__ int bound[MAX_SHARDS + 1];
    const int total = *list_n;
    for (int b = threadIdx.x; b <= nshards; b += blockDim.x) {
        const int64_t key = (int64_t)b * cap;
        int lo = 0, hi = total;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (list[mid] < key) lo = mid + 1; else hi = mid;
        }
        bound[b] = b == nshards ? total : lo;
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nshards; b += blockDim.x) counts[b] = bound[b + 1] - bound[b];
    if (threadIdx.x == 0) counts[nshards] = total;
}

// owned slots: fixed-order incidence sums packed as exchange rows (slot order: the rows and
// the incidence runs are both contiguous)
__global__ void k_gather_pack(int p_lo, int cnt, int cap, const int* __restrict__ ids,
                              const int* __restrict__ inc_base, const int* __restrict__ deg,
                              const double* __restrict__ part, const uint8_t* __restrict__ obtuse,
                              int64_t n_inc, double* __restrict__ out, int split) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= cap) return;
    double* row = out + (int64_t)q * RES_ROW;
    if (q >= cnt) {
        row[0] = -1.0;
        for (int c = 1; c < RES_ROW; ++c) row[c] = 0.0;
        return;
    }
    int i = ids[p_lo + q];
    const int u0 = inc_base[i], u1 = u0 + deg[i];
    double v5[5], ob = 0;
    incidence_sums(part, u0, u1, split, v5);
    for (int u = u0; u < u1; ++u) ob += obtuse[u];
    row[0] = (double)i; row[1] = v5[0]; row[2] = v5[1]; row[3] = v5[2]; row[4] = v5[3];
    row[5] = v5[4]; row[6] = ob; row[7] = 0.0;
}

__global__ void k_unpack_results(const double* __restrict__ rows, int nrows, int n,
                                 const double* __restrict__ z, double* __restrict__ grad,
                                 double* __restrict__ first, double* __restrict__ mass,
                                 double* __restrict__ diag, double* __restrict__ e_gen,
                                 double* __restrict__ g2_gen, double* __restrict__ ob_gen,
                                 int* __restrict__ seen) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const double* row = rows + (int64_t)r * RES_ROW;
    if (row[0] < 0.0) return;
    int i = (int)row[0];
    if (i >= n) return;
    double cx = row[2], cy = row[3], cz = row[4];
    epilogue(z, i, cx, cy, cz, grad, diag, g2_gen);
    first[3 * (int64_t)i] = cx; first[3 * (int64_t)i + 1] = cy; first[3 * (int64_t)i + 2] = cz;
    if (mass) mass[i] = row[1];
    e_gen[i] = row[5];
    ob_gen[i] = row[6];
    atomicAdd(seen, 1);
}

// arithmetic-layout finish: the rows of ids in [lo, hi) -> slice-local outputs (index i - lo);
// E_i, |g_i|^2, obtuse_i by id (the caller NaN-fills E of the slice first: coverage check)
__global__ void k_unpack_slice(const double* __restrict__ rows, int nrows, int64_t lo,
                               int64_t hi, const double* __restrict__ z, double* __restrict__ grad,
                               double* __restrict__ first, double* __restrict__ mass,
                               double* __restrict__ diag, double* __restrict__ e_gen,
                               double* __restrict__ g2_gen, double* __restrict__ ob_gen) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const double* row = rows + (int64_t)r * RES_ROW;
    if (row[0] < 0.0) return;
    const int64_t i = (int64_t)row[0];
    if (i < lo || i >= hi) return;
    const int64_t k = i - lo;
    const double cx = row[2], cy = row[3], cz = row[4];
    V3 zi = load3(z, (int)i);
    const double czd = cx * zi.x + cy * zi.y + cz * zi.z;
    const double gx = 2.0 * czd * zi.x - 2.0 * cx;
    const double gy = 2.0 * czd * zi.y - 2.0 * cy;
    const double gz = 2.0 * czd * zi.z - 2.0 * cz;
    grad[3 * k] = gx; grad[3 * k + 1] = gy; grad[3 * k + 2] = gz;
    diag[k] = 2.0 * czd;
    g2_gen[i] = gx * gx + gy * gy + gz * gz;
    first[3 * k] = cx; first[3 * k + 1] = cy; first[3 * k + 2] = cz;
    if (mass) mass[k] = row[1];
    e_gen[i] = row[5];
    ob_gen[i] = row[6];
}

// ------------------------------------------------------------------ deterministic reductions
// op 0 = sum, 1 = max, 2 = min.  Stage 1 writes RED_BLOCKS partials per array.
template <int OP>
__device__ __forceinline__ double red_op(double a, double b) {
    return OP == 0 ? a + b : (OP == 1 ? fmax(a, b) : fmin(a, b));
}
template <int OP>
__device__ __forceinline__ double red_identity() {
    return OP == 0 ? 0.0 : (OP == 1 ? -INFINITY : INFINITY);
}

template <int OP>
__device__ double block_reduce(double v) {
    __shared__ double sh[RED_THREADS];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = RED_THREADS / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = red_op<OP>(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    double r = sh[0];
    __syncthreads();
    return r;
}

// partials[slot * RED_BLOCKS + block] = op over x[k] (k = block*T + tid + j*RED_BLOCKS*T)
template <int OP>
__global__ void __launch_bounds__(RED_THREADS)
k_reduce_stage1(const double* __restrict__ x, int64_t len, double* __restrict__ partials) {
    double v = red_identity<OP>();
    for (int64_t k = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; k < len;
         k += (int64_t)RED_BLOCKS * RED_THREADS)
        v = red_op<OP>(v, x[k]);
    v = block_reduce<OP>(v);
    if (threadIdx.x == 0) partials[blockIdx.x] = v;
}

// dot products: partials of sum a[k]*b[k]
__global__ void __launch_bounds__(RED_THREADS)
k_dot_stage1(const double* __restrict__ a, const double* __restrict__ b, int64_t len,
             double* __restrict__ partials) {
    double v = 0.0;
    for (int64_t k = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; k < len;
         k += (int64_t)RED_BLOCKS * RED_THREADS)
        v += a[k] * b[k];
    v = block_reduce<0>(v);
    if (threadIdx.x == 0) partials[blockIdx.x] = v;
}

// partials of max |a[k] - b[k]| (movement, optimizer.py:355)
__global__ void __launch_bounds__(RED_THREADS)
k_absdiff_stage1(const double* __restrict__ a, const double* __restrict__ b, int64_t len,
                 double* __restrict__ partials);

// sum over the RED_BLOCKS partials in a fixed order (called by every block that needs it)
template <int OP>
__device__ double finish_partials(const double* __restrict__ partials) {
    double v = red_identity<OP>();
    for (int k = threadIdx.x; k < RED_BLOCKS; k += RED_THREADS) v = red_op<OP>(v, partials[k]);
    return block_reduce<OP>(v);
}

template <int OP>
__global__ void __launch_bounds__(RED_THREADS)
k_reduce_stage2(const double* __restrict__ partials, int nslots, double* __restrict__ out) {
    for (int s = 0; s < nslots; ++s) {
        double v = finish_partials<OP>(partials + s * RED_BLOCKS);
        if (threadIdx.x == 0) out[s] = v;
    }
}

__global__ void __launch_bounds__(RED_THREADS)
k_absdiff_stage1(const double* __restrict__ a, const double* __restrict__ b, int64_t len,
                 double* __restrict__ partials) {
    double v = 0.0;
    for (int64_t k = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; k < len;
         k += (int64_t)RED_BLOCKS * RED_THREADS)
        v = fmax(v, fabs(a[k] - b[k]));
    v = block_reduce<1>(v);
    if (threadIdx.x == 0) partials[blockIdx.x] = v;
}

// ------------------------------------------------------------------ Gram-form two-loop
// two_loop_direction (optimizer.py:147-167) needs, besides the host-side y_i.s_j matrix kept up
// to date at push time, only s_i.g, y_i.H0 g, y_i.H0 y_j and g.H0 g: one fused pass over the
// history computes them all; one block runs the scalar recursion; one combine pass forms
// q = -(H0 (g - sum a_j y_j) + sum c_l s_l), projects it to the tangent planes and reduces
// q.g and g.q3.  Mathematically the reference's two loops; 2K+3 vector reads instead of 4K.
constexpr int MAXM = 16;

struct HistPtrs {
    const double* S[MAXM];   // ordered oldest -> newest
    const double* Y[MAXM];
};

// A slice of the generator ids [lo, lo + len) made of the chunks [c_lo, c_lo + nc); block b of a
// chunked launch (grid = nc) owns the slice-local ids [b ch, min(len, (b + 1) ch)).  Pointers
// handed to the kernels are slice-local (index 0 = id lo).
struct Chunks {
    int64_t lo, len, ch;
    int c_lo, nc;
};

__device__ __forceinline__ void chunk_span(const Chunks& c, int64_t* b, int64_t* e) {
    *b = (int64_t)blockIdx.x * c.ch;
    *e = min(c.len, *b + c.ch);
}

__device__ __forceinline__ double* chunk_slot(double* red, const Chunks& c, int v) {
    return red + (int64_t)v * CHUNKS + c.c_lo + blockIdx.x;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

constexpr int GRAM_THREADS = 128;

// Gram pass of the two-loop (one read of the history): per chunk, s_k.g, y_k.H0 g, y_k.H0 y_l
// (packed upper triangle) and g.H0 g
template <int K>
__global__ void __launch_bounds__(GRAM_THREADS)
k_gram(const double* __restrict__ g, const double* __restrict__ diag, double gamma, HistPtrs h,
       Chunks ck, double* __restrict__ red) {
    constexpr int A = 2 * K + K * (K + 1) / 2 + 1;
    double acc[A];
#pragma unroll
    for (int a = 0; a < A; ++a) acc[a] = 0.0;
    int64_t i0, i1;
    chunk_span(ck, &i0, &i1);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += GRAM_THREADS) {
        const double hw = diag ? 1.0 / diag[i] : gamma;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int64_t e = 3 * i + c;
            const double ge = g[e];
            double yv[K > 0 ? K : 1];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                yv[k] = h.Y[k][e];
                acc[k] += h.S[k][e] * ge;               // s_k . g
                acc[K + k] += yv[k] * (hw * ge);        // y_k . H0 g
            }
            int a = 2 * K;
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int l = k; l < K; ++l) acc[a++] += yv[k] * (hw * yv[l]);   // y_k . H0 y_l
            acc[A - 1] += ge * (hw * ge);                                      // g . H0 g
        }
    }
    __shared__ double sh[GRAM_THREADS / 32][A];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int a = 0; a < A; ++a) {
        double v = warp_sum(acc[a]);
        if (lane == 0) sh[w][a] = v;
    }
    __syncthreads();
    for (int a = threadIdx.x; a < A; a += GRAM_THREADS) {
        double v = 0.0;
        for (int q = 0; q < GRAM_THREADS / 32; ++q) v += sh[q][a];
        *chunk_slot(red, ck, a) = v;
    }
}

struct GramScalars {
    double ys[MAXM][MAXM];   // y_i . s_j, ordered oldest -> newest
    double rho[MAXM];
};

// fixed-order reduction of one value's CHUNKS partials by one warp (lane-strided, then a fixed
// butterfly): the same bits on every rank and for every rank count
template <int OP>
__device__ __forceinline__ double warp_chunks(const double* __restrict__ pv) {
    const int lane = threadIdx.x & 31;
    double v = red_identity<OP>();
    for (int b = lane; b < CHUNKS; b += 32) v = red_op<OP>(v, pv[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = red_op<OP>(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// one block: fixed-order sums of the Gram partials, then the scalar two-loop recursion
__global__ void k_gram_recursion(const double* __restrict__ red, int K, GramScalars gs,
                                 double* __restrict__ coef) {
    __shared__ double val[2 * MAXM + MAXM * (MAXM + 1) / 2 + 1];
    const int A = 2 * K + K * (K + 1) / 2 + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int a = warp; a < A; a += nw) {
        const double v = warp_chunks<0>(red + (int64_t)a * CHUNKS);
        if (lane == 0) val[a] = v;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    auto yhy = [&](int i, int j) {   // packed upper triangle, i <= j
        if (i > j) { int t = i; i = j; j = t; }
        return val[2 * K + i * K - i * (i - 1) / 2 + (j - i)];
    };
    double a[MAXM], c[MAXM];
    for (int i = K - 1; i >= 0; --i) {               // backward: newest -> oldest
        double sq = val[i];                          // s_i . g
        for (int j = i + 1; j < K; ++j) sq -= a[j] * gs.ys[j][i];   // - a_j s_i . y_j
        a[i] = gs.rho[i] * sq;
    }
    for (int i = 0; i < K; ++i) {                    // forward: oldest -> newest
        double yr = val[K + i];                      // y_i . H0 g
        for (int j = 0; j < K; ++j) yr -= a[j] * yhy(i, j);
        for (int l = 0; l < i; ++l) yr += c[l] * gs.ys[i][l];
        c[i] = a[i] - gs.rho[i] * yr;
    }
    for (int i = 0; i < K; ++i) { coef[i] = a[i]; coef[MAXM + i] = c[i]; }
}

// q = -(H0 (g - sum_j a_j y_j) + sum_l c_l s_l); q3 = q - (q.z) z; chunk partials of q.g, g.q3
template <int K>
__global__ void __launch_bounds__(RED_THREADS)
k_combine(const double* __restrict__ g, const double* __restrict__ diag, double gamma,
          HistPtrs h, const double* __restrict__ coef, const double* __restrict__ z, Chunks ck,
          double* __restrict__ q3, double* __restrict__ red) {
    double ca[K > 0 ? K : 1], cc[K > 0 ? K : 1];
#pragma unroll
    for (int k = 0; k < K; ++k) { ca[k] = coef[k]; cc[k] = coef[MAXM + k]; }
    double qg = 0.0, gq3 = 0.0;
    int64_t i0, i1;
    chunk_span(ck, &i0, &i1);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += RED_THREADS) {
        const double hw = diag ? 1.0 / diag[i] : gamma;
        double q[3], gg[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int64_t e = 3 * i + c;
            double v = g[e];
            gg[c] = v;
#pragma unroll
            for (int k = K - 1; k >= 0; --k) v -= ca[k] * h.Y[k][e];
            v *= hw;
#pragma unroll
            for (int k = 0; k < K; ++k) v += cc[k] * h.S[k][e];
            q[c] = -v;
        }
        const double zx = z[3 * i], zy = z[3 * i + 1], zz = z[3 * i + 2];
        const double qd = q[0] * zx + q[1] * zy + q[2] * zz;
        const double ax = q[0] - qd * zx, ay = q[1] - qd * zy, az = q[2] - qd * zz;
        q3[3 * i] = ax; q3[3 * i + 1] = ay; q3[3 * i + 2] = az;
        qg += q[0] * gg[0] + q[1] * gg[1] + q[2] * gg[2];
        gq3 += gg[0] * ax + gg[1] * ay + gg[2] * az;
    }
    qg = block_reduce<0>(qg);
    gq3 = block_reduce<0>(gq3);
    if (threadIdx.x == 0) {
        *chunk_slot(red, ck, 0) = qg;
        *chunk_slot(red, ck, 1) = gq3;
    }
}

// s = z_new - z_old, y = g_new - g_old (staged) and, in the same pass, their products with the
// K stored pairs: chunk partials of y.s, s.s, y.y, max|s| (values 0-3), y_new.s_j (4 .. 4+K)
// and y_j.s_new (4+K .. 4+2K).  Warp butterflies, then the warps in a fixed order.
template <int K>
__global__ void __launch_bounds__(RED_THREADS)
k_history_pair(const double* __restrict__ zo, const double* __restrict__ zn,
               const double* __restrict__ go, const double* __restrict__ gn, HistPtrs h,
               Chunks ck, double* __restrict__ s, double* __restrict__ y,
               double* __restrict__ red) {
    constexpr int A = 4 + 2 * K;
    double acc[A];
#pragma unroll
    for (int a = 0; a < A; ++a) acc[a] = 0.0;
    int64_t i0, i1;
    chunk_span(ck, &i0, &i1);
    for (int64_t e = 3 * i0 + threadIdx.x; e < 3 * i1; e += RED_THREADS) {
        const double sk = zn[e] - zo[e], yk = gn[e] - go[e];
        s[e] = sk; y[e] = yk;
        acc[0] += yk * sk; acc[1] += sk * sk; acc[2] += yk * yk; acc[3] = fmax(acc[3], fabs(sk));
#pragma unroll
        for (int k = 0; k < K; ++k) { acc[4 + k] += yk * h.S[k][e]; acc[4 + K + k] += h.Y[k][e] * sk; }
    }
    __shared__ double sh[RED_THREADS / 32][A];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int a = 0; a < A; ++a) {
        double v = acc[a];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double t = __shfl_xor_sync(0xffffffffu, v, o);
            v = a == 3 ? fmax(v, t) : v + t;
        }
        if (lane == 0) sh[w][a] = v;
    }
    __syncthreads();
    for (int a = threadIdx.x; a < A; a += RED_THREADS) {
        double v = sh[0][a];
        for (int q = 1; q < RED_THREADS / 32; ++q) v = a == 3 ? fmax(v, sh[q][a]) : v + sh[q][a];
        *chunk_slot(red, ck, a) = v;
    }
}

// ------------------------------------------------------------------ evaluation scalars
// Per chunk: sum E_i, sum |g_i|^2, obtuse count, min lloyd_diag (the nonpositive-diagonal test
// of cvt_core.py:184) and, for a line-search trial, the directional derivative
// sum g.(q3/|v|) (optimizer.py:330).  e_gen, g2_gen, ob_gen, diag, grad, q3, norms are
// slice-local.  A missing generator (NaN E) poisons the energy: the coverage check.
__global__ void __launch_bounds__(RED_THREADS)
k_eval_reduce(const double* __restrict__ e_gen, const double* __restrict__ g2_gen,
              const double* __restrict__ ob_gen, const double* __restrict__ diag,
              const double* __restrict__ grad, const double* __restrict__ q3,
              const double* __restrict__ norms, Chunks ck, double* __restrict__ red) {
    double se = 0.0, sg = 0.0, so = 0.0, mn = INFINITY, sd = 0.0;
    int64_t i0, i1;
    chunk_span(ck, &i0, &i1);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += RED_THREADS) {
        se += e_gen[i];
        sg += g2_gen[i];
        so += ob_gen[i];
        mn = fmin(mn, diag[i]);
        if (q3) {
            const double nr = norms[i];
            sd += grad[3 * i] * (q3[3 * i] / nr) + grad[3 * i + 1] * (q3[3 * i + 1] / nr) +
                  grad[3 * i + 2] * (q3[3 * i + 2] / nr);
        }
    }
    se = block_reduce<0>(se); sg = block_reduce<0>(sg); so = block_reduce<0>(so);
    mn = block_reduce<2>(mn); sd = block_reduce<0>(sd);
    if (threadIdx.x == 0) {
        *chunk_slot(red, ck, 0) = se;
        *chunk_slot(red, ck, 1) = sg;
        *chunk_slot(red, ck, 2) = so;
        *chunk_slot(red, ck, 3) = mn;
        *chunk_slot(red, ck, 4) = sd;
    }
}

// fixed-order pass over the chunk partials of nval values (op per value: 0 sum, 1 max, 2 min)
struct RedOps {
    unsigned char op[MAX_RED_VALS];
};

__global__ void k_reduce_chunks(const double* __restrict__ red, int nval, RedOps ops,
                                double* __restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int v = warp; v < nval; v += nw) {
        const double* pv = red + (int64_t)v * CHUNKS;
        const int op = ops.op[v];
        const double r = op == 0 ? warp_chunks<0>(pv) : (op == 1 ? warp_chunks<1>(pv)
                                                                 : warp_chunks<2>(pv));
        if (lane == 0) out[v] = r;
    }
}

// ------------------------------------------------------------------ graph Laplacian
// LaplacianPreconditioner (cvt_core.py:192-229): a_ij = -int over T_ij u T_ji of rho, rows
// summing to zero, perturbed (m2: diagonal x 1.01, a6: + 1e-6 I).  T_ij, the fan
// sub-triangles of cell i next to edge (i, j = row[t]), are half 0 of incidence t and half 1
// of incidence t-1 (delaunay.py:357-361); their masses are the per-half quadrature partials.
// Stored aligned with the cycles: wsym[i][t] = w_ij + w_ji, diag[i] = sum_t wsym[i][t].
__global__ void k_lap_dir(int n, const int* __restrict__ inc_base, const int* __restrict__ deg,
                          const double* __restrict__ part, double* __restrict__ wdir) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int d = deg[i], u0 = inc_base[i];
    for (int t = 0; t < d; ++t)
        wdir[(int64_t)i * MAXDEG + t] = part[(int64_t)(u0 + t) * PART_ROW] +
                                        part[(int64_t)(u0 + (t + d - 1) % d) * PART_ROW + 5];
}

__global__ void k_lap_sym(int n, const int* __restrict__ nbr, const int* __restrict__ deg,
                          const double* __restrict__ wdir, double* __restrict__ wsym,
                          double* __restrict__ diag, int* __restrict__ status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int d = deg[i];
    const int* row = nbr + (int64_t)i * MAXDEG;
    double dsum = 0.0;
    for (int t = 0; t < d; ++t) {
        const int j = row[t];
        const int q = find_in_cycle(nbr + (int64_t)j * MAXDEG, deg[j], i);
        if (q < 0) { atomicOr(status, ST_INCONSISTENT); continue; }
        const double w = wdir[(int64_t)i * MAXDEG + t] + wdir[(int64_t)j * MAXDEG + q];
        wsym[(int64_t)i * MAXDEG + t] = w;
        dsum += w;
    }
    diag[i] = dsum;
}

// Conjugate gradients on the perturbed Laplacian for the three coordinate right-hand sides at
// once (LaplacianPreconditioner.solve, cvt_core.py:231-236; the reference factors it with
// SuperLU).  One chunk per block, fixed-order reductions (bitwise repeatable); the scalars
// live on the device: cg[0..2] r.r, cg[3..5] p.Ap, cg[6..8] new r.r, cg[9..11] b.b.
__device__ __forceinline__ double lap_row(const int* __restrict__ row, int d,
                                          const double* __restrict__ wrow, double dp,
                                          const double* __restrict__ x, int64_t i, int c) {
    double y = dp * x[3 * i + c];
    for (int t = 0; t < d; ++t) y -= wrow[t] * x[3 * (int64_t)row[t] + c];
    return y;
}

__global__ void __launch_bounds__(RED_THREADS)
k_cg_spmv(const int* __restrict__ nbr, const int* __restrict__ deg,
          const double* __restrict__ wsym, const double* __restrict__ dpert,
          const double* __restrict__ p, double* __restrict__ q, Chunks ck,
          double* __restrict__ red) {
    double pq[3] = {0, 0, 0};
    int64_t i0, i1;
    chunk_span(ck, &i0, &i1);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += RED_THREADS) {
        const int d = deg[i];
        const int* row = nbr + i * MAXDEG;
        const double* wrow = wsym + i * MAXDEG;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double y = lap_row(row, d, wrow, dpert[i], p, i, c);
            q[3 * i + c] = y;
            pq[c] += p[3 * i + c] * y;
        }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double v = block_reduce<0>(pq[c]);
        if (threadIdx.x == 0) *chunk_slot(red, ck, c) = v;
    }
}

// Jacobi-preconditioned CG (D = the perturbed diagonal): x += alpha p, r -= alpha q,
// z = r / D (alpha = r.z / p.Ap per coordinate); partials of the new r.z and r.r
__global__ void __launch_bounds__(RED_THREADS)
k_cg_step(double* __restrict__ x, double* __restrict__ r, double* __restrict__ zv,
          const double* __restrict__ p, const double* __restrict__ q,
          const double* __restrict__ dpert, const double* __restrict__ cg, Chunks ck,
          double* __restrict__ red, int* __restrict__ status) {
    double al[3], rz[3] = {0, 0, 0}, rr[3] = {0, 0, 0};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        al[c] = cg[3 + c] != 0.0 ? cg[c] / cg[3 + c] : 0.0;
        if (!(cg[3 + c] > 0.0) && cg[c] > 0.0 && blockIdx.x == 0 && threadIdx.x == 0)
            atomicOr(status, ST_INDEFINITE);
    }
    int64_t i0, i1;
    chunk_span(ck, &i0, &i1);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += RED_THREADS) {
        const double inv_d = 1.0 / dpert[i];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int64_t e = 3 * i + c;
            x[e] = fma(al[c], p[e], x[e]);
            const double rv = fma(-al[c], q[e], r[e]);
            r[e] = rv;
            const double zz = rv * inv_d;
            zv[e] = zz;
            rz[c] += rv * zz;
            rr[c] += rv * rv;
        }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double v = block_reduce<0>(rz[c]);
        if (threadIdx.x == 0) *chunk_slot(red, ck, c) = v;
        const double w = block_reduce<0>(rr[c]);
        if (threadIdx.x == 0) *chunk_slot(red, ck, 3 + c) = w;
    }
}

// start of the preconditioned iteration: r = b, z = p = b / D; chunk partials of r.z and b.b
__global__ void __launch_bounds__(RED_THREADS)
k_cg_start(const double* __restrict__ b, const double* __restrict__ dpert,
           double* __restrict__ r, double* __restrict__ zv, double* __restrict__ p, Chunks ck,
           double* __restrict__ red) {
    double rz[3] = {0, 0, 0}, bb[3] = {0, 0, 0};
    int64_t i0, i1;
    chunk_span(ck, &i0, &i1);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += RED_THREADS) {
        const double inv_d = 1.0 / dpert[i];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int64_t e = 3 * i + c;
            const double bv = b[e], zz = bv * inv_d;
            r[e] = bv;
            zv[e] = zz;
            p[e] = zz;
            rz[c] += bv * zz;
            bb[c] += bv * bv;
        }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double v = block_reduce<0>(rz[c]);
        if (threadIdx.x == 0) *chunk_slot(red, ck, c) = v;
        const double w = block_reduce<0>(bb[c]);
        if (threadIdx.x == 0) *chunk_slot(red, ck, 3 + c) = w;
    }
}

// p = z + beta p (beta = new r.z / r.z), then r.z <- new r.z (one thread, after the pass)
__global__ void k_cg_dir(double* __restrict__ p, const double* __restrict__ zv,
                         double* __restrict__ cg, int64_t len) {
    double be[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) be[c] = cg[c] != 0.0 ? cg[6 + c] / cg[c] : 0.0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len;
         e += (int64_t)gridDim.x * blockDim.x)
        p[e] = fma(be[e % 3], p[e], zv[e]);
}

__global__ void k_cg_roll(double* __restrict__ cg) {
    if (threadIdx.x < 3) cg[threadIdx.x] = cg[6 + threadIdx.x];
}

// ------------------------------------------------------------------ LBFGS vector kernels
__global__ void k_copy(const double* __restrict__ x, int64_t len, double* __restrict__ y) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < len;
         k += (int64_t)gridDim.x * blockDim.x)
        y[k] = x[k];
}

__global__ void k_scale(double a, const double* __restrict__ x, int64_t len,
                        double* __restrict__ y) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < len;
         k += (int64_t)gridDim.x * blockDim.x)
        y[k] = a * x[k];
}

// backward step of the two-loop: a = rho * (s.q) from partials; q -= a*y; store a
__global__ void __launch_bounds__(RED_THREADS)
k_twoloop_back(double* __restrict__ q, const double* __restrict__ y, int64_t len,
               const double* __restrict__ partials, double rho, double* __restrict__ a_store) {
    double a = rho * finish_partials<0>(partials);
    if (blockIdx.x == 0 && threadIdx.x == 0) *a_store = a;
    for (int64_t k = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; k < len;
         k += (int64_t)gridDim.x * RED_THREADS)
        q[k] -= a * y[k];
}

// forward step: b = rho * (y.q); q += s*(a - b); optional negation at the end
__global__ void __launch_bounds__(RED_THREADS)
k_twoloop_fwd(double* __restrict__ q, const double* __restrict__ s, int64_t len,
              const double* __restrict__ partials, double rho, const double* __restrict__ a_store,
              int negate) {
    double b = rho * finish_partials<0>(partials);
    double c = *a_store - b;
    for (int64_t k = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; k < len;
         k += (int64_t)gridDim.x * RED_THREADS) {
        double v = q[k] + s[k] * c;
        q[k] = negate ? -v : v;
    }
}

// h0 application (LloydDiagonal: q * (1/d) blockwise; GammaIdentity: gamma*q), with the
// final negation folded in when there is no forward loop
__global__ void k_apply_h0(double* __restrict__ q, const double* __restrict__ diag, double gamma,
                           int64_t n, int negate) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < 3 * n;
         k += (int64_t)gridDim.x * blockDim.x) {
        double v = diag ? q[k] * (1.0 / diag[k / 3]) : gamma * q[k];
        q[k] = negate ? -v : v;
    }
}

// q3 = q - (q.z) z per row; chunk partials of g.q3
__global__ void __launch_bounds__(RED_THREADS)
k_tangent(const double* __restrict__ q, const double* __restrict__ z,
          const double* __restrict__ g, Chunks ck, double* __restrict__ q3,
          double* __restrict__ red) {
    double v = 0.0;
    int64_t i0, i1;
    chunk_span(ck, &i0, &i1);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += RED_THREADS) {
        double qx = q[3 * i], qy = q[3 * i + 1], qz = q[3 * i + 2];
        double zx = z[3 * i], zy = z[3 * i + 1], zz = z[3 * i + 2];
        double qd = qx * zx + qy * zy + qz * zz;
        double ax = qx - qd * zx, ay = qy - qd * zy, az = qz - qd * zz;
        q3[3 * i] = ax; q3[3 * i + 1] = ay; q3[3 * i + 2] = az;
        v += g[3 * i] * ax + g[3 * i + 1] * ay + g[3 * i + 2] * az;
    }
    v = block_reduce<0>(v);
    if (threadIdx.x == 0) *chunk_slot(red, ck, 0) = v;
}

__global__ void k_trial(const double* __restrict__ z, const double* __restrict__ q3, double alpha,
                        int64_t n, double* __restrict__ zt, double* __restrict__ norms) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double vx = z[3 * i] + alpha * q3[3 * i];
        double vy = z[3 * i + 1] + alpha * q3[3 * i + 1];
        double vz = z[3 * i + 2] + alpha * q3[3 * i + 2];
        double nr = sqrt(vx * vx + vy * vy + vz * vz);
        norms[i] = nr;
        zt[3 * i] = vx / nr; zt[3 * i + 1] = vy / nr; zt[3 * i + 2] = vz / nr;
    }
}

__global__ void __launch_bounds__(RED_THREADS)
k_dirderiv(const double* __restrict__ g, const double* __restrict__ q3,
           const double* __restrict__ norms, Chunks ck, double* __restrict__ red) {
    double v = 0.0;
    int64_t i0, i1;
    chunk_span(ck, &i0, &i1);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += RED_THREADS) {
        double nr = norms[i];
        v += g[3 * i] * (q3[3 * i] / nr) + g[3 * i + 1] * (q3[3 * i + 1] / nr) +
             g[3 * i + 2] * (q3[3 * i + 2] / nr);
    }
    v = block_reduce<0>(v);
    if (threadIdx.x == 0) *chunk_slot(red, ck, 0) = v;
}

__global__ void k_lloyd(const double* __restrict__ c, int64_t n, double* __restrict__ z,
                        int* __restrict__ status) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double x = c[3 * i], y = c[3 * i + 1], w = c[3 * i + 2];
        double nr = sqrt(x * x + y * y + w * w);
        if (!(nr > 1e-12)) atomicOr(status, ST_CENTROID);
        z[3 * i] = x / nr; z[3 * i + 1] = y / nr; z[3 * i + 2] = w / nr;
    }
}

__global__ void k_normalize(double* __restrict__ z, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double x = z[3 * i], y = z[3 * i + 1], w = z[3 * i + 2];
        double nr = sqrt(x * x + y * y + w * w);
        z[3 * i] = x / nr; z[3 * i + 1] = y / nr; z[3 * i + 2] = w / nr;
    }
}

// ------------------------------------------------------------------ covering migration
// Region-mode bookkeeping of the reference (partition.py:123-164, pipeline.py:163-167, 244-259):
// the geometric cell of every point is its Euclidean-nearest covering centre (argmax z.c,
// ties to the lowest index); a fresh decomposition freezes it as the arithmetic cell; later
// evaluations classify the movement: 0 in-place, 1 every moved point stayed in a one-level
// neighbour of its arithmetic cell, 2 out-of-range (max over the points).
__global__ void k_migration(const double* __restrict__ z, int64_t n,
                            const double* __restrict__ centers, int p,
                            const uint32_t* __restrict__ adj, int words,
                            int* __restrict__ arith, int fresh, int* __restrict__ cls) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = z[3 * i], y = z[3 * i + 1], w = z[3 * i + 2];
    double best = -INFINITY;
    int arg = 0;
    for (int c = 0; c < p; ++c) {
        const double sc = x * __ldg(centers + 3 * c) + y * __ldg(centers + 3 * c + 1) +
                          w * __ldg(centers + 3 * c + 2);
        if (sc > best) { best = sc; arg = c; }
    }
    if (fresh) { arith[i] = arg; return; }
    const int a = arith[i];
    if (arg == a) return;
    const bool near = (adj[(int64_t)a * words + (arg >> 5)] >> (arg & 31)) & 1u;
    atomicMax(cls, near ? 1 : 2);
}

// ------------------------------------------------------------------ region-path fallback
// The reference's region path (pipeline.py:62-98, 171-242, 244-259) triangulates every
// Voronoi-sort region of a covering separately and falls back to the global path -- counting
// the evaluation in MeshEvaluator.fallbacks -- when a region fails.  Its moments equal the
// global path's, so only that decision is reproduced here, from the global cycles: a region
// fails when it holds an owned point but < 3 members (InsufficientPointsError,
// pipeline.py:188-191), when a member sits within eps of the antipode of its contact point
// (AntipodeError, geometry.py:76-79), or when a Delaunay triangle at an owned generator is not
// kept by select_region_triangles (delaunay.py:252-273: a vertex outside the region, or
// d_out - d_in < 2 r), which truncates that generator's fan (CoverageError, validate_fans
// delaunay.py:410-426).  Arithmetic as the reference's NumPy: no FMA contraction, canonical
// vertex order for the circumcircle (delaunay.py:150-169 with the cap's `avoid`).
__device__ __forceinline__ bool cov_adj(const uint32_t* adj, int words, int a, int b) {
    return (adj[(int64_t)a * words + (b >> 5)] >> (b & 31)) & 1u;
}

__global__ void k_geo_cells(const double* __restrict__ z, int64_t n,
                            const double* __restrict__ centers, int p, int* __restrict__ geo,
                            int* __restrict__ hist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = z[3 * i], y = z[3 * i + 1], w = z[3 * i + 2];
    double best = -INFINITY;
    int arg = 0;
    for (int c = 0; c < p; ++c) {
        const double sc = x * __ldg(centers + 3 * c) + y * __ldg(centers + 3 * c + 1) +
                          w * __ldg(centers + 3 * c + 2);
        if (sc > best) { best = sc; arg = c; }
    }
    geo[i] = arg;
    atomicAdd(&hist[arg], 1);
}

__device__ __forceinline__ double np_dot3(V3 a, V3 b) {     // ((ax bx + ay by) + az bz)
    return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}

__device__ __forceinline__ V3 np_cross(V3 a, V3 b) {
    return v3(__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)),
              __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
              __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

__device__ __forceinline__ double np_geodesic(V3 a, V3 b) {   // geometry.py:29-40
    const V3 c = np_cross(a, b);
    return atan2(sqrt(np_dot3(c, c)), np_dot3(a, b));
}

// fail[l] bits of region l: 1 coverage (truncated fan), 2 antipode (4, too few members, is
// added on the host)
__global__ void k_region_cover(const double* __restrict__ z, int64_t n, const int* __restrict__ nbr,
                               const int* __restrict__ deg, const double* __restrict__ centers,
                               int p, const uint32_t* __restrict__ adj,
                               const int* __restrict__ geo, const int* __restrict__ hist,
                               double eps_proj, int* __restrict__ fail) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int words = (p + 31) / 32;
    const int g = geo[i];
    const V3 zi = load3(z, i);
    // antipode of the contact point of every region that has i as a member and owns points
    for (int l = 0; l < p; ++l) {
        if (hist[l] == 0 || !(l == g || cov_adj(adj, words, l, g))) continue;
        const V3 t = load3(centers, l);
        const double den = __dadd_rn(__dadd_rn(__dmul_rn(t.x, __dadd_rn(zi.x, t.x)),
                                               __dmul_rn(t.y, __dadd_rn(zi.y, t.y))),
                                     __dmul_rn(t.z, __dadd_rn(zi.z, t.z)));
        if (den <= eps_proj) atomicOr(&fail[l], 2);
    }
    // the triangles at the owned generator i (region g) must all be kept
    const int d = deg[i];
    const int* row = nbr + i * MAXDEG;
    const V3 tc = load3(centers, g);
    for (int k = 0; k < d; ++k) {
        const int a = row[k], b = row[k + 1 == d ? 0 : k + 1];
        const int ga = geo[a], gb = geo[b];
        if (!(ga == g || cov_adj(adj, words, g, ga)) || !(gb == g || cov_adj(adj, words, g, gb))) {
            atomicOr(&fail[g], 1);
            return;
        }
        // canonical rotation (min id first, orientation kept)
        int v0 = (int)i, v1 = a, v2 = b;
        if (a < v0 && a < b) { v0 = a; v1 = b; v2 = (int)i; }
        else if (b < v0 && b < a) { v0 = b; v1 = (int)i; v2 = a; }
        const V3 p0 = load3(z, v0), p1 = load3(z, v1), p2 = load3(z, v2);
        const V3 e1 = v3(__dsub_rn(p1.x, p0.x), __dsub_rn(p1.y, p0.y), __dsub_rn(p1.z, p0.z));
        const V3 e2 = v3(__dsub_rn(p2.x, p0.x), __dsub_rn(p2.y, p0.y), __dsub_rn(p2.z, p0.z));
        const V3 nv = np_cross(e1, e2);
        const double nn = sqrt(np_dot3(nv, nv));
        V3 c = v3(__ddiv_rn(nv.x, nn), __ddiv_rn(nv.y, nn), __ddiv_rn(nv.z, nn));
        double r = np_geodesic(c, p0);
        if (np_geodesic(c, v3(-tc.x, -tc.y, -tc.z)) < r) {    // the cap's `avoid`
            c = v3(-c.x, -c.y, -c.z);
            r = M_PI - r;
        }
        double din = INFINITY, dout = INFINITY;
        for (int l = 0; l < p; ++l) {
            const double cs = fmin(fmax(np_dot3(c, load3(centers, l)), -1.0), 1.0);
            const double dl = acos(cs);
            if (l == g || cov_adj(adj, words, g, l)) din = fmin(din, dl);
            else dout = fmin(dout, dl);
        }
        if (dout != INFINITY && !(__dsub_rn(dout, din) >= __dmul_rn(2.0, r))) {
            atomicOr(&fail[g], 1);
            return;
        }
    }
}

// ------------------------------------------------------------------ canonical triangles
__global__ void k_tri_count(int n, const int* __restrict__ nbr, const int* __restrict__ deg,
                            int* __restrict__ cnt) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i == n) { cnt[n] = 0; return; }
    int d = deg[i], c = 0;
    const int* row = nbr + (int64_t)i * MAXDEG;
    for (int t = 0; t < d; ++t) {
        int a = row[t], b = row[t + 1 == d ? 0 : t + 1];
        c += (i < a && i < b);
    }
    cnt[i] = c;
}

__global__ void k_tri_emit(int n, const int* __restrict__ nbr, const int* __restrict__ deg,
                           const uint8_t* __restrict__ amb, const int* __restrict__ off,
                           int64_t tmax, int64_t* __restrict__ tri, uint8_t* __restrict__ flags) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int d = deg[i];
    const int* row = nbr + (int64_t)i * MAXDEG;
    int la[MAXDEG], lb[MAXDEG], lf[MAXDEG];
    int m = 0;
    for (int t = 0; t < d; ++t) {
        int tp = t + 1 == d ? 0 : t + 1;
        int a = row[t], b = row[tp];
        if (!(i < a && i < b)) continue;
        int f = amb[(int64_t)i * MAXDEG + t] | amb[(int64_t)i * MAXDEG + tp];
        // third edge (a, b) seen from a: b's slot in a's cycle
        int da = deg[a];
        const int* ra = nbr + (int64_t)a * MAXDEG;
        int pb = find_in_cycle(ra, da, b);
        if (pb >= 0) f |= amb[(int64_t)a * MAXDEG + pb];
        int pi = find_in_cycle(ra, da, i);
        if (pi >= 0) f |= amb[(int64_t)a * MAXDEG + pi];
        // insertion sort by second id
        int k = m++;
        while (k > 0 && la[k - 1] > a) { la[k] = la[k - 1]; lb[k] = lb[k - 1]; lf[k] = lf[k - 1]; --k; }
        la[k] = a; lb[k] = b; lf[k] = f;
    }
    int64_t o = off[i];
    for (int k = 0; k < m; ++k) {
        if (o + k >= tmax) break;
        tri[3 * (o + k)] = i; tri[3 * (o + k) + 1] = la[k]; tri[3 * (o + k) + 2] = lb[k];
        if (flags) flags[o + k] = (uint8_t)lf[k];
    }
}

// ------------------------------------------------------------------ cycles from a triangle list
__global__ void k_tl_fill(const int64_t* __restrict__ tri, int64_t t, int* __restrict__ cursor,
                          int* __restrict__ pairs, int* __restrict__ status) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= t) return;
    int v[3] = {(int)tri[3 * r], (int)tri[3 * r + 1], (int)tri[3 * r + 2]};
    for (int c = 0; c < 3; ++c) {
        int i = v[c], j = v[(c + 1) % 3], k = v[(c + 2) % 3];
        int slot = atomicAdd(&cursor[i], 1);
        if (slot >= MAXDEG) { atomicOr(status, ST_DEG_OVERFLOW); continue; }
        pairs[((int64_t)i * MAXDEG + slot) * 2] = j;
        pairs[((int64_t)i * MAXDEG + slot) * 2 + 1] = k;
    }
}

// chain the (next, prev) pairs of each vertex into the CCW cycle starting at its min id
__global__ void k_tl_chain(int n, const int* __restrict__ pairs, const int* __restrict__ cursor,
                           int* __restrict__ nbr, int* __restrict__ deg, int* __restrict__ status) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int d = cursor[i];
    if (d > MAXDEG || d < 3) { deg[i] = 0; atomicOr(status, ST_INCONSISTENT); return; }
    const int* pr = pairs + (int64_t)i * MAXDEG * 2;
    int start = pr[0];
    for (int s = 1; s < d; ++s) start = min(start, pr[2 * s]);
    int* row = nbr + (int64_t)i * MAXDEG;
    int cur = start;
    for (int t = 0; t < d; ++t) {
        row[t] = cur;
        int nx = -1;
        for (int s = 0; s < d; ++s)
            if (pr[2 * s] == cur) { nx = pr[2 * s + 1]; break; }
        if (nx < 0) { atomicOr(status, ST_INCONSISTENT); deg[i] = 0; return; }
        cur = nx;
    }
    if (cur != start) atomicOr(status, ST_INCONSISTENT);
    deg[i] = d;
}

}  // namespace

// ====================================================================== context
struct scvt_ctx {
    int device = 0;
    int64_t n_max = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    int64_t launches = 0;
    // config
    DensityParams dp{};
    int measure = 0;
    int nq = 0;
    bool sym7 = false;           // node table = symmetric 7-node rule on depth-3 leaves
    int m = 7;
    double* d_nodes = nullptr;   // [3][nq]
    double* d_table = nullptr;   // [2][tab_k][TAB_P+1] rho^(1/4) table (tanh4 kinds)
    DensityParams* d_dp = nullptr;   // device copy of dp (tab = d_table)
    // grid
    int g_max = 1;
    uint32_t* d_keys = nullptr; uint32_t* d_skeys = nullptr;
    int* d_vals = nullptr; int* d_ids = nullptr;
    int* d_start = nullptr;
    double* d_zs = nullptr;
    void* d_cub = nullptr; size_t cub_bytes = 0;
    char* arena = nullptr;       // the one device allocation every d_* buffer below lives in
    void* h_arena = nullptr;     // the one pinned allocation of the h_* readback words
    // cells
    int* d_nbr = nullptr; int* d_deg = nullptr; uint8_t* d_amb = nullptr;
    int* d_inc_start = nullptr; int* d_inc_gen = nullptr; int* d_inc_base = nullptr;
    int* d_pairs = nullptr; int* d_cursor = nullptr;
    // quadrature
    double* d_part = nullptr; uint8_t* d_obt = nullptr;
    int* d_defer = nullptr;            // [12 n + 1]: k_quad's queue for k_quad_table, count last
    double* d_egen = nullptr; double* d_g2gen = nullptr; double* d_obgen = nullptr;
    // reductions and status
    double* d_partials = nullptr;      // [MAX_SLOTS][RED_BLOCKS] and [MAX_RED_VALS][CHUNKS]
    double* d_scal = nullptr;          // [MAX_RED_VALS]
    int* d_status = nullptr;           // [64]: status + stats [0,16), d_nbad [16], d_fcnt [24,32), d_fhist [32,48)
    double* h_scal = nullptr;          // pinned [MAX_RED_VALS]
    int* h_status = nullptr;           // pinned [64]: one copy of the whole d_status block
    int* h_small = nullptr;            // pinned [32]: small readbacks (reuse counts, flip rounds)
    double* h_dir = nullptr;           // pinned [2]: scalars of the asynchronous direction
    cudaEvent_t dir_ev = nullptr;      // recorded after their copy
    int* d_rcount = nullptr;           // per-round bad counts of the chained reuse rounds
    int* d_queue = nullptr;            // work queue of the fixed-grid cell rebuilds
    int* d_mig = nullptr;              // covering migration class (scvt_migration)
    // flip repair: candidates {i, a, b, c} (<= 3n), tickets, double-buffered id lists,
    // counters {ncand, nlist[2], nflips}
    int4* d_cand = nullptr;
    double* d_wdir = nullptr;          // graph Laplacian: directed pair masses [n][MAXDEG] (lazy)
    double* d_cgv = nullptr;           // CG work vectors r, p, q: [3][3 n] (lazy)
    double* d_cg = nullptr;            // CG scalars [16] (lazy)
    unsigned long long* d_lock = nullptr;
    int* d_flist = nullptr;            // [2][4 n]: touched cells, four slots per candidate
    int* d_fflag = nullptr;            // [n]
    int* d_fcnt = nullptr;             // [8] flip counters (queues, lists, flips, tail): d_status + 24
    int* d_fhist = nullptr;            // [16] queue length per grid-wide round: d_status + 32
    int flip_grid_rounds = 6;          // grid-wide rounds before k_flip_tail (adapted per evaluation)
    int flip_rounds_enqueued = 0;      // grid-wide rounds of the repair in flight
    int last_nbad = 0;                 // bad cells the previous flip repair left (rebuild path taken)
    bool shard_quad_pending = false;   // a sharded k_quad event pair not yet added to prof_ms
    int deferred_rounds = 0;           // rebuild rounds chained behind the deferred flip repair
    int tail_enter = 128;              // see flip_account (SCVT_TAIL_ENTER)
    int tail_rounds = TAIL_MAX_ROUNDS; // k_flip_tail round limit (SCVT_TAIL_ROUNDS: tests force give-ups)
    int64_t flip_cap = 0;              // flip queue capacity, 0 = n (SCVT_FLIP_CAP: tests force overflows)
    int64_t flip_stats[4] = {0, 0, 0, 0};   // evaluations, rounds, flips, fell back
    int64_t last_flips = 0;                  // flips of the previous repair
    int* d_counts = nullptr;           // sharded reuse: per-shard bad counts [MAX_SHARDS+1]
    int* h_counts = nullptr;           // pinned copy
    // LBFGS history
    double* d_S = nullptr; double* d_Y = nullptr;   // [m][3 n_max]
    double* d_alpha = nullptr;                      // [m]
    std::vector<double> rho, ys, yy;
    double YS[16][16] = {};            // y_slot_i . s_slot_j of the stored pairs (host)
    double* d_coef = nullptr;          // two-loop coefficients a[MAXM], c[MAXM] (device)
    int hist_head = 0, hist_count = 0;
    double* d_tmp_s = nullptr; double* d_tmp_y = nullptr;   // staging for push
    // history pair staged by an evaluation (scvt_evaluate_staged): its scalars came back with
    // the evaluation's, so committing it needs no kernel pass and no host round trip
    bool staged_valid = false;
    const double* staged_z = nullptr; const double* staged_g = nullptr;
    int staged_head = 0, staged_count = 0;
    double staged_sc[4 + 2 * 16] = {};
    // live per-kernel timing (bench roofline): pairs {cells, quad, evaluate}
    bool prof = false;
    cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    double prof_ms[4] = {0, 0, 0, 0};
    unsigned long long* d_diag = nullptr;   // cell-builder work counters (profiling only)
    // cycle reuse across evaluations
    int64_t cycles_n = -1;                  // n of the certified cycles held in d_nbr/d_deg
    int split = 0;                          // k_quad thread per sub-triangle (set per n)
    int* d_bad = nullptr; int* d_nbad = nullptr; uint8_t* d_slotflag = nullptr; int* d_list = nullptr;
    int* d_recheck = nullptr; int* d_nlist = nullptr;   // reuse: cells to re-certify
    int* d_list2 = nullptr; int* d_nlist2 = nullptr;    // sharded reuse: re-check slot list
    int* d_cnt = nullptr;                               // sharded reuse: owned rebuild count
    GridView gv;                                        // grid of the current evaluation
    std::vector<int64_t> plan_counts;                   // bad cells per shard (last plan)
    int64_t reuse_stats[4] = {0, 0, 0, 0};  // checks, bad cells, evaluations fully reused
    int64_t prof_n[4] = {0, 0, 0, 0};
};

namespace {

int fail(scvt_ctx* c, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return code;
}

#define CK(call)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return fail(ctx, SCVT_ERR_CUDA, "%s: %s (%s:%d)", #call,                  \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                  \
    } while (0)

#define LAUNCHED()                                                                    \
    do {                                                                              \
        ++ctx->launches;                                                              \
        cudaError_t e_ = cudaGetLastError();                                          \
        if (e_ != cudaSuccess)                                                        \
            return fail(ctx, SCVT_ERR_CUDA, "launch: %s (%s:%d)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                          \
    } while (0)

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// buckets per face side: ~2 points per bucket at the mean density times a refinement factor
// (SCVT_GRID_REFINE, default 1) so dense regions of very non-uniform sets stay shallow
double grid_refine() {
    const char* e = getenv("SCVT_GRID_REFINE");
    double f = e ? atof(e) : 1.0;
    return f > 0.1 && f < 16.0 ? f : 1.0;
}

// Is the composite node table a depth-3 subdivision of a permutation-symmetric 7-node rule?
// Then k_quad may place nodes leaf by leaf (subtri_moments_sym7): check that the table's
// node set equals that construction and its weights are leaf-independent.
bool is_sym7_depth3(const scvt_config* cfg) {
    if (cfg->n_nodes != 448) return false;
    const double* l1 = cfg->node_l1;
    const double* l2 = cfg->node_l2;
    const double* w = cfg->node_w;
    double nu1[7], nu2[7];
    for (int q = 0; q < 7; ++q) { nu1[q] = 8.0 * l1[q]; nu2[q] = 8.0 * l2[q]; }
    if (!(w[1] == w[2] && w[2] == w[3] && w[4] == w[5] && w[5] == w[6])) return false;
    // symmetric: (nu1, nu2) -> (nu2, nu1) and (nu0, nu1) permutations stay in the set
    auto in_set = [&](double x, double y) {
        for (int q = 0; q < 7; ++q)
            if (fabs(nu1[q] - x) < 1e-13 && fabs(nu2[q] - y) < 1e-13) return true;
        return false;
    };
    for (int q = 0; q < 7; ++q) {
        double nu0 = 1.0 - nu1[q] - nu2[q];
        if (!in_set(nu2[q], nu1[q]) || !in_set(nu0, nu2[q]) || !in_set(nu1[q], nu0)) return false;
    }
    // every table node must be a grid node of the construction, with its orbit's weight
    for (int k = 0; k < 448; ++k) {
        bool found = false;
        for (int pass = 0; pass < 2 && !found; ++pass)
            for (int a = 0; a < 8 - pass && !found; ++a)
                for (int b = 0; b < 8 - pass - a && !found; ++b)
                    for (int q = 0; q < 7 && !found; ++q) {
                        double sg = pass ? -1.0 : 1.0;
                        double x = (a + pass + sg * nu1[q]) / 8.0, y = (b + pass + sg * nu2[q]) / 8.0;
                        if (fabs(x - l1[k]) < 1e-13 && fabs(y - l2[k]) < 1e-13 &&
                            fabs(w[k] - w[q]) <= 1e-15 * fabs(w[q]))
                            found = true;
                    }
        if (!found) return false;
    }
    return true;
}

int grid_for(int64_t n) {
    double g = sqrt((double)n / 12.0) * grid_refine();
    int G = (int)g;
    if (G > 4096) G = 4096;
    return G < 1 ? 1 : G;
}

int status_to_code(scvt_ctx* ctx, int st) {
    if (!st) return SCVT_OK;
    if (st & ST_DUPLICATE)
        return fail(ctx, SCVT_ERR_INSUFFICIENT_POINTS,
                    "duplicate generators: points fell inside the convex hull");
    if (st & ST_UNBOUNDED)
        return fail(ctx, SCVT_ERR_INSUFFICIENT_POINTS,
                    "a Voronoi cell spans a hemisphere (degenerate global point set)");
    if (st & (ST_POLY_OVERFLOW | ST_DEG_OVERFLOW))
        return fail(ctx, SCVT_ERR_CAPACITY, "valence exceeds %d (status 0x%x)", MAXDEG, st);
    if (st & ST_POLE)
        return fail(ctx, SCVT_ERR_POLE_AMBIGUITY, "longitude undefined within 1e-9 of a pole");
    if (st & ST_CENTROID)
        return fail(ctx, SCVT_ERR_CENTROID_AT_ORIGIN, "first moment ~0");
    if (st & ST_DEGENERATE_TRI)
        return fail(ctx, SCVT_ERR_DEGENERATE_TRIANGLE, "degenerate triangle in the fan");
    if (st & ST_INDEFINITE)
        return fail(ctx, SCVT_ERR_FACTORIZATION, "perturbed Laplacian is numerically indefinite");
    return fail(ctx, SCVT_ERR_COVERAGE,
                "triangulation certificate failed (status 0x%x: %s%s%s)", st,
                (st & ST_INCONSISTENT) ? "inconsistent cycles " : "",
                (st & ST_NOT_DELAUNAY) ? "non-Delaunay edge " : "",
                (st & ST_EULER) ? "Euler count" : "");
}

template <typename T>
int dalloc(scvt_ctx* ctx, T** p, size_t count) {
    CK(cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T)));
    return SCVT_OK;
}

#define TRY(x)                 \
    do {                       \
        int r_ = (x);          \
        if (r_) return r_;     \
    } while (0)

// read back `nd` scalars from d_scal and the status block; synchronises the stream
int readback(scvt_ctx* ctx, int nd) {
    if (nd) CK(cudaMemcpyAsync(ctx->h_scal, ctx->d_scal, nd * sizeof(double),
                               cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, 64 * sizeof(int), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return SCVT_OK;
}

int reset_status(scvt_ctx* ctx) {
    CK(cudaMemsetAsync(ctx->d_status, 0, 16 * sizeof(int), ctx->stream));
    return SCVT_OK;
}

// dot(a, b) -> partial slot
int dot_to_slot(scvt_ctx* ctx, const double* a, const double* b, int64_t len, int slot) {
    k_dot_stage1<<<RED_BLOCKS, RED_THREADS, 0, ctx->stream>>>(a, b, len,
                                                             ctx->d_partials + slot * RED_BLOCKS);
    LAUNCHED();
    return SCVT_OK;
}

// sum(slots) -> d_scal[0..nslots) -> host
int finish_slots(scvt_ctx* ctx, int nslots) {
    k_reduce_stage2<0><<<1, RED_THREADS, 0, ctx->stream>>>(ctx->d_partials, nslots, ctx->d_scal);
    LAUNCHED();
    return SCVT_OK;
}

// ---------------------------------------------------------------------- chunked reductions
// rank `rank` of `world` (world divides CHUNKS) owns chunks [rank C/W, (rank+1) C/W)
int make_chunks(scvt_ctx* ctx, int64_t n, int rank, int world, Chunks* c) {
    if (world < 1 || rank < 0 || rank >= world || CHUNKS % world)
        return fail(ctx, SCVT_ERR_CONFIG, "slice %d of %d: the world size must divide %d", rank,
                    world, CHUNKS);
    c->ch = std::max<int64_t>(1, (n + CHUNKS - 1) / CHUNKS);
    c->nc = CHUNKS / world;
    c->c_lo = rank * c->nc;
    c->lo = std::min<int64_t>(n, (int64_t)c->c_lo * c->ch);
    c->len = std::min<int64_t>(n, (int64_t)(c->c_lo + c->nc) * c->ch) - c->lo;
    return SCVT_OK;
}

// partial buffers of a slice: zero outside the owned chunks (the cross-rank SUM is then exact)
int prep_red(scvt_ctx* ctx, double* red, int nval, const Chunks& c) {
    if (c.nc < CHUNKS && nval > 0)
        CK(cudaMemsetAsync(red, 0, (size_t)nval * CHUNKS * sizeof(double), ctx->stream));
    return SCVT_OK;
}

// fixed-order reduction of nval values' chunk partials -> d_scal (device)
int reduce_chunks(scvt_ctx* ctx, const double* red, int nval, const unsigned char* ops) {
    if (nval > MAX_RED_VALS) return fail(ctx, SCVT_ERR_CONFIG, "%d values > %d", nval, MAX_RED_VALS);
    RedOps ro;
    for (int v = 0; v < nval; ++v) ro.op[v] = ops ? ops[v] : 0;
    k_reduce_chunks<<<1, 1024, 0, ctx->stream>>>(red, nval, ro, ctx->d_scal);
    LAUNCHED();
    return SCVT_OK;
}

// ---------------------------------------------------------------------- triangulation core
// cube-map grid over all n points (replicated on every shard; deterministic)
int build_grid(scvt_ctx* ctx, const double* z, int64_t n, GridView* gv) {
    if (n < 4) return fail(ctx, SCVT_ERR_INSUFFICIENT_POINTS,
                           "need >= 4 points on the sphere, got %lld", (long long)n);
    if (n > ctx->n_max) return fail(ctx, SCVT_ERR_CAPACITY, "n=%lld > n_max=%lld",
                                    (long long)n, (long long)ctx->n_max);
    int G = std::min(grid_for(n), ctx->g_max);
    int nb = 6 * G * G;
    cudaStream_t s = ctx->stream;
    k_bucket_keys<<<blocks_for(n, 256), 256, 0, s>>>(z, (int)n, G, ctx->d_keys, ctx->d_vals);
    LAUNCHED();
    int bits = 1;
    while ((1 << bits) < nb) ++bits;
    size_t tb = ctx->cub_bytes;
    CK(cub::DeviceRadixSort::SortPairs(ctx->d_cub, tb, ctx->d_keys, ctx->d_skeys, ctx->d_vals,
                                       ctx->d_ids, (int)n, 0, bits, s));
    k_bucket_start<<<blocks_for(n + 1, 256), 256, 0, s>>>(ctx->d_skeys, (int)n, nb, ctx->d_start);
    LAUNCHED();
    k_gather_sorted<<<blocks_for(n, 256), 256, 0, s>>>(z, ctx->d_ids, (int)n, ctx->d_zs);
    LAUNCHED();
    gv->zs = ctx->d_zs; gv->ids = ctx->d_ids; gv->start = ctx->d_start; gv->z = z; gv->G = G;
    gv->n = n;
    ctx->gv = *gv;
    return SCVT_OK;
}

// Voronoi cells of the generators in sorted slots [lo, hi)
int build_cells_range(scvt_ctx* ctx, const GridView& g, int64_t lo, int64_t hi) {
    cudaStream_t s = ctx->stream;
    int64_t cnt = hi - lo;
    if (cnt <= 0) return SCVT_OK;
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[0], s));
    k_cells_warp<<<blocks_for(cnt, CELL_WARPS), CELL_WARPS * 32, 0, s>>>(
        g, (int)lo, (int)hi, nullptr, nullptr, ctx->d_nbr, ctx->d_deg, ctx->d_status,
        ctx->d_status + 8, ctx->prof ? ctx->d_diag : nullptr);
    LAUNCHED();
    k_cells<<<blocks_for(cnt, CELL_THREADS), CELL_THREADS, 0, s>>>(
        g, (int)lo, (int)hi, nullptr, nullptr, ctx->d_nbr, ctx->d_deg, ctx->d_status,
        ctx->d_status + 8);
    LAUNCHED();
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[1], s));
    return SCVT_OK;
}

int verify_range(scvt_ctx* ctx, const double* z, int64_t lo, int64_t hi, int mode = 0) {
    int64_t cnt = hi - lo;
    if (cnt <= 0) return SCVT_OK;
    k_verify<<<blocks_for(cnt * VERIFY_LANES, 128), 128, 0, ctx->stream>>>(
        z, ctx->d_ids, (int)lo, (int)hi, nullptr, nullptr, ctx->d_nbr, ctx->d_deg, ctx->d_amb,
        ctx->d_status, ctx->d_status + 8, mode, ctx->d_bad, ctx->d_nbad);
    LAUNCHED();
    return SCVT_OK;
}

// compact the sorted slots p in [0, n) whose generator has flag[ids[p]] != 0 into d_list
int compact_slots(scvt_ctx* ctx, int64_t n, const int* flag, int* count_dev) {
    cudaStream_t s = ctx->stream;
    k_flag_slots<<<blocks_for(n, 256), 256, 0, s>>>((int)n, ctx->d_ids, flag, ctx->d_slotflag);
    LAUNCHED();
    size_t tb = ctx->cub_bytes;
    thrust::counting_iterator<int> it(0);
    CK(cub::DeviceSelect::Flagged(ctx->d_cub, tb, it, ctx->d_slotflag, ctx->d_list, count_dev,
                                  (int)n, s));
    return SCVT_OK;
}

bool reuse_enabled() { return getenv("SCVT_NO_REUSE") == nullptr; }

// Reuse the previous evaluation's cycles when they are still a certified Delaunay
// triangulation of the new positions; rebuild (grid method) only the cells of failing
// triangles/quads, re-certify, and escalate to a full rebuild when churn is large.
// fixed grids for lists whose length only the device knows: the resident capacity
constexpr int SPEC_CELL_BLOCKS = 148 * 4;     // k_cells_warp: 4 CTAs x 4 warps per SM
constexpr int SPEC_BLOCKS = 148 * 8;          // thread-per-item kernels

// One rebuild round on the device, no host round trip: the bad cells of the last pass are
// compacted, their re-check set marked, rebuilt (grid-stride over the device count), and the
// re-check list certified; the new bad count lands in d_nbad.
// nbad_host >= 0: the bad count is known on the host (exact grids, hardware block
// scheduling); -1: device-only count (resident grid pulling from a work queue).
int reuse_round_device(scvt_ctx* ctx, const double* z, int64_t n, const GridView& g,
                       int nbad_host) {
    cudaStream_t s = ctx->stream;
    TRY(compact_slots(ctx, n, ctx->d_bad, ctx->d_nbad));
    CK(cudaMemsetAsync(ctx->d_recheck, 0, n * sizeof(int), s));
    const bool known = nbad_host >= 0;
    const int nb = known ? std::max(nbad_host, 1) : 0;
    k_mark_recheck<<<known ? blocks_for(nb, 256) : SPEC_BLOCKS, 256, 0, s>>>(
        ctx->d_list, ctx->d_nbad, ctx->d_ids, ctx->d_nbr, ctx->d_deg, ctx->d_recheck);
    LAUNCHED();
    if (known) {
        k_cells_warp<<<blocks_for(nb, CELL_WARPS), CELL_WARPS * 32, 0, s>>>(
            g, 0, (int)n, ctx->d_list, ctx->d_nbad, ctx->d_nbr, ctx->d_deg, ctx->d_status,
            ctx->d_status + 8, ctx->prof ? ctx->d_diag : nullptr);
    } else {
        CK(cudaMemsetAsync(ctx->d_queue, 0, sizeof(int), s));
        k_cells_warp<<<SPEC_CELL_BLOCKS, CELL_WARPS * 32, 0, s>>>(
            g, 0, (int)n, ctx->d_list, ctx->d_nbad, ctx->d_nbr, ctx->d_deg, ctx->d_status,
            ctx->d_status + 8, ctx->prof ? ctx->d_diag : nullptr, ctx->d_queue);
    }
    LAUNCHED();
    k_cells<<<known ? blocks_for(nb, CELL_THREADS) : SPEC_BLOCKS, CELL_THREADS, 0, s>>>(
        g, 0, (int)n, ctx->d_list, ctx->d_nbad, ctx->d_nbr, ctx->d_deg, ctx->d_status,
        ctx->d_status + 8);
    LAUNCHED();
    TRY(compact_slots(ctx, n, ctx->d_recheck, ctx->d_nlist));
    CK(cudaMemsetAsync(ctx->d_bad, 0, n * sizeof(int), s));
    CK(cudaMemsetAsync(ctx->d_nbad, 0, sizeof(int), s));
    k_verify<<<SPEC_BLOCKS, 128, 0, s>>>(z, ctx->d_ids, 0, (int)n, ctx->d_list, ctx->d_nlist,
                                          ctx->d_nbr, ctx->d_deg, ctx->d_amb, ctx->d_status,
                                          ctx->d_status + 8, 1, ctx->d_bad, ctx->d_nbad);
    LAUNCHED();
    return SCVT_OK;
}

// Reuse the previous evaluation's cycles when they are still a certified Delaunay
// triangulation of the new positions; rebuild (grid method) only the cells of failing
// triangles, re-certify those cells and their previous neighbours, at most 4 passes, and
// escalate to a full rebuild when churn is large.  Pass 0 (every cell) is read back on the
// host (certified evaluations stop there); passes 1-2 with their rebuild rounds are chained
// on the device and read back once.
bool flips_enabled() { return getenv("SCVT_NO_FLIPS") == nullptr; }
constexpr int FLIP_GRID_ROUNDS_MAX = 10;   // grid-wide rounds before the single-block tail
// ctx->tail_enter: queue length below which the remaining rounds go to the cluster tail
// (128 warps); SCVT_TAIL_ENTER at context creation
constexpr int FLIP_HIST = 16;              // d_fhist: queue length at the start of each grid round

// detection pass of the flip repair over the sorted slots [lo, hi): candidates and bad marks
int flip_detect(scvt_ctx* ctx, const double* z, int64_t n, int64_t lo, int64_t hi) {
    cudaStream_t s = ctx->stream;
    int* cnt = ctx->d_fcnt;        // [0] candidates (queue 0); the rounds use the rest
    CK(cudaMemsetAsync(cnt, 0, (8 + FLIP_HIST) * sizeof(int), s));   // d_fcnt and d_fhist
    if (hi <= lo) return SCVT_OK;
    const FlipQueue fq{ctx->d_cand, cnt, (int)(ctx->flip_cap > 0 ? std::min(ctx->flip_cap, n) : n)};
    // a bounded grid: every block certifies many cells and stages its candidates in shared
    // memory (one global atomicAdd per block instead of one per candidate)
    const unsigned vb = (unsigned)std::min<int64_t>(2 * SPEC_BLOCKS,
                                                    blocks_for((hi - lo) * VERIFY_LANES, 128));
    k_verify<<<vb, 128, 0, s>>>(
        z, ctx->d_ids, (int)lo, (int)hi, nullptr, nullptr, ctx->d_nbr, ctx->d_deg, ctx->d_amb,
        ctx->d_status, ctx->d_status + 8, 2, ctx->d_bad, ctx->d_nbad, fq);
    LAUNCHED();
    return SCVT_OK;
}

// Flip rounds on the queued candidates (queue 0, cnt[0]), enqueued without any host read:
// ctx->flip_grid_rounds grid-wide rounds (three launches each: k_round_lock, k_flip_apply,
// k_round_finish; double-buffered queues d_cand / d_cand + 3n and touched-cell lists, no
// memsets), then k_flip_tail runs the remaining rounds in one block and marks what it gives
// up on as bad.  Leaves d_bad / d_nbad as the rebuild path expects them: the cells of
// orientation or consistency failures, of rejected flips and of candidates still open.
int flip_rounds_enqueue(scvt_ctx* ctx, const double* z, int64_t n) {
    cudaStream_t s = ctx->stream;
    int* cnt = ctx->d_fcnt;
    // queue capacity (more candidates: rebuild path)
    const int cap = (int)(ctx->flip_cap > 0 ? std::min(ctx->flip_cap, n) : n);
    int4* cand[2] = {ctx->d_cand, ctx->d_cand + n};
    int* list[2] = {ctx->d_flist, ctx->d_flist + 4 * n};   // four slots per candidate
    int cur = 0;
    // grid-stride kernels over at most n items per round: small meshes get small grids
    // (scheduling 1184 mostly idle blocks costs several microseconds per launch at c1)
    const unsigned fb = (unsigned)std::min<int64_t>(SPEC_BLOCKS, blocks_for(n, 128));
    const unsigned ab = (unsigned)std::min<int64_t>(SPEC_BLOCKS, blocks_for(2 * n, APPLY_THREADS));
    const unsigned vb = (unsigned)std::min<int64_t>(SPEC_BLOCKS, blocks_for(VERIFY_LANES * n, 128));
    const int G = std::max(0, std::min(ctx->flip_grid_rounds, FLIP_GRID_ROUNDS_MAX));
    for (int r = 0; r < G; ++r) {
        const int nxt = 1 - cur;
        k_round_lock<<<fb, 256, 0, s>>>(cand[cur], cnt + cur, cap, ctx->d_lock, cnt + nxt,
                                        ctx->d_fhist + r);
        LAUNCHED();
        k_flip_apply<<<ab, APPLY_THREADS, 0, s>>>(cand[cur], cnt + cur, cap, ctx->d_lock,
                                                  ctx->d_nbr, ctx->d_deg, ctx->d_fflag, list[nxt],
                                                  ctx->d_bad, ctx->d_nbad, cnt + 4);
        LAUNCHED();
        const VerifyArgs v{z, ctx->d_ids, 0, (int)n, list[nxt], nullptr, ctx->d_nbr,
                           ctx->d_deg, ctx->d_amb, ctx->d_status, ctx->d_status + 8, 2,
                           ctx->d_bad, ctx->d_nbad, FlipQueue{cand[nxt], cnt + nxt, cap}, 1, 0};
        k_round_finish<<<vb, 128, 0, s>>>(cand[cur], cnt + cur, cap, ctx->d_lock, ctx->d_fflag, v);
        LAUNCHED();
        cur = nxt;
    }
    const VerifyArgs v{z, ctx->d_ids, 0, (int)n, nullptr, nullptr, ctx->d_nbr, ctx->d_deg,
                       ctx->d_amb, ctx->d_status, ctx->d_status + 8, 2, ctx->d_bad, ctx->d_nbad,
                       FlipQueue{nullptr, nullptr, cap}, 1, 0};
    k_flip_tail<<<TAIL_CTAS, TAIL_THREADS, 0, s>>>(cand[0], cand[1], cnt, cur, cap, ctx->d_lock,
                                           ctx->d_nbr, ctx->d_deg, ctx->d_fflag, list[0], list[1], v,
                                           ctx->tail_rounds);
    LAUNCHED();
    ctx->flip_rounds_enqueued = G;
    return SCVT_OK;
}

// After a readback of the status block (h_status holds d_nbad, d_fcnt and d_fhist): the
// repair's statistics, the number of grid-wide rounds for the next evaluation (as many as
// started with more than ctx->tail_enter candidates this time, one more when the tail was
// entered with more), and the bad count.
int flip_account(scvt_ctx* ctx, bool deferred = false) {
    const int* fc = ctx->h_status + 24;
    const int* hist = ctx->h_status + 32;
    const int G = ctx->flip_rounds_enqueued;
    int big = 0, used = 0;
    for (int r = 0; r < G; ++r) {
        used += hist[r] > 0;
        big += hist[r] > ctx->tail_enter;
    }
    int next = big;
    if (big == G && fc[6] > ctx->tail_enter) next = G + 1 + (fc[6] > 8 * ctx->tail_enter);
    ctx->flip_grid_rounds = std::min(next, FLIP_GRID_ROUNDS_MAX);
    ctx->flip_stats[0] += 1;
    ctx->flip_stats[1] += used + fc[5];
    ctx->flip_stats[2] += fc[4];
    ctx->flip_stats[3] += fc[7] > 0 ? 1 : 0;
    ctx->last_flips = fc[4];
    // the bad count right after the flips (a deferred repair copies it to d_status[17] before
    // any chained rebuild round changes d_nbad): the next evaluation's prediction
    ctx->last_nbad = deferred ? ctx->h_status[17] : ctx->h_status[16];
    if (deferred && ctx->deferred_rounds) {      // the chained rounds' certificate passes
        ctx->reuse_stats[0] += ctx->deferred_rounds;
        ctx->reuse_stats[1] += ctx->h_status[17] + ctx->h_status[18];
    }
    return ctx->h_status[16];
}

// synchronous flip repair (sharded entry points): detection, rounds, one readback
int flip_repair(scvt_ctx* ctx, const double* z, int64_t n, int* nbad_host) {
    TRY(flip_detect(ctx, z, n, 0, n));
    TRY(flip_rounds_enqueue(ctx, z, n));
    TRY(readback(ctx, 0));
    *nbad_host = flip_account(ctx);
    return SCVT_OK;
}

// The reuse path once the certificate's bad count is known on the host (nbad > 0): rebuild
// (grid method) only the cells of failing triangles, re-certify those cells and their previous
// neighbours; the first two rebuild rounds are chained on the device and read back once.
// The bucket grid is only needed to rebuild cells: it is built on demand (*have_grid), so an
// evaluation certified by the flip pass keeps the previous slot order (any permutation is
// valid; outputs do not depend on it).
int rebuild_bad_cells(scvt_ctx* ctx, const double* z, int64_t n, int nbad, GridView& g,
                      bool* have_grid, bool* done) {
    cudaStream_t s = ctx->stream;
    *done = false;
    ctx->reuse_stats[0] += 1;                       // certificate passes run
    ctx->reuse_stats[1] += nbad;
    if (nbad == 0) { *done = true; return SCVT_OK; }
    if (nbad > (3 * n) / 4) return SCVT_OK;         // caller rebuilds everything
    if (!*have_grid) {
        TRY(build_grid(ctx, z, n, &g));
        *have_grid = true;
    }
    for (int r = 0; r < 2; ++r) {
        TRY(reuse_round_device(ctx, z, n, g, r == 0 ? nbad : -1));
        CK(cudaMemcpyAsync(ctx->d_rcount + r, ctx->d_nbad, sizeof(int), cudaMemcpyDeviceToDevice, s));
    }
    CK(cudaMemcpyAsync(ctx->h_small, ctx->d_rcount, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ctx->reuse_stats[0] += 2;
    ctx->reuse_stats[1] += ctx->h_small[0] + ctx->h_small[1];
    nbad = ctx->h_small[1];
    if (nbad == 0) { *done = true; return SCVT_OK; }
    if (nbad > (3 * n) / 4) return SCVT_OK;
    TRY(reuse_round_device(ctx, z, n, g, nbad));    // fourth and last pass
    CK(cudaMemcpyAsync(ctx->h_small, ctx->d_nbad, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ctx->reuse_stats[0] += 1;
    ctx->reuse_stats[1] += ctx->h_small[0];
    if (ctx->h_small[0] == 0) *done = true;
    return SCVT_OK;
}

int build_cells_full(scvt_ctx* ctx, const double* z, int64_t n, GridView& g, bool have_grid) {
    if (!have_grid) TRY(build_grid(ctx, z, n, &g));
    TRY(build_cells_range(ctx, g, 0, n));
    return verify_range(ctx, z, 0, n, 0);
}

// Cells for an evaluation at z.  With certified cycles of the previous evaluation at hand they
// are reused: flip-mode certificate + flip rounds.  deferred != null: the repair is only
// ENQUEUED and *deferred set -- the caller runs the moments behind it (they skip themselves on
// the device when d_nbad != 0), reads d_nbad back with the evaluation's scalars and calls
// build_cells_resume if it is not zero: a certified evaluation costs one host round trip.
int build_cells(scvt_ctx* ctx, const double* z, int64_t n, bool* deferred = nullptr) {
    GridView g;
    bool have_grid = false;
    cudaStream_t s = ctx->stream;
    if (deferred) *deferred = false;
    if (ctx->cycles_n == n && reuse_enabled()) {
        if (ctx->prof) CK(cudaEventRecord(ctx->ev[0], s));
        CK(cudaMemsetAsync(ctx->d_bad, 0, n * sizeof(int), s));
        CK(cudaMemsetAsync(ctx->d_nbad, 0, sizeof(int), s));
        int nbad = 0;
        if (flips_enabled()) {
            if (deferred) {
                // Late in a run a few folded cells (no flip repairs those) need the rebuild
                // path at almost every evaluation.  Predicted from the previous evaluation:
                // the bucket grid is built up front and two rebuild rounds are chained on the
                // device behind the flips (device-side counts, no-ops when nothing is bad), so
                // this case, too, costs one host round trip.
                const bool predicted = ctx->last_nbad > 0;
                if (predicted) {
                    TRY(build_grid(ctx, z, n, &g));
                    have_grid = true;
                }
                TRY(flip_detect(ctx, z, n, 0, n));
                TRY(flip_rounds_enqueue(ctx, z, n));
                CK(cudaMemcpyAsync(ctx->d_status + 17, ctx->d_nbad, sizeof(int),
                                   cudaMemcpyDeviceToDevice, s));
                ctx->deferred_rounds = 0;
                if (predicted) {
                    for (int r = 0; r < 2; ++r) {
                        TRY(reuse_round_device(ctx, z, n, g, -1));
                        if (r == 0)
                            CK(cudaMemcpyAsync(ctx->d_status + 18, ctx->d_nbad, sizeof(int),
                                               cudaMemcpyDeviceToDevice, s));
                    }
                    ctx->deferred_rounds = 2;
                }
                if (ctx->prof) CK(cudaEventRecord(ctx->ev[1], s));
                *deferred = true;
                return SCVT_OK;
            }
            TRY(flip_repair(ctx, z, n, &nbad));
        } else {
            TRY(verify_range(ctx, z, 0, n, 1));
            CK(cudaMemcpyAsync(ctx->h_small, ctx->d_nbad, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            nbad = ctx->h_small[0];
        }
        bool done = false;
        TRY(rebuild_bad_cells(ctx, z, n, nbad, g, &have_grid, &done));
        if (ctx->prof) CK(cudaEventRecord(ctx->ev[1], s));
        if (done) {
            ctx->reuse_stats[2] += 1;
            return SCVT_OK;
        }
        CK(cudaMemsetAsync(ctx->d_status + 8, 0, 8 * sizeof(int), s));
    }
    return build_cells_full(ctx, z, n, g, have_grid);
}

// a deferred flip repair reported nbad > 0 bad cells: the rebuild path, then (if the churn is
// too large or the rounds do not converge) everything from scratch
int build_cells_resume(scvt_ctx* ctx, const double* z, int64_t n, int nbad) {
    GridView g = ctx->gv;
    bool have_grid = ctx->deferred_rounds > 0, done = false;
    cudaStream_t s = ctx->stream;
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[0], s));
    if (ctx->deferred_rounds == 0) {
        TRY(rebuild_bad_cells(ctx, z, n, nbad, g, &have_grid, &done));
    } else if (nbad <= (3 * n) / 4) {
        // two rounds already ran behind the flips: the fourth and last pass
        TRY(reuse_round_device(ctx, z, n, g, nbad));
        CK(cudaMemcpyAsync(ctx->h_small, ctx->d_nbad, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        ctx->reuse_stats[0] += 1;
        ctx->reuse_stats[1] += nbad;
        done = ctx->h_small[0] == 0;
    }
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[1], s));
    if (done) {
        ctx->reuse_stats[2] += 1;
        return SCVT_OK;
    }
    CK(cudaMemsetAsync(ctx->d_status + 8, 0, 8 * sizeof(int), s));
    return build_cells_full(ctx, z, n, g, have_grid);
}

int cells_from_triangles(scvt_ctx* ctx, const int64_t* tri, int64_t t, int64_t n) {
    cudaStream_t s = ctx->stream;
    CK(cudaMemsetAsync(ctx->d_cursor, 0, n * sizeof(int), s));
    k_iota<<<blocks_for(n, 256), 256, 0, s>>>((int)n, ctx->d_ids);
    LAUNCHED();
    k_tl_fill<<<blocks_for(t, 256), 256, 0, s>>>(tri, t, ctx->d_cursor, ctx->d_pairs,
                                                 ctx->d_status);
    LAUNCHED();
    k_tl_chain<<<blocks_for(n, 256), 256, 0, s>>>((int)n, ctx->d_pairs, ctx->d_cursor,
                                                  ctx->d_nbr, ctx->d_deg, ctx->d_status);
    LAUNCHED();
    CK(cudaMemsetAsync(ctx->d_amb, 0, (size_t)n * MAXDEG, s));
    return SCVT_OK;
}

template <int KIND>
int launch_quad_kind(scvt_ctx* ctx, const QuadArgs& a, unsigned grid, size_t smem) {
    if (ctx->measure)
        k_quad<KIND, true, false><<<grid, QUAD_THREADS, smem, ctx->stream>>>(a);
    else if (ctx->sym7) {       // the fast path always runs a thread per fan sub-triangle
        // table kinds: rejected fits go to k_quad_table (see k_quad)
        constexpr bool DEFER = KIND == DEN_TANH4_TAB || KIND == DEN_TANH4X2_TAB;
        const unsigned g2 = blocks_for(2 * (int64_t)a.n_inc, QUAD_THREADS);
        if (DEFER) CK(cudaMemsetAsync(a.defer_cnt, 0, sizeof(int), ctx->stream));
        if (a.n_inc_dev)        // shards: incidence count on the device
            k_quad<KIND, false, true, true, true, DEFER><<<g2, QUAD_THREADS, 21 * sizeof(double),
                                                           ctx->stream>>>(a);
        else
            k_quad<KIND, false, true, true, false, DEFER><<<g2, QUAD_THREADS, 21 * sizeof(double),
                                                            ctx->stream>>>(a);
        if constexpr (DEFER) {
            LAUNCHED();
            // 16 queued sub-triangles per block and pass; the grid covers ~95k of them at once
            // (a c4 launch queues ~65k), longer queues take further grid-stride passes
            const unsigned gt = std::min<unsigned>(blocks_for(8 * (int64_t)a.n_inc, QTAB_THREADS),
                                                   148u * 40u);
            k_quad_table<KIND><<<gt, QTAB_THREADS, 0, ctx->stream>>>(a);
        }
    } else
        k_quad<KIND, false, false><<<grid, QUAD_THREADS, smem, ctx->stream>>>(a);
    LAUNCHED();
    return SCVT_OK;
}

// incidence CSR over the sorted slots [lo, hi) (spatially coherent warps)
int incidences_range(scvt_ctx* ctx, int64_t lo, int64_t hi, int64_t cap,
                     const int* skip = nullptr) {
    cudaStream_t s = ctx->stream;
    int64_t cnt = hi - lo;
    k_deg_sorted<<<blocks_for(cnt + 1, 256), 256, 0, s>>>((int)lo, (int)cnt, ctx->d_ids,
                                                          ctx->d_deg, ctx->d_cursor);
    LAUNCHED();
    size_t tb = ctx->cub_bytes;
    CK(cub::DeviceScan::ExclusiveSum(ctx->d_cub, tb, ctx->d_cursor, ctx->d_inc_start,
                                     (int)cnt + 1, s));
    k_fill_incidences<<<blocks_for(cnt, 256), 256, 0, s>>>((int)lo, (int)cnt, ctx->d_ids,
                                                           ctx->d_deg, ctx->d_inc_start,
                                                           ctx->d_inc_base, ctx->d_inc_gen,
                                                           (int)cap, skip, ctx->d_inc_start + cnt);
    LAUNCHED();
    return SCVT_OK;
}

// fan quadrature over n_inc incidences of the slots [lo, hi)
int quad_range(scvt_ctx* ctx, const double* z, int64_t n, int64_t lo, int64_t hi,
               int64_t n_inc, bool count_on_device = false) {
    QuadArgs a;
    a.z = z; a.nbr = ctx->d_nbr; a.deg = ctx->d_deg; a.inc_start = ctx->d_inc_start;
    a.inc_base = ctx->d_inc_base;
    a.inc_gen = ctx->d_inc_gen; a.n = (int)n; a.cnt = (int)(hi - lo); a.n_inc = (int)n_inc;
    a.n_inc_dev = count_on_device ? 1 : 0;
    a.nodes = ctx->d_nodes;
    a.nq = ctx->nq; a.dp = ctx->dp; a.part = ctx->d_part; a.obtuse = ctx->d_obt;
    a.table = ctx->d_table;
    a.dp.tab = ctx->d_table;
    a.dpg = ctx->d_dp;
    a.status = ctx->d_status;
    a.defer_list = ctx->d_defer;
    a.defer_cnt = ctx->d_defer + 2 * 6 * ctx->n_max;
    if (n_inc <= 0) return SCVT_OK;
    // split mode (thread per fan sub-triangle) on the 7-point fast path: twice the work units,
    // a finer last wave and shorter per-thread chains (c4 k_quad 9.44 -> 8.84 ms, c3 -11 %)
    ctx->split = 1;   // every path stores the two fan sub-triangles of an incidence separately
    unsigned grid = blocks_for(n_inc, QUAD_THREADS);
    size_t smem = 3 * (size_t)ctx->nq * sizeof(double);
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    switch (ctx->dp.kind) {
        case DEN_CONST: TRY(launch_quad_kind<DEN_CONST>(ctx, a, grid, smem)); break;
        case DEN_X3: TRY(launch_quad_kind<DEN_X3>(ctx, a, grid, smem)); break;
        case DEN_X16: TRY(launch_quad_kind<DEN_X16>(ctx, a, grid, smem)); break;
        case DEN_TANH: TRY(launch_quad_kind<DEN_TANH>(ctx, a, grid, smem)); break;
        case DEN_TANH4: TRY(launch_quad_kind<DEN_TANH4>(ctx, a, grid, smem)); break;
        case DEN_TANH4X2: TRY(launch_quad_kind<DEN_TANH4X2>(ctx, a, grid, smem)); break;
        case DEN_TANH4_TAB: TRY(launch_quad_kind<DEN_TANH4_TAB>(ctx, a, grid, smem)); break;
        case DEN_TANH4X2_TAB: TRY(launch_quad_kind<DEN_TANH4X2_TAB>(ctx, a, grid, smem)); break;
        default: return fail(ctx, SCVT_ERR_CONFIG, "bad density kind %d", ctx->dp.kind);
    }
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[3], ctx->stream));
    return SCVT_OK;
}

int pair_phase(scvt_ctx* ctx, const double* zo, const double* zn, const double* go,
               const double* gn, const Chunks& ck, double* red, int* nval);

// fixed-chunk reductions of E_i, |g_i|^2, obtuse_i over ALL n generators (id order), so the
// scalars are bitwise identical whatever the shard count; reads back and checks status
int reduce_finish(scvt_ctx* ctx, int64_t n, double* scalars_host, const double* diag,
                  const double* grad, const double* q3, const double* norms, int nsc,
                  int* deferred_nbad = nullptr, int pair_vals = 0) {
    cudaStream_t s = ctx->stream;
    Chunks ck;
    TRY(make_chunks(ctx, n, 0, 1, &ck));
    k_eval_reduce<<<ck.nc, RED_THREADS, 0, s>>>(ctx->d_egen, ctx->d_g2gen, ctx->d_obgen, diag,
                                                 grad, q3, norms, ck, ctx->d_partials);
    LAUNCHED();
    // values 0-4: the evaluation's scalars; 5 ..: the staged history pair's (max at 5 + 3)
    unsigned char ops[5 + 4 + 2 * MAXM] = {0, 0, 0, 2, 0};
    for (int v = 0; v < pair_vals; ++v) ops[5 + v] = v == 3 ? 1 : 0;
    TRY(reduce_chunks(ctx, ctx->d_partials, 5 + pair_vals, ops));
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[5], s));
    TRY(readback(ctx, 5 + pair_vals));
    if (deferred_nbad) {
        // the flip repair enqueued ahead of these moments: its statistics and bad count
        *deferred_nbad = flip_account(ctx, true);
        if (*deferred_nbad != 0) {     // not certified: the moments skipped themselves
            if (ctx->prof) {
                float a = 0.f;
                CK(cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]));
                ctx->prof_ms[0] += a;   // the resumed rebuild adds its share and the count
            }
            return SCVT_OK;
        }
        ctx->reuse_stats[0] += 1;
        ctx->reuse_stats[2] += 1;
    }
    if (ctx->prof) {
        float a = 0.f, b = 0.f, c = 0.f;
        CK(cudaEventElapsedTime(&b, ctx->ev[2], ctx->ev[3]));
        CK(cudaEventElapsedTime(&c, ctx->ev[4], ctx->ev[5]));
        if (ctx->prof_n[3] == 0) {   // cells pair recorded only on the scvt_evaluate path
            CK(cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]));
            ctx->prof_ms[0] += a; ++ctx->prof_n[0];
        }
        ctx->prof_ms[1] += b; ++ctx->prof_n[1];
        ctx->prof_ms[2] += c; ++ctx->prof_n[2];
    }
    int st = ctx->h_status[0];
    if (st) return status_to_code(ctx, st);
    scalars_host[0] = ctx->h_scal[0];
    scalars_host[1] = sqrt(ctx->h_scal[1]);
    scalars_host[2] = ctx->h_scal[2];
    if (nsc > 3) scalars_host[3] = ctx->h_scal[3];
    if (nsc > 4) scalars_host[4] = q3 ? ctx->h_scal[4] : 0.0;
    return SCVT_OK;
}

int moments(scvt_ctx* ctx, const double* z, int64_t n, double* grad, double* first,
            double* mass, double* diag, double* scalars_host, const double* q3 = nullptr,
            const double* norms = nullptr, int nsc = 3, int* deferred_nbad = nullptr,
            const double* pair_z_old = nullptr, const double* pair_g_old = nullptr) {
    int64_t n_inc = 6 * n - 12;   // Euler: a closed triangulation has exactly 6n-12 incidences
    TRY(incidences_range(ctx, 0, n, n_inc, deferred_nbad ? ctx->d_nbad : nullptr));
    TRY(quad_range(ctx, z, n, 0, n, n_inc));
    k_gather<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(
        z, (int)n, (int)n, ctx->d_inc_start, ctx->d_inc_base, ctx->d_deg, ctx->d_part,
        ctx->d_obt, n_inc, grad, first, mass, diag, ctx->d_egen, ctx->d_g2gen, ctx->d_obgen,
        ctx->split);
    LAUNCHED();
    int pair_vals = 0;
    ctx->staged_valid = false;
    if (pair_z_old && pair_g_old) {
        // the history pair this point would make if the line search accepts it (it usually
        // does): staged now so that its scalars ride on this evaluation's readback
        Chunks ck;
        TRY(make_chunks(ctx, n, 0, 1, &ck));
        TRY(pair_phase(ctx, pair_z_old, z, pair_g_old, grad, ck, ctx->d_partials + 5 * CHUNKS,
                       &pair_vals));
    }
    TRY(reduce_finish(ctx, n, scalars_host, diag, grad, q3, norms, nsc, deferred_nbad, pair_vals));
    if (pair_vals && !(deferred_nbad && *deferred_nbad != 0)) {
        for (int v = 0; v < pair_vals; ++v) ctx->staged_sc[v] = ctx->h_scal[5 + v];
        ctx->staged_valid = true;
        ctx->staged_z = z; ctx->staged_g = grad;
        ctx->staged_head = ctx->hist_head; ctx->staged_count = ctx->hist_count;
    }
    return SCVT_OK;
}

inline void shard_range(int64_t n, int shard, int nshards, int64_t* lo, int64_t* hi) {
    int64_t cap = (n + nshards - 1) / nshards;
    *lo = std::min<int64_t>(n, (int64_t)shard * cap);
    *hi = std::min<int64_t>(n, *lo + cap);
}

}  // namespace

namespace {

// ---------------------------------------------------------------------- Gram dispatch
HistPtrs hist_ptrs(scvt_ctx* ctx) {
    HistPtrs hp;
    const int64_t stride = 3 * ctx->n_max;
    for (int k = 0; k < MAXM; ++k) {
        const int slot = (ctx->hist_head + k) % ctx->m;
        hp.S[k] = k < ctx->hist_count ? ctx->d_S + slot * stride : nullptr;
        hp.Y[k] = k < ctx->hist_count ? ctx->d_Y + slot * stride : nullptr;
    }
    return hp;
}

#define SCVT_K_CASES(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) \
    X(13) X(14) X(15) X(16)

int launch_gram(scvt_ctx* ctx, int K, const double* g, const double* diag, double gamma,
                const HistPtrs& hp, const Chunks& ck, double* red) {
    switch (K) {
#define G(k) case k: k_gram<k><<<ck.nc, GRAM_THREADS, 0, ctx->stream>>>(g, diag, gamma, hp, ck, red); break;
        SCVT_K_CASES(G)
#undef G
        default: return fail(ctx, SCVT_ERR_CONFIG, "history length %d > %d", K, MAXM);
    }
    LAUNCHED();
    return SCVT_OK;
}

int launch_combine(scvt_ctx* ctx, int K, const double* g, const double* diag, double gamma,
                   const HistPtrs& hp, const double* z, const Chunks& ck, double* q3, double* red) {
    switch (K) {
#define C(k) case k: k_combine<k><<<ck.nc, RED_THREADS, 0, ctx->stream>>>(g, diag, gamma, hp, ctx->d_coef, z, ck, q3, red); break;
        SCVT_K_CASES(C)
#undef C
        default: return fail(ctx, SCVT_ERR_CONFIG, "history length %d > %d", K, MAXM);
    }
    LAUNCHED();
    return SCVT_OK;
}

inline int gram_values(int K) { return K ? 2 * K + K * (K + 1) / 2 + 1 : 0; }

// two-loop, phase 1: the Gram partials of the slice (nothing when the history is empty)
int gram_phase(scvt_ctx* ctx, const double* g, const double* diag, double gamma,
               const Chunks& ck, double* red) {
    const int K = ctx->hist_count;
    if (!K) return SCVT_OK;
    TRY(prep_red(ctx, red, gram_values(K), ck));
    return launch_gram(ctx, K, g, diag, gamma, hist_ptrs(ctx), ck, red);
}

// two-loop, phase 2: recursion on the (rank-summed) Gram partials, then the combine pass of the
// slice with the tangent projection; 2 values (q.g, g.q3) into red (may alias red_gram)
int combine_phase(scvt_ctx* ctx, const double* g, const double* diag, double gamma,
                  const double* z, const Chunks& ck, const double* red_gram, double* q3,
                  double* red) {
    const int K = ctx->hist_count;
    if (K) {
        GramScalars gs;
        for (int i = 0; i < K; ++i) {
            const int si = (ctx->hist_head + i) % ctx->m;
            gs.rho[i] = ctx->rho[si];
            for (int j = 0; j < K; ++j) gs.ys[i][j] = ctx->YS[si][(ctx->hist_head + j) % ctx->m];
        }
        k_gram_recursion<<<1, 1024, 0, ctx->stream>>>(red_gram, K, gs, ctx->d_coef);
        LAUNCHED();
    }
    TRY(prep_red(ctx, red, 2, ck));
    return launch_combine(ctx, K, g, diag, gamma, hist_ptrs(ctx), z, ck, q3, red);
}

// history push, phase 1: stage s, y of the slice; 4 + 2K values (y.s, s.s, y.y, max|s|, cross)
int pair_phase(scvt_ctx* ctx, const double* zo, const double* zn, const double* go,
               const double* gn, const Chunks& ck, double* red, int* nval) {
    const int K = ctx->hist_count;
    *nval = 4 + 2 * K;
    TRY(prep_red(ctx, red, *nval, ck));
    const HistPtrs hp = hist_ptrs(ctx);
    switch (K) {
#define P_(k) case k: k_history_pair<k><<<ck.nc, RED_THREADS, 0, ctx->stream>>>(zo, zn, go, gn, hp, ck, ctx->d_tmp_s, ctx->d_tmp_y, red); break;
        SCVT_K_CASES(P_)
#undef P_
        default: return fail(ctx, SCVT_ERR_CONFIG, "history length %d > %d", K, MAXM);
    }
    LAUNCHED();
    return SCVT_OK;
}

// history push, phase 2: fixed-order scalars, curvature test (optimizer.py:98-104), commit of
// the staged slice into the ring slot and of the cross products into the host y.s matrix
int commit_scalars(scvt_ctx* ctx, const double* sc, int64_t len, int32_t* pushed_host,
                   double* movement_host);

int commit_phase(scvt_ctx* ctx, const double* red, int64_t len, int32_t* pushed_host,
                 double* movement_host) {
    const int K = ctx->hist_count;
    unsigned char ops[4 + 2 * MAXM];
    for (int v = 0; v < 4 + 2 * K; ++v) ops[v] = v == 3 ? 1 : 0;
    TRY(reduce_chunks(ctx, red, 4 + 2 * K, ops));
    TRY(readback(ctx, 4 + 2 * K));
    return commit_scalars(ctx, ctx->h_scal, len, pushed_host, movement_host);
}

// the host half of a push: sc = {y.s, s.s, y.y, max|s|, y_new.s_k (K), y_k.s_new (K)} of the
// pair staged in d_tmp_s / d_tmp_y
int commit_scalars(scvt_ctx* ctx, const double* sc, int64_t len, int32_t* pushed_host,
                   double* movement_host) {
    const int K = ctx->hist_count;
    ctx->staged_valid = false;
    double ys = sc[0], ss = sc[1], yy = sc[2];
    *movement_host = sc[3];
    if (ys <= 1e-14 * sqrt(ss) * sqrt(yy)) {
        *pushed_host = 0;
        return SCVT_OK;
    }
    const int slot = (ctx->hist_head + ctx->hist_count) % ctx->m;
    CK(cudaMemcpyAsync(ctx->d_S + (int64_t)slot * 3 * ctx->n_max, ctx->d_tmp_s,
                       3 * len * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_Y + (int64_t)slot * 3 * ctx->n_max, ctx->d_tmp_y,
                       3 * len * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->launches += 2;
    ctx->rho[slot] = 1.0 / ys;
    ctx->ys[slot] = ys;
    ctx->yy[slot] = yy;
    for (int k = 0; k < K; ++k) {                 // cross products with the kept pairs
        const int sk = (ctx->hist_head + k) % ctx->m;
        if (sk == slot) continue;                 // the pair being overwritten
        ctx->YS[slot][sk] = sc[4 + k];       // y_new . s_k
        ctx->YS[sk][slot] = sc[4 + K + k];   // y_k . s_new
    }
    ctx->YS[slot][slot] = ys;
    if (ctx->hist_count < ctx->m) ++ctx->hist_count;
    else ctx->hist_head = (ctx->hist_head + 1) % ctx->m;
    *pushed_host = 1;
    return SCVT_OK;
}

// evaluation scalars of a slice: 5 values (E, |g|^2, obtuse, min diag, dirderiv) into red
int eval_scalars_phase(scvt_ctx* ctx, const Chunks& ck, const double* diag, const double* grad,
                       const double* q3, const double* norms, double* red) {
    TRY(prep_red(ctx, red, 5, ck));
    k_eval_reduce<<<ck.nc, RED_THREADS, 0, ctx->stream>>>(
        ctx->d_egen + ck.lo, ctx->d_g2gen + ck.lo, ctx->d_obgen + ck.lo, diag, grad, q3, norms,
        ck, red);
    LAUNCHED();
    return SCVT_OK;
}

}  // namespace

// Every entry point runs on the context's device and restores the caller's current device
// (a caller may have selected another GPU since scvt_create).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const scvt_ctx* ctx) {
        if (!ctx) return;
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != ctx->device &&
            cudaSetDevice(ctx->device) == cudaSuccess)
            prev = cur;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// ====================================================================== C ABI
extern "C" {

const char* scvt_version(void) { return "scvt_b200 0.1.0 (sm_100a)"; }

#ifdef SCVT_PROBE_FLIPS
// probe build only: {in-circle failures, orientation failures, consistency failures} of the
// reuse certificate passes since the last read
int scvt_probe_flips(unsigned long long* out3) {
    cudaMemcpyFromSymbol(out3, g_probe, 3 * sizeof(unsigned long long));
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_probe, z, sizeof(z));
    return 0;
}
#endif

const char* scvt_last_error(const scvt_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

int64_t scvt_launch_count(const scvt_ctx* ctx) { return ctx ? ctx->launches : 0; }

int scvt_profile_enable(scvt_ctx* ctx, int on) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (on && !ctx->ev[0])
        for (auto& e : ctx->ev) CK(cudaEventCreate(&e));
    ctx->prof = on != 0;
    return SCVT_OK;
}

int scvt_profile_counters(scvt_ctx* ctx, int64_t* out12, int reset) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    CK(cudaMemcpy(out12, ctx->d_diag, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    out12[8] = ctx->reuse_stats[2];   // evaluations whose cycles were certified by reuse
    out12[9] = ctx->reuse_stats[1];   // cells rebuilt by reuse rounds
    out12[10] = ctx->reuse_stats[0];  // certificate passes run by the reuse path
    unsigned long long mx[2];
    CK(cudaMemcpy(mx, ctx->d_diag + 8, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    out12[11] = (int64_t)mx[0] | ((int64_t)mx[1] << 40);   // max scanned | max passes << 40
    if (reset) {
        CK(cudaMemset(ctx->d_diag, 0, 10 * sizeof(int64_t)));
        ctx->reuse_stats[0] = ctx->reuse_stats[1] = ctx->reuse_stats[2] = 0;
    }
    return SCVT_OK;
}

int scvt_profile_flips(scvt_ctx* ctx, int64_t* out4, int reset) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    for (int k = 0; k < 4; ++k) {
        out4[k] = ctx->flip_stats[k];
        if (reset) ctx->flip_stats[k] = 0;
    }
    return SCVT_OK;
}

// the event pair of an asynchronous sharded k_quad launch (scvt_shard_moments_async), added
// to the profile once it has completed
static int flush_shard_quad(scvt_ctx* ctx) {
    if (!ctx->shard_quad_pending) return SCVT_OK;
    ctx->shard_quad_pending = false;
    if (!ctx->prof) return SCVT_OK;
    float ms = 0.f;
    CK(cudaEventSynchronize(ctx->ev[3]));
    CK(cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]));
    ctx->prof_ms[1] += ms;
    ++ctx->prof_n[1];
    return SCVT_OK;
}

int scvt_profile_read(scvt_ctx* ctx, double* ms_out, int64_t* counts_out, int reset) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    TRY(flush_shard_quad(ctx));
    for (int k = 0; k < 3; ++k) {
        ms_out[k] = ctx->prof_ms[k];
        counts_out[k] = ctx->prof_n[k];
        if (reset) { ctx->prof_ms[k] = 0.0; ctx->prof_n[k] = 0; }
    }
    return SCVT_OK;
}

int scvt_set_stream(scvt_ctx* ctx, void* stream) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    ctx->stream = (cudaStream_t)stream;
    return SCVT_OK;
}

int scvt_create(scvt_ctx** out, int device, int64_t n_max, const scvt_config* cfg) {
    if (!out || !cfg) return SCVT_ERR_CONFIG;
    *out = nullptr;
    struct RestoreDevice {
        int d = -1;
        ~RestoreDevice() {
            if (d >= 0) cudaSetDevice(d);
        }
    } restore_;
    if (cudaGetDevice(&restore_.d) != cudaSuccess) restore_.d = -1;
    scvt_ctx* ctx = new scvt_ctx();
    ctx->device = device;
    ctx->n_max = n_max;
    auto bail = [&](int code) { *out = ctx; return code; };
    if (n_max < 4 || n_max > (int64_t)1 << 28)
        return bail(fail(ctx, SCVT_ERR_CONFIG, "n_max=%lld out of range", (long long)n_max));
    if (cfg->n_nodes < 1 || cfg->n_nodes > SCVT_MAX_NODES || !cfg->node_l1 || !cfg->node_l2 ||
        !cfg->node_w)
        return bail(fail(ctx, SCVT_ERR_CONFIG, "bad node table (n_nodes=%d)", cfg->n_nodes));
    if (cfg->density_kind < 0 || cfg->density_kind > 5)
        return bail(fail(ctx, SCVT_ERR_CONFIG, "bad density kind %d", cfg->density_kind));
    if (cfg->lbfgs_m < 1 || cfg->lbfgs_m > MAXM)
        return bail(fail(ctx, SCVT_ERR_CONFIG, "lbfgs_m=%d out of range", cfg->lbfgs_m));
    {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess)
            return bail(fail(ctx, SCVT_ERR_CUDA, "cudaSetDevice(%d): %s", device,
                             cudaGetErrorString(e)));
    }
    {
        // the exact predicate's expansion buffers give the triangulation kernels a ~3 KB
        // stack frame; reserve it once (otherwise the driver grows and shrinks the local
        // memory pool around every launch that needs it)
        size_t stack = 0;
        if (cudaDeviceGetLimit(&stack, cudaLimitStackSize) == cudaSuccess && stack < 4096)
            cudaDeviceSetLimit(cudaLimitStackSize, 4096);
        cudaGetLastError();
    }
    DensityParams& dp = ctx->dp;
    dp.kind = cfg->density_kind;
    dp.gamma = cfg->gamma; dp.beta = cfg->beta; dp.alpha = cfg->alpha;
    dp.c0x = cfg->center[0]; dp.c0y = cfg->center[1]; dp.c0z = cfg->center[2];
    dp.c1x = cfg->center[3]; dp.c1y = cfg->center[4]; dp.c1z = cfg->center[5];
    dp.w_lon = cfg->w_lon; dp.w_lat = cfg->w_lat;
    if (dp.kind == DEN_X16) {
        double horiz = hypot(dp.c0x, dp.c0y);
        if (horiz < 1e-9)
            return bail(fail(ctx, SCVT_ERR_POLE_AMBIGUITY, "x16 centre at a pole"));
        dp.lat_c = atan2(dp.c0z, horiz);
        dp.lon_c = atan2(dp.c0y, dp.c0x);
        dp.cos_lat_c = cos(dp.lat_c);
        dp.sin_lat_c = sin(dp.lat_c);
    }
    dp.tab = nullptr;
    dp.tab_k = 0;
    dp.tab_invw = 0.0;
    if (cfg->table_coef && (dp.kind == DEN_TANH4 || dp.kind == DEN_TANH4X2)) {
        if (cfg->table_degree != TAB_P || cfg->table_intervals < 1 || cfg->table_intervals > 1024 ||
            !(cfg->table_width > 0.0))
            return bail(fail(ctx, SCVT_ERR_CONFIG, "bad density table (degree %d, intervals %d)",
                             cfg->table_degree, cfg->table_intervals));
        dp.tab_k = cfg->table_intervals;
        dp.tab_invw = 1.0 / cfg->table_width;
        dp.kind = dp.kind == DEN_TANH4 ? DEN_TANH4_TAB : DEN_TANH4X2_TAB;
    }
    ctx->measure = cfg->measure;
    ctx->nq = cfg->n_nodes;
    ctx->m = cfg->lbfgs_m;
    int64_t n = n_max;
    int G = grid_for(n);
    ctx->g_max = G;
    int64_t nb = 6LL * G * G;
    int64_t n_inc = 6 * n;
    int r = SCVT_OK;
    // every per-context buffer is a 256-byte aligned range of ONE device allocation (and the
    // pinned readback words of one host allocation): the ~50 cudaMalloc + 5 cudaMallocHost
    // calls they replace cost 20 ms per context at N = 655,362
    struct Slot { void** p; size_t off; };
    std::vector<Slot> slots;
    size_t arena_bytes = 0;
    auto reserve = [&](void** p, size_t bytes) {
        slots.push_back({p, arena_bytes});
        arena_bytes += (std::max<size_t>(bytes, 1) + 255) & ~(size_t)255;
    };
#define AL(p, cnt) \
    reserve((void**)&ctx->p, (size_t)(cnt) * sizeof(*ctx->p))
    AL(d_nodes, 3 * ctx->nq);
    AL(d_table, 2 * (int64_t)dp.tab_k * (TAB_P + 1));
    AL(d_dp, 1);
    AL(d_keys, n); AL(d_skeys, n); AL(d_vals, n); AL(d_ids, n);
    AL(d_start, nb + 1);
    AL(d_zs, 4 * n);
    AL(d_nbr, n * MAXDEG); AL(d_deg, n + 1); AL(d_amb, n * MAXDEG);
    AL(d_inc_start, n + 1); AL(d_inc_gen, n_inc); AL(d_inc_base, n);
    AL(d_pairs, n * MAXDEG * 2); AL(d_cursor, n + 1);
    AL(d_part, PART_ROW * n_inc); AL(d_obt, n_inc); AL(d_defer, 2 * n_inc + 1);   // [n_inc][2][5]: split mode uses both halves
    AL(d_egen, n); AL(d_g2gen, n); AL(d_obgen, n);
    AL(d_partials, std::max<int64_t>((int64_t)MAX_SLOTS * RED_BLOCKS, (int64_t)MAX_RED_VALS * CHUNKS));
    AL(d_scal, MAX_RED_VALS);
    AL(d_status, 64);
    AL(d_diag, 10);
    AL(d_bad, n); AL(d_slotflag, n); AL(d_list, n); AL(d_recheck, n); AL(d_nlist, 1);
    AL(d_list2, n); AL(d_nlist2, 1); AL(d_cnt, 1); AL(d_rcount, 4); AL(d_queue, 1); AL(d_mig, 1); AL(d_cand, 2 * n); AL(d_lock, n); AL(d_flist, 8 * n); AL(d_fflag, n); AL(d_counts, MAX_SHARDS + 1);
    AL(d_S, (int64_t)ctx->m * 3 * n); AL(d_Y, (int64_t)ctx->m * 3 * n);
    AL(d_alpha, ctx->m);
    AL(d_tmp_s, 3 * n); AL(d_tmp_y, 3 * n);
    AL(d_coef, 2 * MAXM);
#undef AL
    // CUB temp storage: max of radix sort (n), scan (n+1) and flagged select (the size queries
    // look at the argument types only)
    {
        size_t b1 = 0, b2 = 0, b3 = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, b1, ctx->d_keys, ctx->d_skeys, ctx->d_vals,
                                        ctx->d_ids, (int)n, 0, 32);
        cub::DeviceScan::ExclusiveSum(nullptr, b2, ctx->d_deg, ctx->d_inc_start, (int)n + 1);
        thrust::counting_iterator<int> it(0);
        cub::DeviceSelect::Flagged(nullptr, b3, it, ctx->d_slotflag, ctx->d_list, ctx->d_nbad,
                                   (int)n);
        ctx->cub_bytes = std::max(std::max(b1, b2), b3);
        reserve(&ctx->d_cub, ctx->cub_bytes);
    }
    if ((r = dalloc(ctx, &ctx->arena, arena_bytes))) return bail(r);
    for (const Slot& sl : slots) *sl.p = ctx->arena + sl.off;
    ctx->d_nbad = ctx->d_status + 16;
    ctx->d_fcnt = ctx->d_status + 24;
    ctx->d_fhist = ctx->d_status + 32;
    if (cudaMemset(ctx->d_status, 0, 64 * sizeof(int)) != cudaSuccess ||
        cudaMemset(ctx->d_lock, 0xFF, (size_t)n * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(ctx->d_fflag, 0, (size_t)n * sizeof(int)) != cudaSuccess)
        return bail(fail(ctx, SCVT_ERR_CUDA, "flip buffers init failed"));
    {
        // pinned readback words: h_scal [MAX_RED_VALS] doubles, h_dir [2] doubles, h_status
        // [64], h_small [32], h_counts [MAX_SHARDS + 1] ints
        size_t nd = MAX_RED_VALS + 2, ni = 64 + 32 + MAX_SHARDS + 1;
        cudaError_t e1 = cudaMallocHost((void**)&ctx->h_arena, nd * sizeof(double) + ni * sizeof(int));
        cudaError_t e2 = cudaEventCreateWithFlags(&ctx->dir_ev, cudaEventDisableTiming);
        if (e1 != cudaSuccess || e2 != cudaSuccess)
            return bail(fail(ctx, SCVT_ERR_CUDA, "cudaMallocHost failed"));
        ctx->h_scal = (double*)ctx->h_arena;
        ctx->h_dir = ctx->h_scal + MAX_RED_VALS;
        ctx->h_status = (int*)(ctx->h_dir + 2);
        ctx->h_small = ctx->h_status + 64;
        ctx->h_counts = ctx->h_small + 32;
    }
    // node table
    std::vector<double> tbl(3 * (size_t)ctx->nq);
    for (int q = 0; q < ctx->nq; ++q) {
        tbl[q] = cfg->node_l1[q];
        tbl[ctx->nq + q] = cfg->node_l2[q];
        tbl[2 * ctx->nq + q] = cfg->node_w[q];
    }
    ctx->sym7 = getenv("SCVT_NO_SYM7") == nullptr && is_sym7_depth3(cfg);
    {
        cudaError_t e = cudaMemcpy(ctx->d_nodes, tbl.data(), tbl.size() * sizeof(double),
                                   cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return bail(fail(ctx, SCVT_ERR_CUDA, "node upload failed"));
    }
    if (dp.tab_k) {
        cudaError_t e = cudaMemcpy(ctx->d_table, cfg->table_coef,
                                   2 * (size_t)dp.tab_k * (TAB_P + 1) * sizeof(double),
                                   cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return bail(fail(ctx, SCVT_ERR_CUDA, "table upload failed"));
    }
    size_t smem = 3 * (size_t)ctx->nq * sizeof(double);   // composite node table (quad_range)
    {
        // the split fast path adds its static per-thread fit slots (up to ~40 KB) to the
        // node table: opt in so that static + dynamic may exceed 48 KB
#define OPT7(K, D) \
    cudaFuncSetAttribute(k_quad<K, false, true, true, false, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    cudaFuncSetAttribute(k_quad<K, false, true, true, true, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
        OPT7(DEN_CONST, false); OPT7(DEN_X3, false); OPT7(DEN_X16, false); OPT7(DEN_TANH, false);
        OPT7(DEN_TANH4, false); OPT7(DEN_TANH4X2, false); OPT7(DEN_TANH4_TAB, true);
        OPT7(DEN_TANH4X2_TAB, true);
#undef OPT7
    }
    DensityParams dpd = dp;          // device copy read by the out-of-line quadrature paths
    dpd.tab = ctx->d_table;
    {
        cudaError_t e = cudaMemcpy(ctx->d_dp, &dpd, sizeof(dpd), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return bail(fail(ctx, SCVT_ERR_CUDA, "density upload failed"));
    }
    if (smem > 48 * 1024) {
        // opt in to large dynamic shared memory for every instantiation
#define OPT(K)                                                                             \
    cudaFuncSetAttribute(k_quad<K, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    cudaFuncSetAttribute(k_quad<K, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    cudaFuncSetAttribute(k_quad<K, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
        OPT(DEN_CONST); OPT(DEN_X3); OPT(DEN_X16); OPT(DEN_TANH); OPT(DEN_TANH4); OPT(DEN_TANH4X2);
        OPT(DEN_TANH4_TAB); OPT(DEN_TANH4X2_TAB);
#undef OPT
    }
    if (const char* e = getenv("SCVT_TAIL_ENTER")) ctx->tail_enter = std::max(0, atoi(e));
    if (const char* e = getenv("SCVT_TAIL_ROUNDS")) ctx->tail_rounds = std::max(0, atoi(e));
    if (const char* e = getenv("SCVT_FLIP_CAP")) ctx->flip_cap = std::max(0, atoi(e));
    ctx->rho.assign(ctx->m, 0.0);
    ctx->ys.assign(ctx->m, 0.0);
    ctx->yy.assign(ctx->m, 0.0);
    *out = ctx;
    return SCVT_OK;
}

int scvt_destroy(scvt_ctx* ctx) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_OK;
    void* dev[] = {ctx->arena, ctx->d_wdir, ctx->d_cgv, ctx->d_cg};   // arena + the lazy ones
    for (void* p : dev)
        if (p) cudaFree(p);
    for (cudaEvent_t e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->h_arena) cudaFreeHost(ctx->h_arena);
    if (ctx->dir_ev) cudaEventDestroy(ctx->dir_ev);
    delete ctx;
    return SCVT_OK;
}

int scvt_triangulate(scvt_ctx* ctx, const double* z, int64_t n, int64_t* tri_out,
                     uint8_t* flags_out, int64_t* stats_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    TRY(reset_status(ctx));
    ctx->cycles_n = -1;
    TRY(build_cells(ctx, z, n));
    cudaStream_t s = ctx->stream;
    // canonical triangles: count per min-id generator, scan, emit sorted
    k_tri_count<<<blocks_for(n + 1, 256), 256, 0, s>>>((int)n, ctx->d_nbr, ctx->d_deg,
                                                       ctx->d_cursor);
    LAUNCHED();
    // counts live in d_cursor[0..n] (n+1 entries incl. trailing 0); scan into inc_start
    size_t tb = ctx->cub_bytes;
    CK(cub::DeviceScan::ExclusiveSum(ctx->d_cub, tb, ctx->d_cursor, ctx->d_inc_start,
                                     (int)n + 1, s));
    k_tri_emit<<<blocks_for(n, 128), 128, 0, s>>>((int)n, ctx->d_nbr, ctx->d_deg, ctx->d_amb,
                                                  ctx->d_inc_start, 2 * n - 4, tri_out, flags_out);
    LAUNCHED();
    int total = 0;
    CK(cudaMemcpyAsync(&total, ctx->d_inc_start + n, sizeof(int), cudaMemcpyDeviceToHost, s));
    TRY(readback(ctx, 0));
    int st = ctx->h_status[0];
    if (stats_host) {
        stats_host[0] = total;
        stats_host[1] = 0;                  // flagged triangles, filled below
        stats_host[2] = ctx->h_status[8];   // max valence
        stats_host[3] = ctx->h_status[11];  // ambiguous (filter-undecided) directed edges
        stats_host[4] = ctx->h_status[12];  // SoS tie-breaks taken while clipping
        stats_host[5] = ctx->h_status[10];  // max candidate passes of one cell
        stats_host[6] = ctx->h_status[14];  // cells that needed the unsorted sweep
        stats_host[7] = ctx->h_status[15];  // 32-point batches visited by those sweeps
    }
    if (st) return status_to_code(ctx, st);
    if (total != 2 * n - 4)
        return fail(ctx, SCVT_ERR_COVERAGE, "triangulation not closed: K=%lld, T=%d (want %lld)",
                    (long long)n, total, (long long)(2 * n - 4));
    ctx->cycles_n = n;
    if (stats_host && flags_out) {
        // flagged triangle count
        std::vector<uint8_t> f((size_t)total);
        CK(cudaMemcpy(f.data(), flags_out, f.size(), cudaMemcpyDeviceToHost));
        int64_t c = 0;
        for (uint8_t v : f) c += v != 0;
        stats_host[1] = c;
    }
    return SCVT_OK;
}

int scvt_evaluate(scvt_ctx* ctx, const double* z, int64_t n, double* grad, double* first,
                  double* mass, double* lloyd_diag, double* scalars_host) {
    DeviceGuard dg_(ctx);
    double sc[5];
    int rc = scvt_evaluate_ex(ctx, z, n, grad, first, mass, lloyd_diag, nullptr, nullptr, sc);
    if (rc == SCVT_OK)
        for (int k = 0; k < 3; ++k) scalars_host[k] = sc[k];
    return rc;
}

static int evaluate_impl(scvt_ctx* ctx, const double* z, int64_t n, double* grad, double* first,
                         double* mass, double* lloyd_diag, const double* q3, const double* norms,
                         const double* z_old, const double* g_old, double* scalars_host) {
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[4], ctx->stream));
    ctx->prof_n[3] = 0;
    TRY(reset_status(ctx));
    const int nsc = q3 ? 5 : (norms ? 4 : 3);
    bool deferred = false;
    int nbad = 0;
    int rc = build_cells(ctx, z, n, &deferred);
    if (rc == SCVT_OK)
        rc = moments(ctx, z, n, grad, first, mass, lloyd_diag, scalars_host, q3, norms,
                     q3 ? 5 : 4, deferred ? &nbad : nullptr, z_old, g_old);
    if (rc == SCVT_OK && deferred && nbad != 0) {
        // the flips left bad cells: rebuild them (host-driven rounds), then the moments again
        rc = reset_status(ctx);
        if (rc == SCVT_OK) rc = build_cells_resume(ctx, z, n, nbad);
        if (rc == SCVT_OK)
            rc = moments(ctx, z, n, grad, first, mass, lloyd_diag, scalars_host, q3, norms,
                         q3 ? 5 : 4, nullptr, z_old, g_old);
    }
    (void)nsc;
    ctx->cycles_n = rc == SCVT_OK ? n : -1;   // certified cycles may seed the next evaluation
    return rc;
}

int scvt_evaluate_ex(scvt_ctx* ctx, const double* z, int64_t n, double* grad, double* first,
                     double* mass, double* lloyd_diag, const double* q3, const double* norms,
                     double* scalars_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    return evaluate_impl(ctx, z, n, grad, first, mass, lloyd_diag, q3, norms, nullptr, nullptr,
                         scalars_host);
}

// scvt_evaluate_ex that also stages the LBFGS pair (z - z_old, grad - g_old) this point would
// push if the line search accepts it; scvt_history_commit_staged then commits it without a
// kernel pass or a host round trip (the pair's scalars came back with the evaluation's).
int scvt_evaluate_staged(scvt_ctx* ctx, const double* z, int64_t n, double* grad, double* first,
                         double* mass, double* lloyd_diag, const double* q3, const double* norms,
                         const double* z_old, const double* g_old, double* scalars_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    return evaluate_impl(ctx, z, n, grad, first, mass, lloyd_diag, q3, norms, z_old, g_old,
                         scalars_host);
}

int scvt_history_commit_staged(scvt_ctx* ctx, const double* z_new, const double* g_new,
                               int64_t n, int32_t* pushed_host, double* movement_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (!ctx->staged_valid || ctx->staged_z != z_new || ctx->staged_g != g_new ||
        ctx->staged_head != ctx->hist_head || ctx->staged_count != ctx->hist_count)
        return fail(ctx, SCVT_ERR_CONFIG, "no staged history pair for this point");
    return commit_scalars(ctx, ctx->staged_sc, n, pushed_host, movement_host);
}

int scvt_evaluate_on_triangles(scvt_ctx* ctx, const double* z, int64_t n, const int64_t* tri,
                               int64_t t, double* grad, double* first, double* mass,
                               double* lloyd_diag, double* scalars_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (n > ctx->n_max) return fail(ctx, SCVT_ERR_CAPACITY, "n > n_max");
    if (t != 2 * n - 4) return fail(ctx, SCVT_ERR_COVERAGE, "T=%lld != 2n-4", (long long)t);
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[4], ctx->stream));
    ctx->prof_n[3] = 1;   // no cell-construction pair on this path
    ctx->cycles_n = -1;
    TRY(reset_status(ctx));
    TRY(cells_from_triangles(ctx, tri, t, n));
    return moments(ctx, z, n, grad, first, mass, lloyd_diag, scalars_host);
}

// ---------------------------------------------------------------------- sharded evaluation
int64_t scvt_shard_rows(int64_t n, int nshards) {
    return nshards > 0 ? (n + nshards - 1) / nshards : 0;
}

int scvt_cell_energy(scvt_ctx* ctx, int64_t n, double* energy_out) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (n < 1 || n > ctx->n_max || !energy_out)
        return fail(ctx, SCVT_ERR_CONFIG, "cell energy: n=%lld", (long long)n);
    CK(cudaMemcpyAsync(energy_out, ctx->d_egen, n * sizeof(double), cudaMemcpyDeviceToDevice,
                       ctx->stream));
    return SCVT_OK;
}

int scvt_shard_cells(scvt_ctx* ctx, const double* z, int64_t n, int shard, int nshards,
                     int32_t* cyc_send) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (nshards < 1 || shard < 0 || shard >= nshards)
        return fail(ctx, SCVT_ERR_CONFIG, "bad shard %d of %d", shard, nshards);
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[4], ctx->stream));
    ctx->prof_n[3] = 0;
    ctx->cycles_n = -1;
    TRY(reset_status(ctx));
    GridView g;
    TRY(build_grid(ctx, z, n, &g));
    int64_t lo, hi, cap = scvt_shard_rows(n, nshards);
    shard_range(n, shard, nshards, &lo, &hi);
    TRY(build_cells_range(ctx, g, lo, hi));
    k_pack_cycles<<<blocks_for(cap, 128), 128, 0, ctx->stream>>>(
        ctx->d_ids, (int)lo, (int)(hi - lo), (int)cap, ctx->d_nbr, ctx->d_deg, cyc_send);
    LAUNCHED();
    return SCVT_OK;
}

// ---- sharded cycle reuse: the single-GPU reuse loop split at its two exchanges
int scvt_shard_flip(scvt_ctx* ctx, const double* z, int64_t n, int32_t* nbad_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    *nbad_host = -1;
    if (ctx->cycles_n != n || !reuse_enabled() || !flips_enabled()) return SCVT_OK;
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[4], ctx->stream));
    ctx->prof_n[3] = 0;
    TRY(reset_status(ctx));
    CK(cudaMemsetAsync(ctx->d_bad, 0, n * sizeof(int), ctx->stream));
    CK(cudaMemsetAsync(ctx->d_nbad, 0, sizeof(int), ctx->stream));
    int nbad = 0;
    TRY(flip_repair(ctx, z, n, &nbad));
    if (nbad == 0) ctx->reuse_stats[2] += 1;   // certified: the evaluation reuses all cycles
    *nbad_host = nbad;
    return SCVT_OK;
}

int scvt_shard_flip_detect(scvt_ctx* ctx, const double* z, int64_t n, int shard, int nshards,
                           int32_t* cand_send, int64_t cap, int32_t* counts_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (nshards < 1 || shard < 0 || shard >= nshards)
        return fail(ctx, SCVT_ERR_CONFIG, "bad shard %d of %d", shard, nshards);
    counts_host[0] = -1;
    counts_host[1] = 0;
    if (ctx->cycles_n != n || !reuse_enabled() || !flips_enabled()) return SCVT_OK;
    cudaStream_t s = ctx->stream;
    if (ctx->prof) CK(cudaEventRecord(ctx->ev[4], s));
    ctx->prof_n[3] = 0;
    TRY(reset_status(ctx));
    CK(cudaMemsetAsync(ctx->d_bad, 0, n * sizeof(int), s));
    CK(cudaMemsetAsync(ctx->d_nbad, 0, sizeof(int), s));
    int64_t lo, hi;
    shard_range(n, shard, nshards, &lo, &hi);
    TRY(flip_detect(ctx, z, n, lo, hi));
    CK(cudaMemcpyAsync(ctx->h_small, ctx->d_fcnt, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctx->h_small + 4, ctx->d_nbad, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int nc = ctx->h_small[0];
    if (nc > 0 && nc <= cap)
        CK(cudaMemcpyAsync(cand_send, ctx->d_cand, (size_t)nc * sizeof(int4),
                           cudaMemcpyDeviceToDevice, s));
    counts_host[0] = nc;                       // > cap: the caller takes the rebuild rounds
    counts_host[1] = ctx->h_small[4];
    return SCVT_OK;
}

int scvt_shard_flip_rounds(scvt_ctx* ctx, const double* z, int64_t n, int nshards,
                           const int32_t* cand_all, int64_t cap, const int64_t* counts,
                           int32_t* nbad_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    cudaStream_t s = ctx->stream;
    int64_t total = 0;
    for (int r = 0; r < nshards; ++r) {        // validate before any copy into d_cand
        if (counts[r] < 0 || counts[r] > cap)
            return fail(ctx, SCVT_ERR_CONFIG, "shard %d: %lld flip candidates > cap %lld", r,
                        (long long)counts[r], (long long)cap);
        total += counts[r];
    }
    if (total > (ctx->flip_cap > 0 ? std::min<int64_t>(ctx->flip_cap, n) : n)) {
        // more than the queue holds: the caller takes the rebuild rounds
        *nbad_host = (int32_t)std::min<int64_t>(total, INT32_MAX);
        return SCVT_OK;
    }
    total = 0;
    for (int r = 0; r < nshards; ++r) {        // the shards' candidates, in rank order
        if (counts[r] > 0)
            CK(cudaMemcpyAsync(ctx->d_cand + total, cand_all + 4 * (int64_t)r * cap,
                               (size_t)counts[r] * sizeof(int4), cudaMemcpyDeviceToDevice, s));
        total += counts[r];
    }
    ctx->h_small[8] = (int)total;
    CK(cudaMemsetAsync(ctx->d_fcnt, 0, (8 + FLIP_HIST) * sizeof(int), s));
    CK(cudaMemcpyAsync(ctx->d_fcnt, ctx->h_small + 8, sizeof(int), cudaMemcpyHostToDevice, s));
    int nbad = 0;
    TRY(flip_rounds_enqueue(ctx, z, n));
    TRY(readback(ctx, 0));
    nbad = flip_account(ctx);
    if (nbad == 0) ctx->reuse_stats[2] += 1;   // certified: the evaluation reuses all cycles
    *nbad_host = nbad;
    return SCVT_OK;
}

int scvt_shard_recheck(scvt_ctx* ctx, const double* z, int64_t n, int shard, int nshards,
                       int round, int32_t* bad_out, int32_t* ready_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (nshards < 1 || shard < 0 || shard >= nshards)
        return fail(ctx, SCVT_ERR_CONFIG, "bad shard %d of %d", shard, nshards);
    cudaStream_t s = ctx->stream;
    *ready_host = 0;
    if (round == 0) {
        if (ctx->cycles_n != n || !reuse_enabled()) return SCVT_OK;   // caller: full path
        if (ctx->prof) CK(cudaEventRecord(ctx->ev[4], s));
        ctx->prof_n[3] = 0;
        TRY(reset_status(ctx));
        GridView g;
        TRY(build_grid(ctx, z, n, &g));
    }
    int64_t lo, hi;
    shard_range(n, shard, nshards, &lo, &hi);
    CK(cudaMemsetAsync(ctx->d_bad, 0, n * sizeof(int), s));
    CK(cudaMemsetAsync(ctx->d_nbad, 0, sizeof(int), s));
    if (round == 0) {
        TRY(verify_range(ctx, z, lo, hi, 1));
    } else {                    // the plan's re-check list; its length stays on the device
        k_verify<<<SPEC_BLOCKS, 128, 0, s>>>(
            z, ctx->d_ids, (int)lo, (int)hi, ctx->d_list2, ctx->d_nlist2, ctx->d_nbr,
            ctx->d_deg, ctx->d_amb, ctx->d_status, ctx->d_status + 8, 1, ctx->d_bad,
            ctx->d_nbad);
        LAUNCHED();
    }
    CK(cudaMemcpyAsync(bad_out, ctx->d_bad, n * sizeof(int), cudaMemcpyDeviceToDevice, s));
    *ready_host = 1;
    return SCVT_OK;
}

int scvt_shard_plan(scvt_ctx* ctx, int64_t n, int nshards, const int32_t* bad_all,
                    int64_t* counts_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (nshards < 1 || nshards > MAX_SHARDS)
        return fail(ctx, SCVT_ERR_CONFIG, "bad shard count %d (max %d)", nshards, MAX_SHARDS);
    cudaStream_t s = ctx->stream;
    CK(cudaMemcpyAsync(ctx->d_bad, bad_all, n * sizeof(int), cudaMemcpyDeviceToDevice, s));
    TRY(compact_slots(ctx, n, ctx->d_bad, ctx->d_nbad));       // bad slots, ascending
    // re-check set of the next round (bad cells and their current neighbours) -> d_list2
    CK(cudaMemsetAsync(ctx->d_recheck, 0, n * sizeof(int), s));
    k_mark_recheck<<<SPEC_BLOCKS, 256, 0, s>>>(ctx->d_list, ctx->d_nbad, ctx->d_ids, ctx->d_nbr,
                                                ctx->d_deg, ctx->d_recheck);
    LAUNCHED();
    k_flag_slots<<<blocks_for(n, 256), 256, 0, s>>>((int)n, ctx->d_ids, ctx->d_recheck,
                                                    ctx->d_slotflag);
    LAUNCHED();
    size_t tb = ctx->cub_bytes;
    thrust::counting_iterator<int> it(0);
    CK(cub::DeviceSelect::Flagged(ctx->d_cub, tb, it, ctx->d_slotflag, ctx->d_list2,
                                  ctx->d_nlist2, (int)n, s));
    // bad cells per shard: boundaries of the ascending slot list, found on the device
    k_shard_counts<<<1, 256, 0, s>>>(ctx->d_list, ctx->d_nbad, nshards,
                                     scvt_shard_rows(n, nshards), ctx->d_counts);
    LAUNCHED();
    CK(cudaMemcpyAsync(ctx->h_counts, ctx->d_counts, (nshards + 1) * sizeof(int),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int nbad = ctx->h_counts[nshards];
    ctx->reuse_stats[0] += 1;
    ctx->reuse_stats[1] += nbad;
    if (nbad == 0) ctx->reuse_stats[2] += 1;   // certified: the evaluation reuses all cycles
    ctx->plan_counts.assign(ctx->h_counts, ctx->h_counts + nshards);
    for (int k = 0; k < nshards; ++k) counts_host[k] = ctx->h_counts[k];
    counts_host[nshards] = nbad;
    return SCVT_OK;
}

int scvt_shard_rebuild(scvt_ctx* ctx, int64_t n, int shard, int nshards, int64_t cap,
                       int32_t* rows_send) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if ((int)ctx->plan_counts.size() != nshards || shard < 0 || shard >= nshards)
        return fail(ctx, SCVT_ERR_CONFIG, "scvt_shard_rebuild without a matching plan");
    cudaStream_t s = ctx->stream;
    int64_t off = 0;
    for (int k = 0; k < shard; ++k) off += ctx->plan_counts[k];
    const int cnt = (int)ctx->plan_counts[shard];
    if (cap < cnt) return fail(ctx, SCVT_ERR_CONFIG, "cap %lld < %d rebuilt cells",
                               (long long)cap, cnt);
    k_set_int<<<1, 1, 0, s>>>(ctx->d_cnt, cnt);
    LAUNCHED();
    const int* list = ctx->d_list + off;
    if (cnt > 0) {
        k_cells_warp<<<blocks_for(cnt, CELL_WARPS), CELL_WARPS * 32, 0, s>>>(
            ctx->gv, 0, (int)n, list, ctx->d_cnt, ctx->d_nbr, ctx->d_deg, ctx->d_status,
            ctx->d_status + 8, ctx->prof ? ctx->d_diag : nullptr);
        LAUNCHED();
        k_cells<<<blocks_for(cnt, CELL_THREADS), CELL_THREADS, 0, s>>>(
            ctx->gv, 0, (int)n, list, ctx->d_cnt, ctx->d_nbr, ctx->d_deg, ctx->d_status,
            ctx->d_status + 8);
        LAUNCHED();
    }
    if (cap > 0) {
        k_pack_list<<<blocks_for(cap, 128), 128, 0, s>>>(list, ctx->d_cnt, (int)cap, ctx->d_ids,
                                                          ctx->d_nbr, ctx->d_deg, rows_send);
        LAUNCHED();
    }
    return SCVT_OK;
}

int scvt_shard_install(scvt_ctx* ctx, int64_t n, const int32_t* rows, int64_t nrows) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (nrows <= 0) return SCVT_OK;
    k_unpack_cycles<<<blocks_for(nrows, 128), 128, 0, ctx->stream>>>(
        rows, (int)nrows, (int)n, ctx->d_nbr, ctx->d_deg, ctx->d_status + 13, ctx->d_status);
    LAUNCHED();
    return SCVT_OK;
}

int scvt_shard_moments(scvt_ctx* ctx, const double* z, int64_t n, int shard, int nshards,
                       const int32_t* cyc_all, double* res_send, int32_t* status_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    cudaStream_t s = ctx->stream;
    int64_t lo, hi, cap = scvt_shard_rows(n, nshards);
    shard_range(n, shard, nshards, &lo, &hi);
    // every rank gets every cycle: needed to certify its own cells against their neighbours
    // (cyc_all == NULL: the cycles were certified by the sharded reuse rounds)
    if (cyc_all) {
        CK(cudaMemsetAsync(ctx->d_status + 13, 0, sizeof(int), s));
        k_unpack_cycles<<<blocks_for(cap * nshards, 128), 128, 0, s>>>(
            cyc_all, (int)(cap * nshards), (int)n, ctx->d_nbr, ctx->d_deg, ctx->d_status + 13,
            ctx->d_status);
        LAUNCHED();
        TRY(verify_range(ctx, z, lo, hi));
    }
    TRY(incidences_range(ctx, lo, hi, 6 * n));
    int tot[2] = {0, (int)(6 * n - 12)};
    CK(cudaMemcpyAsync(&tot[0], ctx->d_inc_start + (hi - lo), sizeof(int), cudaMemcpyDeviceToHost, s));
    if (cyc_all)
        CK(cudaMemcpyAsync(&tot[1], ctx->d_status + 13, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (tot[1] != 6 * n - 12) {
        CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        *status_host = ctx->h_status[0] | ST_EULER;
        return SCVT_OK;
    }
    TRY(quad_range(ctx, z, n, lo, hi, tot[0]));
    k_gather_pack<<<blocks_for(cap, 128), 128, 0, s>>>(
        (int)lo, (int)(hi - lo), (int)cap, ctx->d_ids, ctx->d_inc_base, ctx->d_deg, ctx->d_part,
        ctx->d_obt, tot[0], res_send, ctx->split);
    LAUNCHED();
    CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *status_host = ctx->h_status[0];
    if (ctx->prof && tot[0] > 0) {   // this shard's k_quad launch (quad_range's event pair)
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]));
        ctx->prof_ms[1] += ms;
        ++ctx->prof_n[1];
    }
    return SCVT_OK;
}

// scvt_shard_moments for cycles the sharded reuse rounds certified (cyc_all == NULL), without
// a host read: k_quad takes the shard's incidence count from the device (its grid is sized
// for an upper bound) and the status word is copied to status_dev (device, 1 int32), which
// the caller all-gathers with the other ranks' anyway.
int scvt_shard_moments_async(scvt_ctx* ctx, const double* z, int64_t n, int shard, int nshards,
                             double* res_send, int32_t* status_dev) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (nshards < 1 || shard < 0 || shard >= nshards || !status_dev)
        return fail(ctx, SCVT_ERR_CONFIG, "bad shard %d of %d", shard, nshards);
    cudaStream_t s = ctx->stream;
    TRY(flush_shard_quad(ctx));
    int64_t lo, hi, cap = scvt_shard_rows(n, nshards);
    shard_range(n, shard, nshards, &lo, &hi);
    TRY(incidences_range(ctx, lo, hi, 6 * n));
    int64_t bound;
    if (ctx->sym7 && !ctx->measure) {
        // valence averages < 6 over any large range; a shard that exceeded the bound would set
        // ST_EULER (coverage error), never integrate a truncated range silently
        bound = std::min<int64_t>(6 * n, 8 * (hi - lo) + 4096);
        TRY(quad_range(ctx, z, n, lo, hi, bound, true));
    } else {        // generic quadrature kernels take the exact count: one host read
        int tot = 0;
        CK(cudaMemcpyAsync(&tot, ctx->d_inc_start + (hi - lo), sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        bound = tot;
        TRY(quad_range(ctx, z, n, lo, hi, bound));
    }
    k_gather_pack<<<blocks_for(cap, 128), 128, 0, s>>>(
        (int)lo, (int)(hi - lo), (int)cap, ctx->d_ids, ctx->d_inc_base, ctx->d_deg, ctx->d_part,
        ctx->d_obt, bound, res_send, ctx->split);
    LAUNCHED();
    CK(cudaMemcpyAsync(status_dev, ctx->d_status, sizeof(int), cudaMemcpyDeviceToDevice, s));
    ctx->shard_quad_pending = ctx->prof;   // its event pair is read once it has completed
    return SCVT_OK;
}

int scvt_shard_status(scvt_ctx* ctx, int32_t status) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    return status_to_code(ctx, status);
}

int scvt_shard_finish(scvt_ctx* ctx, const double* z, int64_t n, int nshards,
                      const double* res_all, double* grad, double* first, double* mass,
                      double* lloyd_diag, double* scalars_host) {
    DeviceGuard dg_(ctx);
    double sc[5];
    int rc = scvt_shard_finish_ex(ctx, z, n, nshards, res_all, grad, first, mass, lloyd_diag,
                                  nullptr, nullptr, sc);
    if (rc == SCVT_OK)
        for (int k = 0; k < 3; ++k) scalars_host[k] = sc[k];
    return rc;
}

int scvt_shard_finish_ex(scvt_ctx* ctx, const double* z, int64_t n, int nshards,
                         const double* res_all, double* grad, double* first, double* mass,
                         double* lloyd_diag, const double* q3, const double* norms,
                         double* scalars_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    cudaStream_t s = ctx->stream;
    int64_t cap = scvt_shard_rows(n, nshards);
    CK(cudaMemsetAsync(ctx->d_status + 13, 0, sizeof(int), s));
    k_unpack_results<<<blocks_for(cap * nshards, 128), 128, 0, s>>>(
        res_all, (int)(cap * nshards), (int)n, z, grad, first, mass, lloyd_diag, ctx->d_egen,
        ctx->d_g2gen, ctx->d_obgen, ctx->d_status + 13);
    LAUNCHED();
    TRY(reduce_finish(ctx, n, scalars_host, lloyd_diag, grad, q3, norms, q3 ? 5 : 4));
    int seen = 0;
    CK(cudaMemcpy(&seen, ctx->d_status + 13, sizeof(int), cudaMemcpyDeviceToHost));
    if (seen != n)
        return fail(ctx, SCVT_ERR_COVERAGE, "shard results cover %d of %lld generators", seen,
                    (long long)n);
    // every rank now holds all n certified cycles: the next evaluation may reuse them
    ctx->cycles_n = n;
    return SCVT_OK;
}

// ---------------------------------------------------------------------- arithmetic-layout slices
int scvt_slice_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi) {
    if (world < 1 || rank < 0 || rank >= world || SCVT_CHUNKS % world) return SCVT_ERR_CONFIG;
    const int64_t ch = std::max<int64_t>(1, (n + SCVT_CHUNKS - 1) / SCVT_CHUNKS);
    const int64_t nc = SCVT_CHUNKS / world;
    *lo = std::min<int64_t>(n, rank * nc * ch);
    *hi = std::min<int64_t>(n, (rank + 1) * nc * ch);
    return SCVT_OK;
}

int scvt_slice_finish(scvt_ctx* ctx, const double* z, int64_t n, int nshards,
                      const double* res_all, int rank, int world, double* grad, double* first,
                      double* mass, double* lloyd_diag, const double* q3, const double* norms,
                      double* red) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, rank, world, &ck));
    cudaStream_t s = ctx->stream;
    const int64_t rows = scvt_shard_rows(n, nshards) * nshards;
    if (ck.len)
        CK(cudaMemsetAsync(ctx->d_egen + ck.lo, 0xFF, ck.len * sizeof(double), s));   // NaN
    k_unpack_slice<<<blocks_for(rows, 128), 128, 0, s>>>(
        res_all, (int)rows, ck.lo, ck.lo + ck.len, z, grad, first, mass, lloyd_diag,
        ctx->d_egen, ctx->d_g2gen, ctx->d_obgen);
    LAUNCHED();
    TRY(eval_scalars_phase(ctx, ck, lloyd_diag, grad, q3, norms, red));
    ctx->cycles_n = n;   // every rank holds all n certified cycles: the next evaluation may reuse them
    return SCVT_OK;
}

int scvt_slice_scalars(scvt_ctx* ctx, const double* red, double* scalars_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    static const unsigned char ops[5] = {0, 0, 0, 2, 0};
    TRY(reduce_chunks(ctx, red, 5, ops));
    TRY(readback(ctx, 5));
    if (ctx->h_status[0]) return status_to_code(ctx, ctx->h_status[0]);
    if (std::isnan(ctx->h_scal[0]))
        return fail(ctx, SCVT_ERR_COVERAGE, "shard results do not cover every generator");
    scalars_host[0] = ctx->h_scal[0];
    scalars_host[1] = sqrt(ctx->h_scal[1]);
    scalars_host[2] = ctx->h_scal[2];
    scalars_host[3] = ctx->h_scal[3];
    scalars_host[4] = ctx->h_scal[4];
    return SCVT_OK;
}

int scvt_slice_gram(scvt_ctx* ctx, const double* g, const double* lloyd_diag, double gamma,
                    int64_t n, int rank, int world, double* red, int32_t* nval_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, rank, world, &ck));
    *nval_host = gram_values(ctx->hist_count);
    return gram_phase(ctx, g, lloyd_diag, gamma, ck, red);
}

int scvt_slice_combine(scvt_ctx* ctx, const double* g, const double* lloyd_diag, double gamma,
                       const double* z, int64_t n, int rank, int world, const double* red_gram,
                       double* q3, double* red) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, rank, world, &ck));
    return combine_phase(ctx, g, lloyd_diag, gamma, z, ck, red_gram, q3, red);
}

int scvt_slice_tangent(scvt_ctx* ctx, const double* q, const double* z, const double* g,
                       int64_t n, int rank, int world, double* q3, double* red) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, rank, world, &ck));
    TRY(prep_red(ctx, red, 1, ck));
    k_tangent<<<ck.nc, RED_THREADS, 0, ctx->stream>>>(q, z, g, ck, q3, red);
    LAUNCHED();
    return SCVT_OK;
}

int scvt_slice_history_pair(scvt_ctx* ctx, const double* z_old, const double* z_new,
                            const double* g_old, const double* g_new, int64_t n, int rank,
                            int world, double* red, int32_t* nval_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, rank, world, &ck));
    int nval = 0;
    TRY(pair_phase(ctx, z_old, z_new, g_old, g_new, ck, red, &nval));
    *nval_host = nval;
    return SCVT_OK;
}

int scvt_slice_history_commit(scvt_ctx* ctx, const double* red, int64_t n, int rank, int world,
                              int32_t* pushed_host, double* movement_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, rank, world, &ck));
    return commit_phase(ctx, red, ck.len, pushed_host, movement_host);
}

int scvt_reduce_chunks(scvt_ctx* ctx, const double* red, int32_t nval, const uint8_t* ops,
                       double* out_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    TRY(reduce_chunks(ctx, red, nval, ops));
    TRY(readback(ctx, nval));
    for (int v = 0; v < nval; ++v) out_host[v] = ctx->h_scal[v];
    return SCVT_OK;
}

int scvt_migration(scvt_ctx* ctx, const double* z, int64_t n, const double* centers, int32_t p,
                   const uint32_t* adjacency, int32_t* arithmetic, int32_t fresh,
                   int32_t* class_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (p < 1) return fail(ctx, SCVT_ERR_CONFIG, "covering with %d cells", p);
    cudaStream_t s = ctx->stream;
    CK(cudaMemsetAsync(ctx->d_mig, 0, sizeof(int), s));
    k_migration<<<blocks_for(n, 256), 256, 0, s>>>(z, n, centers, p, adjacency, (p + 31) / 32,
                                                    arithmetic, fresh, ctx->d_mig);
    LAUNCHED();
    CK(cudaMemcpyAsync(ctx->h_small, ctx->d_mig, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *class_host = ctx->h_small[0];
    return SCVT_OK;
}

int scvt_region_cover(scvt_ctx* ctx, const double* z, int64_t n, const double* centers,
                      int32_t p, const uint32_t* adjacency, double eps_proj, int32_t* fail_host,
                      int32_t* region_fail_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (p < 1 || p > MAX_SHARDS / 2)
        return fail(ctx, SCVT_ERR_CONFIG, "covering with %d cells (1..%d)", p, MAX_SHARDS / 2);
    if (ctx->cycles_n != n)
        return fail(ctx, SCVT_ERR_CONFIG, "scvt_region_cover needs the evaluation of these %lld points",
                    (long long)n);
    cudaStream_t s = ctx->stream;
    // geo cells in d_list (n ints); per-cell counts and per-region flags in d_counts
    int* geo = ctx->d_list;
    int* hist = ctx->d_counts;
    int* rfail = ctx->d_counts + p;
    CK(cudaMemsetAsync(hist, 0, 2 * (size_t)p * sizeof(int), s));
    k_geo_cells<<<blocks_for(n, 256), 256, 0, s>>>(z, n, centers, p, geo, hist);
    LAUNCHED();
    k_region_cover<<<blocks_for(n, 128), 128, 0, s>>>(z, n, ctx->d_nbr, ctx->d_deg, centers, p,
                                                     adjacency, geo, hist, eps_proj, rfail);
    LAUNCHED();
    CK(cudaMemcpyAsync(ctx->h_counts, hist, 2 * (size_t)p * sizeof(int), cudaMemcpyDeviceToHost, s));
    std::vector<uint32_t> adj((size_t)p * ((p + 31) / 32));
    CK(cudaMemcpyAsync(adj.data(), adjacency, adj.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int words = (p + 31) / 32;
    int f = 0;
    for (int l = 0; l < p; ++l) {
        int rf = ctx->h_counts[p + l];
        if (ctx->h_counts[l] > 0) {           // regions holding owned points: >= 3 members
            int64_t members = ctx->h_counts[l];
            for (int k = 0; k < p; ++k)
                if (k != l && ((adj[(size_t)l * words + (k >> 5)] >> (k & 31)) & 1u))
                    members += ctx->h_counts[k];
            if (members < 3) rf |= 4;
        } else {
            rf = 0;                            // no payload: the reference skips the region
        }
        if (region_fail_host) region_fail_host[l] = rf;
        f |= rf;
    }
    *fail_host = f;
    return SCVT_OK;
}

// ---------------------------------------------------------------------- graph Laplacian
int scvt_laplacian(scvt_ctx* ctx, int64_t n, double* wsym, double* diag, int32_t* nbr_out,
                   int32_t* deg_out) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (ctx->cycles_n != n)
        return fail(ctx, SCVT_ERR_CONFIG, "scvt_laplacian needs the evaluation of these %lld points",
                    (long long)n);
    if (!ctx->d_wdir) TRY(dalloc(ctx, &ctx->d_wdir, (size_t)ctx->n_max * MAXDEG));
    cudaStream_t s = ctx->stream;
    TRY(reset_status(ctx));
    k_lap_dir<<<blocks_for(n, 256), 256, 0, s>>>((int)n, ctx->d_inc_base, ctx->d_deg, ctx->d_part,
                                                  ctx->d_wdir);
    LAUNCHED();
    k_lap_sym<<<blocks_for(n, 256), 256, 0, s>>>((int)n, ctx->d_nbr, ctx->d_deg, ctx->d_wdir,
                                                  wsym, diag, ctx->d_status);
    LAUNCHED();
    // the matrix keeps its own copy of the sparsity (the context's cycles move on with the
    // next evaluation)
    CK(cudaMemcpyAsync(nbr_out, ctx->d_nbr, (size_t)n * MAXDEG * sizeof(int),
                       cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(deg_out, ctx->d_deg, (size_t)n * sizeof(int), cudaMemcpyDeviceToDevice, s));
    ctx->launches += 2;
    TRY(readback(ctx, 0));
    if (ctx->h_status[0]) return status_to_code(ctx, ctx->h_status[0]);
    return SCVT_OK;
}

int scvt_laplacian_solve(scvt_ctx* ctx, int64_t n, const int32_t* nbr, const int32_t* deg,
                         const double* wsym, const double* dpert, const double* b, double* x,
                         double tol, int32_t max_iter, int32_t* iters_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (n > ctx->n_max) return fail(ctx, SCVT_ERR_CAPACITY, "n > n_max");
    if (!ctx->d_cgv) TRY(dalloc(ctx, &ctx->d_cgv, (size_t)12 * ctx->n_max));
    if (!ctx->d_cg) TRY(dalloc(ctx, &ctx->d_cg, (size_t)16));
    cudaStream_t s = ctx->stream;
    const int64_t len = 3 * n;
    double* r = ctx->d_cgv;
    double* pv = r + 3 * ctx->n_max;
    double* qv = pv + 3 * ctx->n_max;
    double* zv = qv + 3 * ctx->n_max;
    Chunks ck;
    TRY(make_chunks(ctx, n, 0, 1, &ck));
    TRY(reset_status(ctx));
    CK(cudaMemsetAsync(x, 0, len * sizeof(double), s));
    ctx->launches += 1;
    // Jacobi-preconditioned CG: the x64 / x16 Laplacians have diagonals spanning ~1e7, which
    // unpreconditioned CG cannot resolve to 1e-14.  cg: [0..2] r.z, [3..5] p.Ap,
    // [6..8] new r.z, [9..11] new r.r, [12..14] b.b (per coordinate)
    RedOps ro;
    for (int v = 0; v < 6; ++v) ro.op[v] = 0;
    CK(cudaMemsetAsync(ctx->d_cg, 0, 16 * sizeof(double), s));
    k_cg_start<<<ck.nc, RED_THREADS, 0, s>>>(b, dpert, r, zv, pv, ck, ctx->d_partials);
    LAUNCHED();
    k_reduce_chunks<<<1, 1024, 0, s>>>(ctx->d_partials, 6, ro, ctx->d_cg + 9);   // r.z, b.b
    LAUNCHED();
    CK(cudaMemcpyAsync(ctx->d_cg, ctx->d_cg + 9, 3 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    ctx->launches += 1;
    int it = 0;
    constexpr int CHECK = 8;
    for (;;) {
        for (int k = 0; k < CHECK && it < max_iter; ++k, ++it) {
            k_cg_spmv<<<ck.nc, RED_THREADS, 0, s>>>(nbr, deg, wsym, dpert, pv, qv, ck,
                                                     ctx->d_partials);
            LAUNCHED();
            k_reduce_chunks<<<1, 1024, 0, s>>>(ctx->d_partials, 3, ro, ctx->d_cg + 3);   // p.Ap
            LAUNCHED();
            k_cg_step<<<ck.nc, RED_THREADS, 0, s>>>(x, r, zv, pv, qv, dpert, ctx->d_cg, ck,
                                                     ctx->d_partials, ctx->d_status);
            LAUNCHED();
            k_reduce_chunks<<<1, 1024, 0, s>>>(ctx->d_partials, 6, ro, ctx->d_cg + 6);   // r.z, r.r
            LAUNCHED();
            k_cg_dir<<<RED_BLOCKS, VEC_THREADS, 0, s>>>(pv, zv, ctx->d_cg, len);
            LAUNCHED();
            k_cg_roll<<<1, 32, 0, s>>>(ctx->d_cg);
            LAUNCHED();
        }
        CK(cudaMemcpyAsync(ctx->h_scal, ctx->d_cg, 16 * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, 16 * sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (ctx->h_status[0]) return status_to_code(ctx, ctx->h_status[0]);
        bool done = true;
        for (int c = 0; c < 3; ++c) {
            const double rr = ctx->h_scal[9 + c], bb = ctx->h_scal[12 + c];
            if (!std::isfinite(rr))
                return fail(ctx, SCVT_ERR_FACTORIZATION, "Laplacian solve produced non-finite values");
            if (rr > tol * tol * bb) done = false;
        }
        if (done) break;
        if (it >= max_iter)
            return fail(ctx, SCVT_ERR_FACTORIZATION, "Laplacian CG did not reach %.1e in %d iterations",
                        tol, max_iter);
    }
    *iters_host = it;
    return SCVT_OK;
}

int scvt_twoloop_backward(scvt_ctx* ctx, const double* g, int64_t n, double* q) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    const int64_t len = 3 * n;
    cudaStream_t s = ctx->stream;
    k_copy<<<RED_BLOCKS, VEC_THREADS, 0, s>>>(g, len, q);
    LAUNCHED();
    const int64_t stride = 3 * ctx->n_max;
    for (int r = ctx->hist_count - 1; r >= 0; --r) {       // newest -> oldest
        const int slot = (ctx->hist_head + r) % ctx->m;
        TRY(dot_to_slot(ctx, ctx->d_S + slot * stride, q, len, 0));
        k_twoloop_back<<<RED_BLOCKS, RED_THREADS, 0, s>>>(q, ctx->d_Y + slot * stride, len,
                                                          ctx->d_partials, ctx->rho[slot],
                                                          ctx->d_alpha + slot);
        LAUNCHED();
    }
    return SCVT_OK;
}

int scvt_twoloop_forward(scvt_ctx* ctx, double* q, const double* g, int64_t n, double* qg_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    const int64_t len = 3 * n;
    cudaStream_t s = ctx->stream;
    const int64_t stride = 3 * ctx->n_max;
    const int cnt = ctx->hist_count;
    for (int r = 0; r < cnt; ++r) {                         // oldest -> newest, negate last
        const int slot = (ctx->hist_head + r) % ctx->m;
        TRY(dot_to_slot(ctx, ctx->d_Y + slot * stride, q, len, 0));
        k_twoloop_fwd<<<RED_BLOCKS, RED_THREADS, 0, s>>>(q, ctx->d_S + slot * stride, len,
                                                         ctx->d_partials, ctx->rho[slot],
                                                         ctx->d_alpha + slot, r == cnt - 1 ? 1 : 0);
        LAUNCHED();
    }
    if (cnt == 0) {
        k_scale<<<RED_BLOCKS, VEC_THREADS, 0, s>>>(-1.0, q, len, q);
        LAUNCHED();
    }
    TRY(dot_to_slot(ctx, q, g, len, 0));
    TRY(finish_slots(ctx, 1));
    TRY(readback(ctx, 1));
    *qg_host = ctx->h_scal[0];
    return SCVT_OK;
}

// ---------------------------------------------------------------------- optimizer algebra
int scvt_history_clear(scvt_ctx* ctx) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    ctx->hist_head = 0;
    ctx->hist_count = 0;
    ctx->staged_valid = false;
    return SCVT_OK;
}

int scvt_history_size(scvt_ctx* ctx, int32_t* size_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    *size_host = ctx->hist_count;
    return SCVT_OK;
}

int scvt_history_gamma(scvt_ctx* ctx, double* gamma_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    if (ctx->hist_count == 0) { *gamma_host = 1.0; return SCVT_OK; }
    int newest = (ctx->hist_head + ctx->hist_count - 1) % ctx->m;
    *gamma_host = ctx->ys[newest] / ctx->yy[newest];
    return SCVT_OK;
}

int scvt_history_push(scvt_ctx* ctx, const double* z_old, const double* z_new, const double* g_old,
                      const double* g_new, int64_t n, int32_t* pushed_host, double* movement_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, 0, 1, &ck));
    // staged into tmp buffers so a rejected pair never clobbers the oldest stored one
    int nval = 0;
    TRY(pair_phase(ctx, z_old, z_new, g_old, g_new, ck, ctx->d_partials, &nval));
    return commit_phase(ctx, ctx->d_partials, ck.len, pushed_host, movement_host);
}

int scvt_lbfgs_direction_tangent(scvt_ctx* ctx, const double* g, const double* lloyd_diag,
                                 double gamma, const double* z, int64_t n, double* q3,
                                 double* out_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, 0, 1, &ck));
    TRY(gram_phase(ctx, g, lloyd_diag, gamma, ck, ctx->d_partials));
    TRY(combine_phase(ctx, g, lloyd_diag, gamma, z, ck, ctx->d_partials, q3, ctx->d_partials));
    TRY(reduce_chunks(ctx, ctx->d_partials, 2, nullptr));
    TRY(readback(ctx, 2));
    out_host[0] = ctx->h_scal[0];   // q . g
    out_host[1] = ctx->h_scal[1];   // dphi0 = g . q3
    return SCVT_OK;
}

int scvt_lbfgs_direction_tangent_async(scvt_ctx* ctx, const double* g, const double* lloyd_diag,
                                       double gamma, const double* z, int64_t n, double* q3) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, 0, 1, &ck));
    TRY(gram_phase(ctx, g, lloyd_diag, gamma, ck, ctx->d_partials));
    TRY(combine_phase(ctx, g, lloyd_diag, gamma, z, ck, ctx->d_partials, q3, ctx->d_partials));
    TRY(reduce_chunks(ctx, ctx->d_partials, 2, nullptr));
    // the scalars go to their own pinned slots (later readbacks reuse h_scal)
    CK(cudaMemcpyAsync(ctx->h_dir, ctx->d_scal, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaEventRecord(ctx->dir_ev, ctx->stream));
    return SCVT_OK;
}

int scvt_direction_result(scvt_ctx* ctx, double* out_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    CK(cudaEventSynchronize(ctx->dir_ev));
    out_host[0] = ctx->h_dir[0];
    out_host[1] = ctx->h_dir[1];
    return SCVT_OK;
}

int scvt_lbfgs_direction(scvt_ctx* ctx, const double* g, const double* lloyd_diag, double gamma,
                         int64_t n, double* q, double* qg_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    int64_t len = 3 * n;
    cudaStream_t s = ctx->stream;
    unsigned vb = RED_BLOCKS;
    k_copy<<<vb, VEC_THREADS, 0, s>>>(g, len, q);
    LAUNCHED();
    int cnt = ctx->hist_count;
    int64_t stride = 3 * ctx->n_max;
    // backward: newest -> oldest
    for (int r = cnt - 1; r >= 0; --r) {
        int slot = (ctx->hist_head + r) % ctx->m;
        TRY(dot_to_slot(ctx, ctx->d_S + slot * stride, q, len, 0));
        k_twoloop_back<<<vb, RED_THREADS, 0, s>>>(q, ctx->d_Y + slot * stride, len,
                                                   ctx->d_partials, ctx->rho[slot],
                                                   ctx->d_alpha + slot);
        LAUNCHED();
    }
    k_apply_h0<<<vb, VEC_THREADS, 0, s>>>(q, lloyd_diag, gamma, n, cnt == 0 ? 1 : 0);
    LAUNCHED();
    // forward: oldest -> newest, negate on the last
    for (int r = 0; r < cnt; ++r) {
        int slot = (ctx->hist_head + r) % ctx->m;
        TRY(dot_to_slot(ctx, ctx->d_Y + slot * stride, q, len, 0));
        k_twoloop_fwd<<<vb, RED_THREADS, 0, s>>>(q, ctx->d_S + slot * stride, len,
                                                  ctx->d_partials, ctx->rho[slot],
                                                  ctx->d_alpha + slot, r == cnt - 1 ? 1 : 0);
        LAUNCHED();
    }
    TRY(dot_to_slot(ctx, q, g, len, 0));
    TRY(finish_slots(ctx, 1));
    TRY(readback(ctx, 1));
    *qg_host = ctx->h_scal[0];
    return SCVT_OK;
}

int scvt_tangent_project(scvt_ctx* ctx, const double* q, const double* z, const double* g,
                         int64_t n, double* q3, double* dphi0_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, 0, 1, &ck));
    k_tangent<<<ck.nc, RED_THREADS, 0, ctx->stream>>>(q, z, g, ck, q3, ctx->d_partials);
    LAUNCHED();
    TRY(reduce_chunks(ctx, ctx->d_partials, 1, nullptr));
    TRY(readback(ctx, 1));
    *dphi0_host = ctx->h_scal[0];
    return SCVT_OK;
}

int scvt_trial_point(scvt_ctx* ctx, const double* z, const double* q3, double alpha, int64_t n,
                     double* zt, double* norms) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    k_trial<<<RED_BLOCKS, VEC_THREADS, 0, ctx->stream>>>(z, q3, alpha, n, zt, norms);
    LAUNCHED();
    return SCVT_OK;
}

int scvt_directional_derivative(scvt_ctx* ctx, const double* g, const double* q3,
                                const double* norms, int64_t n, double* d_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    Chunks ck;
    TRY(make_chunks(ctx, n, 0, 1, &ck));
    k_dirderiv<<<ck.nc, RED_THREADS, 0, ctx->stream>>>(g, q3, norms, ck, ctx->d_partials);
    LAUNCHED();
    TRY(reduce_chunks(ctx, ctx->d_partials, 1, nullptr));
    TRY(readback(ctx, 1));
    *d_host = ctx->h_scal[0];
    return SCVT_OK;
}

int scvt_lloyd_step(scvt_ctx* ctx, const double* first, int64_t n, double* z_out) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    TRY(reset_status(ctx));
    k_lloyd<<<RED_BLOCKS, VEC_THREADS, 0, ctx->stream>>>(first, n, z_out, ctx->d_status);
    LAUNCHED();
    TRY(readback(ctx, 0));
    if (ctx->h_status[0]) return status_to_code(ctx, ctx->h_status[0]);
    return SCVT_OK;
}

int scvt_min(scvt_ctx* ctx, const double* v, int64_t len, double* min_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    k_reduce_stage1<2><<<RED_BLOCKS, RED_THREADS, 0, ctx->stream>>>(v, len, ctx->d_partials);
    LAUNCHED();
    k_reduce_stage2<2><<<1, RED_THREADS, 0, ctx->stream>>>(ctx->d_partials, 1, ctx->d_scal);
    LAUNCHED();
    TRY(readback(ctx, 1));
    *min_host = ctx->h_scal[0];
    return SCVT_OK;
}

int scvt_max_abs_diff(scvt_ctx* ctx, const double* a, const double* b, int64_t len,
                      double* max_host) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    k_absdiff_stage1<<<RED_BLOCKS, RED_THREADS, 0, ctx->stream>>>(a, b, len, ctx->d_partials);
    LAUNCHED();
    k_reduce_stage2<1><<<1, RED_THREADS, 0, ctx->stream>>>(ctx->d_partials, 1, ctx->d_scal);
    LAUNCHED();
    TRY(readback(ctx, 1));
    *max_host = ctx->h_scal[0];
    return SCVT_OK;
}

int scvt_scale(scvt_ctx* ctx, double a, const double* x, int64_t len, double* y) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    k_scale<<<RED_BLOCKS, VEC_THREADS, 0, ctx->stream>>>(a, x, len, y);
    LAUNCHED();
    return SCVT_OK;
}

int scvt_normalize_rows(scvt_ctx* ctx, double* z, int64_t n) {
    DeviceGuard dg_(ctx);
    if (!ctx) return SCVT_ERR_CONFIG;
    k_normalize<<<RED_BLOCKS, VEC_THREADS, 0, ctx->stream>>>(z, n);
    LAUNCHED();
    return SCVT_OK;
}

}  // extern "C"
