// scvt_cells_warp.cuh — warp-cooperative Voronoi cell construction (sm_100a fast path).
//
// One warp builds the cell of one generator.  The clip polygon lives in registers, one edge
// per lane (line a.u <= b, label, start vertex), so a half-plane clip is a ballot over the
// lanes, two line intersections and one shuffle-compaction — no local memory.  Candidates
// are gathered cooperatively from the cube-map buckets (32 points per step), rank-sorted in
// shared memory and clipped nearest-first with the security-radius early exit (see
// build_cell in scvt_device.cuh for the single-thread restatement and the proof sketch).
// Cells whose polygon would exceed 32 edges fall back to the single-thread builder.
#pragma once

#include "scvt_device.cuh"

namespace scvt {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WCAND = 64;        // sorted candidate capacity per warp
constexpr int CELL_WARPS = 4;    // warps per block of k_cells_warp

struct WPoly {                   // lane k holds edge k (k < n)
    double ax, ay, b, vx, vy;
    int lab;
    int n;
};

__device__ __forceinline__ void wpoly_init(WPoly& P, int lane) {
    const double L = BOX_L;
    P.n = 4;
    P.ax = 0.0; P.ay = 0.0; P.b = L; P.vx = 0.0; P.vy = 0.0; P.lab = -1;
    if (lane == 0) { P.ay = -1.0; P.vx = -L; P.vy = -L; }
    else if (lane == 1) { P.ax = 1.0; P.vx = L; P.vy = -L; }
    else if (lane == 2) { P.ay = 1.0; P.vx = L; P.vy = L; }
    else if (lane == 3) { P.ax = -1.0; P.vx = -L; P.vy = L; }
}

// Clip by a.u <= b (label j at zj).  0 = unchanged, 1 = clipped, <0 = needs fallback.
__device__ __forceinline__ int wpoly_clip(WPoly& P, int lane, double ax, double ay, double b,
                                          int j, V3 zj, ClipCtx& cc) {
    const int n = P.n;
    const bool act = lane < n;
    const int labm = __shfl_sync(FULL, P.lab, lane == 0 ? n - 1 : lane - 1);
    bool o = false;
    if (act) {
        double t1 = ax * P.vx, t2 = ay * P.vy;
        double s = t1 + t2 - b;
        double tol = 1e-9 * (fabs(t1) + fabs(t2) + b);
        if (s > tol) o = true;
        else if (s < -tol) o = false;
        else if (labm >= 0 && P.lab >= 0) {
            int tier;
            o = orient_robust(cc.zi, load3(cc.z, labm), load3(cc.z, P.lab), zj, cc.i, labm, P.lab,
                              j, &tier) > 0;
            cc.tie_breaks += tier == 2;
        } else {
            o = s > 0.0;
        }
    }
    const unsigned mo = __ballot_sync(FULL, o);
    if (mo == 0u) return 0;
    const int nout = __popc(mo);
    if (nout == n) return -1;
    const unsigned full_n = n == 32 ? FULL : ((1u << n) - 1u);
    const unsigned prev = ((mo << 1) | (mo >> (n - 1))) & full_n;   // bit k = out[k-1]
    const unsigned next = ((mo >> 1) | (mo << (n - 1))) & full_n;   // bit k = out[k+1]
    const unsigned firsts = mo & ~prev, lasts = mo & ~next;
    if (__popc(firsts) != 1 || __popc(lasts) != 1) return -2;
    const int first = __ffs(firsts) - 1, last = __ffs(lasts) - 1;
    const int ein = first == 0 ? n - 1 : first - 1;
    const int m = n - nout + 2;
    if (m > 32) return -3;
    double eax = __shfl_sync(FULL, P.ax, ein), eay = __shfl_sync(FULL, P.ay, ein);
    double eb = __shfl_sync(FULL, P.b, ein);
    double lax = __shfl_sync(FULL, P.ax, last), lay = __shfl_sync(FULL, P.ay, last);
    double lb = __shfl_sync(FULL, P.b, last);
    double Ax, Ay, Bx, By;
    line_meet(eax, eay, eb, ax, ay, b, &Ax, &Ay);
    line_meet(ax, ay, b, lax, lay, lb, &Bx, &By);
    // surviving edges last, last+1, ..., ein (cyclic) -> lanes 0..m-2; new edge -> lane m-1
    const int src = (last + lane) % n;
    double nax = __shfl_sync(FULL, P.ax, src), nay = __shfl_sync(FULL, P.ay, src);
    double nb = __shfl_sync(FULL, P.b, src);
    double nvx = __shfl_sync(FULL, P.vx, src), nvy = __shfl_sync(FULL, P.vy, src);
    int nlab = __shfl_sync(FULL, P.lab, src);
    if (lane == 0) { nvx = Bx; nvy = By; }
    if (lane == m - 1) { nax = ax; nay = ay; nb = b; nlab = j; nvx = Ax; nvy = Ay; }
    P.ax = nax; P.ay = nay; P.b = nb; P.vx = nvx; P.vy = nvy; P.lab = nlab;
    P.n = m;
    return 1;
}

__device__ __forceinline__ double wpoly_R2(const WPoly& P, int lane, bool* box) {
    double c = lane < P.n ? vertex_chord2(P.vx, P.vy) : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c = fmax(c, __shfl_xor_sync(FULL, c, off));
    *box = __any_sync(FULL, lane < P.n && P.lab < 0);
    return *box ? 8.0 : c;
}

// Returns valence > 0, -ST_* for genuine failures, or -ST_POLY_OVERFLOW to request the
// single-thread fallback.  All lanes return the same value.
__device__ int build_cell_warp(const GridView& g, int i, V3 zi, int lane, double* s_c2,
                               int* s_j, int* s_p, int* nbr_out, CellStats* st) {
    V3 e1, e2;
    tangent_frame(zi, &e1, &e2);
    WPoly P;
    wpoly_init(P, lane);
    ClipCtx cc;
    cc.z = g.z; cc.zi = zi; cc.i = i; cc.tie_breaks = 0;
    uint32_t key = bucket_key(zi, g.G);
    int cnt = g.start[key + 1] - g.start[key];
    double area_b = 4.0 * M_PI / (6.0 * (double)g.G * (double)g.G);
    double h2 = area_b / (double)(cnt > 0 ? cnt : 1);
    double r2 = 12.25 * h2;                    // first radius 3.5 h
    if (r2 > 4.0) r2 = 4.0000001;
    double lo_c2 = -1.0;                       // exclusive lower bound on c2
    double R2 = 8.0;
    bool box = true;
    int status = 0, rounds = 0, passes = 0;
    const unsigned lt_mask = (1u << lane) - 1u;
    while (true) {
        ++passes;
        if (passes > 64) { status = ST_POLY_OVERFLOW; break; }
        CapBox cb = cap_box(zi, sqrt(r2));
        double lim = 4.0 * R2 * (1.0 + 1e-12);
        int count = 0;
        // ---- gather candidates in (lo_c2, r2] that can still cut the cell
        for (int face = 0; face < 6; ++face) {
            int iu0, iu1, iv0, iv1;
            if (!cap_face_range(cb, face, g.G, &iu0, &iu1, &iv0, &iv1)) continue;
            for (int iu = iu0; iu <= iu1; ++iu) {
                int rowbase = (face * g.G + iu) * g.G;
                int p0 = g.start[rowbase + iv0], p1 = g.start[rowbase + iv1 + 1];
                for (int base = p0; base < p1; base += 32) {
                    int p = base + lane;
                    bool acc = false;
                    double c2 = 0.0;
                    int j = -1;
                    if (p < p1) {
                        j = g.ids[p];
                        const double* q = g.zs + 4 * (int64_t)p;
                        double dx = q[0] - zi.x, dy = q[1] - zi.y, dz = q[2] - zi.z;
                        c2 = dx * dx + dy * dy + dz * dz;
                        acc = j != i && c2 <= r2 && c2 < lim && c2 > lo_c2;
                        if (acc && c2 == 0.0) { status |= ST_DUPLICATE; acc = false; }
                    }
                    unsigned ma = __ballot_sync(FULL, acc);
                    int pos = count + __popc(ma & lt_mask);
                    if (acc && pos < WCAND) { s_c2[pos] = c2; s_j[pos] = j; s_p[pos] = p; }
                    count += __popc(ma);
                }
            }
        }
        status = __reduce_or_sync(FULL, status);
        if (status) break;
        __syncwarp();
        if (count <= WCAND) {
            // ---- rank sort by (c2, id), then clip nearest-first with early exit
            double kc[2];
            int kj[2], kp[2], rk[2];
            for (int h = 0; h < 2; ++h) {
                int e = lane + 32 * h;
                rk[h] = -1;
                if (e < count) {
                    kc[h] = s_c2[e]; kj[h] = s_j[e]; kp[h] = s_p[e];
                    int r = 0;
                    for (int f = 0; f < count; ++f) {
                        double cf = s_c2[f];
                        int jf = s_j[f];
                        r += (cf < kc[h]) || (cf == kc[h] && jf < kj[h]);
                    }
                    rk[h] = r;
                }
            }
            __syncwarp();
            for (int h = 0; h < 2; ++h)
                if (rk[h] >= 0) { s_c2[rk[h]] = kc[h]; s_j[rk[h]] = kj[h]; s_p[rk[h]] = kp[h]; }
            __syncwarp();
            for (int t = 0; t < count; ++t) {
                double c2 = s_c2[t];
                if (c2 >= 4.0 * R2 * (1.0 + 1e-12)) break;
                int j = s_j[t];
                const double* q = g.zs + 4 * (int64_t)s_p[t];
                V3 zj = v3(q[0], q[1], q[2]);
                V3 d = sub(zj, zi);
                int rc = wpoly_clip(P, lane, dot(d, e1), dot(d, e2), 0.5 * c2, j, zj, cc);
                if (rc < 0) { status = ST_POLY_OVERFLOW; break; }
                if (rc == 1) R2 = wpoly_R2(P, lane, &box);
            }
            __syncwarp();
        } else {
            // ---- dense neighbourhood of a large cell: clip in scan order
            ++passes;
            for (int face = 0; face < 6 && !status; ++face) {
                int iu0, iu1, iv0, iv1;
                if (!cap_face_range(cb, face, g.G, &iu0, &iu1, &iv0, &iv1)) continue;
                for (int iu = iu0; iu <= iu1 && !status; ++iu) {
                    int rowbase = (face * g.G + iu) * g.G;
                    int p0 = g.start[rowbase + iv0], p1 = g.start[rowbase + iv1 + 1];
                    for (int base = p0; base < p1 && !status; base += 32) {
                        int p = base + lane;
                        bool acc = false;
                        double c2 = 0.0;
                        int j = -1;
                        V3 zj = v3(0, 0, 0);
                        double cax = 0.0, cay = 0.0;
                        if (p < p1) {
                            j = g.ids[p];
                            const double* q = g.zs + 4 * (int64_t)p;
                            zj = v3(q[0], q[1], q[2]);
                            V3 d = sub(zj, zi);
                            c2 = dot(d, d);
                            acc = j != i && c2 <= r2 && c2 > lo_c2 && c2 > 0.0 &&
                                  c2 < 4.0 * R2 * (1.0 + 1e-12);
                            cax = dot(d, e1);
                            cay = dot(d, e2);
                        }
                        // vertex-disk test, one candidate per lane: j can cut the cell only if
                        // some current vertex is (about) as close to z_j as to z_i
                        if (__any_sync(FULL, acc)) {
                            bool may = false;
                            const double cb2 = 0.5 * c2;
                            for (int k = 0; k < P.n; ++k) {
                                double vx = __shfl_sync(FULL, P.vx, k);
                                double vy = __shfl_sync(FULL, P.vy, k);
                                double t1 = cax * vx, t2 = cay * vy;
                                may |= t1 + t2 - cb2 > -1e-9 * (fabs(t1) + fabs(t2) + cb2);
                            }
                            acc = acc && may;
                        }
                        unsigned ma = __ballot_sync(FULL, acc);
                        while (ma) {
                            int src = __ffs(ma) - 1;
                            ma &= ma - 1u;
                            double cs = __shfl_sync(FULL, c2, src);
                            int js = __shfl_sync(FULL, j, src);
                            V3 zs = v3(__shfl_sync(FULL, zj.x, src), __shfl_sync(FULL, zj.y, src),
                                       __shfl_sync(FULL, zj.z, src));
                            if (cs >= 4.0 * R2 * (1.0 + 1e-12)) continue;
                            V3 d = sub(zs, zi);
                            int rc = wpoly_clip(P, lane, dot(d, e1), dot(d, e2), 0.5 * cs, js, zs, cc);
                            if (rc < 0) { status = ST_POLY_OVERFLOW; break; }
                            if (rc == 1) R2 = wpoly_R2(P, lane, &box);
                        }
                    }
                }
            }
        }
        if (status) break;
        ++rounds;
        if (r2 >= 4.0) {
            if (box) status = ST_UNBOUNDED;
            break;
        }
        if (!box && 4.0 * R2 * (1.0 + 1e-9) <= r2) break;     // security radius certified
        lo_c2 = r2;
        double want = box ? 4.0 * r2 : 4.0 * R2 * (1.0 + 1e-9);
        r2 = want >= 4.0 ? 4.0000001 : want;
    }
    st->rounds = rounds;
    st->passes = passes;
    st->tie_breaks = __reduce_add_sync(FULL, cc.tie_breaks);
    if (status) return -status;
    const int n = P.n;
    int mylab = lane < n ? P.lab : 0x7fffffff;
    int minlab = __reduce_min_sync(FULL, mylab);
    int lead = __ffs(__ballot_sync(FULL, lane < n && P.lab == minlab)) - 1;
    if (lane < n) {
        int k = lane - lead;
        if (k < 0) k += n;
        nbr_out[k] = P.lab;
    }
    return n;
}

}  // namespace scvt
