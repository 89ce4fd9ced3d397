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
    int src = last + lane;                       // (last + lane) mod n for lanes < m
    if (src >= n) src -= n;
    if (src >= n) src = 0;
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

// max vertex chord^2: chord^2 is monotone in |u|^2, so reduce |u|^2 and convert once
__device__ __forceinline__ double wpoly_R2(const WPoly& P, int lane, bool* box) {
    *box = __any_sync(FULL, lane < P.n && P.lab < 0);
    if (*box) return 8.0;
    double q = lane < P.n ? P.vx * P.vx + P.vy * P.vy : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) q = fmax(q, __shfl_xor_sync(FULL, q, off));
    // chord^2 = 2q / (s (s + 1)), s = sqrt(1 + q); branch-free, ~1 ulp (only compared with
    // candidate distances, and rounded up by the callers' (1 + 1e-12) factors)
    const double is = fast_rsqrt(1.0 + q);
    const double sq = (1.0 + q) * is;
    return 2.0 * q * is * fast_rcp(sq + 1.0) * (1.0 + 1e-15);
}

// local point density from the 3x3 bucket neighbourhood of `key` (same face only)
__device__ __forceinline__ double local_spacing2(const GridView& g, uint32_t key) {
    const int G = g.G;
    const int face = key / (G * G), rem = key % (G * G), iu = rem / G, iv = rem % G;
    const int u0 = max(iu - 1, 0), u1 = min(iu + 1, G - 1);
    const int v0 = max(iv - 1, 0), v1 = min(iv + 1, G - 1);
    int cnt = 0;
    for (int u = u0; u <= u1; ++u) {
        const int row = (face * G + u) * G;
        cnt += g.start[row + v1 + 1] - g.start[row + v0];
    }
    const double nb = (double)((u1 - u0 + 1) * (v1 - v0 + 1));
    const double area_b = 4.0 * M_PI / (6.0 * (double)G * (double)G);
    return nb * area_b / (double)(cnt > 1 ? cnt : 1);
}

// Bounding cap (centre, chord radius) of the bucket block [ua..ub] x [va..vb] on `face`.
// Lines of constant u (or v) are great circles, so the block is a convex spherical
// quadrilateral and its farthest point from the centre is a corner.
__device__ __forceinline__ void face_point(int face, float u, float v, float* x, float* y, float* z) {
    const int a = face >> 1;
    const float sg = (face & 1) ? -1.0f : 1.0f;
    float c[3];
    c[a] = sg;
    c[face_axes_b(a)] = u;
    c[face_axes_c(a)] = v;
    const float inv = rsqrtf(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    *x = c[0] * inv; *y = c[1] * inv; *z = c[2] * inv;
}

__device__ __forceinline__ void block_cap(int face, int G, int ua, int ub, int va, int vb,
                                          float* cx, float* cy, float* cz, float* rad) {
    const float k = 1.5707963267948966f / (float)G;     // equi-angular step
    const float a0 = ua * k - 0.78539816f, a1 = (ub + 1) * k - 0.78539816f;
    const float b0 = va * k - 0.78539816f, b1 = (vb + 1) * k - 0.78539816f;
    face_point(face, tanf(0.5f * (a0 + a1)), tanf(0.5f * (b0 + b1)), cx, cy, cz);
    const float tu[2] = {tanf(a0), tanf(a1)}, tv[2] = {tanf(b0), tanf(b1)};
    float r2 = 0.f;
    for (int q = 0; q < 4; ++q) {
        float x, y, z;
        face_point(face, tu[q & 1], tv[q >> 1], &x, &y, &z);
        const float dx = x - *cx, dy = y - *cy, dz = z - *cz;
        r2 = fmaxf(r2, dx * dx + dy * dy + dz * dz);
    }
    *rad = sqrtf(r2) * 1.0001f + 1e-5f;
}

// Per-lane vertex circumdisk on the sphere (float, conservative): a point can cut the cell
// only inside some disk |y - y_k| < R_k.  Box vertices (and idle lanes) cover everything.
__device__ __forceinline__ void vertex_disk(const WPoly& P, int lane, V3 zi, V3 e1, V3 e2,
                                            float* vyx, float* vyy, float* vyz, float* vR) {
    if (lane < P.n && P.lab >= 0) {
        double x = zi.x + P.vx * e1.x + P.vy * e2.x;
        double y = zi.y + P.vx * e1.y + P.vy * e2.y;
        double w = zi.z + P.vx * e1.z + P.vy * e2.z;
        double inv = rsqrt(x * x + y * y + w * w);
        x *= inv; y *= inv; w *= inv;
        double rx = x - zi.x, ry = y - zi.y, rz = w - zi.z;
        *vyx = (float)x; *vyy = (float)y; *vyz = (float)w;
        *vR = (float)sqrt(rx * rx + ry * ry + rz * rz);
    } else {
        *vyx = *vyy = *vyz = 0.f;
        *vR = lane < P.n ? 3.0f : 0.f;
    }
}

// cap rectangles above this many buckets go to the culled sweep once the polygon is bounded
constexpr int SWEEP_BUCKETS = 8192;

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
    double h2 = local_spacing2(g, bucket_key(zi, g.G));
    double r2 = 9.0 * h2;                      // first radius 3 h
    if (r2 > 4.0) r2 = 4.0000001;
    double lo_c2 = -1.0;                       // exclusive lower bound on c2
    double R2 = 8.0;
    bool box = true;
    int status = 0, rounds = 0, passes = 0, sweep_visits = 0, scanned = 0, ncands = 0, nclips = 0;
    int shrinks = 0;
    const unsigned lt_mask = (1u << lane) - 1u;
    while (true) {
        ++passes;
        if (passes > 64) { status = ST_POLY_OVERFLOW; break; }
        CapBox cb = cap_box(zi, sqrt(r2));
        double lim = 4.0 * R2 * (1.0 + 1e-12);
        int count = 0;
        if (!box) {
            // a bounded polygon with a large security disk (a far vertex, or a coarse cell
            // next to a dense region): the plain gather would rescan every bucket of the cap,
            // inner disk included; the sweep culls 8x8-bucket blocks by the vertex disks
            int nbk = 0;
            for (int face = 0; face < 6; ++face) {
                int iu0, iu1, iv0, iv1;
                if (cap_face_range(cb, face, g.G, &iu0, &iu1, &iv0, &iv1))
                    nbk += (iu1 - iu0 + 1) * (iv1 - iv0 + 1);
            }
            if (nbk > SWEEP_BUCKETS) count = WCAND + 1;
        }
        // ---- gather candidates in (lo_c2, r2] that can still cut the cell
        for (int face = 0; face < 6 && count <= WCAND; ++face) {
            int iu0, iu1, iv0, iv1;
            if (!cap_face_range(cb, face, g.G, &iu0, &iu1, &iv0, &iv1)) continue;
            for (int iu = iu0; iu <= iu1 && count <= WCAND; ++iu) {
                int rowbase = (face * g.G + iu) * g.G;
                int p0 = g.start[rowbase + iv0], p1 = g.start[rowbase + iv1 + 1];
                for (int base = p0; base < p1 && count <= WCAND; base += 32) {
                    int p = base + lane;
                    bool acc = false;
                    double c2 = 0.0;
                    int j = -1;
                    if (p < p1) {
                        j = __ldg(g.ids + p);
                        const double2* q2 = reinterpret_cast<const double2*>(g.zs + 4 * (int64_t)p);
                        double2 xy = __ldg(q2);
                        double zz = __ldg(g.zs + 4 * (int64_t)p + 2);
                        double dx = xy.x - zi.x, dy = xy.y - zi.y, dz = zz - zi.z;
                        c2 = dx * dx + dy * dy + dz * dz;
                        acc = j != i && c2 <= r2 && c2 < lim && c2 > lo_c2;
                        if (acc && c2 == 0.0) { status |= ST_DUPLICATE; acc = false; }
                    }
                    unsigned ma = __ballot_sync(FULL, acc);
                    scanned += min(32, p1 - base);
                    int pos = count + __popc(ma & lt_mask);
                    if (acc && pos < WCAND) { s_c2[pos] = c2; s_j[pos] = j; s_p[pos] = p; }
                    count += __popc(ma);
                }
            }
        }
        status = __reduce_or_sync(FULL, status);
        if (status) break;
        __syncwarp();
        if (count > WCAND && shrinks < 4) {
            // annulus denser than expected (a coarse cell next to the plateau, or a far
            // vertex that inflated R2): narrow it and clip nearest-first instead of sweeping;
            // the sweep, if still needed, then starts from a tighter polygon.  Capped per
            // cell: a coarse cell whose security disk covers a dense region would otherwise
            // crawl through it in thin annuli (the culled sweep is the right tool there)
            ++shrinks;
            r2 = lo_c2 < 0.0 ? 0.25 * r2 : lo_c2 + 0.25 * (r2 - lo_c2);
            continue;
        }
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
            ncands += count;
            for (int t = 0; t < count; ++t) {
                double c2 = s_c2[t];
                if (c2 >= 4.0 * R2 * (1.0 + 1e-12)) break;
                ++nclips;
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
            // ---- dense neighbourhood of a large cell: hierarchical sweep.  Lanes first test
            // 8x8-bucket blocks against the vertex circumdisks (a point can cut the cell only
            // inside some disk |y - y_k| < R_k); only intersecting blocks are scanned, their
            // points tested per lane, and survivors clipped one at a time.
            ++passes;
            float vyx = 0.f, vyy = 0.f, vyz = 0.f, vR = 0.f;
            bool dirty = true;
            for (int face = 0; face < 6 && !status; ++face) {
                int iu0, iu1, iv0, iv1;
                if (!cap_face_range(cb, face, g.G, &iu0, &iu1, &iv0, &iv1)) continue;
                const int bu0 = iu0 >> 3, bu1 = iu1 >> 3, bv0 = iv0 >> 3, bv1 = iv1 >> 3;
                const int nbv = bv1 - bv0 + 1, nblk = (bu1 - bu0 + 1) * nbv;
                for (int b0 = 0; b0 < nblk && !status; b0 += 32) {
                    if (dirty) {
                        vertex_disk(P, lane, zi, e1, e2, &vyx, &vyy, &vyz, &vR);
                        dirty = false;
                    }
                    const int bk = b0 + lane;
                    bool hit = false;
                    int ua = 0, ub = -1, va = 0, vb = -1;
                    float cx = 0.f, cy = 0.f, cz = 0.f, crad = 0.f;
                    if (bk < nblk) {
                        const int bu = bu0 + bk / nbv, bv = bv0 + bk % nbv;
                        ua = max(bu << 3, iu0); ub = min((bu << 3) + 7, iu1);
                        va = max(bv << 3, iv0); vb = min((bv << 3) + 7, iv1);
                        block_cap(face, g.G, ua, ub, va, vb, &cx, &cy, &cz, &crad);
                    }
                    for (int k = 0; k < P.n; ++k) {
                        float kx = __shfl_sync(FULL, vyx, k), ky = __shfl_sync(FULL, vyy, k);
                        float kz = __shfl_sync(FULL, vyz, k), kr = __shfl_sync(FULL, vR, k);
                        float dx = kx - cx, dy = ky - cy, dz = kz - cz;
                        float lim2 = kr + crad + 1e-4f;
                        hit |= dx * dx + dy * dy + dz * dz < lim2 * lim2;
                    }
                    unsigned mb = __ballot_sync(FULL, hit && bk < nblk);
                    while (mb && !status) {
                        const int src = __ffs(mb) - 1;
                        mb &= mb - 1u;
                        const int bua = __shfl_sync(FULL, ua, src), bub = __shfl_sync(FULL, ub, src);
                        const int bva = __shfl_sync(FULL, va, src), bvb = __shfl_sync(FULL, vb, src);
                        if (dirty) {
                            // the polygon shrank since this batch was tested: re-test the
                            // block against the current vertex disks before scanning it
                            vertex_disk(P, lane, zi, e1, e2, &vyx, &vyy, &vyz, &vR);
                            dirty = false;
                            const float bx = __shfl_sync(FULL, cx, src), by = __shfl_sync(FULL, cy, src);
                            const float bz = __shfl_sync(FULL, cz, src), br = __shfl_sync(FULL, crad, src);
                            const float dx = vyx - bx, dy = vyy - by, dz = vyz - bz;
                            const float lim2 = vR + br + 1e-4f;
                            const bool h = lane < P.n && dx * dx + dy * dy + dz * dz < lim2 * lim2;
                            if (!__any_sync(FULL, h)) continue;
                        }
                        for (int iu = bua; iu <= bub && !status; ++iu) {
                            int rowbase = (face * g.G + iu) * g.G;
                            int p0 = g.start[rowbase + bva], p1 = g.start[rowbase + bvb + 1];
                            for (int base = p0; base < p1 && !status; base += 32) {
                                sweep_visits += 32;
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
                                    int sl = __ffs(ma) - 1;
                                    ma &= ma - 1u;
                                    double cs = __shfl_sync(FULL, c2, sl);
                                    int js = __shfl_sync(FULL, j, sl);
                                    V3 zs = v3(__shfl_sync(FULL, zj.x, sl), __shfl_sync(FULL, zj.y, sl),
                                               __shfl_sync(FULL, zj.z, sl));
                                    if (cs >= 4.0 * R2 * (1.0 + 1e-12)) continue;
                                    V3 d = sub(zs, zi);
                                    int rc = wpoly_clip(P, lane, dot(d, e1), dot(d, e2), 0.5 * cs, js, zs, cc);
                                    if (rc < 0) { status = ST_POLY_OVERFLOW; break; }
                                    if (rc == 1) { R2 = wpoly_R2(P, lane, &box); dirty = true; }
                                }
                            }
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
    st->sweep_visits = sweep_visits;
    st->scanned = scanned;
    st->cands = ncands;
    st->clips = nclips;
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
