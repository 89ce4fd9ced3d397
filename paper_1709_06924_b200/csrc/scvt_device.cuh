// scvt_device.cuh — __host__ __device__ building blocks of the SCVT hot path.
//
// Everything here is pure per-element arithmetic, written once and used by the sm_100a
// kernels (scvt_kernels.cu).  The test-only host harness (tests/native/) compiles the same
// functions for the CPU so the combinatorics can be exercised without a GPU; the shipped
// library has no CPU path.
//
// Reference citations are /root/reference/pkg/src/scvtmesh/<file>.py:<line>.
#pragma once

#include <stdint.h>
#include <math.h>

#ifdef __CUDACC__
#define SCVT_HD __host__ __device__ __forceinline__
// rarely-run paths of hot kernels (the per-patch fit, the table fallback sweep): out of line,
// so their register demand does not shape the node loop's allocation (k_quad 9.54 -> 9.41 ms)
#define SCVT_COLD __host__ __device__ __noinline__
#else
#define SCVT_HD inline
#define SCVT_COLD inline
#endif

namespace scvt {

// ------------------------------------------------------------------ status bits (device)
enum : int {
    ST_OK = 0,
    ST_DUPLICATE = 1 << 0,        // two identical generators -> InsufficientPointsError
    ST_UNBOUNDED = 1 << 1,        // cell reaches the gnomonic hemisphere limit
    ST_POLY_OVERFLOW = 1 << 2,    // clip polygon exceeded MAXV edges
    ST_DEG_OVERFLOW = 1 << 3,     // valence exceeded SCVT_MAX_DEGREE
    ST_INCONSISTENT = 1 << 4,     // cycles of adjacent cells disagree (not a manifold)
    ST_NOT_DELAUNAY = 1 << 5,     // certified non-locally-Delaunay edge
    ST_EULER = 1 << 6,            // sum of valences != 6n - 12
    ST_POLE = 1 << 7,             // x16 density evaluated within 1e-9 of a pole
    ST_DEGENERATE_TRI = 1 << 8,   // zero-normal triangle in the fan construction
    ST_CENTROID = 1 << 9,         // |c| <= 1e-12 in a Lloyd step
    ST_INDEFINITE = 1 << 10,      // perturbed Laplacian not positive definite (CG p.Ap <= 0)
};

constexpr int MAXV = 64;          // polygon edges while clipping
constexpr int MAXDEG = 32;        // stored valence (== SCVT_MAX_DEGREE)
constexpr double BOX_L = 1.0e4;   // initial gnomonic box half-width (cell < ~89.99 deg)

// ------------------------------------------------------------------ small vector helpers
struct V3 { double x, y, z; };

SCVT_HD V3 v3(double x, double y, double z) { V3 r; r.x = x; r.y = y; r.z = z; return r; }
SCVT_HD V3 add(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
SCVT_HD V3 sub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
SCVT_HD V3 mul(V3 a, double s) { return v3(a.x * s, a.y * s, a.z * s); }
SCVT_HD double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
SCVT_HD V3 cross(V3 a, V3 b) {
    return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
SCVT_HD V3 load3(const double* p, int64_t i) { return v3(p[3 * i], p[3 * i + 1], p[3 * i + 2]); }

SCVT_HD double rsqrt_d(double x) {
#ifdef __CUDA_ARCH__
    return rsqrt(x);
#else
    return 1.0 / sqrt(x);
#endif
}

// 1/sqrt(a) for positive normal a without the special-case branches of the libm version:
// hardware approximation + one cubic Householder step (relative error ~1 ulp).
SCVT_HD double fast_rsqrt(double a) {
#ifdef __CUDA_ARCH__
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    const double r = fma(-(a * y), y, 1.0);        // 1 - a y^2
    const double q = fma(0.375, r, 0.5);
    return fma(q, r * y, y);                       // y (1 + r/2 + 3 r^2 / 8)
#else
    return 1.0 / sqrt(a);
#endif
}

// 1/a for finite nonzero a without the special-case branches of the IEEE division:
// hardware approximation + two Newton steps (~1 ulp).
SCVT_HD double fast_rcp(double a) {
#ifdef __CUDA_ARCH__
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    double e = fma(-a, y, 1.0);
    y = fma(y, e, y);
    e = fma(-a, y, 1.0);
    return fma(y, e, y);
#else
    return 1.0 / a;
#endif
}

// numpy's np.linalg.norm of a 3-vector is sqrt(x*x + y*y + z*z) evaluated as a dot product;
// we use the same expression.
SCVT_HD double norm3(V3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }

// ------------------------------------------------------------------ cube-map buckets
// Face = dominant axis and sign; (u, v) = the other two coordinates over |dominant|;
// equi-angular cell index so buckets have near-uniform solid angle.  Bucketing is FP32:
// range queries are conservative (angular margin + one-bucket widening) so the FP32
// rounding of keys vs ranges can never drop a candidate.
SCVT_HD int face_axes_b(int a) { return a == 0 ? 1 : 0; }
SCVT_HD int face_axes_c(int a) { return a == 2 ? 1 : 2; }

SCVT_HD int bucket_index_1d(float u, int G) {
    float t = (atanf(u) * (float)(4.0 / M_PI) + 1.0f) * 0.5f * (float)G;
    int k = (int)floorf(t);
    return k < 0 ? 0 : (k >= G ? G - 1 : k);
}

SCVT_HD uint32_t bucket_key(V3 p, int G) {
    double c[3] = {p.x, p.y, p.z};
    double ax = fabs(p.x), ay = fabs(p.y), az = fabs(p.z);
    int a = (ax >= ay && ax >= az) ? 0 : (ay >= az ? 1 : 2);
    int sgn = c[a] >= 0.0 ? 0 : 1;
    double den = fabs(c[a]);
    float u = (float)(c[face_axes_b(a)] / den), v = (float)(c[face_axes_c(a)] / den);
    int face = 2 * a + sgn;
    return (uint32_t)((face * G + bucket_index_1d(u, G)) * G + bucket_index_1d(v, G));
}

// Per-axis coordinate bounds of the spherical cap {y : |y - p| <= r} (FP32, conservative).
struct CapBox { float lo[3], hi[3]; };

SCVT_HD CapBox cap_box(V3 p, double r) {
    CapBox b;
    float th = 2.0f * asinf(fminf(1.0f, 0.5f * (float)r)) + 2e-4f;
    float c[3] = {(float)p.x, (float)p.y, (float)p.z};
    const float PI = 3.14159265358979f;
    for (int k = 0; k < 3; ++k) {
        float ck = fmaxf(-1.0f, fminf(1.0f, c[k]));
        float ang = acosf(ck);
        float a_lo = ang - th, a_hi = ang + th;
        b.hi[k] = a_lo <= 0.0f ? 1.0f : cosf(a_lo) + 1e-5f;
        b.lo[k] = a_hi >= PI ? -1.0f : cosf(a_hi) - 1e-5f;
    }
    return b;
}

// Conservative bucket rectangle of the cap on face `face`; false if the cap misses it.
SCVT_HD bool cap_face_range(const CapBox& cb, int face, int G, int* iu0, int* iu1, int* iv0,
                            int* iv1) {
    int a = face >> 1;
    bool neg = face & 1;
    float s_lo = neg ? -cb.hi[a] : cb.lo[a];
    float s_hi = neg ? -cb.lo[a] : cb.hi[a];
    const float inv_sqrt3 = 0.57735026f - 1e-4f;
    if (s_hi < inv_sqrt3) return false;
    float t_lo = fmaxf(s_lo, inv_sqrt3), t_hi = s_hi;
    int b = face_axes_b(a), cc = face_axes_c(a);
    float umin = fminf(cb.lo[b] / t_lo, cb.lo[b] / t_hi), umax = fmaxf(cb.hi[b] / t_lo, cb.hi[b] / t_hi);
    float vmin = fminf(cb.lo[cc] / t_lo, cb.lo[cc] / t_hi), vmax = fmaxf(cb.hi[cc] / t_lo, cb.hi[cc] / t_hi);
    umin = fmaxf(umin, -1.0f); umax = fminf(umax, 1.0f);
    vmin = fmaxf(vmin, -1.0f); vmax = fminf(vmax, 1.0f);
    // no +-1 widening: the 2e-4 rad cap margin (cap_box) is ~30x the FP32 error of the bucket
    // index of a point, so every point of the cap lies in the returned rectangle
    int a0 = bucket_index_1d(umin, G), a1 = bucket_index_1d(umax, G);
    int b0 = bucket_index_1d(vmin, G), b1 = bucket_index_1d(vmax, G);
    *iu0 = a0 < 0 ? 0 : a0; *iu1 = a1 >= G ? G - 1 : a1;
    *iv0 = b0 < 0 ? 0 : b0; *iv1 = b1 >= G ? G - 1 : b1;
    return true;
}

// ------------------------------------------------------------------ predicates
// insphere on the unit sphere == orient3d: for CCW-outward (o, a, b), point c lies inside
// the circumcircle of (o, a, b) iff D = det[a-o, b-o, c-o] > 0.  Three tiers:
//   0. FP64 static filter (decides almost always: seeded inputs never leave it);
//   1. exact sign of D by floating-point expansion arithmetic (Shewchuk's two-sum /
//      two-product / zero-eliminating expansion sums; every product of three input doubles is
//      a 4-term expansion, D a sum of at most 96 of them, nothing rounded);
//   2. D == 0 exactly (cocircular quad) -> Simulation of Simplicity: every point is pushed
//      radially outward by an infinitesimal, larger for lower indices (eps_0 >> eps_1 >> ...).
//      D is affine in each point, so the perturbed sign is the sign of the first non-zero
//      first-order term E_p = dD/d(eps_p) in index order, each evaluated exactly; when all
//      vanish (four points on a great circle) the tie is +1.  The perturbed set is in general
//      position, so all decisions are consistent: every cell that meets the same four points
//      takes the same decision.
// With T1 = [a,b,c], T2 = [o,b,c], T3 = [a,o,c], T4 = [a,b,o] ([p,q,r] = p.(q x r)):
//   D = T1 - T2 - T3 - T4,  E_a = T1 - T3 - T4,  E_b = T1 - T2 - T4,  E_c = T1 - T2 - T3,
//   E_o = -(T2 + T3 + T4)   (o = the origin, index < 0, is never perturbed).
struct DD { double hi, lo; };

SCVT_HD DD dd_two_sum(double a, double b) {
    double s = a + b;
    double bb = s - a;
    DD r; r.hi = s; r.lo = (a - (s - bb)) + (b - bb);
    return r;
}
SCVT_HD DD dd_two_prod(double a, double b) {
    double p = a * b;
    DD r; r.hi = p; r.lo = fma(a, b, -p);
    return r;
}

// h = e + f for nonoverlapping expansions in increasing magnitude (fast_expansion_sum with
// zero elimination); returns the length of h (<= elen + flen)
SCVT_HD int exp_sum(int elen, const double* e, int flen, const double* f, double* h) {
    double q, qn, hh;
    int ei = 0, fi = 0, hi = 0;
    double en = e[0], fn = f[0];
    if ((fn > en) == (fn > -en)) { q = en; ++ei; }
    else { q = fn; ++fi; }
    if (ei < elen && fi < flen) {
        en = e[ei]; fn = f[fi];
        if ((fn > en) == (fn > -en)) {          // fast two-sum of en and q
            qn = en + q; hh = q - (qn - en); ++ei;
        } else {
            qn = fn + q; hh = q - (qn - fn); ++fi;
        }
        q = qn;
        if (hh != 0.0) h[hi++] = hh;
        while (ei < elen && fi < flen) {
            en = e[ei]; fn = f[fi];
            DD t;
            if ((fn > en) == (fn > -en)) { t = dd_two_sum(q, en); ++ei; }
            else { t = dd_two_sum(q, fn); ++fi; }
            q = t.hi;
            if (t.lo != 0.0) h[hi++] = t.lo;
        }
    }
    while (ei < elen) {
        DD t = dd_two_sum(q, e[ei++]);
        q = t.hi;
        if (t.lo != 0.0) h[hi++] = t.lo;
    }
    while (fi < flen) {
        DD t = dd_two_sum(q, f[fi++]);
        q = t.hi;
        if (t.lo != 0.0) h[hi++] = t.lo;
    }
    if (q != 0.0 || hi == 0) h[hi++] = q;
    return hi;
}

// h = b * e (scale_expansion with zero elimination); returns the length (<= 2 elen)
SCVT_HD int exp_scale(int elen, const double* e, double b, double* h) {
    DD p = dd_two_prod(e[0], b);
    double q = p.hi;
    int hi = 0;
    if (p.lo != 0.0) h[hi++] = p.lo;
    for (int k = 1; k < elen; ++k) {
        DD pk = dd_two_prod(e[k], b);
        DD s = dd_two_sum(q, pk.lo);
        if (s.lo != 0.0) h[hi++] = s.lo;
        DD t = dd_two_sum(pk.hi, s.hi);       // |pk.hi| >= |s.hi|: exact either way
        if (t.lo != 0.0) h[hi++] = t.lo;
        q = t.hi;
    }
    if (q != 0.0 || hi == 0) h[hi++] = q;
    return hi;
}

SCVT_HD double exp_sign(int len, const double* e) {
    for (int k = len - 1; k >= 0; --k)
        if (e[k] != 0.0) return e[k];
    return 0.0;
}

// exact [p, q, r] = p.(q x r) as an expansion (<= 24 terms)
SCVT_HD int exp_det3(V3 p, V3 q, V3 r, double* out) {
    const double px[3] = {p.x, p.y, p.z}, qx[3] = {q.x, q.y, q.z}, rx[3] = {r.x, r.y, r.z};
    const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 2, 0}, {1, 0, 2}, {2, 0, 1}, {2, 1, 0}};
    const double sg[6] = {1, -1, 1, -1, 1, -1};
    double acc[24], tmp[24];
    int n = 0;
    for (int t = 0; t < 6; ++t) {
        DD qr = dd_two_prod(qx[perm[t][1]], rx[perm[t][2]]);
        const double e2[2] = {qr.lo, qr.hi};
        double term[4];
        int tl = e2[0] != 0.0 ? exp_scale(2, e2, sg[t] * px[perm[t][0]], term)
                              : exp_scale(1, e2 + 1, sg[t] * px[perm[t][0]], term);
        if (n == 0) {
            for (int k = 0; k < tl; ++k) acc[k] = term[k];
            n = tl;
        } else {
            n = exp_sum(n, acc, tl, term, tmp);
            for (int k = 0; k < n; ++k) acc[k] = tmp[k];
        }
    }
    for (int k = 0; k < n; ++k) out[k] = acc[k];
    return n;
}

// sign of s1 * A + s2 * B + s3 * C + s4 * D over exact expansions (signs +-1 or 0)
SCVT_HD int exp_combine_sign(const double* const* x, const int* len, const double* sg) {
    double acc[96], tmp[96], neg[24];
    int n = 0;
    for (int t = 0; t < 4; ++t) {
        if (sg[t] == 0.0) continue;
        for (int k = 0; k < len[t]; ++k) neg[k] = sg[t] * x[t][k];
        if (n == 0) {
            for (int k = 0; k < len[t]; ++k) acc[k] = neg[k];
            n = len[t];
        } else {
            n = exp_sum(n, acc, len[t], neg, tmp);
            for (int k = 0; k < n; ++k) acc[k] = tmp[k];
        }
    }
    const double v = n ? exp_sign(n, acc) : 0.0;
    return v > 0.0 ? 1 : (v < 0.0 ? -1 : 0);
}

// tiers 1-2.  io < 0 marks o as the (unperturbed) origin.
// inline: a call site in the certificate / cell kernels costs them ~15 % through the call
// ABI's register constraints (k_verify 282 vs 211 us per c4 iteration); the expansion
// buffers live in local memory and are touched only on this path
SCVT_HD int orient_exact_sos(V3 o, V3 a, V3 b, V3 c, int io, int ia, int ib, int ic, int* tier) {
    double t1[24], t2[24], t3[24], t4[24];
    const int l1 = exp_det3(a, b, c, t1), l2 = exp_det3(o, b, c, t2);
    const int l3 = exp_det3(a, o, c, t3), l4 = exp_det3(a, b, o, t4);
    const double* x[4] = {t1, t2, t3, t4};
    const int len[4] = {l1, l2, l3, l4};
    const double sd[4] = {1, -1, -1, -1};
    const int s = exp_combine_sign(x, len, sd);
    if (s) { *tier = 1; return s; }
    *tier = 2;
    // E_p for the points in increasing index order (the origin is never perturbed)
    const int idx[4] = {io, ia, ib, ic};
    const double se[4][4] = {{0, -1, -1, -1},    // E_o
                             {1, 0, -1, -1},     // E_a
                             {1, -1, 0, -1},     // E_b
                             {1, -1, -1, 0}};    // E_c
    bool used[4] = {false, false, false, false};
    for (int step = 0; step < 4; ++step) {
        int w = -1;
        for (int k = 0; k < 4; ++k)
            if (!used[k] && idx[k] >= 0 && (w < 0 || idx[k] < idx[w])) w = k;
        if (w < 0) break;
        used[w] = true;
        const int e = exp_combine_sign(x, len, se[w]);
        if (e) return e;
    }
    return 1;
}

// FP64 value + static filter; returns sign or 0 when undecided
SCVT_HD int orient_filter(V3 o, V3 a, V3 b, V3 c) {
    V3 ao = sub(a, o), bo = sub(b, o), co = sub(c, o);
    double m1 = bo.y * co.z, m2 = bo.z * co.y;
    double m3 = bo.z * co.x, m4 = bo.x * co.z;
    double m5 = bo.x * co.y, m6 = bo.y * co.x;
    double det = ao.x * (m1 - m2) + ao.y * (m3 - m4) + ao.z * (m5 - m6);
    double perm = fabs(ao.x) * (fabs(m1) + fabs(m2)) + fabs(ao.y) * (fabs(m3) + fabs(m4)) +
                  fabs(ao.z) * (fabs(m5) + fabs(m6));
    const double eps = 1.1102230246251565e-16;   // 2^-53
    double bound = (16.0 * eps) * perm;          // differences carry rounding too
    if (det > bound) return 1;
    if (det < -bound) return -1;
    return 0;
}

// Robust sign of det[a-o, b-o, c-o] with SoS tie-breaking; *tier = 0/1/2 (filter/exact/sos)
SCVT_HD int orient_robust(V3 o, V3 a, V3 b, V3 c, int io, int ia, int ib, int ic, int* tier) {
    int s = orient_filter(o, a, b, c);
    if (s) { *tier = 0; return s; }
    return orient_exact_sos(o, a, b, c, io, ia, ib, ic, tier);
}

// Sign without tie-breaking (0 for an exact tie) and whether the FP64 filter was undecided.
SCVT_HD int insphere_sign(V3 o, V3 a, V3 b, V3 c, bool* ambiguous) {
    int s = orient_filter(o, a, b, c);
    *ambiguous = s == 0;
    if (s) return s;
    int tier;
    s = orient_exact_sos(o, a, b, c, 0, 1, 2, 3, &tier);
    return tier == 2 ? 0 : s;
}

// ------------------------------------------------------------------ Voronoi cell clipping
// The spherical Voronoi cell of z_i is the cone {x : x.(z_j - z_i) <= 0 for all j}.  In the
// gnomonic plane x = z_i + u1 e1 + u2 e2 each neighbour contributes the half-plane
// u.d <= |d|^2 / 2 with d = z_j - z_i (well conditioned for close pairs).  The polygon's
// edge labels in CCW order are the Delaunay neighbours of i in CCW order seen from outside,
// so (i, n_t, n_{t+1}) are exactly the CCW-outward hull facets at i (the triangles Qhull
// returns through convex_hull_delaunay, delaunay.py:181-202).  A polygon vertex between
// edges labelled l and r is the circumcentre of (i, l, r); whether a new neighbour j cuts it
// is the in-circle test of j against (i, l, r), decided by `orient_robust` whenever the
// FP64 value of the half-plane test falls inside its rounding band.
struct Poly {
    int n;
    double ax[MAXV], ay[MAXV], b[MAXV];   // edge k line: ax*u + ay*v <= b
    double vx[MAXV], vy[MAXV];            // vertex k = start of edge k
    int lab[MAXV];                        // neighbour id, -1 for the initial box
};

SCVT_HD void poly_init(Poly& P) {
    const double L = BOX_L;
    // CCW: bottom (v >= -L), right (u <= L), top (v <= L), left (u >= -L)
    P.n = 4;
    P.ax[0] = 0;  P.ay[0] = -1; P.b[0] = L; P.vx[0] = -L; P.vy[0] = -L; P.lab[0] = -1;
    P.ax[1] = 1;  P.ay[1] = 0;  P.b[1] = L; P.vx[1] = L;  P.vy[1] = -L; P.lab[1] = -1;
    P.ax[2] = 0;  P.ay[2] = 1;  P.b[2] = L; P.vx[2] = L;  P.vy[2] = L;  P.lab[2] = -1;
    P.ax[3] = -1; P.ay[3] = 0;  P.b[3] = L; P.vx[3] = -L; P.vy[3] = L;  P.lab[3] = -1;
}

SCVT_HD void line_meet(double a1x, double a1y, double b1, double a2x, double a2y, double b2,
                       double* x, double* y) {
    double det = a1x * a2y - a1y * a2x;
    double inv = fast_rcp(det);
    *x = (b1 * a2y - b2 * a1y) * inv;
    *y = (a1x * b2 - a2x * b1) * inv;
}

// squared chord between z_i and the sphere point above gnomonic vertex (x, y)
SCVT_HD double vertex_chord2(double x, double y) {
    double q = x * x + y * y;
    double s = sqrt(1.0 + q);
    return 2.0 * q / (s * (s + 1.0));
}

struct ClipCtx {
    const double* z;   // (n,3) generator coordinates by id
    V3 zi;
    int i;
    int tie_breaks;    // count of SoS decisions
};

// Clip by a.u <= b (label j, position zj).  Returns 0 = unchanged, 1 = clipped, <0 = error.
SCVT_HD int poly_clip(Poly& P, Poly& T, double ax, double ay, double b, int j, V3 zj,
                      ClipCtx& cc) {
    int n = P.n;
    bool out[MAXV];
    int nout = 0;
    for (int k = 0; k < n; ++k) {
        double t1 = ax * P.vx[k], t2 = ay * P.vy[k];
        double s = t1 + t2 - b;
        double tol = 1e-9 * (fabs(t1) + fabs(t2) + b);
        bool o;
        if (s > tol) o = true;
        else if (s < -tol) o = false;
        else {
            int km = k == 0 ? n - 1 : k - 1;
            int l = P.lab[km], r = P.lab[k];
            if (l >= 0 && r >= 0) {
                int tier;
                o = orient_robust(cc.zi, load3(cc.z, l), load3(cc.z, r), zj, cc.i, l, r, j,
                                  &tier) > 0;
                cc.tie_breaks += tier == 2;
            } else {
                o = s > 0.0;
            }
        }
        out[k] = o;
        nout += o;
    }
    if (nout == 0) return 0;
    if (nout == n) return -1;                 // empty: cannot happen for a true cell
    int first = -1, last = -1, runs = 0;
    for (int k = 0; k < n; ++k) {
        int km = k == 0 ? n - 1 : k - 1;
        int kp = k == n - 1 ? 0 : k + 1;
        if (out[k] && !out[km]) { first = k; ++runs; }
        if (out[k] && !out[kp]) last = k;
    }
    if (runs != 1 || first < 0 || last < 0) return -2;   // non-convex decision pattern
    int ein = first == 0 ? n - 1 : first - 1;    // edge entering the outside run
    double Ax, Ay, Bx, By;
    line_meet(P.ax[ein], P.ay[ein], P.b[ein], ax, ay, b, &Ax, &Ay);
    line_meet(ax, ay, b, P.ax[last], P.ay[last], P.b[last], &Bx, &By);
    // surviving edges: last, last+1, ..., ein (cyclic), then the new edge
    int m = 0;
    int k = last;
    while (true) {
        if (m >= MAXV - 1) return -3;
        T.ax[m] = P.ax[k]; T.ay[m] = P.ay[k]; T.b[m] = P.b[k]; T.lab[m] = P.lab[k];
        if (k == last) { T.vx[m] = Bx; T.vy[m] = By; }
        else { T.vx[m] = P.vx[k]; T.vy[m] = P.vy[k]; }
        ++m;
        if (k == ein) break;
        k = k == n - 1 ? 0 : k + 1;
    }
    T.ax[m] = ax; T.ay[m] = ay; T.b[m] = b; T.lab[m] = j; T.vx[m] = Ax; T.vy[m] = Ay;
    ++m;
    T.n = m;
    return 1;
}

SCVT_HD double poly_max_chord2(const Poly& P, bool* has_box) {
    double r2 = 0.0;
    bool box = false;
    for (int k = 0; k < P.n; ++k) {
        r2 = fmax(r2, vertex_chord2(P.vx[k], P.vy[k]));
        box |= P.lab[k] < 0;
    }
    *has_box = box;
    return r2;
}

// Tangent frame at z (seed = least aligned axis; e1 x e2 = z, right-handed).
SCVT_HD void tangent_frame(V3 z, V3* e1, V3* e2) {
    double ax = fabs(z.x), ay = fabs(z.y), az = fabs(z.z);
    V3 seed = (ax <= ay && ax <= az) ? v3(1, 0, 0) : (ay <= az ? v3(0, 1, 0) : v3(0, 0, 1));
    V3 t = cross(z, seed);
    t = mul(t, 1.0 / norm3(t));
    *e1 = t;
    *e2 = cross(z, t);
}

struct GridView {
    const double* zs;       // (n,4) positions sorted by bucket (x,y,z,pad)
    const int* ids;         // (n,) original id of sorted slot
    const int* start;       // (6G^2+1) bucket start offsets into the sorted arrays
    const double* z;        // (n,3) positions by id
    int G;
    int64_t n;
};

constexpr int CAND = 48;    // nearest-first candidate list per pass

struct CellStats { int rounds; int passes; int tie_breaks; int sweep_visits; int scanned; int cands; int clips; };

// Build the Voronoi cell of generator i by nearest-first half-plane clipping with a
// security-radius certificate: a point j can cut the cell only if |z_j - z_i| < 2R with R
// the largest vertex chord, so once every point within r >= 2R is processed the cell is
// final.  Writes the CCW neighbour cycle rotated so its smallest id leads; returns the
// valence (>0) or -status.
SCVT_HD int build_cell(const GridView& g, int i, V3 zi, int* nbr_out, CellStats* st,
                       Poly& P, Poly& T) {
    V3 e1, e2;
    tangent_frame(zi, &e1, &e2);
    poly_init(P);
    Poly* cur = &P;
    Poly* tmp = &T;
    ClipCtx cc;
    cc.z = g.z; cc.zi = zi; cc.i = i; cc.tie_breaks = 0;
    uint32_t key = bucket_key(zi, g.G);
    int cnt = g.start[key + 1] - g.start[key];
    double area_b = 4.0 * M_PI / (6.0 * (double)g.G * (double)g.G);
    double h = sqrt(area_b / (double)(cnt > 0 ? cnt : 1));
    double r2 = 9.0 * h * h;                  // first pass radius 3h
    if (r2 > 4.0) r2 = 4.0000001;
    double lo_c2 = -1.0;                      // exclusive lower bound (c2, id)
    int lo_id = 0x7fffffff;
    double R2 = 8.0;                          // current max vertex chord^2 (box => all)
    bool box = true;
    int status = 0;
    int rounds = 0, passes = 0;
    double cd[CAND];
    int cid[CAND], cp[CAND];
    while (true) {
        ++passes;
        if (passes > 4096) { status |= ST_POLY_OVERFLOW; break; }
        int m = 0;
        bool overflow = false;
        double lim = 4.0 * R2 * (1.0 + 1e-12);
        CapBox cb = cap_box(zi, sqrt(r2));
        for (int face = 0; face < 6; ++face) {
            int iu0, iu1, iv0, iv1;
            if (!cap_face_range(cb, face, g.G, &iu0, &iu1, &iv0, &iv1)) continue;
            for (int iu = iu0; iu <= iu1; ++iu) {
                int rowbase = (face * g.G + iu) * g.G;
                int p0 = g.start[rowbase + iv0], p1 = g.start[rowbase + iv1 + 1];
                for (int p = p0; p < p1; ++p) {
                    int j = g.ids[p];
                    if (j == i) continue;
                    const double* q = g.zs + 4 * (int64_t)p;
                    double dx = q[0] - zi.x, dy = q[1] - zi.y, dz = q[2] - zi.z;
                    double c2 = dx * dx + dy * dy + dz * dz;
                    if (c2 > r2 || c2 >= lim) continue;
                    if (c2 < lo_c2 || (c2 == lo_c2 && j <= lo_id)) continue;
                    if (c2 == 0.0) { status |= ST_DUPLICATE; continue; }
                    // insert into the sorted list (key = (c2, j))
                    if (m == CAND) {
                        if (c2 > cd[m - 1] || (c2 == cd[m - 1] && j > cid[m - 1])) {
                            overflow = true;
                            continue;
                        }
                        overflow = true;
                        --m;
                    }
                    int t = m++;
                    while (t > 0 && (cd[t - 1] > c2 || (cd[t - 1] == c2 && cid[t - 1] > j))) {
                        cd[t] = cd[t - 1]; cid[t] = cid[t - 1]; cp[t] = cp[t - 1];
                        --t;
                    }
                    cd[t] = c2; cid[t] = j; cp[t] = p;
                }
            }
        }
        bool early = false;
        for (int t = 0; t < m; ++t) {
            if (cd[t] >= 4.0 * R2 * (1.0 + 1e-12)) { early = true; break; }
            const double* q = g.zs + 4 * (int64_t)cp[t];
            V3 zj = v3(q[0], q[1], q[2]);
            V3 d = sub(zj, zi);
            int rc = poly_clip(*cur, *tmp, dot(d, e1), dot(d, e2), 0.5 * cd[t], cid[t], zj, cc);
            if (rc < 0) { status |= ST_POLY_OVERFLOW; break; }
            if (rc == 1) {
                Poly* sw = cur; cur = tmp; tmp = sw;
                R2 = poly_max_chord2(*cur, &box);
                if (box) R2 = 8.0;
            }
        }
        if (status) break;
        if (overflow && !early) {
            // dense neighbourhood of a large cell: sweep the rest of the range unsorted
            ++passes;
            double klo = cd[m - 1];
            int kid = cid[m - 1];
            for (int face = 0; face < 6 && !status; ++face) {
                int iu0, iu1, iv0, iv1;
                if (!cap_face_range(cb, face, g.G, &iu0, &iu1, &iv0, &iv1)) continue;
                for (int iu = iu0; iu <= iu1 && !status; ++iu) {
                    int rowbase = (face * g.G + iu) * g.G;
                    int p0 = g.start[rowbase + iv0], p1 = g.start[rowbase + iv1 + 1];
                    for (int p = p0; p < p1; ++p) {
                        int j = g.ids[p];
                        if (j == i) continue;
                        const double* q = g.zs + 4 * (int64_t)p;
                        V3 zj = v3(q[0], q[1], q[2]);
                        V3 d = sub(zj, zi);
                        double c2 = dot(d, d);
                        if (c2 > r2 || c2 >= 4.0 * R2 * (1.0 + 1e-12)) continue;
                        if (c2 < klo || (c2 == klo && j <= kid)) continue;
                        if (c2 == 0.0) { status |= ST_DUPLICATE; continue; }
                        int rc = poly_clip(*cur, *tmp, dot(d, e1), dot(d, e2), 0.5 * c2, j, zj, cc);
                        if (rc < 0) { status |= ST_POLY_OVERFLOW; break; }
                        if (rc == 1) {
                            Poly* sw = cur; cur = tmp; tmp = sw;
                            R2 = poly_max_chord2(*cur, &box);
                            if (box) R2 = 8.0;
                        }
                    }
                }
            }
            if (status) break;
        }
        ++rounds;
        if (r2 >= 4.0) {
            if (box) status |= ST_UNBOUNDED;
            break;
        }
        if (!box && 4.0 * R2 * (1.0 + 1e-9) <= r2) break;   // security radius certified
        lo_c2 = r2;
        lo_id = 0x7fffffff;
        double want = box ? 4.0 * r2 : 4.0 * R2 * (1.0 + 1e-9);
        r2 = want >= 4.0 ? 4.0000001 : want;
    }
    st->rounds = rounds;
    st->passes = passes;
    st->tie_breaks = cc.tie_breaks;
    st->sweep_visits = 0;
    st->scanned = st->cands = st->clips = 0;
    if (status) return -status;
    int n = cur->n;
    if (n > MAXDEG) return -ST_DEG_OVERFLOW;
    int lead = 0;
    for (int k = 1; k < n; ++k)
        if (cur->lab[k] < cur->lab[lead]) lead = k;
    for (int k = 0; k < n; ++k) {
        int kk = lead + k;
        if (kk >= n) kk -= n;
        nbr_out[k] = cur->lab[kk];
    }
    return n;
}

// ------------------------------------------------------------------ density
enum DensityKind { DEN_CONST = 0, DEN_X3 = 1, DEN_X16 = 2, DEN_TANH = 3, DEN_TANH4 = 4,
                   DEN_TANH4X2 = 5,
                   // internal: tanh4 kinds evaluated through the rho^(1/4) table
                   DEN_TANH4_TAB = 6, DEN_TANH4X2_TAB = 7 };

constexpr int TAB_P = 6;   // polynomial degree of the rho^(1/4) table (SCVT_TABLE_DEGREE)

struct DensityParams {
    int kind;
    double gamma, beta, alpha;
    double c0x, c0y, c0z, c1x, c1y, c1z;
    double w_lon, w_lat;
    double lat_c, lon_c, cos_lat_c, sin_lat_c;   // x16 centre (precomputed on host)
    const double* tab;   // [2][tab_k][TAB_P+1] (shared memory inside the kernel)
    int tab_k;
    double tab_invw;
};

// u = rho^(1/4) of the tanh^4 profile from the table (density.tanh4_table): chord to the
// centre when d <= 90 deg, chord to its antipode otherwise; Horner in tau.
SCVT_HD double tab_u(const DensityParams& p, V3 y, V3 c) {
    // chord to the nearer of c and -c (|y - c|^2 = 2 - 2 y.c for unit vectors): a select,
    // not a predicated second chord
    const int br = dot(y, c) < 0.0;
    const double s = br ? -1.0 : 1.0;
    V3 dm = v3(y.x - s * c.x, y.y - s * c.y, y.z - s * c.z);
    double r2 = dot(dm, dm);
    double t = sqrt(r2) * p.tab_invw;
    int k = (int)t;
    if (k > p.tab_k - 1) k = p.tab_k - 1;
    double tau = 2.0 * (t - (double)k) - 1.0;
    const double* co = p.tab + (br * p.tab_k + k) * (TAB_P + 1);
#if defined(__CUDA_ARCH__)
    double acc = __ldg(co + TAB_P);      // the table lives in global memory (read-only cache)
#pragma unroll
    for (int j = TAB_P - 1; j >= 0; --j) acc = fma(acc, tau, __ldg(co + j));
#else
    double acc = co[TAB_P];
#pragma unroll
    for (int j = TAB_P - 1; j >= 0; --j) acc = fma(acc, tau, co[j]);
#endif
    return acc;
}

SCVT_HD double geodesic(V3 a, V3 b) { return atan2(norm3(cross(a, b)), dot(a, b)); }

// density.py:116-129 with the BASELINE variants; y is unit.  *pole set for x16 near poles.
template <int KIND>
SCVT_HD double density_eval(const DensityParams& p, V3 y, int* pole) {
    if (KIND == DEN_CONST) return 1.0;
    if (KIND == DEN_X3) {
        double z2 = y.z * y.z;
        return (1.0 - p.gamma) * (z2 * z2) + p.gamma;
    }
    if (KIND == DEN_TANH4_TAB || KIND == DEN_TANH4X2_TAB) {
        double u = tab_u(p, y, v3(p.c0x, p.c0y, p.c0z));
        if (KIND == DEN_TANH4X2_TAB) u = fmax(u, tab_u(p, y, v3(p.c1x, p.c1y, p.c1z)));
        double u2 = u * u;
        return u2 * u2;
    }
    if (KIND == DEN_TANH4 || KIND == DEN_TANH4X2) {
        double d = geodesic(y, v3(p.c0x, p.c0y, p.c0z));
        if (KIND == DEN_TANH4X2) d = fmin(d, geodesic(y, v3(p.c1x, p.c1y, p.c1z)));
        double t = 0.5 * (1.0 - p.gamma) * (tanh((p.beta - d) / p.alpha) + 1.0) + p.gamma;
        double t2 = t * t;
        return t2 * t2;
    }
    double d;
    if (KIND == DEN_X16) {
        // density.py:100-113 (elliptical distance)
        double horiz = hypot(y.x, y.y);
        if (horiz < 1e-9) *pole = 1;
        double lat_x = atan2(y.z, horiz), lon_x = atan2(y.y, y.x);
        double clx = cos(lat_x);
        V3 x_ic = v3(clx * cos(p.lon_c), clx * sin(p.lon_c), sin(lat_x));
        V3 x_ci = v3(p.cos_lat_c * cos(lon_x), p.cos_lat_c * sin(lon_x), p.sin_lat_c);
        double dl = geodesic(y, x_ic) / p.w_lon, dt = geodesic(y, x_ci) / p.w_lat;
        d = sqrt(dl * dl + dt * dt);
    } else {
        d = geodesic(y, v3(p.c0x, p.c0y, p.c0z));
    }
    return (tanh((p.beta - d) / p.alpha) + 1.0) / (2.0 * (1.0 - p.gamma)) + p.gamma;
}

// ------------------------------------------------------------------ fan geometry
// One incidence = (generator i, Delaunay triangle (i, j, k) CCW).  The two fan
// sub-triangles owned by i (delaunay.py:357-361) are (v_i, m_ij, oc) and (m_ki, v_i, oc);
// this holds for every rotation of the canonical (a, b, c).
struct SubTri { V3 v0, e1, e2; double area; };

struct FanPair {
    SubTri s[2];
    int obtuse;       // 1 if any of the triangle's 6 signed areas is negative (counted at min id)
    int degenerate;
};

SCVT_HD V3 planar_circumcenter(V3 a, V3 b, V3 c) {
    // geometry.py:105-119
    V3 ab = sub(b, a), ac = sub(c, a);
    V3 n = cross(ab, ac);
    double n2 = dot(n, n), ab2 = dot(ab, ab), ac2 = dot(ac, ac);
    V3 num = add(mul(cross(n, ab), ac2), mul(cross(ac, n), ab2));
    // one division, three products (the reference divides each component; the results agree
    // to an ulp, far inside the 1e-12 parity contract; FP64 divides are long MUFU+Newton chains)
    const double rden = 1.0 / (2.0 * n2);
    return add(a, mul(num, rden));
}

SCVT_HD double signed_area(V3 v0, V3 v1, V3 v2, V3 nhat) {
    return 0.5 * dot(cross(sub(v1, v0), sub(v2, v0)), nhat);
}

SCVT_HD FanPair fan_pair(V3 vi, V3 vj, V3 vk, int i, int j, int k) {
    // canonical rotation: min id first (delaunay.py:133-141); oc and n use that order
    V3 va, vb, vc;
    if (i < j && i < k) { va = vi; vb = vj; vc = vk; }
    else if (j < k) { va = vj; vb = vk; vc = vi; }
    else { va = vk; vb = vi; vc = vj; }
    FanPair f;
    V3 oc = planar_circumcenter(va, vb, vc);
    V3 n = cross(sub(vb, va), sub(vc, va));
    double nn = norm3(n);
    f.degenerate = !(nn > 0.0);
    n = mul(n, 1.0 / nn);
    if (dot(n, add(add(va, vb), vc)) < 0.0) n = mul(n, -1.0);
    V3 mij = mul(add(vi, vj), 0.5);
    V3 mki = mul(add(vk, vi), 0.5);
    f.s[0].v0 = vi;  f.s[0].e1 = sub(mij, vi); f.s[0].e2 = sub(oc, vi);
    f.s[0].area = signed_area(vi, mij, oc, n);
    f.s[1].v0 = mki; f.s[1].e1 = sub(vi, mki); f.s[1].e2 = sub(oc, mki);
    f.s[1].area = signed_area(mki, vi, oc, n);
    // obtuse flag for the whole triangle (delaunay.py:366-369): recompute all six areas
    V3 mjk = mul(add(vj, vk), 0.5);
    double a2 = signed_area(mij, vj, oc, n), a3 = signed_area(vj, mjk, oc, n);
    double a4 = signed_area(mjk, vk, oc, n), a5 = signed_area(vk, mki, oc, n);
    f.obtuse = (f.s[0].area < 0) | (f.s[1].area < 0) | (a2 < 0) | (a3 < 0) | (a4 < 0) | (a5 < 0);
    return f;
}

// One fan sub-triangle of the incidence (half 0: (v_i, m_ij, oc), half 1: (m_ki, v_i, oc)),
// without the other half's geometry; *obtuse (the triangle's six signed areas, as fan_pair)
// is computed for half 0 only.  Same arithmetic as fan_pair, so the same bits.
SCVT_HD SubTri fan_sub(V3 vi, V3 vj, V3 vk, int i, int j, int k, int half, int* obtuse,
                       int* degenerate) {
    V3 va, vb, vc;
    if (i < j && i < k) { va = vi; vb = vj; vc = vk; }
    else if (j < k) { va = vj; vb = vk; vc = vi; }
    else { va = vk; vb = vi; vc = vj; }
    const V3 oc = planar_circumcenter(va, vb, vc);
    V3 n = cross(sub(vb, va), sub(vc, va));
    const double nn = norm3(n);
    *degenerate = !(nn > 0.0);
    n = mul(n, 1.0 / nn);
    if (dot(n, add(add(va, vb), vc)) < 0.0) n = mul(n, -1.0);
    const V3 mij = mul(add(vi, vj), 0.5);
    const V3 mki = mul(add(vk, vi), 0.5);
    SubTri st;
    if (half == 0) {
        st.v0 = vi; st.e1 = sub(mij, vi); st.e2 = sub(oc, vi);
        st.area = signed_area(vi, mij, oc, n);
        const V3 mjk = mul(add(vj, vk), 0.5);
        const double a1 = signed_area(mki, vi, oc, n);
        const double a2 = signed_area(mij, vj, oc, n), a3 = signed_area(vj, mjk, oc, n);
        const double a4 = signed_area(mjk, vk, oc, n), a5 = signed_area(vk, mki, oc, n);
        *obtuse = (st.area < 0) | (a1 < 0) | (a2 < 0) | (a3 < 0) | (a4 < 0) | (a5 < 0);
    } else {
        st.v0 = mki; st.e1 = sub(vi, mki); st.e2 = sub(oc, mki);
        st.area = signed_area(mki, vi, oc, n);
        *obtuse = 0;
    }
    return st;
}

// Accumulate sum_q w_q rho(y_q) {1, y_q, |y_q - z|^2} over the composite nodes of one
// sub-triangle (cvt_core.py:80-100 with the subdivision of delaunay.py:383-407 folded into
// the node table).  acc = {m, cx, cy, cz, E}.
template <int KIND, bool SPHERE>
SCVT_HD void subtri_moments(const SubTri& s, V3 z, const double* l1, const double* l2,
                            const double* w, int nq, const DensityParams& dp, double* acc,
                            int* pole) {
    double m = 0.0, cx = 0.0, cy = 0.0, cz = 0.0, e = 0.0;
    double plane_d = 0.0;
    // (two independent nodes per iteration give the FP64 pipe ILP to hide its latency)
    if (SPHERE) {
        V3 nv = cross(s.e1, s.e2);
        double nn = norm3(nv);
        if (nn == 0.0) nn = 1.0;
        plane_d = fabs(dot(nv, s.v0) / nn);
    }
#pragma unroll 2
    for (int q = 0; q < nq; ++q) {
        double a = l1[q], b = l2[q];
        double x = s.v0.x + a * s.e1.x + b * s.e2.x;
        double y = s.v0.y + a * s.e1.y + b * s.e2.y;
        double zz = s.v0.z + a * s.e1.z + b * s.e2.z;
        double r2 = x * x + y * y + zz * zz;
        double inv = rsqrt_d(r2);
        V3 yv = v3(x * inv, y * inv, zz * inv);
        double rho = density_eval<KIND>(dp, yv, pole);
        if (SPHERE) rho *= plane_d * inv * inv * inv;
        double wr = w[q] * rho;
        m += wr;
        cx += wr * yv.x; cy += wr * yv.y; cz += wr * yv.z;
        V3 d = sub(yv, z);
        e += wr * dot(d, d);
    }
    acc[0] += s.area * m;
    acc[1] += s.area * cx; acc[2] += s.area * cy; acc[3] += s.area * cz;
    acc[4] += s.area * e;
}

// ------------------------------------------------------------------ symmetric 7-point fast path
// For a rule whose node set is invariant under permutations of the barycentric coordinates
// (Radon's 7-point rule, DECISIONS.md D1) the 4^d leaves of the depth-d subdivision form a
// regular grid with L = 2^d cells per side: up-leaves at (a, b), a+b <= L-1, with nodes
// P + o_q, and down-leaves at (a+1, b+1), a+b <= L-2, with nodes P - o_q, where
// o_q = nu1_q/L e1 + nu2_q/L e2 are the rule offsets of the first leaf.  Same node set and
// weights as the composite table (geometry.composite_nodes), cheaper per node: 3 adds to place
// it, no table loads.  rho^(1/4) table coefficients are cached per lane across nodes.
struct TabCache {
    int key;
    double c[TAB_P + 1];
};

SCVT_HD double tab_u_cached(const DensityParams& p, V3 x, double inv, V3 c, TabCache& tc) {
    const int br = dot(x, c) < 0.0;                 // sign of y.c (inv > 0)
    const double sx = br ? -c.x : c.x, sy = br ? -c.y : c.y, sz = br ? -c.z : c.z;
    const double dx = fma(x.x, inv, -sx), dy = fma(x.y, inv, -sy), dz = fma(x.z, inv, -sz);
    double r2 = fmax(dx * dx + dy * dy + dz * dz, 1e-300);
    const double t = r2 * fast_rsqrt(r2) * p.tab_invw;
    int k = (int)t;
    if (k > p.tab_k - 1) k = p.tab_k - 1;
    const double tau = 2.0 * (t - (double)k) - 1.0;
    const int key = br * p.tab_k + k;
    if (key != tc.key) {
        tc.key = key;
        const double* co = p.tab + key * (TAB_P + 1);
#pragma unroll
        for (int j = 0; j <= TAB_P; ++j) tc.c[j] = co[j];
    }
    double acc = tc.c[TAB_P];
#pragma unroll
    for (int j = TAB_P - 1; j >= 0; --j) acc = fma(acc, tau, tc.c[j]);
    return acc;
}

// ---- per-sub-triangle local fit of u = rho^(1/4) in s = |y - sigma c|^2 (no sqrt per node)
// exact table value of u at chord x in branch br
SCVT_HD double tab_u_chord(const DensityParams& p, double x, int br) {
    const double t = x * p.tab_invw;
    int k = (int)t;
    if (k > p.tab_k - 1) k = p.tab_k - 1;
    const double tau = 2.0 * (t - (double)k) - 1.0;
    const double* co = p.tab + (br * p.tab_k + k) * (TAB_P + 1);
#if defined(__CUDA_ARCH__)
    double acc = __ldg(co + TAB_P);      // the table lives in global memory (read-only cache)
#pragma unroll
    for (int j = TAB_P - 1; j >= 0; --j) acc = fma(acc, tau, __ldg(co + j));
#else
    double acc = co[TAB_P];
#pragma unroll
    for (int j = TAB_P - 1; j >= 0; --j) acc = fma(acc, tau, co[j]);
#endif
    return acc;
}

constexpr double FIT_NOISE = 4e-15;   // rounding floor of rho = (table u)^4, relative

struct LocalFit {
    double sc;          // centre of the s interval
    double b[7];        // rho(s) = sum_k b[k] (s - sc)^k
    V3 sgc;             // sigma * c
    double rmin, rmax;  // bounds of rho on the patch (table values at the s-interval ends:
                        // rho is monotone in s on one branch)
};

// Fit rho = u^4 over the patch of sub-triangle `st` (nodes y = normalize(v0 + l1 e1 + l2 e2)).
// Returns false (caller falls back to per-node table evaluation) when the patch straddles
// 90 deg from c, comes too close to the sqrt singularity at s = 0, or the fit misses the table
// by more than 4e-15 relative at any check point (the table itself is within 1.6e-15 of the
// closed form; a degree-6 interpolant evaluated in FP64 has a ~1e-15 rounding floor).
// BOUNDS: also record rho at the ends of the s interval (f.rmin, f.rmax: read only by the
// two-centre dominance test; two table evaluations the single-centre kernels skip).
template <bool BOUNDS = true>
SCVT_HD bool local_fit_impl(const DensityParams& p, const SubTri& st, V3 c, LocalFit& f,
                            int* drop = nullptr, double* tail_stats = nullptr) {
    constexpr double CHEB_V[7] = {0.9749279121818236, 0.7818314824680298, 0.4338837391175582,
                              6.123233995736766e-17, -0.43388373911755806, -0.7818314824680295,
                              -0.9749279121818237};
    constexpr double CHEB_A[7][7] = {
    {0.14285714285714285, 0.14285714285714285, 0.14285714285714285, 0.14285714285714285, 0.14285714285714285, 0.14285714285714285, 0.14285714285714285},
    {0.2785508320519496, 0.2233804235622942, 0.12396678260501662, 1.7494954273533617e-17, -0.12396678260501659, -0.22338042356229412, -0.27855083205194964},
    {0.2574196765435483, 0.06357740970180413, -0.17813994338820957, -0.2857142857142857, -0.17813994338820963, 0.06357740970180381, 0.25741967654354836},
    {0.2233804235622942, -0.12396678260501659, -0.2785508320519496, -5.248486282060085e-17, 0.2785508320519496, 0.12396678260501715, -0.22338042356229448},
    {0.1781399433882096, -0.2574196765435483, -0.06357740970180416, 0.2857142857142857, -0.06357740970180402, -0.2574196765435486, 0.17813994338820988},
    {0.12396678260501662, -0.2785508320519496, 0.22338042356229418, 8.747477136766808e-17, -0.2233804235622943, 0.2785508320519494, -0.12396678260501692},
    {0.06357740970180413, -0.17813994338820963, 0.25741967654354836, -0.2857142857142857, 0.25741967654354825, -0.17813994338820863, 0.06357740970180491},
};

    const V3 P[3] = {st.v0, add(st.v0, st.e1), add(st.v0, st.e2)};
    double tk[3];
    for (int k = 0; k < 3; ++k) tk[k] = dot(P[k], c);
    int br;
    if (tk[0] > 0.0 && tk[1] > 0.0 && tk[2] > 0.0) br = 0;
    else if (tk[0] < 0.0 && tk[1] < 0.0 && tk[2] < 0.0) br = 1;
    else return false;
    const double sg = br ? -1.0 : 1.0;
    f.sgc = mul(c, sg);
    double smin = 1e300, smax = -1e300;
    for (int k = 0; k < 3; ++k) {
        const double inv = fast_rsqrt(dot(P[k], P[k]));
        const V3 d = sub(mul(P[k], inv), f.sgc);
        const double sk = dot(d, d);
        smin = fmin(smin, sk);
        smax = fmax(smax, sk);
    }
    // radial lift bends s by at most ~h^2/4 inside the patch; widen generously
    const double h2 = fmax(fmax(dot(st.e1, st.e1), dot(st.e2, st.e2)), dot(sub(st.e1, st.e2), sub(st.e1, st.e2)));
    const double margin = 2.0 * h2 + 1e-3 * (smax - smin);
    const double lo = smin - margin, hi = smax + margin;
    if (!(lo > 0.0)) return false;
    const double hw = 0.5 * (hi - lo), sc = 0.5 * (hi + lo);
    if (hw > 0.1 * sc) return false;            // hopeless near the s = 0 singularity; the
                                                // check points below are the accuracy guard
    double u[7];   // rho = (table u)^4 at the Chebyshev points: the fit is of rho itself
#pragma unroll
    for (int j = 0; j < 7; ++j) {
        const double sj = fma(hw, CHEB_V[j], sc);
        const double uj = tab_u_chord(p, sj * fast_rsqrt(sj), br);
        const double u2 = uj * uj;
        u[j] = u2 * u2;
    }
    double a[7];
#pragma unroll
    for (int m = 0; m < 7; ++m) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 7; ++j) acc = fma(CHEB_A[m][j], u[j], acc);
        a[m] = acc;
    }
    // a-posteriori truncation estimate from the Chebyshev tail: the coefficients of a
    // function analytic on the interval decay geometrically, so with the decay ratio r of
    // the last coefficients above the rounding floor of the table values (~4e-15 relative)
    // the omitted a7, a8, ... sum to ~|a_last| r^k / (1 - r).  A patch is accepted only when
    // that estimate is below the fit tolerance -- in addition to the check points below.
    {
        double umin = u[0];
#pragma unroll
        for (int j = 1; j < 7; ++j) umin = fmin(umin, u[j]);
        const double a4 = fabs(a[4]), a5 = fabs(a[5]), a6 = fabs(a[6]);
        const double noise = FIT_NOISE * umin, tol = 1.6e-14 * umin;
        // division-free: with r <= 1/2, 1 / (1 - r) <= 2
        bool ok = true;
        if (a6 > noise)                         // a7 ~ a6 r, r = max(a6/a5, a5/a4)
            ok = a6 <= 0.5 * a5 && a5 <= 0.5 * a4 && 2.0 * a6 * a6 <= tol * a5 &&
                 2.0 * a6 * a5 <= tol * a4;
        else if (a5 > noise)                    // a7 ~ a5 r^2, r = a5/a4
            ok = a5 <= 0.5 * a4 && 2.0 * a5 * a5 * a5 <= tol * a4 * a4;
        if (!ok) return false;
    }
    // degree selection: |T_k| <= 1 on the interval, so dropping the last Chebyshev terms
    // moves the polynomial by at most the sum of their magnitudes anywhere on the patch.  At
    // the rounding floor of the table values (FIT_NOISE relative: the same floor the tail
    // estimate above uses) a6, or a5 and a6, carry no information about rho -- they follow the
    // table's rounding noise -- and are set to zero EXACTLY (b6 = 0, or b5 = b6 = 0 below); a
    // warp whose patches all qualify evaluates the fit from b5 or b4 down: one or two steps
    // less on every node's dependent chain.  A degree-6 Horner evaluation of such a fit gives
    // the same bits (0 * s + b5 = b5), so the result of a patch does not depend on which
    // sweep its warp takes (sharded and single-GPU runs group the patches differently).
    {
        double umin = u[0];
#pragma unroll
        for (int j = 1; j < 7; ++j) umin = fmin(umin, u[j]);
        if (tail_stats) {
            tail_stats[0] = fabs(a[6]) / umin;
            tail_stats[1] = (fabs(a[6]) + fabs(a[5])) / umin;
            tail_stats[2] = (fabs(a[6]) + fabs(a[5]) + fabs(a[4])) / umin;
            tail_stats[3] = (fabs(a[6]) + fabs(a[5]) + fabs(a[4]) + fabs(a[3])) / umin;
        }
        const double a5 = fabs(a[5]), a6 = fabs(a[6]);
        int d = 0;
        if (a6 <= FIT_NOISE * umin) {
            d = 1;
            a[6] = 0.0;
            if (a5 + a6 <= FIT_NOISE * umin) {
                d = 2;
                a[5] = 0.0;
            }
        }
        if (drop) *drop = d;
    }
    double b[7];   // monomials in v = (s - sc) / hw
    b[0] = a[0] - a[2] + a[4] - a[6];
    b[1] = a[1] - 3.0 * a[3] + 5.0 * a[5];
    b[2] = 2.0 * a[2] - 8.0 * a[4] + 18.0 * a[6];
    b[3] = 4.0 * a[3] - 20.0 * a[5];
    b[4] = 8.0 * a[4] - 48.0 * a[6];
    b[5] = 16.0 * a[5];
    b[6] = 32.0 * a[6];
    const double vchk[3] = {0.995, -0.995, 0.21};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const double v = vchk[q];
        double pv = b[6];
#pragma unroll
        for (int k = 5; k >= 0; --k) pv = fma(pv, v, b[k]);
        const double sq = fma(hw, v, sc);
        const double eu = tab_u_chord(p, sq * fast_rsqrt(sq), br);
        const double e2 = eu * eu, ex = e2 * e2;
        if (!(fabs(pv - ex) <= 1.6e-14 * ex)) return false;   // = 4e-15 on u = rho^(1/4)
    }
    const double ih = 1.0 / hw;
    double sc_k = 1.0;
#pragma unroll
    for (int k = 0; k < 7; ++k) { f.b[k] = b[k] * sc_k; sc_k *= ih; }
    f.sc = sc;
    if (BOUNDS) {
        const double ul = tab_u_chord(p, lo * fast_rsqrt(lo), br), uh = tab_u_chord(p, hi * fast_rsqrt(hi), br);
        const double rl = (ul * ul) * (ul * ul), rh = (uh * uh) * (uh * uh);
        f.rmin = fmin(rl, rh);
        f.rmax = fmax(rl, rh);
    }
    return true;
}

SCVT_COLD bool local_fit(const DensityParams& p, const SubTri& st, V3 c, LocalFit& f) {
    return local_fit_impl(p, st, c, f);
}

SCVT_HD double fit_u(const LocalFit& f, V3 x, double inv) {
    const double dx = fma(x.x, inv, -f.sgc.x), dy = fma(x.y, inv, -f.sgc.y),
                 dz = fma(x.z, inv, -f.sgc.z);
    const double ds = (dx * dx + dy * dy + dz * dz) - f.sc;
    double acc = f.b[6];
#pragma unroll
    for (int k = 5; k >= 0; --k) acc = fma(acc, ds, f.b[k]);
    return acc;
}

template <int KIND>
SCVT_HD double density_x(const DensityParams& dp, V3 x, double inv, TabCache& t0, TabCache& t1,
                         int* pole) {
    if (KIND == DEN_CONST) return 1.0;
    if (KIND == DEN_TANH4_TAB || KIND == DEN_TANH4X2_TAB) {
        double u = tab_u_cached(dp, x, inv, v3(dp.c0x, dp.c0y, dp.c0z), t0);
        if (KIND == DEN_TANH4X2_TAB) u = fmax(u, tab_u_cached(dp, x, inv, v3(dp.c1x, dp.c1y, dp.c1z), t1));
        const double u2 = u * u;
        return u2 * u2;
    }
    return density_eval<KIND>(dp, v3(x.x * inv, x.y * inv, x.z * inv), pole);
}

// Leaf sweep of one sub-triangle; FIT selects the per-patch fit (loop-invariant, so the two
// density paths are separate loops: the table path's per-lane caches are not live in the
// fitted loop).
// part / nparts: the share of the leaves this call sweeps -- pass = part & 1 and the leaf rows
// a = part >> 1 (mod nparts / 2) when nparts > 1 (k_quad_table splits a sub-triangle over four
// lanes); everything with the defaults.
template <int KIND, int L, bool FIT>
SCVT_COLD void sym7_leaves(const SubTri& s, V3 z, const V3* o, double w0, double w1, double w2,
                         const DensityParams& dp, const LocalFit& f0, const LocalFit& f1,
                         double* mo, int* pole, int part = 0, int nparts = 1) {
    TabCache t0, t1;
    if (!FIT) { t0.key = -1; t1.key = -1; }
    double m = 0.0, cx = 0.0, cy = 0.0, cz = 0.0, e = 0.0;
    const double invL = 1.0 / (double)L;
    const int pass_lo = nparts > 1 ? (part & 1) : 0, pass_hi = nparts > 1 ? pass_lo + 1 : 2;
    const int a_lo = nparts > 1 ? (part >> 1) : 0, a_step = nparts > 1 ? nparts / 2 : 1;
    for (int pass = pass_lo; pass < pass_hi; ++pass) {          // 0: up-leaves, 1: down-leaves
    const double sg = pass ? -1.0 : 1.0;
    const int M = L - pass;
    for (int a = a_lo; a < M; a += a_step)
    for (int b = 0; b < M - a; ++b) {
        const double fa = (a + pass) * invL, fb = (b + pass) * invL;
        const V3 P = v3(s.v0.x + fa * s.e1.x + fb * s.e2.x, s.v0.y + fa * s.e1.y + fb * s.e2.y,
                        s.v0.z + fa * s.e1.z + fb * s.e2.z);
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            const V3 x = v3(fma(sg, o[q].x, P.x), fma(sg, o[q].y, P.y), fma(sg, o[q].z, P.z));
            const double r2 = x.x * x.x + x.y * x.y + x.z * x.z;
            const double inv = fast_rsqrt(r2);
            double rho;
            if (FIT) {
                rho = fit_u(f0, x, inv);                        // the fit is of rho = u^4
                if (KIND == DEN_TANH4X2_TAB) rho = fmax(rho, fit_u(f1, x, inv));
            } else {
                rho = density_x<KIND>(dp, x, inv, t0, t1, pole);
            }
            const double wr = (q == 0 ? w0 : (q < 4 ? w1 : w2)) * rho;
            const double wri = wr * inv;
            m += wr;
            cx = fma(wri, x.x, cx); cy = fma(wri, x.y, cy); cz = fma(wri, x.z, cz);
            const double dx = fma(x.x, inv, -z.x), dy = fma(x.y, inv, -z.y), dz = fma(x.z, inv, -z.z);
            e = fma(wr, dx * dx + dy * dy + dz * dz, e);
        }
    }
    }
    mo[0] = m; mo[1] = cx; mo[2] = cy; mo[3] = cz; mo[4] = e;
}

// Fitted-density sweep, rule node outermost: for node q of every leaf,
//   x = v0 + ((a+pass)/L + sg l1_q) e1 + ((b+pass)/L + sg l2_q) e2 = row_base(a) + (b/L) e2,
// so a node costs 3 FMA to place (the leaf-outer loop recomputes o_q, which does not fit in
// registers), the rule weight is applied once per q, and with the patch's fit of rho in
// s = |y - sigma c|^2 = 2 - 2 y.(sigma c) (|y| = |c| = 1):  s - sc = (2 - sc) + inv x.(-2 sigma c).
// SERIES: 1/|x| = (1 - delta)^(-1/2) = 1 + delta/2 + 3 delta^2/8 + 5 delta^3/16 with
// delta = 1 - |x|^2 <= 1e-4 on the patch (truncation <= 35/128 delta^4 < 3e-17), else the
// MUFU seed + cubic refinement.  31 FP64 instructions per node (one centre).
struct FitEval {
    double b[7];   // rho = sum_k b[k] ds^k
    V3 m2c;        // -2 sigma c
    double k0;     // 2 - sc
};

SCVT_HD FitEval fit_eval(const LocalFit& f) {
    FitEval r;
#pragma unroll
    for (int k = 0; k < 7; ++k) r.b[k] = f.b[k];
    r.m2c = mul(f.sgc, -2.0);
    r.k0 = 2.0 - f.sc;
    return r;
}

SCVT_HD double fit_rho(const FitEval& f, V3 x, double inv) {
    const double t = x.x * f.m2c.x + x.y * f.m2c.y + x.z * f.m2c.z;
    const double ds = fma(inv, t, f.k0);
    double acc = f.b[6];
#pragma unroll
    for (int k = 5; k >= 0; --k) acc = fma(acc, ds, f.b[k]);
    return acc;
}

// DEG: the fit's degree (6, or 5 / 4 when its last coefficients are exact zeros)
template <int DEG = 6>
SCVT_HD void fit_rho2(const FitEval& f, V3 x0, double inv0, V3 x1, double inv1, double* r0,
                      double* r1) {
    const double t0 = fma(x0.z, f.m2c.z, fma(x0.y, f.m2c.y, x0.x * f.m2c.x));
    const double t1 = fma(x1.z, f.m2c.z, fma(x1.y, f.m2c.y, x1.x * f.m2c.x));
    const double s0 = fma(inv0, t0, f.k0), s1 = fma(inv1, t1, f.k0);
    double a0 = f.b[DEG], a1 = f.b[DEG];
#pragma unroll
    for (int k = DEG - 1; k >= 0; --k) { a0 = fma(a0, s0, f.b[k]); a1 = fma(a1, s1, f.b[k]); }
    *r0 = a0; *r1 = a1;
}

// as fit_rho2 / fit_rho with t = x.(-2 sigma c) supplied by the caller
template <int DEG = 6>
SCVT_HD void fit_rho2_t(const FitEval& f, double t0, double inv0, double t1, double inv1,
                        double* r0, double* r1) {
    const double s0 = fma(inv0, t0, f.k0), s1 = fma(inv1, t1, f.k0);
    double a0 = f.b[DEG], a1 = f.b[DEG];
#pragma unroll
    for (int k = DEG - 1; k >= 0; --k) { a0 = fma(a0, s0, f.b[k]); a1 = fma(a1, s1, f.b[k]); }
    *r0 = a0; *r1 = a1;
}

SCVT_HD double fit_rho_t(const FitEval& f, double t, double inv) {
    const double ds = fma(inv, t, f.k0);
    double acc = f.b[6];
#pragma unroll
    for (int k = 5; k >= 0; --k) acc = fma(acc, ds, f.b[k]);
    return acc;
}

template <int KIND, int L, bool SERIES>
SCVT_HD void sym7_fit_leaves(const SubTri& s, V3 z, const double* l1, const double* l2,
                             const double* w, const LocalFit& lf0, const LocalFit& lf1,
                             double* acc) {
    const FitEval f0 = fit_eval(lf0);
    FitEval f1;
    if (KIND == DEN_TANH4X2_TAB) f1 = fit_eval(lf1);
    const double invL = 1.0 / (double)L;
    const V3 de2 = mul(s.e2, invL);
    // single-centre fits: t = x.(-2 sigma c) is linear along a row, so it advances by
    // dt = de2.(-2 sigma c) too (exact dot product at the start of every row)
    constexpr bool TADD = KIND != DEN_TANH4X2_TAB;
    const double dt = fma(de2.z, f0.m2c.z, fma(de2.y, f0.m2c.y, de2.x * f0.m2c.x));
    for (int pass = 0; pass < 2; ++pass) {          // 0: up-leaves, 1: down-leaves
        const double sg = pass ? -1.0 : 1.0;
        const int M = L - pass;
#pragma unroll 1
        for (int q = 0; q < 7; ++q) {
            const double ga = fma(sg, l1[q], pass * invL), gb = fma(sg, l2[q], pass * invL);
            const V3 r0 = v3(fma(gb, s.e2.x, s.v0.x), fma(gb, s.e2.y, s.v0.y),
                             fma(gb, s.e2.z, s.v0.z));
            double mq = 0.0, xq = 0.0, yq = 0.0, zq = 0.0, eq = 0.0;
            for (int a = 0; a < M; ++a) {
                const double fa = fma((double)a, invL, ga);
                const V3 base = v3(fma(fa, s.e1.x, r0.x), fma(fa, s.e1.y, r0.y),
                                   fma(fa, s.e1.z, r0.z));
                const int nb = M - a;
                int b = 0;
                // two nodes per step, interleaved stage by stage in the source (ptxas keeps
                // the order, the two dependency chains hide the DFMA latency); nodes advance
                // along the row by de2 = e2 / L with one add per coordinate
                V3 xn = base;                       // node b of the row
                double tn = TADD ? fma(base.z, f0.m2c.z, fma(base.y, f0.m2c.y, base.x * f0.m2c.x))
                                 : 0.0;
                for (; b + 1 < nb; b += 2) {
                    const V3 x0 = xn;
                    const V3 x1 = add(x0, de2);
                    xn = add(x1, de2);
                    const double t0 = tn, t1 = t0 + dt;
                    tn = t1 + dt;
                    double inv0, inv1;
                    if (SERIES) {
                        const double d0 = fma(-x0.z, x0.z, fma(-x0.y, x0.y, fma(-x0.x, x0.x, 1.0)));
                        const double d1 = fma(-x1.z, x1.z, fma(-x1.y, x1.y, fma(-x1.x, x1.x, 1.0)));
                        const double p0 = fma(d0, 0.3125, 0.375), p1 = fma(d1, 0.3125, 0.375);
                        const double q0 = fma(d0, p0, 0.5), q1 = fma(d1, p1, 0.5);
                        inv0 = fma(d0, q0, 1.0); inv1 = fma(d1, q1, 1.0);
                    } else {
                        inv0 = fast_rsqrt(x0.x * x0.x + x0.y * x0.y + x0.z * x0.z);
                        inv1 = fast_rsqrt(x1.x * x1.x + x1.y * x1.y + x1.z * x1.z);
                    }
                    double rho0, rho1;
                    if (TADD) fit_rho2_t(f0, t0, inv0, t1, inv1, &rho0, &rho1);
                    else
                    fit_rho2(f0, x0, inv0, x1, inv1, &rho0, &rho1);
                    if (KIND == DEN_TANH4X2_TAB) {
                        double r0b, r1b;
                        fit_rho2(f1, x0, inv0, x1, inv1, &r0b, &r1b);
                        rho0 = fmax(rho0, r0b); rho1 = fmax(rho1, r1b);
                    }
                    const double dx0 = fma(x0.x, inv0, -z.x), dx1 = fma(x1.x, inv1, -z.x);
                    const double dy0 = fma(x0.y, inv0, -z.y), dy1 = fma(x1.y, inv1, -z.y);
                    const double dz0 = fma(x0.z, inv0, -z.z), dz1 = fma(x1.z, inv1, -z.z);
                    const double e0 = fma(dz0, dz0, fma(dy0, dy0, dx0 * dx0));
                    const double e1 = fma(dz1, dz1, fma(dy1, dy1, dx1 * dx1));
                    mq += rho0 + rho1;
                    // first moment relative to the generator: sum rho (y - z); z sum rho is
                    // added once per rule node class (saves the rho/|x| product per node)
                    xq = fma(rho1, dx1, fma(rho0, dx0, xq));
                    yq = fma(rho1, dy1, fma(rho0, dy0, yq));
                    zq = fma(rho1, dz1, fma(rho0, dz0, zq));
                    eq = fma(rho1, e1, fma(rho0, e0, eq));
                }
                if (b < nb) {
                    const V3 x = xn;
                    double inv;
                    if (SERIES) {
                        const double dl = fma(-x.z, x.z, fma(-x.y, x.y, fma(-x.x, x.x, 1.0)));
                        inv = fma(dl, fma(dl, fma(dl, 0.3125, 0.375), 0.5), 1.0);
                    } else {
                        inv = fast_rsqrt(x.x * x.x + x.y * x.y + x.z * x.z);
                    }
                    double rho = TADD ? fit_rho_t(f0, tn, inv) : fit_rho(f0, x, inv);
                    if (KIND == DEN_TANH4X2_TAB) rho = fmax(rho, fit_rho(f1, x, inv));
                    mq += rho;
                    const double dx = fma(x.x, inv, -z.x), dy = fma(x.y, inv, -z.y),
                                 dz = fma(x.z, inv, -z.z);
                    xq = fma(rho, dx, xq); yq = fma(rho, dy, yq); zq = fma(rho, dz, zq);
                    eq = fma(rho, dx * dx + dy * dy + dz * dz, eq);
                }
            }
            const double wq = s.area * w[q == 0 ? 0 : (q < 4 ? 1 : 4)];
            xq = fma(z.x, mq, xq); yq = fma(z.y, mq, yq); zq = fma(z.z, mq, zq);
            acc[0] = fma(wq, mq, acc[0]);
            acc[1] = fma(wq, xq, acc[1]); acc[2] = fma(wq, yq, acc[2]);
            acc[3] = fma(wq, zq, acc[3]);
            acc[4] = fma(wq, eq, acc[4]);
        }
    }
}

// Two nodes of the fitted sweep (independent chains): positions x0, x1, fit arguments t0, t1
// (t = x.(-2 sigma c), single-centre fits) accumulated into the rule node's sums.
// SER2: every patch of the warp has 1 - |x|^2 <= SER2_MAX, where the cubic term of the 1/|x|
// series is below the truncation the three-term series is admitted with; such a patch carries
// c3 = 0 (otherwise 5/16), so the three-term form gives it the same bits (d * 0 + 3/8 = 3/8).
template <int KIND, bool SERIES, bool TADD, int DEG = 6, bool SER2 = false>
SCVT_HD void fit_pair(const FitEval& f0, const FitEval& f1, V3 z, V3 x0, V3 x1, double t0,
                      double t1, double c3, double& mq, double& xq, double& yq, double& zq,
                      double& eq) {
    double inv0, inv1;
    if (SERIES) {
        const double d0 = fma(-x0.z, x0.z, fma(-x0.y, x0.y, fma(-x0.x, x0.x, 1.0)));
        const double d1 = fma(-x1.z, x1.z, fma(-x1.y, x1.y, fma(-x1.x, x1.x, 1.0)));
        const double p0 = SER2 ? 0.375 : fma(d0, c3, 0.375), p1 = SER2 ? 0.375 : fma(d1, c3, 0.375);
        const double q0 = fma(d0, p0, 0.5), q1 = fma(d1, p1, 0.5);
        inv0 = fma(d0, q0, 1.0); inv1 = fma(d1, q1, 1.0);
    } else {
        inv0 = fast_rsqrt(x0.x * x0.x + x0.y * x0.y + x0.z * x0.z);
        inv1 = fast_rsqrt(x1.x * x1.x + x1.y * x1.y + x1.z * x1.z);
    }
    double rho0, rho1;
    if (TADD) fit_rho2_t<DEG>(f0, t0, inv0, t1, inv1, &rho0, &rho1);
    else fit_rho2<DEG>(f0, x0, inv0, x1, inv1, &rho0, &rho1);
    if (KIND == DEN_TANH4X2_TAB) {
        double r0b, r1b;
        fit_rho2(f1, x0, inv0, x1, inv1, &r0b, &r1b);
        rho0 = fmax(rho0, r0b); rho1 = fmax(rho1, r1b);
    }
    const double dx0 = fma(x0.x, inv0, -z.x), dx1 = fma(x1.x, inv1, -z.x);
    const double dy0 = fma(x0.y, inv0, -z.y), dy1 = fma(x1.y, inv1, -z.y);
    const double dz0 = fma(x0.z, inv0, -z.z), dz1 = fma(x1.z, inv1, -z.z);
    const double e0 = fma(dz0, dz0, fma(dy0, dy0, dx0 * dx0));
    const double e1 = fma(dz1, dz1, fma(dy1, dy1, dx1 * dx1));
    mq += rho0 + rho1;
    xq = fma(rho1, dx1, fma(rho0, dx0, xq));
    yq = fma(rho1, dy1, fma(rho0, dy0, yq));
    zq = fma(rho1, dz1, fma(rho0, dz0, zq));
    eq = fma(rho1, e1, fma(rho0, e0, eq));
}

// The fitted sweep with the up- and down-leaf rows merged (same result up to the summation
// order).  For rule node q the down-leaf node of leaf row a is the up-leaf node of the same
// row shifted by D_q = (1/L - 2 l1_q) e1 + (1/L - 2 l2_q) e2 (l1_q, l2_q: the node's
// coordinates in the first leaf), so one row carries both as
// two chains (L - 1 - a pairs), and the L up-leaf nodes left over -- the row ends, on the
// leaf-grid diagonal -- are swept as L / 2 pairs along the diagonal: per rule node L + 1 row
// setups instead of 2 L - 1, and no single-node tails.
template <int KIND, int L, bool SERIES, int DEG = 6, bool SER2 = false>
SCVT_HD void sym7_fit_leaves_merged(const SubTri& s, V3 z, const double* l1, const double* l2,
                                    const double* w, const LocalFit& lf0, const LocalFit& lf1,
                                    double* acc, double c3 = 0.3125) {
    static_assert(L % 2 == 0, "diagonal pairs");
    const FitEval f0 = fit_eval(lf0);
    FitEval f1;
    if (KIND == DEN_TANH4X2_TAB) f1 = fit_eval(lf1);
    constexpr bool TADD = KIND != DEN_TANH4X2_TAB;
    const double invL = 1.0 / (double)L;
    const V3 de2 = mul(s.e2, invL);
    const V3 dd = mul(sub(s.e1, s.e2), invL);           // along the diagonal
    const double dt = TADD ? fma(de2.z, f0.m2c.z, fma(de2.y, f0.m2c.y, de2.x * f0.m2c.x)) : 0.0;
    const double ddt = TADD ? fma(dd.z, f0.m2c.z, fma(dd.y, f0.m2c.y, dd.x * f0.m2c.x)) : 0.0;
#pragma unroll 1
    for (int q = 0; q < 7; ++q) {
        // l1, l2: node coordinates in the first leaf (already scaled by 1/L)
        const double ga = l1[q], gb = l2[q];
        const double ka = fma(-2.0, ga, invL), kb = fma(-2.0, gb, invL);
        const V3 D = v3(fma(ka, s.e1.x, kb * s.e2.x), fma(ka, s.e1.y, kb * s.e2.y),
                        fma(ka, s.e1.z, kb * s.e2.z));
        const double tD = TADD ? fma(D.z, f0.m2c.z, fma(D.y, f0.m2c.y, D.x * f0.m2c.x)) : 0.0;
        const V3 r0 = v3(fma(gb, s.e2.x, s.v0.x), fma(gb, s.e2.y, s.v0.y),
                         fma(gb, s.e2.z, s.v0.z));
        double mq = 0.0, xq = 0.0, yq = 0.0, zq = 0.0, eq = 0.0;
        for (int a = 0; a < L - 1; ++a) {
            const double fa = fma((double)a, invL, ga);
            V3 xn = v3(fma(fa, s.e1.x, r0.x), fma(fa, s.e1.y, r0.y), fma(fa, s.e1.z, r0.z));
            double tn = TADD ? fma(xn.z, f0.m2c.z, fma(xn.y, f0.m2c.y, xn.x * f0.m2c.x)) : 0.0;
            for (int b = 0; b < L - 1 - a; ++b) {
                const V3 x1 = add(xn, D);
                fit_pair<KIND, SERIES, TADD, DEG, SER2>(f0, f1, z, xn, x1, tn, tn + tD, c3, mq, xq, yq, zq, eq);
                xn = add(xn, de2);
                tn += dt;
            }
        }
        {   // the row ends: up-leaf (a, L-1-a), a = 0..L-1, in pairs along the diagonal
            const double fb = fma((double)(L - 1), invL, gb);
            V3 xn = v3(fma(ga, s.e1.x, fma(fb, s.e2.x, s.v0.x)),
                       fma(ga, s.e1.y, fma(fb, s.e2.y, s.v0.y)),
                       fma(ga, s.e1.z, fma(fb, s.e2.z, s.v0.z)));
            double tn = TADD ? fma(xn.z, f0.m2c.z, fma(xn.y, f0.m2c.y, xn.x * f0.m2c.x)) : 0.0;
            for (int k = 0; k < L / 2; ++k) {
                const V3 x1 = add(xn, dd);
                fit_pair<KIND, SERIES, TADD, DEG, SER2>(f0, f1, z, xn, x1, tn, tn + ddt, c3, mq, xq, yq, zq, eq);
                xn = add(x1, dd);
                tn += 2.0 * ddt;
            }
        }
        const double wq = s.area * w[q == 0 ? 0 : (q < 4 ? 1 : 4)];
        xq = fma(z.x, mq, xq); yq = fma(z.y, mq, yq); zq = fma(z.z, mq, zq);
        acc[0] = fma(wq, mq, acc[0]);
        acc[1] = fma(wq, xq, acc[1]); acc[2] = fma(wq, yq, acc[2]);
        acc[3] = fma(wq, zq, acc[3]);
        acc[4] = fma(wq, eq, acc[4]);
    }
}

#ifdef SCVT_SWEEP_ROWS
#define SCVT_FIT_SWEEP sym7_fit_leaves
#else
#define SCVT_FIT_SWEEP sym7_fit_leaves_merged
#endif

template <int KIND, int L>
SCVT_HD void subtri_moments_sym7(const SubTri& s, V3 z, const double* l1, const double* l2,
                                 const double* w, const DensityParams& dp, double* acc,
                                 int* pole) {
    const bool TAB = KIND == DEN_TANH4_TAB || KIND == DEN_TANH4X2_TAB;
    LocalFit f0, f1;
    bool fitted = false;
    if (TAB) {
        fitted = local_fit(dp, s, v3(dp.c0x, dp.c0y, dp.c0z), f0);
        if (fitted && KIND == DEN_TANH4X2_TAB)
            fitted = local_fit(dp, s, v3(dp.c1x, dp.c1y, dp.c1z), f1);
    }
    if (TAB && fitted) {
        // 1 - |x|^2 <= 1 - dist(origin, plane)^2 on the patch
        const V3 nv = cross(s.e1, s.e2);
        const double nn = dot(nv, nv), h = dot(nv, s.v0);
        const bool series = nn > 0.0 && nn - h * h <= 1e-4 * nn;
        if (KIND == DEN_TANH4X2_TAB) {
            // one centre dominates the whole patch (its minimum above the other's maximum by
            // more than the fits' error): max(rho0, rho1) is that centre's fit at every node,
            // so the single-centre sweep gives the same result at 2/3 of the cost
            const int dom = f1.rmax < f0.rmin * (1.0 - 1e-13) ? 0
                          : (f0.rmax < f1.rmin * (1.0 - 1e-13) ? 1 : -1);
            if (dom >= 0) {
                const LocalFit& fd = dom ? f1 : f0;
                if (series) sym7_fit_leaves<DEN_TANH4_TAB, L, true>(s, z, l1, l2, w, fd, fd, acc);
                else sym7_fit_leaves<DEN_TANH4_TAB, L, false>(s, z, l1, l2, w, fd, fd, acc);
                return;
            }
        }
        if (series)
            sym7_fit_leaves<KIND, L, true>(s, z, l1, l2, w, f0, f1, acc);
        else
            sym7_fit_leaves<KIND, L, false>(s, z, l1, l2, w, f0, f1, acc);
        return;
    }
    V3 o[7];
#pragma unroll
    for (int q = 0; q < 7; ++q) o[q] = add(mul(s.e1, l1[q]), mul(s.e2, l2[q]));
    const double w0 = w[0], w1 = w[1], w2 = w[4];
    double mo[5];
    sym7_leaves<KIND, L, false>(s, z, o, w0, w1, w2, dp, f0, f1, mo, pole);
    acc[0] += s.area * mo[0];
    acc[1] += s.area * mo[1]; acc[2] += s.area * mo[2]; acc[3] += s.area * mo[3];
    acc[4] += s.area * mo[4];
}

// ---- two-phase form of subtri_moments_sym7 (k_quad): the prologue (fits, sweep choice) runs
// inline and leaves its results in a per-thread shared-memory slot; the sweep reads them back.
// Nothing but the slot crosses from one phase to the other, so the prologue's registers die
// before the node loop and no out-of-line call (with its caller-saved stack frame) sits on the
// per-sub-triangle path.
// bits 3-4: how many of the fit's last coefficients are exact zeros (0, 1, 2: local_fit_impl)
// bit 5: 1 - |x|^2 <= SER2_MAX on the patch (two-term 1/|x| series, see fit_pair)
enum : int { SWEEP_TABLE = 0, SWEEP_FIT0 = 1, SWEEP_FIT1 = 2, SWEEP_FIT2 = 3, SWEEP_SERIES = 4,
             SWEEP_DROP_SHIFT = 3, SWEEP_SER2 = 32 };
// 5 d^3 / 16 <= 3e-17: the bound the three-term series is admitted with (35 d^4 / 128 at
// d = 1e-4)
constexpr double SER2_MAX = 4.6e-6;

template <int KIND>
SCVT_HD int sym7_prologue(const DensityParams& dp, const SubTri& s, LocalFit* f) {
    const bool TAB = KIND == DEN_TANH4_TAB || KIND == DEN_TANH4X2_TAB;
    if (!TAB) return SWEEP_TABLE;
    int drop0 = 0, drop1 = 0;
    if (!local_fit_impl<KIND == DEN_TANH4X2_TAB>(dp, s, v3(dp.c0x, dp.c0y, dp.c0z), f[0], &drop0))
        return SWEEP_TABLE;
    int mode = SWEEP_FIT0;
    if (KIND == DEN_TANH4X2_TAB) {
        if (!local_fit_impl(dp, s, v3(dp.c1x, dp.c1y, dp.c1z), f[1], &drop1)) return SWEEP_TABLE;
        // one centre dominates the whole patch: its fit alone gives max(rho0, rho1)
        mode = f[1].rmax < f[0].rmin * (1.0 - 1e-13) ? SWEEP_FIT0
             : (f[0].rmax < f[1].rmin * (1.0 - 1e-13) ? SWEEP_FIT1 : SWEEP_FIT2);
    }
    mode |= (mode == SWEEP_FIT0 ? drop0 : (mode == SWEEP_FIT1 ? drop1 : 0)) << SWEEP_DROP_SHIFT;
    const V3 nv = cross(s.e1, s.e2);
    const double nn = dot(nv, nv), h = dot(nv, s.v0);
    if (nn > 0.0 && nn - h * h <= 1e-4 * nn) mode |= SWEEP_SERIES;
    if (nn > 0.0 && nn - h * h <= SER2_MAX * nn) mode |= SWEEP_SER2;
    return mode;
}

// per-node table (or closed-form) density on the leaf grid: the sweep of a sub-triangle with
// no accepted fit
template <int KIND, int L>
SCVT_HD void sym7_table_sweep(const SubTri& s, V3 z, const double* l1, const double* l2,
                              const double* w, const DensityParams& dp, double* acc, int* pole,
                              int part = 0, int nparts = 1) {
    V3 o[7];
#pragma unroll
    for (int q = 0; q < 7; ++q) o[q] = add(mul(s.e1, l1[q]), mul(s.e2, l2[q]));
    double mo[5];
    LocalFit none;     // not read (FIT = false)
    sym7_leaves<KIND, L, false>(s, z, o, w[0], w[1], w[4], dp, none, none, mo, pole, part,
                                nparts);
    acc[0] += s.area * mo[0];
    acc[1] += s.area * mo[1]; acc[2] += s.area * mo[2]; acc[3] += s.area * mo[3];
    acc[4] += s.area * mo[4];
}

// NO_TABLE: the caller never passes a SWEEP_TABLE mode (k_quad<..., DEFER> queues those)
template <int KIND, int L, bool NO_TABLE = false>
SCVT_HD void sym7_sweep(int mode, const SubTri& s, V3 z, const double* l1, const double* l2,
                        const double* w, const DensityParams& dp, const LocalFit* f,
                        double* acc, int* pole) {
    const int fit = mode & 3;
    const bool series = (mode & SWEEP_SERIES) != 0;
    if (fit == SWEEP_FIT0 || fit == SWEEP_FIT1) {
        const LocalFit& fd = f[fit - 1];
#ifndef SCVT_SWEEP_ROWS
        if (series) {
            // the lowest degree every patch of the warp on this path allows (same bits as the
            // degree-6 sweep: the dropped coefficients are exact zeros)
            int drop = (mode >> SWEEP_DROP_SHIFT) & 3;
            const bool mine2 = (mode & SWEEP_SER2) != 0;
            bool ser2 = mine2;
#ifdef __CUDA_ARCH__
            const unsigned am = __activemask();
            drop = __reduce_min_sync(am, drop);
            ser2 = __all_sync(am, mine2);
#endif
            // in a mixed warp a two-term patch takes the three-term sweep with c3 = 0: same bits
            const double c3 = mine2 ? 0.0 : 0.3125;
#define SCVT_SWEEP_DEG(DEG)                                                                      \
    do {                                                                                         \
        if (ser2) sym7_fit_leaves_merged<DEN_TANH4_TAB, L, true, DEG, true>(s, z, l1, l2, w, fd, \
                                                                            fd, acc);            \
        else sym7_fit_leaves_merged<DEN_TANH4_TAB, L, true, DEG, false>(s, z, l1, l2, w, fd, fd, \
                                                                        acc, c3);                \
    } while (0)
            if (drop == 2) SCVT_SWEEP_DEG(4);
            else if (drop == 1) SCVT_SWEEP_DEG(5);
            else SCVT_SWEEP_DEG(6);
#undef SCVT_SWEEP_DEG
            return;
        }
#endif
        if (series) SCVT_FIT_SWEEP<DEN_TANH4_TAB, L, true>(s, z, l1, l2, w, fd, fd, acc);
        else SCVT_FIT_SWEEP<DEN_TANH4_TAB, L, false>(s, z, l1, l2, w, fd, fd, acc);
        return;
    }
    if (KIND == DEN_TANH4X2_TAB && fit == SWEEP_FIT2) {
        if (series) SCVT_FIT_SWEEP<KIND, L, true>(s, z, l1, l2, w, f[0], f[1], acc);
        else SCVT_FIT_SWEEP<KIND, L, false>(s, z, l1, l2, w, f[0], f[1], acc);
        return;
    }
    if (NO_TABLE) return;
    sym7_table_sweep<KIND, L>(s, z, l1, l2, w, dp, acc, pole);
}

}  // namespace scvt
