// TEST-ONLY host harness: compiles the same __host__ __device__ functions the sm_100a kernels
// use (paper_1709_06924_b200/csrc/scvt_device.cuh) for the CPU, so the cell-clipping
// combinatorics and the per-incidence quadrature can be checked against the oracle without a
// GPU.  Never linked into, loaded by, or reachable from the shipped package.
#define _USE_MATH_DEFINES
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include "../../paper_1709_06924_b200/csrc/scvt_device.cuh"

using namespace scvt;

extern "C" int harness_cells(const double* z, int n, int* nbr, int* deg, int* stats) {
    int G = std::max(1, (int)std::sqrt(n / 12.0));
    int nb = 6 * G * G;
    std::vector<uint32_t> key(n);
    for (int i = 0; i < n; ++i) key[i] = bucket_key(load3(z, i), G);
    std::vector<int> ids(n);
    std::iota(ids.begin(), ids.end(), 0);
    std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) { return key[a] < key[b]; });
    std::vector<int> start(nb + 1, 0);
    for (int b = 0, p = 0; b <= nb; ++b) {
        while (p < n && key[ids[p]] < (uint32_t)b) ++p;
        start[b] = p;
    }
    std::vector<double> zs(4 * (size_t)n);
    for (int p = 0; p < n; ++p)
        for (int c = 0; c < 3; ++c) zs[4 * p + c] = z[3 * ids[p] + c];
    GridView g{zs.data(), ids.data(), start.data(), z, G, n};
    Poly* P = new Poly;
    Poly* T = new Poly;
    int status = 0;
    stats[0] = stats[1] = stats[2] = stats[3] = 0;
    for (int p = 0; p < n; ++p) {
        int i = ids[p];
        CellStats cs;
        int d = build_cell(g, i, v3(zs[4 * p], zs[4 * p + 1], zs[4 * p + 2]), nbr + (int64_t)i * MAXDEG,
                           &cs, *P, *T);
        if (d < 0) { status |= -d; deg[i] = 0; } else { deg[i] = d; stats[0] = std::max(stats[0], d); }
        stats[1] += cs.rounds > 1;
        stats[2] = std::max(stats[2], cs.passes);
        stats[3] += cs.tie_breaks;
    }
    delete P; delete T;
    return status;
}

extern "C" int harness_insphere(const double* o, const double* a, const double* b, const double* c,
                                int* ambiguous) {
    bool am;
    int s = insphere_sign(load3(o, 0), load3(a, 0), load3(b, 0), load3(c, 0), &am);
    *ambiguous = am;
    return s;
}

// exact orient3d with symbolic perturbation (orient_robust): sign, *tier = 0/1/2
extern "C" int harness_orient(const double* o, const double* a, const double* b, const double* c,
                              int io, int ia, int ib, int ic, int* tier) {
    return orient_robust(load3(o, 0), load3(a, 0), load3(b, 0), load3(c, 0), io, ia, ib, ic, tier);
}

// the exact tiers alone (skipping the FP64 filter)
extern "C" int harness_orient_exact(const double* o, const double* a, const double* b,
                                    const double* c, int io, int ia, int ib, int ic, int* tier) {
    return orient_exact_sos(load3(o, 0), load3(a, 0), load3(b, 0), load3(c, 0), io, ia, ib, ic,
                            tier);
}

template <int K>
static void quad_all(const double* z, int n, const int* nbr, const int* deg, const double* l1,
                     const double* l2, const double* w, int nq, const DensityParams& dp, int sphere,
                     double* out, int* pole, int* obtuse) {
    for (int i = 0; i < n; ++i) {
        double acc[5] = {0, 0, 0, 0, 0};
        const int* row = nbr + (int64_t)i * MAXDEG;
        int d = deg[i];
        for (int t = 0; t < d; ++t) {
            int j = row[t], k = row[(t + 1) % d];
            FanPair f = fan_pair(load3(z, i), load3(z, j), load3(z, k), i, j, k);
            for (int s = 0; s < 2; ++s) {
                if (sphere) subtri_moments<K, true>(f.s[s], load3(z, i), l1, l2, w, nq, dp, acc, pole);
                else subtri_moments<K, false>(f.s[s], load3(z, i), l1, l2, w, nq, dp, acc, pole);
            }
            if (f.obtuse && i < j && i < k) ++*obtuse;
        }
        for (int c = 0; c < 5; ++c) out[5 * (int64_t)i + c] = acc[c];
    }
}

extern "C" int harness_quad(const double* z, int n, const int* nbr, const int* deg, const double* l1,
                            const double* l2, const double* w, int nq, int kind, const double* prm,
                            int sphere, double* out, int* obtuse) {
    DensityParams dp{};
    dp.kind = kind;
    dp.gamma = prm[0]; dp.beta = prm[1]; dp.alpha = prm[2];
    dp.c0x = prm[3]; dp.c0y = prm[4]; dp.c0z = prm[5];
    dp.c1x = prm[6]; dp.c1y = prm[7]; dp.c1z = prm[8];
    dp.w_lon = prm[9]; dp.w_lat = prm[10];
    dp.lat_c = prm[11]; dp.lon_c = prm[12]; dp.cos_lat_c = prm[13]; dp.sin_lat_c = prm[14];
    int pole = 0;
    *obtuse = 0;
    switch (kind) {
        case 0: quad_all<0>(z, n, nbr, deg, l1, l2, w, nq, dp, sphere, out, &pole, obtuse); break;
        case 1: quad_all<1>(z, n, nbr, deg, l1, l2, w, nq, dp, sphere, out, &pole, obtuse); break;
        case 2: quad_all<2>(z, n, nbr, deg, l1, l2, w, nq, dp, sphere, out, &pole, obtuse); break;
        case 3: quad_all<3>(z, n, nbr, deg, l1, l2, w, nq, dp, sphere, out, &pole, obtuse); break;
        case 4: quad_all<4>(z, n, nbr, deg, l1, l2, w, nq, dp, sphere, out, &pole, obtuse); break;
        case 5: quad_all<5>(z, n, nbr, deg, l1, l2, w, nq, dp, sphere, out, &pole, obtuse); break;
    }
    return pole;
}

// single-cell probe for debugging: returns valence or -status, fills the cycle and rounds
extern "C" int harness_one_cell(const double* z, int n, int i, int* nbr, int* rounds) {
    int G = std::max(1, (int)std::sqrt(n / 12.0));
    int nb = 6 * G * G;
    std::vector<uint32_t> key(n);
    for (int q = 0; q < n; ++q) key[q] = bucket_key(load3(z, q), G);
    std::vector<int> ids(n);
    std::iota(ids.begin(), ids.end(), 0);
    std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) { return key[a] < key[b]; });
    std::vector<int> start(nb + 1, 0);
    for (int b = 0, p = 0; b <= nb; ++b) {
        while (p < n && key[ids[p]] < (uint32_t)b) ++p;
        start[b] = p;
    }
    std::vector<double> zs(4 * (size_t)n);
    for (int p = 0; p < n; ++p)
        for (int c = 0; c < 3; ++c) zs[4 * p + c] = z[3 * ids[p] + c];
    GridView g{zs.data(), ids.data(), start.data(), z, G, n};
    Poly* P = new Poly;
    Poly* T = new Poly;
    CellStats cs;
    int d = build_cell(g, i, load3(z, i), nbr, &cs, *P, *T);
    *rounds = cs.passes;
    delete P; delete T;
    return d;
}

// per-sub-triangle local-fit acceptance and sym7-path moments (tanh4 table kinds 6/7)
extern "C" int harness_fit_stats(const double* z, int n, const int* nbr, const int* deg,
                                 const double* table, int tab_k, double tab_w, const double* prm,
                                 int kind, long long* counts) {
    DensityParams dp{};
    dp.kind = kind;
    dp.gamma = prm[0]; dp.beta = prm[1]; dp.alpha = prm[2];
    dp.c0x = prm[3]; dp.c0y = prm[4]; dp.c0z = prm[5];
    dp.c1x = prm[6]; dp.c1y = prm[7]; dp.c1z = prm[8];
    dp.tab = table; dp.tab_k = tab_k; dp.tab_invw = 1.0 / tab_w;
    // counts: {fitted, sub-triangles, fitted on the 1/|x| series path, fitted and
    //          single-centre dominated (two-centre kind)}
    long long ok = 0, tot = 0, series = 0, dom = 0;
    for (int i = 0; i < n; ++i) {
        const int* row = nbr + (int64_t)i * MAXDEG;
        for (int t = 0; t < deg[i]; ++t) {
            int j = row[t], k = row[(t + 1) % deg[i]];
            FanPair f = fan_pair(load3(z, i), load3(z, j), load3(z, k), i, j, k);
            for (int s = 0; s < 2; ++s) {
                LocalFit lf, lf1;
                bool a = local_fit(dp, f.s[s], v3(dp.c0x, dp.c0y, dp.c0z), lf);
                if (a && kind == 7) {
                    a = local_fit(dp, f.s[s], v3(dp.c1x, dp.c1y, dp.c1z), lf1);
                    if (a) dom += lf1.rmax < lf.rmin * (1.0 - 1e-13) || lf.rmax < lf1.rmin * (1.0 - 1e-13);
                }
                if (a) {
                    const V3 nv = cross(f.s[s].e1, f.s[s].e2);
                    const double nn = dot(nv, nv), h = dot(nv, f.s[s].v0);
                    series += nn > 0.0 && nn - h * h <= 1e-4 * nn;
                }
                ok += a;
                ++tot;
            }
        }
    }
    counts[0] = ok;
    counts[1] = tot;
    counts[2] = series;
    counts[3] = dom;
    return 0;
}

extern "C" int harness_quad_sym7(const double* z, int n, const int* nbr, const int* deg,
                                 const double* l1, const double* l2, const double* w,
                                 const double* table, int tab_k, double tab_w, const double* prm,
                                 int kind, double* out) {
    DensityParams dp{};
    dp.kind = kind;
    dp.gamma = prm[0]; dp.beta = prm[1]; dp.alpha = prm[2];
    dp.c0x = prm[3]; dp.c0y = prm[4]; dp.c0z = prm[5];
    dp.c1x = prm[6]; dp.c1y = prm[7]; dp.c1z = prm[8];
    dp.tab = table; dp.tab_k = tab_k; dp.tab_invw = tab_w > 0 ? 1.0 / tab_w : 0.0;
    int pole = 0;
    for (int i = 0; i < n; ++i) {
        double acc[5] = {0, 0, 0, 0, 0};
        const int* row = nbr + (int64_t)i * MAXDEG;
        for (int t = 0; t < deg[i]; ++t) {
            int j = row[t], k = row[(t + 1) % deg[i]];
            for (int s = 0; s < 2; ++s) {
                // the k_quad fast path: this half's fan sub-triangle, prologue, sweep
                int obt, degen;
                const SubTri st = fan_sub(load3(z, i), load3(z, j), load3(z, k), i, j, k, s,
                                          &obt, &degen);
                LocalFit fit[2];
                double h[5] = {0, 0, 0, 0, 0};
                if (kind == 6) {
                    int mode = sym7_prologue<6>(dp, st, fit);
                    sym7_sweep<6, 8>(mode, st, load3(z, i), l1, l2, w, dp, fit, h, &pole);
                } else if (kind == 7) {
                    int mode = sym7_prologue<7>(dp, st, fit);
                    sym7_sweep<7, 8>(mode, st, load3(z, i), l1, l2, w, dp, fit, h, &pole);
                } else {
                    int mode = sym7_prologue<0>(dp, st, fit);
                    sym7_sweep<0, 8>(mode, st, load3(z, i), l1, l2, w, dp, fit, h, &pole);
                }
                for (int c = 0; c < 5; ++c) acc[c] += h[c];
            }
        }
        for (int c = 0; c < 5; ++c) out[5 * (int64_t)i + c] = acc[c];
    }
    return pole;
}


// distribution of the Chebyshev tail of the accepted single-centre fits, in the order given by
// `order` (generator ids; the kernel's incidence order is by cube-map bucket): per
// sub-triangle the tail sums |a6|, |a5|+|a6|, |a4|+|a5|+|a6| relative to min rho and the patch's
// bound of 1 - |x|^2 (tail[4 * idx ...]), and
// the accepted flag; returns the number of sub-triangles
extern "C" long long harness_fit_tails(const double* z, int n, const int* order, const int* nbr,
                                       const int* deg, const double* table, int tab_k,
                                       double tab_w, const double* prm, int kind, double* tail,
                                       int* accepted) {
    DensityParams dp{};
    dp.kind = kind;
    dp.gamma = prm[0]; dp.beta = prm[1]; dp.alpha = prm[2];
    dp.c0x = prm[3]; dp.c0y = prm[4]; dp.c0z = prm[5];
    dp.c1x = prm[6]; dp.c1y = prm[7]; dp.c1z = prm[8];
    dp.tab = table; dp.tab_k = tab_k; dp.tab_invw = 1.0 / tab_w;
    long long idx = 0;
    for (int p = 0; p < n; ++p) {
        const int i = order[p];
        const int* row = nbr + (int64_t)i * MAXDEG;
        for (int t = 0; t < deg[i]; ++t) {
            int j = row[t], k = row[(t + 1) % deg[i]];
            FanPair f = fan_pair(load3(z, i), load3(z, j), load3(z, k), i, j, k);
            for (int s = 0; s < 2; ++s) {
                LocalFit lf;
                int low = 0;
                double ts[4] = {1, 1, 1, 1};
                bool a = local_fit_impl(dp, f.s[s], v3(dp.c0x, dp.c0y, dp.c0z), lf, &low, ts);
                accepted[idx] = a ? 1 + low : 0;
                for (int q = 0; q < 3; ++q) tail[4 * idx + q] = ts[q];
                {   // 1 - |x|^2 bound of the patch (the 1/|x| series criterion of sym7_prologue)
                    const V3 nv = cross(f.s[s].e1, f.s[s].e2);
                    const double nn = dot(nv, nv), hh = dot(nv, f.s[s].v0);
                    tail[4 * idx + 3] = nn > 0.0 ? (nn - hh * hh) / nn : 1.0;
                }
                ++idx;
            }
        }
    }
    return idx;
}
