// amul.cuh -- A7 Amul variants (included by kernels.cu).  All variants compute
// y_c = diag_c x_c + sum_{nbr(c)} upper x + sum_{own(c)} upper x (+ interfaces)
// in the oracle's order (reading Q10) with separate DMUL/DADD (--fmad=false),
// so every variant is bitwise identical to amul_row() and to the oracle.
//
//   0  per-row:   one thread per cell, grid-stride (amul_row)
//   1  tile:      CTA-cooperative products in shared memory, then ordered row sums
//   2  unrolled:  one thread per cell, up to 4 faces per side loaded as one batch
//   4  per-row capped at 32 registers (8 CTAs of 256 threads per SM: more warps in flight)
//   5  unrolled, two cells per thread (c and c + 256 of a 512-cell tile): both cells'
//      loads issued together, twice the bytes in flight per thread
//   6  SELL-C:    chunk-of-32 slot layout, packed neighbour side, one row per thread
//   7  SELL-C:    two rows per thread (chunks k and k+1 of a 64-cell warp tile)
//   8  ELL:       uniform-width SELL + per-solve owner-slot coefficient copy, 1 row/thread
//   9  ELL:       same, two rows per thread
//   3  tma:       warp-specialised pipeline -- a producer warp streams each tile's
//                 contiguous ranges (upper/neighbour of the owner side,
//                 losort/ownerLo of the neighbour side, ownerStart/losortStart,
//                 x, diag) into shared-memory stages with cp.async.bulk (TMA)
//                 completing on mbarriers; consumer warps gather x[column] and
//                 upper[losort] (L2), stage the products and sum rows in order.
#pragma once

namespace spuma {

// Processor-interface terms of row c (after its internal faces, reading Q10); rows
// without interfaces are skipped with one bit of a per-cell mask (1 bit / cell).
__device__ __forceinline__ double add_iface(const MeshArgs& a, int c, double s, const double* __restrict__ iface,
                                            const double* __restrict__ xr)
{
    if (a.ifMask && ((__ldg(a.ifMask + (c >> 5)) >> (c & 31)) & 1u)) {
        const int j1 = a.ifStart[c + 1];
        for (int j = a.ifStart[c]; j < j1; ++j) {
            const int i = a.ifIdx[j];
            s = s + iface[i] * xr[i];
        }
    }
    return s;
}

__device__ __forceinline__ bool is_iface_row(const MeshArgs& a, int c)
{
    return a.ifMask && ((__ldg(a.ifMask + (c >> 5)) >> (c & 31)) & 1u);
}

// ---------------------------------------------------------------------------- variant 2
__device__ __forceinline__ double amul_row_unrolled(const MeshArgs& a, int c, const double* __restrict__ diag,
                                                    const double* __restrict__ upper,
                                                    const double* __restrict__ iface,
                                                    const double* __restrict__ x, const double* __restrict__ xr)
{
    const int k0 = __ldg(a.losortStart + c), k1 = __ldg(a.losortStart + c + 1);
    const int f0 = __ldg(a.ownerStart + c), f1 = __ldg(a.ownerStart + c + 1);
    const double d = __ldg(diag + c), xc = __ldg(x + c);
    if (k1 - k0 > 4 || f1 - f0 > 4) return amul_row(a, c, diag, upper, iface, x, xr, nullptr);
    int fi[4], cn[4], co[4];
    double uo[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const bool vn = k0 + r < k1, vo = f0 + r < f1;
        fi[r] = vn ? __ldg(a.losort + k0 + r) : 0;
        cn[r] = vn ? __ldg(a.ownerLo + k0 + r) : c;
        co[r] = vo ? __ldg(a.neighbour + f0 + r) : c;
        uo[r] = vo ? __ldg(upper + f0 + r) : 0.0;
    }
    double un[4], xn[4], xo[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        un[r] = k0 + r < k1 ? __ldg(upper + fi[r]) : 0.0;
        xn[r] = __ldg(x + cn[r]);
        xo[r] = __ldg(x + co[r]);
    }
    double s = d * xc;
#pragma unroll
    for (int r = 0; r < 4; ++r)
        if (k0 + r < k1) s = s + un[r] * xn[r];
#pragma unroll
    for (int r = 0; r < 4; ++r)
        if (f0 + r < f1) s = s + uo[r] * xo[r];
    if (a.ifStart) {
        const int j1 = a.ifStart[c + 1];
        for (int j = a.ifStart[c]; j < j1; ++j) {
            const int i = a.ifIdx[j];
            s = s + iface[i] * xr[i];
        }
    }
    return s;
}

// ---------------------------------------------------------------------------- variant 5
// Two rows per thread, every load of both rows issued before any use.
__device__ __forceinline__ void amul_rows2(const MeshArgs& a, int c, int e, const double* __restrict__ diag,
                                           const double* __restrict__ upper, const double* __restrict__ iface,
                                           const double* __restrict__ x, const double* __restrict__ xr,
                                           double* __restrict__ y, double& acc, bool dot)
{
    const bool ve = e < a.N;
    const int ec = ve ? e : c;
    const int k0 = __ldg(a.losortStart + c), k1 = __ldg(a.losortStart + c + 1);
    const int f0 = __ldg(a.ownerStart + c), f1 = __ldg(a.ownerStart + c + 1);
    const int q0 = __ldg(a.losortStart + ec), q1 = __ldg(a.losortStart + ec + 1);
    const int g0 = __ldg(a.ownerStart + ec), g1 = __ldg(a.ownerStart + ec + 1);
    const double dc = __ldg(diag + c), xc = __ldg(x + c), de = __ldg(diag + ec), xe = __ldg(x + ec);
    if (k1 - k0 > 3 || f1 - f0 > 3 || q1 - q0 > 3 || g1 - g0 > 3 || a.ifStart) {
        const double r = amul_row(a, c, diag, upper, iface, x, xr, nullptr);
        y[c] = r;
        if (dot) acc += r * xc;
        if (ve) {
            const double t = amul_row(a, e, diag, upper, iface, x, xr, nullptr);
            y[e] = t;
            if (dot) acc += t * xe;
        }
        return;
    }
    int fi[6], cn[6], co[6];
    double uo[6];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        bool vn = k0 + r < k1, vo = f0 + r < f1;
        fi[r] = vn ? __ldg(a.losort + k0 + r) : 0;
        cn[r] = vn ? __ldg(a.ownerLo + k0 + r) : c;
        co[r] = vo ? __ldg(a.neighbour + f0 + r) : c;
        uo[r] = vo ? __ldg(upper + f0 + r) : 0.0;
        vn = q0 + r < q1, vo = g0 + r < g1;
        fi[3 + r] = vn ? __ldg(a.losort + q0 + r) : 0;
        cn[3 + r] = vn ? __ldg(a.ownerLo + q0 + r) : ec;
        co[3 + r] = vo ? __ldg(a.neighbour + g0 + r) : ec;
        uo[3 + r] = vo ? __ldg(upper + g0 + r) : 0.0;
    }
    double un[6], xn[6], xo[6];
#pragma unroll
    for (int r = 0; r < 6; ++r) {
        un[r] = __ldg(upper + fi[r]);
        xn[r] = __ldg(x + cn[r]);
        xo[r] = __ldg(x + co[r]);
    }
    double s = dc * xc, t = de * xe;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        if (k0 + r < k1) s = s + un[r] * xn[r];
        if (q0 + r < q1) t = t + un[3 + r] * xn[3 + r];
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        if (f0 + r < f1) s = s + uo[r] * xo[r];
        if (g0 + r < g1) t = t + uo[3 + r] * xo[3 + r];
    }
    y[c] = s;
    if (dot) acc += s * xc;
    if (ve) {
        y[e] = t;
        if (dot) acc += t * xe;
    }
}

#ifndef SPUMA_LOOP_XLD
#define SPUMA_LOOP_XLD 0  // A/B of the persistent loop's coherent loads: 0 ld.global, 1 ld.global.cg (L2 only)
#endif
template <bool NC>
__device__ __forceinline__ double ldx(const double* p)
{
    if constexpr (NC) return __ldg(p);
    double v;
#if SPUMA_LOOP_XLD == 1
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
#else
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));  // volatile: stays behind the barriers
#endif
    return v;
}

// ---------------------------------------------------------------------------- variants 6, 7 (SELL-C)
// Rows read from the SELL-C slots (host.h build_sell): the neighbour side is one packed
// int32 per entry (owner column << 5 | position of the face in the owner's range), so
// neither losort nor losortStart is streamed: DRAM bytes ~ 16 per face (upper 8, two
// 4-byte slots) + 28 per cell (ownerStart, diag, x, y).  Coefficient of a neighbour-side
// entry = upper[ownerStart[column] + position] (L2 hit: the owner's row streamed it).
// When every chunk has the same widths (hex meshes) the slot bases are arithmetic and
// the per-chunk meta load drops out of the dependency chain.
// IFM (interface mode): 0 no processor faces, 1 add the interface terms inline,
// 2 deferred -- interface rows keep only their internal-face sum (finished later by
// k_iface_rows once the halo has arrived) and are left out of this kernel's dot.
// y_c = (A x)_c by the generic row gather (amul_row's order, reading Q10) with coherent x loads:
// the wide-row fallback of the persistent loop's SELL rows (x rewritten inside the launch)
__device__ __forceinline__ double amul_row_coherent(const MeshArgs& a, int c, const double* __restrict__ diag,
                                                    const double* __restrict__ upper, const double* x)
{
    double s = diag[c] * ldx<false>(x + c);
    const int k1 = a.losortStart[c + 1];
    for (int k = a.losortStart[c]; k < k1; ++k) s = s + upper[a.losort[k]] * ldx<false>(x + a.ownerLo[k]);
    const int f1 = a.ownerStart[c + 1];
    for (int f = a.ownerStart[c]; f < f1; ++f) s = s + upper[f] * ldx<false>(x + a.neighbour[f]);
    return s;
}

template <int R, int IFM = 0, bool NC = true>
__device__ __forceinline__ void amul_rows_sell(const MeshArgs& a, int c, int wn_u, int wo_u,
                                               const double* __restrict__ diag, const double* __restrict__ upper,
                                               const double* __restrict__ iface, const double* __restrict__ x,
                                               const double* __restrict__ xr, double* __restrict__ y, double& acc,
                                               bool dot)
{
    constexpr int W = 3;  // fast-path slot width per side
    const int l = c & 31;
    int cc[R], nbase[R], obase[R], wn[R], wo[R], osc[R];
    double dg[R], xc[R];
    bool ok = true;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        cc[r] = min(c + 32 * r, a.N - 1);
        const int k = cc[r] >> 5;
        if (wn_u >= 0) {
            nbase[r] = k * 32 * wn_u;
            obase[r] = k * 32 * wo_u;
            wn[r] = wn_u;
            wo[r] = wo_u;
        } else {
            const int4 m = __ldg(a.sell_meta + k);
            nbase[r] = m.x, obase[r] = m.y, wn[r] = m.z, wo[r] = m.w;
        }
        ok = ok && wn[r] <= W && wo[r] <= W;
        osc[r] = __ldg(a.ownerStart + cc[r]);
        dg[r] = __ldg(diag + cc[r]);
        xc[r] = ldx<NC>(x + cc[r]);
    }
    if (!ok) {
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (c + 32 * r < a.N) {
                double v;
                if constexpr (NC) v = amul_row(a, cc[r], diag, upper, iface, x, xr, nullptr, IFM != 2);
                else v = amul_row_coherent(a, cc[r], diag, upper, x);  // (single rank: no interfaces)
                y[cc[r]] = v;
                if (dot && (IFM != 2 || !is_iface_row(a, cc[r]))) acc += v * xc[r];
            }
        return;
    }
    unsigned pk[R][W];
    int nb[R][W];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < W; ++j) {
            pk[r][j] = j < wn[r] ? __ldg(a.sell_n + nbase[r] + 32 * j + l) : 0xFFFFFFFFu;
            nb[r][j] = j < wo[r] ? __ldg(a.sell_o + obase[r] + 32 * j + l) : -1;
        }
    int oc[R][W];
    double xn[R][W], xo[R][W], uo[R][W];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const bool vn = pk[r][j] != 0xFFFFFFFFu, vo = nb[r][j] >= 0;
            const int col = vn ? (int)(pk[r][j] >> 5) : cc[r];
            oc[r][j] = vn ? __ldg(a.ownerStart + col) : 0;
            xn[r][j] = ldx<NC>(x + col);
            xo[r][j] = ldx<NC>(x + (vo ? nb[r][j] : cc[r]));
            uo[r][j] = vo ? __ldg(upper + osc[r] + j) : 0.0;
        }
    double un[R][W];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < W; ++j)
            un[r][j] = pk[r][j] != 0xFFFFFFFFu ? __ldg(upper + oc[r][j] + (int)(pk[r][j] & 31u)) : 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double s = dg[r] * xc[r];
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (pk[r][j] != 0xFFFFFFFFu) s = s + un[r][j] * xn[r][j];
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (nb[r][j] >= 0) s = s + uo[r][j] * xo[r][j];
        if constexpr (IFM == 1) s = add_iface(a, cc[r], s, iface, xr);
        if (c + 32 * r < a.N) {
            y[cc[r]] = s;
            if (dot && (IFM != 2 || !is_iface_row(a, cc[r]))) acc += s * xc[r];
        }
    }
}

// ---------------------------------------------------------------------------- variants 8, 9 (ELL + coefficient copy)
// Uniform-width SELL (ELL) layout plus a per-solve copy of the coefficients in owner-side
// slot order, upper_s[32 wo k + 32 j + l] = upper[ownerStart[c] + j] (c = 32 k + l).  The
// owner side then streams (upper_s, neighbour slot) and the neighbour side finds its
// coefficient at upper_s[32 wo (col >> 5) + 32 pos + (col & 31)] -- an L2 hit of the
// owner's chunk -- so no row extent is loaded at all: two dependent levels, DRAM bytes
// ~ 16 per face + 24 per cell (the algorithmic minimum of SURVEY §8(d)).
template <int R, int IFM = 0>
__device__ __forceinline__ void amul_rows_ell(const MeshArgs& a, int c, int wn, int wo,
                                              const double* __restrict__ diag, const double* __restrict__ upper,
                                              const double* __restrict__ upper_s, const double* __restrict__ iface,
                                              const double* __restrict__ x, const double* __restrict__ xr,
                                              double* __restrict__ y, double& acc, bool dot)
{
    constexpr int W = 3;
    const int l = c & 31;
    if (wn > W || wo > W) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int cr = c + 32 * r;
            if (cr < a.N) {
                const double v = amul_row(a, cr, diag, upper, iface, x, xr, nullptr, IFM != 2);
                y[cr] = v;
                if (dot && (IFM != 2 || !is_iface_row(a, cr))) acc += v * x[cr];
            }
        }
        return;
    }
    if constexpr (R == 1) {
        // chunk-stencil rows: the chunk's <= 3 column offsets per side are warp-
        // uniform loads, one 32-bit word per cell replaces the 6 explicit slot indices; same
        // slots, same order (offsets ascending = losort / face order), so the same value
        const int k = c >> 5;
        if (a.cmeta) {
            // one dependent level as in the explicit rows: meta, cell word, diag, x and the
            // owner-side coefficients (compact slots) are all issued before any of them is used
            const int4 m0 = __ldg(reinterpret_cast<const int4*>(a.cmeta) + 2 * k);
            const int4 m1 = __ldg(reinterpret_cast<const int4*>(a.cmeta) + 2 * k + 1);
            const int cr = min(c, a.N - 1);
            const unsigned bits = __ldg(a.clane + cr);
            const double dg = __ldg(diag + cr), xcv = __ldg(x + cr);
            double uc[W];
#pragma unroll
            for (int j = 0; j < W; ++j) uc[j] = j < wo ? __ldg(upper_s + (size_t)32 * wo * k + 32 * j + l) : 0.0;
            if (m0.x) {
                const int dn[W] = {m0.y, m0.z, m0.w}, dq[W] = {m1.x, m1.y, m1.z};
                double un[W], xn[W], xo[W];
#pragma unroll
                for (int t = 0; t < W; ++t) {
                    const bool vn = (bits >> t) & 1u;
                    const int col = vn ? cr + dn[t] : cr;
                    const int pos = (int)((bits >> (6 + 5 * t)) & 31u);
                    un[t] = vn ? __ldg(upper_s + (size_t)32 * wo * (col >> 5) + 32 * pos + (col & 31)) : 0.0;
                    xn[t] = __ldg(x + col);
                    const bool vo = (bits >> (3 + t)) & 1u;
                    xo[t] = __ldg(x + (vo ? cr + dq[t] : cr));
                }
                double s = dg * xcv;
#pragma unroll
                for (int t = 0; t < W; ++t)
                    if ((bits >> t) & 1u) s = s + un[t] * xn[t];
#pragma unroll
                for (int t = 0; t < W; ++t)
                    if ((bits >> (3 + t)) & 1u) {  // owner-side offset t = compact slot popc(lower bits)
                        const int so = __popc((bits >> 3) & ((1u << t) - 1u));
                        const double u = so == 0 ? uc[0] : (so == 1 ? uc[1] : uc[2]);
                        s = s + u * xo[t];
                    }
                if constexpr (IFM == 1) s = add_iface(a, cr, s, iface, xr);
                if (c < a.N) {
                    y[cr] = s;
                    if (dot && (IFM != 2 || !is_iface_row(a, cr))) acc += s * xcv;
                }
                return;
            }
        }
    }
    int cc[R];
    double dg[R], xc[R];
    unsigned pk[R][W];
    int nb[R][W];
    double uo[R][W];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        cc[r] = min(c + 32 * r, a.N - 1);
        const int k = cc[r] >> 5;
        dg[r] = __ldg(diag + cc[r]);
        xc[r] = __ldg(x + cc[r]);
#pragma unroll
        for (int j = 0; j < W; ++j) {
            pk[r][j] = j < wn ? __ldg(a.sell_n + (size_t)32 * wn * k + 32 * j + l) : 0xFFFFFFFFu;
            nb[r][j] = j < wo ? __ldg(a.sell_o + (size_t)32 * wo * k + 32 * j + l) : -1;
            uo[r][j] = j < wo ? __ldg(upper_s + (size_t)32 * wo * k + 32 * j + l) : 0.0;
        }
    }
    double un[R][W], xn[R][W], xo[R][W];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const bool vn = pk[r][j] != 0xFFFFFFFFu;
            const int col = vn ? (int)(pk[r][j] >> 5) : cc[r];
            const int pos = (int)(pk[r][j] & 31u);
            un[r][j] = vn ? __ldg(upper_s + (size_t)32 * wo * (col >> 5) + 32 * pos + (col & 31)) : 0.0;
            xn[r][j] = __ldg(x + col);
            xo[r][j] = __ldg(x + (nb[r][j] >= 0 ? nb[r][j] : cc[r]));
        }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double s = dg[r] * xc[r];
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (pk[r][j] != 0xFFFFFFFFu) s = s + un[r][j] * xn[r][j];
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (nb[r][j] >= 0) s = s + uo[r][j] * xo[r][j];
        if constexpr (IFM == 1) s = add_iface(a, cc[r], s, iface, xr);
        if (c + 32 * r < a.N) {
            y[cc[r]] = s;
            if (dot && (IFM != 2 || !is_iface_row(a, cc[r]))) acc += s * xc[r];
        }
    }
}

// Variant 10: the ELL rows of variant 8 software-pipelined across the grid-stride loop -- the
// first-level loads of the thread's NEXT row (diag, x, the six slots, the owner-side
// coefficients) are issued before the second-level gathers of the current row, so two rows'
// worth of loads are in flight per thread (the row gather is latency-bound at the register-
// capped occupancy).  Same slots, same order: bitwise the variant-8 rows.
struct EllL1 {
    int c;
    double dg, xc;
    unsigned pk[3];
    int nb[3];
    double uo[3];
};

template <bool NC = true>
__device__ __forceinline__ void ell_load1(const MeshArgs& a, int c, int wn, int wo, const double* __restrict__ diag,
                                          const double* __restrict__ upper_s, const double* __restrict__ x, EllL1& L)
{
    L.c = c;
    const int cc = min(c, a.N - 1), k = cc >> 5, l = c & 31;
    L.dg = __ldg(diag + cc);
    L.xc = ldx<NC>(x + cc);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        L.pk[j] = j < wn ? __ldg(a.sell_n + (size_t)32 * wn * k + 32 * j + l) : 0xFFFFFFFFu;
        L.nb[j] = j < wo ? __ldg(a.sell_o + (size_t)32 * wo * k + 32 * j + l) : -1;
        L.uo[j] = j < wo ? __ldg(upper_s + (size_t)32 * wo * k + 32 * j + l) : 0.0;
    }
}

template <int IFM, bool NC = true>
__device__ __forceinline__ void ell_finish(const MeshArgs& a, const EllL1& L, int wo, const double* __restrict__ upper_s,
                                           const double* __restrict__ iface, const double* __restrict__ x,
                                           const double* __restrict__ xr, double* __restrict__ y, double& acc, bool dot)
{
    const int cc = min(L.c, a.N - 1);
    double un[3], xn[3], xo[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const bool vn = L.pk[j] != 0xFFFFFFFFu;
        const int col = vn ? (int)(L.pk[j] >> 5) : cc;
        const int pos = (int)(L.pk[j] & 31u);
        un[j] = vn ? __ldg(upper_s + (size_t)32 * wo * (col >> 5) + 32 * pos + (col & 31)) : 0.0;
        xn[j] = ldx<NC>(x + col);
        xo[j] = ldx<NC>(x + (L.nb[j] >= 0 ? L.nb[j] : cc));
    }
    double s = L.dg * L.xc;
#pragma unroll
    for (int j = 0; j < 3; ++j)
        if (L.pk[j] != 0xFFFFFFFFu) s = s + un[j] * xn[j];
#pragma unroll
    for (int j = 0; j < 3; ++j)
        if (L.nb[j] >= 0) s = s + L.uo[j] * xo[j];
    if constexpr (IFM == 1) s = add_iface(a, cc, s, iface, xr);
    if (L.c < a.N) {
        y[cc] = s;
        if (dot && (IFM != 2 || !is_iface_row(a, cc))) acc += s * L.xc;
    }
}

// the grid-stride row loop of variant 10 (rev: descending, SPUMA_OPT_ALT_SWEEP)
template <int IFM>
__device__ __forceinline__ void amul_ell_pipelined(const MeshArgs& a, const double* __restrict__ diag,
                                                   const double* __restrict__ upper,
                                                   const double* __restrict__ iface, const double* __restrict__ x,
                                                   const double* __restrict__ xr, double* __restrict__ y, double& acc,
                                                   bool dot, int rev)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int st = gridDim.x * blockDim.x, t00 = (blockIdx.x * (blockDim.x / 32) + warp) * 32;
    const int cnt = t00 < a.N ? (a.N - 1 - t00) / st + 1 : 0;
    const int wn = a.ell_wn, wo = a.ell_wo;
    if (wn > 3 || wo > 3) {  // not an ELL mesh: plain per-row gathers
        for (int j = 0; j < cnt; ++j) {
            const int c = t00 + (rev ? cnt - 1 - j : j) * st + lane;
            if (c < a.N) {
                const double v = amul_row(a, c, diag, upper, iface, x, xr, nullptr, IFM != 2);
                y[c] = v;
                if (dot && (IFM != 2 || !is_iface_row(a, c))) acc += v * x[c];
            }
        }
        return;
    }
    EllL1 cur, nxt;
    if (cnt > 0) ell_load1(a, t00 + (rev ? cnt - 1 : 0) * st + lane, wn, wo, diag, a.upper_s, x, cur);
    for (int j = 0; j < cnt; ++j) {
        if (j + 1 < cnt) ell_load1(a, t00 + (rev ? cnt - 2 - j : j + 1) * st + lane, wn, wo, diag, a.upper_s, x, nxt);
        ell_finish<IFM>(a, cur, wo, a.upper_s, iface, x, xr, y, acc, dot);
        cur = nxt;
    }
}

// ---------------------------------------------------------------------------- variant 12 (lattice slots)
// A structured numbering (host.h lattice_offsets: every face's column offset is one of K <= 3
// values D[t], e.g. {1, n, n^2} for an n^3 block) needs no index arrays: slot t of row c is the
// face (c, c + D[t]) with its coefficient at upper_d[t S + c] (kLatAbsent where the row has no
// such face), and the neighbour-side face (c - D[t], c) is slot t of row c - D[t].  Every
// address of a row is therefore a function of c alone -- diag[c], x[c], the K owner-side slots
// (streamed), the K neighbour-side slots and the 2K x values (32-cell windows of the warp, L2
// hits) are all issued at once: ONE dependent level instead of the ELL rows' two, and
// 24 + 8K DRAM bytes per cell instead of 24 + 16 per face.  Same order as the oracle (reading
// Q10): diag x, the neighbour side by ascending owner (t = K-1 .. 0), the owner side by
// ascending neighbour (t = 0 .. K-1) -- bitwise the rows of every other variant.
__device__ __forceinline__ bool lat_present(double u)
{
    return (unsigned long long)__double_as_longlong(u) != kLatAbsent;
}

// one 32R-row chunk of the lattice rows (an interior-chunk version without the range clamps was
// measured 0.3 % slower and removed, profiles/r02_lattice_ab.md)
// x loads of the lattice rows: the read-only path, or (NC = false, the persistent loop of loop.cu,
// where x is rewritten between grid barriers inside one launch) plain coherent loads
template <int R, int IFM, int KT, bool NC = true>
__device__ __forceinline__ void lat_chunk(const MeshArgs& a, int K, int ch, const double* __restrict__ diag,
                                          const double* const (&ud)[3], const double* __restrict__ iface,
                                          const double* __restrict__ x, const double* __restrict__ xr,
                                          double* __restrict__ y, double& acc, bool dot)
{
    const int N = a.N, lane = threadIdx.x & 31;
    int c[R];
    double dg[R], xc[R], uo[R][3], xo[R][3], un[R][3], xn[R][3];
    bool on[R][3];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        c[r] = ch * 32 * R + 32 * r + lane;
        const int cc = min(c[r], N - 1);
        dg[r] = __ldg(diag + cc);
        xc[r] = ldx<NC>(x + cc);
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            if (t < K) {
                const int D = a.lat_D[t];
                const int o = cc - D;
                on[r][t] = o >= 0;
                const int oc = o >= 0 ? o : cc;
                uo[r][t] = __ldg(ud[t] + cc);
                xo[r][t] = ldx<NC>(x + min(cc + D, N - 1));
                un[r][t] = __ldg(ud[t] + oc);
                xn[r][t] = ldx<NC>(x + oc);
            } else {
                on[r][t] = false;
                uo[r][t] = __longlong_as_double((long long)kLatAbsent);
                xo[r][t] = un[r][t] = xn[r][t] = 0.0;
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double s = dg[r] * xc[r];
#pragma unroll
        for (int t = 2; t >= 0; --t)
            if (on[r][t] && lat_present(un[r][t])) s = s + un[r][t] * xn[r][t];
#pragma unroll
        for (int t = 0; t < 3; ++t)
            if (lat_present(uo[r][t])) s = s + uo[r][t] * xo[r][t];
        if (c[r] < N) {
            if constexpr (IFM == 1) s = add_iface(a, c[r], s, iface, xr);
            y[c[r]] = s;
            if (dot && (IFM != 2 || !is_iface_row(a, c[r]))) acc += s * xc[r];
        }
    }
}

template <int R, int IFM, int KT = 0>  // KT: the offset count at compile time (0: a.lat_K at run time)
__device__ __forceinline__ void amul_lattice_k(const MeshArgs& a, const double* __restrict__ diag,
                                               const double* __restrict__ iface, const double* __restrict__ x,
                                               const double* __restrict__ xr, double* __restrict__ y, double& acc,
                                               bool dot, int rev)
{
    const int N = a.N, K = KT ? KT : a.lat_K;
    const long long S = a.lat_S;
    const double* const ud[3] = {a.upper_d, a.upper_d + S, a.upper_d + 2 * S};
    const int warp = threadIdx.x >> 5;
    const int nw = gridDim.x * (blockDim.x >> 5), wid = blockIdx.x * (blockDim.x >> 5) + warp;
    const int nch = (N + 32 * R - 1) / (32 * R);
    const int cnt = wid < nch ? (nch - 1 - wid) / nw + 1 : 0;
    for (int j = 0; j < cnt; ++j) {
        const int ch = wid + (rev ? cnt - 1 - j : j) * nw;
        lat_chunk<R, IFM, KT>(a, K, ch, diag, ud, iface, x, xr, y, acc, dot);
    }
}

// the 3-D lattice (K = 3, every hex-block numbering) with the slot loop unrolled at compile time
template <int R, int IFM>
__device__ __forceinline__ void amul_lattice(const MeshArgs& a, const double* __restrict__ diag,
                                             const double* __restrict__ iface, const double* __restrict__ x,
                                             const double* __restrict__ xr, double* __restrict__ y, double& acc,
                                             bool dot, int rev)
{
#if !defined(SPUMA_LAT_K3) || SPUMA_LAT_K3
    if (a.lat_K == 3) {
        amul_lattice_k<R, IFM, 3>(a, diag, iface, x, xr, y, acc, dot, rev);
        return;
    }
#endif
    amul_lattice_k<R, IFM, 0>(a, diag, iface, x, xr, y, acc, dot, rev);
}

// ---------------------------------------------------------------------------- variant 3 (TMA)
namespace tma {

constexpr int kCells = 128;          // cells per tile == consumer threads
constexpr int kCons = kCells;        // consumer threads
constexpr int kBlock = kCons + 32;   // + one producer warp
constexpr int kCap = 448;            // faces per side per stage (3.5 per cell)
constexpr int kStages = 2;

struct Meta {
    int c0, n, f0, f1, k0, k1;
    int offU, offN, offK, staged;
};

struct Stage {
    alignas(16) double up[kCap + 2];     // upper[a0 .. a1)           owner side
    alignas(16) double xx[kCells];       // x[c0 .. c0+n)
    alignas(16) double dg[kCells];       // diag[c0 .. c0+n)
    alignas(16) int nb[kCap + 4];        // neighbour[b0 .. b1)       owner side
    alignas(16) int lo[kCap + 4];        // losort[q0 .. q1)          neighbour side
    alignas(16) int ol[kCap + 4];        // ownerLo[q0 .. q1)
    alignas(16) int os[kCells + 4];      // ownerStart[c0 .. c0+n]
    alignas(16) int ls[kCells + 4];      // losortStart[c0 .. c0+n]
    Meta meta;
};

struct Smem {
    Stage st[kStages];
    alignas(16) double prodN[kCap];
    alignas(16) double prodO[kCap];
    alignas(8) unsigned long long full[kStages];
    alignas(8) unsigned long long empty[kStages];
};

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(unsigned long long* b, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void bar_arrive(unsigned long long* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void bar_arrive_tx(unsigned long long* b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* b, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(s32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s32(dst)),
                 "l"(src), "r"(bytes), "r"(s32(b))
                 : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory"); }

// Lengths (elements) the windows may not exceed: internal arrays are padded by
// 8 elements; caller arrays (upper, diag, and x in the diagnostic Amul) are not.
struct Bounds {
    long long upper_len, x_len, diag_len;
    int sell_wn, sell_wo;  // uniform SELL widths, or -1 (per-chunk meta)
};

template <bool DOT>
__device__ double amul_tma(const MeshArgs& a, const double* __restrict__ diag, const double* __restrict__ upper,
                           const double* __restrict__ iface, const double* __restrict__ x,
                           const double* __restrict__ xr, double* __restrict__ y, Bounds bd, Smem& sm)
{
    const int tid = threadIdx.x;
    const int n_tiles = (a.N + kCells - 1) / kCells;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            bar_init(&sm.full[s], 1);
            bar_init(&sm.empty[s], 1);
        }
        bar_fence_init();
    }
    __syncthreads();
    double acc = 0.0;
    if (tid >= kCons) {
        // ------------------------------------------------------------ producer warp
        if (tid == kCons) {
            int i = 0;
            int tile = blockIdx.x;
            int nf0 = 0, nf1 = 0, nk0 = 0, nk1 = 0;
            if (tile < n_tiles) {
                const int c0 = tile * kCells, n = min(kCells, a.N - c0);
                nf0 = __ldg(a.ownerStart + c0);
                nf1 = __ldg(a.ownerStart + c0 + n);
                nk0 = __ldg(a.losortStart + c0);
                nk1 = __ldg(a.losortStart + c0 + n);
            }
            for (; tile < n_tiles; ++i, tile += gridDim.x) {
                const int s = i % kStages, u = i / kStages;
                const int c0 = tile * kCells, n = min(kCells, a.N - c0);
                const int f0 = nf0, f1 = nf1, k0 = nk0, k1 = nk1;
                // prefetch the next tile's extents before blocking on the stage
                const int nt = tile + gridDim.x;
                if (nt < n_tiles) {
                    const int d0 = nt * kCells, dn = min(kCells, a.N - d0);
                    nf0 = __ldg(a.ownerStart + d0);
                    nf1 = __ldg(a.ownerStart + d0 + dn);
                    nk0 = __ldg(a.losortStart + d0);
                    nk1 = __ldg(a.losortStart + d0 + dn);
                }
                if (u > 0) bar_wait(&sm.empty[s], (u - 1) & 1);
                Stage& st = sm.st[s];
                const long long a0 = f0 & ~1, a1 = (f1 + 1) & ~1;      // upper (double) window
                const long long b0 = f0 & ~3, b1 = (f1 + 3) & ~3;      // neighbour (int) window
                const long long q0 = k0 & ~3, q1 = (k1 + 3) & ~3;      // losort / ownerLo windows
                const long long x1 = (c0 + n + 1) & ~1;                // x / diag windows [c0, x1)
                const long long o1 = (c0 + n + 1 + 3) & ~3;            // ownerStart / losortStart [c0, o1)
                const bool staged = (f1 - f0) <= kCap && (k1 - k0) <= kCap && a1 <= bd.upper_len &&
                                    x1 <= bd.x_len && x1 <= bd.diag_len;
                st.meta = Meta{c0, n, f0, f1, k0, k1, (int)(f0 - a0), (int)(f0 - b0), (int)(k0 - q0), staged ? 1 : 0};
                if (!staged) {
                    bar_arrive(&sm.full[s]);
                    continue;
                }
                const uint32_t bu = (uint32_t)((a1 - a0) * 8), bn = (uint32_t)((b1 - b0) * 4);
                const uint32_t bq = (uint32_t)((q1 - q0) * 4), bx = (uint32_t)((x1 - c0) * 8);
                const uint32_t bo = (uint32_t)((o1 - c0) * 4);
                bar_arrive_tx(&sm.full[s], bu + bn + 2 * bq + 2 * bx + 2 * bo);
                if (bu) bulk_g2s(st.up, upper + a0, bu, &sm.full[s]);
                if (bn) bulk_g2s(st.nb, a.neighbour + b0, bn, &sm.full[s]);
                if (bq) {
                    bulk_g2s(st.lo, a.losort + q0, bq, &sm.full[s]);
                    bulk_g2s(st.ol, a.ownerLo + q0, bq, &sm.full[s]);
                }
                bulk_g2s(st.xx, x + c0, bx, &sm.full[s]);
                bulk_g2s(st.dg, diag + c0, bx, &sm.full[s]);
                bulk_g2s(st.os, a.ownerStart + c0, bo, &sm.full[s]);
                bulk_g2s(st.ls, a.losortStart + c0, bo, &sm.full[s]);
            }
        }
    } else {
        // ------------------------------------------------------------ consumer warps
        int i = 0;
        for (int tile = blockIdx.x; tile < n_tiles; ++i, tile += gridDim.x) {
            const int s = i % kStages, u = i / kStages;
            bar_wait(&sm.full[s], u & 1);
            Stage& st = sm.st[s];
            const Meta m = st.meta;
            const int c = m.c0 + tid;
            if (m.staged) {
                // products: gathers are independent -> all in flight at once
                const int no = m.f1 - m.f0, nn = m.k1 - m.k0;
#pragma unroll 4
                for (int j = tid; j < nn; j += kCons) {
                    const int f = st.lo[m.offK + j];
                    const int col = st.ol[m.offK + j];
                    sm.prodN[j] = __ldg(upper + f) * __ldg(x + col);
                }
#pragma unroll 4
                for (int j = tid; j < no; j += kCons) sm.prodO[j] = st.up[m.offU + j] * __ldg(x + st.nb[m.offN + j]);
                consumers_sync();
                if (tid < m.n) {
                    const double xc = st.xx[tid];
                    double r = st.dg[tid] * xc;
                    const int ke = st.ls[tid + 1] - m.k0;
                    for (int k = st.ls[tid] - m.k0; k < ke; ++k) r = r + sm.prodN[k];
                    const int fe = st.os[tid + 1] - m.f0;
                    for (int f = st.os[tid] - m.f0; f < fe; ++f) r = r + sm.prodO[f];
                    if (a.ifStart) {
                        const int j1 = a.ifStart[c + 1];
                        for (int j = a.ifStart[c]; j < j1; ++j) {
                            const int q = a.ifIdx[j];
                            r = r + iface[q] * xr[q];
                        }
                    }
                    y[c] = r;
                    if (DOT) acc += r * xc;
                }
            } else if (tid < m.n) {
                const double r = amul_row(a, c, diag, upper, iface, x, xr, nullptr);
                y[c] = r;
                if (DOT) acc += r * x[c];
            }
            consumers_sync();  // stage s and the product buffers are free
            if (tid == 0) bar_arrive(&sm.empty[s]);
        }
    }
    return acc;
}

}  // namespace tma

// ---------------------------------------------------------------------------- variant 11 (bulk ring)
// The ELL rows of variant 8 with the first dependent level moved into a per-warp ring of
// cp.async.bulk copies: each warp owns kD shared-memory stages; lane 0 issues the next chunks'
// slot indices, owner-side coefficients, diag and x (2 KB per 32-cell chunk, one mbarrier per
// stage with expect_tx) kD chunks ahead, so ~kD chunks of streamed bytes are in flight per warp
// while the lanes run the second-level gathers of the current chunk from L2.  Same slots,
// same order: bitwise the variant-8 rows.
namespace ring {

constexpr int kD = 6;              // stages per warp
constexpr int kStageBytes = 2048;  // widths <= 3: 128 wn + 128 wo + 256 wo + 256 (diag) + 256 (x)
constexpr int kWarps = kThreads / 32;
constexpr int kSmem = kWarps * kD * kStageBytes + kWarps * kD * 8;

template <int IFM, bool DOT>
__device__ __forceinline__ double amul_ring(const MeshArgs& a, const double* __restrict__ diag,
                                            const double* __restrict__ upper, const double* __restrict__ iface,
                                            const double* __restrict__ x, const double* __restrict__ xr,
                                            double* __restrict__ y, int rev)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wn = a.ell_wn, wo = a.ell_wo;
    double acc = 0.0;
    if (wn > 3 || wo > 3) {  // not an ELL mesh
        amul_ell_pipelined<IFM>(a, diag, upper, iface, x, xr, y, acc, DOT, rev);
        return acc;
    }
    unsigned char* wbase = smem + (size_t)warp * kD * kStageBytes;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + kWarps * kD * kStageBytes) + warp * kD;
    const int nchunks = (a.N + 31) >> 5, nfull = a.N >> 5;  // chunks < nfull hold 32 cells
    const int wid = blockIdx.x * kWarps + warp, wst = gridDim.x * kWarps;
    const int cnt = wid < nchunks ? (nchunks - 1 - wid) / wst + 1 : 0;
    const uint32_t bn = 128u * wn, bo = 128u * wo, bu = 256u * wo;
    const uint32_t offO = bn, offU = bn + bo, offD = bn + bo + bu, offX = offD + 256u;
    auto chunk = [&](int j) { return wid + (rev ? cnt - 1 - j : j) * wst; };
    auto issue = [&](int j) {  // lane 0: stage j's copies into slot j % kD
        const int k = chunk(j);
        if (k >= nfull) return;
        unsigned char* st = wbase + (size_t)(j % kD) * kStageBytes;
        unsigned long long* b = &bar[j % kD];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the lanes' reads of the slot first
        tma::bar_arrive_tx(b, bn + bo + bu + 512u);
        if (bn) tma::bulk_g2s(st, a.sell_n + (size_t)32 * wn * k, bn, b);
        if (bo) {
            tma::bulk_g2s(st + offO, a.sell_o + (size_t)32 * wo * k, bo, b);
            tma::bulk_g2s(st + offU, a.upper_s + (size_t)32 * wo * k, bu, b);
        }
        tma::bulk_g2s(st + offD, diag + (size_t)32 * k, 256u, b);
        tma::bulk_g2s(st + offX, x + (size_t)32 * k, 256u, b);
    };
    if (lane == 0) {
        for (int s = 0; s < kD; ++s) tma::bar_init(&bar[s], 1);
        tma::bar_fence_init();
        for (int j = 0; j < kD && j < cnt; ++j) issue(j);
    }
    __syncwarp();
    uint32_t phase = 0;  // bit s: the parity slot s completes next
    for (int j = 0; j < cnt; ++j) {
        const int k = chunk(j), s = j % kD;
        EllL1 L;
        if (k < nfull) {
            const unsigned char* st = wbase + (size_t)s * kStageBytes;
            tma::bar_wait(&bar[s], (phase >> s) & 1u);
            phase ^= 1u << s;
            const unsigned* sn = reinterpret_cast<const unsigned*>(st);
            const int* so = reinterpret_cast<const int*>(st + offO);
            const double* su = reinterpret_cast<const double*>(st + offU);
            L.c = 32 * k + lane;
            L.dg = reinterpret_cast<const double*>(st + offD)[lane];
            L.xc = reinterpret_cast<const double*>(st + offX)[lane];
#pragma unroll
            for (int jj = 0; jj < 3; ++jj) {
                L.pk[jj] = jj < wn ? sn[32 * jj + lane] : 0xFFFFFFFFu;
                L.nb[jj] = jj < wo ? so[32 * jj + lane] : -1;
                L.uo[jj] = jj < wo ? su[32 * jj + lane] : 0.0;
            }
        } else {  // the partial last chunk: plain loads (its slot was never filled)
            ell_load1(a, 32 * k + lane, wn, wo, diag, a.upper_s, x, L);
        }
        __syncwarp();
        if (lane == 0 && j + kD < cnt) issue(j + kD);
        ell_finish<IFM>(a, L, wo, a.upper_s, iface, x, xr, y, acc, DOT);
    }
    return acc;
}

}  // namespace ring
}  // namespace spuma
