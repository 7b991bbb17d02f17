// gamg.cu -- sm_100a kernels of GAMG with the Richardson smoother (
// PAPER.md P:665, profile rows P:517-545; readings Q22-Q28 in DESIGN.md §3).
//
// Every level is an lduAddressing mesh, so every operator is a per-row GATHER in the
// oracle's face order (Q10) -- bitwise the oracle's row values (--fmad=false).  The
// V-cycle fuses what the oracle does in separate passes where the data allows:
//   restriction  b_{l+1}[C] = sum over the fine cells of C of (b - A x)  (one kernel per
//                level, per COARSE cell; the residual is formed on the fly)
//   prolongation + scale + first post-sweep: the correction x + alpha xc[ftc[j]] is
//                evaluated inside the sweep's row gather, never stored
//   last post-sweep on level 0 accumulates straight into psi
// Reductions (scale factor, residual norm) use the fixed-shape last-CTA pattern.
#include "device.cuh"
#include "internal.h"

namespace spuma {
namespace {

// row of A applied to an implicit vector x(j), in the oracle's order (Q10, no interfaces).
// ul: the coefficients in losort order (coarse levels, written by k_gamg_agg) -- a stream
// instead of the upper[losort[k]] gather; nullptr: gather.
template <class X>
__device__ __forceinline__ double row_ax(const MeshArgs& a, int c, const double* __restrict__ diag,
                                         const double* __restrict__ upper, const X& x,
                                         const double* __restrict__ ul = nullptr)
{
    double s = diag[c] * x(c);
    const int k1 = a.losortStart[c + 1];
    if (ul)
        for (int k = a.losortStart[c]; k < k1; ++k) s = s + ul[k] * x(a.ownerLo[k]);
    else
        for (int k = a.losortStart[c]; k < k1; ++k) s = s + upper[a.losort[k]] * x(a.ownerLo[k]);
    const int f1 = a.ownerStart[c + 1];
    for (int f = a.ownerStart[c]; f < f1; ++f) s = s + upper[f] * x(a.neighbour[f]);
    return s;
}

// The same row over the ELL layout of a uniform mesh (level 0): slot j of the
// 32-cell chunk of c, neighbour side packed (owner column << 5 | position), coefficients in
// owner-slot order (upper_s).  Same summation order as row_ax, so bitwise the same value.
template <class X>
__device__ __forceinline__ double row_ax_ell(const MeshArgs& a, int c, const double* __restrict__ diag, const X& x)
{
    constexpr int W = 3;
    const int wn = a.ell_wn, wo = a.ell_wo, k = c >> 5, l = c & 31;
    unsigned pk[W];
    int nb[W];
    double uo[W], un[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
        pk[j] = j < wn ? __ldg(a.sell_n + (size_t)32 * wn * k + 32 * j + l) : 0xFFFFFFFFu;
        nb[j] = j < wo ? __ldg(a.sell_o + (size_t)32 * wo * k + 32 * j + l) : -1;
        uo[j] = j < wo ? __ldg(a.upper_s + (size_t)32 * wo * k + 32 * j + l) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < W; ++j) {
        const int col = (int)(pk[j] >> 5), pos = (int)(pk[j] & 31u);
        un[j] = pk[j] != 0xFFFFFFFFu ? __ldg(a.upper_s + (size_t)32 * wo * (col >> 5) + 32 * pos + (col & 31)) : 0.0;
    }
    double s = diag[c] * x(c);
#pragma unroll
    for (int j = 0; j < W; ++j)
        if (pk[j] != 0xFFFFFFFFu) s = s + un[j] * x((int)(pk[j] >> 5));
#pragma unroll
    for (int j = 0; j < W; ++j)
        if (nb[j] >= 0) s = s + uo[j] * x(nb[j]);
    return s;
}

// The same row over a per-level CSR copy of the off-diagonal coefficients (coarse generic levels):
// row c's neighbour-side faces in losort order, then its owner-side faces in face order -- the
// order of row_ax -- as one contiguous (column, value) run; values written by k_gamg_agg.
template <class X>
__device__ __forceinline__ double row_ax_csr(const GLevel& L, int c, const double* __restrict__ diag, const X& x)
{
    double s = diag[c] * x(c);
    const int k1 = L.crp[c + 1];
    for (int k = L.crp[c]; k < k1; ++k) s = s + L.cval[k] * x(L.ccol[k]);
    return s;
}

// + the processor-interface terms of row c in (patch, face) order (Q10), reading the halo xr
// of the same implicit vector (packed by the neighbours before this kernel)
template <bool IF>
__device__ __forceinline__ double add_if(const GLevel& L, const double* __restrict__ ic, int c, double s)
{
    if constexpr (IF) {
        const int k1 = L.a.ifStart[c + 1];
        for (int k = L.a.ifStart[c]; k < k1; ++k) {
            const int i = L.a.ifIdx[k];
            s = s + ic[i] * L.xr[i];
        }
    }
    return s;
}

template <int LAY, bool IF = false, class X>
__device__ __forceinline__ double rowA(const GLevel& L, int c, const double* __restrict__ d,
                                       const double* __restrict__ u, const double* __restrict__ ic, const X& x)
{
    double s;
    if constexpr (LAY == 1) s = row_ax_ell(L.a, c, d, x);
    else if constexpr (LAY == 2) s = row_ax_csr(L, c, d, x);
    else s = row_ax(L.a, c, d, u, x, L.upperLo);
    return add_if<IF>(L, ic, c, s);
}

struct XPlain {
    const double* __restrict__ x;
    __device__ __forceinline__ double operator()(int j) const { return x[j]; }
};

// x(j) = x[j] + alpha xc[ftc[j]]  (prolongation by injection, scaled; x == nullptr: zero)
struct XCorr {
    const double* __restrict__ x;
    const double* __restrict__ xc;
    const int* __restrict__ ftc;
    double alpha;
    __device__ __forceinline__ double operator()(int j) const
    {
        return (x ? x[j] : 0.0) + alpha * xc[ftc[j]];
    }
};

struct XZero {
    __device__ __forceinline__ double operator()(int) const { return 0.0; }
};

struct XInj {  // c(j) = xc[ftc[j]]
    const double* __restrict__ xc;
    const int* __restrict__ ftc;
    __device__ __forceinline__ double operator()(int j) const { return xc[ftc[j]]; }
};

__device__ __forceinline__ const double* level_diag(const GLevel& L, const DevPtrs* P)
{
    return L.diag ? L.diag : P->diag;
}
__device__ __forceinline__ const double* level_upper(const GLevel& L, const DevPtrs* P)
{
    return L.upper ? L.upper : P->upper;
}
__device__ __forceinline__ const double* level_iface(const GLevel& L, const DevPtrs* P)
{
    return L.iface ? L.iface : P->iface;
}

// agglomerateMatrix (Q27): coarse diag = fine diags of the members (ascending) + (u + l) of
// the agglomerate-internal faces (ascending); coarse upper = fine uppers of its faces.
__global__ void __launch_bounds__(kThreads) k_gamg_agg(GLevel F, GLevel C, const DevPtrs* __restrict__ P)
{
    const double* __restrict__ fd = level_diag(F, P);
    const double* __restrict__ fu = level_upper(F, P);
    const int stride = gridDim.x * blockDim.x;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < F.nc; c += stride) {
        double d = 0.0;
        for (int k = F.cStart[c]; k < F.cStart[c + 1]; ++k) d = d + fd[F.cList[k]];
        for (int k = F.ciStart[c]; k < F.ciStart[c + 1]; ++k) {
            const double u = fu[F.ciList[k]];
            d = d + (u + u);
        }
        C.diag[c] = d;
    }
    if (F.cifStart) {  // coarse interface coefficients: sums of the fine ones, ascending (Q37)
        const double* __restrict__ fi = level_iface(F, P);
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < F.ncif; e += stride) {
            double v = 0.0;
            for (int k = F.cifStart[e]; k < F.cifStart[e + 1]; ++k) v = v + fi[F.cifList[k]];
            const_cast<double*>(C.iface)[e] = v;
        }
    }
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < F.ncf; e += stride) {
        double u = 0.0;
        for (int k = F.cfStart[e]; k < F.cfStart[e + 1]; ++k) u = u + fu[F.cfList[k]];
        C.upper[e] = u;
        if (C.upperLo) C.upperLo[C.losortPos[e]] = u;  // losort-ordered copy (generic rows)
        if (C.cval) {                                  // CSR rows: both entries of the face
            C.cval[C.cposU[e]] = u;
            C.cval[C.cposL[e]] = u;
        }
        if (C.ell) {  // owner-slot copy for the ELL rows of the coarse level
            const int c = C.a.owner[e];
            const_cast<double*>(C.a.upper_s)[(size_t)32 * C.a.ell_wo * (c >> 5) + 32 * (e - C.a.ownerStart[c]) + (c & 31)] = u;
        }
    }
}

// restrictField of the residual (Q23): C.b[c] = sum_{i in c} (b_i - (A x)_i); r_i stored
// for the scale step when x is not zero.
template <bool IF>
__global__ void __launch_bounds__(kThreads) k_gamg_restrict(GLevel F, GLevel C, const DevPtrs* __restrict__ P,
                                                            const double* __restrict__ x, double* __restrict__ zero_x)
{
    pdl_wait();  // predecessor complete and visible (PDL launch)
    pdl_trigger();
    const double* __restrict__ fd = level_diag(F, P);
    const double* __restrict__ fu = level_upper(F, P);
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < F.nc; c += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = F.cStart[c]; k < F.cStart[c + 1]; ++k) {
            const int i = F.cList[k];
            double r = F.b[i];
            if (x) {
                r = r - add_if<IF>(F, level_iface(F, P), i, (F.cval ? row_ax_csr(F, i, fd, XPlain{x}) : row_ax(F.a, i, fd, fu, XPlain{x}, F.upperLo)));
                F.r[i] = r;
            }
            s = s + r;
        }
        C.b[c] = s;
        if (zero_x) zero_x[c] = 0.0;
    }
}

// Richardson sweep (Q24): xout = x + omega (rD (b - A x)), x = xin or (xin + alpha xc[ftc])
// when xc is given (the prolonged correction of the first post-sweep); psi_acc: psi += xout.
template <int ELL, bool IF>
__global__ void __launch_bounds__(kThreads) k_gamg_smooth(GLevel L, const DevPtrs* __restrict__ P,
                                                          const double* __restrict__ xin, double* __restrict__ xout,
                                                          double omega, const double* __restrict__ xc,
                                                          const double* __restrict__ alpha, int psi_acc)
{
    pdl_wait();  // predecessor complete and visible (PDL launch)
    pdl_trigger();
    const double* __restrict__ d = level_diag(L, P);
    const double* __restrict__ u = level_upper(L, P);
    const double* __restrict__ ic = level_iface(L, P);
    double* __restrict__ psi = P->psi;
    const double a = alpha ? *alpha : 1.0;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.a.N; c += gridDim.x * blockDim.x) {
        double xi, y;
        if (xc) {
            const XCorr X{xin, xc, L.ftc, a};
            xi = X(c);
            y = rowA<ELL, IF>(L, c, d, u, ic, X);
        } else if (xin) {
            xi = xin[c];
            y = rowA<ELL, IF>(L, c, d, u, ic, XPlain{xin});
        } else {  // x == 0 (first pre-sweep)
            xi = 0.0;
            y = rowA<ELL, IF>(L, c, d, u, ic, XZero{});
        }
        const double xn = xi + omega * ((1.0 / d[c]) * (L.b[c] - y));
        if (psi_acc) psi[c] = psi[c] + xn;
        else xout[c] = xn;
    }
}

// GAMGSolver::scale reading (Q25): alpha = (c.r)/(c.Ac) clamped to [0, 2], c = xc[ftc].
// With pq (nPost >= 1) the first post-sweep is prepared here, split by linearity in alpha
// (reading Q29): with x' = x + alpha c,  A x' = (b - r) + alpha Ac, so the sweep
//   x1 = x' + omega rD (r - alpha Ac) = alpha p + q,
//   p = c - omega rD Ac,  q = x + omega rD r       (x = pre-smoothed correction or 0)
// and k_gamg_post needs two direct loads per neighbour instead of a gather of its own.
template <int ELL, bool IF>
__global__ void __launch_bounds__(kThreads) k_gamg_scale(GLevel L, const DevPtrs* __restrict__ P,
                                                         const double* __restrict__ x, const double* __restrict__ xc,
                                                         const double* __restrict__ r, double omega, int pq,
                                                         double* part, unsigned* ticket, double* alpha,
                                                         double* rank_part)
{
    pdl_wait();  // predecessor complete and visible (PDL launch)
    pdl_trigger();
    const double* __restrict__ d = level_diag(L, P);
    const double* __restrict__ u = level_upper(L, P);
    const double* __restrict__ ic = level_iface(L, P);
    const XInj X{xc, L.ftc};
    double v[2] = {0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.a.N; c += gridDim.x * blockDim.x) {
        const double ci = X(c);
        const double aci = rowA<ELL, IF>(L, c, d, u, ic, X);
        const double ri = r[c];
        if (pq) {
            const double rd = 1.0 / d[c];
            L.p[c] = ci - omega * (rd * aci);
            L.q[c] = (x ? x[c] : 0.0) + omega * (rd * ri);
        }
        v[0] += ci * ri;
        v[1] += aci * ci;
    }
    if (grid_sum<2>(v, part, ticket) && threadIdx.x == 0) {
        if (rank_part) {  // n_ranks > 1: this rank's two dots; alpha by k_gamg_fin after the all-gather
            rank_part[0] = v[0];
            rank_part[1] = v[1];
            rank_part[2] = 0.0;
            rank_part[3] = 0.0;
            return;
        }
        double a = fabs(v[1]) > 1e-300 ? v[0] / v[1] : 1.0;
        a = a < 0.0 ? 0.0 : (a > 2.0 ? 2.0 : a);
        *alpha = a;
    }
}

// x + alpha xc[ftc] without a post-sweep (nPost = 0); psi_acc: psi += it
__global__ void __launch_bounds__(kThreads) k_gamg_correct(GLevel L, const DevPtrs* __restrict__ P,
                                                           const double* __restrict__ x, const double* __restrict__ xc,
                                                           const double* __restrict__ alpha, double* __restrict__ out,
                                                           int psi_acc)
{
    pdl_wait();  // predecessor complete and visible (PDL launch)
    pdl_trigger();
    const XCorr X{x, xc, L.ftc, alpha ? *alpha : 1.0};
    double* __restrict__ psi = P->psi;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.a.N; c += gridDim.x * blockDim.x) {
        const double xn = X(c);
        if (psi_acc) psi[c] = psi[c] + xn;
        else out[c] = xn;
    }
}

struct XPQ {  // x1(j) = alpha p_j + q_j
    const double* __restrict__ p;
    const double* __restrict__ q;
    double alpha;
    __device__ __forceinline__ double operator()(int j) const { return alpha * p[j] + q[j]; }
};

// Post-sweeps 1 (+2) after k_gamg_scale: x1 = alpha p + q; two: x2 = x1 + omega rD (b - A x1)
// in one gather with x1 formed at the neighbours.  psi_acc: psi += result.
template <int ELL, bool IF>
__global__ void __launch_bounds__(kThreads) k_gamg_post(GLevel L, const DevPtrs* __restrict__ P,
                                                        const double* __restrict__ alpha, double omega,
                                                        double* __restrict__ out, int two, int psi_acc)
{
    pdl_wait();  // predecessor complete and visible (PDL launch)
    pdl_trigger();
    const double* __restrict__ d = level_diag(L, P);
    const double* __restrict__ u = level_upper(L, P);
    const double* __restrict__ ic = level_iface(L, P);
    double* __restrict__ psi = P->psi;
    const XPQ X{L.p, L.q, *alpha};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.a.N; c += gridDim.x * blockDim.x) {
        const double x1 = X(c);
        double xn = x1;
        if (two) xn = x1 + omega * ((1.0 / d[c]) * (L.b[c] - rowA<ELL, IF>(L, c, d, u, ic, X)));
        if (psi_acc) psi[c] = psi[c] + xn;
        else out[c] = xn;
    }
}

// Two-stage Gauss-Seidel (Q30), stage 1: r = b - A x' with x' = xin (+ alpha xc[ftc] when xc
// is given: the prolonged correction folded into the first post-sweep; xin nullptr: zero).
template <int ELL, bool IF>
__global__ void __launch_bounds__(kThreads) k_gamg_gs2_res(GLevel L, const DevPtrs* __restrict__ P,
                                                           const double* __restrict__ xin,
                                                           const double* __restrict__ xc,
                                                           const double* __restrict__ alpha, double* __restrict__ r)
{
    pdl_wait();  // predecessor complete and visible (PDL launch)
    pdl_trigger();
    const double* __restrict__ d = level_diag(L, P);
    const double* __restrict__ u = level_upper(L, P);
    const double* __restrict__ ic = level_iface(L, P);
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.a.N; c += gridDim.x * blockDim.x) {
        double y;
        if (xc) y = rowA<ELL, IF>(L, c, d, u, ic, XCorr{xin, xc, L.ftc, alpha ? *alpha : 1.0});
        else if (xin) y = rowA<ELL, IF>(L, c, d, u, ic, XPlain{xin});
        else y = rowA<ELL, IF>(L, c, d, u, ic, XZero{});
        r[c] = L.b[c] - y;
    }
}

// Stage 2, one Jacobi-Richardson iteration of (D + L) z = r:  z = rD (r - L zprev), the
// lower sum over the faces with neighbour c in face (losort) order; zprev = zin, or rD r
// when zin is nullptr (the first iteration).  last: x = x' + z (psi_acc: psi += x) instead
// of storing z.  n_inner == 0 is one launch with skip_lower (z = rD r).
__global__ void __launch_bounds__(kThreads) k_gamg_gs2_upd(GLevel L, const DevPtrs* __restrict__ P,
                                                           const double* __restrict__ xin,
                                                           const double* __restrict__ xc,
                                                           const double* __restrict__ alpha,
                                                           const double* __restrict__ r,
                                                           const double* __restrict__ zin, double* __restrict__ out,
                                                           int skip_lower, int last, int psi_acc)
{
    pdl_wait();  // predecessor complete and visible (PDL launch)
    pdl_trigger();
    const double* __restrict__ d = level_diag(L, P);
    const double* __restrict__ u = level_upper(L, P);
    double* __restrict__ psi = P->psi;
    const double a = alpha ? *alpha : 1.0;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.a.N; c += gridDim.x * blockDim.x) {
        double t = r[c];
        if (!skip_lower) {
            const int k0 = L.a.losortStart[c], k1 = L.a.losortStart[c + 1];
            if (L.cval) {  // the lower part = the first k1 - k0 entries of the row's CSR run
                const int q0 = L.crp[c];
                for (int k = 0; k < k1 - k0; ++k) {
                    const int j = L.ccol[q0 + k];
                    const double zj = zin ? zin[j] : (1.0 / d[j]) * r[j];
                    t = t - L.cval[q0 + k] * zj;
                }
            } else if (L.upperLo) {
                for (int k = k0; k < k1; ++k) {
                    const int j = L.a.ownerLo[k];
                    const double zj = zin ? zin[j] : (1.0 / d[j]) * r[j];
                    t = t - L.upperLo[k] * zj;
                }
            } else {
                for (int k = k0; k < k1; ++k) {
                    const int j = L.a.ownerLo[k];
                    const double zj = zin ? zin[j] : (1.0 / d[j]) * r[j];
                    t = t - u[L.a.losort[k]] * zj;
                }
            }
        }
        const double z = (1.0 / d[c]) * t;
        if (!last) {
            out[c] = z;
            continue;
        }
        const double xp = xc ? XCorr{xin, xc, L.ftc, a}(c) : (xin ? xin[c] : 0.0);
        const double xn = xp + z;
        if (psi_acc) psi[c] = psi[c] + xn;
        else out[c] = xn;
    }
}

// end of a GAMG iteration (Q28): rA = source - A psi, final residual, n++, convergence, done
template <int ELL, bool IF>
__global__ void __launch_bounds__(kThreads) k_gamg_residual(GLevel L, Workspace w, double* rank_part)
{
    pdl_wait();  // predecessor complete and visible (PDL launch)
    pdl_trigger();
    const DevPtrs p = *w.ptrs;
    double v[1] = {0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.a.N; c += gridDim.x * blockDim.x) {
        const double r = p.source[c] - rowA<ELL, IF>(L, c, p.diag, p.upper, p.iface, XPlain{p.psi});
        w.rA[c] = r;
        v[0] += fabs(r);
    }
    if (grid_sum<1>(v, w.part, &w.scal->ticket[2]) && threadIdx.x == 0) {
        if (rank_part) {  // n_ranks > 1: finished by k_gamg_fin after the all-gather
            rank_part[0] = v[0];
            rank_part[1] = rank_part[2] = rank_part[3] = 0.0;
            return;
        }
        DevScal* s = w.scal;
        s->fin = v[0] / s->normFactor;
        s->n = s->n + 1;
        const bool c = conv(s->fin, s->init, s->tol, s->rel_tol);
        s->converged = c;
        if (!((s->n < s->max_iter && !c) || s->n < s->min_iter)) s->done = 1;
    }
}

// halo source of the level's next row kernel (n_ranks > 1): the implicit vector at the
// interface cells, formed exactly as the row kernels form it (same rounding)
__global__ void __launch_bounds__(kThreads) k_gamg_pack(GLevel L, int mode, const double* __restrict__ x,
                                                        const double* __restrict__ xc,
                                                        const double* __restrict__ alpha,
                                                        const double* __restrict__ p, const double* __restrict__ q)
{
    const double a = alpha ? *alpha : 1.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L.n_if; i += gridDim.x * blockDim.x) {
        const int c = L.if_cell[i];
        double v;
        if (mode == 1) v = XCorr{x, xc, L.ftc, a}(c);
        else if (mode == 2) v = XInj{xc, L.ftc}(c);
        else if (mode == 3) v = XPQ{p, q, a}(c);
        else v = x ? x[c] : 0.0;
        L.sendbuf[i] = v;
    }
}

// rank-order sums of the gathered partials (every rank computes the same bits)
__global__ void k_gamg_fin(int what, const double* __restrict__ g, int n_ranks, double* alpha, DevScal* s)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double v0 = 0.0, v1 = 0.0;
    for (int r = 0; r < n_ranks; ++r) {
        v0 += g[4 * r];
        v1 += g[4 * r + 1];
    }
    if (what == 0) {  // Q25
        double a = fabs(v1) > 1e-300 ? v0 / v1 : 1.0;
        *alpha = a < 0.0 ? 0.0 : (a > 2.0 ? 2.0 : a);
        return;
    }
    s->fin = v0 / s->normFactor;  // Q28
    s->n = s->n + 1;
    const bool c = conv(s->fin, s->init, s->tol, s->rel_tol);
    s->converged = c;
    if (!((s->n < s->max_iter && !c) || s->n < s->min_iter)) s->done = 1;
}

// The small levels t..nl-1 of a V-cycle in ONE CTA (Richardson, scaled correction, nPre = 0):
// restrictions down, the coarsest PCG (pcg_single_body), then per level the scale step and the
// fused post-sweeps, phases separated by __syncthreads() instead of ~3 launches per level.
// Same arithmetic as the per-level kernels (only the reduction shape of the scale dots
// differs).  Level t's b comes from the preceding restriction kernel; its result is left in
// lv[t].x or lv[t].x2 exactly as the per-level path leaves it.
__global__ void __launch_bounds__(kSmallThreads) k_gamg_tail(const GLevel* __restrict__ lv, int t, int nl,
                                                             Workspace cws, double omega, int n_post)
{
    pdl_wait();
    const int tid = threadIdx.x;
    __shared__ double s_alpha;
    for (int l = t; l + 1 < nl; ++l) {  // restriction (x_l = 0: r = b)
        const GLevel& L = lv[l];
        const GLevel& C = lv[l + 1];
        for (int c = tid; c < L.nc; c += kSmallThreads) {
            double s = 0.0;
            for (int k = L.cStart[c]; k < L.cStart[c + 1]; ++k) s = s + L.b[L.cList[k]];
            C.b[c] = s;
            if (l + 2 == nl) C.x[c] = 0.0;
        }
        __syncthreads();
    }
    pcg_single_body(lv[nl - 1].a, cws);
    __syncthreads();
    for (int l = nl - 2; l >= t; --l) {
        const GLevel& L = lv[l];
        const GLevel& C = lv[l + 1];
        const double* xc = (l + 1 == nl - 1 || n_post == 1 || ((n_post - 2) & 1) == 0) ? C.x : C.x2;
        const double* d = L.diag;
        const double* u = L.upper;
        const XInj X{xc, L.ftc};
        double v[2] = {0.0, 0.0};
        for (int c = tid; c < L.a.N; c += kSmallThreads) {  // scale + p/q (Q25, Q29)
            const double ci = X(c);
            const double aci = L.ell ? row_ax_ell(L.a, c, d, X) : (L.cval ? row_ax_csr(L, c, d, X) : row_ax(L.a, c, d, u, X, L.upperLo));
            const double ri = L.b[c];
            const double rd = 1.0 / d[c];
            L.p[c] = ci - omega * (rd * aci);
            L.q[c] = 0.0 + omega * (rd * ri);
            v[0] += ci * ri;
            v[1] += aci * ci;
        }
        cta_sum_1024<2>(v);
        if (tid == 0) {
            double a = fabs(v[1]) > 1e-300 ? v[0] / v[1] : 1.0;
            s_alpha = a < 0.0 ? 0.0 : (a > 2.0 ? 2.0 : a);
        }
        __syncthreads();
        const XPQ Y{L.p, L.q, s_alpha};
        for (int c = tid; c < L.a.N; c += kSmallThreads) {  // post-sweeps 1 (+2)
            const double x1 = Y(c);
            double xn = x1;
            if (n_post >= 2)
                xn = x1 + omega * ((1.0 / d[c]) * (L.b[c] - (L.ell ? row_ax_ell(L.a, c, d, Y) : (L.cval ? row_ax_csr(L, c, d, Y) : row_ax(L.a, c, d, u, Y, L.upperLo)))));
            L.x[c] = xn;
        }
        __syncthreads();
        double* xin = L.x;
        double* xout = L.x2;
        for (int i = 2; i < n_post; ++i) {  // further plain sweeps
            for (int c = tid; c < L.a.N; c += kSmallThreads) {
                const XPlain Z{xin};
                const double y = L.ell ? row_ax_ell(L.a, c, d, Z) : (L.cval ? row_ax_csr(L, c, d, Z) : row_ax(L.a, c, d, u, Z, L.upperLo));
                xout[c] = xin[c] + omega * ((1.0 / d[c]) * (L.b[c] - y));
            }
            __syncthreads();
            double* tmp = xin;
            xin = xout;
            xout = tmp;
        }
    }
}

}  // namespace

void launch_gamg_tail(cudaStream_t s, const GLevel* d_lv, int t, int nl, const Workspace& cws, double omega,
                      int n_post)
{
    k_gamg_tail<<<1, kSmallThreads, 0, s>>>(d_lv, t, nl, cws, omega, n_post);
}

// every cycle kernel is launched with programmatic stream serialization (PDL): its CTAs may be
// scheduled while the predecessor drains and wait in griddepcontrol.wait (g_use_pdl)
template <typename... KArgs, typename... Args>
static void glaunch(void (*kernel)(KArgs...), int grid, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_use_pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

static int g_gamg_max_grid = 0;

int gamg_grid(int n)
{
    if (!g_gamg_max_grid) {
        int dev = 0, sms = 148, occ = 4;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gamg_smooth<0, false>, kThreads, 0);
        g_gamg_max_grid = sms * (occ > 0 ? occ : 1);
    }
    const int g = (n + kThreads - 1) / kThreads;
    return g < 1 ? 1 : (g > g_gamg_max_grid ? g_gamg_max_grid : g);
}

namespace {
__global__ void __launch_bounds__(kThreads) k_gamg_csr_values(GLevel L, const double* __restrict__ upper, int F)
{
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
        const double u = upper[f];
        L.cval[L.cposU[f]] = u;
        L.cval[L.cposL[f]] = u;
    }
}
}  // namespace

void launch_gamg_csr_values(cudaStream_t s, const GLevel& L, const double* upper, int F)
{
    k_gamg_csr_values<<<gamg_grid(F), kThreads, 0, s>>>(L, upper, F);
}

void launch_gamg_agg(cudaStream_t s, const GLevel& fine, const GLevel& coarse, const DevPtrs* P)
{
    k_gamg_agg<<<gamg_grid(fine.nc > fine.ncf ? fine.nc : fine.ncf), kThreads, 0, s>>>(fine, coarse, P);
}

// the <ELL, IF> instance of a row kernel for level L (IF: the level has processor interfaces)
#define GAMG_DISPATCH(K, L, ...)                                                  \
    do {                                                                          \
        const bool if_ = (L).a.ifStart != nullptr;                                \
        const int lay_ = (L).ell ? 1 : ((L).cval ? 2 : 0);                        \
        if (lay_ == 1) {                                                          \
            if (if_) glaunch(K<1, true>, (L).grid, s, __VA_ARGS__);               \
            else glaunch(K<1, false>, (L).grid, s, __VA_ARGS__);                  \
        } else if (lay_ == 2) {                                                   \
            if (if_) glaunch(K<2, true>, (L).grid, s, __VA_ARGS__);               \
            else glaunch(K<2, false>, (L).grid, s, __VA_ARGS__);                  \
        } else {                                                                  \
            if (if_) glaunch(K<0, true>, (L).grid, s, __VA_ARGS__);               \
            else glaunch(K<0, false>, (L).grid, s, __VA_ARGS__);                  \
        }                                                                         \
    } while (0)

void launch_gamg_restrict(cudaStream_t s, const GLevel& fine, const GLevel& coarse, const DevPtrs* P, const double* x,
                          double* zero_x)
{
    if (fine.a.ifStart && x) glaunch(k_gamg_restrict<true>, gamg_grid(fine.nc), s, fine, coarse, P, x, zero_x);
    else glaunch(k_gamg_restrict<false>, gamg_grid(fine.nc), s, fine, coarse, P, x, zero_x);
}

void launch_gamg_smooth(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* xin, double* xout,
                        double omega, const double* xc, const double* alpha, bool psi_acc)
{
    GAMG_DISPATCH(k_gamg_smooth, L, L, P, xin, xout, omega, xc, alpha, psi_acc ? 1 : 0);
}

void launch_gamg_scale(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* x, const double* xc,
                       const double* r, double omega, bool pq, double* part, unsigned* ticket, double* alpha,
                       double* rank_part)
{
    GAMG_DISPATCH(k_gamg_scale, L, L, P, x, xc, r, omega, pq ? 1 : 0, part, ticket, alpha, rank_part);
}

void launch_gamg_correct(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* x, const double* xc,
                         const double* alpha, double* out, bool psi_acc)
{
    glaunch(k_gamg_correct, L.grid, s, L, P, x, xc, alpha, out, psi_acc ? 1 : 0);
}

void launch_gamg_post(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* alpha, double omega,
                      double* out, bool two, bool psi_acc)
{
    GAMG_DISPATCH(k_gamg_post, L, L, P, alpha, omega, out, two ? 1 : 0, psi_acc ? 1 : 0);
}

void launch_gamg_gs2_res(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* xin, const double* xc,
                         const double* alpha, double* r)
{
    GAMG_DISPATCH(k_gamg_gs2_res, L, L, P, xin, xc, alpha, r);
}

void launch_gamg_gs2_upd(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* xin, const double* xc,
                         const double* alpha, const double* r, const double* zin, double* out, bool skip_lower,
                         bool last, bool psi_acc)
{
    glaunch(k_gamg_gs2_upd, L.grid, s, L, P, xin, xc, alpha, r, zin, out, skip_lower ? 1 : 0, last ? 1 : 0,
            psi_acc ? 1 : 0);
}

void launch_gamg_residual(cudaStream_t s, const GLevel& L, const Workspace& w, double* rank_part)
{
    GAMG_DISPATCH(k_gamg_residual, L, L, w, rank_part);
}

void launch_gamg_pack(cudaStream_t s, const GLevel& L, int mode, const double* x, const double* xc,
                      const double* alpha, const double* p, const double* q)
{
    if (L.n_if <= 0) return;
    k_gamg_pack<<<gamg_grid(L.n_if), kThreads, 0, s>>>(L, mode, x, xc, alpha, p, q);
}

void launch_gamg_fin(cudaStream_t s, int what, const double* gathered, int n_ranks, double* alpha, DevScal* scal)
{
    k_gamg_fin<<<1, 32, 0, s>>>(what, gathered, n_ranks, alpha, scal);
}

}  // namespace spuma
