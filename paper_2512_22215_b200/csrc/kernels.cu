// kernels.cu -- sm_100a kernels of the SPUMA pressure path.
//
// Everything here is fp64 and bandwidth-bound (~0.16 flop/B,
// no dense contraction), so there are no tensor-core paths: the kernels are
// coalesced streaming passes and deterministic per-cell GATHERS over the
// losort/ownerStart restructuring of the faces, replacing the paper's
// atomic face-loop scatters.
//
// Bit-exactness: the library is compiled with --fmad=false, so a*b+c is a
// DMUL followed by a DADD, exactly as the oracle (-ffp-contract=off); the
// per-row accumulation order is the oracle's face order (reading Q10):
// diag*x, then faces with neighbour == c in losort order, then faces with
// owner == c in face order, then processor interfaces in (patch, face) order.
// Reductions use a fixed shape (per-thread grid-stride order, warp shuffle
// tree, CTA tree, last-CTA sum of the per-CTA partials in CTA order), so
// results are run-to-run bitwise reproducible.
#include "internal.h"
#include "device.cuh"

#include <cstdio>



namespace spuma {

// ---------------------------------------------------------------------------
// A7 tiled Amul: a CTA owns a tile of kThreads consecutive cells.  Phase 1
// computes every face product of the tile cooperatively -- the tile's
// owner-side faces [ownerStart[c0], ownerStart[c1]) and neighbour-side entries
// [losortStart[c0], losortStart[c1]) are CONTIGUOUS ranges, so the coefficient
// and index loads are fully coalesced and independent (kUnroll in flight per
// thread) and only x[column] / upper[losort[k]] are gathers (L1/L2 hits on a
// renumbered mesh).  Phase 2: each thread sums its row from shared memory in
// the oracle's order (Q10), so the result is bitwise that of amul_row().
// ---------------------------------------------------------------------------

constexpr int kTileCap = 1024;  // face products per side held in shared memory per tile
constexpr int kUnroll = 4;      // faces in flight per thread per side (4 * 256 = kTileCap)

struct TileSmem {
    double prodN[kTileCap];  // neighbour side, losort order
    double prodO[kTileCap];  // owner side, face order
    int os[kThreads + 1];
    int ls[kThreads + 1];
};

// Products of one side of the tile: prod[k - k0] = coef[k] * x[col[k]], with
// coef[k] = upper[k] (owner side) or upper[losort[k]] (neighbour side).
template <bool INDIRECT>
__device__ __forceinline__ void tile_products(int k0, int k1, const int* __restrict__ coef_idx,
                                              const int* __restrict__ col, const double* __restrict__ upper,
                                              const double* __restrict__ x, double* __restrict__ prod)
{
    for (int base = k0 + (int)threadIdx.x; base < k1; base += kThreads * kUnroll) {
        int cidx[kUnroll];
        double u[kUnroll];
#pragma unroll
        for (int r = 0; r < kUnroll; ++r) {
            const int k = base + r * kThreads;
            cidx[r] = k < k1 ? __ldg(col + k) : 0;
            if (!INDIRECT) u[r] = k < k1 ? __ldg(upper + k) : 0.0;
        }
        if (INDIRECT) {
            int fi[kUnroll];
#pragma unroll
            for (int r = 0; r < kUnroll; ++r) {
                const int k = base + r * kThreads;
                fi[r] = k < k1 ? __ldg(coef_idx + k) : 0;
            }
#pragma unroll
            for (int r = 0; r < kUnroll; ++r) u[r] = __ldg(upper + fi[r]);
        }
        double xv[kUnroll];
#pragma unroll
        for (int r = 0; r < kUnroll; ++r) xv[r] = __ldg(x + cidx[r]);
#pragma unroll
        for (int r = 0; r < kUnroll; ++r) {
            const int k = base + r * kThreads;
            if (k < k1) prod[k - k0] = u[r] * xv[r];
        }
    }
}

// y = A x over the whole mesh, tiles grid-strided over CTAs; returns this thread's sum of y*x.
template <bool DOT>
__device__ __forceinline__ double amul_tiles(const MeshArgs& a, const double* __restrict__ diag,
                                             const double* __restrict__ upper, const double* __restrict__ iface,
                                             const double* __restrict__ x, const double* __restrict__ xr,
                                             double* __restrict__ y, TileSmem& sm)
{
    double acc = 0.0;
    const int n_tiles = (a.N + kThreads - 1) / kThreads;
    const int t = threadIdx.x;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int c0 = tile * kThreads;
        const int n = min(kThreads, a.N - c0);
        const int c = c0 + t;
        if (t < n) {
            sm.os[t] = __ldg(a.ownerStart + c0 + t);
            sm.ls[t] = __ldg(a.losortStart + c0 + t);
        }
        if (t == 0) {  // row extent end of the tile (n may equal kThreads)
            sm.os[n] = __ldg(a.ownerStart + c0 + n);
            sm.ls[n] = __ldg(a.losortStart + c0 + n);
        }
        double dx = 0.0, xc = 0.0;
        if (t < n) {
            xc = __ldg(x + c);
            dx = __ldg(diag + c) * xc;
        }
        __syncthreads();
        const int f0 = sm.os[0], f1 = sm.os[n], k0 = sm.ls[0], k1 = sm.ls[n];
        const bool staged = (f1 - f0) <= kTileCap && (k1 - k0) <= kTileCap;
        if (staged) {
            tile_products<true>(k0, k1, a.losort, a.ownerLo, upper, x, sm.prodN);
            tile_products<false>(f0, f1, nullptr, a.neighbour, upper, x, sm.prodO);
        }
        __syncthreads();
        if (t < n) {
            double s;
            if (staged) {
                s = dx;
                const int ke = sm.ls[t + 1];
                for (int k = sm.ls[t]; k < ke; ++k) s = s + sm.prodN[k - k0];
                const int fe = sm.os[t + 1];
                for (int f = sm.os[t]; f < fe; ++f) s = s + sm.prodO[f - f0];
                if (a.ifStart) {
                    const int j1 = a.ifStart[c + 1];
                    for (int j = a.ifStart[c]; j < j1; ++j) {
                        const int i = a.ifIdx[j];
                        s = s + iface[i] * xr[i];
                    }
                }
            } else {
                s = amul_row(a, c, diag, upper, iface, x, xr, nullptr);
            }
            y[c] = s;
            if (DOT) acc += s * xc;
        }
        __syncthreads();  // smem reused by the next tile
    }
    return acc;
}

}  // namespace spuma
#include "amul.cuh"
namespace spuma {

// ---------------------------------------------------------------------------
// A3 geometry: nonOrthDeltaCoeffs (stabilised form) and linear weights
// ---------------------------------------------------------------------------

__device__ __forceinline__ void face_geometry(const double* CP, const double* CN, const double* S, double magS,
                                              const double* Cf, double* delta, double* weight)
{
    const double dx = CN[0] - CP[0], dy = CN[1] - CP[1], dz = CN[2] - CP[2];
    const double nx = S[0] / magS, ny = S[1] / magS, nz = S[2] / magS;
    const double nd = nx * dx + ny * dy + nz * dz;
    const double magd = sqrt(dx * dx + dy * dy + dz * dz);
    const double lim = 0.05 * magd;
    *delta = 1.0 / (nd > lim ? nd : lim);
    const double ox = Cf[0] - CP[0], oy = Cf[1] - CP[1], oz = Cf[2] - CP[2];
    const double ex = CN[0] - Cf[0], ey = CN[1] - Cf[1], ez = CN[2] - Cf[2];
    const double so = fabs(S[0] * ox + S[1] * oy + S[2] * oz);
    const double sn = fabs(S[0] * ex + S[1] * ey + S[2] * ez);
    const double den = so + sn;
    *weight = den > 1e-150 ? sn / den : 0.5;
}

__global__ void k_geometry(int F, const int* __restrict__ owner, const int* __restrict__ neighbour,
                           const double* __restrict__ Sf, const double* __restrict__ magSf,
                           const double* __restrict__ C, const double* __restrict__ Cf, double* __restrict__ delta,
                           double* __restrict__ weights)
{
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x)
        face_geometry(C + 3 * (size_t)owner[f], C + 3 * (size_t)neighbour[f], Sf + 3 * (size_t)f, magSf[f],
                      Cf + 3 * (size_t)f, delta + f, weights + f);
}

__global__ void k_bgeometry(int Fb, const int* __restrict__ kind, const int* __restrict__ bcell,
                            const double* __restrict__ bSf, const double* __restrict__ bmagSf,
                            const double* __restrict__ bCf, const double* __restrict__ C,
                            const double* __restrict__ nC, const signed char* __restrict__ is_owner,
                            double* __restrict__ bdelta, double* __restrict__ bweight)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Fb; i += gridDim.x * blockDim.x) {
        const double* cp = C + 3 * (size_t)bcell[i];
        const double* S = bSf + 3 * (size_t)i;
        if (kind[i] == SPUMA_PATCH_PROCESSOR) {
            // global orientation: the rank holding the undecomposed owner plays P (reading Q9)
            double Sg[3];
            const double *CP, *CN;
            if (is_owner[i]) {
                Sg[0] = S[0], Sg[1] = S[1], Sg[2] = S[2];
                CP = cp;
                CN = nC + 3 * (size_t)i;
            } else {
                Sg[0] = -S[0], Sg[1] = -S[1], Sg[2] = -S[2];
                CP = nC + 3 * (size_t)i;
                CN = cp;
            }
            face_geometry(CP, CN, Sg, bmagSf[i], bCf + 3 * (size_t)i, bdelta + i, bweight + i);
        } else if (kind[i] == SPUMA_PATCH_EMPTY) {
            bdelta[i] = 0.0;
            bweight[i] = 0.0;
        } else {
            const double nx = S[0] / bmagSf[i], ny = S[1] / bmagSf[i], nz = S[2] / bmagSf[i];
            const double* cf = bCf + 3 * (size_t)i;
            const double ex = cf[0] - cp[0], ey = cf[1] - cp[1], ez = cf[2] - cp[2];
            bdelta[i] = 1.0 / (nx * ex + ny * ey + nz * ez);
            bweight[i] = 0.0;
        }
    }
}

// ---------------------------------------------------------------------------
// A4 face coefficients and A5 diagonal + reference + boundary (gather)
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kThreads) k_face_coeffs(int F, const int* __restrict__ owner,
                                                         const int* __restrict__ neighbour,
                                                         const double* __restrict__ delta,
                                                         const double* __restrict__ weights,
                                                         const double* __restrict__ magSf,
                                                         const double* __restrict__ gamma,
                                                         double* __restrict__ upper)
{
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
        double gf = 1.0;
        if (gamma) {
            const double gn = gamma[neighbour[f]];
            gf = weights[f] * (gamma[owner[f]] - gn) + gn;
        }
        upper[f] = delta[f] * (gf * magSf[f]);
    }
}

__global__ void __launch_bounds__(kThreads)
    k_diag_gather(MeshArgs a, const double* __restrict__ upper, const int* __restrict__ bStart,
                  const int* __restrict__ bFace, const int* __restrict__ bkind, const int* __restrict__ bproc,
                  const double* __restrict__ bmagSf, const double* __restrict__ bdelta,
                  const double* __restrict__ bweight, const double* __restrict__ bvalue,
                  const double* __restrict__ bgamma_r, const signed char* __restrict__ bis_owner,
                  const double* __restrict__ gamma, int ref_cell, double ref_value, double* __restrict__ diag,
                  double* __restrict__ source, double* __restrict__ iface)
{
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
        double d = 0.0;
        const int k1 = a.losortStart[c + 1];
        for (int k = a.losortStart[c]; k < k1; ++k) d = d - upper[a.losort[k]];
        const int f1 = a.ownerStart[c + 1];
        for (int f = a.ownerStart[c]; f < f1; ++f) d = d - upper[f];
        const int j0 = bStart[c], j1 = bStart[c + 1];
        if (c == ref_cell || j1 > j0) {
            double s = source[c];
            if (c == ref_cell) {  // setReference, before any boundary coefficient (Q7)
                s = s + d * ref_value;
                d = d + d;
            }
            const double gP = gamma ? gamma[c] : 1.0;
            for (int j = j0; j < j1; ++j) {
                const int b = bFace[j];
                if (bkind[b] == SPUMA_PATCH_FIXED_VALUE) {
                    const double gms = gP * bmagSf[b];
                    d = d + gms * (-bdelta[b]);
                    s = s + (-gms) * (bdelta[b] * bvalue[b]);
                } else {  // processor (reading Q9): global-orientation interpolation
                    const int i = bproc[b];
                    double gf = 1.0;
                    if (gamma) {
                        const double gr = bgamma_r[i];
                        const double gO = bis_owner[b] ? gP : gr;
                        const double gN = bis_owner[b] ? gr : gP;
                        gf = bweight[b] * (gO - gN) + gN;
                    }
                    const double gms = gf * bmagSf[b];
                    d = d + gms * (-bdelta[b]);
                    iface[i] = bdelta[b] * gms;
                }
            }
            source[c] = s;
        }
        diag[c] = d;
    }
}

// ---------------------------------------------------------------------------
// A7 Amul (plain; diagnostics and the multi-rank setup)
// ---------------------------------------------------------------------------

// minimum resident CTAs per SM per variant (caps registers: 65536 / (CTAs * threads))
template <int V>
constexpr int amul_min_ctas()
{
    return V == 4 ? 8 : (V == 3 ? 4 : ((V == 5 || V == 7 || V == 9) ? 3 : ((V == 6 || V == 8) ? 5 : (V == 10 ? 4 : (V == 11 ? 2 : (V == 12 ? 4 : (V == 13 ? 3 : 6)))))));
}

template <int V, int IFM = 0>
__global__ void __launch_bounds__(V == 3 ? tma::kBlock : kThreads, amul_min_ctas<V>())
    k_amul(MeshArgs a, const double* __restrict__ diag, const double* __restrict__ upper,
           const double* __restrict__ iface, const double* __restrict__ x, const double* __restrict__ xr,
           double* __restrict__ y, tma::Bounds bd)
{
    if constexpr (V == 1) {
        __shared__ TileSmem sm;
        amul_tiles<false>(a, diag, upper, iface, x, xr, y, sm);
    } else if constexpr (V == 3) {
        __shared__ tma::Smem sm;
        tma::amul_tma<false>(a, diag, upper, iface, x, xr, y, bd, sm);
    } else if constexpr (V == 5) {
        double acc = 0.0;
        for (int t0 = blockIdx.x * 2 * kThreads; t0 < a.N; t0 += gridDim.x * 2 * kThreads) {
            const int c = t0 + threadIdx.x;
            if (c < a.N) amul_rows2(a, c, c + kThreads, diag, upper, iface, x, xr, y, acc, false);
        }
    } else if constexpr (V == 6 || V == 7) {
        constexpr int R = V == 7 ? 2 : 1;
        double acc = 0.0;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int t0 = (blockIdx.x * (kThreads / 32) + warp) * 32 * R; t0 < a.N; t0 += gridDim.x * kThreads * R)
            amul_rows_sell<R, IFM>(a, t0 + lane, bd.sell_wn, bd.sell_wo, diag, upper, iface, x, xr, y, acc, false);
    } else if constexpr (V == 8 || V == 9) {
        constexpr int R = V == 9 ? 2 : 1;
        double acc = 0.0;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int t0 = (blockIdx.x * (kThreads / 32) + warp) * 32 * R; t0 < a.N; t0 += gridDim.x * kThreads * R)
            amul_rows_ell<R, IFM>(a, t0 + lane, a.ell_wn, a.ell_wo, diag, upper, a.upper_s, iface, x, xr, y, acc, false);
    } else if constexpr (V == 10) {
        double acc = 0.0;
        amul_ell_pipelined<IFM>(a, diag, upper, iface, x, xr, y, acc, false, 0);
    } else if constexpr (V == 11) {
        ring::amul_ring<IFM, false>(a, diag, upper, iface, x, xr, y, 0);
    } else if constexpr (V == 12 || V == 13) {
        double acc = 0.0;
        amul_lattice<V == 13 ? 2 : 1, IFM>(a, diag, iface, x, xr, y, acc, false, 0);
    } else {
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x)
            y[c] = V == 2 ? amul_row_unrolled(a, c, diag, upper, iface, x, xr)
                          : amul_row(a, c, diag, upper, iface, x, xr, nullptr);
    }
}

__global__ void k_gather(int n, const int* __restrict__ idx, const double* __restrict__ in, double* __restrict__ out)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[idx[i]];
}

__global__ void k_scatter(int n, const int* __restrict__ idx, const double* __restrict__ in, double* __restrict__ out)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[idx[i]] = in[i];
}

// ---------------------------------------------------------------------------
// A6 PCG setup
// ---------------------------------------------------------------------------

// wA = A psi, sumA = A 1 (lduMatrix::sumA), partial sum(psi) and nCells
__global__ void __launch_bounds__(kThreads) k_setup1(MeshArgs a, Workspace w, int fin)
{
    const DevPtrs p = *w.ptrs;
    double v[2] = {0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
        double rs;
        w.wA[c] = amul_row(a, c, p.diag, p.upper, p.iface, p.psi, w.xr, &rs);
        w.sumA[c] = rs;
        v[0] += p.psi[c];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) v[1] = (double)a.N;
    if (grid_sum<2>(v, w.part, &w.scal->ticket[0]) && threadIdx.x == 0) {
        if (fin) finalize(w.scal, 1, v);
        else w.scal->rank_part[0] = v[0], w.scal->rank_part[1] = v[1];
    }
}

// rA = source - wA; rD = 1/diag; partials of |wA - xRef| + |source - xRef|, |rA|, (rD rA) rA
__global__ void __launch_bounds__(kThreads) k_setup2(MeshArgs a, Workspace w, int fin)
{
    const DevPtrs p = *w.ptrs;
    const double xbar = w.scal->xbar;
    double v[3] = {0.0, 0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
        const double b = p.source[c], wa = w.wA[c];
        const double r = b - wa;
        const double xref = w.sumA[c] * xbar;
        const double rd = 1.0 / p.diag[c];
        w.rA[c] = r;
        w.rD[c] = rd;
        v[0] += fabs(wa - xref) + fabs(b - xref);
        v[1] += fabs(r);
        v[2] += (rd * r) * r;
    }
    if (grid_sum<3>(v, w.part, &w.scal->ticket[1]) && threadIdx.x == 0) {
        if (fin) finalize(w.scal, 2, v);
        else w.scal->rank_part[0] = v[0], w.scal->rank_part[1] = v[1], w.scal->rank_part[2] = v[2];
    }
}

// ---------------------------------------------------------------------------
// A7-A11 hot loop (each kernel is a no-op once the device 'done' flag is set)
// ---------------------------------------------------------------------------

// A11 pA = rD rA + beta pA  (n == 0: pA = rD rA)
// psi_pair (deferred psi updates in the direction, SPUMA_OPT_DEFER_PSI = 2; even k >= 2): the
// pair (k-2, k-1) -- psi = (psi + alpha_{k-2} p_{k-2}) + alpha_{k-1} p_{k-1}, the two roundings of
// two separate updates, so the iterates are bitwise unchanged -- applied here, where p_{k-1}
// (pA_prev) is read anyway and p_{k-2} is the value of pA this pass overwrites (read first).
// halo (peer transport, SPUMA_OPT_PEER_FUSED): every interface cell's new direction value is stored
// straight into the neighbours' mailboxes by the thread that computed it (compute and send in one
// kernel); the last CTA publishes the exchange's epoch (the protocol of k_peer_send, peer.cu).
__device__ __forceinline__ bool halo_store(const MeshArgs& a, const Workspace& w, int par, int c, double v)
{
    if (!((__ldg(a.ifMask + (c >> 5)) >> (c & 31)) & 1u)) return false;
    const int j1 = a.ifStart[c + 1];
    for (int j = a.ifStart[c]; j < j1; ++j) {
        const int q = a.ifIdx[j], p = w.if_patch[q];
        w.px->dst[p][par][q - w.px->off[p]] = v;
    }
    return true;
}

// sent: this thread stored into a peer's mailbox (only those threads need the system-scope fence
// before their CTA's ticket; the last CTA fences again before it publishes the flags)
__device__ __forceinline__ void halo_publish(const Workspace& w, unsigned long long e, bool sent)
{
    if (sent) __threadfence_system();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(w.pst.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence_system();
        const int par = (int)(e & 1ull);
        for (int p = 0; p < w.px->n_patches; ++p) st_release_sys(w.px->dst_flag[p][par], e);
        w.pst.ctr[0] = e;
        *w.pst.ticket = 0u;
    }
}

__global__ void __launch_bounds__(kThreads) k_direction(MeshArgs a, Workspace w, int rev, int psi_pair, int halo)
{
    pdl_wait();
    if (w.scal->done) return;
    const int N = a.N;
    const unsigned long long he = halo ? w.pst.ctr[0] + 1 : 0;  // this exchange's epoch
    const int hpar = (int)(he & 1ull);
    bool sent = false;
    const int n = w.scal->n;
    const bool first = n == 0;
    const bool psi = psi_pair && n >= 2;
    const double beta = w.scal->beta, a1 = w.scal->alpha_prev, a2 = w.scal->alpha_prev2;
    const int np = N >> 1;
    const double2* __restrict__ rD2 = reinterpret_cast<const double2*>(w.rD);
    const double2* __restrict__ rA2 = reinterpret_cast<const double2*>(w.rA);
    const double2* pprev = reinterpret_cast<const double2*>(w.pA_prev);  // may alias pA (in place)
    double2* pA2 = reinterpret_cast<double2*>(w.pA);
    double2* psi2 = psi ? reinterpret_cast<double2*>(w.ptrs->psi) : nullptr;
    const GridStride gs(np, rev);
    for (int j = 0; j < gs.cnt; ++j) {
        const int i = gs.at(j);
        const double2 d = rD2[i], r = rA2[i];
        double2 q;
        if (first) {
            q.x = d.x * r.x;
            q.y = d.y * r.y;
        } else {
            const double2 p = pprev[i];
            if (psi) {
                double2 x = psi2[i];
                const double2 o = pA2[i];  // p_{k-2}
                x.x = x.x + a2 * o.x;
                x.y = x.y + a2 * o.y;
                x.x = x.x + a1 * p.x;
                x.y = x.y + a1 * p.y;
                psi2[i] = x;
            }
            q.x = d.x * r.x + beta * p.x;
            q.y = d.y * r.y + beta * p.y;
        }
        pA2[i] = q;
        if (halo) {
            sent |= halo_store(a, w, hpar, 2 * i, q.x);
            sent |= halo_store(a, w, hpar, 2 * i + 1, q.y);
        }
    }
    if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int c = N - 1;
        if (psi) {
            double* ps = w.ptrs->psi;
            ps[c] = (ps[c] + a2 * w.pA[c]) + a1 * w.pA_prev[c];
        }
        const double v = first ? w.rD[c] * w.rA[c] : w.rD[c] * w.rA[c] + beta * w.pA_prev[c];
        w.pA[c] = v;
        if (halo) sent |= halo_store(a, w, hpar, c, v);
    }
    if (psi && blockIdx.x == 0 && threadIdx.x == 0) w.scal->psi_done = n;
    pdl_trigger();
    if (halo) halo_publish(w, he, sent);
}

// A7 + A8: wA = A pA, partial wA.pA -> alpha
template <int V, int IFM = 0>
__global__ void __launch_bounds__(V == 3 ? tma::kBlock : kThreads, amul_min_ctas<V>())
    k_amul_dot(MeshArgs a, Workspace w, int fin, int sell_wn, int sell_wo, int rev)
{
    pdl_wait();
    if (w.scal->done) return;
    const DevPtrs p = *w.ptrs;
    double v[1] = {0.0};
    if constexpr (V == 1) {
        __shared__ TileSmem sm;
        v[0] = amul_tiles<true>(a, p.diag, p.upper, p.iface, w.pA, w.xr, w.wA, sm);
    } else if constexpr (V == 3) {
        __shared__ tma::Smem sm;
        const tma::Bounds bd{a.F, (long long)a.N + 8, a.N, sell_wn, sell_wo};
        v[0] = tma::amul_tma<true>(a, p.diag, p.upper, p.iface, w.pA, w.xr, w.wA, bd, sm);
    } else if constexpr (V == 5) {
        double acc = 0.0;
        for (int t0 = blockIdx.x * 2 * kThreads; t0 < a.N; t0 += gridDim.x * 2 * kThreads) {
            const int c = t0 + threadIdx.x;
            if (c < a.N) amul_rows2(a, c, c + kThreads, p.diag, p.upper, p.iface, w.pA, w.xr, w.wA, acc, true);
        }
        v[0] = acc;
    } else if constexpr (V == 6 || V == 7) {
        constexpr int R = V == 7 ? 2 : 1;
        double acc = 0.0;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int t0 = (blockIdx.x * (kThreads / 32) + warp) * 32 * R; t0 < a.N; t0 += gridDim.x * kThreads * R)
            amul_rows_sell<R, IFM>(a, t0 + lane, sell_wn, sell_wo, p.diag, p.upper, p.iface, w.pA, w.xr, w.wA, acc, true);
        v[0] = acc;
    } else if constexpr (V == 8 || V == 9) {
        constexpr int R = V == 9 ? 2 : 1;
        double acc = 0.0;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int st = gridDim.x * kThreads * R, t00 = (blockIdx.x * (kThreads / 32) + warp) * 32 * R;
        const int cnt = t00 < a.N ? (a.N - 1 - t00) / st + 1 : 0;
        for (int j = 0; j < cnt; ++j) {  // rev: descending sweep (L2 reuse, see GridStride)
            const int t0 = t00 + (rev ? cnt - 1 - j : j) * st;
            amul_rows_ell<R, IFM>(a, t0 + lane, a.ell_wn, a.ell_wo, p.diag, p.upper, a.upper_s, p.iface, w.pA, w.xr, w.wA,
                             acc, true);
        }
        v[0] = acc;
    } else if constexpr (V == 10) {
        double acc = 0.0;
        amul_ell_pipelined<IFM>(a, p.diag, p.upper, p.iface, w.pA, w.xr, w.wA, acc, true, rev);
        v[0] = acc;
    } else if constexpr (V == 11) {
        v[0] = ring::amul_ring<IFM, true>(a, p.diag, p.upper, p.iface, w.pA, w.xr, w.wA, rev);
    } else if constexpr (V == 12 || V == 13) {
        double acc = 0.0;
        amul_lattice<V == 13 ? 2 : 1, IFM>(a, p.diag, p.iface, w.pA, w.xr, w.wA, acc, true, rev);
        v[0] = acc;
    } else {
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
            const double y = V == 2 ? amul_row_unrolled(a, c, p.diag, p.upper, p.iface, w.pA, w.xr)
                                    : amul_row(a, c, p.diag, p.upper, p.iface, w.pA, w.xr, nullptr);
            w.wA[c] = y;
            v[0] += y * w.pA[c];
        }
    }
    pdl_trigger();
    if (grid_sum<1>(v, w.part, &w.scal->ticket[2]) && threadIdx.x == 0) {
        if (fin) finalize(w.scal, 3, v);
        else w.scal->rank_part[0] = v[0];
    }
}

// A11 + A7 + A8 fused (ELL, single rank, deferred psi => pA / pA_prev are distinct buffers):
// the direction pA = rD rA + beta pA_prev (n == 0: rD rA) is formed for the row AND at its
// neighbours inside the Amul gather, written once for the row, and wA = A pA, wA.pA -> alpha.
// The separate k_direction pass (32 B/cell) disappears.  INL: rD = 1/diag computed in place
// (diag is streamed anyway; IEEE division: bitwise the stored rD), else read rD.  Same values
// in the same order as k_direction + k_amul_dot<8> on the same grid: bitwise the same iterates.
template <bool INL>
__global__ void __launch_bounds__(kThreads, amul_min_ctas<8>()) k_amul_dot_dir(MeshArgs a, Workspace w)
{
    pdl_wait();
    if (w.scal->done) return;
    const DevPtrs p = *w.ptrs;
    const bool first = w.scal->n == 0;
    const double beta = w.scal->beta;
    const double* __restrict__ diag = p.diag;
    const double* __restrict__ rD = w.rD;
    const double* __restrict__ rA = w.rA;
    const double* __restrict__ pprev = w.pA_prev;
    auto P = [&](int j) -> double {
        const double rd = INL ? 1.0 / __ldg(diag + j) : __ldg(rD + j);
        return first ? rd * __ldg(rA + j) : rd * __ldg(rA + j) + beta * __ldg(pprev + j);
    };
    constexpr int W = 3;
    const int wn = a.ell_wn, wo = a.ell_wo;
    double acc = 0.0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t0 = (blockIdx.x * (kThreads / 32) + warp) * 32; t0 < a.N; t0 += gridDim.x * kThreads) {
        const int c0 = t0 + lane;
        const int c = min(c0, a.N - 1);
        const int k = c >> 5;
        unsigned pk[W];
        int nb[W];
        double uo[W], un[W];
#pragma unroll
        for (int j = 0; j < W; ++j) {
            pk[j] = j < wn ? __ldg(a.sell_n + (size_t)32 * wn * k + 32 * j + lane) : 0xFFFFFFFFu;
            nb[j] = j < wo ? __ldg(a.sell_o + (size_t)32 * wo * k + 32 * j + lane) : -1;
            uo[j] = j < wo ? __ldg(a.upper_s + (size_t)32 * wo * k + 32 * j + lane) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const int col = (int)(pk[j] >> 5), pos = (int)(pk[j] & 31u);
            un[j] = pk[j] != 0xFFFFFFFFu ? __ldg(a.upper_s + (size_t)32 * wo * (col >> 5) + 32 * pos + (col & 31)) : 0.0;
        }
        const double xc = P(c);
        double xn[W], xo[W];
#pragma unroll
        for (int j = 0; j < W; ++j) {
            xn[j] = P(pk[j] != 0xFFFFFFFFu ? (int)(pk[j] >> 5) : c);
            xo[j] = P(nb[j] >= 0 ? nb[j] : c);
        }
        double sum = __ldg(diag + c) * xc;
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (pk[j] != 0xFFFFFFFFu) sum = sum + un[j] * xn[j];
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (nb[j] >= 0) sum = sum + uo[j] * xo[j];
        if (c0 < a.N) {
            w.pA[c] = xc;
            w.wA[c] = sum;
            acc += sum * xc;
        }
    }
    double v[1] = {acc};
    pdl_trigger();
    if (grid_sum<1>(v, w.part, &w.scal->ticket[2]) && threadIdx.x == 0) finalize(w.scal, 3, v);
}

// A9 + A10: psi += alpha pA; rA -= alpha wA; partials (rD rA) rA and |rA|
// psi_mode 0: psi += alpha pA; 1: psi left for the next iteration (deferred); 2: the
// deferred pair, psi = (psi + alpha_prev pA_prev) + alpha pA -- the same two roundings as
// two separate updates, so every iterate is bitwise unchanged.
__global__ void __launch_bounds__(kThreads) k_update(int N, Workspace w, int fin, int psi_mode, int rev)
{
    pdl_wait();
    if (w.scal->done) return;
    const DevPtrs p = *w.ptrs;
    const double alpha = w.scal->alpha, alpha_prev = w.scal->alpha_prev;
    double v[2] = {0.0, 0.0};
    const int np = N >> 1;
    double2* __restrict__ psi2 = reinterpret_cast<double2*>(p.psi);
    double2* __restrict__ rA2 = reinterpret_cast<double2*>(w.rA);
    const double2* __restrict__ pA2 = reinterpret_cast<const double2*>(w.pA);
    const double2* __restrict__ pP2 = reinterpret_cast<const double2*>(w.pA_prev);
    const double2* __restrict__ wA2 = reinterpret_cast<const double2*>(w.wA);
    const double2* __restrict__ rD2 = reinterpret_cast<const double2*>(w.rD);
    const GridStride gs(np, rev);
    for (int j = 0; j < gs.cnt; ++j) {
        const int i = gs.at(j);
        double2 r = rA2[i];
        const double2 ww = wA2[i], d = rD2[i];
        if (psi_mode != 1) {
            double2 x = psi2[i];
            const double2 pp = pA2[i];
            if (psi_mode == 2) {
                const double2 q = pP2[i];
                x.x = x.x + alpha_prev * q.x;
                x.y = x.y + alpha_prev * q.y;
            }
            x.x = x.x + alpha * pp.x;
            x.y = x.y + alpha * pp.y;
            psi2[i] = x;
        }
        r.x = r.x - alpha * ww.x;
        r.y = r.y - alpha * ww.y;
        rA2[i] = r;
        v[0] += (d.x * r.x) * r.x;
        v[0] += (d.y * r.y) * r.y;
        v[1] += fabs(r.x);
        v[1] += fabs(r.y);
    }
    if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int c = N - 1;
        if (psi_mode != 1) {
            double x = p.psi[c];
            if (psi_mode == 2) x = x + alpha_prev * w.pA_prev[c];
            p.psi[c] = x + alpha * w.pA[c];
        }
        const double r = w.rA[c] - alpha * w.wA[c];
        w.rA[c] = r;
        v[0] += (w.rD[c] * r) * r;
        v[1] += fabs(r);
    }
    pdl_trigger();
    if (grid_sum<2>(v, w.part, &w.scal->ticket[3])) {  // true in every thread of the last CTA
        if (threadIdx.x == 0) {
            if (fin == 1) finalize(w.scal, 4, v);
            else w.scal->rank_part[0] = v[0], w.scal->rank_part[1] = v[1];
        }
        if (fin == 2) {  // the peer all-gather of the rank partials and the finalisation, here
            __syncthreads();
            peer_gather_finalize(*w.pg, w.pst, w.scal->rank_part, w.part, 4, w.scal);
        }
    }
}

// ---------------------------------------------------------------------------
// Small meshes (BASELINE config 1, 400 cells): the whole solve (A6-A12) in ONE
// CTA of 1024 threads -- phases separated by __syncthreads() instead of kernel
// launches, so an iteration costs a few CTA barriers instead of 3 launches.
// Same row order (bitwise Amul) and the same finalisation code.
// ---------------------------------------------------------------------------



__global__ void __launch_bounds__(kSmallThreads) k_pcg_single(MeshArgs a, Workspace w) { pcg_single_body(a, w); }

// threads of the single-CTA solves: one per cell up to kSmallThreads (fewer warps at the CTA barriers
// of a small mesh); both launchers use the same count, so their reductions have the same shape
static int small_threads(int N) { return N >= kSmallThreads ? kSmallThreads : (N < 32 ? 32 : (N + 31) / 32 * 32); }

void launch_pcg_single(cudaStream_t s, const MeshArgs& a, const Workspace& w)
{
    k_pcg_single<<<1, small_threads(a.N), 0, s>>>(a, w);
}

// The single-CTA solve with everything in shared memory (BASELINE config 1, the 400-cell cavity:
// a latency problem).  The matrix (diag, upper), source, psi, the row addressing and the PCG
// vectors and scalars are staged into shared memory once, the whole solve runs there (every
// gather an SMEM load, every finalisation an SMEM store), and psi / the scalars are written back
// at the end.  The same row order and the same reduction tree as k_pcg_single: bitwise the same
// iterates.  Layout: doubles diag, upper, source, psi, wA, rA, rD, pA, sumA, then the DevScal,
// then ints ownerStart, losortStart [N+1], losort, ownerLo, neighbour [F].
size_t pcg_single_smem_bytes(int N, int F)
{
    const size_t dbl = sizeof(double) * (8 * (size_t)N + (size_t)F) + sizeof(DevScal);
    return ((dbl + 15) & ~(size_t)15) + sizeof(int) * (2 * ((size_t)N + 1) + 3 * (size_t)F);
}

__global__ void __launch_bounds__(kSmallThreads) k_pcg_single_smem(MeshArgs a, Workspace w)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int N = a.N, F = a.F, t = threadIdx.x;
    double* d = reinterpret_cast<double*>(smem);
    double* up = d + N;
    double* src = up + F;
    double* psi = src + N;
    Workspace ws = w;
    ws.wA = psi + N;
    ws.rA = ws.wA + N;
    ws.rD = ws.rA + N;
    ws.pA = ws.rD + N;
    ws.sumA = ws.pA + N;
    DevScal* sc = reinterpret_cast<DevScal*>(ws.sumA + N);
    const size_t dbl = sizeof(double) * (8 * (size_t)N + (size_t)F) + sizeof(DevScal);
    int* os = reinterpret_cast<int*>(smem + ((dbl + 15) & ~(size_t)15));
    int* ls = os + N + 1;
    int* lo = ls + N + 1;
    int* ol = lo + F;
    int* nb = ol + F;
    const DevPtrs g = *w.ptrs;
    for (int i = t; i < N; i += blockDim.x) {
        d[i] = g.diag[i];
        src[i] = g.source[i];
        psi[i] = g.psi[i];
    }
    for (int i = t; i < F; i += blockDim.x) {
        up[i] = g.upper[i];
        lo[i] = a.losort[i];
        ol[i] = a.ownerLo[i];
        nb[i] = a.neighbour[i];
    }
    for (int i = t; i <= N; i += blockDim.x) {
        os[i] = a.ownerStart[i];
        ls[i] = a.losortStart[i];
    }
    if (t == 0) *sc = *w.scal;
    __syncthreads();
    MeshArgs as = a;
    as.ownerStart = os;
    as.losortStart = ls;
    as.losort = lo;
    as.ownerLo = ol;
    as.neighbour = nb;
    as.ifStart = nullptr;
    as.ifIdx = nullptr;
    as.ifMask = nullptr;
    const DevPtrs ps{d, up, nullptr, src, psi};
    pcg_single_body(as, ws, ps, sc);
    __syncthreads();
    for (int i = t; i < N; i += blockDim.x) g.psi[i] = psi[i];
    if (t == 0) *w.scal = *sc;
}

bool launch_pcg_single_smem(cudaStream_t s, const MeshArgs& a, const Workspace& w)
{
    const size_t bytes = pcg_single_smem_bytes(a.N, a.F);
    static int max_dyn = -1;  // opt-in shared memory per block minus the kernel's static shared memory
    if (max_dyn < 0) {
        int dev = 0, optin = 0;
        cudaFuncAttributes fa{};
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
            cudaFuncGetAttributes(&fa, k_pcg_single_smem) != cudaSuccess ||
            cudaFuncSetAttribute(k_pcg_single_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - (int)fa.sharedSizeBytes) != cudaSuccess) {
            cudaGetLastError();  // not sticky: fall back to the global-memory kernel
            max_dyn = 0;
        } else {
            max_dyn = optin - (int)fa.sharedSizeBytes;
        }
    }
    if (a.ifStart || bytes > (size_t)max_dyn) return false;
    k_pcg_single_smem<<<1, small_threads(a.N), bytes, s>>>(a, w);
    return true;
}

// ---------------------------------------------------------------------------
// Around the path: fvc::surfaceIntegrate and fvMatrix::flux
// ---------------------------------------------------------------------------

// out[c] = (-phi of faces with neighbour c in losort order, +phi of faces with owner c
// in face order, +bphi of c's non-empty boundary faces in (patch, face) order) / V[c]:
// the oracle's face-loop order, so bitwise ("surfaceIntegrate").
__global__ void __launch_bounds__(kThreads)
    k_surface_integrate(MeshArgs a, const double* __restrict__ phi, const int* __restrict__ bStart,
                        const int* __restrict__ bFace, const double* __restrict__ bphi,
                        const double* __restrict__ V, double* __restrict__ out)
{
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
        double s = 0.0;
        const int k1 = a.losortStart[c + 1];
        for (int k = a.losortStart[c]; k < k1; ++k) s = s - phi[a.losort[k]];
        const int f1 = a.ownerStart[c + 1];
        for (int f = a.ownerStart[c]; f < f1; ++f) s = s + phi[f];
        const int j1 = bStart[c + 1];
        for (int j = bStart[c]; j < j1; ++j) s = s + bphi[bFace[j]];
        out[c] = s / V[c];
    }
}

// fvMatrix::flux, internal faces: faceH = Upper psi_N - Lower psi_P;
// phi != nullptr: the SIMPLE correction phi -= flux in place.
__global__ void __launch_bounds__(kThreads)
    k_face_flux(int F, const int* __restrict__ owner, const int* __restrict__ neighbour,
                const double* __restrict__ upper, const double* __restrict__ psi, const double* __restrict__ cflux,
                double* __restrict__ flux, double* __restrict__ phi)
{
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
        const double u = upper[f];
        double q = u * psi[neighbour[f]] - u * psi[owner[f]];
        if (cflux) q = q + cflux[f];  // fvMatrix::flux adds faceFluxCorrection
        if (flux) flux[f] = q;
        if (phi) phi[f] = phi[f] - q;
    }
}

// boundary faces: internalCoeffs psi_P - boundaryCoeffs (x psi_remote for processor faces)
__global__ void __launch_bounds__(kThreads)
    k_bface_flux(int Fb, const int* __restrict__ bkind, const int* __restrict__ bcell, const int* __restrict__ bproc,
                 const double* __restrict__ bmagSf, const double* __restrict__ bdelta,
                 const double* __restrict__ bweight, const double* __restrict__ bvalue,
                 const double* __restrict__ bgamma_r, const signed char* __restrict__ bis_owner,
                 const double* __restrict__ gamma, const double* __restrict__ psi, const double* __restrict__ psi_r,
                 const double* __restrict__ bcflux, double* __restrict__ bflux, double* __restrict__ bphi)
{
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < Fb; b += gridDim.x * blockDim.x) {
        const int P = bcell[b];
        const double gP = gamma ? gamma[P] : 1.0;
        double q = 0.0;
        if (bkind[b] == SPUMA_PATCH_FIXED_VALUE) {
            const double gms = gP * bmagSf[b];
            q = (gms * (-bdelta[b])) * psi[P] - ((-gms) * (bdelta[b] * bvalue[b]));
        } else if (bkind[b] == SPUMA_PATCH_PROCESSOR) {
            const int i = bproc[b];
            double gf = 1.0;
            if (gamma) {
                const double gr = bgamma_r[i];
                const double gO = bis_owner[b] ? gP : gr;
                const double gN = bis_owner[b] ? gr : gP;
                gf = bweight[b] * (gO - gN) + gN;
            }
            const double gms = gf * bmagSf[b];
            q = (gms * (-bdelta[b])) * psi[P] - (((-gms) * bdelta[b]) * psi_r[i]);
        }
        if (bcflux) q = q + bcflux[b];
        bflux[b] = q;
        if (bphi) bphi[b] = bphi[b] - q;
    }
}

// oriented face field <-> internal numbering: out[i] = sign(flip[i]) in[idx[i]] (gather)
// or out[idx[i]] = sign(flip[i]) in[i] (scatter)
__global__ void k_gather_signed(int n, const int* __restrict__ idx, const signed char* __restrict__ flip,
                                const double* __restrict__ in, double* __restrict__ out)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = flip[i] ? -in[idx[i]] : in[idx[i]];
}
__global__ void k_scatter_signed(int n, const int* __restrict__ idx, const signed char* __restrict__ flip,
                                 const double* __restrict__ in, double* __restrict__ out)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[idx[i]] = flip[i] ? -in[i] : in[i];
}

// ---------------------------------------------------------------------------
// Explicit non-orthogonal correction of "Gauss linear corrected" (P:1112, P:1135,
// P:1145): Gauss gradient, correction vectors, correction flux (reading Q21)
// ---------------------------------------------------------------------------

// nonOrthCorrectionVectors (mesh time): cv = Sf/|Sf| - (C_N - C_P) delta, per component
__global__ void k_corrvec(int F, const int* __restrict__ owner, const int* __restrict__ neighbour,
                          const double* __restrict__ Sf, const double* __restrict__ magSf,
                          const double* __restrict__ C, const double* __restrict__ delta, double* __restrict__ cv)
{
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
        const double* CP = C + 3 * (size_t)owner[f];
        const double* CN = C + 3 * (size_t)neighbour[f];
        for (int k = 0; k < 3; ++k) cv[3 * (size_t)f + k] = Sf[3 * (size_t)f + k] / magSf[f] - (CN[k] - CP[k]) * delta[f];
    }
}

__device__ __forceinline__ double bface_value(int kind, double pP, double value, double w, signed char own, double pr)
{
    if (kind == SPUMA_PATCH_FIXED_VALUE) return value;
    if (kind == SPUMA_PATCH_PROCESSOR) {
        const double pO = own ? pP : pr;
        const double pN = own ? pr : pP;
        return w * (pO - pN) + pN;
    }
    return pP;  // zeroGradient
}

// Gauss linear gradient, per-cell gather in the oracle's face order (bitwise)
__global__ void __launch_bounds__(kThreads)
    k_gauss_grad(MeshArgs a, const double* __restrict__ Sf, const double* __restrict__ weights,
                 const double* __restrict__ p, const int* __restrict__ bStart, const int* __restrict__ bFace,
                 const int* __restrict__ bkind, const int* __restrict__ bproc, const double* __restrict__ bSf,
                 const double* __restrict__ bvalue, const double* __restrict__ bweight,
                 const signed char* __restrict__ bis_owner, const double* __restrict__ p_r,
                 const double* __restrict__ V, double* __restrict__ G)
{
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
        const double pc = p[c];
        double g0 = 0.0, g1 = 0.0, g2 = 0.0;
        const int k1 = a.losortStart[c + 1];
        for (int k = a.losortStart[c]; k < k1; ++k) {  // c is the neighbour: G -= Sf p_f
            const int f = a.losort[k];
            const double pf = weights[f] * (p[a.ownerLo[k]] - pc) + pc;
            g0 = g0 - Sf[3 * (size_t)f] * pf;
            g1 = g1 - Sf[3 * (size_t)f + 1] * pf;
            g2 = g2 - Sf[3 * (size_t)f + 2] * pf;
        }
        const int f1 = a.ownerStart[c + 1];
        for (int f = a.ownerStart[c]; f < f1; ++f) {  // c is the owner: G += Sf p_f
            const double pn = p[a.neighbour[f]];
            const double pf = weights[f] * (pc - pn) + pn;
            g0 = g0 + Sf[3 * (size_t)f] * pf;
            g1 = g1 + Sf[3 * (size_t)f + 1] * pf;
            g2 = g2 + Sf[3 * (size_t)f + 2] * pf;
        }
        const int j1 = bStart[c + 1];
        for (int j = bStart[c]; j < j1; ++j) {
            const int b = bFace[j];
            const int i = bproc[b];
            const double pb = bface_value(bkind[b], pc, bvalue[b], bweight[b], bis_owner[b], i >= 0 ? p_r[i] : 0.0);
            g0 = g0 + bSf[3 * (size_t)b] * pb;
            g1 = g1 + bSf[3 * (size_t)b + 1] * pb;
            g2 = g2 + bSf[3 * (size_t)b + 2] * pb;
        }
        G[c] = g0 / V[c];  // structure of arrays: G[k N + c]
        G[(size_t)a.N + c] = g1 / V[c];
        G[2 * (size_t)a.N + c] = g2 / V[c];
    }
}

// correction flux on internal faces: (gamma_f |S|) (cv . (w (G_P - G_N) + G_N))
__global__ void __launch_bounds__(kThreads)
    k_nonorth_flux(int F, int NC, const int* __restrict__ owner, const int* __restrict__ neighbour,
                   const double* __restrict__ cv, const double* __restrict__ magSf, const double* __restrict__ weights,
                   const double* __restrict__ gamma, const double* __restrict__ G, double* __restrict__ cflux)
{
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
        const size_t P = owner[f], N = neighbour[f];
        const double w = weights[f];
        double g[3];
        for (int k = 0; k < 3; ++k) g[k] = w * (G[k * (size_t)NC + P] - G[k * (size_t)NC + N]) + G[k * (size_t)NC + N];
        const double corr = cv[3 * (size_t)f] * g[0] + cv[3 * (size_t)f + 1] * g[1] + cv[3 * (size_t)f + 2] * g[2];
        double gf = 1.0;
        if (gamma) gf = w * (gamma[P] - gamma[N]) + gamma[N];
        cflux[f] = (gf * magSf[f]) * corr;
    }
}

// correction flux on boundary faces: processor faces in global orientation (outward sign), else 0
__global__ void __launch_bounds__(kThreads)
    k_bnonorth_flux(int Fb, int NC, int NI, const int* __restrict__ bkind, const int* __restrict__ bcell,
                    const int* __restrict__ bproc,
                    const double* __restrict__ bSf, const double* __restrict__ bmagSf, const double* __restrict__ bdelta,
                    const double* __restrict__ bweight, const signed char* __restrict__ bis_owner,
                    const double* __restrict__ bnC, const double* __restrict__ C, const double* __restrict__ G,
                    const double* __restrict__ G_r, const double* __restrict__ gamma,
                    const double* __restrict__ bgamma_r, double* __restrict__ bcflux)
{
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < Fb; b += gridDim.x * blockDim.x) {
        double q = 0.0;
        if (bkind[b] == SPUMA_PATCH_PROCESSOR) {
            const int L = bcell[b], i = bproc[b];
            const bool own = bis_owner[b];
            const double* CL = C + 3 * (size_t)L;
            const double* CR = bnC + 3 * (size_t)b;
            double cv[3], g[3];
            for (int k = 0; k < 3; ++k) {
                const double S = own ? bSf[3 * (size_t)b + k] : -bSf[3 * (size_t)b + k];
                const double cP = own ? CL[k] : CR[k], cN = own ? CR[k] : CL[k];
                cv[k] = S / bmagSf[b] - (cN - cP) * bdelta[b];
                const double gL = G[k * (size_t)NC + L], gR = G_r[k * (size_t)NI + i];
                const double gO = own ? gL : gR;
                const double gN = own ? gR : gL;
                g[k] = bweight[b] * (gO - gN) + gN;
            }
            const double corr = cv[0] * g[0] + cv[1] * g[1] + cv[2] * g[2];
            double gf = 1.0;
            if (gamma) {
                const double gO = own ? gamma[L] : bgamma_r[i];
                const double gN = own ? bgamma_r[i] : gamma[L];
                gf = bweight[b] * (gO - gN) + gN;
            }
            const double v = (gf * bmagSf[b]) * corr;
            q = own ? v : -v;
        }
        bcflux[b] = q;
    }
}

// source -= V div  (div = surfaceIntegrate of the correction flux)
__global__ void k_sub_vdiv(int N, const double* __restrict__ V, const double* __restrict__ div, double* __restrict__ src)
{
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x)
        src[c] = src[c] - V[c] * div[c];
}

// add a (correction) flux: out += in
__global__ void k_add(int n, const double* __restrict__ in, double* __restrict__ out)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = out[i] + in[i];
}

// A7 interface rows (P > 1, deferred mode): rows[] = cells with processor faces
// (ascending).  wA[c] already holds the internal-face sum; add the interface terms
// in (patch, face) order (bitwise the one-pass row, Q10) and the rows' share of
// wA.pA, then complete this rank's partial: rank_part[0] = interior + interface rows.
// peer (SPUMA_OPT_PEER_FUSED): the halo's receive is fused in -- each CTA waits for the neighbours'
// epoch flags of the exchange k_direction published, then reads the remote values straight from
// its mailbox -- and the last CTA runs the rank-partial all-gather + finalisation (stage 3).
__global__ void __launch_bounds__(kThreads) k_iface_rows(MeshArgs a, Workspace w, const int* __restrict__ rows,
                                                         int n_rows, int peer)
{
    if (w.scal->done) return;
    const DevPtrs p = *w.ptrs;
    int par = 0;
    if (peer) {
        __shared__ int ok;
        const unsigned long long e = w.pst.ctr[0];  // set by this rank's k_direction of the same exchange
        par = (int)(e & 1ull);
        if (threadIdx.x == 0) {
            ok = 1;
            for (int q = 0; q < w.px->n_patches && ok; ++q)
                if (!wait_flag(w.px->src_flag[q][par], e, w.pst.err, w.pst.poll_cycles)) ok = 0;
        }
        __syncthreads();
        if (!ok) n_rows = 0;  // timed out: the error word is set, the gather below stops the loop
    }
    double v[1] = {0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_rows; i += gridDim.x * blockDim.x) {
        const int c = rows[i];
        double y = w.wA[c];
        const int j1 = a.ifStart[c + 1];
        for (int j = a.ifStart[c]; j < j1; ++j) {
            const int q = a.ifIdx[j];
            double xr;
            if (peer) {
                const int pp = w.if_patch[q];
                xr = __ldcg(w.px->src[pp][par] + (q - w.px->off[pp]));
            } else {
                xr = w.xr[q];
            }
            y = y + p.iface[q] * xr;
        }
        w.wA[c] = y;
        v[0] += y * w.pA[c];
    }
    if (grid_sum<1>(v, w.part, &w.scal->ticket[4])) {
        if (threadIdx.x == 0) w.scal->rank_part[0] = w.scal->rank_part[0] + v[0];
        if (peer) {
            __syncthreads();
            peer_gather_finalize(*w.pg, w.pst, w.scal->rank_part, w.part, 3, w.scal);
        }
    }
}

// P > 1: global sums of the gathered rank partials in rank order, then finalise
__global__ void k_finalize(int stage, const double* __restrict__ gathered, int n_ranks, Workspace w)
{
    if (stage >= 3 && w.scal->done) return;
    double g[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r = 0; r < n_ranks; ++r)
        for (int i = 0; i < 4; ++i) g[i] += gathered[4 * r + i];
    finalize(w.scal, stage, g);
}

__global__ void k_scal_init(DevScal* s, double tol, double rel_tol, int max_iter, int min_iter, int n_ranks)
{
    s->tol = tol;
    s->rel_tol = rel_tol;
    s->max_iter = max_iter;
    s->min_iter = min_iter;
    s->n_ranks = n_ranks;
    s->n = 0;
    s->done = 0;
    s->singular = 0;
    s->converged = 0;
    s->alpha = s->beta = s->alpha_prev = s->alpha_prev2 = 0.0;
    s->psi_done = 0;
    for (int i = 0; i < 4; ++i) s->rank_part[i] = 0.0;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

template <class K>
static int kernel_block(K kernel)
{
    return ((const void*)kernel == (const void*)k_amul_dot<3> || (const void*)kernel == (const void*)k_amul<3>)
               ? tma::kBlock
               : kThreads;
}

bool g_use_pdl = true;

// launch with the programmatic-stream-serialization attribute when PDL is on
template <typename... KArgs, typename... Args>
static void launch_hot(void (*kernel)(KArgs...), int grid, int block, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_use_pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <typename... KArgs, typename... Args>
static void launch_hot_smem(void (*kernel)(KArgs...), int grid, int smem, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_use_pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}

static int g_sms = 0;

static int sms()
{
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    return g_sms;
}

// grid = min(CTAs the work needs, CTAs resident at full occupancy): one wave, grid-stride loops.
// work / (work_per_thread * threads_per_work_unit) CTAs are needed; for tile kernels pass
// work = tiles and threads_per_work_unit = 1 (one tile per CTA per step).
template <class K>
static int grid_for(K kernel, long long work, int per_thread = 1, int threads_per_unit = kThreads)
{
    int occ = 0;
    const int block = kernel_block(kernel);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, 0);
    if (occ <= 0) occ = 1;
    long long need = (work + (long long)threads_per_unit * per_thread - 1) / ((long long)threads_per_unit * per_thread);
    long long cap = (long long)occ * sms();
    long long g = need < cap ? need : cap;
    return (int)(g < 1 ? 1 : g);
}

// variant 11: dynamic shared memory ring (ring::kSmem per CTA)
template <class K>
static int ring_grid(K kernel, int N)
{
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ring::kSmem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, ring::kSmem);
    if (occ <= 0) occ = 1;
    const long long chunks = ((long long)N + 31) / 32;
    long long need = (chunks + ring::kWarps - 1) / ring::kWarps;
    long long cap = (long long)occ * sms();
    long long g = need < cap ? need : cap;
    return (int)(g < 1 ? 1 : g);
}

int occupancy_grid(int N, int* grid_faces, int F)
{
    // the largest grid any reduction kernel uses (sizes the partials buffer)
    int g = grid_for(k_setup1, N);
    g = std::max(g, grid_for(k_setup2, N));
    g = std::max(g, grid_for(k_amul_dot<0>, N));
    g = std::max(g, grid_for(k_amul_dot<1>, N));
    g = std::max(g, grid_for(k_amul_dot<2>, N));
    g = std::max(g, grid_for(k_amul_dot<3>, (N + tma::kCells - 1) / tma::kCells, 1, 1));
    g = std::max(g, grid_for(k_amul_dot<4>, N));
    g = std::max(g, grid_for(k_amul_dot<5>, N, 2));
    g = std::max(g, grid_for(k_amul_dot<6>, N));
    g = std::max(g, grid_for(k_amul_dot<7>, N, 2));
    g = std::max(g, grid_for(k_amul_dot<8>, N));
    g = std::max(g, grid_for(k_amul_dot<9>, N, 2));
    g = std::max(g, grid_for(k_amul_dot<6, 1>, N));
    g = std::max(g, grid_for(k_amul_dot<7, 1>, N, 2));
    g = std::max(g, grid_for(k_amul_dot<8, 1>, N));
    g = std::max(g, grid_for(k_amul_dot<9, 1>, N, 2));
    g = std::max(g, grid_for(k_amul_dot<6, 2>, N));
    g = std::max(g, grid_for(k_amul_dot<7, 2>, N, 2));
    g = std::max(g, grid_for(k_amul_dot<8, 2>, N));
    g = std::max(g, grid_for(k_amul_dot<9, 2>, N, 2));
    g = std::max(g, ring_grid(k_amul_dot<11>, N));
    g = std::max(g, ring_grid(k_amul_dot<11, 1>, N));
    g = std::max(g, ring_grid(k_amul_dot<11, 2>, N));
    g = std::max(g, grid_for(k_amul_dot<10>, N));
    g = std::max(g, grid_for(k_amul_dot<10, 1>, N));
    g = std::max(g, grid_for(k_amul_dot<10, 2>, N));
    g = std::max(g, grid_for(k_amul_dot<12>, N));
    g = std::max(g, grid_for(k_amul_dot<12, 1>, N));
    g = std::max(g, grid_for(k_amul_dot<12, 2>, N));
    g = std::max(g, grid_for(k_amul_dot<13>, N, 2));
    g = std::max(g, grid_for(k_amul_dot<13, 1>, N, 2));
    g = std::max(g, grid_for(k_amul_dot<13, 2>, N, 2));
    g = std::max(g, grid_for(k_iface_rows, N));
    g = std::max(g, grid_for(k_update, N, 2));
    if (grid_faces) *grid_faces = grid_for(k_face_coeffs, F);
    return g;
}

void launch_geometry(cudaStream_t s, int F, const int* owner, const int* neighbour, const double* Sf,
                     const double* magSf, const double* C, const double* Cf, double* delta, double* weights)
{
    if (F <= 0) return;
    k_geometry<<<grid_for(k_geometry, F), kThreads, 0, s>>>(F, owner, neighbour, Sf, magSf, C, Cf, delta, weights);
}

void launch_bgeometry(cudaStream_t s, int Fb, const int* kind, const int* bcell, const double* bSf,
                      const double* bmagSf, const double* bCf, const double* C, const double* nC,
                      const signed char* is_owner, double* bdelta, double* bweight)
{
    if (Fb <= 0) return;
    k_bgeometry<<<grid_for(k_bgeometry, Fb), kThreads, 0, s>>>(Fb, kind, bcell, bSf, bmagSf, bCf, C, nC, is_owner,
                                                               bdelta, bweight);
}

void launch_face_coeffs(cudaStream_t s, int grid, int F, const int* owner, const int* neighbour,
                        const double* delta, const double* weights, const double* magSf, const double* gamma,
                        double* upper)
{
    if (F <= 0) return;
    (void)grid;
    k_face_coeffs<<<grid_for(k_face_coeffs, F), kThreads, 0, s>>>(F, owner, neighbour, delta, weights, magSf, gamma,
                                                                  upper);
}

void launch_diag_gather(cudaStream_t s, int grid, const MeshArgs& a, const double* upper, const int* bStart,
                        const int* bFace, const int* bkind, const int* bcell, const int* bproc,
                        const double* bmagSf, const double* bdelta, const double* bweight, const double* bvalue,
                        const double* bgamma_r, const signed char* bis_owner, const double* gamma, int ref_cell,
                        double ref_value, double* diag, double* source, double* iface)
{
    if (a.N <= 0) return;
    (void)grid;
    (void)bcell;
    k_diag_gather<<<grid_for(k_diag_gather, a.N), kThreads, 0, s>>>(a, upper, bStart, bFace, bkind, bproc, bmagSf,
                                                                    bdelta, bweight, bvalue, bgamma_r, bis_owner,
                                                                    gamma, ref_cell, ref_value, diag, source, iface);
}

void launch_amul(cudaStream_t s, int variant, const MeshArgs& a, const double* diag, const double* upper,
                 const double* iface, const double* x, const double* xr, double* y, long long x_len, int sell_wn,
                 int sell_wo)
{
    if (a.N <= 0) return;
    variant = resolve_amul_variant(variant, a);
    const tma::Bounds bd{a.F, x_len, a.N, sell_wn, sell_wo};
    switch (variant) {
    case 12:
        if (a.ifMask) k_amul<12, 1><<<grid_for(k_amul<12, 1>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        else k_amul<12><<<grid_for(k_amul<12>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        break;
    case 13:
        if (a.ifMask) k_amul<13, 1><<<grid_for(k_amul<13, 1>, a.N, 2), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        else k_amul<13><<<grid_for(k_amul<13>, a.N, 2), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        break;
    case 1: k_amul<1><<<grid_for(k_amul<1>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd); break;
    case 2: k_amul<2><<<grid_for(k_amul<2>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd); break;
    case 3:
        k_amul<3><<<grid_for(k_amul<3>, (a.N + tma::kCells - 1) / tma::kCells, 1, 1), tma::kBlock, 0, s>>>(a, diag, upper, iface,
                                                                                            x, xr, y, bd);
        break;
    case 4: k_amul<4><<<grid_for(k_amul<4>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd); break;
    case 5: k_amul<5><<<grid_for(k_amul<5>, a.N, 2), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd); break;
    case 6:
        if (a.ifMask) k_amul<6, 1><<<grid_for(k_amul<6, 1>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        else k_amul<6><<<grid_for(k_amul<6>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        break;
    case 7:
        if (a.ifMask) k_amul<7, 1><<<grid_for(k_amul<7, 1>, a.N, 2), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        else k_amul<7><<<grid_for(k_amul<7>, a.N, 2), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        break;
    case 8:
        if (a.ifMask) k_amul<8, 1><<<grid_for(k_amul<8, 1>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        else k_amul<8><<<grid_for(k_amul<8>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        break;
    case 9:
        if (a.ifMask) k_amul<9, 1><<<grid_for(k_amul<9, 1>, a.N, 2), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        else k_amul<9><<<grid_for(k_amul<9>, a.N, 2), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        break;
    case 10:
        if (a.ifMask) k_amul<10, 1><<<grid_for(k_amul<10, 1>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        else k_amul<10><<<grid_for(k_amul<10>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd);
        break;
    case 11:
        if (a.ifMask) k_amul<11, 1><<<ring_grid(k_amul<11, 1>, a.N), kThreads, ring::kSmem, s>>>(a, diag, upper, iface, x, xr, y, bd);
        else k_amul<11><<<ring_grid(k_amul<11>, a.N), kThreads, ring::kSmem, s>>>(a, diag, upper, iface, x, xr, y, bd);
        break;
    default: k_amul<0><<<grid_for(k_amul<0>, a.N), kThreads, 0, s>>>(a, diag, upper, iface, x, xr, y, bd); break;
    }
}

// owner-slot ordered coefficient copy for variants 8/9 (once per solve / Amul call)
__global__ void k_ell_coeffs(MeshArgs a, const double* __restrict__ upper, double* __restrict__ upper_s)
{
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < a.F; f += gridDim.x * blockDim.x) {
        const int o = a.owner[f];
        const int j = f - a.ownerStart[o];
        upper_s[(size_t)32 * a.ell_wo * (o >> 5) + 32 * j + (o & 31)] = upper[f];
    }
}

bool amul_uses_ell(int variant) { return variant >= 8 && variant <= 11; }

// lattice slot coefficient copy for variant 12 (once per solve / Amul call): face f is slot t of
// its owner row, D[t] = neighbour - owner (absent slots keep kLatAbsent from mesh_create)
__global__ void k_lattice_coeffs(MeshArgs a, const double* __restrict__ upper, double* __restrict__ ud)
{
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < a.F; f += gridDim.x * blockDim.x) {
        const int o = __ldg(a.owner + f), d = __ldg(a.neighbour + f) - o;
        const int t = d == a.lat_D[0] ? 0 : (d == a.lat_D[1] ? 1 : 2);
        ud[t * a.lat_S + o] = __ldg(upper + f);
    }
}

void launch_lattice_coeffs(cudaStream_t s, const MeshArgs& a, const double* upper)
{
    if (a.F <= 0 || !a.upper_d) return;
    k_lattice_coeffs<<<grid_for(k_lattice_coeffs, a.F), kThreads, 0, s>>>(a, upper, const_cast<double*>(a.upper_d));
}

__global__ void k_fill_u64(long long n, unsigned long long* __restrict__ p, unsigned long long v)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

void launch_fill_u64(cudaStream_t s, long long n, double* p, unsigned long long v)
{
    if (n <= 0) return;
    k_fill_u64<<<grid_for(k_fill_u64, n), kThreads, 0, s>>>(n, reinterpret_cast<unsigned long long*>(p), v);
}

void launch_ell_coeffs(cudaStream_t s, const MeshArgs& a, const double* upper, double* upper_s)
{
    if (a.F <= 0 || !upper_s) return;
    k_ell_coeffs<<<grid_for(k_ell_coeffs, a.F), kThreads, 0, s>>>(a, upper, upper_s);
}

void launch_gather(cudaStream_t s, int n, const int* idx, const double* in, double* out)
{
    if (n <= 0) return;
    k_gather<<<grid_for(k_gather, n), kThreads, 0, s>>>(n, idx, in, out);
}

void launch_scatter(cudaStream_t s, int n, const int* idx, const double* in, double* out)
{
    if (n <= 0) return;
    k_scatter<<<grid_for(k_scatter, n), kThreads, 0, s>>>(n, idx, in, out);
}

void launch_pack(cudaStream_t s, int n, const int* cell, const double* x, double* out)
{
    launch_gather(s, n, cell, x, out);
}

void launch_setup1(cudaStream_t s, int grid, const MeshArgs& a, const Workspace& w, bool fin)
{
    (void)grid;
    k_setup1<<<grid_for(k_setup1, a.N), kThreads, 0, s>>>(a, w, fin ? 1 : 0);
}

void launch_setup2(cudaStream_t s, int grid, const MeshArgs& a, const Workspace& w, bool fin)
{
    (void)grid;
    k_setup2<<<grid_for(k_setup2, a.N), kThreads, 0, s>>>(a, w, fin ? 1 : 0);
}

void launch_direction(cudaStream_t s, int grid, const MeshArgs& a, const Workspace& w, bool reverse, bool psi_pair,
                      bool halo)
{
    (void)grid;
    launch_hot(k_direction, grid_for(k_direction, a.N, 2), kThreads, s, a, w, reverse ? 1 : 0, psi_pair ? 1 : 0,
               halo ? 1 : 0);
}

int resolve_amul_variant(int variant, const MeshArgs& a)
{
    if ((variant == 12 || variant == 13) && !(a.upper_d && a.lat_K > 0)) variant = 10;  // not a lattice numbering
    if ((variant == 10 || variant == 11) && !a.upper_s) variant = 6;
    if ((variant == 8 || variant == 9) && !a.upper_s) variant -= 2;  // no uniform-width layout: SELL
    if ((variant == 6 || variant == 7) && !a.sell_n) variant = 5;    // layout not encodable on this mesh
    return variant;
}

void launch_amul_dot(cudaStream_t s, int variant, const MeshArgs& a, const Workspace& w, bool fin, int sell_wn,
                     int sell_wo, bool deferred, bool reverse)
{
    const int f = fin ? 1 : 0, r = reverse ? 1 : 0;
    variant = resolve_amul_variant(variant, a);
    if (deferred && a.ifMask) {  // interface rows finished by k_iface_rows after the halo
        switch (variant) {
        case 6: launch_hot(k_amul_dot<6, 2>, grid_for(k_amul_dot<6, 2>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r); return;
        case 7: launch_hot(k_amul_dot<7, 2>, grid_for(k_amul_dot<7, 2>, a.N, 2), kThreads, s, a, w, f, sell_wn, sell_wo, r); return;
        case 8: launch_hot(k_amul_dot<8, 2>, grid_for(k_amul_dot<8, 2>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r); return;
        case 9: launch_hot(k_amul_dot<9, 2>, grid_for(k_amul_dot<9, 2>, a.N, 2), kThreads, s, a, w, f, sell_wn, sell_wo, r); return;
        case 10: launch_hot(k_amul_dot<10, 2>, grid_for(k_amul_dot<10, 2>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r); return;
        case 12: launch_hot(k_amul_dot<12, 2>, grid_for(k_amul_dot<12, 2>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r); return;
        case 13: launch_hot(k_amul_dot<13, 2>, grid_for(k_amul_dot<13, 2>, a.N, 2), kThreads, s, a, w, f, sell_wn, sell_wo, r); return;
        case 11: launch_hot_smem(k_amul_dot<11, 2>, ring_grid(k_amul_dot<11, 2>, a.N), ring::kSmem, s, a, w, f, sell_wn, sell_wo, r); return;
        default: break;  // other variants add the interface terms inline (halo must precede them)
        }
    }
    switch (variant) {
    case 1: k_amul_dot<1><<<grid_for(k_amul_dot<1>, a.N), kThreads, 0, s>>>(a, w, f, sell_wn, sell_wo, r); break;
    case 2: k_amul_dot<2><<<grid_for(k_amul_dot<2>, a.N), kThreads, 0, s>>>(a, w, f, sell_wn, sell_wo, r); break;
    case 3:
        k_amul_dot<3><<<grid_for(k_amul_dot<3>, (a.N + tma::kCells - 1) / tma::kCells, 1, 1), tma::kBlock, 0, s>>>(a, w, f, sell_wn, sell_wo, r);
        break;
    case 4: k_amul_dot<4><<<grid_for(k_amul_dot<4>, a.N), kThreads, 0, s>>>(a, w, f, sell_wn, sell_wo, r); break;
    case 5: launch_hot(k_amul_dot<5>, grid_for(k_amul_dot<5>, a.N, 2), kThreads, s, a, w, f, sell_wn, sell_wo, r); break;
    case 6:
        if (a.ifMask) launch_hot(k_amul_dot<6, 1>, grid_for(k_amul_dot<6, 1>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        else launch_hot(k_amul_dot<6>, grid_for(k_amul_dot<6>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        break;
    case 7:
        if (a.ifMask) launch_hot(k_amul_dot<7, 1>, grid_for(k_amul_dot<7, 1>, a.N, 2), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        else launch_hot(k_amul_dot<7>, grid_for(k_amul_dot<7>, a.N, 2), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        break;
    case 8:
        if (a.ifMask) launch_hot(k_amul_dot<8, 1>, grid_for(k_amul_dot<8, 1>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        else launch_hot(k_amul_dot<8>, grid_for(k_amul_dot<8>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        break;
    case 9:
        if (a.ifMask) launch_hot(k_amul_dot<9, 1>, grid_for(k_amul_dot<9, 1>, a.N, 2), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        else launch_hot(k_amul_dot<9>, grid_for(k_amul_dot<9>, a.N, 2), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        break;
    case 10:
        if (a.ifMask) launch_hot(k_amul_dot<10, 1>, grid_for(k_amul_dot<10, 1>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        else launch_hot(k_amul_dot<10>, grid_for(k_amul_dot<10>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        break;
    case 12:
        if (a.ifMask) launch_hot(k_amul_dot<12, 1>, grid_for(k_amul_dot<12, 1>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        else launch_hot(k_amul_dot<12>, grid_for(k_amul_dot<12>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        break;
    case 13:
        if (a.ifMask) launch_hot(k_amul_dot<13, 1>, grid_for(k_amul_dot<13, 1>, a.N, 2), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        else launch_hot(k_amul_dot<13>, grid_for(k_amul_dot<13>, a.N, 2), kThreads, s, a, w, f, sell_wn, sell_wo, r);
        break;
    case 11:
        if (a.ifMask) launch_hot_smem(k_amul_dot<11, 1>, ring_grid(k_amul_dot<11, 1>, a.N), ring::kSmem, s, a, w, f, sell_wn, sell_wo, r);
        else launch_hot_smem(k_amul_dot<11>, ring_grid(k_amul_dot<11>, a.N), ring::kSmem, s, a, w, f, sell_wn, sell_wo, r);
        break;
    default: launch_hot(k_amul_dot<0>, grid_for(k_amul_dot<0>, a.N), kThreads, s, a, w, f, sell_wn, sell_wo, r); break;
    }
}

bool fused_direction_ok(const MeshArgs& a)
{
    return a.ell_wn >= 0 && a.ell_wn <= 3 && a.ell_wo >= 0 && a.ell_wo <= 3 && a.upper_s && a.sell_n && !a.ifMask;
}

void launch_amul_dot_dir(cudaStream_t s, const MeshArgs& a, const Workspace& w, bool inline_rd)
{
    const int g = grid_for(k_amul_dot<8>, a.N);  // the unfused kernel's grid: same reduction shape
    if (inline_rd) launch_hot(k_amul_dot_dir<true>, g, kThreads, s, a, w);
    else launch_hot(k_amul_dot_dir<false>, g, kThreads, s, a, w);
}

void launch_update(cudaStream_t s, int grid, const MeshArgs& a, const Workspace& w, int fin, int psi_mode,
                   bool reverse)
{
    (void)grid;
    launch_hot(k_update, grid_for(k_update, a.N, 2), kThreads, s, a.N, w, fin, psi_mode, reverse ? 1 : 0);
}

// the pending half of a deferred pair when the loop stopped after an even-indexed iteration
__global__ void k_psi_flush(int N, Workspace w)
{
    const DevPtrs p = *w.ptrs;
    const double a = w.scal->alpha_prev;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x)
        p.psi[c] = p.psi[c] + a * w.pA[c];
}

__global__ void k_psi_flush2(int N, Workspace w, int n, int pending)
{
    const DevPtrs p = *w.ptrs;
    const double a1 = w.scal->alpha_prev, a2 = w.scal->alpha_prev2;
    const double* p1 = ((n - 1) & 1) ? w.pA2 : w.pA;  // p_{n-1}
    const double* p2 = ((n - 2) & 1) ? w.pA2 : w.pA;  // p_{n-2}
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
        double x = p.psi[c];
        if (pending == 2) x = x + a2 * p2[c];
        p.psi[c] = x + a1 * p1[c];
    }
}

void launch_psi_flush2(cudaStream_t s, int N, const Workspace& w, int n, int pending)
{
    if (N <= 0 || pending <= 0) return;
    k_psi_flush2<<<grid_for(k_psi_flush2, N), kThreads, 0, s>>>(N, w, n, pending);
}

void launch_psi_flush(cudaStream_t s, int N, const Workspace& w)
{
    if (N <= 0) return;
    k_psi_flush<<<grid_for(k_psi_flush, N), kThreads, 0, s>>>(N, w);
}

void launch_surface_integrate(cudaStream_t s, const MeshArgs& a, const double* phi, const int* bStart,
                              const int* bFace, const double* bphi, const double* V, double* out)
{
    if (a.N <= 0) return;
    k_surface_integrate<<<grid_for(k_surface_integrate, a.N), kThreads, 0, s>>>(a, phi, bStart, bFace, bphi, V, out);
}

void launch_face_flux(cudaStream_t s, int F, const int* owner, const int* neighbour, const double* upper,
                      const double* psi, const double* cflux, double* flux, double* phi)
{
    if (F <= 0) return;
    k_face_flux<<<grid_for(k_face_flux, F), kThreads, 0, s>>>(F, owner, neighbour, upper, psi, cflux, flux, phi);
}

void launch_bface_flux(cudaStream_t s, int Fb, const int* bkind, const int* bcell, const int* bproc,
                       const double* bmagSf, const double* bdelta, const double* bweight, const double* bvalue,
                       const double* bgamma_r, const signed char* bis_owner, const double* gamma, const double* psi,
                       const double* psi_r, const double* bcflux, double* bflux, double* bphi)
{
    if (Fb <= 0) return;
    k_bface_flux<<<grid_for(k_bface_flux, Fb), kThreads, 0, s>>>(Fb, bkind, bcell, bproc, bmagSf, bdelta, bweight,
                                                                 bvalue, bgamma_r, bis_owner, gamma, psi, psi_r,
                                                                 bcflux, bflux, bphi);
}

void launch_gather_signed(cudaStream_t s, int n, const int* idx, const signed char* flip, const double* in,
                          double* out)
{
    if (n <= 0) return;
    k_gather_signed<<<grid_for(k_gather_signed, n), kThreads, 0, s>>>(n, idx, flip, in, out);
}

void launch_scatter_signed(cudaStream_t s, int n, const int* idx, const signed char* flip, const double* in,
                           double* out)
{
    if (n <= 0) return;
    k_scatter_signed<<<grid_for(k_scatter_signed, n), kThreads, 0, s>>>(n, idx, flip, in, out);
}

void launch_corrvec(cudaStream_t s, int F, const int* owner, const int* neighbour, const double* Sf,
                    const double* magSf, const double* C, const double* delta, double* cv)
{
    if (F <= 0) return;
    k_corrvec<<<grid_for(k_corrvec, F), kThreads, 0, s>>>(F, owner, neighbour, Sf, magSf, C, delta, cv);
}

void launch_gauss_grad(cudaStream_t s, const MeshArgs& a, const double* Sf, const double* weights, const double* p,
                       const int* bStart, const int* bFace, const int* bkind, const int* bproc, const double* bSf,
                       const double* bvalue, const double* bweight, const signed char* bis_owner, const double* p_r,
                       const double* V, double* G)
{
    if (a.N <= 0) return;
    k_gauss_grad<<<grid_for(k_gauss_grad, a.N), kThreads, 0, s>>>(a, Sf, weights, p, bStart, bFace, bkind, bproc, bSf,
                                                                  bvalue, bweight, bis_owner, p_r, V, G);
}

void launch_nonorth_flux(cudaStream_t s, int F, int NC, const int* owner, const int* neighbour, const double* cv,
                         const double* magSf, const double* weights, const double* gamma, const double* G,
                         double* cflux)
{
    if (F <= 0) return;
    k_nonorth_flux<<<grid_for(k_nonorth_flux, F), kThreads, 0, s>>>(F, NC, owner, neighbour, cv, magSf, weights,
                                                                    gamma, G, cflux);
}

void launch_bnonorth_flux(cudaStream_t s, int Fb, int NC, int NI, const int* bkind, const int* bcell, const int* bproc,
                          const double* bSf, const double* bmagSf, const double* bdelta, const double* bweight,
                          const signed char* bis_owner, const double* bnC, const double* C, const double* G,
                          const double* G_r, const double* gamma, const double* bgamma_r, double* bcflux)
{
    if (Fb <= 0) return;
    k_bnonorth_flux<<<grid_for(k_bnonorth_flux, Fb), kThreads, 0, s>>>(Fb, NC, NI, bkind, bcell, bproc, bSf, bmagSf,
                                                                       bdelta, bweight, bis_owner, bnC, C, G, G_r,
                                                                       gamma, bgamma_r, bcflux);
}

void launch_sub_vdiv(cudaStream_t s, int N, const double* V, const double* div, double* src)
{
    if (N <= 0) return;
    k_sub_vdiv<<<grid_for(k_sub_vdiv, N), kThreads, 0, s>>>(N, V, div, src);
}

void launch_add(cudaStream_t s, int n, const double* in, double* out)
{
    if (n <= 0) return;
    k_add<<<grid_for(k_add, n), kThreads, 0, s>>>(n, in, out);
}

void launch_iface_rows(cudaStream_t s, const MeshArgs& a, const Workspace& w, const int* rows, int n_rows, bool peer)
{
    if (n_rows <= 0 && !peer) return;
    const int g = n_rows > 0 ? grid_for(k_iface_rows, n_rows) : 1;  // peer: the gather runs even without rows
    k_iface_rows<<<g, kThreads, 0, s>>>(a, w, rows, n_rows, peer ? 1 : 0);
}

void launch_finalize(cudaStream_t s, int stage, const double* gathered, int n_ranks, const Workspace& w)
{
    k_finalize<<<1, 1, 0, s>>>(stage, gathered, n_ranks, w);
}

void launch_scal_init(cudaStream_t s, const Workspace& w, const spuma_solver_controls& c, int n_ranks)
{
    k_scal_init<<<1, 1, 0, s>>>(w.scal, c.tolerance, c.rel_tol, c.max_iter, c.min_iter, n_ranks);
}

}  // namespace spuma
