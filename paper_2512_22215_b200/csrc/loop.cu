// loop.cu -- the persistent PCG loop (SPUMA_OPT_PERSISTENT): A7-A11 of every iteration of one
// solve (P:506-523 the PCG iteration, P:616 the per-kernel synchronisation the
// paper's profile is dominated by) in ONE cooperative launch of one 896-thread CTA per SM.
//
// Why: the hot loop is HBM-bound (124 B/cell per iteration over three kernels).  A kernel
// boundary forgets everything a CTA held; a persistent CTA does not.  Each CTA owns a fixed
// set of cell pairs for the vector phases, so the residual rA -- read and written by the
// update and read again by the direction, 24 B/cell per iteration -- never leaves the SM:
// the first pairs of every thread live in tensor memory (TMEM, 512 columns x 128 lanes x
// 32 bit per SM, tcgen05.ld / tcgen05.st; the tensor cores themselves stay idle), the next
// ones in shared memory, any rest in HBM (meshes above ~8.2M cells on a 148-SM B200).
// Per iteration: direction (C) -> grid barrier -> Amul + wA.pA (A) -> grid barrier ->
// alpha -> update + (rD rA).rA, |rA| (B) -> grid barrier -> beta / convergence.  Every CTA
// sums the CTA partials in the same fixed order and runs the same finalisation on its own
// copy of the scalars (DevScal in shared memory), so all CTAs take the same decisions
// without a second barrier; CTA 0 writes the scalars back at the end.
//
// The Amul phase runs over the lattice slots (variant 12) on structured numberings, else over
// the ELL rows (variant 8's layout) or the SELL-C rows (variant 6; a permuted mesh as given).
// Element arithmetic is that of k_direction / k_amul_dot / k_update (same operations in the
// same order, deferred psi pairs in the direction, SPUMA_OPT_DEFER_PSI = 2): the rows of A are
// bitwise those of every other variant; the dot products are summed in another (fixed) shape,
// so iterates agree with the graph path to rounding (deterministic run to run).  The host
// (api.cu run_pcg_loop) falls back to the graph batches below half residency and when the
// cooperative launch does not fit.
#include <cstdint>

#include "internal.h"
#include "device.cuh"
#include "amul.cuh"

namespace spuma {
namespace ploop {

#ifndef SPUMA_LOOP_THREADS
#define SPUMA_LOOP_THREADS 896  // same box: 135.0 (896, 72 registers) / 135.7 (1024, 64) / 141.8 (768, 80) us
#endif
constexpr int kT = SPUMA_LOOP_THREADS;           // threads per CTA (one CTA per SM)
constexpr int kWarps = kT / 32;
constexpr int kGroups = kWarps / 4;              // warps sharing one TMEM lane quarter
constexpr int kTmemCols = 512;
constexpr int kColsPerThread = kTmemCols / kGroups / 4 * 4;  // 896 threads: 72 columns = 18 double2
constexpr int kTmemPairs = kColsPerThread / 4;
static_assert(kT % 128 == 0, "whole TMEM lane quarters");

// ---------------------------------------------------------------------------- TMEM access
// A warp reaches only its lane quarter (lanes 32 (warp % 4) ..); thread l of the warp owns
// lane 32 (warp % 4) + l and, of the 512 columns, the kColsPerThread of its warp group.
// Load and completion wait in one asm statement: the registers are defined when it ends.
__device__ __forceinline__ double2 tm_ld(uint32_t addr)
{
    uint32_t r0, r1, r2, r3;
    asm volatile(
        "{\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        "}\n"
        : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
        : "r"(addr));
    double2 v;
    v.x = __hiloint2double((int)r1, (int)r0);
    v.y = __hiloint2double((int)r3, (int)r2);
    return v;
}

__device__ __forceinline__ void tm_st(uint32_t addr, double2 v)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr),
                 "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)),
                 "r"(__double2hiint(v.y))
                 : "memory");
}

__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#ifndef SPUMA_LOOP_PSI_PF
#define SPUMA_LOOP_PSI_PF 1  // A/B: the psi pair's loads (psi, p_{n-2}) prefetched one tile ahead too
#endif
#ifndef SPUMA_LOOP_BAR
#define SPUMA_LOOP_BAR 1  // A/B: 0 fence + atomicAdd + acquire poll + fence, 1 red.release + acquire poll
#endif

// coherent 16-byte load (data another CTA wrote before the last grid barrier)
__device__ __forceinline__ double2 ld2(const double2* p)
{
    double2 v;
#if SPUMA_LOOP_XLD == 1
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
#else
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
#endif
    return v;
}

// The residency of rA: pair slot k of this thread (the CTA's k-th tile) in TMEM (k < tp),
// shared memory (k < tp + sp) or HBM.
struct Res {
    uint32_t taddr;  // this thread's first TMEM column (lane quarter in bits 31..16)
    int tp, sp;
    double2* sm;     // [sp][kT]
    double2* g;      // rA as pairs (HBM)

    __device__ __forceinline__ double2 load(int k, int i) const
    {
        if (k < tp) return tm_ld(taddr + 4u * (uint32_t)k);
        if (k < tp + sp) return sm[(k - tp) * kT + threadIdx.x];
        return g[i];
    }
    __device__ __forceinline__ void store(int k, int i, double2 v) const
    {
        if (k < tp) tm_st(taddr + 4u * (uint32_t)k, v);
        else if (k < tp + sp) sm[(k - tp) * kT + threadIdx.x] = v;
        else g[i] = v;
    }
};

// ---------------------------------------------------------------------------- grid barrier
// Monotone arrival counter: the s-th barrier of the launch waits for s * gridDim.x arrivals.
// A CTA that waits longer than spin_limit cycles (a bug, never a slow peer: the launch is
// cooperative, every CTA is resident) raises the abort word; every later barrier then fails
// at once and the loop stops with SPUMA_ERR_STATE reported by the host.
__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}

// prof (SPUMA_LOOP_PROF builds / LoopArgs::prof): per CTA and phase slot, the ns from the previous
// barrier's release to this CTA's arrival (work) and from arrival to release (wait)
__device__ __forceinline__ bool grid_bar(const LoopArgs& L, unsigned long long target, int slot,
                                         unsigned long long& t_rel)
{
    __shared__ int ok;
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long t_arr = L.prof ? gtime() : 0ull;
#if SPUMA_LOOP_BAR == 1
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(L.bar) : "memory");
#else
        __threadfence();
        atomicAdd(L.bar, 1ull);
#endif
        const long long t0 = clock64();
        int good = 1;
        unsigned spins = 0;
        for (;;) {
            unsigned long long v;
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(L.bar) : "memory");
            if (v >= target) break;
            if ((++spins & 63u) == 0u &&
                (*reinterpret_cast<volatile unsigned long long*>(L.bar + 1) || clock64() - t0 > L.spin_limit)) {
                atomicExch(L.bar + 1, 1ull);
                good = 0;
                break;
            }
        }
#if SPUMA_LOOP_BAR != 1
        __threadfence();
#endif
        ok = good;
        if (L.prof) {
            const unsigned long long t = gtime();
            unsigned long long* q = L.prof + (size_t)blockIdx.x * 8 + 2 * slot;
            q[0] += t_arr - t_rel;
            q[1] += t - t_arr;
            t_rel = t;
        }
    }
    __syncthreads();
    return ok != 0;
}

// Sum NV values over the CTA (warp shuffle tree, then the 32 warp sums in warp 0); result in
// thread 0.
template <int NV>
__device__ __forceinline__ void cta_reduce(double (&v)[NV], double (*sh)[kWarps])
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_down_sync(0xffffffffu, v[i], o);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) sh[i][warp] = v[i];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double t = lane < kWarps ? sh[i][lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
            v[i] = t;
        }
    }
}

// Grid-wide sums of the CTA partials part[i * G + b], the same fixed order in every CTA
// (lane-strided ascending, then the shuffle tree): valid in thread 0.
template <int NV>
__device__ __forceinline__ void grid_sums(const double* part, int off, double (&g)[NV])
{
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double t = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) t += __ldcg(part + (off + i) * gridDim.x + b);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
            g[i] = t;
        }
    }
}

// KT: the lattice offset count at compile time (0: a.lat_K at run time); ELL: the Amul runs over
// the ELL rows of variant 10 (uniform slot widths <= 3, per-solve coefficient copy upper_s) on a
// mesh that is not a lattice numbering (C2 / C4 renumbered by RCM)
// LAY: 0 lattice slots, 1 ELL rows, 2 SELL-C rows (variant 6: a permuted mesh as given, C2)
template <int KT, int LAY>
__global__ void __launch_bounds__(kT, 1) k_pcg_loop(MeshArgs a, Workspace w, LoopArgs L)
{
    extern __shared__ double2 rs[];
    __shared__ uint32_t tmem_base;
    __shared__ DevScal S;
    __shared__ double sh[3][kWarps];

    const int t = threadIdx.x, warp = t >> 5;
    const int G = gridDim.x, b = blockIdx.x;
    const int N = a.N, np = N >> 1;
    const int ntile = (np + kT - 1) / kT;
    const int nk = b < ntile ? (ntile - 1 - b) / G + 1 : 0;  // this CTA's tiles (CTA-uniform)
    const bool use_tmem = L.tmem_pairs > 0;

    if (use_tmem && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (t == 0) S = *w.scal;  // after k_setup2 (stream order): n = 0, wArA, normFactor, done
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    Res R;
    R.tp = use_tmem ? min(nk, min(L.tmem_pairs, kTmemPairs)) : 0;
    R.sp = min(nk - R.tp, L.smem_pairs);
    R.taddr = use_tmem ? tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * kColsPerThread) : 0u;
    R.sm = rs;
    R.g = reinterpret_cast<double2*>(w.rA);

    // rA (k_setup2) into its residency
    for (int k = 0; k < R.tp + R.sp; ++k) {
        const int i = (b + k * G) * kT + t;
        R.store(k, i, i < np ? R.g[i] : make_double2(0.0, 0.0));
    }
    if (use_tmem) tm_wait_st();

    const double* __restrict__ rD = w.rD;
    const double2* __restrict__ rD2 = reinterpret_cast<const double2*>(w.rD);
    const DevPtrs P = *w.ptrs;
    double2* psi2 = reinterpret_cast<double2*>(P.psi);
    const double* const ud[3] = {a.upper_d, a.upper_d + a.lat_S, a.upper_d + 2 * a.lat_S};
    const int K = KT ? KT : a.lat_K;
    unsigned long long target = 0, t_rel = L.prof && t == 0 ? gtime() : 0ull;
    bool ok = true;

    while (!S.done) {
        const int n = S.n;
        const bool odd = L.alt && (n & 1);
        double* pc = (n & 1) ? w.pA2 : w.pA;  // this iteration's direction (slot parity, as the graphs)
        const double* pp = (n & 1) ? w.pA : w.pA2;
        double2* pc2 = reinterpret_cast<double2*>(pc);
        const double2* pp2 = reinterpret_cast<const double2*>(pp);

        // ---- C (A11): pA = rD rA + beta pA_prev; the deferred psi pair on even n >= 2
        {
            const bool first = n == 0;
            const bool psi = n >= 2 && !(n & 1);
            const double beta = S.beta, a1 = S.alpha_prev, a2 = S.alpha_prev2;
            // one tile ahead: the next tile's rD / pA_prev loads are in flight while this one computes
            // (rA pairs kept in HBM -- meshes beyond the on-chip capacity -- are loaded here too)
            double2 dn = make_double2(0.0, 0.0), pn = dn, rn = dn;
#if SPUMA_LOOP_PSI_PF
            double2 xn = dn, on = dn;  // psi and p_{n-2} of the next tile (psi iterations)
#endif
            const int kon = R.tp + R.sp;
            auto pf = [&](int j) {
                const int kk = odd ? nk - 1 - j : j;
                const int i = (b + kk * G) * kT + t;
                if (i < np) {
                    dn = __ldg(rD2 + i);
                    if (!first) pn = ld2(pp2 + i);
#if SPUMA_LOOP_PSI_PF
                    if (psi) {
                        xn = psi2[i];
                        on = ld2(pc2 + i);
                    }
#endif
                    if (kk >= kon) rn = R.g[i];
                }
            };
            if (nk > 0) pf(0);
            for (int j = 0; j < nk; ++j) {
                const int k = odd ? nk - 1 - j : j;
                const int i = (b + k * G) * kT + t;
                const double2 d = dn, p = pn, rh = rn;
#if SPUMA_LOOP_PSI_PF
                const double2 xc = xn, oc = on;
#endif
                if (j + 1 < nk) pf(j + 1);
                const double2 r = k < kon ? R.load(k, 0) : rh;
                if (i < np) {
                    double2 q;
                    if (first) {
                        q.x = d.x * r.x;
                        q.y = d.y * r.y;
                    } else {
                        if (psi) {
#if SPUMA_LOOP_PSI_PF
                            double2 x = xc;
                            const double2 o = oc;  // p_{n-2}
#else
                            double2 x = psi2[i];
                            const double2 o = pc2[i];  // p_{n-2}
#endif
                            x.x = x.x + a2 * o.x;
                            x.y = x.y + a2 * o.y;
                            x.x = x.x + a1 * p.x;
                            x.y = x.y + a1 * p.y;
                            psi2[i] = x;
                        }
                        q.x = d.x * r.x + beta * p.x;
                        q.y = d.y * r.y + beta * p.y;
                    }
                    pc2[i] = q;
                }
            }
            if ((N & 1) && b == 0 && t == 0) {  // the odd cell (rA in HBM)
                const int c = N - 1;
                if (psi) P.psi[c] = (P.psi[c] + a2 * pc[c]) + a1 * pp[c];
                pc[c] = first ? rD[c] * w.rA[c] : rD[c] * w.rA[c] + beta * pp[c];
            }
            if (psi && t == 0) S.psi_done = n;  // every CTA (the same value); CTA 0's copy is written back
        }
        target += (unsigned long long)G;
        if (!(ok = grid_bar(L, target, 0, t_rel))) break;

        // ---- A (A7 + A8): wA = A pA (lattice rows), wA.pA -> alpha
        {
            const int rev = L.alt && !odd;
            const int nw = G * kWarps, wid = b * kWarps + warp;
            const int nch = (N + 31) / 32;
            const int cnt = wid < nch ? (nch - 1 - wid) / nw + 1 : 0;
            double acc = 0.0;
            if constexpr (LAY == 2) {  // variant 6's SELL-C rows (per-chunk widths, wide-row fallback)
                const int lane = t & 31;
                for (int j = 0; j < cnt; ++j)
                    amul_rows_sell<1, 0, false>(a, (wid + (rev ? cnt - 1 - j : j) * nw) * 32 + lane, a.ell_wn, a.ell_wo,
                                                P.diag, P.upper, nullptr, pc, nullptr, w.wA, acc, true);
            } else if constexpr (LAY == 1) {  // variant 8's rows: one row's loads at a time (64 registers; the
                                  // software-pipelined rows of variant 10 spill here: 249 vs 189 us per
                                  // iteration at 8M cells, profiles/r02aa_*)
                const int wn = a.ell_wn, wo = a.ell_wo, lane = t & 31;
                for (int j = 0; j < cnt; ++j) {
                    EllL1 cur;
                    ell_load1<false>(a, (wid + (rev ? cnt - 1 - j : j) * nw) * 32 + lane, wn, wo, P.diag, a.upper_s, pc, cur);
                    ell_finish<0, false>(a, cur, wo, a.upper_s, nullptr, pc, nullptr, w.wA, acc, true);
                }
            } else {
                for (int j = 0; j < cnt; ++j) {
                    const int ch = wid + (rev ? cnt - 1 - j : j) * nw;
                    lat_chunk<1, 0, KT, false>(a, K, ch, P.diag, ud, nullptr, pc, nullptr, w.wA, acc, true);
                }
            }
            double v[1] = {acc};
            cta_reduce<1>(v, sh);
            if (t == 0) w.part[b] = v[0];
        }
        target += (unsigned long long)G;
        if (!(ok = grid_bar(L, target, 1, t_rel))) break;
        {
            double g[1];
            grid_sums<1>(w.part, 0, g);
            if (t == 0) finalize(&S, 3, g);
            __syncthreads();
        }
        if (S.done) break;  // singular

        // ---- B (A9 + A10): rA -= alpha wA; (rD rA).rA, |rA| -> final residual, beta, done
        {
            const double alpha = S.alpha;
            const double2* wA2 = reinterpret_cast<const double2*>(w.wA);
            double v[2] = {0.0, 0.0};
            const int kon = R.tp + R.sp;
            auto pf = [&](int j, double2& wn, double2& dn, double2& rn) {
                const int kk = odd ? nk - 1 - j : j;
                const int i = (b + kk * G) * kT + t;
                if (i < np) {
                    wn = ld2(wA2 + i);
                    dn = __ldg(rD2 + i);
                    if (kk >= kon) rn = R.g[i];
                }
            };
            auto body = [&](int j, double2 ww, double2 d, double2 rh) {
                const int k = odd ? nk - 1 - j : j;
                const int i = (b + k * G) * kT + t;
                double2 r = k < kon ? R.load(k, 0) : rh;
                if (i < np) {
                    r.x = r.x - alpha * ww.x;
                    r.y = r.y - alpha * ww.y;
                    v[0] += (d.x * r.x) * r.x;
                    v[0] += (d.y * r.y) * r.y;
                    v[1] += fabs(r.x);
                    v[1] += fabs(r.y);
                }
                if (k < kon || i < np) R.store(k, i, r);  // on-chip: every lane (TMEM stores are warp-collective)
            };
            // two tiles ahead: slots 0 / 1 hold the loads of tiles j and j + 1 while tile j - 1
            // computes (896 threads: 134.4 vs 135.0 us per iteration for one ahead, same box,
            // profiles/r02bi_*; at 1024 threads / 64 registers it had not paid, r02ah_*)
            double2 w0 = make_double2(0.0, 0.0), d0 = w0, r0 = w0, w1 = w0, d1 = w0, r1 = w0;
            if (nk > 0) pf(0, w0, d0, r0);
            if (nk > 1) pf(1, w1, d1, r1);
            for (int j = 0; j < nk; j += 2) {
                {
                    const double2 ww = w0, d = d0, rh = r0;
                    if (j + 2 < nk) pf(j + 2, w0, d0, r0);
                    body(j, ww, d, rh);
                }
                if (j + 1 < nk) {
                    const double2 ww = w1, d = d1, rh = r1;
                    if (j + 3 < nk) pf(j + 3, w1, d1, r1);
                    body(j + 1, ww, d, rh);
                }
            }
            if ((N & 1) && b == 0 && t == 0) {
                const int c = N - 1;
                const double r = w.rA[c] - alpha * w.wA[c];
                w.rA[c] = r;
                v[0] += (rD[c] * r) * r;
                v[1] += fabs(r);
            }
            if (use_tmem) tm_wait_st();
            cta_reduce<2>(v, sh);
            if (t == 0) {
                w.part[1 * G + b] = v[0];
                w.part[2 * G + b] = v[1];
            }
        }
        target += (unsigned long long)G;
        if (!(ok = grid_bar(L, target, 2, t_rel))) break;
        {
            double g[2];
            grid_sums<2>(w.part, 1, g);
            if (t == 0) finalize(&S, 4, g);
            __syncthreads();
        }
    }

    // rA back to HBM (the handle's workspace stays what the graph path leaves), scalars, TMEM
    for (int k = 0; k < R.tp + R.sp; ++k) {
        const int i = (b + k * G) * kT + t;
        const double2 r = R.load(k, 0);
        if (i < np) R.g[i] = r;
    }
    __syncthreads();
    if (b == 0 && t == 0) {
        if (!ok) S.done = 1;
        *w.scal = S;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (use_tmem && warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols)
                     : "memory");
    }
}

}  // namespace ploop

// ---------------------------------------------------------------------------- host side
int loop_threads() { return ploop::kT; }
int loop_tmem_pairs() { return ploop::kTmemPairs; }

// K: the lattice offset count, 0 = the ELL rows, -1 = the SELL-C rows
static void* loop_fn(int K)
{
    if (K == 3) return (void*)ploop::k_pcg_loop<3, 0>;
    if (K > 0) return (void*)ploop::k_pcg_loop<0, 0>;
    return K == 0 ? (void*)ploop::k_pcg_loop<0, 1> : (void*)ploop::k_pcg_loop<0, 2>;
}

// CTAs per SM the loop kernel reaches with `smem` bytes of dynamic shared memory (0: it
// cannot run, e.g. the shared-memory request is too large)
int loop_occupancy(int K, size_t smem)
{
    void* f = loop_fn(K);
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, ploop::kT, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return nb;
}

cudaError_t launch_pcg_loop(cudaStream_t s, int grid, size_t smem, const MeshArgs& a, const Workspace& w,
                            const LoopArgs& L, const cudaAccessPolicyWindow* win, int layout)
{
    MeshArgs aa = a;
    Workspace ww = w;
    LoopArgs ll = L;
    void* args[] = {(void*)&aa, (void*)&ww, (void*)&ll};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    int na = 1;
    if (win) {
        attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[1].val.accessPolicyWindow = *win;
        na = 2;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(ploop::kT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelExC(&cfg, loop_fn(layout == 1 ? a.lat_K : (layout == 2 ? 0 : -1)), args);
}

}  // namespace spuma
