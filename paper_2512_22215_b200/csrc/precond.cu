// precond.cu -- sm_100a kernels of the preconditioned solvers around the path
// (readings Q31-Q35): DIC / DILU factor and sweeps, aDILU passes,
// the PCG/PBiCG vector kernels, asymmetric Amul/Tmul, LDU -> CSR value gather.
//
// The DIC/DILU recurrences are sequential in face order.  They run as ONE persistent
// "sync-free" kernel per sweep: threads claim rows in level-schedule order (host-built,
// rows sorted by dependency depth) from an atomic counter, spin (acquire loads) on the
// ready flags of the rows they depend on, then publish their value (release store).  Each
// row sums its faces in the oracle's order, so the result is bitwise that of the
// sequential loop for ANY cell numbering; the critical path is the dependency depth.  A
// row only waits on rows claimed earlier, whose threads are already running: no deadlock.
#include "device.cuh"
#include "internal.h"

namespace spuma {
namespace {

__device__ __forceinline__ int ld_acquire(const int* p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v)
{
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Deadlock guard: a dependency that never arrives (a corrupted schedule) must not hang the GPU.
// After kSpinLimit polls (~2 s with the back-off) the row gives up, raises flag[N] (the error
// word past the row flags, read by the host after the solve) and continues.
constexpr unsigned kSpinLimit = 1u << 22;
__device__ __forceinline__ void spin_fail(int* err) { atomicExch(err, 1); }

__device__ __forceinline__ void wait_ready(const int* flag, int j, int* err)
{
    if (ld_acquire(flag + j)) return;
    unsigned ns = 32, polls = 0;
    while (!ld_acquire(flag + j)) {  // back off: keep the L2 free for the rows that can progress
        __nanosleep(ns);
        ns = ns < 512 ? 2 * ns : 512;
        if (++polls > kSpinLimit) {
            spin_fail(err);
            return;
        }
    }
}

// wait until the flags of all n (<= kDep) dependencies are set: all polls in flight at once
constexpr int kDep = 8;
__device__ __forceinline__ void wait_all(const int* flag, const int* js, int n, int* err)
{
    unsigned ns = 32, polls = 0;
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int d = 0; d < kDep; ++d)
            if (d < n && !ld_acquire(flag + js[d])) ok = false;
        if (ok) return;
        __nanosleep(ns);
        ns = ns < 512 ? 2 * ns : 512;
        if (++polls > kSpinLimit) {
            spin_fail(err);
            return;
        }
    }
}

// a warp claims 32 consecutive rows of the schedule with one atomic
__device__ __forceinline__ unsigned claim_rows(unsigned* counter)
{
    unsigned base = 0;
    if ((threadIdx.x & 31) == 0) base = atomicAdd(counter, 32u);
    return __shfl_sync(0xffffffffu, base, 0) + (threadIdx.x & 31);
}

// Factor (Q31): raw[c] = diag[c] - sum over faces with neighbour c (face order) of
// upper*lower/raw[owner]; the reciprocal is taken by k_ilu_recip afterwards.
__global__ void __launch_bounds__(kThreads) k_ilu_factor(MeshArgs a, const int* __restrict__ order,
                                                         const double* __restrict__ diag,
                                                         const double* __restrict__ upper,
                                                         const double* __restrict__ lower, double* raw, int* flag,
                                                         unsigned* counter)
{
    for (;;) {
        const unsigned i = claim_rows(counter);
        if (i - (threadIdx.x & 31) >= (unsigned)a.N) break;  // warp-uniform exit
        if (i >= (unsigned)a.N) continue;
        const int c = order[i];
        const int k0 = a.losortStart[c], nd = a.losortStart[c + 1] - k0;
        int js[kDep];
        double cf[kDep], v[kDep];
#pragma unroll
        for (int d = 0; d < kDep; ++d)
            if (d < nd) {
                const int f = a.losort[k0 + d];
                js[d] = a.ownerLo[k0 + d];
                cf[d] = upper[f] * lower[f];
            }
        wait_all(flag, js, nd < kDep ? nd : kDep, flag + a.N);
#pragma unroll
        for (int d = 0; d < kDep; ++d)
            if (d < nd) v[d] = __ldcg(raw + js[d]);
        double t = diag[c];
#pragma unroll
        for (int d = 0; d < kDep; ++d)
            if (d < nd) t = t - cf[d] / v[d];
        for (int k = k0 + kDep; k < k0 + nd; ++k) {  // rows with more than kDep lower faces
            const int j = a.ownerLo[k], f = a.losort[k];
            wait_ready(flag, j, flag + a.N);
            t = t - upper[f] * lower[f] / __ldcg(raw + j);
        }
        __stcg(raw + c, t);
        st_release(flag + c, 1);
    }
}

__global__ void k_ilu_recip(int N, const double* __restrict__ raw, double* __restrict__ rD)
{
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) rD[c] = 1.0 / raw[c];
}

// The sweeps publish each row's VALUE as its ready flag: the output array is pre-filled with
// kPending (a NaN payload no arithmetic on finite data produces) and a row's result is written
// with one release store, so a consumer's acquire load of the dependency returns the value
// itself -- one L2 round trip per dependency level instead of flag + value.
constexpr unsigned long long kPending = 0x7FF4DEADBEEF0001ull;

__device__ __forceinline__ unsigned long long ld_acquire_u64(const double* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_f64(double* p, double v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"((unsigned long long)__double_as_longlong(v))
                 : "memory");
}

// the values of all n (<= kDep) dependencies, polled together (bounded, back-off)
__device__ __forceinline__ void wait_values(const double* w, const int* js, int n, double* v, int* err)
{
    bool have[kDep];
#pragma unroll
    for (int d = 0; d < kDep; ++d) have[d] = d >= n;
    unsigned ns = 32, polls = 0;
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int d = 0; d < kDep; ++d)
            if (!have[d]) {
                const unsigned long long u = ld_acquire_u64(w + js[d]);
                if (u != kPending) {
                    v[d] = __longlong_as_double((long long)u);
                    have[d] = true;
                } else {
                    ok = false;
                }
            }
        if (ok) return;
        __nanosleep(ns);
        ns = ns < 64 ? 2 * ns : 64;  // short back-off: the sweep is latency-bound (-2 % vs 512 ns)
        if (++polls > kSpinLimit) {
            spin_fail(err);
#pragma unroll
            for (int d = 0; d < kDep; ++d)
                if (!have[d]) v[d] = 0.0;
            return;
        }
    }
}

__device__ __forceinline__ double wait_value(const double* w, int j, int* err)
{
    double v;
    wait_values(w, &j, 1, &v, err);
    return v;
}

__global__ void k_fill_pending(int N, double* __restrict__ w, const DevScal* scal)
{
    if (scal && scal->done) return;  // the sweeps are no-ops then: leave w as it is
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x)
        w[c] = __longlong_as_double((long long)kPending);
}

// Forward sweep: y[c] = rD[c] r[c], then y[c] -= rD[c]*lo[f]*y[owner] over the faces with
// neighbour c in face order.  y: pre-filled with kPending.
__global__ void __launch_bounds__(kThreads) k_ilu_fwd(MeshArgs a, const int* __restrict__ order,
                                                      const double* __restrict__ rD, const double* __restrict__ lo,
                                                      const double* __restrict__ r, double* y, int* err,
                                                      unsigned* counter, const DevScal* scal)
{
    if (scal && scal->done) return;
    for (;;) {
        const unsigned i = claim_rows(counter);
        if (i - (threadIdx.x & 31) >= (unsigned)a.N) break;
        if (i >= (unsigned)a.N) continue;
        const int c = order[i];
        const double rd = rD[c];
        const int k0 = a.losortStart[c], nd = a.losortStart[c + 1] - k0;
        int js[kDep];
        double cf[kDep], v[kDep];
#pragma unroll
        for (int d = 0; d < kDep; ++d)
            if (d < nd) {
                js[d] = a.ownerLo[k0 + d];
                cf[d] = rd * lo[a.losort[k0 + d]];
            }
        double t = rd * r[c];
        wait_values(y, js, nd < kDep ? nd : kDep, v, err);
#pragma unroll
        for (int d = 0; d < kDep; ++d)
            if (d < nd) t = t - cf[d] * v[d];
        for (int k = k0 + kDep; k < k0 + nd; ++k) t = t - rd * lo[a.losort[k]] * wait_value(y, a.ownerLo[k], err);
        st_release_f64(y + c, t);
    }
}

// Backward sweep (rows in reverse dependency order): w[c] = y[c] - rD[c]*up[f]*w[neighbour] over
// the faces with owner c in DESCENDING face order.  y: the forward result; w pre-filled with kPending.
__global__ void __launch_bounds__(kThreads) k_ilu_bwd(MeshArgs a, const int* __restrict__ order,
                                                      const double* __restrict__ rD, const double* __restrict__ up,
                                                      const double* __restrict__ y, double* w, int* err,
                                                      unsigned* counter, const DevScal* scal)
{
    if (scal && scal->done) return;
    for (;;) {
        const unsigned i = claim_rows(counter);
        if (i - (threadIdx.x & 31) >= (unsigned)a.N) break;
        if (i >= (unsigned)a.N) continue;
        const int c = order[i];
        const double rd = rD[c];
        const int f1 = a.ownerStart[c + 1] - 1, nd = f1 + 1 - a.ownerStart[c];
        int js[kDep];
        double cf[kDep], v[kDep];
#pragma unroll
        for (int d = 0; d < kDep; ++d)
            if (d < nd) {
                js[d] = a.neighbour[f1 - d];
                cf[d] = rd * up[f1 - d];
            }
        double t = y[c];
        wait_values(w, js, nd < kDep ? nd : kDep, v, err);
#pragma unroll
        for (int d = 0; d < kDep; ++d)
            if (d < nd) t = t - cf[d] * v[d];
        for (int f = f1 - kDep; f >= a.ownerStart[c]; --f) t = t - rd * up[f] * wait_value(w, a.neighbour[f], err);
        st_release_f64(w + c, t);
    }
}

// aDILU (Q33) forward pass: out[c] = y0[c] - sum (rD[c]*lo[f]) * prev[owner] (face order);
// y0 == nullptr: y0 = rD r.  Backward pass: out[c] = y0[c] - sum over owner faces in
// descending order of (rD[c]*up[f]) * prev[neighbour].
__global__ void __launch_bounds__(kThreads) k_adilu_pass(MeshArgs a, int backward, const double* __restrict__ rD,
                                                         const double* __restrict__ coef,
                                                         const double* __restrict__ r,
                                                         const double* __restrict__ y0,
                                                         const double* __restrict__ prev, double* __restrict__ out,
                                                         const DevScal* scal)
{
    if (scal && scal->done) return;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
        const double rd = rD[c];
        double t = y0 ? y0[c] : rd * r[c];
        if (!backward) {
            for (int k = a.losortStart[c]; k < a.losortStart[c + 1]; ++k)
                t = t - rd * coef[a.losort[k]] * prev[a.ownerLo[k]];
        } else {
            for (int f = a.ownerStart[c + 1] - 1; f >= a.ownerStart[c]; --f) t = t - rd * coef[f] * prev[a.neighbour[f]];
        }
        out[c] = t;
    }
}

// aDILU with the pass coefficients rD[c]*coef[f] formed once per solve in the pass's row order
// (forward: losort order, contiguous per row -- no face indirection; backward: face order):
// fco/bco for M^-1, fcoT/bcoT for M^-T (lower/upper swapped).  (rD*coef)*prev is the pass's own
// rounding, so the passes below are bitwise k_adilu_pass.
__global__ void __launch_bounds__(kThreads) k_adilu_coefs(MeshArgs a, const double* __restrict__ rD,
                                                          const double* __restrict__ up,
                                                          const double* __restrict__ lo, double* __restrict__ fco,
                                                          double* __restrict__ bco, double* __restrict__ fcoT,
                                                          double* __restrict__ bcoT)
{
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
        const double rd = rD[c];
        for (int k = a.losortStart[c]; k < a.losortStart[c + 1]; ++k) {
            const int f = a.losort[k];
            fco[k] = rd * lo[f];
            fcoT[k] = rd * up[f];
        }
        for (int f = a.ownerStart[c]; f < a.ownerStart[c + 1]; ++f) {
            bco[f] = rd * up[f];
            bcoT[f] = rd * lo[f];
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_adilu_pass_pre(MeshArgs a, int backward, const double* __restrict__ pre,
                                                             const double* __restrict__ rD,
                                                             const double* __restrict__ r,
                                                             const double* __restrict__ y0,
                                                             const double* __restrict__ prev,
                                                             double* __restrict__ out, const DevScal* scal)
{
    if (scal && scal->done) return;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
        double t = y0 ? y0[c] : rD[c] * r[c];
        if (!backward) {
            const int k1 = a.losortStart[c + 1];
            for (int k = a.losortStart[c]; k < k1; ++k) t = t - pre[k] * prev[a.ownerLo[k]];
        } else {
            for (int f = a.ownerStart[c + 1] - 1; f >= a.ownerStart[c]; --f) t = t - pre[f] * prev[a.neighbour[f]];
        }
        out[c] = t;
    }
}

// w = rD r (diagonal preconditioner; also aDILU with k = 0)
__global__ void k_pc_diag(int N, const double* __restrict__ rD, const double* __restrict__ r, double* __restrict__ w,
                          const DevScal* scal)
{
    if (scal && scal->done) return;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) w[c] = rD[c] * r[c];
}

// wArA (PCG) / wArT (PBiCG) = w . r; beta = wArA / wArAold (used from the second iteration)
__global__ void __launch_bounds__(kThreads) k_pc_dot(int N, const double* __restrict__ w, const double* __restrict__ r,
                                                     double* part, DevScal* scal, int fin)
{
    if (scal->done) return;
    double v[1] = {0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) v[0] += w[c] * r[c];
    if (grid_sum<1>(v, part, &scal->ticket[5]) && threadIdx.x == 0) {
        if (fin) finalize(scal, 5, v);
        else scal->rank_part[0] = v[0];  // P > 1: global sum + finalize(5) by reduce_finalize
    }
}

// pA = wA (+ beta pA); pT = wT (+ beta pT) when pT != nullptr
__global__ void k_pc_direction(int N, const double* __restrict__ wA, double* __restrict__ pA,
                               const double* __restrict__ wT, double* __restrict__ pT, const DevScal* scal)
{
    if (scal->done) return;
    const bool first = scal->n == 0;
    const double beta = scal->beta;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
        pA[c] = first ? wA[c] : wA[c] + beta * pA[c];
        if (pT) pT[c] = first ? wT[c] : wT[c] + beta * pT[c];
    }
}

// asymmetric row of A (upper on the owner side, lower on the neighbour side) and of A^T, then the
// processor-interface terms icoef * x_remote in (patch, face) order (Q10) when icoef is given
__device__ __forceinline__ double row_asym(const MeshArgs& a, int c, const double* __restrict__ diag,
                                           const double* __restrict__ nbr_coef, const double* __restrict__ own_coef,
                                           const double* __restrict__ x, const double* __restrict__ icoef = nullptr,
                                           const double* __restrict__ xr = nullptr)
{
    double s = diag[c] * x[c];
    for (int k = a.losortStart[c]; k < a.losortStart[c + 1]; ++k) s = s + nbr_coef[a.losort[k]] * x[a.ownerLo[k]];
    for (int f = a.ownerStart[c]; f < a.ownerStart[c + 1]; ++f) s = s + own_coef[f] * x[a.neighbour[f]];
    if (icoef && a.ifStart)
        for (int j = a.ifStart[c]; j < a.ifStart[c + 1]; ++j) s = s + icoef[a.ifIdx[j]] * xr[a.ifIdx[j]];
    return s;
}

// PBiCG: wA = A pA, wT = A^T pT, wApT = wA . pT -> alpha, singularity (Q32; finalize stage 3)
__global__ void __launch_bounds__(kThreads) k_bicg_amul_tmul(MeshArgs a, const double* __restrict__ diag,
                                                             const double* __restrict__ upper,
                                                             const double* __restrict__ lower,
                                                             const double* __restrict__ iface,
                                                             const double* __restrict__ iface_t,
                                                             const double* __restrict__ pA,
                                                             const double* __restrict__ pT,
                                                             const double* __restrict__ xr,
                                                             const double* __restrict__ xrT, double* __restrict__ wA,
                                                             double* __restrict__ wT, double* part, DevScal* scal,
                                                             int fin)
{
    if (scal->done) return;
    double v[1] = {0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
        const double ya = row_asym(a, c, diag, lower, upper, pA, iface, xr);
        const double yt = row_asym(a, c, diag, upper, lower, pT, iface_t, xrT);
        wA[c] = ya;
        wT[c] = yt;
        v[0] += ya * pT[c];
    }
    if (grid_sum<1>(v, part, &scal->ticket[6]) && threadIdx.x == 0) {
        if (fin) finalize(scal, 3, v);
        else scal->rank_part[0] = v[0];
    }
}

// PBiCG update: psi += alpha pA, rA -= alpha wA, rT -= alpha wT; |rA| -> finalize stage 4
__global__ void __launch_bounds__(kThreads) k_bicg_update(int N, double* __restrict__ psi,
                                                          const double* __restrict__ pA,
                                                          double* __restrict__ rA, const double* __restrict__ wA,
                                                          double* __restrict__ rT, const double* __restrict__ wT,
                                                          double* part, DevScal* scal, int fin)
{
    if (scal->done) return;
    const double alpha = scal->alpha;
    double v[2] = {0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
        psi[c] = psi[c] + alpha * pA[c];
        const double r = rA[c] - alpha * wA[c];
        rA[c] = r;
        if (rT) rT[c] = rT[c] - alpha * wT[c];
        v[1] += fabs(r);
    }
    if (grid_sum<2>(v, part, &scal->ticket[7]) && threadIdx.x == 0) {
        if (fin) finalize(scal, 4, v);
        else scal->rank_part[0] = v[0], scal->rank_part[1] = v[1];
    }
}

// PBiCG setup: wA = A psi, wT = A^T psi, rA = b - wA, rT = b - wT, sumA = row sums incl. the
// Amul interface coefficients (Q17, Q35); sum of psi and N -> finalize stage 1 (gAverage)
__global__ void __launch_bounds__(kThreads) k_bicg_setup(MeshArgs a, const double* __restrict__ diag,
                                                         const double* __restrict__ upper,
                                                         const double* __restrict__ lower,
                                                         const double* __restrict__ iface,
                                                         const double* __restrict__ iface_t,
                                                         const double* __restrict__ xr,
                                                         const double* __restrict__ source,
                                                         const double* __restrict__ psi, double* __restrict__ wA,
                                                         double* __restrict__ wT, double* __restrict__ rA,
                                                         double* __restrict__ rT, double* __restrict__ sumA,
                                                         double* part, DevScal* scal, int fin)
{
    double v[2] = {0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
        const double ya = row_asym(a, c, diag, lower, upper, psi, iface, xr);
        const double yt = row_asym(a, c, diag, upper, lower, psi, iface_t, xr);
        double s = diag[c];
        for (int k = a.losortStart[c]; k < a.losortStart[c + 1]; ++k) s = s + lower[a.losort[k]];
        for (int f = a.ownerStart[c]; f < a.ownerStart[c + 1]; ++f) s = s + upper[f];
        if (iface && a.ifStart)
            for (int j = a.ifStart[c]; j < a.ifStart[c + 1]; ++j) s = s + iface[a.ifIdx[j]];
        wA[c] = ya;
        wT[c] = yt;
        rA[c] = source[c] - ya;
        rT[c] = source[c] - yt;
        sumA[c] = s;
        v[0] += psi[c];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) v[1] = (double)a.N;
    if (grid_sum<2>(v, part, &scal->ticket[0]) && threadIdx.x == 0) {
        if (fin) finalize(scal, 1, v);
        else scal->rank_part[0] = v[0], scal->rank_part[1] = v[1];
    }
}

// normFactor and initial residual from wA, sumA, rA (Q1) -> finalize stage 2 (loop decision)
__global__ void __launch_bounds__(kThreads) k_pc_setup2(int N, const double* __restrict__ wA,
                                                        const double* __restrict__ sumA,
                                                        const double* __restrict__ source,
                                                        const double* __restrict__ rA, double* part, DevScal* s,
                                                        int fin)
{
    const double xbar = s->xbar;
    double v[3] = {0.0, 0.0, 0.0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
        const double xref = sumA[c] * xbar;
        v[0] += fabs(wA[c] - xref) + fabs(source[c] - xref);
        v[1] += fabs(rA[c]);
    }
    if (grid_sum<3>(v, part, &s->ticket[1]) && threadIdx.x == 0) {
        if (fin) finalize(s, 2, v);
        else s->rank_part[0] = v[0], s->rank_part[1] = v[1], s->rank_part[2] = 0.0;
    }
}

// CSR values: vals[k] = [diag | upper | lower][map[k]]
__global__ void k_csr_values(int nnz, int N, int F, const int* __restrict__ map, const double* __restrict__ diag,
                             const double* __restrict__ upper, const double* __restrict__ lower,
                             double* __restrict__ vals)
{
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += gridDim.x * blockDim.x) {
        const int m = map[k];
        vals[k] = m < N ? diag[m] : (m < N + F ? upper[m - N] : lower[m - N - F]);
    }
}

// internal (upper, lower) from the caller's through the face map; faces whose orientation RCM
// reversed swap their two coefficients
__global__ void k_gather_pair(int F, const int* __restrict__ map, const signed char* __restrict__ flip,
                              const double* __restrict__ u, const double* __restrict__ l, double* __restrict__ uo,
                              double* __restrict__ lo)
{
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
        const int g = map[f];
        const bool sw = flip && flip[f];
        uo[f] = sw ? l[g] : u[g];
        lo[f] = sw ? u[g] : l[g];
    }
}

__global__ void k_amul_asym(MeshArgs a, const double* __restrict__ diag, const double* __restrict__ upper,
                            const double* __restrict__ lower, const double* __restrict__ x, double* __restrict__ y,
                            int transpose)
{
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x)
        y[c] = transpose ? row_asym(a, c, diag, upper, lower, x) : row_asym(a, c, diag, lower, upper, x);
}

int persistent_grid(const void* kernel, int cap_threads = 1 << 30)
{
    static int sms = 0;
    int dev = 0, occ = 1;
    if (!sms) {
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0);
    const int full = sms * (occ > 0 ? occ : 1);
    const int want = (cap_threads + kThreads - 1) / kThreads;
    return want < 1 ? 1 : (want < full ? want : full);
}

int cell_grid(int n)
{
    const int g = (n + kThreads - 1) / kThreads;
    return g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g);
}

}  // namespace

// grids of the reduction kernels are fixed per N (deterministic partial order)
int pc_grid(int n) { return cell_grid(n); }

void launch_ilu_factor(cudaStream_t s, const MeshArgs& a, const int* order, const double* diag, const double* upper,
                       const double* lower, double* raw, double* rD, int* flag, unsigned* counter, int width)
{
    cudaMemsetAsync(flag, 0, sizeof(int) * a.N, s);
    cudaMemsetAsync(counter, 0, sizeof(unsigned), s);
    k_ilu_factor<<<persistent_grid((const void*)k_ilu_factor, 2 * width), kThreads, 0, s>>>(a, order, diag, upper,
                                                                                           lower, raw, flag, counter);
    k_ilu_recip<<<cell_grid(a.N), kThreads, 0, s>>>(a.N, raw, rD);
}

// w = M^-1 r (transpose: M^-T r).  k < 0: exact sweeps; k >= 0: aDILU with k passes per sweep.
void launch_ilu_precondition(cudaStream_t s, const MeshArgs& a, const int* order_f, const int* order_b,
                             const double* rD, const double* upper, const double* lower, const double* r, double* w,
                             double* t1, double* t2, int* flag, unsigned* counter, int k, bool transpose,
                             const DevScal* scal, int width_f, int width_b, const double* fpre, const double* bpre)
{
    const double* lo = transpose ? upper : lower;
    const double* up = transpose ? lower : upper;
    if (k < 0) {  // forward result in t1, backward into w (values as flags, kPending = not yet)
        k_fill_pending<<<cell_grid(a.N), kThreads, 0, s>>>(a.N, t1, scal);
        cudaMemsetAsync(counter, 0, sizeof(unsigned), s);
        k_ilu_fwd<<<persistent_grid((const void*)k_ilu_fwd, 2 * width_f), kThreads, 0, s>>>(a, order_f, rD, lo, r, t1,
                                                                                           flag + a.N, counter, scal);
        k_fill_pending<<<cell_grid(a.N), kThreads, 0, s>>>(a.N, w, scal);
        cudaMemsetAsync(counter, 0, sizeof(unsigned), s);
        k_ilu_bwd<<<persistent_grid((const void*)k_ilu_bwd, 2 * width_b), kThreads, 0, s>>>(a, order_b, rD, up, t1, w,
                                                                                           flag + a.N, counter, scal);
        return;
    }
    if (k == 0) {
        k_pc_diag<<<cell_grid(a.N), kThreads, 0, s>>>(a.N, rD, r, w, scal);
        return;
    }
    // forward passes: prev_0 = y_0 = rD r in t1; out_i alternates t2, t1, ... (y_0 stays implicit via r)
    k_pc_diag<<<cell_grid(a.N), kThreads, 0, s>>>(a.N, rD, r, t1, scal);
    double* prev = t1;
    for (int it = 0; it < k; ++it) {
        double* out = prev == t1 ? t2 : t1;
        if (fpre) k_adilu_pass_pre<<<cell_grid(a.N), kThreads, 0, s>>>(a, 0, fpre, rD, r, nullptr, prev, out, scal);
        else k_adilu_pass<<<cell_grid(a.N), kThreads, 0, s>>>(a, 0, rD, lo, r, nullptr, prev, out, scal);
        prev = out;
    }
    // backward passes from w_0 = y (kept in Y): out_i alternates Z / w so that out_k = w
    double* Y = prev;
    double* Z = Y == t1 ? t2 : t1;
    const double* bprev = Y;
    for (int it = 0; it < k; ++it) {
        double* out = ((k - 1 - it) & 1) ? Z : w;
        if (bpre) k_adilu_pass_pre<<<cell_grid(a.N), kThreads, 0, s>>>(a, 1, bpre, rD, r, Y, bprev, out, scal);
        else k_adilu_pass<<<cell_grid(a.N), kThreads, 0, s>>>(a, 1, rD, up, r, Y, bprev, out, scal);
        bprev = out;
    }
}

void launch_adilu_coefs(cudaStream_t s, const MeshArgs& a, const double* rD, const double* upper,
                        const double* lower, double* fco, double* bco, double* fcoT, double* bcoT)
{
    if (a.N <= 0) return;
    k_adilu_coefs<<<cell_grid(a.N), kThreads, 0, s>>>(a, rD, upper, lower, fco, bco, fcoT, bcoT);
}

void launch_recip(cudaStream_t s, int N, const double* in, double* out)
{
    k_ilu_recip<<<cell_grid(N), kThreads, 0, s>>>(N, in, out);
}

void launch_pc_dot(cudaStream_t s, int N, const double* w, const double* r, double* part, DevScal* scal, bool fin)
{
    k_pc_dot<<<cell_grid(N), kThreads, 0, s>>>(N, w, r, part, scal, fin ? 1 : 0);
}

void launch_pc_direction(cudaStream_t s, int N, const double* wA, double* pA, const double* wT, double* pT,
                         const DevScal* scal)
{
    k_pc_direction<<<cell_grid(N), kThreads, 0, s>>>(N, wA, pA, wT, pT, scal);
}

void launch_bicg_amul_tmul(cudaStream_t s, const MeshArgs& a, const double* diag, const double* upper,
                           const double* lower, const double* iface, const double* iface_t, const double* pA,
                           const double* pT, const double* xr, const double* xrT, double* wA, double* wT,
                           double* part, DevScal* scal, bool fin)
{
    k_bicg_amul_tmul<<<cell_grid(a.N), kThreads, 0, s>>>(a, diag, upper, lower, iface, iface_t, pA, pT, xr, xrT, wA,
                                                        wT, part, scal, fin ? 1 : 0);
}

void launch_bicg_update(cudaStream_t s, int N, double* psi, const double* pA, double* rA, const double* wA, double* rT,
                        const double* wT, double* part, DevScal* scal, bool fin)
{
    k_bicg_update<<<cell_grid(N), kThreads, 0, s>>>(N, psi, pA, rA, wA, rT, wT, part, scal, fin ? 1 : 0);
}

void launch_bicg_setup1(cudaStream_t s, const MeshArgs& a, const double* diag, const double* upper,
                        const double* lower, const double* iface, const double* iface_t, const double* xr,
                        const double* source, const double* psi, double* wA, double* wT, double* rA, double* rT,
                        double* sumA, double* part, DevScal* scal, bool fin)
{
    k_bicg_setup<<<cell_grid(a.N), kThreads, 0, s>>>(a, diag, upper, lower, iface, iface_t, xr, source, psi, wA, wT,
                                                    rA, rT, sumA, part, scal, fin ? 1 : 0);
}

void launch_pc_setup2(cudaStream_t s, int N, const double* wA, const double* sumA, const double* source,
                      const double* rA, double* part, DevScal* scal, bool fin)
{
    k_pc_setup2<<<cell_grid(N), kThreads, 0, s>>>(N, wA, sumA, source, rA, part, scal, fin ? 1 : 0);
}

void launch_gather_pair(cudaStream_t s, int F, const int* map, const signed char* flip, const double* u,
                        const double* l, double* uo, double* lo)
{
    k_gather_pair<<<cell_grid(F), kThreads, 0, s>>>(F, map, flip, u, l, uo, lo);
}

void launch_amul_asym(cudaStream_t s, const MeshArgs& a, const double* diag, const double* upper,
                      const double* lower, const double* x, double* y, bool transpose)
{
    k_amul_asym<<<cell_grid(a.N), kThreads, 0, s>>>(a, diag, upper, lower, x, y, transpose ? 1 : 0);
}

void launch_csr_values(cudaStream_t s, int nnz, int N, int F, const int* map, const double* diag,
                       const double* upper, const double* lower, double* vals)
{
    k_csr_values<<<cell_grid(nnz), kThreads, 0, s>>>(nnz, N, F, map, diag, upper, lower, vals);
}

}  // namespace spuma
