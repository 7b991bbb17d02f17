// device.cuh -- device helpers shared by the libspuma kernel files (reductions, the
// oracle-order row gather).  Header-only; every function is inlined into its caller.
#pragma once
#include "internal.h"

namespace spuma {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------

// Grid-stride index sequence of this thread over [0, n): ascending, or descending when rev
// (consecutive kernels that alternate the direction start on the lines the previous one
// touched last, which are still in L2).  The same indices either way; only the order (and
// hence the rounding of per-thread partial sums) changes.
struct GridStride {
    int i0, st, cnt, rev;
    __device__ __forceinline__ GridStride(int n, int r)
        : i0(blockIdx.x * blockDim.x + threadIdx.x), st(gridDim.x * blockDim.x), rev(r)
    {
        cnt = i0 < n ? (n - 1 - i0) / st + 1 : 0;
    }
    __device__ __forceinline__ int at(int j) const { return i0 + (rev ? cnt - 1 - j : j) * st; }
};

// Sum NV values over the CTA; the result is valid in thread 0.
template <int NV>
__device__ __forceinline__ void cta_sum(double (&v)[NV])
{
    __shared__ double sh[NV][kThreads / 32];
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
        const int nw = blockDim.x >> 5;  // <= kThreads / 32
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double t = lane < nw ? sh[i][lane] : 0.0;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
            v[i] = t;
        }
    }
    __syncthreads();
}

// Store this CTA's partials; return true in the LAST CTA to finish, which then
// holds the grid-wide sums (CTA order) in v (thread 0).
template <int NV>
__device__ __forceinline__ bool grid_sum(double (&v)[NV], double* part, unsigned int* ticket)
{
    __shared__ bool last;
    cta_sum<NV>(v);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) part[i * gridDim.x + blockIdx.x] = v[i];
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double t = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) t += __ldcg(part + i * gridDim.x + b);
        v[i] = t;
    }
    cta_sum<NV>(v);
    if (threadIdx.x == 0) *ticket = 0u;
    return true;
}

// Programmatic dependent launch (sm_90+): a hot-loop kernel launched with the PDL
// attribute may start while its predecessor drains; it must wait before reading the
// predecessor's results, and lets its own successor launch once its main loop is done.
// Both are no-ops for a normal launch.
#ifndef SPUMA_NO_PDL_INSTR
static __device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
static __device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#else
static __device__ __forceinline__ void pdl_wait() {}
static __device__ __forceinline__ void pdl_trigger() {}
#endif

static __device__ __forceinline__ bool conv(double r, double init, double tol, double rel_tol)
{
    return (r < tol) || (rel_tol > 1e-20 && r < rel_tol * init);
}

// y_c = (A x)_c in the oracle's face order (reading Q10).
static __device__ __forceinline__ double amul_row(const MeshArgs& a, int c, const double* __restrict__ diag,
                                           const double* __restrict__ upper, const double* __restrict__ iface,
                                           const double* __restrict__ x, const double* __restrict__ xr,
                                           double* rowsum, bool iface_terms = true)
{
    double s = diag[c] * x[c];
    double r = diag[c];
    const int k1 = a.losortStart[c + 1];
    for (int k = a.losortStart[c]; k < k1; ++k) {
        const double u = upper[a.losort[k]];
        s = s + u * x[a.ownerLo[k]];
        r = r + u;
    }
    const int f1 = a.ownerStart[c + 1];
    for (int f = a.ownerStart[c]; f < f1; ++f) {
        const double u = upper[f];
        s = s + u * x[a.neighbour[f]];
        r = r + u;
    }
    if (a.ifStart && iface_terms) {
        const int j1 = a.ifStart[c + 1];
        for (int j = a.ifStart[c]; j < j1; ++j) {
            const int i = a.ifIdx[j];
            s = s + iface[i] * xr[i];
            r = r + iface[i];
        }
    }
    if (rowsum) *rowsum = r;
    return s;
}

// Finalisation steps of the PCG scalars, from global sums g[].
static __device__ void finalize(DevScal* s, int stage, const double* g)
{
    switch (stage) {
    case 1:  // gAverage(psi) = gSum(psi) / gSum(nCells)
        s->xbar = g[0] / g[1];
        break;
    case 2: {  // normFactor, initial residual, first wArA, iterate-at-all decision (Q1, Q3)
        s->normFactor = g[0] + 1e-20;
        s->init = g[1] / s->normFactor;
        s->fin = s->init;
        s->wArA = g[2];
        s->wArAold = 1e20;
        s->n = 0;
        s->singular = 0;
        s->converged = conv(s->fin, s->init, s->tol, s->rel_tol);
        s->done = !(s->min_iter > 0 || !s->converged);
        break;
    }
    case 3: {  // alpha = wArA / wApA, checkSingularity (Q4)
        s->wApA = g[0];
        if (fabs(s->wApA) / s->normFactor < 1e-300) {
            s->singular = 1;
            s->done = 1;
        } else {
            s->alpha = s->wArA / s->wApA;
        }
        break;
    }
    case 4: {  // final residual, convergence, loop condition, beta for the next direction
        s->fin = g[1] / s->normFactor;
        s->n = s->n + 1;
        const bool c = conv(s->fin, s->init, s->tol, s->rel_tol);
        s->converged = c;
        if (!((s->n < s->max_iter && !c) || s->n < s->min_iter)) s->done = 1;
        s->wArAold = s->wArA;
        s->wArA = g[0];
        s->beta = s->wArA / s->wArAold;
        s->alpha_prev2 = s->alpha_prev;
        s->alpha_prev = s->alpha;  // a deferred psi update of this iteration uses it
        break;
    }
    case 5:  // preconditioned loops (§8(f4)): wArA = wA.rA from the general preconditioner, beta
        s->wArA = g[0];
        s->beta = s->wArA / s->wArAold;
        break;
    }
}

// ---------------------------------------------------------------------------
// peer-memory transport primitives (peer.cu, and the PCG loop's fused halo / all-gather)
// ---------------------------------------------------------------------------
static __device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

static __device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// wait until *f >= e (thread-local poll); false on timeout (error word set)
static __device__ bool wait_flag(const unsigned long long* f, unsigned long long e, int* err, long long limit)
{
    const long long t0 = clock64();
    unsigned ns = 32;
    while (ld_acquire_sys(f) < e) {
        if (*reinterpret_cast<volatile int*>(err)) return false;  // an earlier exchange already failed
        if (clock64() - t0 > limit) {
            atomicExch(err, 1);
            return false;
        }
        __nanosleep(ns);
        ns = ns < 4096 ? 2 * ns : ns;
    }
    return true;
}

// The rank-partial all-gather of the peer transport, then the PCG finalisation: publish this
// rank's 4 partials (in) into every rank's mailbox slot + flag, wait for every rank's flag, copy
// the rank-ordered block to out, and (stage > 0) finalise the scalars from it in rank order --
// the sums of k_finalize, so every rank takes bitwise the same decisions.  Called by every
// thread of ONE CTA (blockDim >= n_ranks): k_peer_allgather4, or the last CTA of a reduction
// kernel of the fused PCG loop (compute and collective in one kernel).  A timed-out gather stops
// the loop (done) instead of finalising stale values.
static __device__ void peer_gather_finalize(const PeerGather& g, const PeerState& st, const double* in,
                                            double* out, int stage, DevScal* sc)
{
    __shared__ unsigned long long se;
    __shared__ int ok;
    if (threadIdx.x == 0) {
        se = st.ctr[1] + 1;
        ok = 1;
    }
    __syncthreads();
    const unsigned long long e = se;
    const int par = (int)(e & 1ull);
    const int t = threadIdx.x;
    if (t < g.n_ranks) {
        double* dst = g.part[t][par] + 4 * g.rank;
#pragma unroll
        for (int k = 0; k < 4; ++k) dst[k] = in[k];
        __threadfence_system();
        st_release_sys(g.flag[t][par] + g.rank, e);
    }
    __syncthreads();
    if (t < g.n_ranks && !wait_flag(g.my_flag[par] + t, e, st.err, st.poll_cycles)) ok = 0;
    __syncthreads();
    if (ok && t < g.n_ranks)
#pragma unroll
        for (int k = 0; k < 4; ++k) out[4 * t + k] = g.my_part[par][4 * t + k];
    if (t == 0) st.ctr[1] = e;
    if (stage > 0) {
        __syncthreads();
        if (t == 0) {
            if (!ok) {
                sc->done = 1;
            } else if (!(stage >= 3 && sc->done)) {
                double v[4] = {0.0, 0.0, 0.0, 0.0};
                for (int r = 0; r < g.n_ranks; ++r)
                    for (int i = 0; i < 4; ++i) v[i] += out[4 * r + i];
                finalize(sc, stage, v);
            }
        }
    }
}

template <int NV>
__device__ __forceinline__ void cta_sum_1024(double (&v)[NV])
{
    __shared__ double sh[NV][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
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
            double t = lane < nw ? sh[i][lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
            v[i] = t;
        }
    }
    __syncthreads();
}

// The whole PCG solve (A6-A12) by one CTA of up to kSmallThreads threads (small meshes, GAMG coarsest
// level); rows strided by the block size (the small-solve launchers size it to the mesh).
// p / sc / w's vectors / a's addressing may live in global or shared memory (k_pcg_single_smem).
static __device__ void pcg_single_body(const MeshArgs& a, const Workspace& w, const DevPtrs& p, DevScal* sc)
{
    const int N = a.N, t = threadIdx.x;
    {  // A6: wA = A psi, sumA, gAverage(psi)
        double v[2] = {0.0, 0.0};
        for (int c = t; c < N; c += (int)blockDim.x) {
            double rs;
            w.wA[c] = amul_row(a, c, p.diag, p.upper, p.iface, p.psi, w.xr, &rs);
            w.sumA[c] = rs;
            v[0] += p.psi[c];
        }
        if (t == 0) v[1] = (double)N;
        cta_sum_1024<2>(v);
        if (t == 0) finalize(sc, 1, v);
        __syncthreads();
    }
    {  // A6: residual, normFactor, rD, first wArA
        const double xbar = sc->xbar;
        double v[3] = {0.0, 0.0, 0.0};
        for (int c = t; c < N; c += (int)blockDim.x) {
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
        cta_sum_1024<3>(v);
        if (t == 0) finalize(sc, 2, v);
        __syncthreads();
    }
    while (!sc->done) {
        const bool first = sc->n == 0;
        const double beta = sc->beta;
        for (int c = t; c < N; c += (int)blockDim.x)  // A11
            w.pA[c] = first ? w.rD[c] * w.rA[c] : w.rD[c] * w.rA[c] + beta * w.pA[c];
        __syncthreads();
        double v[2] = {0.0, 0.0};
        for (int c = t; c < N; c += (int)blockDim.x) {  // A7
            const double y = amul_row(a, c, p.diag, p.upper, p.iface, w.pA, w.xr, nullptr);
            w.wA[c] = y;
            v[0] += y * w.pA[c];
        }
        cta_sum_1024<1>(reinterpret_cast<double(&)[1]>(v[0]));
        if (t == 0) finalize(sc, 3, v);  // A8
        __syncthreads();
        if (sc->done) break;
        const double alpha = sc->alpha;
        v[0] = v[1] = 0.0;
        for (int c = t; c < N; c += (int)blockDim.x) {  // A9
            p.psi[c] = p.psi[c] + alpha * w.pA[c];
            const double r = w.rA[c] - alpha * w.wA[c];
            w.rA[c] = r;
            v[0] += (w.rD[c] * r) * r;
            v[1] += fabs(r);
        }
        cta_sum_1024<2>(v);
        if (t == 0) finalize(sc, 4, v);  // A10
        __syncthreads();
    }
}

}  // namespace spuma

namespace spuma {
static __device__ void pcg_single_body(const MeshArgs& a, const Workspace& w)
{
    const DevPtrs p = *w.ptrs;
    pcg_single_body(a, w, p, w.scal);
}
}  // namespace spuma
