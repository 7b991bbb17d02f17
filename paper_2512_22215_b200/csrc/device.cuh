// device.cuh -- device helpers shared by the libspuma kernel files (reductions, the
// oracle-order row gather).  Header-only; every function is inlined into its caller.
#pragma once
#include "internal.h"

namespace spuma {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------

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

}  // namespace spuma
