// peer.cu -- the device-side transport over peer memory (SURVEY §8(e), §5 "one-shot P2P via
// CUDA IPC"): every rank exports one mailbox (CUDA IPC handle); every rank maps the others'.
// Over NVLink / NVSwitch the stores below are P2P writes into the neighbour's HBM; ranks that
// share one GPU (the tests) map the same device memory.
//
//   halo (processor patches): the sender's kernel gathers x at its interface cells and stores
//     the values straight into the receiver's mailbox (pack and send fused, no staging buffer,
//     no NCCL), then -- after a system-scope fence by every CTA and a ticket -- the last CTA
//     publishes the exchange's epoch in the receiver's flag slot for this sender
//     (st.release.sys).  The receiver's kernel polls its flags (ld.acquire.sys, bounded,
//     nanosleep back-off) and copies its mailbox into x_remote.
//   all-gather of the 4 rank partials: one CTA stores this rank's partials into every rank's
//     mailbox slot [parity][rank] + flag, then waits for all ranks' flags and copies the rank-
//     ordered [n_ranks][4] block out -- every rank then finalises the same bits (rank order).
//
// Epochs: each rank counts its exchanges on the device (all ranks run the same sequence), so
// the kernels are graph-capturable.  Two mailbox halves (epoch parity) make reuse safe: a rank
// can only be one exchange ahead of a neighbour that has not yet consumed (it needs that
// neighbour's next message first).  A poll that exceeds its limit (~20 s by default,
// SPUMA_OPT_PEER_POLL_MS) sets the handle's error word instead of hanging the GPU; every
// collective call reads and clears it afterwards (api.cu peer_guard -> SPUMA_ERR_STATE).
#include "internal.h"
#include "device.cuh"

namespace spuma {
namespace {

// fused pack + send: dst[p][par][i] = (idx ? x[idx[off_p + i]] : x[off_p + i]) for every
// patch p, then the epoch into each receiver's flag slot (last CTA)
__global__ void __launch_bounds__(kThreads) k_peer_send(PeerXfer d, const double* __restrict__ x,
                                                        const int* __restrict__ idx, PeerState st)
{
    const unsigned long long e = st.ctr[0] + 1;
    const int par = (int)(e & 1ull);
    for (int p = 0; p < d.n_patches; ++p) {
        double* __restrict__ dst = d.dst[p][par];
        const int o = d.off[p], n = d.count[p];
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
            dst[i] = idx ? x[idx[o + i]] : x[o + i];
    }
    __threadfence_system();  // this thread's peer stores before the ticket
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(st.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int p = 0; p < d.n_patches; ++p) st_release_sys(d.dst_flag[p][par], e);
        st.ctr[0] = e;
        *st.ticket = 0u;
    }
}

// receive: wait for every patch's sender, then recv[off_p + i] = my mailbox region of p
__global__ void __launch_bounds__(kThreads) k_peer_recv(PeerXfer d, double* __restrict__ recv, PeerState st)
{
    const unsigned long long e = st.ctr[0];  // set by this rank's k_peer_send of the same exchange
    const int par = (int)(e & 1ull);
    __shared__ int ok;
    if (threadIdx.x == 0) {
        ok = 1;
        for (int p = 0; p < d.n_patches && ok; ++p)
            if (!wait_flag(d.src_flag[p][par], e, st.err, st.poll_cycles)) ok = 0;
    }
    __syncthreads();
    if (!ok) return;
    for (int p = 0; p < d.n_patches; ++p) {
        const double* __restrict__ src = d.src[p][par];
        const int o = d.off[p], n = d.count[p];
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) recv[o + i] = src[i];
    }
}

// all-gather of 4 doubles per rank (one CTA) and, stage > 0, the finalisation (device.cuh)
__global__ void k_peer_allgather4(PeerGather g, const double* __restrict__ in, double* __restrict__ out, PeerState st,
                                  int stage, Workspace w)
{
    peer_gather_finalize(g, st, in, out, stage, w.scal);
}

}  // namespace

void launch_peer_exchange(cudaStream_t s, const PeerXfer& d, const double* x, const int* idx, double* recv,
                          const PeerState& st)
{
    int total = 0;
    for (int p = 0; p < d.n_patches; ++p) total = d.count[p] > total ? d.count[p] : total;
    int grid = (total + kThreads - 1) / kThreads;
    grid = grid < 1 ? 1 : (grid > 592 ? 592 : grid);
    k_peer_send<<<grid, kThreads, 0, s>>>(d, x, idx, st);
    // the receiver polls: few CTAs, so that while it waits (on the comm stream, overlapped with
    // the interior Amul) it does not hold the SM slots the Amul runs in
    k_peer_recv<<<grid < 32 ? grid : 32, kThreads, 0, s>>>(d, recv, st);
}

void launch_peer_allgather4(cudaStream_t s, const PeerGather& g, const double* in, double* out, const PeerState& st,
                            int stage, const Workspace* w)
{
    k_peer_allgather4<<<1, 32 * ((g.n_ranks + 31) / 32), 0, s>>>(g, in, out, st, w ? stage : 0, w ? *w : Workspace{});
}

}  // namespace spuma
