// api.cu -- the C-ABI of libspuma (include/spuma.h): mesh handle, assembly,
// PCG orchestration (graph-captured iteration batches), NCCL halo exchange.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <string>
#include <vector>

#include "host.h"
#include "internal.h"

using namespace spuma;

namespace spuma {

static thread_local std::string g_err;

spuma_status set_error(spuma_status s, const std::string& msg)
{
    g_err = msg;
    return s;
}

}  // namespace spuma

namespace {

// every internal array carries kPad zeroed elements past its end (TMA windows); the
// zero-fill is synchronous so no stream can overtake it
template <class T>
spuma_status dalloc(T** p, size_t n)
{
    *p = nullptr;
    SPUMA_CUDA(cudaMalloc(reinterpret_cast<void**>(p), (n + kPad) * sizeof(T)));
    SPUMA_CUDA(cudaMemset(*p, 0, (n + kPad) * sizeof(T)));
    SPUMA_CUDA(cudaDeviceSynchronize());
    return SPUMA_OK;
}

template <class T>
spuma_status upload(T** p, const std::vector<T>& v, cudaStream_t s)
{
    SPUMA_TRY(dalloc(p, v.size()));
    if (!v.empty()) SPUMA_CUDA(cudaMemcpyAsync(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return SPUMA_OK;
}

bool is_device_ptr(const void* p)
{
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// host copy of a caller array that may live on the device
template <class T>
spuma_status fetch(std::vector<T>& out, const T* p, size_t n, bool on_device)
{
    out.resize(n);
    if (n == 0) return SPUMA_OK;
    if (!p) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array in mesh description");
    if (on_device) SPUMA_CUDA(cudaMemcpy(out.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost));
    else std::memcpy(out.data(), p, n * sizeof(T));
    return SPUMA_OK;
}

MeshArgs mesh_args(const spuma_mesh m)
{
    MeshArgs a{};
    a.N = m->N;
    a.F = m->F;
    a.ownerStart = m->d_ownerStart;
    a.losortStart = m->d_losortStart;
    a.losort = m->d_losort;
    a.ownerLo = m->d_ownerLo;
    a.neighbour = m->d_neighbour;
    a.owner = m->d_owner;
    a.ifStart = m->n_iface ? m->d_ifStart : nullptr;
    a.ifIdx = m->d_ifIdx;
    a.ifMask = m->n_iface ? m->d_ifMask : nullptr;
    a.n_iface = m->n_iface;
    a.sell_meta = reinterpret_cast<const int4*>(m->d_sell_meta);
    a.sell_n = m->d_sell_n;
    a.sell_o = m->d_sell_o;
    a.ell_wn = m->sell_wn;
    a.ell_wo = m->sell_wo;
    a.upper_s = m->d_upper_s;
    a.cmeta = m->ell_stencil ? m->d_cmeta : nullptr;
    a.clane = m->ell_stencil ? m->d_clane : nullptr;
    a.lat_K = m->d_upper_d ? m->lat_K : 0;
    for (int t = 0; t < 3; ++t) a.lat_D[t] = m->lat_D[t];
    a.lat_S = m->lat_S;
    a.upper_d = m->d_upper_d;
    return a;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// the loop runs while (n < max_iter && !converged) || n < min_iter (reading Q3): min_iter may
// exceed max_iter, so the host-side termination guards are bounded by the larger of the two
static int iter_bound(const spuma_solver_controls* c) { return std::max(c->max_iter, c->min_iter); }

// Peer transport (peer.cu): a poll that exceeds its limit sets the handle's error word and the
// kernels then skip the stale exchange -- every collective call reads (and clears) that word
// after its work, so such a call returns SPUMA_ERR_STATE instead of SPUMA_OK with wrong results.
spuma_status peer_guard(spuma_mesh m)
{
    if (!m->peer || !m->pst.err) return SPUMA_OK;
    int e = 0;
    SPUMA_CUDA(cudaMemcpyAsync(&e, m->pst.err, sizeof e, cudaMemcpyDeviceToHost, m->stream));
    SPUMA_CUDA(cudaStreamSynchronize(m->stream));
    if (!e) return SPUMA_OK;
    SPUMA_CUDA(cudaMemsetAsync(m->pst.err, 0, sizeof(int), m->stream));
    SPUMA_CUDA(cudaStreamSynchronize(m->stream));
    return set_error(SPUMA_ERR_STATE, "peer transport: a neighbour did not answer within the poll limit");
}

enum CellRole { R_GAMMA = 0, R_DIAG, R_SOURCE, R_PSI, R_X, R_Y, R_COUNT };

double** cell_buf(spuma_mesh m, int role)
{
    double** bufs[R_COUNT] = {&m->d_cell_a, &m->d_cell_b, &m->d_cell_c, &m->d_cell_d, &m->d_cell_e, &m->d_cell_t};
    return bufs[role];
}

// caller cell array -> device array in internal numbering
// (the vector kernels access cell arrays as double2: a caller device array that is only 8-byte
// aligned -- e.g. a torch slice at an odd offset -- is staged through the handle's buffer)
spuma_status cells_in(spuma_mesh m, const double* p, int role, const double** out)
{
    const bool dev = is_device_ptr(p);
    if (!m->renumber && dev && aligned16(p)) {
        *out = p;
        return SPUMA_OK;
    }
    double** buf = cell_buf(m, role);
    if (!*buf) SPUMA_TRY(dalloc(buf, m->N));
    if (!m->renumber) {
        SPUMA_CUDA(cudaMemcpyAsync(*buf, p, sizeof(double) * m->N, cudaMemcpyDefault, m->stream));
    } else {
        const double* src = p;
        if (!dev) {
            if (!m->d_face_t) SPUMA_TRY(dalloc(&m->d_face_t, std::max(m->F, m->N)));
            SPUMA_CUDA(cudaMemcpyAsync(m->d_face_t, p, sizeof(double) * m->N, cudaMemcpyHostToDevice, m->stream));
            src = m->d_face_t;
        }
        launch_scatter(m->stream, m->N, m->d_perm, src, *buf);  // buf[perm[i]] = p[i]
    }
    *out = *buf;
    return SPUMA_OK;
}

// internal device array -> caller cell array
spuma_status cells_out(spuma_mesh m, double* p, const double* buf)
{
    if (buf == p) return SPUMA_OK;
    if (!m->renumber) {
        SPUMA_CUDA(cudaMemcpyAsync(p, buf, sizeof(double) * m->N, cudaMemcpyDefault, m->stream));
        return SPUMA_OK;
    }
    if (!m->d_face_t) SPUMA_TRY(dalloc(&m->d_face_t, std::max(m->F, m->N)));
    launch_gather(m->stream, m->N, m->d_perm, buf, m->d_face_t);  // t[i] = buf[perm[i]]
    SPUMA_CUDA(cudaMemcpyAsync(p, m->d_face_t, sizeof(double) * m->N, cudaMemcpyDefault, m->stream));
    return SPUMA_OK;
}

spuma_status faces_in(spuma_mesh m, const double* p, const double** out)
{
    const bool dev = is_device_ptr(p);
    if (!m->renumber && dev) {
        *out = p;
        return SPUMA_OK;
    }
    if (!m->d_face_a) SPUMA_TRY(dalloc(&m->d_face_a, m->F));
    if (!m->renumber) {
        SPUMA_CUDA(cudaMemcpyAsync(m->d_face_a, p, sizeof(double) * m->F, cudaMemcpyHostToDevice, m->stream));
    } else {
        const double* src = p;
        if (!dev) {
            if (!m->d_face_t) SPUMA_TRY(dalloc(&m->d_face_t, std::max(m->F, m->N)));
            SPUMA_CUDA(cudaMemcpyAsync(m->d_face_t, p, sizeof(double) * m->F, cudaMemcpyHostToDevice, m->stream));
            src = m->d_face_t;
        }
        launch_gather(m->stream, m->F, m->d_face_map, src, m->d_face_a);  // a[new] = p[face_map[new]]
    }
    *out = m->d_face_a;
    return SPUMA_OK;
}

spuma_status faces_out(spuma_mesh m, double* p, const double* buf)
{
    if (buf == p) return SPUMA_OK;
    if (!m->renumber) {
        SPUMA_CUDA(cudaMemcpyAsync(p, buf, sizeof(double) * m->F, cudaMemcpyDefault, m->stream));
        return SPUMA_OK;
    }
    if (!m->d_face_t) SPUMA_TRY(dalloc(&m->d_face_t, std::max(m->F, m->N)));
    launch_scatter(m->stream, m->F, m->d_face_map, buf, m->d_face_t);  // t[face_map[new]] = buf[new]
    SPUMA_CUDA(cudaMemcpyAsync(p, m->d_face_t, sizeof(double) * m->F, cudaMemcpyDefault, m->stream));
    return SPUMA_OK;
}

spuma_status iface_in(spuma_mesh m, const double* p, const double** out)
{
    if (m->n_iface == 0 || is_device_ptr(p)) {
        *out = p;
        return SPUMA_OK;
    }
    if (!m->d_iface_a) SPUMA_TRY(dalloc(&m->d_iface_a, m->n_iface));
    SPUMA_CUDA(cudaMemcpyAsync(m->d_iface_a, p, sizeof(double) * m->n_iface, cudaMemcpyHostToDevice, m->stream));
    *out = m->d_iface_a;
    return SPUMA_OK;
}

// oriented face field (e.g. a flux, owner -> neighbour) -> internal numbering/orientation
spuma_status oriented_in(spuma_mesh m, const double* p, double** buf, double** out)
{
    const bool dev = is_device_ptr(p);
    if (!m->renumber && dev) {
        *out = const_cast<double*>(p);
        return SPUMA_OK;
    }
    if (!*buf) SPUMA_TRY(dalloc(buf, m->F));
    if (!m->renumber) {
        SPUMA_CUDA(cudaMemcpyAsync(*buf, p, sizeof(double) * m->F, cudaMemcpyHostToDevice, m->stream));
    } else {
        const double* src = p;
        if (!dev) {
            if (!m->d_face_t) SPUMA_TRY(dalloc(&m->d_face_t, std::max(m->F, m->N)));
            SPUMA_CUDA(cudaMemcpyAsync(m->d_face_t, p, sizeof(double) * m->F, cudaMemcpyHostToDevice, m->stream));
            src = m->d_face_t;
        }
        launch_gather_signed(m->stream, m->F, m->d_face_map, m->d_face_flip, src, *buf);
    }
    *out = *buf;
    return SPUMA_OK;
}

spuma_status oriented_out(spuma_mesh m, double* p, const double* buf)
{
    if (buf == p) return SPUMA_OK;
    if (!m->renumber) {
        SPUMA_CUDA(cudaMemcpyAsync(p, buf, sizeof(double) * m->F, cudaMemcpyDefault, m->stream));
        return SPUMA_OK;
    }
    if (!m->d_face_t) SPUMA_TRY(dalloc(&m->d_face_t, std::max(m->F, m->N)));
    launch_scatter_signed(m->stream, m->F, m->d_face_map, m->d_face_flip, buf, m->d_face_t);
    SPUMA_CUDA(cudaMemcpyAsync(p, m->d_face_t, sizeof(double) * m->F, cudaMemcpyDefault, m->stream));
    return SPUMA_OK;
}

// per-patch face values (array of per-patch pointers, NULL entries = 0) -> concatenated device buffer
spuma_status patches_in(spuma_mesh m, const double* const* pv, double* dst, bool skip_empty_kinds)
{
    SPUMA_CUDA(cudaMemsetAsync(dst, 0, sizeof(double) * std::max(m->Fb, 1), m->stream));
    if (!pv) return SPUMA_OK;
    for (size_t p = 0; p < m->patches.size(); ++p) {
        const Patch& P = m->patches[p];
        if (!pv[p] || P.n_faces == 0 || (skip_empty_kinds && P.kind == SPUMA_PATCH_EMPTY)) continue;
        SPUMA_CUDA(cudaMemcpyAsync(dst + P.offset, pv[p], sizeof(double) * P.n_faces, cudaMemcpyDefault, m->stream));
    }
    return SPUMA_OK;
}

spuma_status patches_out(spuma_mesh m, double* const* pv, const double* src)
{
    if (!pv) return SPUMA_OK;
    for (size_t p = 0; p < m->patches.size(); ++p) {
        const Patch& P = m->patches[p];
        if (!pv[p] || P.n_faces == 0) continue;
        SPUMA_CUDA(cudaMemcpyAsync(pv[p], src + P.offset, sizeof(double) * P.n_faces, cudaMemcpyDefault, m->stream));
    }
    return SPUMA_OK;
}

// ---------------------------------------------------------------------------
// halo exchange over NCCL (processor patches)
// ---------------------------------------------------------------------------

spuma_status halo_exchange(spuma_mesh m, const double* x, double* xr, cudaStream_t s)
{
    if (m->peer) {  // pack fused into the peer stores (peer.cu)
        if (m->px.n_patches == 0) return SPUMA_OK;
        PeerXfer d = m->px;
        for (int p = 0; p < d.n_patches; ++p) d.off[p] = m->cb_offsets[p], d.count[p] = m->cb_counts[p];
        launch_peer_exchange(s, d, x, m->d_if_cell, xr, m->pst);
        m->stats.kernel_launches += 2;
        return SPUMA_OK;
    }
    if (m->n_ranks == 1) return SPUMA_OK;
    if (m->external_comm) {
        if (!m->cb.exchange) return set_error(SPUMA_ERR_STATE, "external comm: callbacks not set");
        if (m->n_iface) {
            launch_pack(s, m->n_iface, m->d_if_cell, x, m->d_sendbuf);
            m->stats.kernel_launches += 1;
            SPUMA_CUDA(cudaMemcpyAsync(m->h_send, m->d_sendbuf, sizeof(double) * m->n_iface, cudaMemcpyDeviceToHost, s));
        }
        SPUMA_CUDA(cudaStreamSynchronize(s));
        if (m->cb.exchange(m->cb.ctx, (int)m->cb_peers.size(), m->cb_peers.data(), m->cb_offsets.data(),
                           m->cb_counts.data(), m->h_send, m->h_recv) != 0)
            return set_error(SPUMA_ERR_NCCL, "external comm: exchange callback failed");
        if (m->n_iface)
            SPUMA_CUDA(cudaMemcpyAsync(xr, m->h_recv, sizeof(double) * m->n_iface, cudaMemcpyHostToDevice, s));
        return SPUMA_OK;
    }
    if (m->n_iface == 0) return SPUMA_OK;
    launch_pack(s, m->n_iface, m->d_if_cell, x, m->d_sendbuf);
    m->stats.kernel_launches += 1;
    SPUMA_NCCL(ncclGroupStart());
    for (const auto& p : m->patches) {
        if (p.kind != SPUMA_PATCH_PROCESSOR || p.n_faces == 0) continue;
        SPUMA_NCCL(ncclSend(m->d_sendbuf + p.iface_offset, p.n_faces, ncclDouble, p.neighbour_rank, m->comm, s));
        SPUMA_NCCL(ncclRecv(xr + p.iface_offset, p.n_faces, ncclDouble, p.neighbour_rank, m->comm, s));
    }
    SPUMA_NCCL(ncclGroupEnd());
    return SPUMA_OK;
}

// NCCL communicator health, polled when an iteration batch ends (SURVEY §5 failure detection):
// an asynchronous NCCL error (a peer died, a network failure) surfaces as SPUMA_ERR_NCCL
spuma_status nccl_async_check(spuma_mesh m)
{
    if (!m->comm) return SPUMA_OK;
    ncclResult_t r = ncclSuccess;
    SPUMA_NCCL(ncclCommGetAsyncError(m->comm, &r));
    if (r != ncclSuccess && r != ncclInProgress)
        return set_error(SPUMA_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(r));
    return SPUMA_OK;
}

// all ranks' 4 partials (device, [4]) into out ([4 * n_ranks], rank order) on stream s
spuma_status allgather4(spuma_mesh m, const double* in, double* out, cudaStream_t s)
{
    if (m->peer) {
        launch_peer_allgather4(s, m->pg, in, out, m->pst);
        m->stats.kernel_launches += 1;
        return SPUMA_OK;
    }
    if (m->external_comm) {
        if (!m->cb.allgather) return set_error(SPUMA_ERR_STATE, "external comm: callbacks not set");
        SPUMA_CUDA(cudaMemcpyAsync(m->h_part, in, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
        SPUMA_CUDA(cudaStreamSynchronize(s));
        if (m->cb.allgather(m->cb.ctx, m->h_part, m->h_part + 4, 4) != 0)
            return set_error(SPUMA_ERR_NCCL, "external comm: allgather callback failed");
        SPUMA_CUDA(cudaMemcpyAsync(out, m->h_part + 4, 4 * sizeof(double) * m->n_ranks, cudaMemcpyHostToDevice, s));
        return SPUMA_OK;
    }
    SPUMA_NCCL(ncclAllGather(in, out, 4, ncclDouble, m->comm, s));
    return SPUMA_OK;
}

// every rank gets all ranks' 4 partials (rank order) and finalises identically
spuma_status reduce_finalize_ws(spuma_mesh m, const Workspace& w, int stage, cudaStream_t s)
{
    double* gathered = w.part;  // free after the reduction kernel finished
    if (m->peer) {  // the all-gather kernel finalises too
        launch_peer_allgather4(s, m->pg, w.scal->rank_part, gathered, m->pst, stage, &w);
        m->stats.kernel_launches += 1;
        return SPUMA_OK;
    }
    SPUMA_TRY(allgather4(m, w.scal->rank_part, gathered, s));
    launch_finalize(s, stage, gathered, m->n_ranks, w);
    m->stats.kernel_launches += 1;
    return SPUMA_OK;
}

spuma_status reduce_finalize(spuma_mesh m, int stage, cudaStream_t s) { return reduce_finalize_ws(m, m->ws, stage, s); }

// processor-patch exchange of a level's interface values (device buffers; per-patch counts of
// the level, peers and order of level 0's patches): recv[offset_p ..) <- the neighbour's send
spuma_status exchange_counts(spuma_mesh m, const std::vector<int>& counts, const double* send, double* recv,
                             cudaStream_t s)
{
    int n = 0;
    std::vector<int> offsets(counts.size());
    for (size_t p = 0; p < counts.size(); ++p) offsets[p] = n, n += counts[p];
    if (m->peer) {  // each patch's data lands in the receiver's level-0 region of that patch
        if (m->px.n_patches == 0) return SPUMA_OK;
        PeerXfer d = m->px;
        for (int p = 0; p < d.n_patches; ++p) d.off[p] = offsets[p], d.count[p] = counts[p];
        launch_peer_exchange(s, d, send, nullptr, recv, m->pst);
        m->stats.kernel_launches += 2;
        return SPUMA_OK;
    }
    if (m->external_comm) {
        if (!m->cb.exchange) return set_error(SPUMA_ERR_STATE, "external comm: callbacks not set");
        std::vector<double> hs(n + 1), hr(n + 1);
        if (n) SPUMA_CUDA(cudaMemcpyAsync(hs.data(), send, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        SPUMA_CUDA(cudaStreamSynchronize(s));
        if (m->cb.exchange(m->cb.ctx, (int)counts.size(), m->cb_peers.data(), offsets.data(), counts.data(), hs.data(),
                           hr.data()) != 0)
            return set_error(SPUMA_ERR_NCCL, "external comm: exchange callback failed");
        if (n) SPUMA_CUDA(cudaMemcpyAsync(recv, hr.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
        SPUMA_CUDA(cudaStreamSynchronize(s));  // hr is a stack buffer
        return SPUMA_OK;
    }
    SPUMA_NCCL(ncclGroupStart());
    for (size_t p = 0; p < counts.size(); ++p) {
        if (counts[p] == 0) continue;
        SPUMA_NCCL(ncclSend(send + offsets[p], counts[p], ncclDouble, m->cb_peers[p], m->comm, s));
        SPUMA_NCCL(ncclRecv(recv + offsets[p], counts[p], ncclDouble, m->cb_peers[p], m->comm, s));
    }
    SPUMA_NCCL(ncclGroupEnd());
    return SPUMA_OK;
}

// timing event of a captured batch, recorded on a LEAF branch (timing stream): the event node
// depends on the work captured on s so far, nothing on s depends on it, so the programmatic
// (PDL) edges between the timed kernels are the untimed ones (an event node in line would
// serialise the next kernel's launch behind it).  "Before kernel k" = "after kernel k - 1".
void record(spuma_mesh m, std::vector<cudaEvent_t>& ev, int idx, cudaStream_t s)
{
    if (!m->tstream) {  // outside a timed capture (not expected): in line
        cudaEventRecordWithFlags(ev[idx], s, cudaEventRecordExternal);
        return;
    }
    cudaEventRecord(m->tfork, s);
    cudaStreamWaitEvent(m->tstream, m->tfork, 0);
    cudaEventRecordWithFlags(ev[idx], m->tstream, cudaEventRecordExternal);
}

// one PCG iteration (A11, A7h, A7-A8, A9-A10) on stream s.  P > 1 with processor faces
// and an ELL/SELL Amul: the halo (pack + NCCL send/recv on the comm stream) overlaps
// the Amul of every row, whose interface rows are finished by k_iface_rows once the
// halo has arrived (SURVEY §8(e) "overlapped with the interior Amul").
// the per-call coefficient copy the selected Amul layout reads (ELL owner-slot order, or the
// lattice slots of variant 12)
void prepare_amul_coeffs(spuma_mesh m, cudaStream_t s, const MeshArgs& a, const double* upper)
{
    const int rv = resolve_amul_variant(m->amul_variant, a);
    if (rv == 12 || rv == 13) {
        launch_lattice_coeffs(s, a, upper);
        m->stats.kernel_launches += 1;
    } else if (amul_uses_ell(rv) && m->d_upper_s) {
        launch_ell_coeffs(s, a, upper, m->d_upper_s);
        m->stats.kernel_launches += 1;
    }
}

spuma_status enqueue_iteration(spuma_mesh m, cudaStream_t s, std::vector<cudaEvent_t>* ev, int slot)
{
    const MeshArgs a = mesh_args(m);
    const bool fin = m->n_ranks == 1;
    // deferred psi updates: iteration k (slot parity = k parity) writes direction buffer k % 2,
    // reads the previous one, and applies psi for the pair (k-1, k) when k is odd
    Workspace ws = m->ws;
    int psi_mode = 0;
    if (m->defer_psi) {
        ws.pA = (slot & 1) ? m->ws.pA2 : m->ws.pA;
        ws.pA_prev = (slot & 1) ? m->ws.pA : m->ws.pA2;
        psi_mode = (slot & 1) ? 2 : 1;
    }
    const int rv = resolve_amul_variant(m->amul_variant, a);
    // alternating sweeps (slot parity): C asc, A desc, B asc | C desc, A asc, B desc | ...
    const bool odd = m->alt_sweep && (slot & 1);
    const bool alt = m->alt_sweep;
    const bool overlap = !fin && m->n_iface > 0 && rv >= 6 && rv <= 13;
    // SPUMA_OPT_DEFER_PSI = 2: the pairs are applied by the direction of every even iteration
    const bool psi_in_dir = m->defer_psi == 2;
    if (psi_in_dir) psi_mode = 1;
    if (fin && m->defer_psi == 1 && m->fuse_direction && rv == 8 && fused_direction_ok(a)) {
        // direction formed inside the Amul gather (one pass less per iteration)
        if (ev) record(m, *ev, slot * 6 + 0, s);
        if (ev) record(m, *ev, slot * 6 + 1, s);
        if (ev) record(m, *ev, slot * 6 + 2, s);
        launch_amul_dot_dir(s, a, ws, m->fuse_direction == 2);
        if (ev) record(m, *ev, slot * 6 + 3, s);
        if (ev) record(m, *ev, slot * 6 + 4, s);
        launch_update(s, m->grid, a, ws, fin, psi_mode);
        if (ev) record(m, *ev, slot * 6 + 5, s);
        m->stats.kernel_launches += 2;
        return SPUMA_OK;
    }
    if (overlap && m->peer && m->peer_fused && m->px.n_patches > 0) {
        // peer transport, fused: four kernels per iteration -- the direction stores the interface
        // values into the neighbours' mailboxes; the Amul's interior rows overlap the transfer;
        // the interface rows wait for the neighbours' flags, read their mailbox and all-gather the
        // rank partials of wA.pA (alpha); the update all-gathers its own (beta, convergence)
        ws.pst = m->pst;
        if (ev) record(m, *ev, slot * 6 + 0, s);
        launch_direction(s, m->grid, a, ws, odd, psi_in_dir && !(slot & 1), true);
        if (ev) record(m, *ev, slot * 6 + 1, s);
        if (ev) record(m, *ev, slot * 6 + 2, s);
        launch_amul_dot(s, m->amul_variant, a, ws, false, m->sell_wn, m->sell_wo, true);
        launch_iface_rows(s, a, ws, m->d_ifRows, m->n_ifRows, true);
        if (ev) record(m, *ev, slot * 6 + 3, s);
        if (ev) record(m, *ev, slot * 6 + 4, s);
        launch_update(s, m->grid, a, ws, 2, psi_mode, odd);
        if (ev) record(m, *ev, slot * 6 + 5, s);
        m->stats.kernel_launches += 4;
        return SPUMA_OK;
    }
    if (ev) record(m, *ev, slot * 6 + 0, s);
    launch_direction(s, m->grid, a, ws, odd, psi_in_dir && !(slot & 1));
    if (ev) record(m, *ev, slot * 6 + 1, s);
    if (overlap) {
        if (!m->external_comm) {
            SPUMA_CUDA(cudaEventRecord(m->ev_fork, s));
            SPUMA_CUDA(cudaStreamWaitEvent(m->comm_stream, m->ev_fork, 0));
            SPUMA_TRY(halo_exchange(m, ws.pA, ws.xr, m->comm_stream));
            SPUMA_CUDA(cudaEventRecord(m->ev_join, m->comm_stream));
        }
        if (ev) record(m, *ev, slot * 6 + 2, s);
        launch_amul_dot(s, m->amul_variant, a, ws, fin, m->sell_wn, m->sell_wo, true);
        if (ev) record(m, *ev, slot * 6 + 3, s);
        if (m->external_comm) SPUMA_TRY(halo_exchange(m, ws.pA, ws.xr, s));
        else SPUMA_CUDA(cudaStreamWaitEvent(s, m->ev_join, 0));
        launch_iface_rows(s, a, ws, m->d_ifRows, m->n_ifRows);
        m->stats.kernel_launches += 1;
    } else {
        SPUMA_TRY(halo_exchange(m, ws.pA, ws.xr, s));
        if (ev) record(m, *ev, slot * 6 + 2, s);
        launch_amul_dot(s, m->amul_variant, a, ws, fin, m->sell_wn, m->sell_wo, false, alt && !odd);
        if (ev) record(m, *ev, slot * 6 + 3, s);
    }
    if (!fin) SPUMA_TRY(reduce_finalize(m, 3, s));
    if (ev) record(m, *ev, slot * 6 + 4, s);
    launch_update(s, m->grid, a, ws, fin, psi_mode, odd);
    if (ev) record(m, *ev, slot * 6 + 5, s);
    if (!fin) SPUMA_TRY(reduce_finalize(m, 4, s));
    m->stats.kernel_launches += 3;
    return SPUMA_OK;
}

// iterations per captured batch: even when psi updates are deferred (pairs must not straddle batches)
int batch_eff(spuma_mesh m) { return m->batch + ((m->defer_psi && (m->batch & 1)) ? 1 : 0); }

void destroy_graphs(spuma_mesh m)
{
    for (int i = 0; i < 2; ++i) {
        if (m->gexec[i]) cudaGraphExecDestroy(m->gexec[i]);
        m->gexec[i] = nullptr;
        for (auto e : m->tev[i]) cudaEventDestroy(e);
        m->tev[i].clear();
    }
}

// An L2 access-policy window (persisting hits, streaming misses) over one workspace vector
// (1 pA, 2 rA, 3 rD, 4 wA), with the device-wide persisting-L2 limit raised to cover it.  The lines
// another target left persisting are released first (they would hold the set-aside otherwise).
// *use = false when the vector does not fit the persisting set-aside (a partly persisting window
// over a larger vector thrashes: 252^3 graph batches 314 -> 379 us per iteration, C4 64M 1525 ->
// 2378 us, profiles/r02x2_*): no window then.
spuma_status l2_policy(spuma_mesh m, int target, cudaAccessPolicyWindow* out, bool* use)
{
    int dev = 0, maxp = 0, maxw = 0;
    SPUMA_CUDA(cudaGetDevice(&dev));
    SPUMA_CUDA(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
    SPUMA_CUDA(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    const size_t win = std::min((size_t)maxw, sizeof(double) * (size_t)m->N);
    *use = win <= (size_t)maxp && sizeof(double) * (size_t)m->N <= (size_t)maxw;
    if (!*use) {
        if (m->l2_lines) {
            SPUMA_CUDA(cudaCtxResetPersistingL2Cache());
            m->l2_lines = nullptr;
        }
        return SPUMA_OK;
    }
    SPUMA_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min((size_t)maxp, win)));
    m->l2_limit_set = true;
    double* const tg[5] = {nullptr, m->ws.pA, m->ws.rA, m->ws.rD, m->ws.wA};
    if (m->l2_lines != tg[target]) {
        SPUMA_CUDA(cudaCtxResetPersistingL2Cache());
        m->l2_lines = tg[target];
    }
    *out = cudaAccessPolicyWindow{};
    out->base_ptr = tg[target];
    out->num_bytes = win;
    out->hitRatio = (float)std::min(1.0, (double)maxp / (double)win);
    out->hitProp = cudaAccessPropertyPersisting;
    out->missProp = cudaAccessPropertyStreaming;
    return SPUMA_OK;
}

// SPUMA_OPT_L2_PERSIST: the window captured into the iteration graphs' kernel nodes; 0 = none.
// The window is set on the stream only for the duration of the capture (the kernel nodes keep
// it); the stream's previous policy -- it may be the caller's stream -- is restored afterwards.
spuma_status l2_window(spuma_mesh m, cudaStreamAttrValue* saved)
{
    cudaStreamAttrValue v{};
    if (!m->l2_persist || m->N == 0) return SPUMA_OK;
    SPUMA_CUDA(cudaStreamGetAttribute(m->stream, cudaStreamAttributeAccessPolicyWindow, saved));
    bool use = false;
    SPUMA_TRY(l2_policy(m, m->l2_persist, &v.accessPolicyWindow, &use));
    if (!use) v.accessPolicyWindow = cudaAccessPolicyWindow{};  // num_bytes 0: no window on the captured nodes
    SPUMA_CUDA(cudaStreamSetAttribute(m->stream, cudaStreamAttributeAccessPolicyWindow, &v));
    return SPUMA_OK;
}

// undo SPUMA_OPT_L2_PERSIST's device-wide state: the persisting-L2 limit and the lines
// already marked persisting
void l2_reset(spuma_mesh m)
{
    if (!m->l2_limit_set) return;
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
    cudaCtxResetPersistingL2Cache();
    m->l2_lines = nullptr;
    m->l2_limit_set = false;
}

constexpr int kTimedSlots = 2;  // iterations per batch carrying timing events (spuma_set_timing)

spuma_status build_graphs(spuma_mesh m)
{
    if (m->gexec[0] && m->gexec_timed == m->timing && m->gexec_batch == batch_eff(m)) return SPUMA_OK;
    destroy_graphs(m);
    const uint64_t launches_before = m->stats.kernel_launches;
    for (int g = 0; g < 2; ++g) {
        std::vector<cudaEvent_t>* ev = nullptr;
        if (m->timing) {
            m->tev[g].resize(6 * kTimedSlots);
            for (auto& e : m->tev[g]) SPUMA_CUDA(cudaEventCreate(&e));
            ev = &m->tev[g];
        }
        cudaGraph_t graph = nullptr;
        cudaStreamAttrValue saved{};
        SPUMA_TRY(l2_window(m, &saved));
        if (m->timing && !m->tstream) {
            SPUMA_CUDA(cudaStreamCreateWithFlags(&m->tstream, cudaStreamNonBlocking));
            SPUMA_CUDA(cudaEventCreateWithFlags(&m->tfork, cudaEventDisableTiming));
        }
        SPUMA_CUDA(cudaStreamBeginCapture(m->stream, cudaStreamCaptureModeThreadLocal));
        spuma_status st = SPUMA_OK;
        // timing samples the first two iterations of every batch -- one even, one odd, so both
        // halves of the deferred-psi pattern are in the averages (6 event nodes per timed
        // iteration on a leaf branch; ~200 samples per 1600-iteration solve)
        for (int k = 0; k < batch_eff(m) && st == SPUMA_OK; ++k)
            st = enqueue_iteration(m, m->stream, k < kTimedSlots ? ev : nullptr, k);
        if (m->timing) {  // the timing branch rejoins the origin stream at the end of the batch
            cudaEventRecord(m->tfork, m->tstream);
            cudaStreamWaitEvent(m->stream, m->tfork, 0);
        }
        cudaError_t e = cudaStreamEndCapture(m->stream, &graph);
        if (m->l2_persist && m->N > 0) cudaStreamSetAttribute(m->stream, cudaStreamAttributeAccessPolicyWindow, &saved);
        if (st != SPUMA_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        SPUMA_CUDA(e);
        e = cudaGraphInstantiate(&m->gexec[g], graph, 0);
        cudaGraphDestroy(graph);
        SPUMA_CUDA(e);
    }
    m->stats.kernel_launches = launches_before;  // capture launches nothing
    m->gexec_timed = m->timing;
    m->gexec_batch = batch_eff(m);
    return SPUMA_OK;
}

// every timed iteration of a batch that ran (slot < executed) contributes one sample per phase
spuma_status account_timing(spuma_mesh m, int g, int executed)
{
    static const int from[3] = {0, 2, 4};
    for (int k = 0; k < kTimedSlots && k < executed && 6 * k + 5 < (int)m->tev[g].size(); ++k)
        for (int ph = 0; ph < 3; ++ph) {
            float ms = 0.f;
            SPUMA_CUDA(cudaEventElapsedTime(&ms, m->tev[g][6 * k + from[ph]], m->tev[g][6 * k + from[ph] + 1]));
            m->stats.phase_ms[ph] += ms;
            m->stats.phase_count[ph] += 1;
        }
    return SPUMA_OK;
}


// ---------------------------------------------------------------------------
// GAMG: hierarchy on the device, per-solve Galerkin products, one
// captured V-cycle + residual per iteration (kernels in gamg.cu)
// ---------------------------------------------------------------------------
}  // namespace

struct GamgState {
    int n_coarsest = -1, max_levels = -1;            // key of the hierarchy
    std::vector<spuma::GLevel> lv;
    std::vector<int> cells, faces;
    std::vector<std::vector<int>> ftc;               // host copies (diagnostics)
    std::vector<void*> allocs;
    double *alpha = nullptr, *part = nullptr;        // per-level scale factors, reduction partials
    unsigned* ticket = nullptr;
    spuma::Workspace cws{};                          // coarsest-level PCG
    spuma::DevPtrs* h_cptrs = nullptr;               // pinned
    cudaGraphExec_t gexec = nullptr;
    spuma_gamg_params gkey{};
    int gkey_tail = -1;                              // tail threshold the graph was captured with
    int launches_per_cycle = 0;
    spuma::GLevel* d_lv = nullptr;                   // device copy of lv (the single-CTA tail reads it)
    // n_ranks > 1 (readings Q36-Q38): per-level per-patch interface counts, this rank's
    // reduction partials and the gathered ones
    std::vector<std::vector<int>> if_count;
    double *rank_part = nullptr, *gathered = nullptr;
    bool dd = false;
};

namespace {

// SPUMA_OPT_PERSISTENT: can this solve run as one cooperative launch (loop.cu)?
// layout of the loop's Amul: 1 lattice slots, 2 ELL rows, 3 SELL-C rows, 0 = not eligible
int loop_layout(spuma_mesh m, const MeshArgs& a)
{
    if (!(m->persistent > 0 && m->n_ranks == 1 && !m->external_comm && m->defer_psi == 2 && m->N > 0)) return 0;
    const int rv = resolve_amul_variant(m->amul_variant, a);
    if ((rv == 12 || rv == 13) && a.lat_K >= 1 && a.lat_K <= 3) return 1;
    if ((rv == 8 || rv == 10) && a.upper_s && !m->ell_stencil && a.ell_wn >= 0 && a.ell_wn <= 3 && a.ell_wo >= 0 &&
        a.ell_wo <= 3)
        return 2;
    if (rv == 6 && a.sell_n) return 3;
    return 0;
}

// A7-A11 of the whole solve in one cooperative launch after the A6 setup; *ran = false when the
// device cannot host it (the caller then runs the graph batches)
spuma_status run_pcg_loop(spuma_mesh m, cudaStream_t s, const MeshArgs& a, int layout, bool* ran)
{
    *ran = false;
    const int kkey = layout == 3 ? -1 : (layout == 2 ? 0 : a.lat_K);  // loop_fn key: lattice K, 0 ELL, -1 SELL
    const int T = loop_threads();
    if (!m->loop_grid) {
        int dev = 0, sms = 0;
        SPUMA_CUDA(cudaGetDevice(&dev));
        SPUMA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        SPUMA_TRY(dalloc(&m->d_loop_bar, 2));
        SPUMA_TRY(dalloc(&m->d_loop_part, (size_t)3 * sms));
        for (int i = 0; i < 2; ++i) SPUMA_CUDA(cudaEventCreate(&m->loop_ev[i]));
        m->loop_grid = sms;
    }
    // CTAs (SPUMA_OPT_LOOP_GRID): explicit, or 32 per started 16384 cells up to one per SM -- a
    // few thousand cells run faster on fewer CTAs (8000 cells: 9.0 us per iteration on 32 CTAs,
    // 11.0 on 148; 64000: 148 best; profiles/r02at_loop_grid_ab.jsonl)
    const int G_auto = (int)std::min<long long>(m->loop_grid, 32LL * (((long long)m->N + 16383) / 16384));
    const int G = m->loop_ctas > 0 ? std::min(m->loop_ctas, m->loop_grid) : std::max(1, G_auto);
    // rA pairs per thread: the CTA's tiles of T pairs, grid-strided
    const long long np = m->N / 2, ntile = (np + T - 1) / T;
    const int need = (int)((ntile + G - 1) / G);
    int tp = m->persistent >= 3 ? std::min(need, loop_tmem_pairs()) : 0;
    // <= 186 KB of shared memory: the rest of the SM's 256 KB stays L1 for the Amul's pA windows
    // (896 threads with 14 pairs = 201 KB: 252^3 413 vs 303 us per iteration, profiles/r02av_*)
    const int sp_cap = (186 * 1024) / (T * (int)sizeof(double2));
    int sp = m->persistent >= 2 ? std::min(need - tp, sp_cap) : 0;
    // less than half of rA on chip: the graph batches are as fast or faster (C4 64M cells, 13 % on
    // chip: 1695 vs 1571 us per iteration; 252^3, 52 %: loop 312 vs 321 us, profiles/r02y_*)
    if (m->persistent >= 2 && 2 * (tp + sp) < need) return SPUMA_OK;
    size_t smem = (size_t)sp * T * sizeof(double2);
    if (loop_occupancy(kkey, smem) < 1) {
        if (loop_occupancy(kkey, 0) < 1) return SPUMA_OK;  // cannot run here: graph batches
        sp = 0;
        smem = 0;
    }
    LoopArgs L{};
    L.bar = m->d_loop_bar;
    L.tmem_pairs = tp;
    L.smem_pairs = sp;
    L.alt = m->alt_sweep ? 1 : 0;
    L.spin_limit = m->pst.poll_cycles;  // SPUMA_OPT_PEER_POLL_MS (default ~20 s): only a bug waits that long
    Workspace w = m->ws;
    w.part = m->d_loop_part;
    if (m->loop_profile) {
        if (!m->d_loop_prof) SPUMA_TRY(dalloc(&m->d_loop_prof, (size_t)8 * m->loop_grid));  // G <= SMs
        SPUMA_CUDA(cudaMemsetAsync(m->d_loop_prof, 0, sizeof(unsigned long long) * 8 * G, s));
        L.prof = m->d_loop_prof;
    }
    SPUMA_CUDA(cudaMemsetAsync(m->d_loop_bar, 0, 2 * sizeof(unsigned long long), s));
    if (m->timing) SPUMA_CUDA(cudaEventRecord(m->loop_ev[0], s));
    cudaAccessPolicyWindow win{};
    bool use_win = false;
    if (m->loop_l2) {
        SPUMA_TRY(l2_policy(m, m->loop_l2, &win, &use_win));
    } else if (m->l2_lines) {  // lines a graph window left persisting would hold the set-aside
        SPUMA_CUDA(cudaCtxResetPersistingL2Cache());
        m->l2_lines = nullptr;
    }
    {
        const cudaError_t e = launch_pcg_loop(s, G, smem, a, w, L, use_win ? &win : nullptr, layout);
        if (e == cudaErrorCooperativeLaunchTooLarge) {  // SMs taken (e.g. MPS limits): graph batches instead
            cudaGetLastError();
            return SPUMA_OK;
        }
        SPUMA_CUDA(e);
    }
    if (m->timing) SPUMA_CUDA(cudaEventRecord(m->loop_ev[1], s));
    m->stats.kernel_launches += 1;
    unsigned long long abort_word = 0;
    SPUMA_CUDA(cudaMemcpyAsync(&abort_word, m->d_loop_bar + 1, sizeof(abort_word), cudaMemcpyDeviceToHost, s));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    if (m->timing) {
        float ms = 0.f;
        SPUMA_CUDA(cudaEventElapsedTime(&ms, m->loop_ev[0], m->loop_ev[1]));
        m->stats.loop_ms += ms;
        m->stats.loop_count += 1;
    }
    if (m->loop_profile) {
        std::vector<unsigned long long> pr((size_t)8 * G);
        SPUMA_CUDA(cudaMemcpy(pr.data(), m->d_loop_prof, sizeof(unsigned long long) * pr.size(), cudaMemcpyDeviceToHost));
        for (int ph = 0; ph < 3; ++ph) {
            double wsum = 0, tsum = 0, wmax = 0;
            for (int bb = 0; bb < G; ++bb) {
                wsum += (double)pr[(size_t)bb * 8 + 2 * ph];
                tsum += (double)pr[(size_t)bb * 8 + 2 * ph + 1];
                wmax = std::max(wmax, (double)pr[(size_t)bb * 8 + 2 * ph]);
            }
            m->stats.loop_work_ms[ph] += wsum / G * 1e-6;
            m->stats.loop_wait_ms[ph] += tsum / G * 1e-6;
            m->stats.loop_work_max_ms[ph] += wmax * 1e-6;
        }
    }
    m->stats.loop_mode = m->persistent;
    m->stats.loop_threads = T;
    m->stats.loop_grid = G;
    m->stats.loop_tmem_pairs = tp;
    m->stats.loop_smem_pairs = sp;
    if (abort_word) return set_error(SPUMA_ERR_STATE, "persistent PCG loop: grid barrier timed out");
    *ran = true;
    return SPUMA_OK;
}

void gamg_release(spuma_mesh m)
{
    GamgState* G = m->gamg;
    if (!G) return;
    if (m->stream) cudaStreamSynchronize(m->stream);
    if (G->gexec) cudaGraphExecDestroy(G->gexec);
    for (void* p : G->allocs)
        if (p) cudaFree(p);
    if (G->h_cptrs) cudaFreeHost(G->h_cptrs);
    delete G;
    m->gamg = nullptr;
}

template <class T>
spuma_status galloc(GamgState* G, T** p, size_t n)
{
    SPUMA_TRY(dalloc(p, n));
    G->allocs.push_back(*p);
    return SPUMA_OK;
}

template <class T>
spuma_status gupload(GamgState* G, T** p, const std::vector<T>& v, cudaStream_t s)
{
    SPUMA_TRY(upload(p, v, s));
    G->allocs.push_back(*p);
    return SPUMA_OK;
}

// host collectives of the decomposed hierarchy build (GamgComm, gamg_host.cpp)
bool host_allgather4(void* ctx, const double* in, double* out)
{
    spuma_mesh m = static_cast<spuma_mesh>(ctx);
    if (m->external_comm) return m->cb.allgather && m->cb.allgather(m->cb.ctx, in, out, 4) == 0;
    double* d = nullptr;
    if (cudaMalloc(reinterpret_cast<void**>(&d), sizeof(double) * 4 * (m->n_ranks + 1)) != cudaSuccess) return false;
    bool ok = cudaMemcpy(d, in, 4 * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess &&
              allgather4(m, d, d + 4, m->stream) == SPUMA_OK &&
              cudaMemcpyAsync(out, d + 4, 4 * sizeof(double) * m->n_ranks, cudaMemcpyDeviceToHost, m->stream) ==
                  cudaSuccess &&
              cudaStreamSynchronize(m->stream) == cudaSuccess;
    cudaFree(d);
    return ok;
}

bool host_exchange(void* ctx, const std::vector<int>& counts, const std::vector<double>& send,
                   std::vector<double>& recv)
{
    spuma_mesh m = static_cast<spuma_mesh>(ctx);
    const size_t n = send.size();
    if (m->external_comm) {
        std::vector<int> offsets(counts.size());
        int o = 0;
        for (size_t p = 0; p < counts.size(); ++p) offsets[p] = o, o += counts[p];
        std::vector<double> hs(send), hr(n + 1);
        hs.push_back(0.0);
        if (!m->cb.exchange ||
            m->cb.exchange(m->cb.ctx, (int)counts.size(), m->cb_peers.data(), offsets.data(), counts.data(), hs.data(),
                           hr.data()) != 0)
            return false;
        recv.assign(hr.begin(), hr.begin() + n);
        return true;
    }
    double* d = nullptr;
    if (cudaMalloc(reinterpret_cast<void**>(&d), sizeof(double) * (2 * n + 1)) != cudaSuccess) return false;
    bool ok = (n == 0 || cudaMemcpy(d, send.data(), sizeof(double) * n, cudaMemcpyHostToDevice) == cudaSuccess) &&
              exchange_counts(m, counts, d, d + n, m->stream) == SPUMA_OK &&
              (n == 0 || cudaMemcpyAsync(recv.data(), d + n, sizeof(double) * n, cudaMemcpyDeviceToHost, m->stream) ==
                             cudaSuccess) &&
              cudaStreamSynchronize(m->stream) == cudaSuccess;
    cudaFree(d);
    return ok;
}

spuma_status gamg_ensure(spuma_mesh m, const spuma_gamg_params& gp)
{
    if (m->gamg && m->gamg->n_coarsest == gp.n_cells_in_coarsest_level && m->gamg->max_levels == gp.max_levels)
        return SPUMA_OK;
    gamg_release(m);
    cudaStream_t s = m->stream;
    std::vector<double> w(m->F);
    if (m->F) SPUMA_CUDA(cudaMemcpy(w.data(), m->d_magSf, sizeof(double) * m->F, cudaMemcpyDeviceToHost));
    std::vector<int> ownerLo(m->F);
    for (int k = 0; k < m->F; ++k) ownerLo[k] = m->h_owner[m->h_losort[k]];
    const bool dd = m->n_ranks > 1;
    std::vector<GamgHostLevel> H;
    if (dd) {  // decomposed hierarchy (Q36, Q37): collective over the ranks
        GamgComm comm;
        comm.n_ranks = m->n_ranks;
        comm.allgather4 = host_allgather4;
        comm.exchange = host_exchange;
        comm.ctx = m;
        bool ok = true;
        H = gamg_hierarchy_dd(m->N, m->F, m->h_owner, m->h_neighbour, m->h_ownerStart, m->h_losortStart, m->h_losort,
                              ownerLo, w, m->h_if_cell, m->cb_counts, gp.n_cells_in_coarsest_level, gp.max_levels,
                              comm, &ok);
        if (!ok) return set_error(SPUMA_ERR_NCCL, "GAMG hierarchy: collective failed");
    } else {
        H = gamg_hierarchy(m->N, m->F, m->h_owner, m->h_neighbour, m->h_ownerStart, m->h_losortStart, m->h_losort,
                           ownerLo, w, gp.n_cells_in_coarsest_level, gp.max_levels);
    }
    GamgState* G = new GamgState();
    m->gamg = G;
    G->dd = dd;
    G->n_coarsest = gp.n_cells_in_coarsest_level;
    G->max_levels = gp.max_levels;
    const int nl = (int)H.size();
    G->lv.resize(nl);
    int max_grid = 1;
    for (int l = 0; l < nl; ++l) {
        GamgHostLevel& h = H[l];
        GLevel& L = G->lv[l];
        L = GLevel{};
        const int n = h.n;
        G->cells.push_back(n);
        G->faces.push_back(h.F);
        if (l == 0) {
            L.a = mesh_args(m);
            L.a.ifStart = nullptr;
            L.a.ifMask = nullptr;
            L.a.n_iface = 0;
            L.rD = m->ws.rD;
            L.b = m->ws.rA;
            L.ell = (m->d_upper_s && m->d_sell_n && m->sell_wn >= 0 && m->sell_wn <= 3 && m->sell_wo >= 0 &&
                     m->sell_wo <= 3) ? 1 : 0;
            if (!L.ell && m->gamg_csr && m->F > 0) {  // irregular fine mesh: CSR rows, values per solve
                std::vector<int> rp(n + 1, 0), col(2 * (size_t)m->F), pu(m->F), pl(m->F);
                int k = 0;
                for (int c = 0; c < n; ++c) {
                    for (int q = m->h_losortStart[c]; q < m->h_losortStart[c + 1]; ++q) {
                        col[k] = m->h_owner[m->h_losort[q]];
                        pl[m->h_losort[q]] = k++;
                    }
                    for (int f = m->h_ownerStart[c]; f < m->h_ownerStart[c + 1]; ++f) {
                        col[k] = m->h_neighbour[f];
                        pu[f] = k++;
                    }
                    rp[c + 1] = k;
                }
                int *crp, *ccol, *cpu, *cpl;
                SPUMA_TRY(gupload(G, &crp, rp, s));
                SPUMA_TRY(gupload(G, &ccol, col, s));
                SPUMA_TRY(gupload(G, &cpu, pu, s));
                SPUMA_TRY(gupload(G, &cpl, pl, s));
                SPUMA_TRY(galloc(G, &L.cval, 2 * (size_t)m->F));
                L.crp = crp;
                L.ccol = ccol;
                L.cposU = cpu;
                L.cposL = cpl;
            }
        } else {
            L.a = MeshArgs{};
            L.a.N = n;
            L.a.F = h.F;
            int *os, *ls, *lo, *olo, *nb, *ow;
            SPUMA_TRY(gupload(G, &os, h.ownerStart, s));
            SPUMA_TRY(gupload(G, &ls, h.losortStart, s));
            SPUMA_TRY(gupload(G, &lo, h.losort, s));
            SPUMA_TRY(gupload(G, &olo, h.ownerLo, s));
            SPUMA_TRY(gupload(G, &nb, h.neighbour, s));
            SPUMA_TRY(gupload(G, &ow, h.owner, s));
            L.a.ownerStart = os;
            L.a.losortStart = ls;
            L.a.losort = lo;
            L.a.ownerLo = olo;
            L.a.neighbour = nb;
            L.a.owner = ow;
            SPUMA_TRY(galloc(G, &L.diag, n));
            SPUMA_TRY(galloc(G, &L.upper, h.F));
            SPUMA_TRY(galloc(G, &L.b, n));
            // coarse levels of hex meshes stay structured: rows over ELL when the widths are
            // uniform (<= 3 per side); k_gamg_agg then also writes the owner-slot coefficients
            const SellHost sh = build_sell(n, h.ownerStart, h.losortStart, h.losort, h.ownerLo, h.neighbour);
            if (sh.ok && sh.uniform_wn >= 0 && sh.uniform_wn <= 3 && sh.uniform_wo >= 0 && sh.uniform_wo <= 3) {
                unsigned* sn;
                int* so;
                double* us;
                SPUMA_TRY(gupload(G, &sn, sh.nslot, s));
                SPUMA_TRY(gupload(G, &so, sh.oslot, s));
                SPUMA_TRY(galloc(G, &us, (size_t)32 * sh.uniform_wo * ((n + 31) / 32)));
                L.a.sell_n = sn;
                L.a.sell_o = so;
                L.a.upper_s = us;
                L.a.ell_wn = sh.uniform_wn;
                L.a.ell_wo = sh.uniform_wo;
                L.ell = 1;
            } else if (h.F > 0 && m->gamg_csr) {
                // generic rows as CSR runs (row_ax order: neighbour side in losort order, then owner
                // side); k_gamg_agg writes both entries of every coarse face
                std::vector<int> rp(n + 1, 0), col(2 * (size_t)h.F), pu(h.F), pl(h.F);
                int k = 0;
                for (int c = 0; c < n; ++c) {
                    for (int q = h.losortStart[c]; q < h.losortStart[c + 1]; ++q) {
                        col[k] = h.ownerLo[q];
                        pl[h.losort[q]] = k++;
                    }
                    for (int f = h.ownerStart[c]; f < h.ownerStart[c + 1]; ++f) {
                        col[k] = h.neighbour[f];
                        pu[f] = k++;
                    }
                    rp[c + 1] = k;
                }
                int *crp, *ccol, *cpu, *cpl;
                SPUMA_TRY(gupload(G, &crp, rp, s));
                SPUMA_TRY(gupload(G, &ccol, col, s));
                SPUMA_TRY(gupload(G, &cpu, pu, s));
                SPUMA_TRY(gupload(G, &cpl, pl, s));
                SPUMA_TRY(galloc(G, &L.cval, 2 * (size_t)h.F));
                L.crp = crp;
                L.ccol = ccol;
                L.cposU = cpu;
                L.cposL = cpl;
            } else if (h.F > 0) {  // generic rows: a losort-ordered coefficient copy (one dependent load less)
                std::vector<int> pos(h.F);
                for (int k = 0; k < h.F; ++k) pos[h.losort[k]] = k;
                int* lp;
                SPUMA_TRY(gupload(G, &lp, pos, s));
                SPUMA_TRY(galloc(G, &L.upperLo, h.F));
                L.losortPos = lp;
            }
        }
        SPUMA_TRY(galloc(G, &L.x, n));
        SPUMA_TRY(galloc(G, &L.x2, n));
        SPUMA_TRY(galloc(G, &L.r, n));
        SPUMA_TRY(galloc(G, &L.p, n));
        SPUMA_TRY(galloc(G, &L.q, n));
        L.grid = gamg_grid(n);
        max_grid = std::max(max_grid, L.grid);
        if (dd) {  // processor interfaces of the level (a.ifStart / a.ifIdx per cell, Q10 order)
            const int ni = (int)h.if_cell.size();
            G->if_count.push_back(h.if_count);
            L.n_if = ni;
            int *ifs, *ifi, *ifc;
            SPUMA_TRY(gupload(G, &ifs, h.ifStart, s));
            SPUMA_TRY(gupload(G, &ifi, h.ifIdx, s));
            SPUMA_TRY(gupload(G, &ifc, h.if_cell, s));
            L.a.ifStart = ifs;
            L.a.ifIdx = ifi;
            L.a.ifMask = nullptr;
            L.a.n_iface = ni;
            L.if_cell = ifc;
            SPUMA_TRY(galloc(G, &L.xr, ni));
            SPUMA_TRY(galloc(G, &L.sendbuf, ni));
            if (l > 0) {
                double* ic;
                SPUMA_TRY(galloc(G, &ic, ni));
                L.iface = ic;
            }
            if (l + 1 < nl) {
                int *cs, *cl;
                SPUMA_TRY(gupload(G, &cs, h.cifStart, s));
                SPUMA_TRY(gupload(G, &cl, h.cifList, s));
                L.cifStart = cs;
                L.cifList = cl;
                L.ncif = (int)H[l + 1].if_cell.size();
            }
        }
        if (l + 1 < nl) {
            int *ftc, *cs, *cl, *cis, *cil, *cfs, *cfl;
            SPUMA_TRY(gupload(G, &ftc, h.ftc, s));
            SPUMA_TRY(gupload(G, &cs, h.cStart, s));
            SPUMA_TRY(gupload(G, &cl, h.cList, s));
            SPUMA_TRY(gupload(G, &cis, h.ciStart, s));
            SPUMA_TRY(gupload(G, &cil, h.ciList, s));
            SPUMA_TRY(gupload(G, &cfs, h.cfStart, s));
            SPUMA_TRY(gupload(G, &cfl, h.cfList, s));
            L.ftc = ftc;
            L.cStart = cs;
            L.cList = cl;
            L.ciStart = cis;
            L.ciList = cil;
            L.cfStart = cfs;
            L.cfList = cfl;
            L.nc = H[l + 1].n;
            L.ncf = H[l + 1].F;
            G->ftc.push_back(h.ftc);
        }
        h = GamgHostLevel{};  // release host memory early
    }
    SPUMA_TRY(galloc(G, &G->d_lv, nl));
    SPUMA_CUDA(cudaMemcpyAsync(G->d_lv, G->lv.data(), sizeof(GLevel) * nl, cudaMemcpyHostToDevice, s));
    SPUMA_TRY(galloc(G, &G->alpha, nl));
    SPUMA_TRY(galloc(G, &G->part, (size_t)kMaxPartials * max_grid));
    SPUMA_TRY(galloc(G, &G->ticket, 4));
    const int nc = G->cells[nl - 1];
    Workspace& c = G->cws;
    SPUMA_TRY(galloc(G, &c.wA, nc));
    SPUMA_TRY(galloc(G, &c.rA, nc));
    SPUMA_TRY(galloc(G, &c.pA, nc));
    SPUMA_TRY(galloc(G, &c.rD, nc));
    SPUMA_TRY(galloc(G, &c.sumA, nc));
    c.pA_prev = c.pA;
    SPUMA_TRY(galloc(G, &c.part, (size_t)kMaxPartials * std::max(occupancy_grid(nc, nullptr, 0), m->n_ranks)));
    SPUMA_TRY(galloc(G, &c.scal, 1));
    if (dd) {
        c.xr = G->lv[nl - 1].xr;
        SPUMA_TRY(galloc(G, &G->rank_part, 4));
        SPUMA_TRY(galloc(G, &G->gathered, (size_t)4 * m->n_ranks));
    }
    SPUMA_TRY(galloc(G, &c.ptrs, 1));
    SPUMA_CUDA(cudaMallocHost(reinterpret_cast<void**>(&G->h_cptrs), sizeof(DevPtrs)));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    return SPUMA_OK;
}

// The coarsest level of a decomposed hierarchy (Q38): PCG + diagonal over all ranks (O8
// semantics) from x = 0 -- the main path's multi-rank kernels (setup, direction, Amul with
// inline interface terms after the halo, update) and rank-order finalisation, with the
// coarsest level's addressing and interfaces and the coarsest workspace.
spuma_status gamg_coarsest_dd(spuma_mesh m, const spuma_gamg_params& gp, cudaStream_t s, int* k)
{
    GamgState* G = m->gamg;
    GLevel& Lc = G->lv.back();
    const std::vector<int>& cnt = G->if_count.back();
    Workspace c = G->cws;
    const MeshArgs a = Lc.a;
    const spuma_solver_controls cc{gp.coarsest_tolerance, gp.coarsest_rel_tol, gp.coarsest_max_iter, 0};
    launch_scal_init(s, c, cc, m->n_ranks);
    SPUMA_CUDA(cudaMemsetAsync(Lc.x, 0, sizeof(double) * (a.N + kPad), s));
    launch_pack(s, Lc.n_if, Lc.if_cell, Lc.x, Lc.sendbuf);
    SPUMA_TRY(exchange_counts(m, cnt, Lc.sendbuf, Lc.xr, s));
    launch_setup1(s, 0, a, c, false);
    SPUMA_TRY(reduce_finalize_ws(m, c, 1, s));
    launch_setup2(s, 0, a, c, false);
    SPUMA_TRY(reduce_finalize_ws(m, c, 2, s));
    *k += 4;
    DevScal* hs = &m->h_scal[1];
    SPUMA_CUDA(cudaMemcpyAsync(hs, c.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    const int per_check = m->external_comm ? 1 : 8;  // no-op kernels past 'done' (same on every rank)
    int it = 0;
    while (!hs->done) {
        for (int b = 0; b < per_check; ++b) {
            launch_direction(s, 0, a, c);
            launch_pack(s, Lc.n_if, Lc.if_cell, c.pA, Lc.sendbuf);
            SPUMA_TRY(exchange_counts(m, cnt, Lc.sendbuf, Lc.xr, s));
            launch_amul_dot(s, 0, a, c, false, -1, -1);
            SPUMA_TRY(reduce_finalize_ws(m, c, 3, s));
            launch_update(s, 0, a, c, false, 0);
            SPUMA_TRY(reduce_finalize_ws(m, c, 4, s));
            *k += 4;
        }
        SPUMA_CUDA(cudaMemcpyAsync(hs, c.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
        SPUMA_CUDA(cudaStreamSynchronize(s));
        it += per_check;
        if (it > gp.coarsest_max_iter + 16) return set_error(SPUMA_ERR_STATE, "coarsest PCG did not terminate");
    }
    return SPUMA_OK;
}

// One V-cycle (Q23) + the outer residual (Q28), enqueued on s (captured or direct).  On a
// decomposed mesh (G->dd; direct launches only) every row kernel is preceded by the halo of the
// vector it gathers, every reduction is finished from the gathered rank partials, and the
// coarsest level is gamg_coarsest_dd (readings Q36-Q38).
int gamg_enqueue_cycle(spuma_mesh m, const spuma_gamg_params& gp, cudaStream_t s, spuma_status* st = nullptr)
{
    GamgState* G = m->gamg;
    const DevPtrs* P = m->ws.ptrs;
    const int nl = (int)G->lv.size();
    std::vector<GLevel>& lv = G->lv;
    int k = 0;
    Workspace w0 = m->ws;
    w0.part = G->part;
    const bool dd = G->dd;
    spuma_status err = SPUMA_OK;
    if (st) *st = SPUMA_OK;
    // dd: the neighbours' values of the vector the next row kernel of level L gathers
    auto halo = [&](const GLevel& L, int mode, const double* x, const double* xc, const double* alpha,
                    const double* p, const double* q) {
        if (!dd || err != SPUMA_OK) return;
        launch_gamg_pack(s, L, mode, x, xc, alpha, p, q);
        ++k;
        err = exchange_counts(m, G->if_count[&L - lv.data()], L.sendbuf, L.xr, s);
    };
    auto reduce = [&](int what, double* alpha) {
        if (err != SPUMA_OK) return;
        err = allgather4(m, G->rank_part, G->gathered, s);
        launch_gamg_fin(s, what, G->gathered, m->n_ranks, alpha, m->ws.scal);
        ++k;
    };
    double* rp = dd ? G->rank_part : nullptr;
    if (nl == 1) {  // the finest level is the coarsest: exact-ish solve of A x = r, psi += x
        if (dd) {
            err = gamg_coarsest_dd(m, gp, s, &k);
        } else {
            cudaMemsetAsync(lv[0].x, 0, sizeof(double) * lv[0].a.N, s);
            launch_pcg_single(s, lv[0].a, G->cws);
        }
        launch_add(s, lv[0].a.N, lv[0].x, m->h_ptrs->psi);
        halo(lv[0], 0, m->h_ptrs->psi, nullptr, nullptr, nullptr, nullptr);
        launch_gamg_residual(s, lv[0], w0, rp);
        if (dd) reduce(1, nullptr);
        if (st) *st = err;
        return k + 3;
    }
    // one smoother sweep on level L: from x' = xin (+ alpha xc[ftc] if xc) into out (acc: psi += x)
    auto sweep = [&](GLevel& L, const double* xin, const double* xc, const double* alpha, double* out,
                     bool acc) {
        halo(L, xc ? 1 : 0, xin, xc, alpha, nullptr, nullptr);
        if (gp.smoother != SPUMA_SMOOTHER_GS2) {
            launch_gamg_smooth(s, L, P, xin, out, gp.omega, xc, alpha, acc);
            ++k;
            return;
        }
        launch_gamg_gs2_res(s, L, P, xin, xc, alpha, L.r);  // two-stage Gauss-Seidel (Q30)
        ++k;
        if (gp.n_inner == 0) {
            launch_gamg_gs2_upd(s, L, P, xin, xc, alpha, L.r, nullptr, out, true, true, acc);
            ++k;
            return;
        }
        const double* zin = nullptr;
        double* zb[2] = {L.p, L.q};
        for (int it = 0; it < gp.n_inner; ++it, ++k) {
            const bool last = it + 1 == gp.n_inner;
            double* zo = last ? out : zb[it & 1];
            launch_gamg_gs2_upd(s, L, P, xin, xc, alpha, L.r, zin, zo, false, last, acc);
            zin = zo;
        }
    };
    // the small levels t..nl-1 in one CTA (k_gamg_tail) when the configuration allows it
    int t = nl;
    if (!dd && m->gamg_tail_cells > 0 && gp.smoother == SPUMA_SMOOTHER_RICHARDSON && gp.scale_correction &&
        gp.n_pre_sweeps == 0 && gp.n_post_sweeps >= 1) {
        for (int l = 1; l < nl; ++l)
            if (lv[l].a.N <= m->gamg_tail_cells) {
                t = l;
                break;
            }
        if (t >= nl - 1) t = nl;
    }
    std::vector<double*> xcur(nl, nullptr);  // buffer holding x_l; nullptr: x_l == 0
    for (int l = 0; l + 1 < nl && l < t; ++l) {
        GLevel& L = lv[l];
        double* xl = nullptr;
        if (gp.n_pre_sweeps > 0) {
            double *xin = nullptr, *xout = L.x;
            for (int i = 0; i < gp.n_pre_sweeps; ++i) {
                sweep(L, xin, nullptr, nullptr, xout, false);
                xin = xout;
                xout = xout == L.x ? L.x2 : L.x;
            }
            xl = xin;
        }
        if (xl) halo(L, 0, xl, nullptr, nullptr, nullptr, nullptr);
        launch_gamg_restrict(s, L, lv[l + 1], P, xl, l + 2 == nl ? lv[l + 1].x : nullptr);  // zeroes x_coarsest
        ++k;
        xcur[l] = xl;
    }
    GLevel& Lc = lv[nl - 1];
    if (t < nl) {
        launch_gamg_tail(s, G->d_lv, t, nl, G->cws, gp.omega, gp.n_post_sweeps);
        ++k;
        const bool in_x = gp.n_post_sweeps <= 2 || ((gp.n_post_sweeps - 2) & 1) == 0;
        xcur[t] = in_x ? lv[t].x : lv[t].x2;
    } else if (dd) {
        if (err == SPUMA_OK) err = gamg_coarsest_dd(m, gp, s, &k);
        xcur[nl - 1] = Lc.x;
    } else {
        launch_pcg_single(s, Lc.a, G->cws);
        ++k;
        xcur[nl - 1] = Lc.x;
    }
    const bool pq = gp.smoother != SPUMA_SMOOTHER_GS2 && gp.scale_correction && gp.n_post_sweeps > 0;
    for (int l = (t < nl ? t - 1 : nl - 2); l >= 0; --l) {
        GLevel& L = lv[l];
        const double* xc = xcur[l + 1];
        const double* r = xcur[l] ? L.r : L.b;
        double* out = xcur[l] == L.x ? L.x2 : L.x;
        double* other = out == L.x ? L.x2 : L.x;
        const double* alpha = gp.scale_correction ? G->alpha + l : nullptr;
        int done_sweeps = 0;
        if (gp.scale_correction) {
            halo(L, 2, nullptr, xc, nullptr, nullptr, nullptr);
            launch_gamg_scale(s, L, P, xcur[l], xc, r, gp.omega, pq, G->part, G->ticket, G->alpha + l, rp);
            ++k;
            if (dd) reduce(0, G->alpha + l);
        }
        bool acc = false;
        if (pq) {  // Richardson: sweeps 1 (+2) in one kernel, sweep 1 prepared by the scale (Q29)
            const bool two = gp.n_post_sweeps >= 2;
            done_sweeps = two ? 2 : 1;
            acc = l == 0 && done_sweeps == gp.n_post_sweeps;
            if (two) halo(L, 3, nullptr, nullptr, G->alpha + l, L.p, L.q);
            launch_gamg_post(s, L, P, G->alpha + l, gp.omega, out, two, acc);
            ++k;
        } else if (gp.n_post_sweeps > 0) {  // the correction folded into the first sweep
            done_sweeps = 1;
            acc = l == 0 && gp.n_post_sweeps == 1;
            sweep(L, xcur[l], xc, alpha, out, acc);
        } else {
            acc = l == 0;
            launch_gamg_correct(s, L, P, xcur[l], xc, alpha, out, acc);
            ++k;
        }
        if (!acc) {
            xcur[l] = out;
            std::swap(out, other);
        }
        for (int i = done_sweeps; i < gp.n_post_sweeps; ++i) {
            const bool last = i + 1 == gp.n_post_sweeps;
            sweep(L, xcur[l], nullptr, nullptr, out, l == 0 && last);
            if (!(l == 0 && last)) {
                xcur[l] = out;
                std::swap(out, other);
            }
        }
    }
    halo(lv[0], 0, m->h_ptrs->psi, nullptr, nullptr, nullptr, nullptr);
    launch_gamg_residual(s, lv[0], w0, rp);
    if (dd) reduce(1, nullptr);
    if (st) *st = err;
    return k + 1;
}

// ---------------------------------------------------------------------------
// preconditioned solvers (§8(f3)/(f4)): level schedules + buffers, kept by the handle
// ---------------------------------------------------------------------------
}  // namespace

struct PcState {
    int *order_f = nullptr, *order_b = nullptr, *flag = nullptr;
    unsigned* counter = nullptr;
    int depth_f = 0, depth_b = 0;
    int width_f = 0, width_b = 0;  // widest dependency level (rows that can run concurrently)
    double *raw = nullptr, *rD = nullptr, *t1 = nullptr, *t2 = nullptr;
    double *wT = nullptr, *rT = nullptr, *pT = nullptr, *part = nullptr;
    double *u_in = nullptr, *l_in = nullptr, *u_int = nullptr, *l_int = nullptr;
    int* csr_map = nullptr;  // device copy of the CSR map
    double *fco = nullptr, *bco = nullptr, *fcoT = nullptr, *bcoT = nullptr;  // aDILU pass coefficients (per solve)
    double *iface_t = nullptr, *xrT = nullptr;  // PBiCG: Tmul interface coefficients (staging), pT halo
    int nnz = 0;
};

namespace {

void pc_release(spuma_mesh m)
{
    PcState* P = m->pc;
    if (!P) return;
    void* ptrs[] = {P->order_f, P->order_b, P->flag, P->counter, P->raw, P->rD, P->t1, P->t2, P->wT, P->rT,
                    P->pT, P->part, P->u_in, P->l_in, P->u_int, P->l_int, P->csr_map, P->iface_t, P->xrT,
                    P->fco, P->bco, P->fcoT, P->bcoT};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    delete P;
    m->pc = nullptr;
}

// dependency levels: forward row c waits on the owners of its neighbour-side faces, backward
// row c on the neighbours of its owner-side faces; rows sorted by level (ascending cell within)
spuma_status pc_ensure(spuma_mesh m)
{
    if (m->pc) return SPUMA_OK;
    PcState* P = new PcState();
    m->pc = P;
    const int N = m->N;
    std::vector<int> of, ob;
    level_schedule(N, m->h_owner, m->h_neighbour, m->h_ownerStart, m->h_losortStart, m->h_losort, of, ob, P->depth_f,
                   P->depth_b, P->width_f, P->width_b);
    cudaStream_t s = m->stream;
    SPUMA_TRY(upload(&P->order_f, of, s));
    SPUMA_TRY(upload(&P->order_b, ob, s));
    SPUMA_TRY(dalloc(&P->flag, N + 1));
    SPUMA_TRY(dalloc(&P->counter, 1));
    for (double** b : {&P->raw, &P->rD, &P->t1, &P->t2, &P->wT, &P->rT, &P->pT}) SPUMA_TRY(dalloc(b, N));
    for (double** b : {&P->fco, &P->bco, &P->fcoT, &P->bcoT}) SPUMA_TRY(dalloc(b, m->F));
    SPUMA_TRY(dalloc(&P->part, (size_t)kMaxPartials * pc_grid(N)));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    return SPUMA_OK;
}

// (upper, lower) in internal numbering; lower == nullptr: lower = upper
spuma_status pair_in(spuma_mesh m, const double* u, const double* l, const double** uo, const double** lo)
{
    if (!l) {
        SPUMA_TRY(faces_in(m, u, uo));
        *lo = *uo;
        return SPUMA_OK;
    }
    PcState* P = m->pc;
    cudaStream_t s = m->stream;
    const bool du = is_device_ptr(u), dl = is_device_ptr(l);
    if (!m->renumber && du && dl) {
        *uo = u;
        *lo = l;
        return SPUMA_OK;
    }
    for (double** b : {&P->u_in, &P->l_in, &P->u_int, &P->l_int})
        if (!*b) SPUMA_TRY(dalloc(b, m->F));
    const double* su = u;
    const double* sl = l;
    if (!du) {
        SPUMA_CUDA(cudaMemcpyAsync(P->u_in, u, sizeof(double) * m->F, cudaMemcpyHostToDevice, s));
        su = P->u_in;
    }
    if (!dl) {
        SPUMA_CUDA(cudaMemcpyAsync(P->l_in, l, sizeof(double) * m->F, cudaMemcpyHostToDevice, s));
        sl = P->l_in;
    }
    if (!m->renumber) {
        *uo = su;
        *lo = sl;
        return SPUMA_OK;
    }
    launch_gather_pair(s, m->F, m->d_face_map, m->d_face_flip, su, sl, P->u_int, P->l_int);
    *uo = P->u_int;
    *lo = P->l_int;
    return SPUMA_OK;
}

spuma_status pc_check(spuma_mesh m, const spuma_preconditioner& pc, bool multi_rank_ok = false)
{
    if (m->n_ranks > 1 && !multi_rank_ok)
        return set_error(SPUMA_ERR_STATE, "this preconditioned solver is single-rank (DESIGN.md §3)");
    if (pc.kind < SPUMA_PC_DIAGONAL || pc.kind > SPUMA_PC_ADILU || pc.n_sweeps < 0)
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "invalid preconditioner");
    return SPUMA_OK;
}

// M from (diag, upper, lower): rD into P->rD (diagonal: 1/diag)
void pc_setup(spuma_mesh m, const spuma_preconditioner& pc, const double* d, const double* u, const double* l)
{
    PcState* P = m->pc;
    const MeshArgs a = mesh_args(m);
    if (pc.kind == SPUMA_PC_DIAGONAL) {
        launch_recip(m->stream, m->N, d, P->rD);
        return;
    }
    launch_ilu_factor(m->stream, a, P->order_f, d, u, pc.kind == SPUMA_PC_DIC ? u : l, P->raw, P->rD, P->flag,
                      P->counter, P->width_f);
    if (pc.kind == SPUMA_PC_ADILU && P->fco)
        launch_adilu_coefs(m->stream, a, P->rD, u, l, P->fco, P->bco, P->fcoT, P->bcoT);
}

void pc_apply(spuma_mesh m, const spuma_preconditioner& pc, const double* u, const double* l, const double* r,
              double* w, bool transpose, const DevScal* scal)
{
    PcState* P = m->pc;
    const int k = pc.kind == SPUMA_PC_DIAGONAL ? 0 : (pc.kind == SPUMA_PC_ADILU ? pc.n_sweeps : -1);
    const bool pre = pc.kind == SPUMA_PC_ADILU && P->fco;
    launch_ilu_precondition(m->stream, mesh_args(m), P->order_f, P->order_b, P->rD, u,
                            pc.kind == SPUMA_PC_DIC ? u : l, r, w, P->t1, P->t2, P->flag, P->counter, k, transpose,
                            scal, P->width_f, P->width_b, pre ? (transpose ? P->fcoT : P->fco) : nullptr,
                            pre ? (transpose ? P->bcoT : P->bco) : nullptr);
}

// the sweeps' deadlock guard (flag[N], precond.cu): read and clear after a solve
spuma_status pc_guard(spuma_mesh m)
{
    int err = 0;
    SPUMA_CUDA(cudaMemcpy(&err, m->pc->flag + m->N, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
        SPUMA_CUDA(cudaMemset(m->pc->flag + m->N, 0, sizeof(int)));
        return set_error(SPUMA_ERR_STATE, "DIC/DILU sweep: a dependency never became ready (deadlock guard)");
    }
    return SPUMA_OK;
}

uint64_t pc_launches(const spuma_preconditioner& pc)
{
    if (pc.kind == SPUMA_PC_DIAGONAL) return 1;
    if (pc.kind == SPUMA_PC_ADILU) return pc.n_sweeps ? 1 + 2 * (uint64_t)pc.n_sweeps : 1;
    return 2;
}

// our kernels per captured iteration: direction, Amul, update; with ranks: the two reduction
// finalisations (k_finalize after NCCL's all-gather, or the fused peer all-gather + finalise), the
// halo (fused pack + P2P send and the receive, or the NCCL pack kernel) and the interface rows
// finished after the overlapped halo (ELL / lattice rows)
uint64_t launches_per_iteration(spuma_mesh m)
{
    uint64_t k = 3;
    if (m->n_ranks > 1) {
        const int rv = resolve_amul_variant(m->amul_variant, mesh_args(m));
        const bool overlap = m->n_iface && rv >= 6 && rv <= 13;
        if (overlap && m->peer && m->peer_fused && m->px.n_patches > 0) return 4;  // fused peer loop
        k += 2;
        if (m->n_iface) {
            k += m->peer ? (m->px.n_patches ? 2 : 0) : 1;
            if (overlap) k += 1;
        }
    }
    return k;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================

extern "C" {

const char* spuma_last_error(void) { return g_err.c_str(); }

int spuma_abi_version(void) { return SPUMA_ABI_VERSION; }

spuma_status spuma_nccl_get_unique_id(void* out128)
{
    if (!out128) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "out128 is NULL");
    ncclUniqueId id;
    SPUMA_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return SPUMA_OK;
}

void spuma_free(spuma_mesh m)
{
    if (!m) return;
    if (m->stream) cudaStreamSynchronize(m->stream);
    destroy_graphs(m);
    gamg_release(m);
    pc_release(m);
    l2_reset(m);
    for (int i = 0; i < 2; ++i) {
        if (m->batch_done[i]) cudaEventDestroy(m->batch_done[i]);
        if (m->asm_ev[i]) cudaEventDestroy(m->asm_ev[i]);
    }
    void* dptrs[] = {m->d_sell_meta, m->d_sell_n, m->d_sell_o, m->d_upper_s, m->d_cmeta, m->d_clane, m->d_upper_d,
                     m->d_owner, m->d_neighbour, m->d_ownerStart, m->d_losortStart, m->d_losort, m->d_ownerLo,
                     m->d_perm, m->d_face_map, m->d_delta, m->d_weights, m->d_magSf, m->d_bkind, m->d_bcell,
                     m->d_bproc, m->d_bmagSf, m->d_bdelta, m->d_bweight, m->d_bvalue, m->d_bgamma_r,
                     m->d_bis_owner, m->d_bStart, m->d_bFace, m->d_bAllStart, m->d_bAllFace, m->d_face_flip,
                     m->d_bphi, m->d_bflux, m->d_face_b, m->d_face_c, m->d_Sf, m->d_C, m->d_corrvec, m->d_bSf,
                     m->d_bnC, m->d_G, m->d_Gr, m->d_pr, m->d_bcflux, m->d_face_d, m->d_div, m->d_cell_v, m->d_ifStart, m->d_ifIdx, m->d_if_cell, m->d_ifMask, m->d_ifRows,
                     m->d_sendbuf, m->d_cell_a, m->d_cell_b, m->d_cell_c, m->d_cell_d, m->d_cell_e, m->d_cell_t,
                     m->d_face_a, m->d_face_t, m->d_iface_a, m->ws.wA, m->ws.rA, m->ws.pA, m->ws.pA2, m->ws.rD, m->ws.sumA,
                     m->ws.xr, m->ws.part, m->ws.scal, m->ws.ptrs};
    for (void* p : dptrs)
        if (p) cudaFree(p);
    if (m->h_ptrs) cudaFreeHost(m->h_ptrs);
    if (m->h_send) cudaFreeHost(m->h_send);
    if (m->h_recv) cudaFreeHost(m->h_recv);
    if (m->h_part) cudaFreeHost(m->h_part);
    if (m->h_scal) cudaFreeHost(m->h_scal);
    for (void* p : m->peer_mapped)
        if (p) cudaIpcCloseMemHandle(p);
    if (m->d_mail) cudaFree(m->d_mail);
    if (m->pst.ctr) cudaFree(m->pst.ctr);
    if (m->d_px) cudaFree(m->d_px);
    if (m->d_pg) cudaFree(m->d_pg);
    if (m->d_if_patch) cudaFree(m->d_if_patch);
    if (m->comm) ncclCommDestroy(m->comm);
    if (m->comm_stream) cudaStreamDestroy(m->comm_stream);
    if (m->ev_fork) cudaEventDestroy(m->ev_fork);
    if (m->tfork) cudaEventDestroy(m->tfork);
    if (m->tstream) cudaStreamDestroy(m->tstream);
    if (m->ev_join) cudaEventDestroy(m->ev_join);
    if (m->d_loop_bar) cudaFree(m->d_loop_bar);
    if (m->d_loop_part) cudaFree(m->d_loop_part);
    if (m->d_loop_prof) cudaFree(m->d_loop_prof);
    for (int i = 0; i < 2; ++i)
        if (m->loop_ev[i]) cudaEventDestroy(m->loop_ev[i]);
    if (m->own_stream && m->stream) cudaStreamDestroy(m->stream);
    delete m;
}

static spuma_status mesh_create_impl(const spuma_mesh_desc* d, spuma_mesh m)
{
    const int N = d->n_cells, F = d->n_faces;
    int ndev = 0;
    SPUMA_CUDA(cudaGetDeviceCount(&ndev));
    SPUMA_CUDA(cudaGetDevice(&m->device));
    if (d->cuda_stream) {
        m->stream = static_cast<cudaStream_t>(d->cuda_stream);
    } else {
        // blocking (cudaStreamDefault): a caller that filled psi / zeroed y on the legacy default
        // stream (torch's default) is ordered before the handle's work without an explicit sync
        SPUMA_CUDA(cudaStreamCreateWithFlags(&m->stream, cudaStreamDefault));
        m->own_stream = true;
    }
    m->N = N;
    m->F = F;
    m->renumber = d->renumber ? 1 : 0;
    m->rank = d->rank;
    m->n_ranks = d->n_ranks;
    const bool od = d->pointers_on_device != 0;

    // ---- A0: host copies + validation
    std::vector<int> owner, neighbour;
    std::vector<double> Sf, magSf, C, Cf;
    SPUMA_TRY(fetch(owner, d->owner, F, od));
    SPUMA_TRY(fetch(neighbour, d->neighbour, F, od));
    SPUMA_TRY(fetch(Sf, d->Sf, 3 * (size_t)F, od));
    SPUMA_TRY(fetch(magSf, d->magSf, F, od));
    SPUMA_TRY(fetch(C, d->C, 3 * (size_t)N, od));
    SPUMA_TRY(fetch(Cf, d->Cf, 3 * (size_t)F, od));
    std::string why;
    if (!valid_addressing(N, F, owner.data(), neighbour.data(), &why)) return set_error(SPUMA_ERR_ADDRESSING, why);

    struct HP {
        int kind, n, rank;
        std::vector<int> cells, gface;
        std::vector<double> Sf, magSf, Cf, nC;
        std::vector<signed char> own;
    };
    std::vector<HP> hp(d->n_patches);
    for (int p = 0; p < d->n_patches; ++p) {
        const spuma_patch_desc& pd = d->patches[p];
        HP& h = hp[p];
        h.kind = pd.kind;
        h.n = pd.n_faces;
        h.rank = pd.neighbour_rank;
        if (pd.kind < SPUMA_PATCH_ZERO_GRADIENT || pd.kind > SPUMA_PATCH_PROCESSOR)
            return set_error(SPUMA_ERR_INVALID_ARGUMENT, "patch " + std::to_string(p) + ": bad kind");
        if (pd.n_faces < 0) return set_error(SPUMA_ERR_LENGTH_MISMATCH, "patch " + std::to_string(p) + ": n_faces < 0");
        SPUMA_TRY(fetch(h.cells, pd.face_cells, pd.n_faces, od));
        SPUMA_TRY(fetch(h.Sf, pd.Sf, 3 * (size_t)pd.n_faces, od));
        SPUMA_TRY(fetch(h.magSf, pd.magSf, pd.n_faces, od));
        SPUMA_TRY(fetch(h.Cf, pd.Cf, 3 * (size_t)pd.n_faces, od));
        for (int c : h.cells)
            if (c < 0 || c >= N)
                return set_error(SPUMA_ERR_ADDRESSING, "patch " + std::to_string(p) + ": face cell out of range");
        if (pd.kind == SPUMA_PATCH_PROCESSOR) {
            if (d->n_ranks <= 1 || pd.neighbour_rank < 0 || pd.neighbour_rank >= d->n_ranks ||
                pd.neighbour_rank == d->rank)
                return set_error(SPUMA_ERR_INVALID_ARGUMENT, "patch " + std::to_string(p) + ": bad neighbour_rank");
            SPUMA_TRY(fetch(h.gface, pd.global_face, pd.n_faces, od));
            SPUMA_TRY(fetch(h.nC, pd.neighbour_C, 3 * (size_t)pd.n_faces, od));
            SPUMA_TRY(fetch(h.own, pd.is_owner, pd.n_faces, od));
            for (int i = 1; i < pd.n_faces; ++i)
                if (h.gface[i] <= h.gface[i - 1])
                    return set_error(SPUMA_ERR_ADDRESSING, "processor patch " + std::to_string(p) +
                                                               ": global_face not strictly ascending (Q13)");
        }
    }

    // ---- A1: renumbering
    if (m->renumber) {
        m->h_perm = rcm_permutation(N, F, owner.data(), neighbour.data());
        std::vector<int> o2, n2;
        std::vector<char> flip;
        rekey_faces(N, F, m->h_perm.data(), owner.data(), neighbour.data(), o2, n2, m->h_face_map, flip);
        m->h_face_flip.assign(flip.begin(), flip.end());
        std::vector<double> Sf2(3 * (size_t)F), magSf2(F), Cf2(3 * (size_t)F), C2(3 * (size_t)N);
        for (int g = 0; g < F; ++g) {
            const int f = m->h_face_map[g];
            const double sg = flip[g] ? -1.0 : 1.0;
            for (int k = 0; k < 3; ++k) {
                Sf2[3 * (size_t)g + k] = flip[g] ? -Sf[3 * (size_t)f + k] : Sf[3 * (size_t)f + k];
                Cf2[3 * (size_t)g + k] = Cf[3 * (size_t)f + k];
            }
            (void)sg;
            magSf2[g] = magSf[f];
        }
        for (int c = 0; c < N; ++c)
            for (int k = 0; k < 3; ++k) C2[3 * (size_t)m->h_perm[c] + k] = C[3 * (size_t)c + k];
        owner.swap(o2);
        neighbour.swap(n2);
        Sf.swap(Sf2);
        magSf.swap(magSf2);
        Cf.swap(Cf2);
        C.swap(C2);
        for (auto& h : hp)
            for (int& c : h.cells) c = m->h_perm[c];
    } else {
        m->h_perm.resize(N);
        for (int c = 0; c < N; ++c) m->h_perm[c] = c;
        m->h_face_map.resize(F);
        for (int f = 0; f < F; ++f) m->h_face_map[f] = f;
    }

    // ---- A2: derived addressing
    std::vector<int> ownerLo;
    derived_addressing(N, F, owner.data(), neighbour.data(), m->h_ownerStart, m->h_losort, m->h_losortStart, ownerLo);
    m->h_owner = owner;
    m->h_neighbour = neighbour;

    // boundary faces, concatenated in patch order
    std::vector<int> bkind, bcell, bproc, if_cell;
    std::vector<double> bSf, bmagSf, bCf, bnC;
    std::vector<signed char> bown;
    std::vector<char> contributes;
    int iface_off = 0;
    for (int p = 0; p < (int)hp.size(); ++p) {
        const HP& h = hp[p];
        Patch P{h.kind, h.n, (int)bkind.size(), h.rank, h.kind == SPUMA_PATCH_PROCESSOR ? iface_off : -1};
        m->patches.push_back(P);
        for (int i = 0; i < h.n; ++i) {
            bkind.push_back(h.kind);
            bcell.push_back(h.cells[i]);
            for (int k = 0; k < 3; ++k) {
                bSf.push_back(h.Sf[3 * (size_t)i + k]);
                bCf.push_back(h.Cf[3 * (size_t)i + k]);
                bnC.push_back(h.kind == SPUMA_PATCH_PROCESSOR ? h.nC[3 * (size_t)i + k] : 0.0);
            }
            bmagSf.push_back(h.magSf[i]);
            bown.push_back(h.kind == SPUMA_PATCH_PROCESSOR ? h.own[i] : 0);
            contributes.push_back(h.kind == SPUMA_PATCH_FIXED_VALUE || h.kind == SPUMA_PATCH_PROCESSOR);
            if (h.kind == SPUMA_PATCH_PROCESSOR) {
                bproc.push_back(iface_off++);
                if_cell.push_back(h.cells[i]);
            } else {
                bproc.push_back(-1);
            }
        }
    }
    m->Fb = (int)bkind.size();
    m->n_iface = iface_off;
    std::vector<int> bStart, bFace;
    cell_lists(N, bcell, contributes, bStart, bFace);
    std::vector<int> bAllStart, bAllFace;
    {
        std::vector<char> nonempty(bkind.size());
        for (size_t i = 0; i < bkind.size(); ++i) nonempty[i] = bkind[i] != SPUMA_PATCH_EMPTY;
        cell_lists(N, bcell, nonempty, bAllStart, bAllFace);
    }
    std::vector<int> ifStart, ifIdx;
    cell_lists(N, if_cell, std::vector<char>(if_cell.size(), 1), ifStart, ifIdx);

    // ---- uploads
    cudaStream_t s = m->stream;
    SPUMA_TRY(upload(&m->d_owner, owner, s));
    SPUMA_TRY(upload(&m->d_neighbour, neighbour, s));
    SPUMA_TRY(upload(&m->d_ownerStart, m->h_ownerStart, s));
    SPUMA_TRY(upload(&m->d_losortStart, m->h_losortStart, s));
    SPUMA_TRY(upload(&m->d_losort, m->h_losort, s));
    SPUMA_TRY(upload(&m->d_ownerLo, ownerLo, s));
    {
        const SellHost sell = build_sell(N, m->h_ownerStart, m->h_losortStart, m->h_losort, ownerLo, neighbour);
        if (sell.ok) {
            m->sell_wn = sell.uniform_wn;
            m->sell_wo = sell.uniform_wo;
            if (m->sell_wo >= 0) SPUMA_TRY(dalloc(&m->d_upper_s, (size_t)32 * m->sell_wo * ((N + 31) / 32)));
            if (m->sell_wn >= 0 && m->sell_wn <= 3 && m->sell_wo >= 0 && m->sell_wo <= 3) {
                const EllStencil st =
                    build_ell_stencil(N, m->h_ownerStart, m->h_losortStart, m->h_losort, ownerLo, neighbour);
                if (st.compressed > 0) {
                    SPUMA_TRY(upload(&m->d_cmeta, st.meta, s));
                    SPUMA_TRY(upload(&m->d_clane, st.lane, s));
                }
            }
            SPUMA_TRY(upload(&m->d_sell_meta, sell.meta, s));
            SPUMA_TRY(upload(&m->d_sell_n, sell.nslot, s));
            SPUMA_TRY(upload(&m->d_sell_o, sell.oslot, s));
        }
    }
    {  // lattice slots (variant 12): absent slots are filled once here, present ones per solve
        int D[3] = {0, 0, 0};
        const int K = F > 0 ? lattice_offsets(N, F, owner.data(), neighbour.data(), D) : 0;
        if (K > 0) {
            m->lat_K = K;
            for (int t = 0; t < 3; ++t) m->lat_D[t] = D[t];
            m->lat_S = ((long long)N + 31) / 32 * 32;
            SPUMA_TRY(dalloc(&m->d_upper_d, (size_t)(K * m->lat_S)));
            launch_fill_u64(s, (long long)K * m->lat_S, m->d_upper_d, kLatAbsent);
        }
    }
    if (m->renumber) {
        SPUMA_TRY(upload(&m->d_perm, m->h_perm, s));
        SPUMA_TRY(upload(&m->d_face_map, m->h_face_map, s));
        SPUMA_TRY(upload(&m->d_face_flip, m->h_face_flip, s));
    }
    SPUMA_TRY(upload(&m->d_magSf, magSf, s));
    SPUMA_TRY(upload(&m->d_bkind, bkind, s));
    SPUMA_TRY(upload(&m->d_bcell, bcell, s));
    SPUMA_TRY(upload(&m->d_bproc, bproc, s));
    SPUMA_TRY(upload(&m->d_bmagSf, bmagSf, s));
    SPUMA_TRY(upload(&m->d_bis_owner, bown, s));
    SPUMA_TRY(upload(&m->d_bStart, bStart, s));
    SPUMA_TRY(upload(&m->d_bFace, bFace, s));
    SPUMA_TRY(upload(&m->d_bAllStart, bAllStart, s));
    SPUMA_TRY(upload(&m->d_bAllFace, bAllFace, s));
    SPUMA_TRY(dalloc(&m->d_bphi, m->Fb));
    SPUMA_TRY(dalloc(&m->d_bflux, m->Fb));
    SPUMA_TRY(upload(&m->d_ifStart, ifStart, s));
    SPUMA_TRY(upload(&m->d_ifIdx, ifIdx, s));
    SPUMA_TRY(upload(&m->d_if_cell, if_cell, s));
    m->h_if_cell = if_cell;
    {
        std::vector<unsigned> mask((N + 31) / 32 + 1, 0u);
        for (int c : if_cell) mask[c >> 5] |= 1u << (c & 31);
        SPUMA_TRY(upload(&m->d_ifMask, mask, s));
        std::vector<int> rows;
        for (int c = 0; c < N; ++c)
            if ((mask[c >> 5] >> (c & 31)) & 1u) rows.push_back(c);
        m->n_ifRows = (int)rows.size();
        SPUMA_TRY(upload(&m->d_ifRows, rows, s));
    }
    SPUMA_TRY(dalloc(&m->d_bdelta, m->Fb));
    SPUMA_TRY(dalloc(&m->d_bweight, m->Fb));
    SPUMA_TRY(dalloc(&m->d_bvalue, m->Fb));
    SPUMA_CUDA(cudaMemsetAsync(m->d_bvalue, 0, sizeof(double) * std::max(m->Fb, 1), s));
    SPUMA_TRY(dalloc(&m->d_bgamma_r, m->n_iface));
    SPUMA_TRY(dalloc(&m->d_sendbuf, m->n_iface));
    SPUMA_TRY(dalloc(&m->d_delta, F));
    SPUMA_TRY(dalloc(&m->d_weights, F));

    // ---- A3: geometry on the device
    {
        double *dSf = nullptr, *dC = nullptr, *dCf = nullptr, *dbSf = nullptr, *dbCf = nullptr, *dbnC = nullptr;
        SPUMA_TRY(upload(&dSf, Sf, s));
        SPUMA_TRY(upload(&dC, C, s));
        SPUMA_TRY(upload(&dCf, Cf, s));
        SPUMA_TRY(upload(&dbSf, bSf, s));
        SPUMA_TRY(upload(&dbCf, bCf, s));
        SPUMA_TRY(upload(&dbnC, bnC, s));
        launch_geometry(s, F, m->d_owner, m->d_neighbour, dSf, m->d_magSf, dC, dCf, m->d_delta, m->d_weights);
        launch_bgeometry(s, m->Fb, m->d_bkind, m->d_bcell, dbSf, m->d_bmagSf, dbCf, dC, dbnC, m->d_bis_owner,
                         m->d_bdelta, m->d_bweight);
        SPUMA_TRY(dalloc(&m->d_corrvec, 3 * (size_t)F));
        launch_corrvec(s, F, m->d_owner, m->d_neighbour, dSf, m->d_magSf, dC, m->d_delta, m->d_corrvec);
        m->stats.kernel_launches += (F > 0) * 2 + (m->Fb > 0);
        SPUMA_CUDA(cudaStreamSynchronize(s));
        // kept for the non-orthogonal correction (gradient and processor correction vectors)
        m->d_Sf = dSf;
        m->d_C = dC;
        m->d_bSf = dbSf;
        m->d_bnC = dbnC;
        cudaFree(dCf);
        cudaFree(dbCf);
    }

    // ---- workspaces (allocated once: the paper's memory-pool lesson)
    m->grid = occupancy_grid(N, &m->grid_faces, F);
    SPUMA_TRY(dalloc(&m->ws.wA, N + 1));
    SPUMA_TRY(dalloc(&m->ws.rA, N + 1));
    SPUMA_TRY(dalloc(&m->ws.pA, N + 1));
    SPUMA_TRY(dalloc(&m->ws.pA2, N + 1));
    m->ws.pA_prev = m->ws.pA;
    SPUMA_TRY(dalloc(&m->ws.rD, N + 1));
    SPUMA_TRY(dalloc(&m->ws.sumA, N + 1));
    SPUMA_TRY(dalloc(&m->ws.xr, m->n_iface));
    SPUMA_TRY(dalloc(&m->ws.part, (size_t)kMaxPartials * std::max(m->grid, 4 * std::max(m->n_ranks, 1))));
    SPUMA_TRY(dalloc(&m->ws.scal, 1));
    SPUMA_TRY(dalloc(&m->ws.ptrs, 1));
    SPUMA_CUDA(cudaMemsetAsync(m->ws.scal, 0, sizeof(DevScal), s));
    SPUMA_CUDA(cudaMemsetAsync(m->ws.pA, 0, sizeof(double) * (N + 1), s));
    SPUMA_CUDA(cudaMallocHost(reinterpret_cast<void**>(&m->h_ptrs), sizeof(DevPtrs)));
    SPUMA_CUDA(cudaMallocHost(reinterpret_cast<void**>(&m->h_scal), 2 * sizeof(DevScal)));
    for (int i = 0; i < 2; ++i) {
        SPUMA_CUDA(cudaEventCreateWithFlags(&m->batch_done[i], cudaEventDisableTiming));
        SPUMA_CUDA(cudaEventCreate(&m->asm_ev[i]));
    }

    // ---- communicator
    if (m->n_ranks > 1) {
        for (const auto& P : m->patches)
            if (P.kind == SPUMA_PATCH_PROCESSOR && P.n_faces > 0) {
                m->cb_peers.push_back(P.neighbour_rank);
                m->cb_offsets.push_back(P.iface_offset);
                m->cb_counts.push_back(P.n_faces);
            }
        SPUMA_CUDA(cudaStreamCreateWithFlags(&m->comm_stream, cudaStreamNonBlocking));
        SPUMA_CUDA(cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming));
        SPUMA_CUDA(cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming));
        if (!d->nccl_unique_id) {
            m->external_comm = true;
            SPUMA_CUDA(cudaMallocHost(reinterpret_cast<void**>(&m->h_send), sizeof(double) * (m->n_iface + 1)));
            SPUMA_CUDA(cudaMallocHost(reinterpret_cast<void**>(&m->h_recv), sizeof(double) * (m->n_iface + 1)));
            SPUMA_CUDA(cudaMallocHost(reinterpret_cast<void**>(&m->h_part), sizeof(double) * 4 * (m->n_ranks + 1)));
        } else {
            ncclUniqueId id;
            std::memcpy(&id, d->nccl_unique_id, sizeof(id));
            SPUMA_NCCL(ncclCommInitRank(&m->comm, m->n_ranks, id, m->rank));
        }
    }
    SPUMA_CUDA(cudaStreamSynchronize(s));
    m->stats.blocks_per_grid = m->grid;
    m->stats.threads_per_block = kThreads;
    m->stats.batch_iterations = m->batch;
    return SPUMA_OK;
}

spuma_status spuma_mesh_create(const spuma_mesh_desc* d, spuma_mesh* out)
{
    SPUMA_NVTX("spuma_mesh_create");
    if (!out) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!d) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "desc is NULL");
    if (d->abi_version != SPUMA_ABI_VERSION) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "abi_version mismatch");
    if (d->n_cells < 0 || d->n_faces < 0) return set_error(SPUMA_ERR_LENGTH_MISMATCH, "negative size");
    if (d->n_patches < 0 || (d->n_patches > 0 && !d->patches))
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "patches is NULL");
    if (d->n_ranks < 1 || d->rank < 0 || d->rank >= d->n_ranks)
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "bad rank / n_ranks");
    if (d->n_faces > 0 && (!d->owner || !d->neighbour || !d->Sf || !d->magSf || !d->Cf))
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL face array");
    if (d->n_cells > 0 && !d->C) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "C is NULL");
    spuma_mesh m = new spuma_mesh_s();
    spuma_status st = mesh_create_impl(d, m);
    if (st != SPUMA_OK) {
        spuma_free(m);
        return st;
    }
    g_err.clear();
    *out = m;
    return SPUMA_OK;
}

spuma_status spuma_assemble_laplacian(spuma_mesh m, const spuma_scalar* gamma, const spuma_scalar* const* patch_value,
                                      spuma_label ref_cell, spuma_scalar ref_value, spuma_scalar* diag,
                                      spuma_scalar* upper, spuma_scalar* source, spuma_scalar* iface_coeffs)
{
    SPUMA_NVTX("spuma_assemble_laplacian");
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if ((m->N > 0 && (!diag || !source)) || (m->F > 0 && !upper))
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL diag/upper/source");
    if (m->n_iface > 0 && !iface_coeffs) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "iface_coeffs is NULL");
    if (ref_cell >= m->N) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "ref_cell out of range");
    cudaStream_t s = m->stream;
    // fixedValue values -> concatenated boundary buffer
    for (size_t p = 0; p < m->patches.size(); ++p) {
        const Patch& P = m->patches[p];
        if (P.kind != SPUMA_PATCH_FIXED_VALUE || P.n_faces == 0) continue;
        if (!patch_value || !patch_value[p])
            return set_error(SPUMA_ERR_INVALID_ARGUMENT, "missing fixedValue values for patch " + std::to_string(p));
        SPUMA_CUDA(cudaMemcpyAsync(m->d_bvalue + P.offset, patch_value[p], sizeof(double) * P.n_faces,
                                   cudaMemcpyDefault, s));
    }
    const double* g = nullptr;
    if (gamma) SPUMA_TRY(cells_in(m, gamma, R_GAMMA, &g));
    // internal outputs
    const double* src_in = nullptr;
    SPUMA_TRY(cells_in(m, source, R_SOURCE, &src_in));
    double* src_i = const_cast<double*>(src_in);
    double* diag_i = diag;
    if (m->renumber || !is_device_ptr(diag) || !aligned16(diag)) {
        if (!m->d_cell_b) SPUMA_TRY(dalloc(&m->d_cell_b, m->N));
        diag_i = m->d_cell_b;
    }
    double* upper_i = upper;
    if (m->renumber || !is_device_ptr(upper)) {
        if (!m->d_face_a) SPUMA_TRY(dalloc(&m->d_face_a, m->F));
        upper_i = m->d_face_a;
    }
    double* iface_i = iface_coeffs;
    if (m->n_iface && !is_device_ptr(iface_coeffs)) {
        if (!m->d_iface_a) SPUMA_TRY(dalloc(&m->d_iface_a, m->n_iface));
        iface_i = m->d_iface_a;
    }
    // gamma halo (processor faces interpolate gamma in global orientation)
    if (g && m->n_iface) SPUMA_TRY(halo_exchange(m, g, m->d_bgamma_r, s));
    const int rc = ref_cell < 0 ? -1 : (m->renumber ? m->h_perm[ref_cell] : ref_cell);
    const MeshArgs a = mesh_args(m);
    if (m->timing) SPUMA_CUDA(cudaEventRecord(m->asm_ev[0], s));
    launch_face_coeffs(s, m->grid_faces, m->F, m->d_owner, m->d_neighbour, m->d_delta, m->d_weights, m->d_magSf, g,
                       upper_i);
    launch_diag_gather(s, m->grid, a, upper_i, m->d_bStart, m->d_bFace, m->d_bkind, m->d_bcell, m->d_bproc,
                       m->d_bmagSf, m->d_bdelta, m->d_bweight, m->d_bvalue, m->d_bgamma_r, m->d_bis_owner, g, rc,
                       ref_value, diag_i, src_i, iface_i);
    if (m->timing) SPUMA_CUDA(cudaEventRecord(m->asm_ev[1], s));
    m->stats.kernel_launches += 2;
    SPUMA_TRY(cells_out(m, diag, diag_i));
    SPUMA_TRY(faces_out(m, upper, upper_i));
    SPUMA_TRY(cells_out(m, source, src_i));
    if (iface_i != iface_coeffs)
        SPUMA_CUDA(cudaMemcpyAsync(iface_coeffs, iface_i, sizeof(double) * m->n_iface, cudaMemcpyDefault, s));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    SPUMA_CUDA(cudaGetLastError());
    if (m->timing) {
        float ms = 0.f;
        SPUMA_CUDA(cudaEventElapsedTime(&ms, m->asm_ev[0], m->asm_ev[1]));
        m->stats.phase_ms[3] += ms;
        m->stats.phase_count[3] += 1;
    }
    return peer_guard(m);
}

spuma_status spuma_amul(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                        const spuma_scalar* iface_coeffs, const spuma_scalar* x, spuma_scalar* y)
{
    SPUMA_NVTX("spuma_amul");
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (m->N > 0 && (!diag || !x || !y)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array");
    if (m->F > 0 && !upper) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "upper is NULL");
    if (m->n_iface > 0 && !iface_coeffs) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "iface_coeffs is NULL");
    cudaStream_t s = m->stream;
    const double *d_i, *u_i, *x_i, *if_i = nullptr;
    SPUMA_TRY(cells_in(m, diag, R_DIAG, &d_i));
    SPUMA_TRY(faces_in(m, upper, &u_i));
    SPUMA_TRY(cells_in(m, x, R_X, &x_i));
    if (m->n_iface) SPUMA_TRY(iface_in(m, iface_coeffs, &if_i));
    double* y_i = y;
    if (m->renumber || !is_device_ptr(y) || !aligned16(y)) {
        if (!m->d_cell_t) SPUMA_TRY(dalloc(&m->d_cell_t, m->N));
        y_i = m->d_cell_t;
    }
    SPUMA_TRY(halo_exchange(m, x_i, m->ws.xr, s));
    prepare_amul_coeffs(m, s, mesh_args(m), u_i);
    launch_amul(s, m->amul_variant, mesh_args(m), d_i, u_i, if_i, x_i, m->ws.xr, y_i,
                (x_i == x) ? (long long)m->N : (long long)m->N + kPad, m->sell_wn, m->sell_wo);
    m->stats.kernel_launches += 1;
    SPUMA_TRY(cells_out(m, y, y_i));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    SPUMA_CUDA(cudaGetLastError());
    return peer_guard(m);
}

spuma_status spuma_pcg_solve(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                             const spuma_scalar* iface_coeffs, const spuma_scalar* source, spuma_scalar* psi,
                             const spuma_solver_controls* ctl, spuma_solver_perf* perf)
{
    SPUMA_NVTX("spuma_pcg_solve");
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (!ctl || !perf) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL controls/perf");
    if (m->N > 0 && (!diag || !source || !psi)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array");
    if (m->F > 0 && !upper) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "upper is NULL");
    if (m->n_iface > 0 && !iface_coeffs) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "iface_coeffs is NULL");
    if (ctl->max_iter < 0 || ctl->min_iter < 0) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "negative iteration limit");
    cudaStream_t s = m->stream;
    DevPtrs P{};
    const double* psi_in = nullptr;
    SPUMA_TRY(cells_in(m, diag, R_DIAG, &P.diag));
    SPUMA_TRY(faces_in(m, upper, &P.upper));
    SPUMA_TRY(cells_in(m, source, R_SOURCE, &P.source));
    SPUMA_TRY(cells_in(m, psi, R_PSI, &psi_in));
    P.psi = const_cast<double*>(psi_in);
    if (m->n_iface) SPUMA_TRY(iface_in(m, iface_coeffs, &P.iface));
    *m->h_ptrs = P;
    SPUMA_CUDA(cudaMemcpyAsync(m->ws.ptrs, m->h_ptrs, sizeof(DevPtrs), cudaMemcpyHostToDevice, s));
    launch_scal_init(s, m->ws, *ctl, m->n_ranks);

    // ---- small meshes: the whole solve in one single-CTA launch (latency path) -- up to 3072 cells
    // when the persistent loop could run instead (it takes ~10-11 us per iteration at any small size;
    // one CTA 9.4 us at 2197 cells, 12.2 at 4096, 22.1 at 8000: profiles/r02ar_small_threshold_ab.jsonl)
    constexpr int kLoopBeatsSmallCells = 3072;
    if (m->n_ranks == 1 && m->N <= m->small_max_cells && !m->timing &&
        (m->N <= kLoopBeatsSmallCells || !loop_layout(m, mesh_args(m)))) {
        if (!(m->small_smem && launch_pcg_single_smem(s, mesh_args(m), m->ws))) launch_pcg_single(s, mesh_args(m), m->ws);
        m->stats.kernel_launches += 2;
        DevScal fs;
        SPUMA_CUDA(cudaMemcpyAsync(m->h_scal, m->ws.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
        SPUMA_CUDA(cudaStreamSynchronize(s));
        fs = m->h_scal[0];
        SPUMA_CUDA(cudaGetLastError());
        perf->initial_residual = fs.init;
        perf->final_residual = fs.fin;
        perf->n_iterations = fs.n;
        perf->converged = fs.converged;
        perf->singular = fs.singular;
        m->stats.solves += 1;
        m->stats.iterations += fs.n;
        SPUMA_TRY(cells_out(m, psi, P.psi));
        SPUMA_CUDA(cudaStreamSynchronize(s));
        return SPUMA_OK;
    }

    // ---- A6 setup
    spuma::NvtxRange nvtx_loop("A6 setup + A7-A11 loop");
    const MeshArgs a = mesh_args(m);
    prepare_amul_coeffs(m, s, a, P.upper);
    const bool fin = m->n_ranks == 1;
    SPUMA_TRY(halo_exchange(m, P.psi, m->ws.xr, s));
    launch_setup1(s, m->grid, a, m->ws, fin);
    if (!fin) SPUMA_TRY(reduce_finalize(m, 1, s));
    launch_setup2(s, m->grid, a, m->ws, fin);
    if (!fin) SPUMA_TRY(reduce_finalize(m, 2, s));
    m->stats.kernel_launches += 3;

    bool looped = false;
    m->stats.loop_mode = 0;
    if (const int lay = loop_layout(m, a)) SPUMA_TRY(run_pcg_loop(m, s, a, lay, &looped));
    if (looped) {
        // the whole loop ran in one launch (scalars in ws.scal)
    } else if (m->external_comm) {  // host callbacks cannot be captured: iterate with direct launches
        SPUMA_CUDA(cudaMemcpyAsync(&m->h_scal[0], m->ws.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
        SPUMA_CUDA(cudaStreamSynchronize(s));
        int it = 0;
        while (!m->h_scal[0].done) {
            SPUMA_TRY(enqueue_iteration(m, s, nullptr, it));
            SPUMA_CUDA(cudaMemcpyAsync(&m->h_scal[0], m->ws.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
            SPUMA_CUDA(cudaStreamSynchronize(s));
            if (++it > iter_bound(ctl) + 1) return set_error(SPUMA_ERR_STATE, "PCG loop did not terminate");
        }
    } else {
    // ---- A7-A11 in captured batches, ping-pong; host reads the scalars once per batch
    SPUMA_TRY(build_graphs(m));
    if (m->l2_persist) {  // the graphs' window makes its target's lines persisting; release another target's first
        double* const tg[5] = {nullptr, m->ws.pA, m->ws.rA, m->ws.rD, m->ws.wA};
        cudaAccessPolicyWindow unused{};
        bool use = false;
        SPUMA_TRY(l2_policy(m, m->l2_persist, &unused, &use));  // also releases stale lines when no window
        if (use) m->l2_lines = tg[m->l2_persist];
    }
    SPUMA_CUDA(cudaMemcpyAsync(&m->h_scal[1], m->ws.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    uint64_t launched_batches = 0;
    int done = m->h_scal[1].done;
    int b = 0;
    int prev_n = 0;
    while (!done) {
        const int g = b & 1;
        SPUMA_CUDA(cudaGraphLaunch(m->gexec[g], s));
        SPUMA_CUDA(cudaMemcpyAsync(&m->h_scal[g], m->ws.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
        SPUMA_CUDA(cudaEventRecord(m->batch_done[g], s));
        ++launched_batches;
        if (b > 0) {  // wait for the previous batch while this one runs
            const int pg = (b - 1) & 1;
            SPUMA_CUDA(cudaEventSynchronize(m->batch_done[pg]));
            if (m->timing) {
                SPUMA_TRY(account_timing(m, pg, m->h_scal[pg].n - prev_n));
                prev_n = m->h_scal[pg].n;
            }
            done = m->h_scal[pg].done;
            SPUMA_TRY(nccl_async_check(m));
        }
        ++b;
        if (b > 2 + (iter_bound(ctl) + m->gexec_batch - 1) / m->gexec_batch + 1) {
            cudaStreamSynchronize(s);
            return set_error(SPUMA_ERR_STATE, "PCG batch loop did not terminate");
        }
    }
    SPUMA_CUDA(cudaStreamSynchronize(s));
    if (m->timing && b > 0) SPUMA_TRY(account_timing(m, (b - 1) & 1, m->h_scal[(b - 1) & 1].n - prev_n));
    m->stats.kernel_launches += launched_batches * (uint64_t)m->gexec_batch * launches_per_iteration(m);
    }
    DevScal fs;
    SPUMA_CUDA(cudaMemcpy(&fs, m->ws.scal, sizeof(DevScal), cudaMemcpyDeviceToHost));
    if (m->defer_psi == 1 && (fs.n & 1)) {  // the last iteration's psi update is still pending
        launch_psi_flush(s, m->N, m->ws);
        m->stats.kernel_launches += 1;
        SPUMA_CUDA(cudaStreamSynchronize(s));
    } else if (m->defer_psi == 2 && fs.n > fs.psi_done) {  // the last one or two updates are pending
        launch_psi_flush2(s, m->N, m->ws, fs.n, fs.n - fs.psi_done);
        m->stats.kernel_launches += 1;
        SPUMA_CUDA(cudaStreamSynchronize(s));
    }
    SPUMA_CUDA(cudaGetLastError());
    perf->initial_residual = fs.init;
    perf->final_residual = fs.fin;
    perf->n_iterations = fs.n;
    perf->converged = fs.converged;
    perf->singular = fs.singular;
    m->stats.solves += 1;
    m->stats.iterations += fs.n;
    SPUMA_TRY(cells_out(m, psi, P.psi));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    return peer_guard(m);
}

spuma_status spuma_surface_integrate(spuma_mesh m, const spuma_scalar* phi, const spuma_scalar* const* patch_phi,
                                     const spuma_scalar* V, spuma_scalar* out)
{
    SPUMA_NVTX("spuma_surface_integrate");
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if ((m->F > 0 && !phi) || (m->N > 0 && (!V || !out))) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array");
    cudaStream_t s = m->stream;
    double* phi_i = nullptr;
    SPUMA_TRY(oriented_in(m, phi, &m->d_face_b, &phi_i));
    SPUMA_TRY(patches_in(m, patch_phi, m->d_bphi, true));
    const double* V_i = nullptr;
    SPUMA_TRY(cells_in(m, V, R_X, &V_i));
    double* out_i = out;
    if (m->renumber || !is_device_ptr(out) || !aligned16(out)) {
        if (!m->d_cell_t) SPUMA_TRY(dalloc(&m->d_cell_t, m->N));
        out_i = m->d_cell_t;
    }
    launch_surface_integrate(s, mesh_args(m), phi_i, m->d_bAllStart, m->d_bAllFace, m->d_bphi, V_i, out_i);
    m->stats.kernel_launches += 1;
    SPUMA_TRY(cells_out(m, out, out_i));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    SPUMA_CUDA(cudaGetLastError());
    return peer_guard(m);
}

spuma_status spuma_face_flux(spuma_mesh m, const spuma_scalar* gamma, const spuma_scalar* const* patch_value,
                             const spuma_scalar* upper, const spuma_scalar* psi, const spuma_scalar* corr_flux,
                             const spuma_scalar* const* patch_corr_flux, spuma_scalar* flux,
                             spuma_scalar* const* patch_flux, spuma_scalar* phi, spuma_scalar* const* patch_phi)
{
    SPUMA_NVTX("spuma_face_flux");
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if ((m->F > 0 && !upper) || (m->N > 0 && !psi)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array");
    cudaStream_t s = m->stream;
    for (size_t p = 0; p < m->patches.size(); ++p)
        if (m->patches[p].kind == SPUMA_PATCH_FIXED_VALUE && m->patches[p].n_faces > 0 && (!patch_value || !patch_value[p]))
            return set_error(SPUMA_ERR_INVALID_ARGUMENT, "missing fixedValue values for patch " + std::to_string(p));
    SPUMA_TRY(patches_in(m, patch_value, m->d_bvalue, true));
    const double *u_i = nullptr, *psi_i = nullptr, *g = nullptr;
    SPUMA_TRY(faces_in(m, upper, &u_i));
    SPUMA_TRY(cells_in(m, psi, R_PSI, &psi_i));
    if (gamma) SPUMA_TRY(cells_in(m, gamma, R_GAMMA, &g));
    if (m->n_ranks > 1) {  // psi (and gamma) of the remote cells of processor faces
        SPUMA_TRY(halo_exchange(m, psi_i, m->ws.xr, s));
        if (g) SPUMA_TRY(halo_exchange(m, g, m->d_bgamma_r, s));
    }
    double* phi_i = nullptr;
    if (phi) SPUMA_TRY(oriented_in(m, phi, &m->d_face_b, &phi_i));
    double* flux_i = nullptr;
    if (flux) {
        flux_i = flux;
        if (m->renumber || !is_device_ptr(flux)) {
            if (!m->d_face_c) SPUMA_TRY(dalloc(&m->d_face_c, m->F));
            flux_i = m->d_face_c;
        }
    }
    if (patch_phi) SPUMA_TRY(patches_in(m, patch_phi, m->d_bphi, false));
    double* cf_i = nullptr;
    if (corr_flux) SPUMA_TRY(oriented_in(m, corr_flux, &m->d_face_d, &cf_i));
    if (patch_corr_flux) {
        if (!m->d_bcflux) SPUMA_TRY(dalloc(&m->d_bcflux, m->Fb));
        SPUMA_TRY(patches_in(m, patch_corr_flux, m->d_bcflux, false));
    }
    launch_face_flux(s, m->F, m->d_owner, m->d_neighbour, u_i, psi_i, cf_i, flux_i, phi_i);
    launch_bface_flux(s, m->Fb, m->d_bkind, m->d_bcell, m->d_bproc, m->d_bmagSf, m->d_bdelta, m->d_bweight,
                      m->d_bvalue, m->d_bgamma_r, m->d_bis_owner, g, psi_i, m->ws.xr,
                      patch_corr_flux ? m->d_bcflux : nullptr, m->d_bflux, patch_phi ? m->d_bphi : nullptr);
    m->stats.kernel_launches += 2;
    if (flux) SPUMA_TRY(oriented_out(m, flux, flux_i));
    if (phi) SPUMA_TRY(oriented_out(m, phi, phi_i));
    SPUMA_TRY(patches_out(m, patch_flux, m->d_bflux));
    if (patch_phi) SPUMA_TRY(patches_out(m, patch_phi, m->d_bphi));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    SPUMA_CUDA(cudaGetLastError());
    return peer_guard(m);
}

spuma_status spuma_laplacian_correction(spuma_mesh m, const spuma_scalar* gamma,
                                        const spuma_scalar* const* patch_value, const spuma_scalar* p,
                                        const spuma_scalar* V, spuma_scalar* source, spuma_scalar* corr_flux,
                                        spuma_scalar* const* patch_corr_flux)
{
    SPUMA_NVTX("spuma_laplacian_correction");
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (m->N > 0 && (!p || !V || !source)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array");
    cudaStream_t s = m->stream;
    for (size_t q = 0; q < m->patches.size(); ++q)
        if (m->patches[q].kind == SPUMA_PATCH_FIXED_VALUE && m->patches[q].n_faces > 0 && (!patch_value || !patch_value[q]))
            return set_error(SPUMA_ERR_INVALID_ARGUMENT, "missing fixedValue values for patch " + std::to_string(q));
    SPUMA_TRY(patches_in(m, patch_value, m->d_bvalue, true));
    const double *p_i = nullptr, *g = nullptr, *src_in = nullptr;
    SPUMA_TRY(cells_in(m, p, R_PSI, &p_i));
    if (gamma) SPUMA_TRY(cells_in(m, gamma, R_GAMMA, &g));
    SPUMA_TRY(cells_in(m, source, R_SOURCE, &src_in));
    double* src_i = const_cast<double*>(src_in);
    // V: its own staging buffer (the other cell roles are in use)
    const double* V_i = V;
    if (m->renumber || !is_device_ptr(V) || !aligned16(V)) {
        if (!m->d_cell_v) SPUMA_TRY(dalloc(&m->d_cell_v, m->N));
        if (!m->renumber) {
            SPUMA_CUDA(cudaMemcpyAsync(m->d_cell_v, V, sizeof(double) * m->N, cudaMemcpyDefault, s));
        } else {
            const double* src = V;
            if (!is_device_ptr(V)) {
                if (!m->d_face_t) SPUMA_TRY(dalloc(&m->d_face_t, std::max(m->F, m->N)));
                SPUMA_CUDA(cudaMemcpyAsync(m->d_face_t, V, sizeof(double) * m->N, cudaMemcpyHostToDevice, s));
                src = m->d_face_t;
            }
            launch_scatter(s, m->N, m->d_perm, src, m->d_cell_v);
        }
        V_i = m->d_cell_v;
    }
    if (!m->d_G) SPUMA_TRY(dalloc(&m->d_G, 3 * (size_t)m->N));
    if (!m->d_Gr) SPUMA_TRY(dalloc(&m->d_Gr, 3 * (size_t)m->n_iface));
    if (!m->d_pr) SPUMA_TRY(dalloc(&m->d_pr, m->n_iface));
    if (!m->d_bcflux) SPUMA_TRY(dalloc(&m->d_bcflux, m->Fb));
    if (!m->d_face_d) SPUMA_TRY(dalloc(&m->d_face_d, m->F));
    if (!m->d_div) SPUMA_TRY(dalloc(&m->d_div, m->N));
    const MeshArgs a = mesh_args(m);
    if (m->n_ranks > 1) {
        SPUMA_TRY(halo_exchange(m, p_i, m->d_pr, s));
        if (g) SPUMA_TRY(halo_exchange(m, g, m->d_bgamma_r, s));
    }
    launch_gauss_grad(s, a, m->d_Sf, m->d_weights, p_i, m->d_bAllStart, m->d_bAllFace, m->d_bkind, m->d_bproc,
                      m->d_bSf, m->d_bvalue, m->d_bweight, m->d_bis_owner, m->d_pr, V_i, m->d_G);
    if (m->n_ranks > 1)
        for (int k = 0; k < 3; ++k)
            SPUMA_TRY(halo_exchange(m, m->d_G + (size_t)k * m->N, m->d_Gr + (size_t)k * m->n_iface, s));
    launch_nonorth_flux(s, m->F, m->N, m->d_owner, m->d_neighbour, m->d_corrvec, m->d_magSf, m->d_weights, g,
                        m->d_G, m->d_face_d);
    launch_bnonorth_flux(s, m->Fb, m->N, m->n_iface, m->d_bkind, m->d_bcell, m->d_bproc, m->d_bSf, m->d_bmagSf,
                         m->d_bdelta, m->d_bweight, m->d_bis_owner, m->d_bnC, m->d_C, m->d_G, m->d_Gr, g,
                         m->d_bgamma_r, m->d_bcflux);
    launch_surface_integrate(s, a, m->d_face_d, m->d_bAllStart, m->d_bAllFace, m->d_bcflux, V_i, m->d_div);
    launch_sub_vdiv(s, m->N, V_i, m->d_div, src_i);  // fvm.source() -= V fvc::div(correction flux)
    m->stats.kernel_launches += 5;
    SPUMA_TRY(cells_out(m, source, src_i));
    if (corr_flux) SPUMA_TRY(oriented_out(m, corr_flux, m->d_face_d));
    SPUMA_TRY(patches_out(m, patch_corr_flux, m->d_bcflux));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    SPUMA_CUDA(cudaGetLastError());
    return peer_guard(m);
}

spuma_status spuma_mesh_get_addressing(spuma_mesh m, spuma_label* perm, spuma_label* owner, spuma_label* neighbour,
                                       spuma_label* owner_start, spuma_label* losort, spuma_label* losort_start,
                                       spuma_label* face_map)
{
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    auto cp = [](spuma_label* dst, const std::vector<int>& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(int));
    };
    cp(perm, m->h_perm);
    cp(owner, m->h_owner);
    cp(neighbour, m->h_neighbour);
    cp(owner_start, m->h_ownerStart);
    cp(losort, m->h_losort);
    cp(losort_start, m->h_losortStart);
    cp(face_map, m->h_face_map);
    return SPUMA_OK;
}

spuma_status spuma_mesh_get_geometry(spuma_mesh m, spuma_scalar* delta, spuma_scalar* weights, spuma_scalar* bdelta)
{
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    std::vector<double> d(m->F), w(m->F);
    SPUMA_CUDA(cudaMemcpy(d.data(), m->d_delta, sizeof(double) * m->F, cudaMemcpyDeviceToHost));
    SPUMA_CUDA(cudaMemcpy(w.data(), m->d_weights, sizeof(double) * m->F, cudaMemcpyDeviceToHost));
    for (int g = 0; g < m->F; ++g) {
        if (delta) delta[m->h_face_map[g]] = d[g];
        if (weights) weights[m->h_face_map[g]] = w[g];
    }
    if (bdelta && m->Fb) SPUMA_CUDA(cudaMemcpy(bdelta, m->d_bdelta, sizeof(double) * m->Fb, cudaMemcpyDeviceToHost));
    return SPUMA_OK;
}

spuma_status spuma_get_stats(spuma_mesh m, spuma_stats* out)
{
    if (!m || !out) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument");
    m->stats.timing_enabled = m->timing;
    m->stats.batch_iterations = m->batch;
    m->stats.amul_variant = resolve_amul_variant(m->amul_variant, mesh_args(m));
    *out = m->stats;
    return SPUMA_OK;
}

spuma_status spuma_reset_stats(spuma_mesh m)
{
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    const int g = m->stats.blocks_per_grid, t = m->stats.threads_per_block;
    m->stats = spuma_stats{};
    m->stats.blocks_per_grid = g;
    m->stats.threads_per_block = t;
    return SPUMA_OK;
}

spuma_status spuma_set_timing(spuma_mesh m, int enable)
{
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    m->timing = enable != 0;
    return SPUMA_OK;
}

spuma_status spuma_set_option(spuma_mesh m, int option, int value)
{
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    switch (option) {
    case SPUMA_OPT_FUSE_DIRECTION:
        if (value < 0 || value > 2) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "fuse_direction is 0, 1 or 2");
        if (m->fuse_direction != value) destroy_graphs(m);
        m->fuse_direction = value;
        return SPUMA_OK;
    case SPUMA_OPT_ELL_STENCIL:
        if (value < 0 || value > 1) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "ell_stencil is 0 or 1");
        if (m->ell_stencil != (value != 0)) destroy_graphs(m);
        m->ell_stencil = value != 0;
        return SPUMA_OK;
    case SPUMA_OPT_L2_PERSIST:
        if (value < 0 || value > 4) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "l2_persist is 0..4");
        if (m->l2_persist != value) destroy_graphs(m);
        m->l2_persist = value;
        if (!m->l2_persist) l2_reset(m);
        return SPUMA_OK;
    case SPUMA_OPT_GAMG_CSR:
        if (value < 0 || value > 1) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "gamg_csr is 0 or 1");
        if (m->gamg_csr != (value != 0)) gamg_release(m);  // the hierarchy is rebuilt at the next solve
        m->gamg_csr = value != 0;
        return SPUMA_OK;
    case SPUMA_OPT_PEER_POLL_MS:
        if (value < 1) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "peer_poll_ms must be >= 1");
        m->pst.poll_cycles = (long long)value * 2'000'000LL;
        destroy_graphs(m);  // the captured kernels (PCG batches, GAMG cycles) hold the old limit
        gamg_release(m);
        return SPUMA_OK;
    case SPUMA_OPT_ALT_SWEEP:
        if (value < 0 || value > 1) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "alt_sweep is 0 or 1");
        if (m->alt_sweep != (value != 0)) destroy_graphs(m);
        m->alt_sweep = value != 0;
        return SPUMA_OK;
    case SPUMA_OPT_GAMG_TAIL_CELLS:
        if (value < 0) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "negative GAMG tail size");
        m->gamg_tail_cells = value;  // the captured V-cycle is re-captured at the next solve
        return SPUMA_OK;
    case SPUMA_OPT_DEFER_PSI:
        if (value < 0 || value > 2) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "defer_psi is 0, 1 or 2");
        if (m->defer_psi != value) destroy_graphs(m);
        m->defer_psi = value;
        return SPUMA_OK;
    case SPUMA_OPT_PDL:
        if (g_use_pdl != (value != 0)) {
            destroy_graphs(m);
            if (m->gamg && m->gamg->gexec) {  // the captured V-cycle embeds the launch attribute too
                cudaGraphExecDestroy(m->gamg->gexec);
                m->gamg->gexec = nullptr;
            }
        }
        g_use_pdl = value != 0;
        return SPUMA_OK;
    case SPUMA_OPT_LOOP_PROFILE:
        if (value < 0 || value > 1) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "loop_profile is 0 or 1");
        m->loop_profile = value != 0;
        return SPUMA_OK;
    case SPUMA_OPT_LOOP_GRID:
        if (value < 0) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "loop grid must be >= 0");
        m->loop_ctas = value;
        return SPUMA_OK;
    case SPUMA_OPT_LOOP_L2:
        if (value < 0 || value > 4) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "loop_l2 is 0..4");
        m->loop_l2 = value;
        return SPUMA_OK;
    case SPUMA_OPT_PERSISTENT:
        if (value < 0 || value > 3) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "persistent is 0..3");
        m->persistent = value;
        return SPUMA_OK;
    case SPUMA_OPT_PEER_FUSED:
        if (value < 0 || value > 1) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "peer_fused is 0 or 1");
        if (m->peer_fused != (value != 0)) destroy_graphs(m);
        m->peer_fused = value != 0;
        return SPUMA_OK;
    case SPUMA_OPT_SMALL_SMEM:
        if (value < 0 || value > 1) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "small_smem is 0 or 1");
        m->small_smem = value != 0;
        return SPUMA_OK;
    case SPUMA_OPT_SMALL_SOLVE_MAX_CELLS:
        if (value < 0) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "small-solve threshold must be >= 0");
        m->small_max_cells = value;
        return SPUMA_OK;
    case SPUMA_OPT_AMUL_VARIANT:
        if (value < 0 || value > 13) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "amul variant must be 0..13");
        if (value != m->amul_variant) destroy_graphs(m);
        m->amul_variant = value;
        return SPUMA_OK;
    default: return set_error(SPUMA_ERR_INVALID_ARGUMENT, "unknown option");
    }
}

// ---------------------------------------------------------------------------
// peer-memory transport (peer.cu): blob = {IPC handle of the mailbox, rank, n_ranks, n_iface,
// processor patches (peer, offset, count)}; import maps every other rank's mailbox
// ---------------------------------------------------------------------------
namespace {
struct PeerBlob {
    cudaIpcMemHandle_t handle;
    int32_t magic, rank, n_ranks, n_iface, n_patches;
    int32_t peer[kMaxPeerPatches], offset[kMaxPeerPatches], count[kMaxPeerPatches];
};
static_assert(sizeof(PeerBlob) <= SPUMA_PEER_BLOB_BYTES, "peer blob too large");
constexpr int32_t kPeerMagic = 0x53504d41;  // "SPMA"

// mailbox layout (8-byte units): halo [2][n_iface] | partials [2][n_ranks][4] |
// halo flags [2][n_ranks] | partial flags [2][n_ranks]
inline size_t mail_units(int n_iface, int P) { return 2 * (size_t)n_iface + 12 * (size_t)P; }
}  // namespace

spuma_status spuma_peer_export(spuma_mesh m, void* blob)
{
    SPUMA_NVTX("spuma_peer_export");
    if (!m || !blob) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (m->n_ranks < 2) return set_error(SPUMA_ERR_STATE, "peer transport needs n_ranks > 1");
    if (m->n_ranks > kMaxPeerRanks || (int)m->cb_peers.size() > kMaxPeerPatches)
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "too many ranks or processor patches for the peer transport");
    if (!m->d_mail) {
        m->mail_units = mail_units(m->n_iface, m->n_ranks);
        SPUMA_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->d_mail), sizeof(double) * m->mail_units));
        SPUMA_CUDA(cudaMemset(m->d_mail, 0, sizeof(double) * m->mail_units));
        SPUMA_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->pst.ctr), 64));
        SPUMA_CUDA(cudaMemset(m->pst.ctr, 0, 64));
        m->pst.ticket = reinterpret_cast<unsigned*>(m->pst.ctr + 2);
        m->pst.err = reinterpret_cast<int*>(m->pst.ctr + 3);
        SPUMA_CUDA(cudaDeviceSynchronize());
    }
    PeerBlob b{};
    SPUMA_CUDA(cudaIpcGetMemHandle(&b.handle, m->d_mail));
    b.magic = kPeerMagic;
    b.rank = m->rank;
    b.n_ranks = m->n_ranks;
    b.n_iface = m->n_iface;
    b.n_patches = (int)m->cb_peers.size();
    for (int p = 0; p < b.n_patches; ++p) b.peer[p] = m->cb_peers[p], b.offset[p] = m->cb_offsets[p], b.count[p] = m->cb_counts[p];
    std::memset(blob, 0, SPUMA_PEER_BLOB_BYTES);
    std::memcpy(blob, &b, sizeof b);
    return SPUMA_OK;
}

spuma_status spuma_peer_import(spuma_mesh m, const void* blobs, int n_blobs)
{
    SPUMA_NVTX("spuma_peer_import");
    if (!m || !blobs) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!m->d_mail) return set_error(SPUMA_ERR_STATE, "spuma_peer_export first");
    if (m->peer) return set_error(SPUMA_ERR_STATE, "peer transport already imported on this handle");
    if (n_blobs != m->n_ranks) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "one blob per rank (rank order)");
    const int P = m->n_ranks;
    std::vector<PeerBlob> B(P);
    for (int r = 0; r < P; ++r) {
        std::memcpy(&B[r], static_cast<const char*>(blobs) + (size_t)r * SPUMA_PEER_BLOB_BYTES, sizeof(PeerBlob));
        if (B[r].magic != kPeerMagic || B[r].rank != r || B[r].n_ranks != P)
            return set_error(SPUMA_ERR_INVALID_ARGUMENT, "peer blob " + std::to_string(r) + " invalid or out of order");
    }
    std::vector<double*> base(P, nullptr);
    for (int r = 0; r < P; ++r) {
        if (r == m->rank) {
            base[r] = m->d_mail;
            continue;
        }
        void* p = nullptr;
        SPUMA_CUDA(cudaIpcOpenMemHandle(&p, B[r].handle, cudaIpcMemLazyEnablePeerAccess));
        m->peer_mapped.push_back(p);
        base[r] = static_cast<double*>(p);
    }
    auto halo = [&](int r, int par) { return base[r] + (size_t)par * B[r].n_iface; };
    auto part = [&](int r, int par) { return base[r] + 2 * (size_t)B[r].n_iface + (size_t)par * 4 * P; };
    auto hflag = [&](int r, int par) {
        return reinterpret_cast<unsigned long long*>(base[r] + 2 * (size_t)B[r].n_iface + 8 * (size_t)P) + par * P;
    };
    auto pflag = [&](int r, int par) {
        return reinterpret_cast<unsigned long long*>(base[r] + 2 * (size_t)B[r].n_iface + 10 * (size_t)P) + par * P;
    };
    PeerXfer& d = m->px;
    d = PeerXfer{};
    d.n_patches = (int)m->cb_peers.size();
    std::vector<int> used(P, 0);  // k-th patch of mine to rank q <-> k-th patch of q to me
    for (int p = 0; p < d.n_patches; ++p) {
        const int q = m->cb_peers[p];
        if (q < 0 || q >= P || q == m->rank) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "bad processor patch peer");
        int k = used[q]++, j = -1;
        for (int t = 0; t < B[q].n_patches; ++t)
            if (B[q].peer[t] == m->rank && k-- == 0) {
                j = t;
                break;
            }
        if (j < 0 || B[q].count[j] != m->cb_counts[p])
            return set_error(SPUMA_ERR_ADDRESSING, "processor patches of ranks " + std::to_string(m->rank) + " and " +
                                                       std::to_string(q) + " do not match");
        for (int par = 0; par < 2; ++par) {
            d.dst[p][par] = halo(q, par) + B[q].offset[j];
            d.dst_flag[p][par] = hflag(q, par) + m->rank;
            d.src[p][par] = halo(m->rank, par) + m->cb_offsets[p];
            d.src_flag[p][par] = hflag(m->rank, par) + q;
        }
    }
    PeerGather& g = m->pg;
    g = PeerGather{};
    g.n_ranks = P;
    g.rank = m->rank;
    for (int r = 0; r < P; ++r)
        for (int par = 0; par < 2; ++par) {
            g.part[r][par] = part(r, par);
            g.flag[r][par] = pflag(r, par);
        }
    for (int par = 0; par < 2; ++par) {
        g.my_part[par] = part(m->rank, par);
        g.my_flag[par] = pflag(m->rank, par);
    }
    // device copies for the fused PCG loop (halo inside k_direction / k_iface_rows, all-gather
    // inside the reductions' last CTA): the level-0 exchange and the gather descriptors, and the
    // processor patch of every interface face
    {
        PeerXfer x = d;
        for (int p = 0; p < x.n_patches; ++p) x.off[p] = m->cb_offsets[p], x.count[p] = m->cb_counts[p];
        std::vector<int> ifp(std::max(m->n_iface, 1), 0);
        for (int p = 0; p < x.n_patches; ++p)
            for (int i = 0; i < x.count[p]; ++i) ifp[x.off[p] + i] = p;
        SPUMA_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->d_px), sizeof(PeerXfer)));
        SPUMA_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->d_pg), sizeof(PeerGather)));
        SPUMA_CUDA(cudaMemcpy(m->d_px, &x, sizeof(PeerXfer), cudaMemcpyHostToDevice));
        SPUMA_CUDA(cudaMemcpy(m->d_pg, &g, sizeof(PeerGather), cudaMemcpyHostToDevice));
        SPUMA_TRY(upload(&m->d_if_patch, ifp, m->stream));
        SPUMA_CUDA(cudaStreamSynchronize(m->stream));
        m->ws.px = m->d_px;
        m->ws.pg = m->d_pg;
        m->ws.if_patch = m->d_if_patch;
    }
    m->peer = true;
    m->external_comm = false;  // graph-capturable from now on
    destroy_graphs(m);
    return SPUMA_OK;
}

spuma_status spuma_peer_check(spuma_mesh m)
{
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (!m->peer) return SPUMA_OK;
    int e = 0;
    SPUMA_CUDA(cudaMemcpy(&e, m->pst.err, sizeof e, cudaMemcpyDeviceToHost));
    if (e) return set_error(SPUMA_ERR_STATE, "peer transport: a neighbour did not answer within the poll limit");
    return SPUMA_OK;
}

spuma_status spuma_set_comm_callbacks(spuma_mesh m, const spuma_comm_callbacks* cb)
{
    if (!m || !cb || !cb->exchange || !cb->allgather) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL callbacks");
    if (!m->external_comm) return set_error(SPUMA_ERR_STATE, "handle uses NCCL (or n_ranks == 1)");
    m->cb = *cb;
    return SPUMA_OK;
}

spuma_status spuma_set_batch(spuma_mesh m, int iterations)
{
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (iterations < 1 || iterations > 256) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "batch out of range");
    m->batch = iterations;
    return SPUMA_OK;
}


void spuma_gamg_default_params(spuma_gamg_params* p)
{
    if (!p) return;
    p->n_pre_sweeps = 0;
    p->n_post_sweeps = 2;
    p->scale_correction = 1;
    p->n_cells_in_coarsest_level = 10;
    p->max_levels = 50;
    p->omega = 0.75;
    p->coarsest_tolerance = 0.0;
    p->coarsest_rel_tol = 1e-6;
    p->coarsest_max_iter = 1000;
    p->smoother = SPUMA_SMOOTHER_RICHARDSON;
    p->n_inner = 1;
}

static spuma_status gamg_check_params(const spuma_gamg_params& gp)
{
    if (gp.n_pre_sweeps < 0 || gp.n_post_sweeps < 0 || gp.max_levels < 1 || gp.coarsest_max_iter < 0 ||
        gp.n_inner < 0 || (gp.smoother != SPUMA_SMOOTHER_RICHARDSON && gp.smoother != SPUMA_SMOOTHER_GS2))
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "invalid GAMG parameters");
    return SPUMA_OK;
}

spuma_status spuma_gamg_solve(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                              const spuma_scalar* iface_coeffs, const spuma_scalar* source, spuma_scalar* psi,
                              const spuma_solver_controls* ctl, const spuma_gamg_params* params,
                              spuma_solver_perf* perf)
{
    SPUMA_NVTX("spuma_gamg_solve");
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (!ctl || !perf) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL controls/perf");
    if (m->N > 0 && (!diag || !source || !psi)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array");
    if (m->n_iface > 0 && !iface_coeffs) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "iface_coeffs is NULL");
    if (m->F > 0 && !upper) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "upper is NULL");
    if (ctl->max_iter < 0 || ctl->min_iter < 0) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "negative iteration limit");
    spuma_gamg_params gp;
    spuma_gamg_default_params(&gp);
    if (params) gp = *params;
    SPUMA_TRY(gamg_check_params(gp));
    if (m->N == 0 && m->n_ranks == 1) {
        *perf = spuma_solver_perf{};
        return SPUMA_OK;
    }
    cudaStream_t s = m->stream;
    DevPtrs P{};
    const double* psi_in = nullptr;
    SPUMA_TRY(cells_in(m, diag, R_DIAG, &P.diag));
    SPUMA_TRY(faces_in(m, upper, &P.upper));
    SPUMA_TRY(cells_in(m, source, R_SOURCE, &P.source));
    SPUMA_TRY(cells_in(m, psi, R_PSI, &psi_in));
    P.psi = const_cast<double*>(psi_in);
    if (m->n_iface) SPUMA_TRY(iface_in(m, iface_coeffs, &P.iface));
    SPUMA_TRY(gamg_ensure(m, gp));
    const bool dd = m->gamg->dd;
    GamgState* G = m->gamg;
    const int nl = (int)G->lv.size();
    *m->h_ptrs = P;
    SPUMA_CUDA(cudaMemcpyAsync(m->ws.ptrs, m->h_ptrs, sizeof(DevPtrs), cudaMemcpyHostToDevice, s));
    const GLevel& Lc = G->lv[nl - 1];
    *G->h_cptrs = DevPtrs{nl == 1 ? P.diag : Lc.diag, nl == 1 ? P.upper : Lc.upper, nl == 1 ? P.iface : Lc.iface,
                          Lc.b ? Lc.b : m->ws.rA, Lc.x};
    SPUMA_CUDA(cudaMemcpyAsync(G->cws.ptrs, G->h_cptrs, sizeof(DevPtrs), cudaMemcpyHostToDevice, s));
    // per-solve: Galerkin coarse matrices (Q27), outer scalars, coarsest PCG controls, A6 setup
    if (G->lv[0].cval) {  // level 0 over CSR runs: this call's coefficients into them
        launch_gamg_csr_values(s, G->lv[0], P.upper, m->F);
        m->stats.kernel_launches += 1;
    }
    for (int l = 0; l + 1 < nl; ++l) launch_gamg_agg(s, G->lv[l], G->lv[l + 1], m->ws.ptrs);
    if (G->lv[0].ell) {  // level 0 rows over ELL: this call's coefficients in owner-slot order
        launch_ell_coeffs(s, G->lv[0].a, P.upper, m->d_upper_s);
        m->stats.kernel_launches += 1;
    }
    launch_scal_init(s, m->ws, *ctl, dd ? m->n_ranks : 1);
    const spuma_solver_controls cc{gp.coarsest_tolerance, gp.coarsest_rel_tol, gp.coarsest_max_iter, 0};
    launch_scal_init(s, G->cws, cc, 1);
    if (dd) {  // A6 over the ranks: normFactor, initial residual (interface terms after the psi halo)
        const MeshArgs a0 = mesh_args(m);
        SPUMA_TRY(halo_exchange(m, P.psi, m->ws.xr, s));
        launch_setup1(s, m->grid, a0, m->ws, false);
        SPUMA_TRY(reduce_finalize(m, 1, s));
        launch_setup2(s, m->grid, a0, m->ws, false);
        SPUMA_TRY(reduce_finalize(m, 2, s));
    } else {
        const MeshArgs a0 = G->lv[0].a;
        launch_setup1(s, m->grid, a0, m->ws, true);
        launch_setup2(s, m->grid, a0, m->ws, true);
    }
    m->stats.kernel_launches += (uint64_t)(nl - 1) + 4;

    // one V-cycle per graph launch (nl == 1 or a decomposed mesh: direct launches)
    const bool use_graph = nl > 1 && !dd;
    if (use_graph && (!G->gexec || std::memcmp(&G->gkey, &gp, sizeof gp) != 0 || G->gkey_tail != m->gamg_tail_cells)) {
        if (G->gexec) cudaGraphExecDestroy(G->gexec);
        G->gexec = nullptr;
        cudaGraph_t graph = nullptr;
        SPUMA_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        G->launches_per_cycle = gamg_enqueue_cycle(m, gp, s);
        cudaError_t e = cudaStreamEndCapture(s, &graph);
        SPUMA_CUDA(e);
        e = cudaGraphInstantiate(&G->gexec, graph, 0);
        cudaGraphDestroy(graph);
        SPUMA_CUDA(e);
        G->gkey = gp;
        G->gkey_tail = m->gamg_tail_cells;
    }
    SPUMA_CUDA(cudaMemcpyAsync(&m->h_scal[0], m->ws.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    int cycles = 0;
    while (!m->h_scal[0].done) {
        if (use_graph) {
            SPUMA_CUDA(cudaGraphLaunch(G->gexec, s));
        } else {
            spuma_status st = SPUMA_OK;
            G->launches_per_cycle = gamg_enqueue_cycle(m, gp, s, &st);
            if (st != SPUMA_OK) return st;
        }
        SPUMA_CUDA(cudaMemcpyAsync(&m->h_scal[0], m->ws.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
        SPUMA_CUDA(cudaStreamSynchronize(s));
        if (++cycles > iter_bound(ctl) + 1) return set_error(SPUMA_ERR_STATE, "GAMG loop did not terminate");
    }
    SPUMA_CUDA(cudaGetLastError());
    m->stats.kernel_launches += (uint64_t)cycles * (uint64_t)G->launches_per_cycle;
    const DevScal fs = m->h_scal[0];
    perf->initial_residual = fs.init;
    perf->final_residual = fs.fin;
    perf->n_iterations = fs.n;
    perf->converged = fs.converged;
    perf->singular = 0;
    m->stats.solves += 1;
    m->stats.iterations += fs.n;
    SPUMA_TRY(cells_out(m, psi, P.psi));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    return peer_guard(m);
}

spuma_status spuma_gamg_get_hierarchy(spuma_mesh m, const spuma_gamg_params* params, int max_levels,
                                      int* n_levels, int* level_cells, int* level_faces, int level,
                                      spuma_label* ftc)
{
    if (!m || !n_levels) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument");
    spuma_gamg_params gp;
    spuma_gamg_default_params(&gp);
    if (params) gp = *params;
    else if (m->gamg) gp.n_cells_in_coarsest_level = m->gamg->n_coarsest, gp.max_levels = m->gamg->max_levels;
    SPUMA_TRY(gamg_check_params(gp));
    SPUMA_TRY(gamg_ensure(m, gp));  // collective on a decomposed mesh when the hierarchy is (re)built
    const GamgState* G = m->gamg;
    const int nl = (int)G->lv.size();
    *n_levels = nl;
    for (int l = 0; l < nl && l < max_levels; ++l) {
        if (level_cells) level_cells[l] = G->cells[l];
        if (level_faces) level_faces[l] = G->faces[l];
    }
    if (ftc) {
        if (level < 0 || level >= nl - 1) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "level has no coarser level");
        std::memcpy(ftc, G->ftc[level].data(), sizeof(int) * G->ftc[level].size());
    }
    return SPUMA_OK;
}

spuma_status spuma_pcg_solve_pc(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                                const spuma_scalar* iface_coeffs, const spuma_scalar* source, spuma_scalar* psi,
                                const spuma_solver_controls* ctl, const spuma_preconditioner* pcp,
                                spuma_solver_perf* perf)
{
    SPUMA_NVTX("spuma_pcg_solve_pc");
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (!ctl || !perf) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL controls/perf");
    if (m->N > 0 && (!diag || !source || !psi)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array");
    if (m->F > 0 && !upper) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "upper is NULL");
    if (m->n_iface > 0 && !iface_coeffs) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "iface_coeffs is NULL");
    if (ctl->max_iter < 0 || ctl->min_iter < 0) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "negative iteration limit");
    const spuma_preconditioner pc = pcp ? *pcp : spuma_preconditioner{SPUMA_PC_DIAGONAL, 0};
    SPUMA_TRY(pc_check(m, pc, true));
    if (m->N == 0 && m->n_ranks == 1) {
        *perf = spuma_solver_perf{};
        return SPUMA_OK;
    }
    SPUMA_TRY(pc_ensure(m));
    cudaStream_t s = m->stream;
    DevPtrs Pp{};
    const double* psi_in = nullptr;
    SPUMA_TRY(cells_in(m, diag, R_DIAG, &Pp.diag));
    SPUMA_TRY(faces_in(m, upper, &Pp.upper));
    SPUMA_TRY(cells_in(m, source, R_SOURCE, &Pp.source));
    SPUMA_TRY(cells_in(m, psi, R_PSI, &psi_in));
    Pp.psi = const_cast<double*>(psi_in);
    if (m->n_iface) SPUMA_TRY(iface_in(m, iface_coeffs, &Pp.iface));
    *m->h_ptrs = Pp;
    SPUMA_CUDA(cudaMemcpyAsync(m->ws.ptrs, m->h_ptrs, sizeof(DevPtrs), cudaMemcpyHostToDevice, s));
    launch_scal_init(s, m->ws, *ctl, m->n_ranks);
    const MeshArgs a = mesh_args(m);
    const bool fin = m->n_ranks == 1;
    prepare_amul_coeffs(m, s, a, Pp.upper);
    SPUMA_TRY(halo_exchange(m, Pp.psi, m->ws.xr, s));
    launch_setup1(s, m->grid, a, m->ws, fin);
    if (!fin) SPUMA_TRY(reduce_finalize(m, 1, s));
    launch_setup2(s, m->grid, a, m->ws, fin);
    if (!fin) SPUMA_TRY(reduce_finalize(m, 2, s));
    pc_setup(m, pc, Pp.diag, Pp.upper, Pp.upper);  // processor-local factorisation (Q31)
    m->stats.kernel_launches += 5;
    PcState* P = m->pc;
    Workspace w = m->ws;
    SPUMA_CUDA(cudaMemcpyAsync(&m->h_scal[0], w.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    // external comm (host callbacks): one iteration per check; otherwise 8 (no-op kernels past
    // 'done'; every rank runs the same launches and collectives)
    const int per_check = m->external_comm ? 1 : 8;
    int it = 0;
    while (!m->h_scal[0].done) {
        for (int b = 0; b < per_check; ++b) {
            pc_apply(m, pc, Pp.upper, Pp.upper, w.rA, w.wA, false, w.scal);
            launch_pc_dot(s, m->N, w.wA, w.rA, P->part, w.scal, fin);
            if (!fin) SPUMA_TRY(reduce_finalize(m, 5, s));
            launch_pc_direction(s, m->N, w.wA, w.pA, nullptr, nullptr, w.scal);
            SPUMA_TRY(halo_exchange(m, w.pA, w.xr, s));
            launch_amul_dot(s, m->amul_variant, a, w, fin, m->sell_wn, m->sell_wo);
            if (!fin) SPUMA_TRY(reduce_finalize(m, 3, s));
            launch_update(s, m->grid, a, w, fin, 0);
            if (!fin) SPUMA_TRY(reduce_finalize(m, 4, s));
            m->stats.kernel_launches += pc_launches(pc) + 4;
        }
        SPUMA_CUDA(cudaMemcpyAsync(&m->h_scal[0], w.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
        SPUMA_CUDA(cudaStreamSynchronize(s));
        it += per_check;
        if (it > iter_bound(ctl) + 16) return set_error(SPUMA_ERR_STATE, "PCG loop did not terminate");
    }
    SPUMA_CUDA(cudaGetLastError());
    SPUMA_TRY(pc_guard(m));
    const DevScal fs = m->h_scal[0];
    perf->initial_residual = fs.init;
    perf->final_residual = fs.fin;
    perf->n_iterations = fs.n;
    perf->converged = fs.converged;
    perf->singular = fs.singular;
    m->stats.solves += 1;
    m->stats.iterations += fs.n;
    SPUMA_TRY(cells_out(m, psi, Pp.psi));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    return peer_guard(m);
}

spuma_status spuma_pbicg_solve(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                               const spuma_scalar* lower, const spuma_scalar* iface_coeffs,
                               const spuma_scalar* iface_coeffs_t, const spuma_scalar* source, spuma_scalar* psi,
                               const spuma_solver_controls* ctl, const spuma_preconditioner* pcp,
                               spuma_solver_perf* perf)
{
    SPUMA_NVTX("spuma_pbicg_solve");
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (!ctl || !perf) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL controls/perf");
    if (m->N > 0 && (!diag || !source || !psi)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array");
    if (m->F > 0 && (!upper || !lower)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "upper/lower is NULL");
    if (m->n_iface > 0 && (!iface_coeffs || !iface_coeffs_t))
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "iface_coeffs / iface_coeffs_t is NULL");
    if (ctl->max_iter < 0 || ctl->min_iter < 0) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "negative iteration limit");
    const spuma_preconditioner pc = pcp ? *pcp : spuma_preconditioner{SPUMA_PC_ADILU, 2};
    SPUMA_TRY(pc_check(m, pc, true));
    if (m->N == 0 && m->n_ranks == 1) {
        *perf = spuma_solver_perf{};
        return SPUMA_OK;
    }
    SPUMA_TRY(pc_ensure(m));
    PcState* P = m->pc;
    cudaStream_t s = m->stream;
    const bool fin = m->n_ranks == 1;
    const double *d_i, *s_i, *psi_c, *u_i, *l_i, *if_i = nullptr, *ift_i = nullptr;
    SPUMA_TRY(cells_in(m, diag, R_DIAG, &d_i));
    SPUMA_TRY(cells_in(m, source, R_SOURCE, &s_i));
    SPUMA_TRY(cells_in(m, psi, R_PSI, &psi_c));
    SPUMA_TRY(pair_in(m, upper, lower, &u_i, &l_i));
    if (m->n_iface) {
        SPUMA_TRY(iface_in(m, iface_coeffs, &if_i));
        if (!P->iface_t) SPUMA_TRY(dalloc(&P->iface_t, m->n_iface));
        if (!P->xrT) SPUMA_TRY(dalloc(&P->xrT, m->n_iface));
        if (is_device_ptr(iface_coeffs_t)) ift_i = iface_coeffs_t;
        else {
            SPUMA_CUDA(cudaMemcpyAsync(P->iface_t, iface_coeffs_t, sizeof(double) * m->n_iface, cudaMemcpyHostToDevice,
                                       s));
            ift_i = P->iface_t;
        }
    }
    double* psi_i = const_cast<double*>(psi_c);
    Workspace w = m->ws;
    const MeshArgs a = mesh_args(m);
    launch_scal_init(s, w, *ctl, m->n_ranks);
    SPUMA_TRY(halo_exchange(m, psi_i, w.xr, s));
    launch_bicg_setup1(s, a, d_i, u_i, l_i, if_i, ift_i, w.xr, s_i, psi_i, w.wA, P->wT, w.rA, P->rT, w.sumA, P->part,
                       w.scal, fin);
    if (!fin) SPUMA_TRY(reduce_finalize(m, 1, s));
    launch_pc_setup2(s, m->N, w.wA, w.sumA, s_i, w.rA, P->part, w.scal, fin);
    if (!fin) SPUMA_TRY(reduce_finalize(m, 2, s));
    pc_setup(m, pc, d_i, u_i, l_i);  // processor-local (Q31)
    m->stats.kernel_launches += 4;
    SPUMA_CUDA(cudaMemcpyAsync(&m->h_scal[0], w.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    const int per_check = m->external_comm ? 1 : 8;
    int it = 0;
    while (!m->h_scal[0].done) {
        for (int b = 0; b < per_check; ++b) {
            pc_apply(m, pc, u_i, l_i, w.rA, w.wA, false, w.scal);
            pc_apply(m, pc, u_i, l_i, P->rT, P->wT, true, w.scal);
            launch_pc_dot(s, m->N, w.wA, P->rT, P->part, w.scal, fin);
            if (!fin) SPUMA_TRY(reduce_finalize(m, 5, s));
            launch_pc_direction(s, m->N, w.wA, w.pA, P->wT, P->pT, w.scal);
            SPUMA_TRY(halo_exchange(m, w.pA, w.xr, s));
            SPUMA_TRY(halo_exchange(m, P->pT, P->xrT, s));
            launch_bicg_amul_tmul(s, a, d_i, u_i, l_i, if_i, ift_i, w.pA, P->pT, w.xr, P->xrT, w.wA, P->wT, P->part,
                                  w.scal, fin);
            if (!fin) SPUMA_TRY(reduce_finalize(m, 3, s));
            launch_bicg_update(s, m->N, psi_i, w.pA, w.rA, w.wA, P->rT, P->wT, P->part, w.scal, fin);
            if (!fin) SPUMA_TRY(reduce_finalize(m, 4, s));
            m->stats.kernel_launches += 2 * pc_launches(pc) + 4;
        }
        SPUMA_CUDA(cudaMemcpyAsync(&m->h_scal[0], w.scal, sizeof(DevScal), cudaMemcpyDeviceToHost, s));
        SPUMA_CUDA(cudaStreamSynchronize(s));
        it += per_check;
        if (it > iter_bound(ctl) + 16) return set_error(SPUMA_ERR_STATE, "PBiCG loop did not terminate");
    }
    SPUMA_CUDA(cudaGetLastError());
    SPUMA_TRY(pc_guard(m));
    const DevScal fs = m->h_scal[0];
    perf->initial_residual = fs.init;
    perf->final_residual = fs.fin;
    perf->n_iterations = fs.n;
    perf->converged = fs.converged;
    perf->singular = fs.singular;
    m->stats.solves += 1;
    m->stats.iterations += fs.n;
    SPUMA_TRY(cells_out(m, psi, psi_i));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    return peer_guard(m);
}

spuma_status spuma_precondition(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                                const spuma_scalar* lower, const spuma_preconditioner* pcp, const spuma_scalar* r,
                                spuma_scalar* wout, int transpose)
{
    SPUMA_NVTX("spuma_precondition");
    if (!m || !pcp) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (m->N > 0 && (!diag || !r || !wout)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array");
    if (m->F > 0 && !upper) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "upper is NULL");
    SPUMA_TRY(pc_check(m, *pcp));
    if (m->N == 0) return SPUMA_OK;
    SPUMA_TRY(pc_ensure(m));
    cudaStream_t s = m->stream;
    const double *d_i, *r_i, *u_i, *l_i;
    SPUMA_TRY(cells_in(m, diag, R_DIAG, &d_i));
    SPUMA_TRY(cells_in(m, r, R_X, &r_i));
    SPUMA_TRY(pair_in(m, upper, lower, &u_i, &l_i));
    pc_setup(m, *pcp, d_i, u_i, l_i);
    if (!m->d_cell_t) SPUMA_TRY(dalloc(&m->d_cell_t, m->N));
    pc_apply(m, *pcp, u_i, l_i, r_i, m->d_cell_t, transpose != 0, nullptr);
    m->stats.kernel_launches += 2 + pc_launches(*pcp);
    SPUMA_CUDA(cudaStreamSynchronize(s));
    SPUMA_TRY(pc_guard(m));
    SPUMA_TRY(cells_out(m, wout, m->d_cell_t));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    SPUMA_CUDA(cudaGetLastError());
    return SPUMA_OK;
}

spuma_status spuma_amul_asym(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                             const spuma_scalar* lower, const spuma_scalar* x, spuma_scalar* y, int transpose)
{
    SPUMA_NVTX("spuma_amul_asym");
    if (!m) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (m->N > 0 && (!diag || !x || !y)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL array");
    if (m->F > 0 && (!upper || !lower)) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "upper/lower is NULL");
    if (m->N == 0) return SPUMA_OK;
    SPUMA_TRY(pc_ensure(m));
    cudaStream_t s = m->stream;
    const double *d_i, *x_i, *u_i, *l_i;
    SPUMA_TRY(cells_in(m, diag, R_DIAG, &d_i));
    SPUMA_TRY(cells_in(m, x, R_X, &x_i));
    SPUMA_TRY(pair_in(m, upper, lower, &u_i, &l_i));
    if (!m->d_cell_t) SPUMA_TRY(dalloc(&m->d_cell_t, m->N));
    launch_amul_asym(s, mesh_args(m), d_i, u_i, l_i, x_i, m->d_cell_t, transpose != 0);
    m->stats.kernel_launches += 1;
    SPUMA_TRY(cells_out(m, y, m->d_cell_t));
    SPUMA_CUDA(cudaStreamSynchronize(s));
    SPUMA_CUDA(cudaGetLastError());
    return SPUMA_OK;
}

spuma_status spuma_ldu_to_csr(spuma_mesh m, spuma_label* row_ptr, spuma_label* col, spuma_label* map)
{
    if (!m || !row_ptr || !col || !map) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (m->renumber) return set_error(SPUMA_ERR_STATE, "LDU->CSR needs a handle built with renumber = 0");
    std::vector<int> rp, cl, mp;
    ldu_to_csr_host(m->N, m->F, m->h_owner, m->h_neighbour, m->h_ownerStart, m->h_losortStart, m->h_losort, rp, cl,
                    mp);
    const int nnz = m->N + 2 * m->F;
    auto put = [&](spuma_label* dst, const std::vector<int>& v) -> spuma_status {
        if (is_device_ptr(dst)) SPUMA_CUDA(cudaMemcpy(dst, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice));
        else std::memcpy(dst, v.data(), sizeof(int) * v.size());
        return SPUMA_OK;
    };
    SPUMA_TRY(put(row_ptr, rp));
    SPUMA_TRY(put(col, cl));
    SPUMA_TRY(put(map, mp));
    SPUMA_TRY(pc_ensure(m));
    if (!m->pc->csr_map) SPUMA_TRY(upload(&m->pc->csr_map, mp, m->stream));
    m->pc->nnz = nnz;
    SPUMA_CUDA(cudaStreamSynchronize(m->stream));
    return SPUMA_OK;
}

spuma_status spuma_csr_values(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                              const spuma_scalar* lower, spuma_scalar* values)
{
    SPUMA_NVTX("spuma_csr_values");
    if (!m || !diag || !values || (m->F > 0 && (!upper || !lower)))
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!m->pc || !m->pc->csr_map) return set_error(SPUMA_ERR_STATE, "call spuma_ldu_to_csr first");
    if (!is_device_ptr(diag) || !is_device_ptr(upper) || !is_device_ptr(lower) || !is_device_ptr(values))
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "spuma_csr_values takes device arrays");
    launch_csr_values(m->stream, m->pc->nnz, m->N, m->F, m->pc->csr_map, diag, upper, lower, values);
    m->stats.kernel_launches += 1;
    SPUMA_CUDA(cudaStreamSynchronize(m->stream));
    SPUMA_CUDA(cudaGetLastError());
    return SPUMA_OK;
}

// ---------------- host-only diagnostics (no device access; CPU-testable host logic) ----------------
static spuma_status host_addressing(int n, int F, const spuma_label* owner, const spuma_label* neighbour,
                                    std::vector<int>& o, std::vector<int>& nb, std::vector<int>& os,
                                    std::vector<int>& ls, std::vector<int>& lo, std::vector<int>& olo)
{
    if (n < 0 || F < 0 || (F > 0 && (!owner || !neighbour))) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "bad sizes");
    std::string why;
    if (!valid_addressing(n, F, owner, neighbour, &why)) return set_error(SPUMA_ERR_ADDRESSING, why);
    o.assign(owner, owner + F);
    nb.assign(neighbour, neighbour + F);
    derived_addressing(n, F, o.data(), nb.data(), os, lo, ls, olo);
    return SPUMA_OK;
}

spuma_status spuma_host_rcm(int n_cells, int n_faces, const spuma_label* owner, const spuma_label* neighbour,
                            spuma_label* perm)
{
    std::vector<int> o, nb, os, ls, lo, olo;
    SPUMA_TRY(host_addressing(n_cells, n_faces, owner, neighbour, o, nb, os, ls, lo, olo));
    if (!perm) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "perm is NULL");
    const std::vector<int> p = rcm_permutation(n_cells, n_faces, owner, neighbour);
    std::memcpy(perm, p.data(), sizeof(int) * p.size());
    return SPUMA_OK;
}

spuma_status spuma_host_lattice_offsets(int n_cells, int n_faces, const spuma_label* owner,
                                        const spuma_label* neighbour, int* n_offsets, int* offsets)
{
    std::vector<int> o, nb, os, ls, lo, olo;
    SPUMA_TRY(host_addressing(n_cells, n_faces, owner, neighbour, o, nb, os, ls, lo, olo));
    if (!n_offsets || !offsets) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL output");
    int D[3] = {0, 0, 0};
    *n_offsets = n_faces > 0 ? lattice_offsets(n_cells, n_faces, owner, neighbour, D) : 0;
    for (int t = 0; t < 3; ++t) offsets[t] = t < *n_offsets ? D[t] : 0;
    return SPUMA_OK;
}

spuma_status spuma_host_gamg_hierarchy(int n_cells, int n_faces, const spuma_label* owner,
                                       const spuma_label* neighbour, const spuma_scalar* face_weights,
                                       int n_coarsest, int max_levels, int max_out, int* n_levels,
                                       int* level_cells, int* level_faces, spuma_label* ftc)
{
    std::vector<int> o, nb, os, ls, lo, olo;
    SPUMA_TRY(host_addressing(n_cells, n_faces, owner, neighbour, o, nb, os, ls, lo, olo));
    if (!n_levels || (n_faces > 0 && !face_weights) || max_levels < 1)
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument / max_levels < 1");
    std::vector<double> w(face_weights, face_weights + n_faces);
    const std::vector<GamgHostLevel> H = gamg_hierarchy(n_cells, n_faces, o, nb, os, ls, lo, olo, w, n_coarsest,
                                                        max_levels);
    *n_levels = (int)H.size();
    size_t off = 0;
    for (int l = 0; l < (int)H.size(); ++l) {
        if (l < max_out) {
            if (level_cells) level_cells[l] = H[l].n;
            if (level_faces) level_faces[l] = H[l].F;
        }
        if (ftc && l + 1 < (int)H.size()) {  // concatenated fine-to-coarse maps of every level but the coarsest
            std::memcpy(ftc + off, H[l].ftc.data(), sizeof(int) * H[l].ftc.size());
            off += H[l].ftc.size();
        }
    }
    return SPUMA_OK;
}

namespace {
// in-process transport of spuma_host_gamg_hierarchy_dd: one thread per rank, a shared gather
// array and a mailbox per (source, destination, k-th patch between them), barrier-separated
struct SimComm {
    int P = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long gen = 0;
    std::vector<double> gather;
    std::map<std::tuple<int, int, int>, std::vector<double>> box;
    void barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        const long long g = gen;
        if (++arrived == P) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
struct SimRank {
    SimComm* sc;
    int rank;
    std::vector<int> peers;
};
bool sim_allgather4(void* ctx, const double* in, double* out)
{
    SimRank* r = static_cast<SimRank*>(ctx);
    {
        std::lock_guard<std::mutex> lk(r->sc->mu);
        std::copy(in, in + 4, r->sc->gather.begin() + 4 * r->rank);
    }
    r->sc->barrier();
    {
        std::lock_guard<std::mutex> lk(r->sc->mu);
        std::copy(r->sc->gather.begin(), r->sc->gather.end(), out);
    }
    r->sc->barrier();
    return true;
}
bool sim_exchange(void* ctx, const std::vector<int>& counts, const std::vector<double>& send, std::vector<double>& recv)
{
    SimRank* r = static_cast<SimRank*>(ctx);
    std::map<int, int> kth;
    {
        std::lock_guard<std::mutex> lk(r->sc->mu);
        int off = 0;
        for (size_t p = 0; p < counts.size(); ++p) {
            const int q = r->peers[p], k = kth[q]++;
            r->sc->box[std::make_tuple(r->rank, q, k)] =
                std::vector<double>(send.begin() + off, send.begin() + off + counts[p]);
            off += counts[p];
        }
    }
    r->sc->barrier();
    kth.clear();
    {
        std::lock_guard<std::mutex> lk(r->sc->mu);
        recv.assign(send.size(), 0.0);
        int off = 0;
        for (size_t p = 0; p < counts.size(); ++p) {
            const int q = r->peers[p], k = kth[q]++;
            const std::vector<double>& v = r->sc->box[std::make_tuple(q, r->rank, k)];
            if ((int)v.size() != counts[p]) return false;
            std::copy(v.begin(), v.end(), recv.begin() + off);
            off += counts[p];
        }
    }
    r->sc->barrier();
    return true;
}
}  // namespace

spuma_status spuma_host_gamg_hierarchy_dd(int n_ranks, const int* n_cells, const int* n_faces,
                                          const spuma_label* const* owner, const spuma_label* const* neighbour,
                                          const spuma_scalar* const* face_weights, const int* n_patches,
                                          const int* const* patch_peer, const int* const* patch_count,
                                          const spuma_label* const* if_cell, int n_coarsest, int max_levels,
                                          int* n_levels, int* level_cells, int* level_ifaces)
{
    if (n_ranks < 1 || !n_cells || !n_faces || !owner || !neighbour || !face_weights || !n_patches || !n_levels ||
        max_levels < 1)
        return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument / n_ranks < 1 / max_levels < 1");
    SimComm sc;
    sc.P = n_ranks;
    sc.gather.assign(4 * (size_t)n_ranks, 0.0);
    std::vector<SimRank> ranks(n_ranks);
    std::vector<std::vector<GamgHostLevel>> H(n_ranks);
    std::vector<spuma_status> st(n_ranks, SPUMA_OK);
    std::vector<std::string> err(n_ranks);
    auto work = [&](int r) {
        std::vector<int> o, nb, os, ls, lo, olo;
        st[r] = host_addressing(n_cells[r], n_faces[r], owner[r], neighbour[r], o, nb, os, ls, lo, olo);
        if (st[r] != SPUMA_OK) err[r] = spuma_last_error();
        std::vector<double> w(face_weights[r], face_weights[r] + n_faces[r]);
        std::vector<int> counts(patch_count[r], patch_count[r] + n_patches[r]);
        int n_if = 0;
        for (int c : counts) n_if += c;
        std::vector<int> ic(if_cell[r], if_cell[r] + n_if);
        ranks[r] = SimRank{&sc, r, std::vector<int>(patch_peer[r], patch_peer[r] + n_patches[r])};
        GamgComm comm;
        comm.n_ranks = n_ranks;
        comm.allgather4 = sim_allgather4;
        comm.exchange = sim_exchange;
        comm.ctx = &ranks[r];
        bool ok = true;
        H[r] = gamg_hierarchy_dd(n_cells[r], n_faces[r], o, nb, os, ls, lo, olo, w, ic, counts, n_coarsest, max_levels,
                                 comm, &ok);
        if (!ok && st[r] == SPUMA_OK) st[r] = SPUMA_ERR_NCCL;
    };
    // every rank must run (the collectives are lockstep), so validation errors are reported after
    std::vector<std::thread> th;
    for (int r = 0; r < n_ranks; ++r) th.emplace_back(work, r);
    for (auto& t : th) t.join();
    for (int r = 0; r < n_ranks; ++r)
        if (st[r] != SPUMA_OK) return set_error(st[r], "rank " + std::to_string(r) + ": " + err[r]);
    *n_levels = (int)H[0].size();
    for (int r = 0; r < n_ranks; ++r) {
        if ((int)H[r].size() != *n_levels) return set_error(SPUMA_ERR_STATE, "ranks disagree on the level count");
        for (int l = 0; l < (int)H[r].size() && l < 64; ++l) {
            if (level_cells) level_cells[64 * r + l] = H[r][l].n;
            if (level_ifaces) level_ifaces[64 * r + l] = (int)H[r][l].if_cell.size();
        }
    }
    return SPUMA_OK;
}

spuma_status spuma_host_level_schedule(int n_cells, int n_faces, const spuma_label* owner,
                                       const spuma_label* neighbour, spuma_label* order_f, spuma_label* order_b,
                                       int* depth_f, int* depth_b)
{
    std::vector<int> o, nb, os, ls, lo, olo;
    SPUMA_TRY(host_addressing(n_cells, n_faces, owner, neighbour, o, nb, os, ls, lo, olo));
    if (!order_f || !order_b || !depth_f || !depth_b) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument");
    std::vector<int> of, ob;
    int wf, wb;
    level_schedule(n_cells, o, nb, os, ls, lo, of, ob, *depth_f, *depth_b, wf, wb);
    std::memcpy(order_f, of.data(), sizeof(int) * of.size());
    std::memcpy(order_b, ob.data(), sizeof(int) * ob.size());
    return SPUMA_OK;
}

spuma_status spuma_host_ldu_to_csr(int n_cells, int n_faces, const spuma_label* owner, const spuma_label* neighbour,
                                   spuma_label* row_ptr, spuma_label* col, spuma_label* map)
{
    std::vector<int> o, nb, os, ls, lo, olo;
    SPUMA_TRY(host_addressing(n_cells, n_faces, owner, neighbour, o, nb, os, ls, lo, olo));
    if (!row_ptr || !col || !map) return set_error(SPUMA_ERR_INVALID_ARGUMENT, "NULL argument");
    std::vector<int> rp, cl, mp;
    ldu_to_csr_host(n_cells, n_faces, o, nb, os, ls, lo, rp, cl, mp);
    std::memcpy(row_ptr, rp.data(), sizeof(int) * rp.size());
    std::memcpy(col, cl.data(), sizeof(int) * cl.size());
    std::memcpy(map, mp.data(), sizeof(int) * mp.size());
    return SPUMA_OK;
}

}  // extern "C"
