// internal.h -- libspuma internals (not part of the C-ABI; see include/spuma.h).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges are no-ops unless a profiler is attached

#include <cstdint>
#include <string>
#include <vector>

#include "spuma.h"

namespace spuma {

constexpr int kThreads = 256;      // threads per CTA of every cell/face kernel (8 warps)
constexpr int kSmallThreads = 1024;  // the single-CTA solves (small meshes, GAMG coarsest level / tail)
constexpr int kMaxPartials = 4;    // reduction values per kernel
constexpr int kPhases = 4;         // timing phases (spuma_stats.phase_ms)

// Device-resident PCG state (A6-A12).  Written only by the finalisation code
// (last CTA of a reduction kernel, or the 1-CTA finalise kernel when P > 1).
struct DevScal {
    double wArA, wArAold, wApA, alpha, beta, alpha_prev;
    double alpha_prev2;    // alpha of the iteration before alpha_prev (psi updates in the direction)
    double normFactor, init, fin, xbar;
    double tol, rel_tol;
    double rank_part[4];   // this rank's partial sums of the current reduction (P > 1)
    int n, done, singular, converged;
    int max_iter, min_iter, n_ranks;
    int psi_done;          // psi updates applied so far (SPUMA_OPT_DEFER_PSI = 2: by k_direction)
    unsigned int ticket[8];
};

// Per-call pointers of the hot loop (device copy read by the captured kernels,
// so one captured graph serves every spuma_pcg_solve call on the handle).
struct DevPtrs {
    const double* diag;
    const double* upper;
    const double* iface;
    const double* source;
    double* psi;
};

// Mesh-constant kernel arguments (captured by value).
struct MeshArgs {
    int N, F;
    const int* ownerStart;   // [N+1]
    const int* losortStart;  // [N+1]
    const int* losort;       // [F]  faces sorted by neighbour (stable)
    const int* ownerLo;      // [F]  owner[losort[k]]
    const int* neighbour;    // [F]
    const int* owner;        // [F]
    // processor interfaces, per cell in (patch, face) order
    const int* ifStart;      // [N+1] or nullptr (no interfaces)
    const int* ifIdx;        // [n_iface] index into iface / x_remote arrays
    const unsigned* ifMask;  // [ceil(N/32)] bit c: cell c has interface faces (nullptr: none)
    int n_iface;
    // SELL-C layout (variants 6/7; see host.h build_sell), nullptr if not encodable
    const int4* sell_meta;   // [chunks] {nbase, obase, wn, wo}
    const unsigned* sell_n;  // neighbour-side slots (owner column << 5 | position in the owner's faces)
    const int* sell_o;       // owner-side slots (neighbour column)
    int ell_wn, ell_wo;      // uniform chunk widths (ELL) or -1
    const double* upper_s;   // owner-slot ordered coefficient copy (variants 8/9), refreshed per call
    const int* cmeta;        // chunk-stencil compression of the ELL rows (variant 8; host.h build_ell_stencil)
    const unsigned* clane;   //   or nullptr
    // lattice slots (variant 12; host.h lattice_offsets): slot t of row c holds the coefficient of
    // the face (c, c + lat_D[t]) at upper_d[t * lat_S + c], kLatAbsent where there is no such face
    int lat_K;               // 0: the numbering is not a lattice (variant 12 unavailable)
    int lat_D[3];            // column offsets, ascending
    long long lat_S;         // slot stride (elements)
    const double* upper_d;   // [lat_K * lat_S], refreshed per solve / Amul call (k_lattice_coeffs)
};

// absent lattice slot: a NaN with a payload the assembly never produces (a caller upper array
// holding exactly this bit pattern would be read as "no face")
constexpr unsigned long long kLatAbsent = 0x7FF4A5A5C3C3A5A5ull;

// Peer-memory transport (peer.cu): kernel-parameter descriptors of one exchange / all-gather
constexpr int kMaxPeerPatches = 32;
constexpr int kMaxPeerRanks = 64;
struct PeerXfer {
    int n_patches;
    int off[kMaxPeerPatches], count[kMaxPeerPatches];           // this exchange: local offsets / counts
    double* dst[kMaxPeerPatches][2];                              // receiver's region for my patch (parity)
    unsigned long long* dst_flag[kMaxPeerPatches][2];             // receiver's flag slot for me (parity)
    const double* src[kMaxPeerPatches][2];                        // my region written by patch p's peer
    const unsigned long long* src_flag[kMaxPeerPatches][2];       // my flag slot for patch p's peer
};
struct PeerGather {
    int n_ranks, rank;
    double* part[kMaxPeerRanks][2];               // rank t's partials block [n_ranks][4] (parity)
    unsigned long long* flag[kMaxPeerRanks][2];   // rank t's partial flags [n_ranks] (parity)
    const double* my_part[2];
    const unsigned long long* my_flag[2];
};
struct PeerState {
    unsigned long long* ctr;  // [2] exchange / all-gather epochs (device)
    unsigned* ticket;
    int* err;                 // set on a poll timeout
    long long poll_cycles = 40'000'000'000LL;  // poll limit, SM clocks (~20 s at 2 GHz; SPUMA_OPT_PEER_POLL_MS)
};

struct Workspace {
    double *wA, *rA, *pA, *rD, *sumA;
    double* pA_prev;   // direction of the previous iteration (== pA unless psi updates are deferred)
    double* pA2;       // second direction buffer (deferred psi updates)
    double* xr;        // [n_iface] x_remote received from the neighbours
    double* part;      // [kMaxPartials * grid] per-CTA partials
    DevScal* scal;
    DevPtrs* ptrs;
    // the peer transport's fused PCG loop (SPUMA_OPT_PEER_FUSED): the halo stores inside the
    // direction kernel and the receive inside the interface rows, the rank-partial all-gather
    // and finalisation inside the reductions' last CTA; nullptr without the peer transport
    const PeerXfer* px;      // device copy of the level-0 exchange descriptor
    const PeerGather* pg;    // device copy of the all-gather descriptor
    const int* if_patch;     // [n_iface] processor patch (px order) of each interface face
    PeerState pst;
};

// The persistent PCG loop (loop.cu, SPUMA_OPT_PERSISTENT)
struct LoopArgs {
    unsigned long long* bar;  // [0] grid-barrier arrivals (zeroed before every launch), [1] abort word
    int tmem_pairs;           // rA pairs per thread held in tensor memory (0: no TMEM)
    int smem_pairs;           // ... then in shared memory (the rest in HBM)
    int alt;                  // alternating sweep directions (SPUMA_OPT_ALT_SWEEP)
    long long spin_limit;     // clock64 cycles a grid barrier waits before it aborts the loop
    unsigned long long* prof; // [8 * grid] per-CTA phase work / barrier-wait ns (nullptr: off)
};

// One GAMG level on the device, captured by value.  Level 0 reads its
// matrix, source and psi through DevPtrs (per-call pointers); its b is Workspace::rA.
struct GLevel {
    MeshArgs a;                   // this level's lduAddressing (no interfaces, no SELL)
    double* diag;                 // nullptr on level 0
    double* upper;                // nullptr on level 0
    double* rD;                   // 1/diag
    double* b;                    // right-hand side of the level's correction equation
    double *x, *x2, *r;           // correction (ping-pong) and residual after pre-smoothing
    double *p, *q;                // first post-sweep = alpha p + q (k_gamg_scale / k_gamg_post)
    const int* ftc;               // [N] -> next level's cell, nullptr on the coarsest
    const int *cStart, *cList;    // next level: coarse cell -> fine cells
    const int *ciStart, *ciList;  // next level: coarse cell -> agglomerate-internal fine faces
    const int *cfStart, *cfList;  // next level: coarse face -> fine faces
    int nc, ncf;                  // next level's size
    int grid;                     // CTAs of this level's cell kernels (fixed: deterministic reductions)
    int ell;                      // 1: rows over the ELL layout (a.sell_*, a.upper_s; level 0 of a uniform mesh)
    double* upperLo;              // coarse generic levels: coefficients in losort order (nullptr: gather)
    const int* losortPos;         //   face -> its losort position (k_gamg_agg writes upperLo through it)
    const int *crp, *ccol;        // coarse generic levels: CSR rows of the off-diagonal entries (row_ax order)
    double* cval;                 //   their values (k_gamg_agg), nullptr: no CSR copy
    const int *cposU, *cposL;     //   face -> its positions in the owner / neighbour row
    // processor interfaces (n_ranks > 1, readings Q36-Q38): a.ifStart / a.ifIdx per cell
    const double* iface;          // [n_if] coefficients (nullptr on level 0: DevPtrs::iface)
    double* xr;                   // [n_if] the neighbours' values of the vector a row kernel gathers
    double* sendbuf;              // [n_if] packed local values for the neighbours
    const int* if_cell;           // [n_if] local cell of each interface face
    int n_if;
    const int *cifStart, *cifList;  // next level: coarse interface face -> fine interface faces
    int ncif;                     // next level's interface faces
};


struct Patch {
    int kind, n_faces, offset;   // offset into the concatenated boundary arrays
    int neighbour_rank;          // processor
    int iface_offset;            // processor: offset into the iface arrays
};

}  // namespace spuma

struct GamgState;  // api.cu
struct PcState;    // api.cu: preconditioned solvers (§8(f3)/(f4))

struct spuma_mesh_s {
    int N = 0, F = 0, Fb = 0, n_iface = 0;
    int renumber = 0;
    int rank = 0, n_ranks = 1;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaStream_t comm_stream = nullptr;
    ncclComm_t comm = nullptr;
    bool external_comm = false;          // n_ranks > 1 without an NCCL id: host callbacks
    spuma_comm_callbacks cb{};
    double *h_send = nullptr, *h_recv = nullptr, *h_part = nullptr;  // pinned (external comm)
    std::vector<int> cb_peers, cb_offsets, cb_counts;
    std::vector<int> h_if_cell;          // [n_iface] local cell of each processor face, (patch, face) order
    // peer-memory transport (spuma_peer_export / spuma_peer_import; peer.cu)
    bool peer = false;
    double* d_mail = nullptr;            // this rank's mailbox (IPC-exported)
    spuma::PeerXfer* d_px = nullptr;     // device copies for the fused PCG loop (Workspace::px, pg)
    spuma::PeerGather* d_pg = nullptr;
    int* d_if_patch = nullptr;
    size_t mail_units = 0;
    std::vector<void*> peer_mapped;      // opened IPC mappings (to close)
    spuma::PeerXfer px{};                // level-0 exchange descriptor (off/count per call)
    spuma::PeerGather pg{};
    spuma::PeerState pst{};

    std::vector<spuma::Patch> patches;
    // host copies of the derived addressing (internal numbering) for diagnostics
    std::vector<int> h_perm, h_face_map, h_owner, h_neighbour, h_ownerStart, h_losort, h_losortStart;
    std::vector<signed char> h_face_flip;

    // device: addressing (internal numbering)
    int *d_owner = nullptr, *d_neighbour = nullptr, *d_ownerStart = nullptr, *d_losortStart = nullptr;
    int *d_losort = nullptr, *d_ownerLo = nullptr;
    int *d_perm = nullptr, *d_face_map = nullptr;  // renumber only
    int* d_sell_meta = nullptr;
    int sell_wn = -1, sell_wo = -1;  // uniform chunk widths (ELL-like) or -1
    double* d_upper_s = nullptr;     // [32 * sell_wo * chunks] (uniform layout only)
    int* d_cmeta = nullptr;          // chunk-stencil ELL compression (uniform layout only)
    unsigned* d_clane = nullptr;
    bool ell_stencil = false;        // use it (SPUMA_OPT_ELL_STENCIL; measured neutral -> off)
    int lat_K = 0;                   // lattice slots (variant 12): offsets, stride, coefficient copy
    int lat_D[3] = {0, 0, 0};
    long long lat_S = 0;
    double* d_upper_d = nullptr;
    unsigned* d_sell_n = nullptr;
    int* d_sell_o = nullptr;
    // device: geometry
    double *d_delta = nullptr, *d_weights = nullptr, *d_magSf = nullptr;
    // device: boundary faces, concatenated in patch order (all patches)
    int *d_bkind = nullptr, *d_bcell = nullptr, *d_bproc = nullptr;  // bproc: iface ordinal or -1
    double *d_bmagSf = nullptr, *d_bdelta = nullptr, *d_bweight = nullptr, *d_bvalue = nullptr;
    double* d_bgamma_r = nullptr;    // [n_iface] remote gamma (gamma halo)
    signed char* d_bis_owner = nullptr;
    int *d_bStart = nullptr, *d_bFace = nullptr;   // per-cell lists of contributing boundary faces
    int *d_bAllStart = nullptr, *d_bAllFace = nullptr;  // per-cell lists of all non-empty boundary faces
    signed char* d_face_flip = nullptr;  // renumber: internal face orientation reversed w.r.t. the caller
    double *d_bphi = nullptr, *d_bflux = nullptr;       // [Fb] staging of per-patch face fields
    double *d_face_b = nullptr, *d_face_c = nullptr;    // [F] staging of oriented face fields
    // non-orthogonal correction: geometry kept from mesh_create (internal numbering)
    double *d_Sf = nullptr, *d_C = nullptr, *d_corrvec = nullptr, *d_bSf = nullptr, *d_bnC = nullptr;
    double *d_G = nullptr, *d_Gr = nullptr, *d_pr = nullptr;  // gradient [3N], remote gradient [3 n_iface], remote p
    double *d_bcflux = nullptr, *d_face_d = nullptr;          // boundary / internal correction flux staging
    double *d_div = nullptr, *d_cell_v = nullptr;             // [N] divergence, V staging
    // device: interfaces
    int *d_ifStart = nullptr, *d_ifIdx = nullptr, *d_if_cell = nullptr;  // if_cell: [n_iface] local cell
    unsigned* d_ifMask = nullptr;
    int* d_ifRows = nullptr;          // cells with processor faces, ascending
    int n_ifRows = 0;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // halo / interior overlap
    cudaStream_t tstream = nullptr;   // leaf branch of the timing event nodes (captured batches)
    cudaEvent_t tfork = nullptr;
    double* d_sendbuf = nullptr;     // [n_iface] packed x for the neighbours
    // staging (renumbering / host pointers), allocated on first use
    double *d_cell_a = nullptr, *d_cell_b = nullptr, *d_cell_c = nullptr, *d_cell_d = nullptr,
           *d_cell_e = nullptr, *d_cell_t = nullptr;
    double *d_face_a = nullptr, *d_face_t = nullptr, *d_iface_a = nullptr;

    spuma::Workspace ws{};
    spuma::DevPtrs* h_ptrs = nullptr;   // pinned
    spuma::DevScal* h_scal = nullptr;   // pinned [2]
    int grid = 0;                       // CTAs of the cell kernels (fixed: deterministic partials)
    int grid_faces = 0;

    // captured iteration batches (ping-pong) and timing events
    int batch = 16;
    int small_max_cells = 8192;  // single-CTA solve at or below this many cells (1 rank)
    bool small_smem = true;      // ... staged in shared memory when it fits (SPUMA_OPT_SMALL_SMEM)
    bool peer_fused = true;      // peer transport: halo + all-gather fused into the PCG loop's kernels
    int amul_variant = 12;  // lattice slots (falls back to 10 -> 6 -> 5 off lattice / uniform meshes)
    int defer_psi = 2;      // 0: psi += alpha pA every iteration; 1: pairs in k_update; 2: pairs in k_direction  // psi += alpha pA applied every second iteration (same rounding, fewer bytes)  // ELL + coefficient copy (falls back to 6 -> 5 when the mesh is not uniform)
    bool timing = false;
    int fuse_direction = 0;      // 0: k_direction + k_amul_dot (default: faster); 1: fused, rD read; 2: fused, 1/diag inline
    bool gamg_csr = true;        // GAMG coarse generic levels as CSR runs (SPUMA_OPT_GAMG_CSR)
    int l2_persist = 2;          // L2 access-policy window (SPUMA_OPT_L2_PERSIST): 0 none, 1 pA, 2 rA (default), 3 rD, 4 wA
    bool l2_limit_set = false;   // the persisting-L2 limit was raised (reset on option off / free)
    const double* l2_lines = nullptr;  // the vector whose L2 lines the last window made persisting
    bool alt_sweep = true;       // alternate the sweep direction of consecutive hot-loop kernels (L2 reuse)
    int gamg_tail_cells = 512;   // GAMG: levels from the first one at or below this size run in one CTA (0: off)
    // persistent PCG loop (loop.cu, SPUMA_OPT_PERSISTENT): 0 off, 1 rA in HBM, 2 + shared memory,
    // 3 + tensor memory (default)
    int persistent = 3;
    bool loop_profile = false;   // per-phase work / barrier-wait profile of the loop (SPUMA_OPT_LOOP_PROFILE)
    int loop_ctas = 0;           // CTAs of the persistent loop (SPUMA_OPT_LOOP_GRID; 0 = one per SM)
    int loop_l2 = 1;             // L2 window of the persistent loop (SPUMA_OPT_LOOP_L2, targets as l2_persist): pA
    unsigned long long* d_loop_bar = nullptr;  // [2] barrier arrivals, abort word
    double* d_loop_part = nullptr;             // [3 * SMs] CTA partials
    unsigned long long* d_loop_prof = nullptr; // [8 * SMs] phase work / wait ns (timing on)
    int loop_grid = 0;                         // SMs (one CTA each), 0 until first use
    cudaEvent_t loop_ev[2] = {nullptr, nullptr};  // timing of the launch (spuma_set_timing)
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    bool gexec_timed = false;
    int gexec_batch = 0;
    std::vector<cudaEvent_t> tev[2];     // [batch * 3 * 2] per graph
    cudaEvent_t batch_done[2] = {nullptr, nullptr};
    cudaEvent_t asm_ev[2] = {nullptr, nullptr};

    spuma_stats stats{};
    GamgState* gamg = nullptr;  // GAMG hierarchy + captured cycle, built on first spuma_gamg_solve
    PcState* pc = nullptr;      // level schedules + buffers of the DIC/DILU/PBiCG solvers
};

// NVTX range per C-ABI call and solver phase (SURVEY §5 tracing): visible in nsys / ncu
// --nvtx timelines, free otherwise
namespace spuma {
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace spuma
#define SPUMA_NVTX(name) spuma::NvtxRange spuma_nvtx_range_(name)

// error plumbing (api.cu)
namespace spuma {
spuma_status set_error(spuma_status s, const std::string& msg);
}

#define SPUMA_CUDA(call)                                                                             \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess)                                                                       \
            return spuma::set_error(e_ == cudaErrorMemoryAllocation ? SPUMA_ERR_OUT_OF_MEMORY : SPUMA_ERR_CUDA, \
                                    std::string(#call) + ": " + cudaGetErrorString(e_));             \
    } while (0)

#define SPUMA_NCCL(call)                                                                             \
    do {                                                                                             \
        ncclResult_t r_ = (call);                                                                    \
        if (r_ != ncclSuccess)                                                                       \
            return spuma::set_error(SPUMA_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

#define SPUMA_TRY(call)                      \
    do {                                     \
        spuma_status s_ = (call);            \
        if (s_ != SPUMA_OK) return s_;       \
    } while (0)

// kernels.cu launchers (all asynchronous on `s`)
namespace spuma {
void launch_geometry(cudaStream_t s, int F, const int* owner, const int* neighbour, const double* Sf,
                     const double* magSf, const double* C, const double* Cf, double* delta, double* weights);
void launch_bgeometry(cudaStream_t s, int Fb, const int* kind, const int* bcell, const double* bSf,
                      const double* bmagSf, const double* bCf, const double* C, const double* nC,
                      const signed char* is_owner, double* bdelta, double* bweight);
void launch_face_coeffs(cudaStream_t s, int grid, int F, const int* owner, const int* neighbour,
                        const double* delta, const double* weights, const double* magSf, const double* gamma,
                        double* upper);
void launch_diag_gather(cudaStream_t s, int grid, const MeshArgs& a, const double* upper, const int* bStart,
                        const int* bFace, const int* bkind, const int* bcell, const int* bproc,
                        const double* bmagSf, const double* bdelta, const double* bweight, const double* bvalue,
                        const double* bgamma_r, const signed char* bis_owner, const double* gamma, int ref_cell,
                        double ref_value, double* diag, double* source, double* iface);
void launch_amul(cudaStream_t s, int variant, const MeshArgs& a, const double* diag, const double* upper,
                 const double* iface, const double* x, const double* xr, double* y, long long x_len, int sell_wn,
                 int sell_wo);
void launch_gather(cudaStream_t s, int n, const int* idx, const double* in, double* out);   // out[i] = in[idx[i]]
void launch_ell_coeffs(cudaStream_t s, const MeshArgs& a, const double* upper, double* upper_s);
bool amul_uses_ell(int variant);
void launch_lattice_coeffs(cudaStream_t s, const MeshArgs& a, const double* upper);  // variant 12 slots
void launch_fill_u64(cudaStream_t s, long long n, double* p, unsigned long long v);
void launch_scatter(cudaStream_t s, int n, const int* idx, const double* in, double* out);  // out[idx[i]] = in[i]
void launch_pack(cudaStream_t s, int n, const int* cell, const double* x, double* out);     // out[i] = x[cell[i]]

// PCG (A6-A12). `fin` = true when this rank finalises itself (P == 1).
void launch_setup1(cudaStream_t s, int grid, const MeshArgs& a, const Workspace& w, bool fin);
void launch_setup2(cudaStream_t s, int grid, const MeshArgs& a, const Workspace& w, bool fin);
// psi_pair (SPUMA_OPT_DEFER_PSI = 2, even iterations k >= 2): also psi = (psi + alpha_{k-2} p_{k-2}) +
// alpha_{k-1} p_{k-1}, p_{k-2} being the buffer the new direction overwrites
void launch_direction(cudaStream_t s, int grid, const MeshArgs& a, const Workspace& w, bool reverse = false,
                      bool psi_pair = false, bool halo = false);
void launch_amul_dot(cudaStream_t s, int variant, const MeshArgs& a, const Workspace& w, bool fin, int sell_wn,
                     int sell_wo, bool deferred = false, bool reverse = false);
// reverse: the kernel sweeps its cells in descending order (alternating sweep directions between
// consecutive kernels lets each one start on the lines its predecessor left in L2)
int resolve_amul_variant(int variant, const MeshArgs& a);  // variant actually run on this mesh
// peer: the halo's receive (flags + mailbox reads) and the stage-3 all-gather + finalisation fused in
void launch_iface_rows(cudaStream_t s, const MeshArgs& a, const Workspace& w, const int* rows, int n_rows,
                       bool peer = false);
void launch_surface_integrate(cudaStream_t s, const MeshArgs& a, const double* phi, const int* bStart,
                              const int* bFace, const double* bphi, const double* V, double* out);
void launch_face_flux(cudaStream_t s, int F, const int* owner, const int* neighbour, const double* upper,
                      const double* psi, const double* cflux, double* flux, double* phi);
void launch_bface_flux(cudaStream_t s, int Fb, const int* bkind, const int* bcell, const int* bproc,
                       const double* bmagSf, const double* bdelta, const double* bweight, const double* bvalue,
                       const double* bgamma_r, const signed char* bis_owner, const double* gamma, const double* psi,
                       const double* psi_r, const double* bcflux, double* bflux, double* bphi);
void launch_gather_signed(cudaStream_t s, int n, const int* idx, const signed char* flip, const double* in,
                          double* out);
void launch_corrvec(cudaStream_t s, int F, const int* owner, const int* neighbour, const double* Sf,
                    const double* magSf, const double* C, const double* delta, double* cv);
void launch_gauss_grad(cudaStream_t s, const MeshArgs& a, const double* Sf, const double* weights, const double* p,
                       const int* bStart, const int* bFace, const int* bkind, const int* bproc, const double* bSf,
                       const double* bvalue, const double* bweight, const signed char* bis_owner, const double* p_r,
                       const double* V, double* G);
void launch_nonorth_flux(cudaStream_t s, int F, int NC, const int* owner, const int* neighbour, const double* cv,
                         const double* magSf, const double* weights, const double* gamma, const double* G,
                         double* cflux);
void launch_bnonorth_flux(cudaStream_t s, int Fb, int NC, int NI, const int* bkind, const int* bcell, const int* bproc,
                          const double* bSf, const double* bmagSf, const double* bdelta, const double* bweight,
                          const signed char* bis_owner, const double* bnC, const double* C, const double* G,
                          const double* G_r, const double* gamma, const double* bgamma_r, double* bcflux);
void launch_sub_vdiv(cudaStream_t s, int N, const double* V, const double* div, double* src);
void launch_add(cudaStream_t s, int n, const double* in, double* out);
void launch_scatter_signed(cudaStream_t s, int n, const int* idx, const signed char* flip, const double* in,
                           double* out);
constexpr int kPad = 8;  // padding elements on internal arrays (16-byte TMA windows may overrun by <= 3)
// fin: 1 finalise (one rank); 0 leave the rank partials; 2 the peer all-gather + finalisation in the last CTA
void launch_update(cudaStream_t s, int grid, const MeshArgs& a, const Workspace& w, int fin, int psi_mode = 0,
                   bool reverse = false);
// psi_mode: 0 psi += alpha pA; 1 defer (psi untouched); 2 psi = (psi + alpha_prev pA_prev) + alpha pA
void launch_psi_flush(cudaStream_t s, int N, const Workspace& w);
// SPUMA_OPT_DEFER_PSI = 2: the pending updates j = n - pending .. n - 1 (pending <= 2), p_j in pA if
// j is even, else pA2; alpha_{n-1} = alpha_prev, alpha_{n-2} = alpha_prev2
void launch_psi_flush2(cudaStream_t s, int N, const Workspace& w, int n, int pending);
// loop.cu: the persistent PCG loop (one cooperative launch per solve)
int loop_threads();
int loop_tmem_pairs();
int loop_occupancy(int K, size_t smem);
cudaError_t launch_pcg_loop(cudaStream_t s, int grid, size_t smem, const MeshArgs& a, const Workspace& w,
                            const LoopArgs& L, const cudaAccessPolicyWindow* win, int layout);  // 1 lattice, 2 ELL, 3 SELL
// A11+A7+A8 in one kernel (ELL, single rank, deferred psi): see kernels.cu
bool fused_direction_ok(const MeshArgs& a);
void launch_amul_dot_dir(cudaStream_t s, const MeshArgs& a, const Workspace& w, bool inline_rd);  // psi += alpha_prev pA (pending update)
// P > 1: finalise from the gathered rank partials ([n_ranks][4], rank order)
void launch_finalize(cudaStream_t s, int stage, const double* gathered, int n_ranks, const Workspace& w);
void launch_scal_init(cudaStream_t s, const Workspace& w, const spuma_solver_controls& c, int n_ranks);
void launch_pcg_single(cudaStream_t s, const MeshArgs& a, const Workspace& w);  // whole solve, 1 CTA
// the same with everything in shared memory; false (nothing launched) if the mesh does not fit
bool launch_pcg_single_smem(cudaStream_t s, const MeshArgs& a, const Workspace& w);
int occupancy_grid(int N, int* grid_faces, int F);
// preconditioned solvers (precond.cu)
int pc_grid(int n);
void launch_recip(cudaStream_t s, int N, const double* in, double* out);  // out = 1 / in
void launch_ilu_factor(cudaStream_t s, const MeshArgs& a, const int* order, const double* diag, const double* upper,
                       const double* lower, double* raw, double* rD, int* flag, unsigned* counter, int width);
void launch_ilu_precondition(cudaStream_t s, const MeshArgs& a, const int* order_f, const int* order_b,
                             const double* rD, const double* upper, const double* lower, const double* r, double* w,
                             double* t1, double* t2, int* flag, unsigned* counter, int k, bool transpose,
                             const DevScal* scal, int width_f = 1 << 30, int width_b = 1 << 30,
                             const double* fpre = nullptr, const double* bpre = nullptr);
// aDILU pass coefficients rD*lower / rD*upper in pass order, for M^-1 (fco, bco) and M^-T (fcoT, bcoT)
void launch_adilu_coefs(cudaStream_t s, const MeshArgs& a, const double* rD, const double* upper,
                        const double* lower, double* fco, double* bco, double* fcoT, double* bcoT);
void launch_pc_dot(cudaStream_t s, int N, const double* w, const double* r, double* part, DevScal* scal,
                   bool fin = true);
void launch_pc_direction(cudaStream_t s, int N, const double* wA, double* pA, const double* wT, double* pT,
                         const DevScal* scal);
void launch_bicg_amul_tmul(cudaStream_t s, const MeshArgs& a, const double* diag, const double* upper,
                           const double* lower, const double* iface, const double* iface_t, const double* pA,
                           const double* pT, const double* xr, const double* xrT, double* wA, double* wT,
                           double* part, DevScal* scal, bool fin);
void launch_bicg_update(cudaStream_t s, int N, double* psi, const double* pA, double* rA, const double* wA, double* rT,
                        const double* wT, double* part, DevScal* scal, bool fin);
void launch_bicg_setup1(cudaStream_t s, const MeshArgs& a, const double* diag, const double* upper,
                        const double* lower, const double* iface, const double* iface_t, const double* xr,
                        const double* source, const double* psi, double* wA, double* wT, double* rA, double* rT,
                        double* sumA, double* part, DevScal* scal, bool fin);
void launch_pc_setup2(cudaStream_t s, int N, const double* wA, const double* sumA, const double* source,
                      const double* rA, double* part, DevScal* scal, bool fin);
void launch_csr_values(cudaStream_t s, int nnz, int N, int F, const int* map, const double* diag,
                       const double* upper, const double* lower, double* vals);
void launch_gather_pair(cudaStream_t s, int F, const int* map, const signed char* flip, const double* u,
                        const double* l, double* uo, double* lo);
void launch_amul_asym(cudaStream_t s, const MeshArgs& a, const double* diag, const double* upper,
                      const double* lower, const double* x, double* y, bool transpose);
// GAMG (gamg.cu).  P = the handle's DevPtrs (level 0's matrix, source, psi).
int gamg_grid(int n);
void launch_gamg_agg(cudaStream_t s, const GLevel& fine, const GLevel& coarse, const DevPtrs* P);
void launch_gamg_csr_values(cudaStream_t s, const GLevel& L, const double* upper, int F);  // level-0 CSR values
void launch_gamg_restrict(cudaStream_t s, const GLevel& fine, const GLevel& coarse, const DevPtrs* P,
                          const double* x, double* zero_x = nullptr);  // x nullptr: the level's x is zero
void launch_gamg_smooth(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* xin, double* xout,
                        double omega, const double* xc, const double* alpha, bool psi_acc);
void launch_gamg_scale(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* x, const double* xc,
                       const double* r, double omega, bool pq, double* part, unsigned* ticket, double* alpha,
                       double* rank_part = nullptr);  // rank_part: write the two dots there (n_ranks > 1)
void launch_gamg_correct(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* x, const double* xc,
                         const double* alpha, double* out, bool psi_acc);
void launch_gamg_residual(cudaStream_t s, const GLevel& L, const Workspace& w, double* rank_part = nullptr);
// n_ranks > 1: L.sendbuf[i] = X(if_cell[i]) for X = 0: x (nullptr: 0), 1: x + alpha xc[ftc],
// 2: xc[ftc], 3: alpha p + q -- the vector the next row kernel of the level gathers
void launch_gamg_pack(cudaStream_t s, const GLevel& L, int mode, const double* x, const double* xc,
                      const double* alpha, const double* p, const double* q);
// n_ranks > 1: finish a reduction from the gathered rank partials ([n_ranks][4], rank order):
// what 0: alpha = clamp(sum g0 / sum g1) (Q25); what 1: the outer residual (Q28) into scal
void launch_gamg_fin(cudaStream_t s, int what, const double* gathered, int n_ranks, double* alpha, DevScal* scal);
// levels t..nl-1 of the V-cycle in one CTA (Richardson, scaled, nPre = 0); d_lv: device copy of the levels
void launch_gamg_tail(cudaStream_t s, const GLevel* d_lv, int t, int nl, const Workspace& cws, double omega,
                      int n_post);
void launch_gamg_post(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* alpha, double omega,
                      double* out, bool two, bool psi_acc);
void launch_gamg_gs2_res(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* xin, const double* xc,
                         const double* alpha, double* r);
void launch_gamg_gs2_upd(cudaStream_t s, const GLevel& L, const DevPtrs* P, const double* xin, const double* xc,
                         const double* alpha, const double* r, const double* zin, double* out, bool skip_lower,
                         bool last, bool psi_acc);
// peer-memory transport (peer.cu)
void launch_peer_exchange(cudaStream_t s, const PeerXfer& d, const double* x, const int* idx, double* recv,
                          const PeerState& st);
// stage > 0 with w: also finalise the PCG scalars of w from the gathered block (k_finalize's sums)
void launch_peer_allgather4(cudaStream_t s, const PeerGather& g, const double* in, double* out, const PeerState& st,
                            int stage = 0, const Workspace* w = nullptr);
extern bool g_use_pdl;  // programmatic dependent launch of the hot-loop kernels (process-wide)
}  // namespace spuma
