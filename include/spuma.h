/*
 * spuma.h -- C-ABI of libspuma: the B200-native pressure-equation hot path of
 * SPUMA (Bna et al., arXiv 2512.22215, "SPUMA: a minimally invasive approach
 * to the GPU porting of OPENFOAM").
 *
 * What it computes (citations are PAPER.md line numbers, "P:n"):
 *   - the LDU matrix of fvm::laplacian(gamma, p) on an unstructured finite-
 *     volume mesh ("P assembly"; lduMatrix / lduAddressing with an
 *     implicit DOF map; "Gauss linear corrected" with linear
 *     interpolation; negSumDiag P:520; pRefCell/pRefValue
 *     P:1083-1084),
 *   - its solve by PCG with the diagonal (Jacobi) preconditioner (the
 *     "pcgDiag" solver), including the SpMV Amul
 *     (21.79% of the paper's kernel time), the PCG vector updates and
 *     the dot-product reductions,
 *   - over a domain decomposition, one rank per GPU, with processor-patch halo
 *     exchange -- done here with NCCL over NVLink.
 * OpenFOAM semantics the paper relies on but does not print ("SPUMA
 * reproduces OpenFOAM-v2412") are the readings Q1..Q16 of DESIGN.md §3.
 *
 * Conventions (all calls):
 *   - Types: labels are int32 (spuma_label), scalars fp64 (spuma_scalar).  The
 *     path is fp64 only (reading Q16; the paper never states precision).
 *   - Numbering: every per-cell / per-face array at this API is in the
 *     CALLER's numbering, even with renumber = 1 (the library permutes on entry
 *     and exit).  Internal faces are the lduAddressing faces: owner < neighbour,
 *     sorted by (owner, neighbour).  "lower" is not passed: the Laplacian is
 *     symmetric, lower == upper.
 *   - Memory space: hot-path arrays (gamma, patch values, diag, upper, source,
 *     psi, iface_coeffs, x, y) may be device pointers (cudaMalloc / torch CUDA
 *     tensors) or host pointers (pageable or pinned); the library detects the
 *     space with cudaPointerGetAttributes and stages host arrays through its own
 *     device buffers (host<->device copies are then part of the call).
 *     spuma_mesh_create accepts host or device arrays (pointers_on_device).
 *   - Ownership: the caller owns every array it passes; the library never
 *     frees or retains a caller pointer after a call returns.  The handle owns
 *     its derived addressing, geometry, permutation, halo plan, NCCL
 *     communicator and every PCG workspace, all allocated once in
 *     spuma_mesh_create (the paper's memory-pool lesson) and released
 *     by spuma_free.
 *   - Synchrony: every call returns after its work is complete; work is
 *     ordered on the handle's CUDA stream (desc.cuda_stream, or a stream the
 *     handle creates).
 *   - Errors: a non-OK spuma_status is returned; spuma_last_error() gives a
 *     thread-local message.  Non-convergence and singularity are NOT errors
 *     (reported in spuma_solver_perf, OpenFOAM behaviour).  There is no CPU
 *     fallback: without a usable CUDA device every compute call fails with
 *     SPUMA_ERR_CUDA.
 *   - Thread safety: a handle is not thread-safe; distinct handles are
 *     independent.
 */
#ifndef SPUMA_H
#define SPUMA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPUMA_ABI_VERSION 1

typedef int32_t spuma_label;
typedef double spuma_scalar;
typedef struct spuma_mesh_s* spuma_mesh;

typedef enum {
    SPUMA_OK = 0,
    SPUMA_ERR_INVALID_ARGUMENT = 1, /* NULL where required, bad enum, bad size, abi mismatch   */
    SPUMA_ERR_ADDRESSING = 2,       /* owner >= neighbour, unsorted faces, index out of range  */
    SPUMA_ERR_LENGTH_MISMATCH = 3,  /* inconsistent array sizes (e.g. processor patch lengths) */
    SPUMA_ERR_CUDA = 4,             /* CUDA runtime error (incl. no device)                    */
    SPUMA_ERR_NCCL = 5,             /* NCCL error                                              */
    SPUMA_ERR_OUT_OF_MEMORY = 6,
    SPUMA_ERR_STATE = 7             /* call not valid in the handle's state                    */
} spuma_status;

/* Boundary condition of p on a patch (the kinds the pressure path needs; P:87,
 * P:536 for processor patches; zeroGradient/fixedValue/empty are [OF]). */
typedef enum {
    SPUMA_PATCH_ZERO_GRADIENT = 0, /* no matrix contribution                                      */
    SPUMA_PATCH_FIXED_VALUE = 1,   /* diag += (g|S|)(-delta_b); source += -(g|S|)(delta_b p_b)      */
    SPUMA_PATCH_EMPTY = 2,         /* 2-D front/back: ignored entirely                             */
    SPUMA_PATCH_PROCESSOR = 3      /* coupled face to cell of neighbour_rank (domain decomposition) */
} spuma_patch_kind;

typedef struct {
    spuma_patch_kind kind;
    spuma_label n_faces;
    const spuma_label* face_cells;   /* [n_faces] cell owning the face (local numbering)          */
    const spuma_scalar* Sf;          /* [3*n_faces] face area vectors, pointing OUT of the domain */
    const spuma_scalar* magSf;       /* [n_faces] |Sf|                                             */
    const spuma_scalar* Cf;          /* [3*n_faces] face centres                                   */
    /* PROCESSOR only (ignored otherwise): */
    int neighbour_rank;              /* rank holding the other cell                                */
    const spuma_label* global_face;  /* [n_faces] face id in the undecomposed mesh; faces must be
                                        ascending in it (reading Q13) -- both sides then agree   */
    const spuma_scalar* neighbour_C; /* [3*n_faces] centre of the remote cell                      */
    const signed char* is_owner;     /* [n_faces] 1 if the local cell is the owner of the
                                        undecomposed face (face evaluated in global orientation) */
} spuma_patch_desc;

typedef struct {
    int abi_version;                 /* SPUMA_ABI_VERSION                                           */
    spuma_label n_cells;             /* cells of this (sub-)domain                                  */
    spuma_label n_faces;             /* internal faces only                                         */
    const spuma_label* owner;        /* [n_faces] lowerAddr; owner < neighbour; sorted    */
    const spuma_label* neighbour;    /* [n_faces] upperAddr                                         */
    const spuma_scalar* Sf;          /* [3*n_faces] owner -> neighbour                              */
    const spuma_scalar* magSf;       /* [n_faces]                                                   */
    const spuma_scalar* C;           /* [3*n_cells] cell centres                                    */
    const spuma_scalar* Cf;          /* [3*n_faces] face centres (interpolation weights)            */
    int n_patches;
    const spuma_patch_desc* patches; /* [n_patches], boundary coefficients applied in this order    */
    int renumber;                    /* 0: keep caller numbering; 1: reverse Cuthill-McKee inside   */
    int pointers_on_device;          /* 0: arrays above are host memory; 1: device memory           */
    void* cuda_stream;               /* cudaStream_t to order work on; NULL: handle makes its own
                                        BLOCKING stream (ordered with the legacy default stream, so
                                        e.g. torch fills on the default stream precede each call)   */
    int rank, n_ranks;               /* n_ranks == 1: no communication                              */
    const void* nccl_unique_id;      /* 128-byte ncclUniqueId from rank 0 (n_ranks > 1)             */
} spuma_mesh_desc;

/* SolverControls (P:1033-1041 key names). converged := r < tolerance ||
 * (rel_tol > 1e-20 && r < rel_tol * initial_residual), r the normalised L1
 * residual (reading Q1/Q2); at least min_iter, at most max_iter iterations. */
typedef struct {
    spuma_scalar tolerance, rel_tol;
    int max_iter, min_iter;
} spuma_solver_controls;

typedef struct {
    spuma_scalar initial_residual, final_residual;
    int n_iterations;
    int converged, singular;
} spuma_solver_perf;

/*
 * Build a handle for one (sub-)mesh: validate the addressing (A0), optionally
 * renumber cells by reverse Cuthill-McKee (A1, reading O2/Q12), derive
 * ownerStart / losort / losortStart and the per-cell boundary lists (A2),
 * compute nonOrthDeltaCoeffs and linear weights on the device (A3),
 * build the halo plan and the NCCL communicator (n_ranks > 1), and allocate
 * every workspace.  Errors: INVALID_ARGUMENT, ADDRESSING, LENGTH_MISMATCH,
 * CUDA, NCCL, OUT_OF_MEMORY.  *out is NULL on error.
 */
spuma_status spuma_mesh_create(const spuma_mesh_desc* desc, spuma_mesh* out);

/*
 * Assemble fvm::laplacian(gamma, p) ("P assembly"):
 *   gamma_f  = w (gamma_P - gamma_N) + gamma_N         (linear; gamma == NULL: gamma = 1)
 *   upper[f] = delta_f (gamma_f |S_f|)                 lower == upper
 *   diag[c]  = -sum of the off-diagonals of row c      (negSumDiag)
 *   setReference(ref_cell, ref_value) if ref_cell >= 0:
 *            source[ref] += diag[ref] ref_value; diag[ref] += diag[ref]
 *   then boundary coefficients in (patch, face) order (fixedValue, processor).
 * gamma: [n_cells]. patch_value: [n_patches] array of pointers, fixedValue
 * values per patch face (entries for other kinds ignored; may be NULL if no
 * fixedValue patch).  diag [n_cells], upper [n_faces] are written; source
 * [n_cells] is read-modified-written.  iface_coeffs: [sum of processor faces]
 * written with the true matrix entries A[P][remote] (reading Q9), in patch
 * order; NULL allowed when there is no processor patch.  n_ranks > 1: the gamma
 * halo is exchanged with the neighbours (collective: all ranks must call).
 */
spuma_status spuma_assemble_laplacian(spuma_mesh m, const spuma_scalar* gamma,
                                      const spuma_scalar* const* patch_value, spuma_label ref_cell,
                                      spuma_scalar ref_value, spuma_scalar* diag, spuma_scalar* upper,
                                      spuma_scalar* source, spuma_scalar* iface_coeffs);

/*
 * Solve A psi = source by PCG with the diagonal preconditioner, OpenFOAM
 * semantics (normFactor Q1, convergence Q2, loop Q3, singularity
 * Q4).  psi [n_cells] is the initial guess on entry and the solution on exit.
 * diag/upper/iface_coeffs as produced by spuma_assemble_laplacian (or any
 * symmetric LDU matrix on this mesh).  perf must be non-NULL.  n_ranks > 1:
 * collective; dot products and norms are global and every rank returns the
 * same perf.
 */
spuma_status spuma_pcg_solve(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                             const spuma_scalar* iface_coeffs, const spuma_scalar* source, spuma_scalar* psi,
                             const spuma_solver_controls* ctl, spuma_solver_perf* perf);

/* Release everything the handle owns (NULL-safe). */
void spuma_free(spuma_mesh m);

/* ---------------- GAMG with the Richardson smoother ----------------
 * PAPER.md P:665 ("GAMG ... Richardson smoother ... diagonal at the coarsest level"),
 * pGAMG controls P:1043-1052, profile rows restrictField / prolongField /
 * agglomerateMatrix / scale / Vcycle P:517-545.  Readings Q22-Q28:
 * faceAreaPair pairwise agglomeration on |S_f| (Q22), Galerkin coarse matrices (Q27),
 * V-cycle in correction form (Q23) with weighted-Jacobi sweeps (Q24) or two-stage
 * Gauss-Seidel sweeps (Q30, the paper's second GPU smoother), energy-optimal
 * correction scaling clamped to [0, 2] (Q25), PCG + diagonal at the coarsest level (Q26),
 * PCG's normFactor / convergence / loop semantics with one V-cycle per iteration (Q28). */
typedef struct spuma_gamg_params {
    int n_pre_sweeps;               /* Richardson sweeps before restriction (default 0)           */
    int n_post_sweeps;              /* sweeps after the coarse correction (default 2)             */
    int scale_correction;           /* 1: scale the prolonged correction (default 1)              */
    int n_cells_in_coarsest_level;  /* coarsening stops at or below this many cells (default 10)  */
    int max_levels;                 /* including the finest (default 50)                          */
    double omega;                   /* Richardson weight (default 0.75)                           */
    double coarsest_tolerance;      /* coarsest PCG tolerance (default 0)                         */
    double coarsest_rel_tol;        /* coarsest PCG relTol (default 1e-6)                         */
    int coarsest_max_iter;          /* coarsest PCG maxIter (default 1000)                        */
    int smoother;                   /* SPUMA_SMOOTHER_RICHARDSON (default) or _GS2 (Q30)          */
    int n_inner;                    /* two-stage Gauss-Seidel: inner Jacobi-Richardson iterations (default 1) */
} spuma_gamg_params;
enum { SPUMA_SMOOTHER_RICHARDSON = 0, SPUMA_SMOOTHER_GS2 = 1 };

/* Fill *p with the defaults above. */
void spuma_gamg_default_params(spuma_gamg_params* p);

/*
 * Solve A psi = source by GAMG (arguments as spuma_pcg_solve; params NULL: defaults).
 * The level hierarchy depends only on the mesh, n_cells_in_coarsest_level and max_levels:
 * it is built on the host at the first call (and when those change) and kept by the
 * handle; every call re-forms the coarse matrices from diag/upper on the device.
 * perf->n_iterations counts V-cycles.  Decomposed meshes (n_ranks > 1; collective, every
 * rank calls it; iface_coeffs as spuma_pcg_solve): readings Q36-Q38 -- processor-local
 * agglomeration with the level count decided on the global cell count, coarse processor
 * interfaces = distinct (local, remote) agglomerate pairs by first occurrence with summed
 * coefficients, the halo of every gathered vector before each row kernel, rank-order sums
 * for the scale factors and the residual, and PCG + diagonal over all ranks on the
 * coarsest level; V-cycles are launched directly (not captured).
 * Errors: INVALID_ARGUMENT (NULL arrays/perf, negative limits, max_levels < 1,
 * n_post_sweeps/n_pre_sweeps < 0), STATE, CUDA, OUT_OF_MEMORY.
 */
spuma_status spuma_gamg_solve(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                              const spuma_scalar* iface_coeffs, const spuma_scalar* source, spuma_scalar* psi,
                              const spuma_solver_controls* ctl, const spuma_gamg_params* params,
                              spuma_solver_perf* perf);

/*
 * Diagnostics of the hierarchy built by the last spuma_gamg_solve (or built now from
 * params, NULL: defaults): *n_levels; level_cells / level_faces [max_levels] (may be
 * NULL); ftc: if non-NULL and level < *n_levels - 1, the fine-to-coarse map of that
 * level [cells of the level], in the handle's INTERNAL numbering (spuma_mesh_get_addressing).
 */
spuma_status spuma_gamg_get_hierarchy(spuma_mesh m, const spuma_gamg_params* params, int max_levels,
                                      int* n_levels, int* level_cells, int* level_faces, int level,
                                      spuma_label* ftc);

/* ---------------- preconditioned solvers (readings Q31-Q35) ----------------
 * DIC / DILU (OpenFOAM's incomplete factorisations with a diagonal-only factor, P:566, P:665,
 * P:672), aDILU (DILU factor, each triangular sweep replaced by n_sweeps Jacobi-style passes,
 * reading Q33 — the paper's "aDILUPreconditioner", never defined), diagonal.  The
 * factor and the exact sweeps are sequential recurrences in face order; libspuma runs them
 * as dependency-scheduled persistent kernels, bitwise equal to the sequential loops for any
 * numbering (their critical path is the mesh's dependency depth: a colour / wavefront
 * numbering makes them fast, the natural order of an n^3 box has depth ~3n).
 * spuma_pcg_solve_pc and spuma_pbicg_solve run on decomposed meshes too; the diagnostics
 * are single-rank (n_ranks > 1 -> SPUMA_ERR_STATE). */
typedef enum spuma_precond_kind {
    SPUMA_PC_DIAGONAL = 0,
    SPUMA_PC_DIC = 1,
    SPUMA_PC_DILU = 2,
    SPUMA_PC_ADILU = 3
} spuma_precond_kind;

typedef struct spuma_preconditioner {
    int kind;      /* spuma_precond_kind                                   */
    int n_sweeps;  /* aDILU: Jacobi-style passes per triangular sweep (2)  */
} spuma_preconditioner;

/*
 * PCG (Q1-Q4 semantics) with the preconditioner pc (NULL: diagonal): per iteration
 * wA = M^-1 rA, wArA = wA.rA, pA = wA + beta pA, wA = A pA, alpha = wArA / wA.pA, psi and rA
 * updated.  Arguments as spuma_pcg_solve (symmetric matrix: upper only; iface_coeffs as
 * produced by spuma_assemble_laplacian when n_ranks > 1).  Multi-rank: collective; the
 * preconditioner is factorised and applied on each rank's own faces (processor-local, as
 * OpenFOAM on decomposed meshes, Q31), the Amul and the dot products are global.  Errors as
 * spuma_pcg_solve plus INVALID_ARGUMENT (unknown kind, n_sweeps < 0).
 */
spuma_status spuma_pcg_solve_pc(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                                const spuma_scalar* iface_coeffs, const spuma_scalar* source, spuma_scalar* psi,
                                const spuma_solver_controls* ctl, const spuma_preconditioner* pc,
                                spuma_solver_perf* perf);

/*
 * PBiCG (Q32) for an asymmetric LDU matrix: lower [n_faces] is
 * the coefficient of row neighbour, column owner; upper of row owner, column neighbour.
 * n_ranks > 1 (collective): iface_coeffs [sum of processor faces] = this rank's row entry
 * A[P][remote] of each processor face (used by Amul), iface_coeffs_t = the remote row's entry
 * A[remote][P] (used by Tmul); both NULL on a single rank.  The preconditioner is
 * processor-local (Q31).  pc NULL: aDILU with 2 passes (the paper's setting).  psi in/out.
 */
spuma_status spuma_pbicg_solve(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                               const spuma_scalar* lower, const spuma_scalar* iface_coeffs,
                               const spuma_scalar* iface_coeffs_t, const spuma_scalar* source, spuma_scalar* psi,
                               const spuma_solver_controls* ctl, const spuma_preconditioner* pc,
                               spuma_solver_perf* perf);

/*
 * Diagnostics of the above: w = M^-1 r (transpose != 0: M^-T r) with M built from
 * (diag, upper, lower) (lower NULL: = upper), and y = A x (transpose: A^T x) of the
 * asymmetric matrix.  Arrays [n_cells] / [n_faces] in the caller's numbering.
 */
spuma_status spuma_precondition(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                                const spuma_scalar* lower, const spuma_preconditioner* pc, const spuma_scalar* r,
                                spuma_scalar* w, int transpose);
spuma_status spuma_amul_asym(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                             const spuma_scalar* lower, const spuma_scalar* x, spuma_scalar* y, int transpose);

/*
 * LDU -> CSR (Q34, the map AmgX-style consumers need): row_ptr [n_cells+1],
 * col [n_cells + 2 n_faces] with ascending columns per row, map [same] indexing the
 * concatenation [diag | upper | lower]; host or device pointers.  The values of a matrix are
 * then spuma_csr_values (a device gather).  Handles built with renumber = 0 only
 * (SPUMA_ERR_STATE otherwise): the CSR is in the caller's numbering.
 */
spuma_status spuma_ldu_to_csr(spuma_mesh m, spuma_label* row_ptr, spuma_label* col, spuma_label* map);
spuma_status spuma_csr_values(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                              const spuma_scalar* lower, spuma_scalar* values);

/* ---------------- host-only diagnostics (no device access) ----------------
 * The host logic of libspuma, callable without a GPU so it can be checked on any machine:
 * addressing validation + RCM (A0/A1, Q12), the GAMG hierarchy (Q22: faceAreaPair pairing on
 * face_weights, n_coarsest / max_levels as spuma_gamg_params), the DIC/DILU dependency
 * schedules (rows sorted by dependency level) and the LDU -> CSR map (Q34).  All arrays are
 * host memory in the caller's numbering; owner/neighbour must be valid lduAddressing
 * (SPUMA_ERR_ADDRESSING otherwise).  ftc: the fine-to-coarse maps of every level but the
 * coarsest, concatenated (sum of level_cells[0 .. n_levels-2] entries).  order_*: [n_cells]. */
spuma_status spuma_host_rcm(int n_cells, int n_faces, const spuma_label* owner, const spuma_label* neighbour,
                            spuma_label* perm);
/* The lattice test of Amul variant 12: *n_offsets = K if every internal face's
 * column offset neighbour - owner takes one of K <= 3 values with no repeated (owner, neighbour)
 * pair (offsets[0..K-1] ascending), else 0.  Errors: ADDRESSING for an invalid lduAddressing. */
spuma_status spuma_host_lattice_offsets(int n_cells, int n_faces, const spuma_label* owner,
                                        const spuma_label* neighbour, int* n_offsets, int* offsets);
spuma_status spuma_host_gamg_hierarchy(int n_cells, int n_faces, const spuma_label* owner,
                                       const spuma_label* neighbour, const spuma_scalar* face_weights,
                                       int n_coarsest, int max_levels, int max_out, int* n_levels,
                                       int* level_cells, int* level_faces, spuma_label* ftc);
/* The decomposed GAMG hierarchy (Q36, Q37) of n_ranks sub-domains, built by the library's host code
 * with an in-process transport (one thread per rank standing in for the collectives).  Per rank r:
 * lduAddressing owner[r] / neighbour[r] [n_faces[r]], face_weights[r], its n_patches[r]
 * processor patches (patch_peer[r][p], patch_count[r][p]) and if_cell[r] (their face cells,
 * patch order).  Out: *n_levels; level_cells[64 r + l], level_ifaces[64 r + l] (may be NULL). */
spuma_status spuma_host_gamg_hierarchy_dd(int n_ranks, const int* n_cells, const int* n_faces,
                                          const spuma_label* const* owner, const spuma_label* const* neighbour,
                                          const spuma_scalar* const* face_weights, const int* n_patches,
                                          const int* const* patch_peer, const int* const* patch_count,
                                          const spuma_label* const* if_cell, int n_coarsest, int max_levels,
                                          int* n_levels, int* level_cells, int* level_ifaces);
spuma_status spuma_host_level_schedule(int n_cells, int n_faces, const spuma_label* owner,
                                       const spuma_label* neighbour, spuma_label* order_f, spuma_label* order_b,
                                       int* depth_f, int* depth_b);
spuma_status spuma_host_ldu_to_csr(int n_cells, int n_faces, const spuma_label* owner, const spuma_label* neighbour,
                                   spuma_label* row_ptr, spuma_label* col, spuma_label* map);

/* ---------------- around the path (the pressure step's neighbours) ----------------
 * Oriented face fields (phi, flux) are owner -> neighbour in the CALLER's numbering; with
 * renumber = 1 faces whose owner/neighbour swapped are negated on entry and exit.  Per-patch
 * arrays are arrays of per-patch pointers (NULL entries read as zero / are not written). */

/* fvc::surfaceIntegrate (profile row "surfaceIntegrate") -- the pressure
 * source fvc::div(phiHbyA):  out[c] = (sum of the outward fluxes of c: +phi on faces it owns,
 * -phi on faces where it is the neighbour, +patch_phi on its non-empty boundary faces) / V[c],
 * accumulated in face order, then (patch, face) order.  phi [n_faces], V, out [n_cells]. */
spuma_status spuma_surface_integrate(spuma_mesh m, const spuma_scalar* phi, const spuma_scalar* const* patch_phi,
                                     const spuma_scalar* V, spuma_scalar* out);

/* fvMatrix::flux of the assembled fvm::laplacian(gamma, psi) (lduMatrix::faceH):
 *   internal  flux[f] = upper[f] psi[N] - upper[f] psi[P]  (+ corr_flux[f])
 *   boundary  internalCoeffs psi_P - boundaryCoeffs (x psi_remote on processor faces):
 *             fixedValue (g|S|)(-delta) psi_P - (-(g|S|))(delta p_b); zeroGradient/empty 0
 *             (+ patch_corr_flux).
 * gamma / patch_value as given to spuma_assemble_laplacian; corr_flux / patch_corr_flux: the
 * faceFluxCorrection of spuma_laplacian_correction (NULL: none); flux [n_faces] and patch_flux
 * may be NULL; if phi (and/or patch_phi) is given the SIMPLE correction phi -= flux is applied in
 * place.  n_ranks > 1: collective (psi and gamma halo). */
spuma_status spuma_face_flux(spuma_mesh m, const spuma_scalar* gamma, const spuma_scalar* const* patch_value,
                             const spuma_scalar* upper, const spuma_scalar* psi, const spuma_scalar* corr_flux,
                             const spuma_scalar* const* patch_corr_flux, spuma_scalar* flux,
                             spuma_scalar* const* patch_flux, spuma_scalar* phi, spuma_scalar* const* patch_phi);

/* Explicit non-orthogonal correction of "Gauss linear corrected" (laplacianSchemes P:1135,
 * snGradSchemes corrected P:1145, gradSchemes Gauss linear P:1112; reading Q21):
 *   grad p   Gauss linear: (sum of Sf p_f over the faces of c) / V, p_f = w (p_P - p_N) + p_N,
 *            boundary p_b = p_P (zeroGradient), the patch value (fixedValue), the interpolate
 *            with the remote cell (processor)
 *   corr_f   (gamma_f |S|) (corrVec . (w (grad_P - grad_N) + grad_N)),
 *            corrVec = Sf/|Sf| - (C_N - C_P) nonOrthDeltaCoeff (0 on non-coupled patches)
 *   source  -= V fvc::div(corr)   (read-modified-written, like spuma_assemble_laplacian's)
 * p, V [n_cells]; corr_flux [n_faces] / patch_corr_flux (outputs, may be NULL) for
 * spuma_face_flux.  n_ranks > 1: collective (p, gamma and gradient halo). */
spuma_status spuma_laplacian_correction(spuma_mesh m, const spuma_scalar* gamma,
                                        const spuma_scalar* const* patch_value, const spuma_scalar* p,
                                        const spuma_scalar* V, spuma_scalar* source, spuma_scalar* corr_flux,
                                        spuma_scalar* const* patch_corr_flux);

/* ---------------- diagnostics (parity tests, benchmark harness) ---------------- */

/* y = A x (lduMatrix::Amul), with the processor-interface terms when
 * n_ranks > 1 (collective halo exchange of x). */
spuma_status spuma_amul(spuma_mesh m, const spuma_scalar* diag, const spuma_scalar* upper,
                        const spuma_scalar* iface_coeffs, const spuma_scalar* x, spuma_scalar* y);

/* Host copies of the derived addressing, INTERNAL numbering (after renumbering).
 * perm [n_cells] (perm[caller cell] = internal cell), owner/neighbour [n_faces],
 * owner_start/losort_start [n_cells+1], losort [n_faces], face_map [n_faces]
 * (face_map[internal face] = caller face).  Any pointer may be NULL. */
spuma_status spuma_mesh_get_addressing(spuma_mesh m, spuma_label* perm, spuma_label* owner,
                                       spuma_label* neighbour, spuma_label* owner_start, spuma_label* losort,
                                       spuma_label* losort_start, spuma_label* face_map);

/* Host copies of the A3 geometry in CALLER face order: delta [n_faces]
 * (nonOrthDeltaCoeffs), weights [n_faces], bdelta [total boundary faces in
 * patch order, empty patches included as 0]. Any pointer may be NULL. */
spuma_status spuma_mesh_get_geometry(spuma_mesh m, spuma_scalar* delta, spuma_scalar* weights,
                                     spuma_scalar* bdelta);

typedef struct {
    uint64_t kernel_launches;        /* kernels this handle launched (graph nodes counted per replay) */
    uint64_t solves, iterations;     /* totals over the handle's life                                 */
    int timing_enabled;
    /* phase timing (CUDA events on the handle's stream, enabled by spuma_set_timing):
       [0] direction (pA = rD rA + beta pA), [1] Amul + wA.pA, [2] update + residual dots,
       [3] assembly (face coefficients + diagonal gather) */
    double phase_ms[4];
    uint64_t phase_count[4];
    int blocks_per_grid, threads_per_block, batch_iterations;
    int amul_variant;                /* the A7 layout the hot loop runs on this mesh (after fallbacks:
                                        12 lattice slots -> 10 ELL -> 6 SELL -> 5 per-row)          */
    /* persistent loop (SPUMA_OPT_PERSISTENT) of the last spuma_pcg_solve: the mode it ran (0: the
       captured graph batches), its CTAs (one per SM), the rA pairs per thread held in tensor /
       shared memory, and with timing on the device time of its launches (CUDA events) */
    int loop_mode, loop_grid, loop_tmem_pairs, loop_smem_pairs;
    double loop_ms;
    uint64_t loop_count;
    /* with SPUMA_OPT_LOOP_PROFILE: per phase (0 direction, 1 Amul, 2 update) the time from the previous grid
       barrier's release to a CTA's arrival at the next (work) and from arrival to release (wait),
       summed over the iterations, mean over the CTAs; work_max: the slowest CTA's */
    double loop_work_ms[3], loop_wait_ms[3], loop_work_max_ms[3];
    int loop_threads;                /* threads per CTA of the persistent loop (its tile width in cell pairs) */
} spuma_stats;

spuma_status spuma_get_stats(spuma_mesh m, spuma_stats* out);
spuma_status spuma_reset_stats(spuma_mesh m);
/* Record CUDA events around every hot-loop kernel (adds event nodes to the
 * captured iteration graphs); off by default. */
spuma_status spuma_set_timing(spuma_mesh m, int enable);
/* Iterations per captured CUDA-graph batch (default 16; 1..256). */
spuma_status spuma_set_batch(spuma_mesh m, int iterations);

/* Tuning options.  SPUMA_OPT_AMUL_VARIANT selects the A7 kernel (all variants are
 * bitwise identical): 0 per-row, 1 CTA tile, 2 unrolled per-row, 3 TMA
 * producer/consumer pipeline (cp.async.bulk + mbarrier), 4 per-row at 8 CTAs/SM,
 * 5 unrolled two rows per thread, 6/7 SELL-C-32 slot layout with packed neighbour
 * side (one / two rows per thread), 8/9 ELL with a per-solve owner-slot ordered
 * coefficient copy (no row extents streamed; one / two rows per thread), 10 (default) the
 * ELL rows of 8 software-pipelined (the next row's slot loads issued before the current
 * row's gathers), 11 the ELL rows with the first-level loads streamed by a per-warp
 * cp.async.bulk ring into shared memory (measured slower; A/B only), 12 (default) lattice
 * slots: on a structured numbering (every face offset neighbour - owner one of <= 3 values,
 * spuma_host_lattice_offsets) the rows need no index arrays and every load of a row is
 * independent (falls back to 10 on other meshes), 13 the same with two rows per thread.
 * Errors: INVALID_ARGUMENT. */
typedef enum {
    SPUMA_OPT_AMUL_VARIANT = 0,
    /* meshes with at most this many cells (single rank) are solved by one single-CTA
     * kernel launch (latency path, BASELINE config 1); default 8192; 0 disables.  Above 3072
     * cells the persistent loop takes precedence where it can run (SPUMA_OPT_PERSISTENT). */
    SPUMA_OPT_SMALL_SOLVE_MAX_CELLS = 1,
    /* programmatic dependent launch of the hot-loop kernels (1 = on, default; process-wide) */
    SPUMA_OPT_PDL = 2,
    /* apply psi += alpha pA for two iterations at once (psi = (psi + a1 p1) + a2 p2: the same
     * roundings, fewer bytes): 0 = every iteration, 1 = the pairs in the update pass (which then
     * reads both directions), 2 = the pairs in the direction pass of every even iteration, where
     * the previous direction is read anyway and the one before is the value being overwritten
     * (default: 4 B/cell per iteration fewer than 1) */
    SPUMA_OPT_DEFER_PSI = 3,
    /* GAMG: the levels from the first one (below the finest) with at most this many cells
     * down to the coarsest run in ONE single-CTA kernel per V-cycle (Richardson, scaled
     * correction, nPre = 0); default 512 (same-box A/B r01q: 512 best, 256/1024 within 1.5 %,
     * 2048+ slower); 0 = one
     * launch per level and step */
    SPUMA_OPT_GAMG_TAIL_CELLS = 4,
    /* PCG hot loop: form the direction pA = rD rA + beta pA inside the Amul gather instead of
     * a separate pass (single rank, deferred psi, ELL layout; bitwise the same iterates).
     * 0 = separate k_direction (default: measured faster); 1 = fused, rD read;
     * 2 = fused, rD = 1/diag in place */
    SPUMA_OPT_FUSE_DIRECTION = 5,
    /* PCG hot loop: alternate the cell sweep direction of consecutive kernels (direction
     * ascending, Amul descending, update ascending, next iteration the reverse) so that each
     * kernel starts on the lines its predecessor left in L2.  Same operations per element;
     * only the order of the per-thread partial sums of the dots changes (deterministic).
     * 1 = on (default), 0 = all ascending */
    SPUMA_OPT_ALT_SWEEP = 6,
    /* ELL Amul (variant 8): chunks of 32 cells whose column offsets (col - c) take at most 3
     * values per side store those offsets once per chunk and one 32-bit word per cell instead
     * of 6 explicit 32-bit slot indices (~19 B/cell less; bitwise the same rows).  0 = explicit
     * slots everywhere (default: same-box A/B at 200^3 measured no gain -- the row gather is
     * bound by its two dependent load levels, not by the bytes), 1 = on */
    SPUMA_OPT_ELL_STENCIL = 7,
    /* PCG hot loop: an L2 access-policy window (persisting hits) captured into the iteration
     * graphs over one workspace vector: 0 = none, 1 = pA, 2 = rA (default), 3 = rD, 4 = wA.
     * Sets the device-wide persisting-L2 limit while the handle lives (reset by spuma_free or
     * by setting 0).  Same-box A/B at 200^3: 161 us per iteration without a window, 150.5 with
     * rA or pA (profiles/r02n_l2_target_ab.log). */
    SPUMA_OPT_L2_PERSIST = 8,
    /* GAMG: the coarse levels without uniform widths run their rows over a per-level CSR copy of
     * the off-diagonal coefficients (row_ax order; bitwise the same rows); 1 = on (default),
     * 0 = the losort-addressed rows.  Rebuilds the hierarchy at the next solve. */
    SPUMA_OPT_GAMG_CSR = 9,
    /* peer transport: how long a kernel polls for a neighbour's flag before it gives up, in
     * milliseconds (approximate: SM clocks at 2 GHz); default 20000.  The call that saw the
     * timeout returns SPUMA_ERR_STATE.  Also the persistent loop's grid-barrier limit. */
    SPUMA_OPT_PEER_POLL_MS = 10,
    /* the single-CTA small solve (SPUMA_OPT_SMALL_SOLVE_MAX_CELLS) with the matrix, addressing,
     * vectors and scalars staged in shared memory when they fit (about 1700 cells of a 3-D hex
     * mesh); 1 = on (default), 0 = global memory.  Bitwise the same iterates. */
    SPUMA_OPT_SMALL_SMEM = 11,
    /* peer transport, PCG loop: the halo stores fused into the direction kernel and the receive
     * into the interface rows, the rank-partial all-gather + finalisation into the reductions'
     * last CTA (4 kernels per iteration instead of 7); 1 = on (default), 0 = separate kernels.
     * Bitwise the same iterates. */
    SPUMA_OPT_PEER_FUSED = 12,
    /* single-rank PCG (lattice, ELL or SELL-C layout, deferred psi pairs in the direction): run every
     * iteration of a solve in ONE cooperative launch of one 896-thread CTA per SM, three grid
     * barriers per iteration, each CTA finalising the scalars itself; the residual rA stays on
     * the SM: 0 = off (captured graph batches), 1 = persistent, rA in HBM, 2 = rA in shared
     * memory (the rest in HBM), 3 = rA in tensor memory + shared memory (default; ~8.2M cells
     * fully on chip on 148 SMs).  Modes 2 and 3 fall back to the graph batches when less than
     * half of rA fits on chip (meshes above ~17M cells), and any mode when the cooperative launch
     * does not fit the device.  The Amul runs over the lattice slots (variant 12) or, on other
     * meshes, over the ELL rows (variant 8/10 layout) or the SELL-C rows (variant 6).  Above
     * SPUMA_OPT_SMALL_SOLVE_MAX_CELLS's 3072-cell cut it also replaces the single-CTA solve.  Same
     * element arithmetic as the graph
     * path; the dot products are summed in another fixed shape (iterates equal to rounding,
     * deterministic). */
    SPUMA_OPT_PERSISTENT = 13,
    /* the persistent loop's L2 access-policy window (persisting hits), targets as
     * SPUMA_OPT_L2_PERSIST: 0 = none, 1 = pA (default), 2 = rA, 3 = rD, 4 = wA.  Same-box A/B at
     * 200^3 with the final loop (profiles/r02bk_*, r02bl_*): 155.7 / 137.0 / 142.4 / 138.3 us per
     * iteration for none / pA / rD / wA (pA also ahead at 126^3 and 159^3). */
    SPUMA_OPT_LOOP_L2 = 14,
    /* the persistent loop records, per CTA and phase, the time from one grid barrier's release to
     * its arrival at the next (work) and the wait there (globaltimer; spuma_stats.loop_work_ms /
     * loop_wait_ms / loop_work_max_ms); 0 = off (default), 1 = on */
    SPUMA_OPT_LOOP_PROFILE = 15,
    /* CTAs of the persistent loop: 0 = automatic (default: 32 per started 16384 cells, at most
     * one per SM), else at most this many */
    SPUMA_OPT_LOOP_GRID = 16
} spuma_option;
spuma_status spuma_set_option(spuma_mesh m, int option, int value);

/* External communication, used when n_ranks > 1 and desc.nccl_unique_id == NULL
 * (a host transport instead of NCCL -- e.g. several ranks sharing one GPU in tests).
 * Must be set before the first collective call.  Buffers are host memory; both
 * callbacks are collective across ranks and return 0 on success (else the calling
 * spuma_* function fails with SPUMA_ERR_NCCL).  The device path is unchanged except
 * that the iteration batches are launched directly (host callbacks are not capturable).
 *   exchange:  for i < n_peers send send[offsets[i] .. +counts[i]) to rank peers[i] and
 *              receive counts[i] doubles from it into recv[offsets[i] ..) (processor-patch
 *              halo, faces in ascending undecomposed face id on both sides, Q13)
 *   allgather: n doubles from every rank into recv[n * rank ..), rank order */
typedef struct {
    void* ctx;
    int (*exchange)(void* ctx, int n_peers, const int* peers, const int* offsets, const int* counts,
                    const double* send, double* recv);
    int (*allgather)(void* ctx, const double* send, double* recv, int n);
} spuma_comm_callbacks;
spuma_status spuma_set_comm_callbacks(spuma_mesh m, const spuma_comm_callbacks* cb);

/* Peer-memory transport (halo and rank-partial exchanges as direct stores
 * into the neighbours' device memory over NVLink, no NCCL).  Every rank calls
 * spuma_peer_export (allocates its mailbox and writes a SPUMA_PEER_BLOB_BYTES description:
 * CUDA IPC handle, rank, processor patches), the blobs are all-gathered by the caller (any
 * host transport), and every rank calls spuma_peer_import with the n_ranks blobs in rank
 * order ([n_ranks][SPUMA_PEER_BLOB_BYTES] bytes).  From then on every collective of the handle
 * (PCG, PCG-pc, PBiCG, GAMG, assembly halos) runs as device kernels: the halo pack is fused
 * into the P2P stores, completion is signalled by system-scope release/acquire epoch flags,
 * and the iteration batches stay CUDA-graph captured.  Ranks may share one GPU (tests).
 * spuma_peer_check returns SPUMA_ERR_STATE if a poll ever timed out (~20 s).
 * Errors: INVALID_ARGUMENT (n_ranks > 64, > 32 processor patches, bad or out-of-order blobs),
 * ADDRESSING (the ranks' processor patches do not pair up), STATE, CUDA. */
#define SPUMA_PEER_BLOB_BYTES 512
spuma_status spuma_peer_export(spuma_mesh m, void* blob);
spuma_status spuma_peer_import(spuma_mesh m, const void* blobs, int n_blobs);
spuma_status spuma_peer_check(spuma_mesh m);

/* Fill out128 with a fresh ncclUniqueId (rank 0 calls it and broadcasts). */
spuma_status spuma_nccl_get_unique_id(void* out128);

/* Message of the last non-OK status on this thread ("" if none). */
const char* spuma_last_error(void);

/* ABI version the library was built with. */
int spuma_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPUMA_H */
