/*
 * oracle/oracle.c -- the CPU ORACLE for the SPUMA pressure path (arXiv 2512.22215).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this code.
 * The product (paper_2512_22215_b200, libspuma) never links, imports or
 * executes it, and this file shares no code, header, table or helper with it.
 *
 * Plain, slow, single-threaded, fp64, built with -O2 -ffp-contract=off (no FMA
 * contraction, round-to-nearest-even).  Every function follows the OpenFOAM
 * definitions the paper relies on ("SPUMA ... reproduces OpenFOAM-v2412",
 * PAPER.md P:371) in their plain face-loop form; readings where the
 * paper is silent are DESIGN.md §3 (Q1..Q16).
 *
 *   O1 addressing   or_check_addressing, or_owner_start, or_losort       P:82-83 (lduAddressing)
 *   O2 renumbering  or_rcm, or_renumber_faces                            BASELINE.json "renumbered cells"; reading Q12
 *   O3 geometry     or_geometry, or_boundary_delta, or_processor_geometry P:1133-1146 ("Gauss linear corrected", linear)
 *   O4 assembly     or_assemble                                           P:736 "P assembly", P:520 negSumDiag
 *   O5 Amul         or_amul, or_sumA                                      P:506 "SpMVM (Amul + Tmul)", P:519 sumA
 *   O6 PCG          or_pcg (P >= 1 domains, O8 when P > 1)                P:961, P:1033-1041 (pcgDiag)
 *   O7 dense        or_dense_from_ldu, or_dense_matvec, or_dense_solve    brute force for N <= 64
 *   O9 around       or_surface_integrate, or_face_flux
 *   O10 non-orth    or_gauss_grad, or_nonorth_flux                        P:1112, P:1135, P:1145 (Gauss linear corrected)
 *   O12 precond.    or_ilu_factor, or_ilu_precondition, or_pcg_pc, or_pbicg, or_tmul, or_ldu_to_csr
 *                   P:509
 *   O11 GAMG        or_agglomerate, or_coarse_addressing, or_agglomerate_matrix, or_restrict, or_gamg
 *                   P:517
 *   O11dd GAMG dd   or_gamg_dd, or_gamg_dd_dense_level (decomposed hierarchy, coarse interfaces;
 *                   readings Q36-Q38)
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): SPEC chain examples,
 * closed-form Poisson eigenmodes (Dirichlet / Neumann) and linear exactness,
 * dense brute force, symmetry / zero-row-sum / Sigma diag invariants,
 * decomposition invariance, A-norm monotonicity.
 * Parity unpinned: the normFactor formula (Q1) and the convergence/loop
 * semantics (Q2, Q3) are pinned only by special cases (init residual = 1 for
 * psi0 = 0, and for a constant psi0 on Neumann and Dirichlet matrices -- the
 * latter separating the xRef = sumA mean(psi) term from the reference-free
 * readings; exact start; minIter), not by any number the paper prints -- the
 * paper prints no PCG iteration count, residual or matrix value for this path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* O1 addressing ("the mesh data structure reflects the sparsity     */
/* pattern of the matrix"; SPEC S:275-281 invariants)                         */
/* ------------------------------------------------------------------------- */

/* 0 = valid; 2 = addressing violation (index range, owner >= neighbour, order) */
int or_check_addressing(int n_cells, int n_faces, const int* owner, const int* neighbour)
{
    for (int f = 0; f < n_faces; ++f) {
        if (owner[f] < 0 || owner[f] >= n_cells || neighbour[f] < 0 || neighbour[f] >= n_cells) return 2;
        if (!(owner[f] < neighbour[f])) return 2;
        if (f > 0) {
            if (owner[f] < owner[f - 1]) return 2;
            if (owner[f] == owner[f - 1] && neighbour[f] < neighbour[f - 1]) return 2;
        }
    }
    return 0;
}

/* ownerStart[c] = number of faces with owner < c (faces sorted by owner) */
void or_owner_start(int n_cells, int n_faces, const int* owner, int* owner_start)
{
    for (int c = 0; c <= n_cells; ++c) {
        int lo = 0, hi = n_faces; /* first face with owner >= c */
        while (lo < hi) {
            int mid = lo + (hi - lo) / 2;
            if (owner[mid] < c) lo = mid + 1;
            else hi = mid;
        }
        owner_start[c] = lo;
    }
}

typedef struct { int key; int face; } or_pair;
static int or_pair_cmp(const void* a, const void* b)
{
    const or_pair* x = (const or_pair*)a;
    const or_pair* y = (const or_pair*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->face < y->face ? -1 : (x->face > y->face);
}

/* losort = faces sorted by neighbour, ties by face index; losortStart[c] = #faces with neighbour < c */
void or_losort(int n_cells, int n_faces, const int* neighbour, int* losort, int* losort_start)
{
    or_pair* p = (or_pair*)malloc(sizeof(or_pair) * (size_t)(n_faces > 0 ? n_faces : 1));
    for (int f = 0; f < n_faces; ++f) {
        p[f].key = neighbour[f];
        p[f].face = f;
    }
    qsort(p, (size_t)n_faces, sizeof(or_pair), or_pair_cmp);
    for (int k = 0; k < n_faces; ++k) losort[k] = p[k].face;
    for (int c = 0; c <= n_cells; ++c) {
        int lo = 0, hi = n_faces;
        while (lo < hi) {
            int mid = lo + (hi - lo) / 2;
            if (p[mid].key < c) lo = mid + 1;
            else hi = mid;
        }
        losort_start[c] = lo;
    }
    free(p);
}

/* ------------------------------------------------------------------------- */
/* O2 reverse Cuthill-McKee with fixed tie-breaks (reading Q12)              */
/* ------------------------------------------------------------------------- */

static const int* or_rcm_deg;
static int or_deg_cmp(const void* a, const void* b)
{
    int x = *(const int*)a, y = *(const int*)b;
    if (or_rcm_deg[x] != or_rcm_deg[y]) return or_rcm_deg[x] < or_rcm_deg[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

/*
 * perm[old] = new.  Graph = cells with internal faces as edges; deg(c) = number
 * of internal faces of c.  Start at the unvisited cell of minimum degree (ties:
 * smallest index), BFS with a FIFO queue; a dequeued cell enqueues its
 * unvisited neighbours sorted by (deg, index).  Restart per component.
 * Visit order k -> new[c_k] = N-1-k.
 */
int or_rcm(int n_cells, int n_faces, const int* owner, const int* neighbour, int* perm)
{
    int* deg = (int*)calloc((size_t)n_cells + 1, sizeof(int));
    int* start = (int*)calloc((size_t)n_cells + 2, sizeof(int));
    int* adj = (int*)malloc(sizeof(int) * (size_t)(2 * n_faces + 1));
    int* fill = (int*)calloc((size_t)n_cells + 1, sizeof(int));
    char* seen = (char*)calloc((size_t)n_cells + 1, 1);
    int* queue = (int*)malloc(sizeof(int) * (size_t)(n_cells + 1));
    int* cand = (int*)malloc(sizeof(int) * (size_t)(2 * n_faces + 1));
    if (!deg || !start || !adj || !fill || !seen || !queue || !cand) return 6;
    for (int f = 0; f < n_faces; ++f) {
        deg[owner[f]]++;
        deg[neighbour[f]]++;
    }
    for (int c = 0; c < n_cells; ++c) start[c + 1] = start[c] + deg[c];
    for (int f = 0; f < n_faces; ++f) {
        adj[start[owner[f]] + fill[owner[f]]++] = neighbour[f];
        adj[start[neighbour[f]] + fill[neighbour[f]]++] = owner[f];
    }
    or_rcm_deg = deg;
    int k = 0;
    while (k < n_cells) {
        int s = -1;
        for (int c = 0; c < n_cells; ++c)
            if (!seen[c] && (s < 0 || deg[c] < deg[s])) s = c;
        int head = k, tail = k;
        queue[tail++] = s;
        seen[s] = 1;
        while (head < tail) {
            int c = queue[head++];
            int nc = 0;
            for (int e = start[c]; e < start[c + 1]; ++e) {
                int d = adj[e];
                if (!seen[d]) {
                    seen[d] = 1; /* marks duplicates (several faces to one cell) once */
                    cand[nc++] = d;
                }
            }
            qsort(cand, (size_t)nc, sizeof(int), or_deg_cmp);
            for (int i = 0; i < nc; ++i) queue[tail++] = cand[i];
        }
        k = tail;
    }
    for (int i = 0; i < n_cells; ++i) perm[queue[i]] = n_cells - 1 - i;
    free(deg);
    free(start);
    free(adj);
    free(fill);
    free(seen);
    free(queue);
    free(cand);
    return 0;
}

typedef struct { int o, n, f; } or_triple;
static int or_triple_cmp(const void* a, const void* b)
{
    const or_triple* x = (const or_triple*)a;
    const or_triple* y = (const or_triple*)b;
    if (x->o != y->o) return x->o < y->o ? -1 : 1;
    if (x->n != y->n) return x->n < y->n ? -1 : 1;
    return x->f < y->f ? -1 : (x->f > y->f);
}

/*
 * Re-key faces under perm[old] = new: (a, b) = (new[P], new[N]); owner = min,
 * neighbour = max; flip[g] = 1 iff the pair swapped (Sf must be negated);
 * faces re-sorted by (owner, neighbour), ties by old face index.
 * face_map[new face] = old face.
 */
void or_renumber_faces(int n_faces, const int* perm, const int* owner, const int* neighbour, int* owner_out,
                       int* neighbour_out, int* face_map, signed char* flip)
{
    or_triple* t = (or_triple*)malloc(sizeof(or_triple) * (size_t)(n_faces > 0 ? n_faces : 1));
    for (int f = 0; f < n_faces; ++f) {
        int a = perm[owner[f]], b = perm[neighbour[f]];
        t[f].o = a < b ? a : b;
        t[f].n = a < b ? b : a;
        t[f].f = f;
    }
    qsort(t, (size_t)n_faces, sizeof(or_triple), or_triple_cmp);
    for (int g = 0; g < n_faces; ++g) {
        owner_out[g] = t[g].o;
        neighbour_out[g] = t[g].n;
        face_map[g] = t[g].f;
        flip[g] = (signed char)(perm[owner[t[g].f]] > perm[neighbour[t[g].f]]);
    }
    free(t);
}

/* ------------------------------------------------------------------------- */
/* O3 geometry: [OF] surfaceInterpolation::makeNonOrthDeltaCoeffs (the       */
/* "stabilised form for bad meshes") and makeWeights; "Gauss linear          */
/* corrected" laplacian, "linear" interpolation.  Reading Q6.  */
/* ------------------------------------------------------------------------- */

static void or_face_geometry(const double* CP, const double* CN, const double* S, double magS, const double* Cf,
                             double* delta, double* weight)
{
    double d[3], nh[3];
    for (int k = 0; k < 3; ++k) d[k] = CN[k] - CP[k];
    for (int k = 0; k < 3; ++k) nh[k] = S[k] / magS;
    double nd = nh[0] * d[0] + nh[1] * d[1] + nh[2] * d[2];
    double magd = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double lim = 0.05 * magd;
    *delta = 1.0 / (nd > lim ? nd : lim);

    double eo[3], en[3];
    for (int k = 0; k < 3; ++k) {
        eo[k] = Cf[k] - CP[k];
        en[k] = CN[k] - Cf[k];
    }
    double SfdOwn = fabs(S[0] * eo[0] + S[1] * eo[1] + S[2] * eo[2]);
    double SfdNei = fabs(S[0] * en[0] + S[1] * en[1] + S[2] * en[2]);
    double den = SfdOwn + SfdNei;
    *weight = den > 1e-150 ? SfdNei / den : 0.5;
}

void or_geometry(int n_faces, const int* owner, const int* neighbour, const double* Sf, const double* magSf,
                 const double* C, const double* Cf, double* delta, double* weights)
{
    for (int f = 0; f < n_faces; ++f)
        or_face_geometry(C + 3 * owner[f], C + 3 * neighbour[f], Sf + 3 * f, magSf[f], Cf + 3 * f, delta + f,
                         weights + f);
}

/* non-coupled patch face of cell P: delta_b = 1 / (nhat . (Cf - C_P)) */
void or_boundary_delta(int n, const int* face_cells, const double* Sf, const double* magSf, const double* Cf,
                       const double* C, double* delta)
{
    for (int i = 0; i < n; ++i) {
        const double* cp = C + 3 * face_cells[i];
        double nh[3], e[3];
        for (int k = 0; k < 3; ++k) {
            nh[k] = Sf[3 * i + k] / magSf[i];
            e[k] = Cf[3 * i + k] - cp[k];
        }
        delta[i] = 1.0 / (nh[0] * e[0] + nh[1] * e[1] + nh[2] * e[2]);
    }
}

/* processor face, evaluated in the GLOBAL orientation (reading O3 / Q9) */
void or_processor_geometry(int n, const int* face_cells, const double* Sf_out, const double* magSf,
                           const double* Cf, const double* C, const double* neighbour_C, const signed char* is_owner,
                           double* delta, double* weights)
{
    for (int i = 0; i < n; ++i) {
        double S[3];
        const double *CP, *CN;
        if (is_owner[i]) {
            for (int k = 0; k < 3; ++k) S[k] = Sf_out[3 * i + k];
            CP = C + 3 * face_cells[i];
            CN = neighbour_C + 3 * i;
        } else {
            for (int k = 0; k < 3; ++k) S[k] = -Sf_out[3 * i + k];
            CP = neighbour_C + 3 * i;
            CN = C + 3 * face_cells[i];
        }
        or_face_geometry(CP, CN, S, magSf[i], Cf + 3 * i, delta + i, weights + i);
    }
}

/* ------------------------------------------------------------------------- */
/* O4 assembly of fvm::laplacian(gamma, p): [OF] gaussLaplacianScheme::      */
/* fvmLaplacianUncorrected, lduMatrix::negSumDiag, fvMatrix::        */
/* setReference (P:1083-1084 pRefCell/pRefValue), addBoundaryDiag,           */
/* addBoundarySource.  Readings Q6, Q7, Q9, Q15.                             */
/* ------------------------------------------------------------------------- */

enum { OR_ZERO_GRADIENT = 0, OR_FIXED_VALUE = 1, OR_EMPTY = 2, OR_PROCESSOR = 3 };

/*
 * Boundary faces are given concatenated in patch order; per face:
 *   bkind     patch kind
 *   bcells    local owner cell
 *   bmagSf    |S_b|
 *   bdelta    delta_b (non-coupled) or delta_f in global orientation (processor)
 *   bweight   processor only: global-orientation weight w
 *   bvalue    fixedValue only: p_b
 *   bgamma_r  processor only: gamma of the remote cell
 *   bis_owner processor only: 1 if the local cell is the global owner
 * iface receives, for processor faces only (in boundary order), the true matrix
 * entry A[P][remote] = delta_f (gamma_f |S_f|)  (reading Q9); other slots untouched.
 */
void or_assemble(int n_cells, int n_faces, const int* owner, const int* neighbour, const double* magSf,
                 const double* delta, const double* weights, const double* gamma, int n_bfaces, const int* bkind,
                 const int* bcells, const double* bmagSf, const double* bdelta, const double* bweight,
                 const double* bvalue, const double* bgamma_r, const signed char* bis_owner, int ref_cell,
                 double ref_value, double* diag, double* upper, double* source, double* iface)
{
    /* 1-2: face coefficients, upper = deltaCoeffs * (gamma_f * magSf); lower aliases upper */
    for (int f = 0; f < n_faces; ++f) {
        double gf = 1.0;
        if (gamma) gf = weights[f] * (gamma[owner[f]] - gamma[neighbour[f]]) + gamma[neighbour[f]];
        upper[f] = delta[f] * (gf * magSf[f]);
    }
    /* 3: negSumDiag, face order: Diag[l] -= Lower; Diag[u] -= Upper */
    for (int c = 0; c < n_cells; ++c) diag[c] = 0.0;
    for (int f = 0; f < n_faces; ++f) {
        diag[owner[f]] -= upper[f]; /* lower == upper */
        diag[neighbour[f]] -= upper[f];
    }
    /* 4: setReference before any boundary coefficient */
    if (ref_cell >= 0 && ref_cell < n_cells) {
        source[ref_cell] += diag[ref_cell] * ref_value;
        diag[ref_cell] += diag[ref_cell];
    }
    /* 5: boundary coefficients in (patch, face) order */
    for (int i = 0; i < n_bfaces; ++i) {
        int P = bcells[i];
        double gP = gamma ? gamma[P] : 1.0;
        if (bkind[i] == OR_FIXED_VALUE) {
            double gms = gP * bmagSf[i];
            diag[P] += gms * (-bdelta[i]);                   /* internalCoeffs = pGamma * (-delta)       */
            source[P] += (-gms) * (bdelta[i] * bvalue[i]);  /* boundaryCoeffs = -pGamma * (delta * p_b) */
        } else if (bkind[i] == OR_PROCESSOR) {
            double gf = 1.0;
            if (gamma) {
                double gO = bis_owner[i] ? gP : bgamma_r[i];
                double gN = bis_owner[i] ? bgamma_r[i] : gP;
                gf = bweight[i] * (gO - gN) + gN;
            }
            double gms = gf * bmagSf[i];
            diag[P] += gms * (-bdelta[i]);
            iface[i] = bdelta[i] * gms;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* O5 Amul and sumA: plain face-loop   */
/* scatter, then processor interfaces in order.                              */
/* ------------------------------------------------------------------------- */

void or_amul(int n_cells, int n_faces, const int* owner, const int* neighbour, const double* diag,
             const double* lower, const double* upper, const double* x, int n_iface, const int* iface_cells,
             const double* iface_coeffs, const double* x_remote, double* y)
{
    for (int c = 0; c < n_cells; ++c) y[c] = diag[c] * x[c];
    for (int f = 0; f < n_faces; ++f) {
        y[neighbour[f]] += lower[f] * x[owner[f]];
        y[owner[f]] += upper[f] * x[neighbour[f]];
    }
    for (int i = 0; i < n_iface; ++i) y[iface_cells[i]] += iface_coeffs[i] * x_remote[i];
}

void or_sumA(int n_cells, int n_faces, const int* owner, const int* neighbour, const double* diag,
             const double* lower, const double* upper, int n_iface, const int* iface_cells, const double* iface_coeffs,
             double* sumA)
{
    for (int c = 0; c < n_cells; ++c) sumA[c] = diag[c];
    for (int f = 0; f < n_faces; ++f) {
        sumA[owner[f]] += lower[f];
        sumA[neighbour[f]] += upper[f];
    }
    for (int i = 0; i < n_iface; ++i) sumA[iface_cells[i]] += iface_coeffs[i];
}

/* ------------------------------------------------------------------------- */
/* O9 around the path: fvc::surfaceIntegrate -- the pressure  */
/* source fvc::div(phiHbyA) -- and fvMatrix::flux (lduMatrix::faceH plus the  */
/* boundary contributions) for the flux correction phi = phiHbyA - flux.      */
/* Paper: profile rows "surfaceIntegrate" and "lduMatrix::faceH"      */
/* (P:553); SPEC S:620-626 (surface_integrate), S:325-331 (face_h).           */
/* ------------------------------------------------------------------------- */

/* out[c] = (sum over internal faces in face order of +phi (owner) / -phi (neighbour),
 * then the boundary faces of c in (patch, face) order, empty patches excluded) / V[c] */
void or_surface_integrate(int n_cells, int n_faces, const int* owner, const int* neighbour, const double* phi,
                          int n_bfaces, const int* bkind, const int* bcells, const double* bphi, const double* V,
                          double* out)
{
    for (int c = 0; c < n_cells; ++c) out[c] = 0.0;
    for (int f = 0; f < n_faces; ++f) {
        out[owner[f]] += phi[f];
        out[neighbour[f]] -= phi[f];
    }
    for (int b = 0; b < n_bfaces; ++b)
        if (bkind[b] != OR_EMPTY) out[bcells[b]] += bphi[b];
    for (int c = 0; c < n_cells; ++c) out[c] /= V[c];
}

/* fvMatrix::flux of the assembled fvm::laplacian(gamma, psi):
 *   internal (faceH):  flux[f] = Upper[f] psi[N] - Lower[f] psi[P]
 *   boundary:          internalCoeffs psi_P - boundaryCoeffs (x psi_remote when coupled), i.e.
 *     fixedValue:  (gms (-delta)) psi_P - ((-gms) (delta p_b))
 *     processor:   (gms (-delta)) psi_P - (((-gms) delta) psi_remote)   (global-orientation gms)
 *     zeroGradient / empty: 0 */
void or_face_flux(int n_faces, const int* owner, const int* neighbour, const double* lower, const double* upper,
                  const double* psi, double* flux, int n_bfaces, const int* bkind, const int* bcells,
                  const double* bmagSf, const double* bdelta, const double* bweight, const double* bvalue,
                  const double* bgamma_r, const signed char* bis_owner, const double* gamma,
                  const double* bpsi_r, double* bflux)
{
    for (int f = 0; f < n_faces; ++f) flux[f] = upper[f] * psi[neighbour[f]] - lower[f] * psi[owner[f]];
    for (int b = 0; b < n_bfaces; ++b) {
        const int P = bcells[b];
        const double gP = gamma ? gamma[P] : 1.0;
        bflux[b] = 0.0;
        if (bkind[b] == OR_FIXED_VALUE) {
            const double gms = gP * bmagSf[b];
            bflux[b] = (gms * (-bdelta[b])) * psi[P] - ((-gms) * (bdelta[b] * bvalue[b]));
        } else if (bkind[b] == OR_PROCESSOR) {
            double gf = 1.0;
            if (gamma) {
                const double gO = bis_owner[b] ? gP : bgamma_r[b];
                const double gN = bis_owner[b] ? bgamma_r[b] : gP;
                gf = bweight[b] * (gO - gN) + gN;
            }
            const double gms = gf * bmagSf[b];
            bflux[b] = (gms * (-bdelta[b])) * psi[P] - (((-gms) * bdelta[b]) * bpsi_r[b]);
        }
    }
}

/* ------------------------------------------------------------------------- */
/* O10 explicit non-orthogonal correction of "Gauss linear corrected"          */
/* (laplacianSchemes P:1135, snGradSchemes corrected P:1145, gradSchemes      */
/* default Gauss linear P:1112): [OF] gaussLaplacianScheme::fvmLaplacian,      */
/* correctedSnGrad::fullGradCorrection, gaussGrad::gradf,                     */
/* surfaceInterpolation::makeNonOrthCorrectionVectors.  Reading Q21.          */
/* ------------------------------------------------------------------------- */

/* gaussGrad (Gauss linear): p_f = w (p_P - p_N) + p_N on internal faces; G[owner] += Sf p_f,
 * G[neighbour] -= Sf p_f in face order; then every non-empty boundary face in (patch, face)
 * order adds bSf p_b, with p_b = p_P (zeroGradient), the patch value (fixedValue) or the
 * global-orientation interpolate with the remote cell (processor); then G /= V.
 * G is [3 N] (x, y, z per cell). */
void or_gauss_grad(int n_cells, int n_faces, const int* owner, const int* neighbour, const double* Sf,
                   const double* weights, const double* p, int n_bfaces, const int* bkind, const int* bcells,
                   const double* bSf, const double* bvalue, const double* bweight, const signed char* bis_owner,
                   const double* bp_r, const double* V, double* G)
{
    double* bp = (double*)malloc(sizeof(double) * (size_t)(n_bfaces > 0 ? n_bfaces : 1));
    for (int b = 0; b < n_bfaces; ++b) {
        const double pP = p[bcells[b]];
        if (bkind[b] == OR_FIXED_VALUE) bp[b] = bvalue[b];
        else if (bkind[b] == OR_PROCESSOR) {
            const double pO = bis_owner[b] ? pP : bp_r[b];
            const double pN = bis_owner[b] ? bp_r[b] : pP;
            bp[b] = bweight[b] * (pO - pN) + pN;
        } else bp[b] = pP;
    }
    for (int i = 0; i < 3 * n_cells; ++i) G[i] = 0.0;
    for (int f = 0; f < n_faces; ++f) {
        const double pf = weights[f] * (p[owner[f]] - p[neighbour[f]]) + p[neighbour[f]];
        for (int k = 0; k < 3; ++k) {
            G[3 * owner[f] + k] += Sf[3 * f + k] * pf;
            G[3 * neighbour[f] + k] -= Sf[3 * f + k] * pf;
        }
    }
    for (int b = 0; b < n_bfaces; ++b)
        if (bkind[b] != OR_EMPTY)
            for (int k = 0; k < 3; ++k) G[3 * bcells[b] + k] += bSf[3 * b + k] * bp[b];
    for (int c = 0; c < n_cells; ++c)
        for (int k = 0; k < 3; ++k) G[3 * c + k] /= V[c];
    free(bp);
}

/* nonOrthCorrectionVectors: corr = Sf/|Sf| - (C_N - C_P) nonOrthDeltaCoeff (per component) */
static void or_corr_vec(const double* S, double magS, const double* CP, const double* CN, double delta, double* cv)
{
    for (int k = 0; k < 3; ++k) cv[k] = S[k] / magS - (CN[k] - CP[k]) * delta;
}

/* correction flux gammaMagSf * (corrVec . linearInterpolate(grad p)) on internal faces (face
 * orientation) and processor faces (outward: the owner side carries the global value, the other
 * side its negation); 0 on non-coupled boundary faces. */
void or_nonorth_flux(int n_faces, const int* owner, const int* neighbour, const double* Sf, const double* magSf,
                     const double* C, const double* delta, const double* weights, const double* gamma,
                     const double* G, double* cflux, int n_bfaces, const int* bkind, const int* bcells,
                     const double* bSf, const double* bmagSf, const double* bdelta, const double* bweight,
                     const signed char* bis_owner, const double* bnC, const double* bgamma_r, const double* bG_r,
                     double* bcflux)
{
    for (int f = 0; f < n_faces; ++f) {
        const int P = owner[f], N = neighbour[f];
        double cv[3], g[3];
        or_corr_vec(Sf + 3 * f, magSf[f], C + 3 * P, C + 3 * N, delta[f], cv);
        for (int k = 0; k < 3; ++k) g[k] = weights[f] * (G[3 * P + k] - G[3 * N + k]) + G[3 * N + k];
        const double corr = cv[0] * g[0] + cv[1] * g[1] + cv[2] * g[2];
        double gf = 1.0;
        if (gamma) gf = weights[f] * (gamma[P] - gamma[N]) + gamma[N];
        cflux[f] = (gf * magSf[f]) * corr;
    }
    for (int b = 0; b < n_bfaces; ++b) {
        bcflux[b] = 0.0;
        if (bkind[b] != OR_PROCESSOR) continue;
        const int L = bcells[b];
        const int own = bis_owner[b];
        double S[3], cv[3], g[3];
        for (int k = 0; k < 3; ++k) S[k] = own ? bSf[3 * b + k] : -bSf[3 * b + k];
        const double* CL = C + 3 * L;
        const double* CR = bnC + 3 * b;
        or_corr_vec(S, bmagSf[b], own ? CL : CR, own ? CR : CL, bdelta[b], cv);
        for (int k = 0; k < 3; ++k) {
            const double gO = own ? G[3 * L + k] : bG_r[3 * b + k];
            const double gN = own ? bG_r[3 * b + k] : G[3 * L + k];
            g[k] = bweight[b] * (gO - gN) + gN;
        }
        const double corr = cv[0] * g[0] + cv[1] * g[1] + cv[2] * g[2];
        double gf = 1.0;
        if (gamma) {
            const double gO = own ? gamma[L] : bgamma_r[b];
            const double gN = own ? bgamma_r[b] : gamma[L];
            gf = bweight[b] * (gO - gN) + gN;
        }
        const double q = (gf * bmagSf[b]) * corr;
        bcflux[b] = own ? q : -q;
    }
}

/* ------------------------------------------------------------------------- */
/* O6 PCG + diagonal preconditioner ([OF] PCG::scalarSolve,                  */
/* lduMatrix::solver::normFactor, SolverPerformance::checkConvergence /      */
/* checkSingularity; controls P:1033-1041).  Readings Q1-Q5, Q11.            */
/* P > 1 domains = O8 decomposed oracle: x_remote copied between domains     */
/* before each Amul, global sums = per-domain sums added in rank order.      */
/* ------------------------------------------------------------------------- */

typedef struct {
    int n_cells, n_faces;
    const int* owner;
    const int* neighbour;
    const double* diag;
    const double* upper; /* symmetric: lower == upper */
    const double* source;
    double* psi;
    int n_iface;
    const int* iface_cells;
    const double* iface_coeffs;
    const int* iface_src_domain; /* x_remote[i] = x of domain iface_src_domain[i] ... */
    const int* iface_src_cell;   /* ... at its local cell iface_src_cell[i]           */
} or_domain;

typedef struct { double tolerance, rel_tol; int max_iter, min_iter; } or_controls;
typedef struct { double initial_residual, final_residual; int n_iterations, converged, singular; } or_perf;

typedef struct { double *wA, *rA, *pA, *rD, *xr, *sumA; } or_work;

static int or_conv(double r, double init, const or_controls* c)
{
    return (r < c->tolerance) || (c->rel_tol > 1e-20 && r < c->rel_tol * init);
}

static void or_dom_amul(int nd, or_domain* D, or_work* W, double* const* x, double* const* y)
{
    for (int p = 0; p < nd; ++p)
        for (int i = 0; i < D[p].n_iface; ++i) W[p].xr[i] = x[D[p].iface_src_domain[i]][D[p].iface_src_cell[i]];
    for (int p = 0; p < nd; ++p)
        or_amul(D[p].n_cells, D[p].n_faces, D[p].owner, D[p].neighbour, D[p].diag, D[p].upper, D[p].upper, x[p],
                D[p].n_iface, D[p].iface_cells, D[p].iface_coeffs, W[p].xr, y[p]);
}

static void or_pc_setup(int kind, int n, int F, const int* owner, const int* neighbour, const double* diag,
                        const double* upper, const double* lower, double* rD);
static void or_pc_apply(int kind, int k, int n, int F, const int* owner, const int* neighbour, const double* rD,
                        const double* upper, const double* lower, const double* r, double* w, int transpose);

/* PCG over nd domains (O6/O8) with the preconditioner `kind` (O12) applied per domain on its
 * own faces: the processor-local factorisation OpenFOAM uses on decomposed meshes (Q31); kind 0
 * (diagonal) is the A9 fused form rD rA. */
static int or_pcg_impl(int nd, or_domain* D, const or_controls* ctl, int kind, int k, or_perf* perf);

int or_pcg(int nd, or_domain* D, const or_controls* ctl, or_perf* perf) { return or_pcg_impl(nd, D, ctl, 0, 0, perf); }

int or_pcg_dd_pc(int nd, or_domain* D, const or_controls* ctl, int kind, int k, or_perf* perf)
{
    return or_pcg_impl(nd, D, ctl, kind, k, perf);
}

static int or_pcg_impl(int nd, or_domain* D, const or_controls* ctl, int kind, int k, or_perf* perf)
{
    or_work* W = (or_work*)calloc((size_t)nd, sizeof(or_work));
    double** X = (double**)malloc(sizeof(double*) * (size_t)nd);
    double** Y = (double**)malloc(sizeof(double*) * (size_t)nd);
    for (int p = 0; p < nd; ++p) {
        size_t n = (size_t)D[p].n_cells + 1;
        W[p].wA = (double*)calloc(n, sizeof(double));
        W[p].rA = (double*)calloc(n, sizeof(double));
        W[p].pA = (double*)calloc(n, sizeof(double));
        W[p].rD = (double*)calloc(n, sizeof(double));
        W[p].sumA = (double*)calloc(n, sizeof(double));
        W[p].xr = (double*)calloc((size_t)D[p].n_iface + 1, sizeof(double));
        if (!W[p].wA || !W[p].rA || !W[p].pA || !W[p].rD || !W[p].sumA || !W[p].xr) return 6;
    }
    perf->n_iterations = 0;
    perf->converged = 0;
    perf->singular = 0;

    /* wA = A psi ; rA = source - wA */
    for (int p = 0; p < nd; ++p) { X[p] = D[p].psi; Y[p] = W[p].wA; }
    or_dom_amul(nd, D, W, X, Y);
    for (int p = 0; p < nd; ++p)
        for (int c = 0; c < D[p].n_cells; ++c) W[p].rA[c] = D[p].source[c] - W[p].wA[c];

    /* normFactor = gSum(|wA - xRef| + |source - xRef|) + small, xRef = sumA * gAverage(psi) */
    double spsi = 0.0, ncell = 0.0;
    for (int p = 0; p < nd; ++p) {
        double s = 0.0;
        for (int c = 0; c < D[p].n_cells; ++c) s += D[p].psi[c];
        spsi += s;
        ncell += (double)D[p].n_cells;
    }
    double xbar = spsi / ncell;
    double normFactor = 0.0;
    for (int p = 0; p < nd; ++p) {
        or_sumA(D[p].n_cells, D[p].n_faces, D[p].owner, D[p].neighbour, D[p].diag, D[p].upper, D[p].upper,
                D[p].n_iface, D[p].iface_cells, D[p].iface_coeffs, W[p].sumA);
        double s = 0.0;
        for (int c = 0; c < D[p].n_cells; ++c) {
            double xref = W[p].sumA[c] * xbar;
            s += fabs(W[p].wA[c] - xref) + fabs(D[p].source[c] - xref);
        }
        normFactor += s;
    }
    normFactor += 1e-20;

    double smag = 0.0;
    for (int p = 0; p < nd; ++p) {
        double s = 0.0;
        for (int c = 0; c < D[p].n_cells; ++c) s += fabs(W[p].rA[c]);
        smag += s;
    }
    perf->initial_residual = smag / normFactor;
    perf->final_residual = perf->initial_residual;

    for (int p = 0; p < nd; ++p) {
        if (kind == 0) {
            for (int c = 0; c < D[p].n_cells; ++c) W[p].rD[c] = 1.0 / D[p].diag[c];
        } else {
            or_pc_setup(kind, D[p].n_cells, D[p].n_faces, D[p].owner, D[p].neighbour, D[p].diag, D[p].upper,
                        D[p].upper, W[p].rD);
        }
    }

    double wArA = 1e20, wArAold;
    if (ctl->min_iter > 0 || !or_conv(perf->final_residual, perf->initial_residual, ctl)) {
        do {
            wArAold = wArA;
            /* precondition wA = M^-1 rA (per domain) ; wArA = gSumProd(wA, rA) */
            wArA = 0.0;
            for (int p = 0; p < nd; ++p) {
                if (kind != 0)
                    or_pc_apply(kind, k, D[p].n_cells, D[p].n_faces, D[p].owner, D[p].neighbour, W[p].rD,
                                D[p].upper, D[p].upper, W[p].rA, W[p].wA, 0);
                double s = 0.0;
                for (int c = 0; c < D[p].n_cells; ++c) {
                    if (kind == 0) W[p].wA[c] = W[p].rD[c] * W[p].rA[c];
                    s += W[p].wA[c] * W[p].rA[c];
                }
                wArA += s;
            }
            /* update search direction */
            if (perf->n_iterations == 0) {
                for (int p = 0; p < nd; ++p)
                    for (int c = 0; c < D[p].n_cells; ++c) W[p].pA[c] = W[p].wA[c];
            } else {
                double beta = wArA / wArAold;
                for (int p = 0; p < nd; ++p)
                    for (int c = 0; c < D[p].n_cells; ++c) W[p].pA[c] = W[p].wA[c] + beta * W[p].pA[c];
            }
            /* wA = A pA ; wApA = gSumProd(wA, pA) */
            for (int p = 0; p < nd; ++p) { X[p] = W[p].pA; Y[p] = W[p].wA; }
            or_dom_amul(nd, D, W, X, Y);
            double wApA = 0.0;
            for (int p = 0; p < nd; ++p) {
                double s = 0.0;
                for (int c = 0; c < D[p].n_cells; ++c) s += W[p].wA[c] * W[p].pA[c];
                wApA += s;
            }
            if (fabs(wApA) / normFactor < 1e-300) { /* checkSingularity: vSmall */
                perf->singular = 1;
                break;
            }
            double alpha = wArA / wApA;
            smag = 0.0;
            for (int p = 0; p < nd; ++p) {
                double s = 0.0;
                for (int c = 0; c < D[p].n_cells; ++c) {
                    D[p].psi[c] += alpha * W[p].pA[c];
                    W[p].rA[c] -= alpha * W[p].wA[c];
                }
                for (int c = 0; c < D[p].n_cells; ++c) s += fabs(W[p].rA[c]);
                smag += s;
            }
            perf->final_residual = smag / normFactor;
        } while ((++perf->n_iterations < ctl->max_iter && !or_conv(perf->final_residual, perf->initial_residual, ctl)) ||
                 perf->n_iterations < ctl->min_iter);
    }
    perf->converged = or_conv(perf->final_residual, perf->initial_residual, ctl);

    for (int p = 0; p < nd; ++p) {
        free(W[p].wA);
        free(W[p].rA);
        free(W[p].pA);
        free(W[p].rD);
        free(W[p].sumA);
        free(W[p].xr);
    }
    free(W);
    free(X);
    free(Y);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O11 GAMG with the Richardson smoother (paper: "GAMG ...      */
/* Richardson (or weighted Jacobi) ... diagonal at the coarsest" P:665,       */
/* pGAMG P:1043-1052; profile rows restrictField P:527, prolongField P:537,   */
/* agglomerateMatrix P:538, scale P:525, Vcycle P:545, RichardsonSmoother     */
/* P:517).  Readings Q22-Q28; SPEC S:479-569 for the rest.      */
/* ------------------------------------------------------------------------- */

/* faceAreaPair-style pairwise agglomeration (Q22): cells in ascending order; an
 * unagglomerated cell pairs with its unagglomerated neighbour across the face of largest
 * weight (faces of the cell in ascending face index, first maximum wins); with no such
 * neighbour it joins the agglomerate of its neighbour across the largest-weight face;
 * an isolated cell becomes its own agglomerate.  Returns the number of coarse cells. */
int or_agglomerate(int n, int F, const int* owner, const int* neighbour, const double* w, int* ftc)
{
    int* start = (int*)calloc((size_t)n + 1, sizeof(int));
    int* faces = (int*)malloc(sizeof(int) * (size_t)(2 * F + 1));
    int* fill = (int*)calloc((size_t)n + 1, sizeof(int));
    for (int f = 0; f < F; ++f) {
        start[owner[f] + 1]++;
        start[neighbour[f] + 1]++;
    }
    for (int c = 0; c < n; ++c) start[c + 1] += start[c];
    for (int f = 0; f < F; ++f) { /* ascending f: each cell's list is in ascending face index */
        faces[start[owner[f]] + fill[owner[f]]++] = f;
        faces[start[neighbour[f]] + fill[neighbour[f]]++] = f;
    }
    for (int c = 0; c < n; ++c) ftc[c] = -1;
    int nc = 0;
    for (int c = 0; c < n; ++c) {
        if (ftc[c] >= 0) continue;
        int best = -1;
        double bw = -1.0;
        for (int e = start[c]; e < start[c + 1]; ++e) {
            const int f = faces[e];
            const int o = owner[f] == c ? neighbour[f] : owner[f];
            if (ftc[o] < 0 && w[f] > bw) {
                bw = w[f];
                best = o;
            }
        }
        if (best >= 0) {
            ftc[c] = ftc[best] = nc++;
            continue;
        }
        bw = -1.0;
        for (int e = start[c]; e < start[c + 1]; ++e) {
            const int f = faces[e];
            const int o = owner[f] == c ? neighbour[f] : owner[f];
            if (w[f] > bw) {
                bw = w[f];
                best = o;
            }
        }
        ftc[c] = best >= 0 ? ftc[best] : nc++;
    }
    free(start);
    free(faces);
    free(fill);
    return nc;
}

static int or_pair2_cmp(const void* a, const void* b)
{
    const int* x = (const int*)a;
    const int* y = (const int*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    return x[1] < y[1] ? -1 : (x[1] > y[1]);
}

/* coarse lduAddressing: coarse faces = distinct (min, max) agglomerate pairs of the fine faces,
 * sorted; frestrict[f] = coarse face of fine face f, or -1 when both cells are in one
 * agglomerate.  Coarse face weights = sums of the fine ones (ascending fine face).
 * Returns the number of coarse faces (arrays sized F suffice). */
int or_coarse_addressing(int F, const int* owner, const int* neighbour, const int* ftc, const double* w,
                         int* cowner, int* cneighbour, int* frestrict, double* cw)
{
    int* pairs = (int*)malloc(sizeof(int) * 2 * (size_t)(F > 0 ? F : 1));
    int np = 0;
    for (int f = 0; f < F; ++f) {
        const int a = ftc[owner[f]], b = ftc[neighbour[f]];
        if (a == b) continue;
        pairs[2 * np] = a < b ? a : b;
        pairs[2 * np + 1] = a < b ? b : a;
        ++np;
    }
    qsort(pairs, (size_t)np, 2 * sizeof(int), or_pair2_cmp);
    int ncf = 0;
    for (int i = 0; i < np; ++i)
        if (i == 0 || pairs[2 * i] != pairs[2 * i - 2] || pairs[2 * i + 1] != pairs[2 * i - 1]) {
            cowner[ncf] = pairs[2 * i];
            cneighbour[ncf] = pairs[2 * i + 1];
            ++ncf;
        }
    for (int i = 0; i < ncf; ++i) cw[i] = 0.0;
    for (int f = 0; f < F; ++f) {
        const int a = ftc[owner[f]], b = ftc[neighbour[f]];
        if (a == b) {
            frestrict[f] = -1;
            continue;
        }
        const int lo = a < b ? a : b, hi = a < b ? b : a;
        int l = 0, h = ncf; /* binary search (lo, hi) */
        while (l < h) {
            const int m = l + (h - l) / 2;
            if (cowner[m] < lo || (cowner[m] == lo && cneighbour[m] < hi)) l = m + 1;
            else h = m;
        }
        frestrict[f] = l;
        cw[l] += w[f];
    }
    free(pairs);
    return ncf;
}

/* agglomerateMatrix (Galerkin with summation restriction / injection prolongation):
 * cdiag = restrict(diag) (ascending fine cells); then fine faces ascending: cupper[frestrict]
 * += upper, or cdiag[ftc[owner]] += (upper + lower) for agglomerate-internal faces. */
void or_agglomerate_matrix(int n, int F, const int* owner, const int* ftc, const int* frestrict, const double* diag,
                           const double* upper, int nc, int ncf, double* cdiag, double* cupper)
{
    for (int c = 0; c < nc; ++c) cdiag[c] = 0.0;
    for (int i = 0; i < ncf; ++i) cupper[i] = 0.0;
    for (int i = 0; i < n; ++i) cdiag[ftc[i]] += diag[i];
    for (int f = 0; f < F; ++f) {
        if (frestrict[f] >= 0) cupper[frestrict[f]] += upper[f];
        else cdiag[ftc[owner[f]]] += upper[f] + upper[f];
    }
}

/* restrictField: coarse[c] = sum of fine[i] over ftc[i] = c, ascending i */
void or_restrict(int n, const int* ftc, const double* fine, int nc, double* coarse)
{
    for (int c = 0; c < nc; ++c) coarse[c] = 0.0;
    for (int i = 0; i < n; ++i) coarse[ftc[i]] += fine[i];
}

typedef struct {
    int n_pre, n_post, scale, n_coarsest_cells, max_levels;
    double omega, coarsest_tol, coarsest_rel_tol;
    int coarsest_max_iter;
    int smoother; /* 0 Richardson (Q24), 1 two-stage Gauss-Seidel (Q30) */
    int n_inner;  /* two-stage GS: Jacobi-Richardson inner iterations */
} or_gamg_params;

typedef struct {
    int n, F;
    int *owner, *neighbour, *ftc, *frestrict; /* ftc/frestrict map this level to the next */
    double *w, *diag, *upper, *b, *x, *r, *y, *c, *rD;
} or_level;

/* Richardson / weighted-Jacobi sweep (Q24): y = A x; x = x + omega (rD (b - y)) */
static void or_jacobi_sweep(or_level* L, double omega)
{
    or_amul(L->n, L->F, L->owner, L->neighbour, L->diag, L->upper, L->upper, L->x, 0, 0, 0, 0, L->y);
    for (int i = 0; i < L->n; ++i) L->x[i] = L->x[i] + omega * (L->rD[i] * (L->b[i] - L->y[i]));
}

/* Two-stage Gauss-Seidel sweep (Q30, Berger-Vergiat et al. 2021): x = x + z with
 * z ~ (D + L)^-1 r, r = b - A x, L = strictly lower part (row c: faces with neighbour c,
 * coefficient lower = upper), by n_inner Jacobi-Richardson iterations
 * z_0 = rD r,  z_{k+1} = rD (r - L z_k)  (lower sums in face order). */
static void or_gs2_sweep(or_level* L, int n_inner)
{
    or_amul(L->n, L->F, L->owner, L->neighbour, L->diag, L->upper, L->upper, L->x, 0, 0, 0, 0, L->y);
    double* r = (double*)malloc(sizeof(double) * (size_t)(L->n + 1));
    double* z = (double*)malloc(sizeof(double) * (size_t)(L->n + 1));
    double* t = (double*)malloc(sizeof(double) * (size_t)(L->n + 1));
    for (int i = 0; i < L->n; ++i) {
        r[i] = L->b[i] - L->y[i];
        z[i] = L->rD[i] * r[i];
    }
    for (int k = 0; k < n_inner; ++k) {
        for (int i = 0; i < L->n; ++i) t[i] = r[i];
        for (int f = 0; f < L->F; ++f) t[L->neighbour[f]] -= L->upper[f] * z[L->owner[f]];
        for (int i = 0; i < L->n; ++i) z[i] = L->rD[i] * t[i];
    }
    for (int i = 0; i < L->n; ++i) L->x[i] = L->x[i] + z[i];
    free(r);
    free(z);
    free(t);
}

static void or_smooth(or_level* L, const or_gamg_params* gp)
{
    if (gp->smoother == 1) or_gs2_sweep(L, gp->n_inner);
    else or_jacobi_sweep(L, gp->omega);
}

/* GAMGSolver::scale reading (Q25): alpha = (c.r)/(c.Ac) clamped to [0, 2]
 * (1 when c.Ac <= 1e-300); c *= alpha.  The lower clamp is pinned (omega = 1.6 case); the
 * upper clamp is PARITY UNPINNED: no pin found reaches alpha > 2 (with Galerkin operators the
 * raw factor stayed <= 2 in every searched configuration). */
static void or_scale(or_level* L, double* r)
{
    or_amul(L->n, L->F, L->owner, L->neighbour, L->diag, L->upper, L->upper, L->c, 0, 0, 0, 0, L->y);
    double num = 0.0, den = 0.0;
    for (int i = 0; i < L->n; ++i) num += L->c[i] * r[i];
    for (int i = 0; i < L->n; ++i) den += L->y[i] * L->c[i];
    double a = fabs(den) > 1e-300 ? num / den : 1.0;
    if (a < 0.0) a = 0.0;
    if (a > 2.0) a = 2.0;
    for (int i = 0; i < L->n; ++i) L->c[i] = a * L->c[i];
}

static void or_coarsest_solve(or_level* L, const or_gamg_params* gp)
{
    for (int i = 0; i < L->n; ++i) L->x[i] = 0.0;
    or_domain d = {L->n, L->F, L->owner, L->neighbour, L->diag, L->upper, L->b, L->x, 0, 0, 0, 0, 0};
    or_controls c = {gp->coarsest_tol, gp->coarsest_rel_tol, gp->coarsest_max_iter, 0};
    or_perf pf;
    or_pcg(1, &d, &c, &pf);
}

/* one V-cycle (Q23): correction form, zero initial guess on every coarse level */
static void or_vcycle(int nl, or_level* Lv, const or_gamg_params* gp)
{
    for (int l = 0; l < nl - 1; ++l) {
        or_level* L = &Lv[l];
        for (int i = 0; i < L->n; ++i) L->x[i] = 0.0;
        for (int s = 0; s < gp->n_pre; ++s) or_smooth(L, gp);
        or_amul(L->n, L->F, L->owner, L->neighbour, L->diag, L->upper, L->upper, L->x, 0, 0, 0, 0, L->y);
        for (int i = 0; i < L->n; ++i) L->r[i] = L->b[i] - L->y[i];
        or_restrict(L->n, L->ftc, L->r, Lv[l + 1].n, Lv[l + 1].b);
    }
    or_coarsest_solve(&Lv[nl - 1], gp);
    for (int l = nl - 2; l >= 0; --l) {
        or_level* L = &Lv[l];
        for (int i = 0; i < L->n; ++i) L->c[i] = Lv[l + 1].x[L->ftc[i]]; /* prolongField: injection */
        if (gp->scale) or_scale(L, L->r);
        for (int i = 0; i < L->n; ++i) L->x[i] = L->x[i] + L->c[i];
        for (int s = 0; s < gp->n_post; ++s) or_smooth(L, gp);
    }
}

/* Build the hierarchy (faceAreaPair weights = face areas): returns the number of levels;
 * levels[0] is the fine mesh (arrays borrowed), coarser levels allocated. */
int or_gamg_hierarchy(int n, int F, const int* owner, const int* neighbour, const double* weights,
                      const or_gamg_params* gp, or_level* Lv, int max_out)
{
    int nl = 1;
    Lv[0].n = n;
    Lv[0].F = F;
    Lv[0].owner = (int*)owner;
    Lv[0].neighbour = (int*)neighbour;
    Lv[0].w = (double*)weights;
    while (nl < max_out && nl < gp->max_levels && Lv[nl - 1].n > gp->n_coarsest_cells) {
        or_level* L = &Lv[nl - 1];
        L->ftc = (int*)malloc(sizeof(int) * (size_t)(L->n + 1));
        const int nc = or_agglomerate(L->n, L->F, L->owner, L->neighbour, L->w, L->ftc);
        if (nc >= L->n) {
            free(L->ftc);
            L->ftc = 0;
            break;
        }
        or_level* C = &Lv[nl];
        C->owner = (int*)malloc(sizeof(int) * (size_t)(L->F + 1));
        C->neighbour = (int*)malloc(sizeof(int) * (size_t)(L->F + 1));
        C->w = (double*)malloc(sizeof(double) * (size_t)(L->F + 1));
        L->frestrict = (int*)malloc(sizeof(int) * (size_t)(L->F + 1));
        C->F = or_coarse_addressing(L->F, L->owner, L->neighbour, L->ftc, L->w, C->owner, C->neighbour,
                                    L->frestrict, C->w);
        C->n = nc;
        ++nl;
    }
    Lv[nl - 1].ftc = 0;
    Lv[nl - 1].frestrict = 0;
    return nl;
}

/* GAMG solve, OpenFOAM loop semantics (Q26): normFactor / residual as PCG (Q1);
 * iterate V-cycles while ((++n < maxIter && !converged) || n < minIter). */
int or_gamg(int n, int F, const int* owner, const int* neighbour, const double* weights, const double* diag,
            const double* upper, const double* source, double* psi, const or_gamg_params* gp,
            const or_controls* ctl, or_perf* perf, int* levels_out, int* level_cells)
{
    or_level Lv[64];
    memset(Lv, 0, sizeof(Lv));
    const int nl = or_gamg_hierarchy(n, F, owner, neighbour, weights, gp, Lv, 64);
    for (int l = 0; l < nl; ++l) {
        or_level* L = &Lv[l];
        const size_t m = (size_t)L->n + 1;
        L->b = (double*)calloc(m, sizeof(double));
        L->x = (double*)calloc(m, sizeof(double));
        L->r = (double*)calloc(m, sizeof(double));
        L->y = (double*)calloc(m, sizeof(double));
        L->c = (double*)calloc(m, sizeof(double));
        L->rD = (double*)calloc(m, sizeof(double));
        if (l == 0) {
            L->diag = (double*)diag;
            L->upper = (double*)upper;
        } else {
            L->diag = (double*)calloc(m, sizeof(double));
            L->upper = (double*)calloc((size_t)L->F + 1, sizeof(double));
            or_level* P = &Lv[l - 1];
            or_agglomerate_matrix(P->n, P->F, P->owner, P->ftc, P->frestrict, P->diag, P->upper, L->n, L->F,
                                  L->diag, L->upper);
        }
        for (int i = 0; i < L->n; ++i) L->rD[i] = 1.0 / L->diag[i];
        if (level_cells && l < 64) level_cells[l] = L->n;
    }
    if (levels_out) *levels_out = nl;

    /* residual and normFactor exactly as PCG (Q1) */
    double* wA = (double*)calloc((size_t)n + 1, sizeof(double));
    double* sumA = (double*)calloc((size_t)n + 1, sizeof(double));
    double* r = (double*)calloc((size_t)n + 1, sizeof(double));
    or_amul(n, F, owner, neighbour, diag, upper, upper, psi, 0, 0, 0, 0, wA);
    for (int i = 0; i < n; ++i) r[i] = source[i] - wA[i];
    double spsi = 0.0;
    for (int i = 0; i < n; ++i) spsi += psi[i];
    const double xbar = spsi / (double)n;
    or_sumA(n, F, owner, neighbour, diag, upper, upper, 0, 0, 0, sumA);
    double nf = 0.0;
    for (int i = 0; i < n; ++i) {
        const double xref = sumA[i] * xbar;
        nf += fabs(wA[i] - xref) + fabs(source[i] - xref);
    }
    const double normFactor = nf + 1e-20;
    double smag = 0.0;
    for (int i = 0; i < n; ++i) smag += fabs(r[i]);
    perf->initial_residual = smag / normFactor;
    perf->final_residual = perf->initial_residual;
    perf->n_iterations = 0;
    perf->singular = 0;
    if (ctl->min_iter > 0 || !or_conv(perf->final_residual, perf->initial_residual, ctl)) {
        do {
            for (int i = 0; i < n; ++i) Lv[0].b[i] = r[i];
            if (nl == 1) {
                or_coarsest_solve(&Lv[0], gp);
            } else {
                or_vcycle(nl, Lv, gp);
            }
            for (int i = 0; i < n; ++i) psi[i] = psi[i] + Lv[0].x[i];
            or_amul(n, F, owner, neighbour, diag, upper, upper, psi, 0, 0, 0, 0, wA);
            smag = 0.0;
            for (int i = 0; i < n; ++i) {
                r[i] = source[i] - wA[i];
                smag += fabs(r[i]);
            }
            perf->final_residual = smag / normFactor;
        } while ((++perf->n_iterations < ctl->max_iter && !or_conv(perf->final_residual, perf->initial_residual, ctl)) ||
                 perf->n_iterations < ctl->min_iter);
    }
    perf->converged = or_conv(perf->final_residual, perf->initial_residual, ctl);
    for (int l = 0; l < nl; ++l) {
        or_level* L = &Lv[l];
        free(L->b); free(L->x); free(L->r); free(L->y); free(L->c); free(L->rD);
        free(L->ftc); free(L->frestrict);
        if (l > 0) { free(L->diag); free(L->upper); free(L->owner); free(L->neighbour); free(L->w); }
    }
    free(wA);
    free(sumA);
    free(r);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O11dd GAMG on a decomposed mesh (nd domains; readings Q36-Q38, DESIGN.md   */
/* §3).  OpenFOAM's parallel GAMG keeps the agglomeration processor-local and */
/* agglomerates the processor interfaces alongside ([OF] GAMGAgglomeration,   */
/* processorGAMGInterface); the paper runs GAMG decomposed on 1-8 GPUs with   */
/* the coarsening unchanged.                        */
/*   Q36 levels: every domain agglomerates its own internal faces (Q22); a    */
/*       level is added while sum_p n_p > nd * nCellsInCoarsestLevel and the  */
/*       pass reduces sum_p n_p (nd = 1: exactly Q22's rule).                 */
/*   Q37 coarse interfaces: per domain, the fine interface faces in their     */
/*       (patch, face) order map to coarse interface faces = distinct         */
/*       (neighbour domain, local coarse cell, remote coarse cell) triples    */
/*       numbered by first occurrence; coefficient = sum of the fine ones in  */
/*       ascending fine order (both sides see the same faces in the same      */
/*       order, Q13, so both get bitwise the same coarse coefficients).       */
/*   Q38 cycle: the single-domain V-cycle (Q23-Q30) with every A x a          */
/*       decomposed Amul (remote x copied across the interfaces first), every */
/*       dot a per-domain sum added in domain order, the two-stage GS lower   */
/*       sweep domain-local (like DILU, Q31), and the coarsest level solved   */
/*       by the decomposed PCG (O8) over the coarsest interfaces.             */
/* ------------------------------------------------------------------------- */

typedef struct {
    or_level l;          /* per-domain level (borrowed arrays on level 0) */
    int n_if;
    int *if_cell, *if_src_dom, *if_src_cell;
    double* if_coef;
    int* if_restrict;    /* fine interface face -> coarse interface face of the next level */
    double* xr;
} or_dlevel;

static void or_dd_amul(int nd, or_dlevel* L, double* const* x, double* const* y)
{
    for (int p = 0; p < nd; ++p)
        for (int i = 0; i < L[p].n_if; ++i) L[p].xr[i] = x[L[p].if_src_dom[i]][L[p].if_src_cell[i]];
    for (int p = 0; p < nd; ++p)
        or_amul(L[p].l.n, L[p].l.F, L[p].l.owner, L[p].l.neighbour, L[p].l.diag, L[p].l.upper, L[p].l.upper, x[p],
                L[p].n_if, L[p].if_cell, L[p].if_coef, L[p].xr, y[p]);
}

/* y_p = A x_p over all domains with x = the level's x (or c when use_c) */
static void or_dd_amul_field(int nd, or_dlevel* L, int use_c)
{
    double* X[256];
    double* Y[256];
    for (int p = 0; p < nd; ++p) {
        X[p] = use_c ? L[p].l.c : L[p].l.x;
        Y[p] = L[p].l.y;
    }
    or_dd_amul(nd, L, X, Y);
}

/* Build the decomposed hierarchy (Q36, Q37) and, with diag != NULL, the Galerkin matrices
 * (Q27 per domain + coarse interface coefficients).  Returns the number of levels. */
static int or_dd_build(int nd, const or_domain* D, const double* const* weights, const or_gamg_params* gp,
                       or_dlevel** Lv, int max_out)
{
    Lv[0] = (or_dlevel*)calloc((size_t)nd, sizeof(or_dlevel));
    for (int p = 0; p < nd; ++p) {
        or_dlevel* d = &Lv[0][p];
        d->l.n = D[p].n_cells;
        d->l.F = D[p].n_faces;
        d->l.owner = (int*)D[p].owner;
        d->l.neighbour = (int*)D[p].neighbour;
        d->l.w = (double*)weights[p];
        d->l.diag = (double*)D[p].diag;
        d->l.upper = (double*)D[p].upper;
        d->n_if = D[p].n_iface;
        d->if_cell = (int*)D[p].iface_cells;
        d->if_src_dom = (int*)D[p].iface_src_domain;
        d->if_src_cell = (int*)D[p].iface_src_cell;
        d->if_coef = (double*)D[p].iface_coeffs;
    }
    int nl = 1;
    for (;;) {
        or_dlevel* F = Lv[nl - 1];
        long long nfine = 0;
        for (int p = 0; p < nd; ++p) nfine += F[p].l.n;
        if (!(nl < max_out && nl < gp->max_levels && nfine > (long long)nd * gp->n_coarsest_cells)) break;
        long long ncoarse = 0;
        int* nc = (int*)calloc((size_t)nd, sizeof(int));
        for (int p = 0; p < nd; ++p) {
            F[p].l.ftc = (int*)malloc(sizeof(int) * (size_t)(F[p].l.n + 1));
            nc[p] = or_agglomerate(F[p].l.n, F[p].l.F, F[p].l.owner, F[p].l.neighbour, F[p].l.w, F[p].l.ftc);
            ncoarse += nc[p];
        }
        if (ncoarse >= nfine) {
            for (int p = 0; p < nd; ++p) {
                free(F[p].l.ftc);
                F[p].l.ftc = 0;
            }
            free(nc);
            break;
        }
        or_dlevel* C = (or_dlevel*)calloc((size_t)nd, sizeof(or_dlevel));
        for (int p = 0; p < nd; ++p) {
            or_level* L = &F[p].l;
            or_level* K = &C[p].l;
            K->owner = (int*)malloc(sizeof(int) * (size_t)(L->F + 1));
            K->neighbour = (int*)malloc(sizeof(int) * (size_t)(L->F + 1));
            K->w = (double*)malloc(sizeof(double) * (size_t)(L->F + 1));
            L->frestrict = (int*)malloc(sizeof(int) * (size_t)(L->F + 1));
            K->F = or_coarse_addressing(L->F, L->owner, L->neighbour, L->ftc, L->w, K->owner, K->neighbour,
                                        L->frestrict, K->w);
            K->n = nc[p];
            /* Q37: coarse interface faces by first occurrence of (domain, local, remote) */
            const int m = F[p].n_if;
            C[p].if_cell = (int*)malloc(sizeof(int) * (size_t)(m + 1));
            C[p].if_src_dom = (int*)malloc(sizeof(int) * (size_t)(m + 1));
            C[p].if_src_cell = (int*)malloc(sizeof(int) * (size_t)(m + 1));
            F[p].if_restrict = (int*)malloc(sizeof(int) * (size_t)(m + 1));
            int k = 0;
            for (int i = 0; i < m; ++i) {
                const int q = F[p].if_src_dom[i];
                const int a = L->ftc[F[p].if_cell[i]];
                const int b = F[q].l.ftc[F[p].if_src_cell[i]];
                int j = 0;
                while (j < k && !(C[p].if_src_dom[j] == q && C[p].if_cell[j] == a && C[p].if_src_cell[j] == b)) ++j;
                if (j == k) {
                    C[p].if_src_dom[k] = q;
                    C[p].if_cell[k] = a;
                    C[p].if_src_cell[k] = b;
                    ++k;
                }
                F[p].if_restrict[i] = j;
            }
            C[p].n_if = k;
        }
        free(nc);
        Lv[nl++] = C;
    }
    for (int p = 0; p < nd; ++p) {
        Lv[nl - 1][p].l.ftc = 0;
        Lv[nl - 1][p].l.frestrict = 0;
        Lv[nl - 1][p].if_restrict = 0;
    }
    /* Galerkin matrices (Q27) + coarse interface coefficients (Q37) */
    for (int l = 1; l < nl; ++l)
        for (int p = 0; p < nd; ++p) {
            or_dlevel* f = &Lv[l - 1][p];
            or_dlevel* c = &Lv[l][p];
            c->l.diag = (double*)calloc((size_t)c->l.n + 1, sizeof(double));
            c->l.upper = (double*)calloc((size_t)c->l.F + 1, sizeof(double));
            or_agglomerate_matrix(f->l.n, f->l.F, f->l.owner, f->l.ftc, f->l.frestrict, f->l.diag, f->l.upper,
                                  c->l.n, c->l.F, c->l.diag, c->l.upper);
            c->if_coef = (double*)calloc((size_t)c->n_if + 1, sizeof(double));
            for (int i = 0; i < f->n_if; ++i) c->if_coef[f->if_restrict[i]] += f->if_coef[i];
        }
    for (int l = 0; l < nl; ++l)
        for (int p = 0; p < nd; ++p) {
            or_level* L = &Lv[l][p].l;
            const size_t m = (size_t)L->n + 1;
            L->b = (double*)calloc(m, sizeof(double));
            L->x = (double*)calloc(m, sizeof(double));
            L->r = (double*)calloc(m, sizeof(double));
            L->y = (double*)calloc(m, sizeof(double));
            L->c = (double*)calloc(m, sizeof(double));
            L->rD = (double*)calloc(m, sizeof(double));
            for (int i = 0; i < L->n; ++i) L->rD[i] = 1.0 / L->diag[i];
            Lv[l][p].xr = (double*)calloc((size_t)Lv[l][p].n_if + 1, sizeof(double));
        }
    return nl;
}

static void or_dd_free(int nd, or_dlevel** Lv, int nl)
{
    for (int l = 0; l < nl; ++l) {
        for (int p = 0; p < nd; ++p) {
            or_dlevel* d = &Lv[l][p];
            or_level* L = &d->l;
            free(L->b); free(L->x); free(L->r); free(L->y); free(L->c); free(L->rD);
            free(L->ftc); free(L->frestrict); free(d->if_restrict); free(d->xr);
            if (l > 0) {
                free(L->diag); free(L->upper); free(L->owner); free(L->neighbour); free(L->w);
                free(d->if_cell); free(d->if_src_dom); free(d->if_src_cell); free(d->if_coef);
            }
        }
        free(Lv[l]);
    }
}

static void or_dd_smooth(int nd, or_dlevel* Lv, const or_gamg_params* gp)
{
    or_dd_amul_field(nd, Lv, 0);
    for (int p = 0; p < nd; ++p) {
        or_level* L = &Lv[p].l;
        if (gp->smoother != 1) {
            for (int i = 0; i < L->n; ++i) L->x[i] = L->x[i] + gp->omega * (L->rD[i] * (L->b[i] - L->y[i]));
            continue;
        }
        /* two-stage Gauss-Seidel (Q30), the lower sweep on the domain's own faces (Q38) */
        double* r = (double*)malloc(sizeof(double) * (size_t)(L->n + 1));
        double* z = (double*)malloc(sizeof(double) * (size_t)(L->n + 1));
        double* t = (double*)malloc(sizeof(double) * (size_t)(L->n + 1));
        for (int i = 0; i < L->n; ++i) {
            r[i] = L->b[i] - L->y[i];
            z[i] = L->rD[i] * r[i];
        }
        for (int k = 0; k < gp->n_inner; ++k) {
            for (int i = 0; i < L->n; ++i) t[i] = r[i];
            for (int f = 0; f < L->F; ++f) t[L->neighbour[f]] -= L->upper[f] * z[L->owner[f]];
            for (int i = 0; i < L->n; ++i) z[i] = L->rD[i] * t[i];
        }
        for (int i = 0; i < L->n; ++i) L->x[i] = L->x[i] + z[i];
        free(r);
        free(z);
        free(t);
    }
}

/* Q25 over domains: alpha = (sum_p c.r) / (sum_p Ac.c), clamped to [0, 2] */
static void or_dd_scale(int nd, or_dlevel* Lv)
{
    or_dd_amul_field(nd, Lv, 1);
    double num = 0.0, den = 0.0;
    for (int p = 0; p < nd; ++p) {
        or_level* L = &Lv[p].l;
        double s = 0.0;
        for (int i = 0; i < L->n; ++i) s += L->c[i] * L->r[i];
        num += s;
    }
    for (int p = 0; p < nd; ++p) {
        or_level* L = &Lv[p].l;
        double s = 0.0;
        for (int i = 0; i < L->n; ++i) s += L->y[i] * L->c[i];
        den += s;
    }
    double a = fabs(den) > 1e-300 ? num / den : 1.0;
    if (a < 0.0) a = 0.0;
    if (a > 2.0) a = 2.0;
    for (int p = 0; p < nd; ++p)
        for (int i = 0; i < Lv[p].l.n; ++i) Lv[p].l.c[i] = a * Lv[p].l.c[i];
}

static void or_dd_coarsest(int nd, or_dlevel* Lv, const or_gamg_params* gp)
{
    or_domain* d = (or_domain*)calloc((size_t)nd, sizeof(or_domain));
    for (int p = 0; p < nd; ++p) {
        or_level* L = &Lv[p].l;
        for (int i = 0; i < L->n; ++i) L->x[i] = 0.0;
        or_domain q = {L->n, L->F, L->owner, L->neighbour, L->diag, L->upper, L->b, L->x,
                       Lv[p].n_if, Lv[p].if_cell, Lv[p].if_coef, Lv[p].if_src_dom, Lv[p].if_src_cell};
        d[p] = q;
    }
    or_controls c = {gp->coarsest_tol, gp->coarsest_rel_tol, gp->coarsest_max_iter, 0};
    or_perf pf;
    or_pcg(nd, d, &c, &pf);
    free(d);
}

static void or_dd_vcycle(int nd, int nl, or_dlevel** Lv, const or_gamg_params* gp)
{
    for (int l = 0; l < nl - 1; ++l) {
        for (int p = 0; p < nd; ++p)
            for (int i = 0; i < Lv[l][p].l.n; ++i) Lv[l][p].l.x[i] = 0.0;
        for (int s = 0; s < gp->n_pre; ++s) or_dd_smooth(nd, Lv[l], gp);
        or_dd_amul_field(nd, Lv[l], 0);
        for (int p = 0; p < nd; ++p) {
            or_level* L = &Lv[l][p].l;
            for (int i = 0; i < L->n; ++i) L->r[i] = L->b[i] - L->y[i];
            or_restrict(L->n, L->ftc, L->r, Lv[l + 1][p].l.n, Lv[l + 1][p].l.b);
        }
    }
    or_dd_coarsest(nd, Lv[nl - 1], gp);
    for (int l = nl - 2; l >= 0; --l) {
        for (int p = 0; p < nd; ++p) {
            or_level* L = &Lv[l][p].l;
            for (int i = 0; i < L->n; ++i) L->c[i] = Lv[l + 1][p].l.x[L->ftc[i]];
        }
        if (gp->scale) or_dd_scale(nd, Lv[l]);
        for (int p = 0; p < nd; ++p) {
            or_level* L = &Lv[l][p].l;
            for (int i = 0; i < L->n; ++i) L->x[i] = L->x[i] + L->c[i];
        }
        for (int s = 0; s < gp->n_post; ++s) or_dd_smooth(nd, Lv[l], gp);
    }
}

/* Decomposed GAMG solve (Q36-Q38 + the outer loop of Q28 with decomposed sums, as O8).
 * level_cells[p * 64 + l] / level_ifaces[p * 64 + l]: per-domain level sizes (may be NULL). */
int or_gamg_dd(int nd, or_domain* D, const double* const* weights, const or_gamg_params* gp, const or_controls* ctl,
               or_perf* perf, int* levels_out, int* level_cells, int* level_ifaces)
{
    if (nd < 1 || nd > 256) return 1;
    or_dlevel* Lv[64];
    const int nl = or_dd_build(nd, D, weights, gp, Lv, 64);
    if (levels_out) *levels_out = nl;
    for (int p = 0; p < nd; ++p)
        for (int l = 0; l < nl; ++l) {
            if (level_cells) level_cells[p * 64 + l] = Lv[l][p].l.n;
            if (level_ifaces) level_ifaces[p * 64 + l] = Lv[l][p].n_if;
        }
    double* wA[256];
    double* r[256];
    double* sumA[256];
    double* psi[256];
    for (int p = 0; p < nd; ++p) {
        wA[p] = (double*)calloc((size_t)D[p].n_cells + 1, sizeof(double));
        r[p] = (double*)calloc((size_t)D[p].n_cells + 1, sizeof(double));
        sumA[p] = (double*)calloc((size_t)D[p].n_cells + 1, sizeof(double));
        psi[p] = D[p].psi;
    }
    /* residual and normFactor exactly as the decomposed PCG (Q1, O8) */
    or_dd_amul(nd, Lv[0], psi, wA);
    double spsi = 0.0, ncell = 0.0;
    for (int p = 0; p < nd; ++p) {
        double s = 0.0;
        for (int c = 0; c < D[p].n_cells; ++c) s += psi[p][c];
        spsi += s;
        ncell += (double)D[p].n_cells;
    }
    const double xbar = spsi / ncell;
    double normFactor = 0.0, smag = 0.0;
    for (int p = 0; p < nd; ++p) {
        or_sumA(D[p].n_cells, D[p].n_faces, D[p].owner, D[p].neighbour, D[p].diag, D[p].upper, D[p].upper,
                D[p].n_iface, D[p].iface_cells, D[p].iface_coeffs, sumA[p]);
        double s = 0.0;
        for (int c = 0; c < D[p].n_cells; ++c) {
            const double xref = sumA[p][c] * xbar;
            s += fabs(wA[p][c] - xref) + fabs(D[p].source[c] - xref);
        }
        normFactor += s;
    }
    normFactor += 1e-20;
    for (int p = 0; p < nd; ++p) {
        double s = 0.0;
        for (int c = 0; c < D[p].n_cells; ++c) {
            r[p][c] = D[p].source[c] - wA[p][c];
            s += fabs(r[p][c]);
        }
        smag += s;
    }
    perf->initial_residual = smag / normFactor;
    perf->final_residual = perf->initial_residual;
    perf->n_iterations = 0;
    perf->singular = 0;
    if (ctl->min_iter > 0 || !or_conv(perf->final_residual, perf->initial_residual, ctl)) {
        do {
            for (int p = 0; p < nd; ++p)
                for (int c = 0; c < D[p].n_cells; ++c) Lv[0][p].l.b[c] = r[p][c];
            if (nl == 1) or_dd_coarsest(nd, Lv[0], gp);
            else or_dd_vcycle(nd, nl, Lv, gp);
            for (int p = 0; p < nd; ++p)
                for (int c = 0; c < D[p].n_cells; ++c) psi[p][c] = psi[p][c] + Lv[0][p].l.x[c];
            or_dd_amul(nd, Lv[0], psi, wA);
            smag = 0.0;
            for (int p = 0; p < nd; ++p) {
                double s = 0.0;
                for (int c = 0; c < D[p].n_cells; ++c) {
                    r[p][c] = D[p].source[c] - wA[p][c];
                    s += fabs(r[p][c]);
                }
                smag += s;
            }
            perf->final_residual = smag / normFactor;
        } while ((++perf->n_iterations < ctl->max_iter && !or_conv(perf->final_residual, perf->initial_residual, ctl)) ||
                 perf->n_iterations < ctl->min_iter);
    }
    perf->converged = or_conv(perf->final_residual, perf->initial_residual, ctl);
    for (int p = 0; p < nd; ++p) {
        free(wA[p]);
        free(r[p]);
        free(sumA[p]);
    }
    or_dd_free(nd, Lv, nl);
    return 0;
}

/* The global operator of level `level` of the decomposed hierarchy as a dense matrix (cells
 * numbered domain-major: domain p's cells after those of domains < p) and, for level > 0, the
 * global fine-to-coarse map of level - 1 -- for the Galerkin pin R^T A R (tests only).
 * Returns the global cell count of the level, or -1 (no such level / capacity too small). */
int or_gamg_dd_dense_level(int nd, const or_domain* D, const double* const* weights, const or_gamg_params* gp,
                           int level, int cap, double* A, int* ftc_global)
{
    if (nd < 1 || nd > 256) return -1;
    or_dlevel* Lv[64];
    const int nl = or_dd_build(nd, D, weights, gp, Lv, 64);
    int ret = -1;
    if (level >= 0 && level < nl) {
        int off[257];
        off[0] = 0;
        for (int p = 0; p < nd; ++p) off[p + 1] = off[p] + Lv[level][p].l.n;
        const int n = off[nd];
        if (n <= cap) {
            for (int i = 0; i < n * n; ++i) A[i] = 0.0;
            for (int p = 0; p < nd; ++p) {
                const or_dlevel* d = &Lv[level][p];
                for (int c = 0; c < d->l.n; ++c) A[(off[p] + c) * n + off[p] + c] += d->l.diag[c];
                for (int f = 0; f < d->l.F; ++f) {
                    const int o = off[p] + d->l.owner[f], nb = off[p] + d->l.neighbour[f];
                    A[o * n + nb] += d->l.upper[f];
                    A[nb * n + o] += d->l.upper[f];
                }
                for (int i = 0; i < d->n_if; ++i)
                    A[(off[p] + d->if_cell[i]) * n + off[d->if_src_dom[i]] + d->if_src_cell[i]] += d->if_coef[i];
            }
            if (level > 0 && ftc_global) {
                int offf[257];
                offf[0] = 0;
                for (int p = 0; p < nd; ++p) offf[p + 1] = offf[p] + Lv[level - 1][p].l.n;
                for (int p = 0; p < nd; ++p)
                    for (int i = 0; i < Lv[level - 1][p].l.n; ++i)
                        ftc_global[offf[p] + i] = off[p] + Lv[level - 1][p].l.ftc[i];
            }
            ret = n;
        }
    }
    or_dd_free(nd, Lv, nl);
    return ret;
}

/* ------------------------------------------------------------------------- */
/* O12 preconditioners (readings Q31-Q35): diagonal, DIC,  */
/* DILU, aDILU; PCG with any of them; PBiCG (*/
/* P:566); LDU -> CSR map.                           */
/* ------------------------------------------------------------------------- */

/* [OF] DIC/DILU calcReciprocalD: rD = diag; faces in order: rD[nbr] -= upper*lower/rD[own];
 * then rD = 1/rD (DIC: lower = upper). */
void or_ilu_factor(int n, int F, const int* owner, const int* neighbour, const double* diag, const double* upper,
                   const double* lower, double* rD)
{
    for (int c = 0; c < n; ++c) rD[c] = diag[c];
    for (int f = 0; f < F; ++f) rD[neighbour[f]] -= upper[f] * lower[f] / rD[owner[f]];
    for (int c = 0; c < n; ++c) rD[c] = 1.0 / rD[c];
}

/* [OF] DIC/DILU precondition: w = rD r; forward over faces: w[nbr] -= rD[nbr]*lower*w[own];
 * backward over faces in reverse: w[own] -= rD[own]*upper*w[nbr].  transpose (preconditionT)
 * swaps the roles of lower and upper.  k >= 0 (aDILU, Q33): each sweep replaced by k
 * Jacobi-style passes of the same face update reading the previous pass's values. */
void or_ilu_precondition(int n, int F, const int* owner, const int* neighbour, const double* rD, const double* upper,
                         const double* lower, const double* r, double* w, int transpose, int k)
{
    const double* lo = transpose ? upper : lower;
    const double* up = transpose ? lower : upper;
    for (int c = 0; c < n; ++c) w[c] = rD[c] * r[c];
    if (k < 0) {
        for (int f = 0; f < F; ++f) w[neighbour[f]] -= rD[neighbour[f]] * lo[f] * w[owner[f]];
        for (int f = F - 1; f >= 0; --f) w[owner[f]] -= rD[owner[f]] * up[f] * w[neighbour[f]];
        return;
    }
    double* y0 = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    double* prev = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    for (int c = 0; c < n; ++c) y0[c] = w[c];
    for (int it = 0; it < k; ++it) { /* forward: w = rD r - (rD lower) w_prev */
        for (int c = 0; c < n; ++c) prev[c] = w[c];
        for (int c = 0; c < n; ++c) w[c] = y0[c];
        for (int f = 0; f < F; ++f) w[neighbour[f]] -= rD[neighbour[f]] * lo[f] * prev[owner[f]];
    }
    for (int c = 0; c < n; ++c) y0[c] = w[c];
    for (int it = 0; it < k; ++it) { /* backward: w = y - (rD upper) w_prev */
        for (int c = 0; c < n; ++c) prev[c] = w[c];
        for (int c = 0; c < n; ++c) w[c] = y0[c];
        for (int f = F - 1; f >= 0; --f) w[owner[f]] -= rD[owner[f]] * up[f] * prev[neighbour[f]];
    }
    free(y0);
    free(prev);
}

enum { OR_PC_DIAGONAL = 0, OR_PC_DIC = 1, OR_PC_DILU = 2, OR_PC_ADILU = 3 };

static void or_pc_setup(int kind, int n, int F, const int* owner, const int* neighbour, const double* diag,
                        const double* upper, const double* lower, double* rD)
{
    if (kind == OR_PC_DIAGONAL) {
        for (int c = 0; c < n; ++c) rD[c] = 1.0 / diag[c];
    } else {
        or_ilu_factor(n, F, owner, neighbour, diag, upper, kind == OR_PC_DIC ? upper : lower, rD);
    }
}

static void or_pc_apply(int kind, int k, int n, int F, const int* owner, const int* neighbour, const double* rD,
                        const double* upper, const double* lower, const double* r, double* w, int transpose)
{
    if (kind == OR_PC_DIAGONAL) {
        for (int c = 0; c < n; ++c) w[c] = rD[c] * r[c];
    } else {
        or_ilu_precondition(n, F, owner, neighbour, rD, upper, kind == OR_PC_DIC ? upper : lower, r, w, transpose,
                            kind == OR_PC_ADILU ? k : -1);
    }
}

/* normFactor (Q1) of a single domain */
static double or_norm_factor(int n, int F, const int* owner, const int* neighbour, const double* diag,
                             const double* lower, const double* upper, const double* source, const double* psi,
                             const double* wA)
{
    double* sumA = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    for (int c = 0; c < n; ++c) sumA[c] = diag[c]; /* row sums: row owner holds upper, row neighbour lower */
    for (int f = 0; f < F; ++f) {
        sumA[owner[f]] += upper[f];
        sumA[neighbour[f]] += lower[f];
    }
    double spsi = 0.0;
    for (int c = 0; c < n; ++c) spsi += psi[c];
    const double xbar = spsi / (double)n;
    double nf = 0.0;
    for (int c = 0; c < n; ++c) {
        const double xref = sumA[c] * xbar;
        nf += fabs(wA[c] - xref) + fabs(source[c] - xref);
    }
    free(sumA);
    return nf + 1e-20;
}

/* PCG with a general preconditioner (single domain), OpenFOAM PCG::solve (Q1-Q4):
 * wA = M^-1 rA; wArA = wA.rA; pA = wA (+ beta pA); wA = A pA; alpha = wArA / wA.pA;
 * psi += alpha pA; rA -= alpha wA; final = |rA| / normFactor. */
int or_pcg_pc(int n, int F, const int* owner, const int* neighbour, const double* diag, const double* upper,
              const double* source, double* psi, const or_controls* ctl, int kind, int k, or_perf* perf)
{
    double* wA = (double*)calloc((size_t)n + 1, sizeof(double));
    double* rA = (double*)calloc((size_t)n + 1, sizeof(double));
    double* pA = (double*)calloc((size_t)n + 1, sizeof(double));
    double* rD = (double*)calloc((size_t)n + 1, sizeof(double));
    or_amul(n, F, owner, neighbour, diag, upper, upper, psi, 0, 0, 0, 0, wA);
    for (int c = 0; c < n; ++c) rA[c] = source[c] - wA[c];
    const double normFactor = or_norm_factor(n, F, owner, neighbour, diag, upper, upper, source, psi, wA);
    double s = 0.0;
    for (int c = 0; c < n; ++c) s += fabs(rA[c]);
    perf->initial_residual = s / normFactor;
    perf->final_residual = perf->initial_residual;
    perf->n_iterations = 0;
    perf->singular = 0;
    if (ctl->min_iter > 0 || !or_conv(perf->final_residual, perf->initial_residual, ctl)) {
        or_pc_setup(kind, n, F, owner, neighbour, diag, upper, upper, rD);
        double wArA = 1e20, wArAold;
        do {
            wArAold = wArA;
            or_pc_apply(kind, k, n, F, owner, neighbour, rD, upper, upper, rA, wA, 0);
            wArA = 0.0;
            for (int c = 0; c < n; ++c) wArA += wA[c] * rA[c];
            if (perf->n_iterations == 0) {
                for (int c = 0; c < n; ++c) pA[c] = wA[c];
            } else {
                const double beta = wArA / wArAold;
                for (int c = 0; c < n; ++c) pA[c] = wA[c] + beta * pA[c];
            }
            or_amul(n, F, owner, neighbour, diag, upper, upper, pA, 0, 0, 0, 0, wA);
            double wApA = 0.0;
            for (int c = 0; c < n; ++c) wApA += wA[c] * pA[c];
            if (fabs(wApA) / normFactor < 1e-300) {
                perf->singular = 1;
                break;
            }
            const double alpha = wArA / wApA;
            s = 0.0;
            for (int c = 0; c < n; ++c) {
                psi[c] += alpha * pA[c];
                rA[c] -= alpha * wA[c];
                s += fabs(rA[c]);
            }
            perf->final_residual = s / normFactor;
        } while ((++perf->n_iterations < ctl->max_iter && !or_conv(perf->final_residual, perf->initial_residual, ctl)) ||
                 perf->n_iterations < ctl->min_iter);
    }
    perf->converged = or_conv(perf->final_residual, perf->initial_residual, ctl);
    free(wA); free(rA); free(pA); free(rD);
    return 0;
}

/* Tmul: y = A^T x (upper and lower swap roles) */
void or_tmul(int n, int F, const int* owner, const int* neighbour, const double* diag, const double* upper,
             const double* lower, const double* x, double* y)
{
    or_amul(n, F, owner, neighbour, diag, upper, lower, x, 0, 0, 0, 0, y); /* or_amul(diag, lower, upper): swapped */
}

/* [OF] PBiCG::solve (Q32): rA = b - A psi, rT = b - A^T psi; per iteration wA = M^-1 rA,
 * wT = M^-T rT, wArT = wA.rT, pA/pT = w + beta p, wA = A pA, wT = A^T pT, wApT = wA.pT,
 * alpha = wArT/wApT, psi += alpha pA, rA -= alpha wA, rT -= alpha wT. */
int or_pbicg(int n, int F, const int* owner, const int* neighbour, const double* diag, const double* upper,
             const double* lower, const double* source, double* psi, const or_controls* ctl, int kind, int k,
             or_perf* perf)
{
    double* wA = (double*)calloc((size_t)n + 1, sizeof(double));
    double* wT = (double*)calloc((size_t)n + 1, sizeof(double));
    double* rA = (double*)calloc((size_t)n + 1, sizeof(double));
    double* rT = (double*)calloc((size_t)n + 1, sizeof(double));
    double* pA = (double*)calloc((size_t)n + 1, sizeof(double));
    double* pT = (double*)calloc((size_t)n + 1, sizeof(double));
    double* rD = (double*)calloc((size_t)n + 1, sizeof(double));
    or_amul(n, F, owner, neighbour, diag, lower, upper, psi, 0, 0, 0, 0, wA);
    or_tmul(n, F, owner, neighbour, diag, upper, lower, psi, wT);
    for (int c = 0; c < n; ++c) {
        rA[c] = source[c] - wA[c];
        rT[c] = source[c] - wT[c];
    }
    const double normFactor = or_norm_factor(n, F, owner, neighbour, diag, lower, upper, source, psi, wA);
    double s = 0.0;
    for (int c = 0; c < n; ++c) s += fabs(rA[c]);
    perf->initial_residual = s / normFactor;
    perf->final_residual = perf->initial_residual;
    perf->n_iterations = 0;
    perf->singular = 0;
    if (ctl->min_iter > 0 || !or_conv(perf->final_residual, perf->initial_residual, ctl)) {
        or_pc_setup(kind, n, F, owner, neighbour, diag, upper, lower, rD);
        double wArT = 1e300, wArTold;
        do {
            wArTold = wArT;
            or_pc_apply(kind, k, n, F, owner, neighbour, rD, upper, lower, rA, wA, 0);
            or_pc_apply(kind, k, n, F, owner, neighbour, rD, upper, lower, rT, wT, 1);
            wArT = 0.0;
            for (int c = 0; c < n; ++c) wArT += wA[c] * rT[c];
            if (perf->n_iterations == 0) {
                for (int c = 0; c < n; ++c) {
                    pA[c] = wA[c];
                    pT[c] = wT[c];
                }
            } else {
                const double beta = wArT / wArTold;
                for (int c = 0; c < n; ++c) {
                    pA[c] = wA[c] + beta * pA[c];
                    pT[c] = wT[c] + beta * pT[c];
                }
            }
            or_amul(n, F, owner, neighbour, diag, lower, upper, pA, 0, 0, 0, 0, wA);
            or_tmul(n, F, owner, neighbour, diag, upper, lower, pT, wT);
            double wApT = 0.0;
            for (int c = 0; c < n; ++c) wApT += wA[c] * pT[c];
            if (fabs(wApT) / normFactor < 1e-300) {
                perf->singular = 1;
                break;
            }
            const double alpha = wArT / wApT;
            s = 0.0;
            for (int c = 0; c < n; ++c) {
                psi[c] += alpha * pA[c];
                rA[c] -= alpha * wA[c];
                rT[c] -= alpha * wT[c];
                s += fabs(rA[c]);
            }
            perf->final_residual = s / normFactor;
        } while ((++perf->n_iterations < ctl->max_iter && !or_conv(perf->final_residual, perf->initial_residual, ctl)) ||
                 perf->n_iterations < ctl->min_iter);
    }
    perf->converged = or_conv(perf->final_residual, perf->initial_residual, ctl);
    free(wA); free(wT); free(rA); free(rT); free(pA); free(pT); free(rD);
    return 0;
}

/* [OF] PBiCG over nd domains (O8 + Q32): lower[p] the domain's lower coefficients; iface_t[p]
 * the coefficients Tmul uses on its processor faces (A^T couples row P to the remote cell with
 * A[remote][P]); the preconditioner is processor-local (Q31); sums in rank order; sumA of the
 * normFactor = diag + row's upper/lower + its Amul interface coefficients (Q17, Q35). */
int or_pbicg_dd(int nd, or_domain* D, const double* const* lower, const double* const* iface_t,
                const or_controls* ctl, int kind, int k, or_perf* perf)
{
    double **wA = (double**)calloc((size_t)nd, sizeof(double*)), **wT = (double**)calloc((size_t)nd, sizeof(double*));
    double **rA = (double**)calloc((size_t)nd, sizeof(double*)), **rT = (double**)calloc((size_t)nd, sizeof(double*));
    double **pA = (double**)calloc((size_t)nd, sizeof(double*)), **pT = (double**)calloc((size_t)nd, sizeof(double*));
    double **rD = (double**)calloc((size_t)nd, sizeof(double*)), **xr = (double**)calloc((size_t)nd, sizeof(double*));
    for (int p = 0; p < nd; ++p) {
        const size_t n = (size_t)D[p].n_cells + 1;
        wA[p] = (double*)calloc(n, sizeof(double));
        wT[p] = (double*)calloc(n, sizeof(double));
        rA[p] = (double*)calloc(n, sizeof(double));
        rT[p] = (double*)calloc(n, sizeof(double));
        pA[p] = (double*)calloc(n, sizeof(double));
        pT[p] = (double*)calloc(n, sizeof(double));
        rD[p] = (double*)calloc(n, sizeof(double));
        xr[p] = (double*)calloc((size_t)D[p].n_iface + 1, sizeof(double));
    }
    /* y = A x (T = 0) or A^T x (T = 1) on every domain, x_remote from the other domains */
#define OR_DD_MUL(T, X, Y)                                                                                         \
    do {                                                                                                           \
        for (int p = 0; p < nd; ++p)                                                                               \
            for (int i = 0; i < D[p].n_iface; ++i) xr[p][i] = (X)[D[p].iface_src_domain[i]][D[p].iface_src_cell[i]]; \
        for (int p = 0; p < nd; ++p)                                                                               \
            or_amul(D[p].n_cells, D[p].n_faces, D[p].owner, D[p].neighbour, D[p].diag, (T) ? D[p].upper : lower[p], \
                    (T) ? lower[p] : D[p].upper, (X)[p], D[p].n_iface, D[p].iface_cells,                          \
                    (T) ? iface_t[p] : D[p].iface_coeffs, xr[p], (Y)[p]);                                          \
    } while (0)
    double** psi = (double**)calloc((size_t)nd, sizeof(double*));
    for (int p = 0; p < nd; ++p) psi[p] = D[p].psi;
    OR_DD_MUL(0, psi, wA);
    OR_DD_MUL(1, psi, wT);
    for (int p = 0; p < nd; ++p)
        for (int c = 0; c < D[p].n_cells; ++c) {
            rA[p][c] = D[p].source[c] - wA[p][c];
            rT[p][c] = D[p].source[c] - wT[p][c];
        }
    double spsi = 0.0, ncell = 0.0;
    for (int p = 0; p < nd; ++p) {
        double t = 0.0;
        for (int c = 0; c < D[p].n_cells; ++c) t += D[p].psi[c];
        spsi += t;
        ncell += (double)D[p].n_cells;
    }
    const double xbar = spsi / ncell;
    double normFactor = 0.0;
    for (int p = 0; p < nd; ++p) {
        double* sumA = (double*)calloc((size_t)D[p].n_cells + 1, sizeof(double));
        for (int c = 0; c < D[p].n_cells; ++c) sumA[c] = D[p].diag[c];
        for (int f = 0; f < D[p].n_faces; ++f) {
            sumA[D[p].owner[f]] += D[p].upper[f];
            sumA[D[p].neighbour[f]] += lower[p][f];
        }
        for (int i = 0; i < D[p].n_iface; ++i) sumA[D[p].iface_cells[i]] += D[p].iface_coeffs[i];
        double t = 0.0;
        for (int c = 0; c < D[p].n_cells; ++c) {
            const double xref = sumA[c] * xbar;
            t += fabs(wA[p][c] - xref) + fabs(D[p].source[c] - xref);
        }
        normFactor += t;
        free(sumA);
    }
    normFactor += 1e-20;
    double smag = 0.0;
    for (int p = 0; p < nd; ++p) {
        double t = 0.0;
        for (int c = 0; c < D[p].n_cells; ++c) t += fabs(rA[p][c]);
        smag += t;
    }
    perf->initial_residual = smag / normFactor;
    perf->final_residual = perf->initial_residual;
    perf->n_iterations = 0;
    perf->singular = 0;
    if (ctl->min_iter > 0 || !or_conv(perf->final_residual, perf->initial_residual, ctl)) {
        for (int p = 0; p < nd; ++p)
            or_pc_setup(kind, D[p].n_cells, D[p].n_faces, D[p].owner, D[p].neighbour, D[p].diag, D[p].upper,
                        lower[p], rD[p]);
        double wArT = 1e300, wArTold;
        do {
            wArTold = wArT;
            wArT = 0.0;
            for (int p = 0; p < nd; ++p) {
                or_pc_apply(kind, k, D[p].n_cells, D[p].n_faces, D[p].owner, D[p].neighbour, rD[p], D[p].upper,
                            lower[p], rA[p], wA[p], 0);
                or_pc_apply(kind, k, D[p].n_cells, D[p].n_faces, D[p].owner, D[p].neighbour, rD[p], D[p].upper,
                            lower[p], rT[p], wT[p], 1);
                double t = 0.0;
                for (int c = 0; c < D[p].n_cells; ++c) t += wA[p][c] * rT[p][c];
                wArT += t;
            }
            for (int p = 0; p < nd; ++p) {
                if (perf->n_iterations == 0) {
                    for (int c = 0; c < D[p].n_cells; ++c) {
                        pA[p][c] = wA[p][c];
                        pT[p][c] = wT[p][c];
                    }
                } else {
                    const double beta = wArT / wArTold;
                    for (int c = 0; c < D[p].n_cells; ++c) {
                        pA[p][c] = wA[p][c] + beta * pA[p][c];
                        pT[p][c] = wT[p][c] + beta * pT[p][c];
                    }
                }
            }
            OR_DD_MUL(0, pA, wA);
            OR_DD_MUL(1, pT, wT);
            double wApT = 0.0;
            for (int p = 0; p < nd; ++p) {
                double t = 0.0;
                for (int c = 0; c < D[p].n_cells; ++c) t += wA[p][c] * pT[p][c];
                wApT += t;
            }
            if (fabs(wApT) / normFactor < 1e-300) {
                perf->singular = 1;
                break;
            }
            const double alpha = wArT / wApT;
            smag = 0.0;
            for (int p = 0; p < nd; ++p) {
                double t = 0.0;
                for (int c = 0; c < D[p].n_cells; ++c) {
                    D[p].psi[c] += alpha * pA[p][c];
                    rA[p][c] -= alpha * wA[p][c];
                    rT[p][c] -= alpha * wT[p][c];
                    t += fabs(rA[p][c]);
                }
                smag += t;
            }
            perf->final_residual = smag / normFactor;
        } while ((++perf->n_iterations < ctl->max_iter && !or_conv(perf->final_residual, perf->initial_residual, ctl)) ||
                 perf->n_iterations < ctl->min_iter);
    }
#undef OR_DD_MUL
    perf->converged = or_conv(perf->final_residual, perf->initial_residual, ctl);
    for (int p = 0; p < nd; ++p) {
        free(wA[p]); free(wT[p]); free(rA[p]); free(rT[p]); free(pA[p]); free(pT[p]); free(rD[p]); free(xr[p]);
    }
    free(wA); free(wT); free(rA); free(rT); free(pA); free(pT); free(rD); free(xr); free(psi);
    return 0;
}

/* LDU -> CSR (Q34; "a map computed by the Radix sort ... of the sparsity pattern"):
 * rows ascending, columns ascending within a row; map[k] indexes [diag (n) | upper (F) | lower (F)]:
 * row P col N (P = owner) is upper[f], row N col P is lower[f].  row_ptr [n+1], col/map [n+2F]. */
static int or_csr_cmp(const void* a, const void* b)
{
    const int* x = (const int*)a;
    const int* y = (const int*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    return x[1] < y[1] ? -1 : (x[1] > y[1]);
}

void or_ldu_to_csr(int n, int F, const int* owner, const int* neighbour, int* row_ptr, int* col, int* map)
{
    const int nnz = n + 2 * F;
    int* t = (int*)malloc(sizeof(int) * 3 * (size_t)(nnz + 1));
    int m = 0;
    for (int c = 0; c < n; ++c, ++m) t[3 * m] = c, t[3 * m + 1] = c, t[3 * m + 2] = c;
    for (int f = 0; f < F; ++f, ++m) t[3 * m] = owner[f], t[3 * m + 1] = neighbour[f], t[3 * m + 2] = n + f;
    for (int f = 0; f < F; ++f, ++m) t[3 * m] = neighbour[f], t[3 * m + 1] = owner[f], t[3 * m + 2] = n + F + f;
    qsort(t, (size_t)nnz, 3 * sizeof(int), or_csr_cmp);
    for (int c = 0; c <= n; ++c) row_ptr[c] = 0;
    for (int i = 0; i < nnz; ++i) {
        row_ptr[t[3 * i] + 1]++;
        col[i] = t[3 * i + 1];
        map[i] = t[3 * i + 2];
    }
    for (int c = 0; c < n; ++c) row_ptr[c + 1] += row_ptr[c];
    free(t);
}

/* ------------------------------------------------------------------------- */
/* O7 dense brute force (N <= 64): entries (P,N) = upper, (N,P) = lower       */
/* ------------------------------------------------------------------------- */

void or_dense_from_ldu(int n, int n_faces, const int* owner, const int* neighbour, const double* diag,
                       const double* lower, const double* upper, double* A)
{
    for (int i = 0; i < n * n; ++i) A[i] = 0.0;
    for (int c = 0; c < n; ++c) A[c * n + c] = diag[c];
    for (int f = 0; f < n_faces; ++f) {
        A[owner[f] * n + neighbour[f]] += upper[f];
        A[neighbour[f] * n + owner[f]] += lower[f];
    }
}

void or_dense_matvec(int n, const double* A, const double* x, double* y)
{
    for (int i = 0; i < n; ++i) {
        long double s = 0.0L;
        for (int j = 0; j < n; ++j) s += (long double)A[i * n + j] * (long double)x[j];
        y[i] = (double)s;
    }
}

/* Gaussian elimination with partial pivoting in long double; 0 ok, 1 singular */
int or_dense_solve(int n, const double* A, const double* b, double* x)
{
    long double* M = (long double*)malloc(sizeof(long double) * (size_t)n * (size_t)(n + 1));
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) M[i * (n + 1) + j] = A[i * n + j];
        M[i * (n + 1) + n] = b[i];
    }
    for (int k = 0; k < n; ++k) {
        int piv = k;
        for (int i = k + 1; i < n; ++i)
            if (fabsl(M[i * (n + 1) + k]) > fabsl(M[piv * (n + 1) + k])) piv = i;
        if (M[piv * (n + 1) + k] == 0.0L) {
            free(M);
            return 1;
        }
        if (piv != k)
            for (int j = 0; j <= n; ++j) {
                long double t = M[k * (n + 1) + j];
                M[k * (n + 1) + j] = M[piv * (n + 1) + j];
                M[piv * (n + 1) + j] = t;
            }
        for (int i = k + 1; i < n; ++i) {
            long double m = M[i * (n + 1) + k] / M[k * (n + 1) + k];
            for (int j = k; j <= n; ++j) M[i * (n + 1) + j] -= m * M[k * (n + 1) + j];
        }
    }
    long double* xs = (long double*)malloc(sizeof(long double) * (size_t)(n > 0 ? n : 1));
    for (int i = n - 1; i >= 0; --i) {
        long double s = M[i * (n + 1) + n];
        for (int j = i + 1; j < n; ++j) s -= M[i * (n + 1) + j] * xs[j];
        xs[i] = s / M[i * (n + 1) + i];
    }
    for (int i = 0; i < n; ++i) x[i] = (double)xs[i];
    free(xs);
    free(M);
    return 0;
}
