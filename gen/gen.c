/*
 * gen/gen.c -- seeded synthetic INPUTS shared by the oracle tests and the CUDA path.
 *
 * This module holds none of the method's arithmetic (no delta coefficients,
 * no interpolation weights, no matrix coefficients, no solver step).  It only
 * produces what a mesh generator / case setup would hand to OpenFOAM:
 * owner/neighbour addressing, face area vectors Sf, face centres Cf, cell
 * centres C, cell volumes V, boundary faces, and seeded cell fields.
 *
 * Recipe (SURVEY.md §8(d) "Synthetic inputs"):
 *   RNG      counter-based splitmix64(seed ^ (stream << 40) ^ id), U = (x >> 11) * 2^-53
 *   lattice  nx*ny*nz hex cells on [0,Lx]x[0,Ly]x[0,Lz], cell id i + nx*(j + ny*k)
 *   jitter   interior vertex components moved by U(-a*h, a*h) (seed, streams 0/1/2,
 *            keyed by the global vertex id) -- boundary planes stay planar
 *   faces    quad vector area Sf = 1/2 (x2 - x0) x (x3 - x1), Cf = mean of 4 vertices,
 *            C = mean of 8 vertices, V = 1/3 sum_out Cf.Sf
 *   order    internal faces sorted by (owner, neighbour) -- OpenFOAM upper-triangular
 *            order (lduAddressing)
 *
 * Build: gcc -O2 -fPIC -shared (see gen/__init__.py).  int32 labels, fp64 scalars.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

uint64_t gen_splitmix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

double gen_uniform(uint64_t seed, uint64_t stream, uint64_t id)
{
    return (double)(gen_splitmix64(seed ^ (stream << 40) ^ id) >> 11) * 0x1.0p-53;
}

void gen_uniform_fill(uint64_t seed, uint64_t stream, int64_t n, const int32_t* ids, double* out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = gen_uniform(seed, stream, ids ? (uint64_t)ids[i] : (uint64_t)i);
}

/* ------------------------------------------------------------------------- */
/* hex lattice                                                               */
/* ------------------------------------------------------------------------- */

void gen_hex_counts(int nx, int ny, int nz, int64_t* n_cells, int64_t* n_faces, int64_t* patch_sizes)
{
    *n_cells = (int64_t)nx * ny * nz;
    *n_faces = (int64_t)(nx - 1) * ny * nz + (int64_t)nx * (ny - 1) * nz + (int64_t)nx * ny * (nz - 1);
    patch_sizes[0] = patch_sizes[1] = (int64_t)ny * nz; /* xmin, xmax */
    patch_sizes[2] = patch_sizes[3] = (int64_t)nx * nz; /* ymin, ymax */
    patch_sizes[4] = patch_sizes[5] = (int64_t)nx * ny; /* zmin, zmax */
}

typedef struct {
    int nx, ny, nz;
    const double* X; /* vertices [(nx+1)(ny+1)(nz+1)][3] */
} lattice;

static inline const double* vtx(const lattice* L, int i, int j, int k)
{
    return L->X + 3 * ((int64_t)i + (int64_t)(L->nx + 1) * ((int64_t)j + (int64_t)(L->ny + 1) * k));
}

static void quad(const double* x0, const double* x1, const double* x2, const double* x3, double sign,
                 double* Sf, double* Cf, double* magSf)
{
    double a[3], b[3];
    for (int d = 0; d < 3; ++d) {
        a[d] = x2[d] - x0[d];
        b[d] = x3[d] - x1[d];
    }
    double s[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
    for (int d = 0; d < 3; ++d) {
        Sf[d] = sign * (0.5 * s[d]);
        Cf[d] = 0.25 * (((x0[d] + x1[d]) + x2[d]) + x3[d]);
    }
    *magSf = sqrt(Sf[0] * Sf[0] + Sf[1] * Sf[1] + Sf[2] * Sf[2]);
}

/* +x face on vertex plane i, row (j,k) */
static void xface(const lattice* L, int i, int j, int k, double sign, double* Sf, double* Cf, double* m)
{
    quad(vtx(L, i, j, k), vtx(L, i, j + 1, k), vtx(L, i, j + 1, k + 1), vtx(L, i, j, k + 1), sign, Sf, Cf, m);
}
static void yface(const lattice* L, int i, int j, int k, double sign, double* Sf, double* Cf, double* m)
{
    quad(vtx(L, i, j, k), vtx(L, i, j, k + 1), vtx(L, i + 1, j, k + 1), vtx(L, i + 1, j, k), sign, Sf, Cf, m);
}
static void zface(const lattice* L, int i, int j, int k, double sign, double* Sf, double* Cf, double* m)
{
    quad(vtx(L, i, j, k), vtx(L, i + 1, j, k), vtx(L, i + 1, j + 1, k), vtx(L, i, j + 1, k), sign, Sf, Cf, m);
}

/*
 * Fill a lattice mesh.  Boundary faces are concatenated in patch order
 * xmin, xmax, ymin, ymax, zmin, zmax, each in ascending cell-id order.
 * Returns 0 on success, 1 on allocation failure.
 */
int gen_hex_fill(int nx, int ny, int nz, double Lx, double Ly, double Lz, double jitter, uint64_t seed,
                 int32_t* owner, int32_t* neighbour, double* Sf, double* magSf, double* Cf,
                 double* C, double* V, int32_t* bcells, double* bSf, double* bmagSf, double* bCf)
{
    int64_t nv = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
    double* X = (double*)malloc(sizeof(double) * 3 * nv);
    if (!X) return 1;
    const double hx = Lx / nx, hy = Ly / ny, hz = Lz / nz;
    for (int k = 0; k <= nz; ++k)
        for (int j = 0; j <= ny; ++j)
            for (int i = 0; i <= nx; ++i) {
                int64_t id = (int64_t)i + (int64_t)(nx + 1) * ((int64_t)j + (int64_t)(ny + 1) * k);
                double* x = X + 3 * id;
                x[0] = Lx * i / nx;
                x[1] = Ly * j / ny;
                x[2] = Lz * k / nz;
                if (jitter > 0.0) {
                    if (i > 0 && i < nx) x[0] += (2.0 * gen_uniform(seed, 0, (uint64_t)id) - 1.0) * jitter * hx;
                    if (j > 0 && j < ny) x[1] += (2.0 * gen_uniform(seed, 1, (uint64_t)id) - 1.0) * jitter * hy;
                    if (k > 0 && k < nz) x[2] += (2.0 * gen_uniform(seed, 2, (uint64_t)id) - 1.0) * jitter * hz;
                }
            }
    lattice L = {nx, ny, nz, X};
    const int64_t N = (int64_t)nx * ny * nz;

    for (int64_t c = 0; c < N; ++c) V[c] = 0.0;

    /* cell centres */
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                int64_t c = (int64_t)i + (int64_t)nx * ((int64_t)j + (int64_t)ny * k);
                for (int d = 0; d < 3; ++d) {
                    double s = 0.0;
                    for (int dk = 0; dk < 2; ++dk)
                        for (int dj = 0; dj < 2; ++dj)
                            for (int di = 0; di < 2; ++di) s += vtx(&L, i + di, j + dj, k + dk)[d];
                    C[3 * c + d] = 0.125 * s;
                }
            }

    /* internal faces in (owner, neighbour) order */
    int64_t f = 0;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                int64_t c = (int64_t)i + (int64_t)nx * ((int64_t)j + (int64_t)ny * k);
                if (i < nx - 1) {
                    owner[f] = (int32_t)c;
                    neighbour[f] = (int32_t)(c + 1);
                    xface(&L, i + 1, j, k, 1.0, Sf + 3 * f, Cf + 3 * f, magSf + f);
                    ++f;
                }
                if (j < ny - 1) {
                    owner[f] = (int32_t)c;
                    neighbour[f] = (int32_t)(c + nx);
                    yface(&L, i, j + 1, k, 1.0, Sf + 3 * f, Cf + 3 * f, magSf + f);
                    ++f;
                }
                if (k < nz - 1) {
                    owner[f] = (int32_t)c;
                    neighbour[f] = (int32_t)(c + (int64_t)nx * ny);
                    zface(&L, i, j, k + 1, 1.0, Sf + 3 * f, Cf + 3 * f, magSf + f);
                    ++f;
                }
            }
    const int64_t F = f;
    for (f = 0; f < F; ++f) {
        double cs = Cf[3 * f] * Sf[3 * f] + Cf[3 * f + 1] * Sf[3 * f + 1] + Cf[3 * f + 2] * Sf[3 * f + 2];
        V[owner[f]] += cs;
        V[neighbour[f]] -= cs;
    }

    /* boundary faces */
    int64_t b = 0;
#define BFACE(FN, I, J, K, SIGN, CELL)                                                   \
    do {                                                                                 \
        bcells[b] = (int32_t)(CELL);                                                     \
        FN(&L, I, J, K, SIGN, bSf + 3 * b, bCf + 3 * b, bmagSf + b);                     \
        V[CELL] += bCf[3 * b] * bSf[3 * b] + bCf[3 * b + 1] * bSf[3 * b + 1] + bCf[3 * b + 2] * bSf[3 * b + 2]; \
        ++b;                                                                             \
    } while (0)
    for (int side = 0; side < 2; ++side) /* xmin, xmax */
        for (int k = 0; k < nz; ++k)
            for (int j = 0; j < ny; ++j) {
                int i = side ? nx - 1 : 0;
                int64_t c = (int64_t)i + (int64_t)nx * ((int64_t)j + (int64_t)ny * k);
                BFACE(xface, side ? nx : 0, j, k, side ? 1.0 : -1.0, c);
            }
    for (int side = 0; side < 2; ++side) /* ymin, ymax */
        for (int k = 0; k < nz; ++k)
            for (int i = 0; i < nx; ++i) {
                int j = side ? ny - 1 : 0;
                int64_t c = (int64_t)i + (int64_t)nx * ((int64_t)j + (int64_t)ny * k);
                BFACE(yface, i, side ? ny : 0, k, side ? 1.0 : -1.0, c);
            }
    for (int side = 0; side < 2; ++side) /* zmin, zmax */
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                int k = side ? nz - 1 : 0;
                int64_t c = (int64_t)i + (int64_t)nx * ((int64_t)j + (int64_t)ny * k);
                BFACE(zface, i, j, side ? nz : 0, side ? 1.0 : -1.0, c);
            }
#undef BFACE
    for (int64_t c = 0; c < N; ++c) V[c] = V[c] / 3.0;
    free(X);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* cell permutation (Fisher-Yates, counter-based)                            */
/* ------------------------------------------------------------------------- */

/* perm[old] = new.  order[k] starts as k; for i = n-1..1 swap order[i], order[j],
 * j = floor(U(seed, 1, i) * (i + 1)). */
void gen_random_perm(int64_t n, uint64_t seed, int32_t* perm)
{
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t k = 0; k < n; ++k) order[k] = (int32_t)k;
    for (int64_t i = n - 1; i >= 1; --i) {
        int64_t j = (int64_t)(gen_uniform(seed, 1, (uint64_t)i) * (double)(i + 1));
        if (j > i) j = i;
        int32_t t = order[i];
        order[i] = order[j];
        order[j] = t;
    }
    for (int64_t k = 0; k < n; ++k) perm[order[k]] = (int32_t)k;
    free(order);
}

/*
 * Re-key the internal faces under a cell permutation perm[old] = new:
 * (a, b) = (perm[owner], perm[neighbour]); owner' = min, neighbour' = max;
 * if a > b the face is flipped (Sf is negated by the caller via flip[]).
 * Faces are then stably re-sorted by (owner', neighbour'), ties by old face
 * index (two stable counting-sort passes).  face_map[new] = old.
 */
int gen_permute_faces(int64_t n_cells, int64_t n_faces, const int32_t* perm, const int32_t* owner,
                      const int32_t* neighbour, int32_t* owner_out, int32_t* neighbour_out, int32_t* face_map,
                      int8_t* flip)
{
    int32_t* a = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_faces + 1));
    int32_t* bb = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_faces + 1));
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_faces + 1));
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_cells + 1));
    if (!a || !bb || !tmp || !cnt) return 1;
    for (int64_t f = 0; f < n_faces; ++f) {
        int32_t x = perm[owner[f]], y = perm[neighbour[f]];
        a[f] = x < y ? x : y;
        bb[f] = x < y ? y : x;
    }
    /* pass 1: stable by neighbour' */
    memset(cnt, 0, sizeof(int64_t) * (size_t)(n_cells + 1));
    for (int64_t f = 0; f < n_faces; ++f) cnt[bb[f] + 1]++;
    for (int64_t c = 0; c < n_cells; ++c) cnt[c + 1] += cnt[c];
    for (int64_t f = 0; f < n_faces; ++f) tmp[cnt[bb[f]]++] = (int32_t)f;
    /* pass 2: stable by owner' */
    memset(cnt, 0, sizeof(int64_t) * (size_t)(n_cells + 1));
    for (int64_t f = 0; f < n_faces; ++f) cnt[a[f] + 1]++;
    for (int64_t c = 0; c < n_cells; ++c) cnt[c + 1] += cnt[c];
    for (int64_t t = 0; t < n_faces; ++t) {
        int32_t f = tmp[t];
        face_map[cnt[a[f]]++] = f;
    }
    for (int64_t g = 0; g < n_faces; ++g) {
        int32_t f = face_map[g];
        owner_out[g] = a[f];
        neighbour_out[g] = bb[f];
        flip[g] = (int8_t)(perm[owner[f]] > perm[neighbour[f]]);
    }
    free(a);
    free(bb);
    free(tmp);
    free(cnt);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* cell fields                                                               */
/* ------------------------------------------------------------------------- */

/* gamma_c = exp(0.5 xi_c), xi ~ N(0,1) by Box-Muller keyed by the global cell id */
void gen_gamma_lognormal(int64_t n, const int32_t* gid, uint64_t seed, double* gamma)
{
    const double two_pi = 6.283185307179586476925286766559;
    for (int64_t c = 0; c < n; ++c) {
        double u1 = gen_uniform(seed, 0, (uint64_t)gid[c]);
        double u2 = gen_uniform(seed, 1, (uint64_t)gid[c]);
        double xi = sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2);
        gamma[c] = exp(0.5 * xi);
    }
}

/* b_c = V_c (2 U_c - 1), then b -= mean(b) (sum in array order) */
void gen_rhs(int64_t n, const int32_t* gid, const double* V, uint64_t seed, double* b)
{
    double s = 0.0;
    for (int64_t c = 0; c < n; ++c) {
        b[c] = V[c] * (2.0 * gen_uniform(seed, 0, (uint64_t)gid[c]) - 1.0);
        s += b[c];
    }
    double mean = n > 0 ? s / (double)n : 0.0;
    for (int64_t c = 0; c < n; ++c) b[c] -= mean;
}

/* ------------------------------------------------------------------------- */
/* window of a global lattice (one rank's block of a decomposed lattice)     */
/* ------------------------------------------------------------------------- */

typedef struct {
    int NX, NY, NZ;
    double Lx, Ly, Lz, jitter;
    uint64_t seed;
} glat;

static void gvtx(const glat* g, int i, int j, int k, double* x)
{
    int64_t id = (int64_t)i + (int64_t)(g->NX + 1) * ((int64_t)j + (int64_t)(g->NY + 1) * k);
    x[0] = g->Lx * i / g->NX;
    x[1] = g->Ly * j / g->NY;
    x[2] = g->Lz * k / g->NZ;
    if (g->jitter > 0.0) {
        if (i > 0 && i < g->NX) x[0] += (2.0 * gen_uniform(g->seed, 0, (uint64_t)id) - 1.0) * g->jitter * (g->Lx / g->NX);
        if (j > 0 && j < g->NY) x[1] += (2.0 * gen_uniform(g->seed, 1, (uint64_t)id) - 1.0) * g->jitter * (g->Ly / g->NY);
        if (k > 0 && k < g->NZ) x[2] += (2.0 * gen_uniform(g->seed, 2, (uint64_t)id) - 1.0) * g->jitter * (g->Lz / g->NZ);
    }
}

static void gquad(const glat* g, int axis, int i, int j, int k, double sign, double* Sf, double* Cf, double* m)
{
    double v[4][3];
    if (axis == 0) {
        gvtx(g, i, j, k, v[0]); gvtx(g, i, j + 1, k, v[1]); gvtx(g, i, j + 1, k + 1, v[2]); gvtx(g, i, j, k + 1, v[3]);
    } else if (axis == 1) {
        gvtx(g, i, j, k, v[0]); gvtx(g, i, j, k + 1, v[1]); gvtx(g, i + 1, j, k + 1, v[2]); gvtx(g, i + 1, j, k, v[3]);
    } else {
        gvtx(g, i, j, k, v[0]); gvtx(g, i + 1, j, k, v[1]); gvtx(g, i + 1, j + 1, k, v[2]); gvtx(g, i, j + 1, k, v[3]);
    }
    quad(v[0], v[1], v[2], v[3], sign, Sf, Cf, m);
}

static void gcentre(const glat* g, int i, int j, int k, double* C)
{
    double v[8][3];
    int n = 0;
    for (int dk = 0; dk < 2; ++dk)
        for (int dj = 0; dj < 2; ++dj)
            for (int di = 0; di < 2; ++di) gvtx(g, i + di, j + dj, k + dk, v[n++]);
    for (int d = 0; d < 3; ++d) {
        double s = 0.0;
        for (int q = 0; q < 8; ++q) s += v[q][d];
        C[d] = 0.125 * s;
    }
}

/* global face id of the face of cell (i,j,k) along axis (owner side) in the
 * undecomposed lattice: faces owned by earlier cells + earlier axes of this cell */
static int64_t gface_id(const glat* g, int i, int j, int k, int axis)
{
    const int64_t NX = g->NX, NY = g->NY, NZ = g->NZ;
    const int64_t c = (int64_t)i + NX * ((int64_t)j + NY * k);
    int64_t cx = ((int64_t)j + NY * k) * (NX - 1) + (i < NX - 1 ? i : NX - 1);
    int64_t cy = (int64_t)k * NX * (NY - 1) + (j < NY - 1 ? (int64_t)j * NX + i : (NY - 1) * NX);
    int64_t cz = k < NZ - 1 ? c : NX * NY * (NZ - 1);
    int64_t id = cx + cy + cz;
    if (axis >= 1 && i < NX - 1) id += 1;
    if (axis >= 2 && j < NY - 1) id += 1;
    return id;
}

void gen_window_counts(int nx, int ny, int nz, int64_t* n_cells, int64_t* n_faces, int64_t* side_sizes)
{
    gen_hex_counts(nx, ny, nz, n_cells, n_faces, side_sizes);
}

/*
 * Cells [i0, i0+nx) x [j0, j0+ny) x [k0, k0+nz) of the global lattice NX x NY x NZ
 * on [0,Lx]x[0,Ly]x[0,Lz].  Local cell id = li + nx (lj + ny lk).  Internal faces
 * (both cells inside) in local (owner, neighbour) order.  The 6 sides of the window
 * (xmin, xmax, ymin, ymax, zmin, zmax; cells in local id order) are returned as
 * boundary faces with outward Sf; for each, if the side is interior to the global
 * lattice, also the centre of the cell across (bnC), its global id (bngid) and
 * the global face id (bgface); else bngid = -1.
 * gid[c] = global cell id.  Vertex coordinates use the global formula, so both
 * sides of a cut agree bitwise.
 */
int gen_hex_window(int NX, int NY, int NZ, double Lx, double Ly, double Lz, double jitter, uint64_t seed,
                   int i0, int j0, int k0, int nx, int ny, int nz, int32_t* owner, int32_t* neighbour, double* Sf,
                   double* magSf, double* Cf, double* C, double* V, int32_t* gid, int32_t* bcells, double* bSf,
                   double* bmagSf, double* bCf, double* bnC, int32_t* bngid, int32_t* bgface)
{
    glat g = {NX, NY, NZ, Lx, Ly, Lz, jitter, seed};
    const int64_t N = (int64_t)nx * ny * nz;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                int64_t c = (int64_t)i + (int64_t)nx * ((int64_t)j + (int64_t)ny * k);
                gcentre(&g, i0 + i, j0 + j, k0 + k, C + 3 * c);
                gid[c] = (int32_t)((int64_t)(i0 + i) + (int64_t)NX * ((int64_t)(j0 + j) + (int64_t)NY * (k0 + k)));
                V[c] = 0.0;
            }
    int64_t f = 0;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                int64_t c = (int64_t)i + (int64_t)nx * ((int64_t)j + (int64_t)ny * k);
                const int I = i0 + i, J = j0 + j, K = k0 + k;
                if (i < nx - 1) {
                    owner[f] = (int32_t)c; neighbour[f] = (int32_t)(c + 1);
                    gquad(&g, 0, I + 1, J, K, 1.0, Sf + 3 * f, Cf + 3 * f, magSf + f); ++f;
                }
                if (j < ny - 1) {
                    owner[f] = (int32_t)c; neighbour[f] = (int32_t)(c + nx);
                    gquad(&g, 1, I, J + 1, K, 1.0, Sf + 3 * f, Cf + 3 * f, magSf + f); ++f;
                }
                if (k < nz - 1) {
                    owner[f] = (int32_t)c; neighbour[f] = (int32_t)(c + (int64_t)nx * ny);
                    gquad(&g, 2, I, J, K + 1, 1.0, Sf + 3 * f, Cf + 3 * f, magSf + f); ++f;
                }
            }
    const int64_t F = f;
    for (f = 0; f < F; ++f) {
        double cs = Cf[3 * f] * Sf[3 * f] + Cf[3 * f + 1] * Sf[3 * f + 1] + Cf[3 * f + 2] * Sf[3 * f + 2];
        V[owner[f]] += cs;
        V[neighbour[f]] -= cs;
    }
    int64_t b = 0;
    for (int axis = 0; axis < 3; ++axis)
        for (int side = 0; side < 2; ++side) {
            const int na = axis == 0 ? nx : (axis == 1 ? ny : nz);
            const int la = side ? na - 1 : 0; /* local index along axis of the side's cells */
            for (int k = 0; k < nz; ++k)
                for (int j = 0; j < ny; ++j)
                    for (int i = 0; i < nx; ++i) {
                        const int li = axis == 0 ? la : i, lj = axis == 1 ? la : j, lk = axis == 2 ? la : k;
                        if ((axis == 0 && i != 0) || (axis == 1 && j != 0) || (axis == 2 && k != 0)) continue;
                        const int64_t c = (int64_t)li + (int64_t)nx * ((int64_t)lj + (int64_t)ny * lk);
                        const int I = i0 + li, J = j0 + lj, K = k0 + lk;
                        /* vertex plane of the face along the axis */
                        int pi = I, pj = J, pk = K;
                        if (side) { if (axis == 0) pi++; else if (axis == 1) pj++; else pk++; }
                        bcells[b] = (int32_t)c;
                        gquad(&g, axis, pi, pj, pk, side ? 1.0 : -1.0, bSf + 3 * b, bCf + 3 * b, bmagSf + b);
                        V[c] += bCf[3 * b] * bSf[3 * b] + bCf[3 * b + 1] * bSf[3 * b + 1] + bCf[3 * b + 2] * bSf[3 * b + 2];
                        int RI = I, RJ = J, RK = K; /* cell across */
                        int inside;
                        if (axis == 0) { RI += side ? 1 : -1; inside = RI >= 0 && RI < NX; }
                        else if (axis == 1) { RJ += side ? 1 : -1; inside = RJ >= 0 && RJ < NY; }
                        else { RK += side ? 1 : -1; inside = RK >= 0 && RK < NZ; }
                        if (inside) {
                            gcentre(&g, RI, RJ, RK, bnC + 3 * b);
                            bngid[b] = (int32_t)((int64_t)RI + (int64_t)NX * ((int64_t)RJ + (int64_t)NY * RK));
                            /* the global owner is the smaller id: the + side's local cell, the - side's remote cell */
                            bgface[b] = side ? (int32_t)gface_id(&g, I, J, K, axis) : (int32_t)gface_id(&g, RI, RJ, RK, axis);
                        } else {
                            bnC[3 * b] = bnC[3 * b + 1] = bnC[3 * b + 2] = 0.0;
                            bngid[b] = -1;
                            bgface[b] = -1;
                        }
                        ++b;
                    }
        }
    for (int64_t c = 0; c < N; ++c) V[c] = V[c] / 3.0;
    return 0;
}
