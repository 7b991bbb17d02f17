// host.h -- host-side mesh logic (mesh_host.cpp).
#pragma once
#include <string>
#include <vector>

namespace spuma {
bool valid_addressing(int N, int F, const int* owner, const int* neighbour, std::string* why);
std::vector<int> rcm_permutation(int N, int F, const int* owner, const int* neighbour);  // perm[old] = new
void rekey_faces(int N, int F, const int* perm, const int* owner, const int* neighbour, std::vector<int>& owner_out,
                 std::vector<int>& neighbour_out, std::vector<int>& face_map, std::vector<char>& flip);
void derived_addressing(int N, int F, const int* owner, const int* neighbour, std::vector<int>& ownerStart,
                        std::vector<int>& losort, std::vector<int>& losortStart, std::vector<int>& ownerLo);
// SELL-C (C = 32) layout of the Amul rows (variant 6/7).  Per chunk of 32 cells:
// meta = {nbase, obase, wn, wo}; neighbour-side slot j of lane l at nslot[nbase + 32 j + l]
// = (ownerLo << 5) | (face - ownerStart[ownerLo]) in losort order, 0xFFFFFFFF = empty;
// owner-side slot j at oslot[obase + 32 j + l] = neighbour[ownerStart[c] + j], -1 = empty.
struct SellHost {
    std::vector<int> meta;          // [4 * chunks]
    std::vector<unsigned> nslot;
    std::vector<int> oslot;
    bool ok = false;                // false: a column >= 2^27 - 1 or a position >= 31 (not encodable)
    int uniform_wn = -1, uniform_wo = -1;  // >= 0: every chunk has these widths (bases = 32 k w)
};
SellHost build_sell(int N, const std::vector<int>& ownerStart, const std::vector<int>& losortStart,
                    const std::vector<int>& losort, const std::vector<int>& ownerLo,
                    const std::vector<int>& neighbour);

// Chunk-stencil compression of the uniform ELL rows (variant 8): per 32-cell
// chunk, the distinct column offsets (col - c) of each side when there are at most 3 per side
// (meta[8 k] = 1; meta[8 k + 1 .. 3] neighbour side, [8 k + 4 .. 6] owner side, ascending,
// unused = 0); per cell one word: bit t = neighbour-side offset t present, bit 3 + t =
// owner-side offset t present, bits 6 + 5 t = position of the neighbour-side face t in its
// owner's faces.  Chunks with more distinct offsets keep meta[8 k] = 0 (explicit slots).
struct EllStencil {
    std::vector<int> meta;
    std::vector<unsigned> lane;
    int compressed = 0;  // chunks encoded
};
EllStencil build_ell_stencil(int N, const std::vector<int>& ownerStart, const std::vector<int>& losortStart,
                             const std::vector<int>& losort, const std::vector<int>& ownerLo,
                             const std::vector<int>& neighbour);

// Lattice slots (Amul variant 12): if every internal face's column offset
// d = neighbour - owner takes one of at most 3 values and no owner has two faces with the same
// offset (a structured numbering, e.g. an n^3 block: d in {1, n, n^2}), return their number K and
// the offsets D[0] < ... < D[K-1]; otherwise 0.  Face f then lives in slot t (D[t] = d) of its
// owner row, and the rows of the Amul need no index arrays at all.
int lattice_offsets(int N, int F, const int* owner, const int* neighbour, int D[3]);

// per-cell lists of the items i with keep[i], in input order
void cell_lists(int N, const std::vector<int>& cell_of, const std::vector<char>& keep, std::vector<int>& start,
                std::vector<int>& items);

// Dependency levels of the DIC/DILU recurrences (§8(f3)/(f4)): forward row c waits on the owners
// of its neighbour-side faces, backward row c on the neighbours of its owner-side faces.  order_*
// = rows sorted by level (ascending cell within a level); depth = number of levels; width = the
// widest level.
void level_schedule(int N, const std::vector<int>& owner, const std::vector<int>& neighbour,
                    const std::vector<int>& ownerStart, const std::vector<int>& losortStart,
                    const std::vector<int>& losort, std::vector<int>& order_f, std::vector<int>& order_b,
                    int& depth_f, int& depth_b, int& width_f, int& width_b);
// LDU -> CSR (Q34): per row the neighbour-side faces in losort order (owners ascending), the
// diagonal, the owner-side faces; map into [diag (N) | upper (F) | lower (F)].
void ldu_to_csr_host(int N, int F, const std::vector<int>& owner, const std::vector<int>& neighbour,
                     const std::vector<int>& ownerStart, const std::vector<int>& losortStart,
                     const std::vector<int>& losort, std::vector<int>& row_ptr, std::vector<int>& col,
                     std::vector<int>& map);

// GAMG hierarchy (readings Q22, Q27).  Level l's arrays; ftc and the
// next level's agglomeration lists are empty on the coarsest level.
struct GamgHostLevel {
    int n = 0, F = 0;
    std::vector<int> owner, neighbour, ownerStart, losort, losortStart, ownerLo;  // l >= 1 (level 0: the mesh's)
    std::vector<double> w;                      // face weights (level 0: |Sf|)
    std::vector<int> ftc;                       // [n] fine -> coarse cell of the next level
    std::vector<int> frestrict;                 // [F] fine face -> coarse face, -1 inside an agglomerate
    std::vector<int> cStart, cList;             // next level: coarse cell -> fine cells (ascending)
    std::vector<int> ciStart, ciList;           // next level: coarse cell -> agglomerate-internal fine faces
    std::vector<int> cfStart, cfList;           // next level: coarse face -> fine faces (ascending)
    // processor interfaces of the level (n_ranks > 1; readings Q36-Q38): faces in (patch, face)
    // order, per-patch counts, per-cell lists (Q10 order) and, towards the next level, the
    // coarse interface face -> fine interface faces lists (ascending) of the Galerkin sums
    std::vector<int> if_cell, if_count, ifStart, ifIdx, cifStart, cifList;
};
// Levels are added while the current level has more than n_coarsest cells, the pairwise
// pass reduces the count and fewer than max_levels exist.  Level 0 takes the given
// addressing (sorted lduAddressing + derived arrays) and weights.
std::vector<GamgHostLevel> gamg_hierarchy(int N, int F, const std::vector<int>& owner,
                                          const std::vector<int>& neighbour, const std::vector<int>& ownerStart,
                                          const std::vector<int>& losortStart, const std::vector<int>& losort,
                                          const std::vector<int>& ownerLo, const std::vector<double>& w,
                                          int n_coarsest, int max_levels);

// Decomposed hierarchy (readings Q36, Q37): processor-local agglomeration; a level is added
// while sum over ranks of the level's cells > n_ranks * n_coarsest and the pass reduces that
// sum; coarse interface faces per patch = distinct (local coarse, remote coarse) pairs by
// first occurrence over the fine interface faces.  The two collectives are passed in:
// allgather4(in[4], out[4 * n_ranks]) and exchange(per-patch counts, send, recv) over the
// processor patches (same peers as level 0).  Level 0's if_cell / if_count are given.
struct GamgComm {
    int n_ranks = 1;
    bool (*allgather4)(void* ctx, const double* in, double* out) = nullptr;
    bool (*exchange)(void* ctx, const std::vector<int>& counts, const std::vector<double>& send,
                     std::vector<double>& recv) = nullptr;
    void* ctx = nullptr;
};
std::vector<GamgHostLevel> gamg_hierarchy_dd(int N, int F, const std::vector<int>& owner,
                                             const std::vector<int>& neighbour, const std::vector<int>& ownerStart,
                                             const std::vector<int>& losortStart, const std::vector<int>& losort,
                                             const std::vector<int>& ownerLo, const std::vector<double>& w,
                                             const std::vector<int>& if_cell, const std::vector<int>& if_count,
                                             int n_coarsest, int max_levels, const GamgComm& comm, bool* ok);
}  // namespace spuma
