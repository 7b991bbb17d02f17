// gamg_host.cpp -- host construction of the GAMG level hierarchy.
//
// faceAreaPair agglomeration (reading Q22; PAPER.md P:665 keeps the
// original coarsening) and the coarse lduAddressing of each level (Q27).  Run once per
// (mesh, n_coarsest, max_levels); the per-solve Galerkin products run on the device
// (gamg.cu) over the lists built here.
#include <algorithm>
#include <map>
#include <numeric>

#include "host.h"

namespace spuma {
namespace {

// Pairwise pass (Q22).  Cell c's faces in ascending face index are its neighbour-side
// faces (losort range, owners < c: always already agglomerated when c is visited) and
// then its owner-side faces, so a FREE partner can only be across an owner-side face.
int pair_cells(int n, const int* ownerStart, const int* neighbour, const int* losortStart, const int* losort,
               const int* ownerLo, const double* w, std::vector<int>& ftc)
{
    ftc.assign(n, -1);
    int nc = 0;
    for (int c = 0; c < n; ++c) {
        if (ftc[c] >= 0) continue;
        int partner = -1;
        double best = -1.0;
        for (int f = ownerStart[c]; f < ownerStart[c + 1]; ++f) {
            const int o = neighbour[f];
            if (ftc[o] < 0 && w[f] > best) best = w[f], partner = o;
        }
        if (partner >= 0) {
            ftc[c] = ftc[partner] = nc++;
            continue;
        }
        best = -1.0;  // every neighbour is taken: join the strongest neighbouring agglomerate
        for (int k = losortStart[c]; k < losortStart[c + 1]; ++k)
            if (w[losort[k]] > best) best = w[losort[k]], partner = ownerLo[k];
        for (int f = ownerStart[c]; f < ownerStart[c + 1]; ++f)
            if (w[f] > best) best = w[f], partner = neighbour[f];
        ftc[c] = partner >= 0 ? ftc[partner] : nc++;
    }
    return nc;
}

// The coarse level of L given its agglomeration (Q22, Q27): distinct (lo, hi) agglomerate
// pairs bucketed by lo and sorted by hi, face weights summed in ascending fine order, and the
// device lists of the Galerkin product and the restriction.  L.ftc takes ftc.
GamgHostLevel coarsen(GamgHostLevel& L, const std::vector<int>& Lo, const std::vector<int>& Ln, std::vector<int>& ftc,
                      int nc)
{
    std::vector<int> bstart(nc + 1, 0);
    for (int f = 0; f < L.F; ++f) {
        const int a = ftc[Lo[f]], b = ftc[Ln[f]];
        if (a != b) bstart[std::min(a, b) + 1]++;
    }
    for (int c = 0; c < nc; ++c) bstart[c + 1] += bstart[c];
    std::vector<int> his(bstart[nc]), fill(bstart.begin(), bstart.end() - 1);
    for (int f = 0; f < L.F; ++f) {
        const int a = ftc[Lo[f]], b = ftc[Ln[f]];
        if (a != b) his[fill[std::min(a, b)]++] = std::max(a, b);
    }
    GamgHostLevel C;
    C.n = nc;
    std::vector<int> ustart(nc + 1, 0);  // per lo: start of its distinct coarse faces
    for (int lo = 0; lo < nc; ++lo) {
        auto b0 = his.begin() + bstart[lo], b1 = his.begin() + bstart[lo + 1];
        std::sort(b0, b1);
        auto e = std::unique(b0, b1);
        ustart[lo] = (int)C.owner.size();
        for (auto it = b0; it != e; ++it) {
            C.owner.push_back(lo);
            C.neighbour.push_back(*it);
        }
    }
    ustart[nc] = (int)C.owner.size();
    C.F = (int)C.owner.size();
    L.frestrict.assign(L.F, -1);
    C.w.assign(C.F, 0.0);
    for (int f = 0; f < L.F; ++f) {  // ascending fine face: coarse weights summed in this order
        const int a = ftc[Lo[f]], b = ftc[Ln[f]];
        if (a == b) continue;
        const int lo = std::min(a, b), hi = std::max(a, b);
        const int cf = (int)(std::lower_bound(C.neighbour.begin() + ustart[lo], C.neighbour.begin() + ustart[lo + 1], hi) -
                             C.neighbour.begin());
        L.frestrict[f] = cf;
        C.w[cf] += L.w[f];
    }
    // the device-side lists of the Galerkin product and the restriction
    std::vector<char> all(L.n, 1), inside(L.F), across(L.F);
    std::vector<int> inner_of(L.F), cface_of(L.F);
    for (int f = 0; f < L.F; ++f) {
        inside[f] = L.frestrict[f] < 0;
        across[f] = !inside[f];
        inner_of[f] = ftc[Lo[f]];
        cface_of[f] = inside[f] ? 0 : L.frestrict[f];
    }
    cell_lists(nc, ftc, all, L.cStart, L.cList);
    cell_lists(nc, inner_of, inside, L.ciStart, L.ciList);
    cell_lists(C.F, cface_of, across, L.cfStart, L.cfList);
    L.ftc = std::move(ftc);
    derived_addressing(C.n, C.F, C.owner.data(), C.neighbour.data(), C.ownerStart, C.losort, C.losortStart,
                       C.ownerLo);
    return C;
}

struct LevelRef {
    const std::vector<int>&o, &nb, &os, &ls, &l, &lo;
};

}  // namespace

std::vector<GamgHostLevel> gamg_hierarchy(int N, int F, const std::vector<int>& owner,
                                          const std::vector<int>& neighbour, const std::vector<int>& ownerStart,
                                          const std::vector<int>& losortStart, const std::vector<int>& losort,
                                          const std::vector<int>& ownerLo, const std::vector<double>& w,
                                          int n_coarsest, int max_levels)
{
    std::vector<GamgHostLevel> lv(1);
    lv[0].n = N;
    lv[0].F = F;
    lv[0].w = w;
    while ((int)lv.size() < max_levels && lv.back().n > n_coarsest) {
        GamgHostLevel& L = lv.back();
        const bool fine = lv.size() == 1;
        const LevelRef r{fine ? owner : L.owner, fine ? neighbour : L.neighbour, fine ? ownerStart : L.ownerStart,
                         fine ? losortStart : L.losortStart, fine ? losort : L.losort, fine ? ownerLo : L.ownerLo};
        std::vector<int> ftc;
        const int nc = pair_cells(L.n, r.os.data(), r.nb.data(), r.ls.data(), r.l.data(), r.lo.data(), L.w.data(), ftc);
        if (nc >= L.n) break;
        GamgHostLevel C = coarsen(L, r.o, r.nb, ftc, nc);
        lv.push_back(std::move(C));
    }
    return lv;
}

std::vector<GamgHostLevel> gamg_hierarchy_dd(int N, int F, const std::vector<int>& owner,
                                             const std::vector<int>& neighbour, const std::vector<int>& ownerStart,
                                             const std::vector<int>& losortStart, const std::vector<int>& losort,
                                             const std::vector<int>& ownerLo, const std::vector<double>& w,
                                             const std::vector<int>& if_cell, const std::vector<int>& if_count,
                                             int n_coarsest, int max_levels, const GamgComm& comm, bool* ok)
{
    *ok = true;
    const int P = comm.n_ranks;
    std::vector<GamgHostLevel> lv(1);
    lv[0].n = N;
    lv[0].F = F;
    lv[0].w = w;
    lv[0].if_cell = if_cell;
    lv[0].if_count = if_count;
    std::vector<double> g(4 * (size_t)P);
    for (;;) {
        GamgHostLevel& L = lv.back();
        const bool fine = lv.size() == 1;
        const LevelRef r{fine ? owner : L.owner, fine ? neighbour : L.neighbour, fine ? ownerStart : L.ownerStart,
                         fine ? losortStart : L.losortStart, fine ? losort : L.losort, fine ? ownerLo : L.ownerLo};
        std::vector<int> ftc;
        const int nc = pair_cells(L.n, r.os.data(), r.nb.data(), r.ls.data(), r.l.data(), r.lo.data(), L.w.data(), ftc);
        const double in[4] = {(double)L.n, (double)nc, 0.0, 0.0};
        if (!comm.allgather4(comm.ctx, in, g.data())) {
            *ok = false;
            return lv;
        }
        double nfine = 0.0, ncoarse = 0.0;  // integers < 2^53: exact
        for (int q = 0; q < P; ++q) nfine += g[4 * q], ncoarse += g[4 * q + 1];
        if (!((int)lv.size() < max_levels && nfine > (double)P * n_coarsest)) break;  // Q36
        if (ncoarse >= nfine) break;
        // the neighbours' coarse cells of this level's interface faces (Q37)
        const int m = (int)L.if_cell.size();
        std::vector<double> send(m), recv(m);
        for (int i = 0; i < m; ++i) send[i] = (double)ftc[L.if_cell[i]];
        if (!comm.exchange(comm.ctx, L.if_count, send, recv)) {
            *ok = false;
            return lv;
        }
        GamgHostLevel C = coarsen(L, r.o, r.nb, ftc, nc);
        std::vector<int> ifr(m);
        C.if_count.assign(L.if_count.size(), 0);
        int off = 0;
        for (size_t p = 0; p < L.if_count.size(); ++p) {
            std::map<std::pair<int, int>, int> seen;  // (local, remote) -> coarse face, first occurrence
            for (int i = off; i < off + L.if_count[p]; ++i) {
                const std::pair<int, int> key(L.ftc[L.if_cell[i]], (int)recv[i]);
                auto it = seen.find(key);
                if (it == seen.end()) {
                    it = seen.emplace(key, (int)C.if_cell.size()).first;
                    C.if_cell.push_back(key.first);
                    C.if_count[p]++;
                }
                ifr[i] = it->second;
            }
            off += L.if_count[p];
        }
        std::vector<char> all_if(m, 1);
        cell_lists((int)C.if_cell.size(), ifr, all_if, L.cifStart, L.cifList);
        lv.push_back(std::move(C));
    }
    for (GamgHostLevel& L : lv) {  // per-cell interface lists (Q10: (patch, face) order)
        std::vector<char> all_if(L.if_cell.size(), 1);
        cell_lists(L.n, L.if_cell, all_if, L.ifStart, L.ifIdx);
    }
    return lv;
}

}  // namespace spuma
