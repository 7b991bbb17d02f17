// gamg_host.cpp -- host construction of the GAMG level hierarchy.
//
// faceAreaPair agglomeration (reading Q22; PAPER.md P:665 keeps the
// original coarsening) and the coarse lduAddressing of each level (Q27).  Run once per
// (mesh, n_coarsest, max_levels); the per-solve Galerkin products run on the device
// (gamg.cu) over the lists built here.
#include <algorithm>
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
        const std::vector<int>& Lo = fine ? owner : L.owner;
        const std::vector<int>& Ln = fine ? neighbour : L.neighbour;
        const std::vector<int>& Los = fine ? ownerStart : L.ownerStart;
        const std::vector<int>& Lls = fine ? losortStart : L.losortStart;
        const std::vector<int>& Ll = fine ? losort : L.losort;
        const std::vector<int>& Llo = fine ? ownerLo : L.ownerLo;
        std::vector<int> ftc;
        const int nc = pair_cells(L.n, Los.data(), Ln.data(), Lls.data(), Ll.data(), Llo.data(), L.w.data(), ftc);
        if (nc >= L.n) break;
        // coarse faces: distinct (lo, hi) agglomerate pairs, bucketed by lo, sorted by hi
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
        lv.push_back(std::move(C));
    }
    return lv;
}

}  // namespace spuma
