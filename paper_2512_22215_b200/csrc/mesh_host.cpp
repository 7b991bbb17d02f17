// mesh_host.cpp -- host-side mesh logic of libspuma: addressing validation (A0),
// reverse Cuthill-McKee renumbering (A1), face re-keying, and the derived
// addressing ownerStart / losort / losortStart (A2).  Runs once per mesh.
//
// A1's rule (the paper is silent, BASELINE.json asks for "renumbered cells";
// reading Q12): start at the unvisited cell of minimum degree
// (ties: smallest index), FIFO BFS, a dequeued cell enqueues its unvisited
// neighbours sorted by (degree, index), restart per component, reverse.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "host.h"

namespace spuma {

bool valid_addressing(int N, int F, const int* owner, const int* neighbour, std::string* why)
{
    for (int f = 0; f < F; ++f) {
        const int o = owner[f], n = neighbour[f];
        if (o < 0 || o >= N || n < 0 || n >= N) {
            *why = "face " + std::to_string(f) + ": cell index out of range";
            return false;
        }
        if (o >= n) {
            *why = "face " + std::to_string(f) + ": owner >= neighbour";
            return false;
        }
        if (f && (o < owner[f - 1] || (o == owner[f - 1] && n < neighbour[f - 1]))) {
            *why = "face " + std::to_string(f) + ": faces not sorted by (owner, neighbour)";
            return false;
        }
    }
    return true;
}

std::vector<int> rcm_permutation(int N, int F, const int* owner, const int* neighbour)
{
    std::vector<int> deg(N, 0), start(N + 1, 0), adj(2 * (size_t)F);
    for (int f = 0; f < F; ++f) {
        ++deg[owner[f]];
        ++deg[neighbour[f]];
    }
    for (int c = 0; c < N; ++c) start[c + 1] = start[c] + deg[c];
    {
        std::vector<int> pos(start.begin(), start.end() - 1);
        for (int f = 0; f < F; ++f) {
            adj[pos[owner[f]]++] = neighbour[f];
            adj[pos[neighbour[f]]++] = owner[f];
        }
    }
    auto less = [&](int a, int b) { return deg[a] != deg[b] ? deg[a] < deg[b] : a < b; };
    std::vector<int> by_degree(N);
    std::iota(by_degree.begin(), by_degree.end(), 0);
    std::sort(by_degree.begin(), by_degree.end(), less);

    std::vector<char> seen(N, 0);
    std::vector<int> order;
    order.reserve(N);
    std::vector<int> cand;
    size_t next_start = 0;
    while ((int)order.size() < N) {
        while (seen[by_degree[next_start]]) ++next_start;
        const int s = by_degree[next_start];
        seen[s] = 1;
        size_t head = order.size();
        order.push_back(s);
        while (head < order.size()) {
            const int c = order[head++];
            cand.clear();
            for (int e = start[c]; e < start[c + 1]; ++e) {
                const int d = adj[e];
                if (!seen[d]) {
                    seen[d] = 1;
                    cand.push_back(d);
                }
            }
            std::sort(cand.begin(), cand.end(), less);
            order.insert(order.end(), cand.begin(), cand.end());
        }
    }
    std::vector<int> perm(N);
    for (int k = 0; k < N; ++k) perm[order[k]] = N - 1 - k;
    return perm;
}

void rekey_faces(int N, int F, const int* perm, const int* owner, const int* neighbour, std::vector<int>& owner_out,
                 std::vector<int>& neighbour_out, std::vector<int>& face_map, std::vector<char>& flip)
{
    std::vector<int> lo(F), hi(F), tmp(F);
    for (int f = 0; f < F; ++f) {
        const int a = perm[owner[f]], b = perm[neighbour[f]];
        lo[f] = std::min(a, b);
        hi[f] = std::max(a, b);
    }
    // stable by (lo, hi, old face): LSD counting sort, hi then lo
    std::vector<int64_t> cnt(N + 1);
    std::fill(cnt.begin(), cnt.end(), 0);
    for (int f = 0; f < F; ++f) ++cnt[hi[f] + 1];
    for (int c = 0; c < N; ++c) cnt[c + 1] += cnt[c];
    for (int f = 0; f < F; ++f) tmp[cnt[hi[f]]++] = f;
    std::fill(cnt.begin(), cnt.end(), 0);
    for (int f = 0; f < F; ++f) ++cnt[lo[f] + 1];
    for (int c = 0; c < N; ++c) cnt[c + 1] += cnt[c];
    face_map.assign(F, 0);
    for (int t = 0; t < F; ++t) {
        const int f = tmp[t];
        face_map[cnt[lo[f]]++] = f;
    }
    owner_out.resize(F);
    neighbour_out.resize(F);
    flip.resize(F);
    for (int g = 0; g < F; ++g) {
        const int f = face_map[g];
        owner_out[g] = lo[f];
        neighbour_out[g] = hi[f];
        flip[g] = perm[owner[f]] > perm[neighbour[f]];
    }
}

void derived_addressing(int N, int F, const int* owner, const int* neighbour, std::vector<int>& ownerStart,
                        std::vector<int>& losort, std::vector<int>& losortStart, std::vector<int>& ownerLo)
{
    ownerStart.assign(N + 1, 0);
    for (int f = 0; f < F; ++f) ++ownerStart[owner[f] + 1];
    for (int c = 0; c < N; ++c) ownerStart[c + 1] += ownerStart[c];
    losortStart.assign(N + 1, 0);
    for (int f = 0; f < F; ++f) ++losortStart[neighbour[f] + 1];
    for (int c = 0; c < N; ++c) losortStart[c + 1] += losortStart[c];
    losort.assign(F, 0);
    ownerLo.assign(F, 0);
    std::vector<int> pos(losortStart.begin(), losortStart.end() - 1);
    for (int f = 0; f < F; ++f) losort[pos[neighbour[f]]++] = f;  // stable: ascending face index
    for (int k = 0; k < F; ++k) ownerLo[k] = owner[losort[k]];
}

void cell_lists(int N, const std::vector<int>& cell_of, const std::vector<char>& keep, std::vector<int>& start,
                std::vector<int>& items)
{
    start.assign(N + 1, 0);
    const int n = (int)cell_of.size();
    for (int i = 0; i < n; ++i)
        if (keep[i]) ++start[cell_of[i] + 1];
    for (int c = 0; c < N; ++c) start[c + 1] += start[c];
    items.assign(start[N], 0);
    std::vector<int> pos(start.begin(), start.end() - 1);
    for (int i = 0; i < n; ++i)
        if (keep[i]) items[pos[cell_of[i]]++] = i;  // stable: input order
}

SellHost build_sell(int N, const std::vector<int>& ownerStart, const std::vector<int>& losortStart,
                    const std::vector<int>& losort, const std::vector<int>& ownerLo,
                    const std::vector<int>& neighbour)
{
    SellHost S;
    const int chunks = (N + 31) / 32;
    S.meta.assign(4 * (size_t)chunks, 0);
    std::vector<int> cwn(chunks), cwo(chunks);
    size_t sell_slots = 0;
    int gwn = 0, gwo = 0;
    for (int k = 0; k < chunks; ++k) {
        int wn = 0, wo = 0;
        for (int c = 32 * k; c < std::min(N, 32 * k + 32); ++c) {
            wn = std::max(wn, losortStart[c + 1] - losortStart[c]);
            wo = std::max(wo, ownerStart[c + 1] - ownerStart[c]);
        }
        cwn[k] = wn;
        cwo[k] = wo;
        gwn = std::max(gwn, wn);
        gwo = std::max(gwo, wo);
        sell_slots += 32 * (size_t)(wn + wo);
    }
    // ELL-like uniform widths when they pad by <= 10 %: slot bases become arithmetic
    const bool uniform = 32 * (size_t)chunks * (gwn + gwo) * 10 <= sell_slots * 11;
    if (uniform) {
        S.uniform_wn = gwn;
        S.uniform_wo = gwo;
    }
    size_t nb = 0, ob = 0;
    for (int k = 0; k < chunks; ++k) {
        const int wn = uniform ? gwn : cwn[k], wo = uniform ? gwo : cwo[k];
        S.meta[4 * k + 0] = (int)std::min(nb, (size_t)INT32_MAX);
        S.meta[4 * k + 1] = (int)std::min(ob, (size_t)INT32_MAX);
        S.meta[4 * k + 2] = wn;
        S.meta[4 * k + 3] = wo;
        nb += 32 * (size_t)wn;
        ob += 32 * (size_t)wo;
    }
    if (nb >= (1ull << 31) || ob >= (1ull << 31)) return S;
    S.nslot.assign(nb, 0xFFFFFFFFu);
    S.oslot.assign(ob, -1);
    for (int c = 0; c < N; ++c) {
        const int k = c >> 5, l = c & 31;
        const int nbase = S.meta[4 * k], obase = S.meta[4 * k + 1];
        for (int q = losortStart[c], j = 0; q < losortStart[c + 1]; ++q, ++j) {
            const int o = ownerLo[q];
            const int pos = losort[q] - ownerStart[o];
            if (o >= (1 << 27) - 1 || pos >= 31) return S;
            S.nslot[nbase + 32 * (size_t)j + l] = ((unsigned)o << 5) | (unsigned)pos;
        }
        for (int f = ownerStart[c], j = 0; f < ownerStart[c + 1]; ++f, ++j)
            S.oslot[obase + 32 * (size_t)j + l] = neighbour[f];
    }
    S.ok = true;
    return S;
}

EllStencil build_ell_stencil(int N, const std::vector<int>& ownerStart, const std::vector<int>& losortStart,
                             const std::vector<int>& losort, const std::vector<int>& ownerLo,
                             const std::vector<int>& neighbour)
{
    EllStencil E;
    const int chunks = (N + 31) / 32;
    E.meta.assign(8 * (size_t)chunks, 0);
    E.lane.assign((size_t)N, 0u);
    for (int k = 0; k < chunks; ++k) {
        const int c0 = 32 * k, c1 = std::min(N, c0 + 32);
        std::vector<long long> dn, dO;
        bool ok = true;
        for (int c = c0; c < c1 && ok; ++c) {
            for (int q = losortStart[c]; q < losortStart[c + 1]; ++q) {
                dn.push_back((long long)ownerLo[q] - c);
                if (losort[q] - ownerStart[ownerLo[q]] >= 32) ok = false;
            }
            for (int f = ownerStart[c]; f < ownerStart[c + 1]; ++f) dO.push_back((long long)neighbour[f] - c);
        }
        std::sort(dn.begin(), dn.end());
        dn.erase(std::unique(dn.begin(), dn.end()), dn.end());
        std::sort(dO.begin(), dO.end());
        dO.erase(std::unique(dO.begin(), dO.end()), dO.end());
        if (!ok || dn.size() > 3 || dO.size() > 3) continue;
        for (size_t t = 0; t < dn.size(); ++t) E.meta[8 * k + 1 + t] = (int)dn[t];
        for (size_t t = 0; t < dO.size(); ++t) E.meta[8 * k + 4 + t] = (int)dO[t];
        for (int c = c0; c < c1; ++c) {
            unsigned w = 0;
            for (int q = losortStart[c]; q < losortStart[c + 1]; ++q) {
                const long long d = (long long)ownerLo[q] - c;
                const int t = (int)(std::lower_bound(dn.begin(), dn.end(), d) - dn.begin());
                w |= 1u << t;
                w |= (unsigned)(losort[q] - ownerStart[ownerLo[q]]) << (6 + 5 * t);
            }
            for (int f = ownerStart[c]; f < ownerStart[c + 1]; ++f) {
                const long long d = (long long)neighbour[f] - c;
                const int t = (int)(std::lower_bound(dO.begin(), dO.end(), d) - dO.begin());
                w |= 1u << (3 + t);
            }
            E.lane[c] = w;
        }
        E.meta[8 * k] = 1;
        E.compressed++;
    }
    return E;
}

void level_schedule(int N, const std::vector<int>& owner, const std::vector<int>& neighbour,
                    const std::vector<int>& ownerStart, const std::vector<int>& losortStart,
                    const std::vector<int>& losort, std::vector<int>& order_f, std::vector<int>& order_b,
                    int& depth_f, int& depth_b, int& width_f, int& width_b)
{
    std::vector<int> lf(N, 0), lb(N, 0);
    for (int c = 0; c < N; ++c)
        for (int k = losortStart[c]; k < losortStart[c + 1]; ++k) lf[c] = std::max(lf[c], lf[owner[losort[k]]] + 1);
    for (int c = N - 1; c >= 0; --c)
        for (int f = ownerStart[c]; f < ownerStart[c + 1]; ++f) lb[c] = std::max(lb[c], lb[neighbour[f]] + 1);
    auto order_by = [N](const std::vector<int>& lev, std::vector<int>& ord, int& depth, int& width) {
        depth = 0;
        for (int c = 0; c < N; ++c) depth = std::max(depth, lev[c] + 1);
        std::vector<int> start(depth + 1, 0);
        for (int c = 0; c < N; ++c) start[lev[c] + 1]++;
        width = 0;
        for (int d = 0; d < depth; ++d) width = std::max(width, start[d + 1]);
        for (int d = 0; d < depth; ++d) start[d + 1] += start[d];
        ord.assign(N, 0);
        for (int c = 0; c < N; ++c) ord[start[lev[c]]++] = c;
    };
    order_by(lf, order_f, depth_f, width_f);
    order_by(lb, order_b, depth_b, width_b);
}

void ldu_to_csr_host(int N, int F, const std::vector<int>& owner, const std::vector<int>& neighbour,
                     const std::vector<int>& ownerStart, const std::vector<int>& losortStart,
                     const std::vector<int>& losort, std::vector<int>& row_ptr, std::vector<int>& col,
                     std::vector<int>& map)
{
    const int nnz = N + 2 * F;
    row_ptr.assign(N + 1, 0);
    col.assign(nnz, 0);
    map.assign(nnz, 0);
    int k = 0;
    for (int c = 0; c < N; ++c) {
        for (int j = losortStart[c]; j < losortStart[c + 1]; ++j) {
            const int f = losort[j];
            col[k] = owner[f];
            map[k++] = N + F + f;
        }
        col[k] = c;
        map[k++] = c;
        for (int f = ownerStart[c]; f < ownerStart[c + 1]; ++f) {
            col[k] = neighbour[f];
            map[k++] = N + f;
        }
        row_ptr[c + 1] = k;
    }
}

int lattice_offsets(int N, int F, const int* owner, const int* neighbour, int D[3])
{
    int K = 0;
    for (int f = 0; f < F; ++f) {
        const int d = neighbour[f] - owner[f];
        int t = 0;
        while (t < K && D[t] != d) ++t;
        if (t == K) {
            if (K == 3) return 0;
            D[K++] = d;
        }
    }
    std::sort(D, D + K);
    // faces are sorted by (owner, neighbour): a repeated offset within one owner is adjacent
    for (int f = 1; f < F; ++f)
        if (owner[f] == owner[f - 1] && neighbour[f] == neighbour[f - 1]) return 0;
    (void)N;
    return K;
}

}  // namespace spuma
