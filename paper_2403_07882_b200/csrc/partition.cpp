// Mode-R domain decomposition (see partition.hpp).  Restates the reference's
// integer algorithms; every ordering rule below is the reference's.
#include "partition.hpp"

#include <algorithm>
#include <cstring>
#include <thread>

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <stdexcept>

namespace bcs {

int Decomposition::rankOfRow(int g) const {
    return static_cast<int>(std::upper_bound(rankRowOffset.begin(), rankRowOffset.end(), g) - rankRowOffset.begin()) - 1;
}

namespace {

// rcbRecurse (partition.cpp:21-53): widest axis (ties favour x, y, z by
// +1e-14), cells ordered by (coordinate, index), left share rounded
// ⌊(|cells|·nLeft + nR/2)/nR⌋ clamped to leave every rank a cell.
void rcb(std::vector<int>& cells, size_t b, size_t e, int r0, int r1, const double* cen, std::vector<int>& c2r) {
    const int nR = r1 - r0;
    if (nR == 1) {
        for (size_t i = b; i < e; ++i) c2r[cells[i]] = r0;
        return;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (size_t i = b; i < e; ++i)
        for (int a = 0; a < 3; ++a) {
            const double v = cen[3 * static_cast<size_t>(cells[i]) + a];
            lo[a] = std::min(lo[a], v);
            hi[a] = std::max(hi[a], v);
        }
    int axis = 0;
    for (int a = 1; a < 3; ++a)
        if (hi[a] - lo[a] > hi[axis] - lo[axis] + 1e-14) axis = a;
    std::sort(cells.begin() + b, cells.begin() + e, [&](int x, int y) {
        const double cx = cen[3 * static_cast<size_t>(x) + axis], cy = cen[3 * static_cast<size_t>(y) + axis];
        return cx != cy ? cx < cy : x < y;
    });
    const long long count = static_cast<long long>(e - b);
    const int nLeft = nR / 2;
    long long cl = (count * nLeft + nR / 2) / nR;
    cl = std::clamp(cl, static_cast<long long>(nLeft), count - (nR - nLeft));
    rcb(cells, b, b + cl, r0, r0 + nLeft, cen, c2r);
    rcb(cells, b + cl, e, r0 + nLeft, r1, cen, c2r);
}

struct Trip {
    int row, col, src;
};

// assembleCsr (partition.cpp:94-111): triplets sorted by (row, col)
void assemble(std::vector<Trip>& t, int nRows, Partition& p) {
    std::sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
    p.ro.assign(nRows + 1, 0);
    for (const Trip& x : t) ++p.ro[x.row + 1];
    for (int r = 0; r < nRows; ++r) p.ro[r + 1] += p.ro[r];
    p.ci.resize(t.size());
    p.src.resize(t.size());
    for (size_t k = 0; k < t.size(); ++k) {
        p.ci[k] = t[k].col;
        p.src[k] = t[k].src;
    }
}

struct Halo {
    int row, col, peer, src;
};

// finalizePartition (partition.cpp:113-119)
void finalize(std::vector<Halo>& h, Partition& p) {
    std::sort(h.begin(), h.end(), [](const Halo& a, const Halo& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
    p.haloRow.resize(h.size());
    p.haloCol.resize(h.size());
    p.haloPeer.resize(h.size());
    p.haloSrc.resize(h.size());
    for (size_t i = 0; i < h.size(); ++i) {
        p.haloRow[i] = h[i].row;
        p.haloCol[i] = h[i].col;
        p.haloPeer[i] = h[i].peer;
        p.haloSrc[i] = h[i].src;
    }
    std::sort(p.sendPlan.begin(), p.sendPlan.end());
    p.sendPlan.erase(std::unique(p.sendPlan.begin(), p.sendPlan.end()), p.sendPlan.end());
}

}  // namespace

Decomposition decompose(int nc, const double* cen, int nRanks) {
    if (nRanks < 1 || nRanks > nc) throw std::invalid_argument("decompose: need 1 <= nRanks <= nCells");
    Decomposition d;
    d.nRanks = nRanks;
    d.cellToRank.assign(nc, 0);
    std::vector<int> all(nc);
    std::iota(all.begin(), all.end(), 0);
    rcb(all, 0, all.size(), 0, nRanks, cen, d.cellToRank);
    d.rankRowOffset.assign(nRanks + 1, 0);
    for (int c = 0; c < nc; ++c) ++d.rankRowOffset[d.cellToRank[c] + 1];
    for (int r = 0; r < nRanks; ++r) d.rankRowOffset[r + 1] += d.rankRowOffset[r];
    std::vector<int> next(d.rankRowOffset.begin(), d.rankRowOffset.end() - 1);
    d.oldToNew.resize(nc);
    d.newToOld.resize(nc);
    for (int c = 0; c < nc; ++c) {
        const int g = next[d.cellToRank[c]]++;
        d.oldToNew[c] = g;
        d.newToOld[g] = c;
    }
    return d;
}

std::vector<Partition> buildPartitioned(int nc, int nf, const int32_t* owner, const int32_t* neigh,
                                        const Decomposition& dec) {
    std::vector<Partition> parts(dec.nRanks);
    std::vector<std::vector<Trip>> trip(dec.nRanks);
    std::vector<std::vector<Halo>> halo(dec.nRanks);
    for (int r = 0; r < dec.nRanks; ++r) {
        parts[r].id = r;
        parts[r].rowStart = dec.rankRowOffset[r];
        parts[r].rowEnd = dec.rankRowOffset[r + 1];
    }
    for (int c = 0; c < nc; ++c) {
        const int g = dec.oldToNew[c], r = dec.cellToRank[c];
        trip[r].push_back({g - parts[r].rowStart, g - parts[r].rowStart, c});
    }
    auto place = [&](int gRow, int gCol, int src) {
        const int r = dec.rankOfRow(gRow), rc = dec.rankOfRow(gCol);
        if (r == rc) {
            trip[r].push_back({gRow - parts[r].rowStart, gCol - parts[r].rowStart, src});
        } else {
            halo[r].push_back({gRow - parts[r].rowStart, gCol, rc, src});
            parts[rc].sendPlan.emplace_back(r, gCol - parts[rc].rowStart);
        }
    };
    for (int f = 0; f < nf; ++f) {
        const int go = dec.oldToNew[owner[f]], gn = dec.oldToNew[neigh[f]];
        place(go, gn, nc + f);       // upper
        place(gn, go, nc + nf + f);  // lower
    }
    for (int r = 0; r < dec.nRanks; ++r) {
        assemble(trip[r], parts[r].nLocalRows(), parts[r]);
        finalize(halo[r], parts[r]);
    }
    return parts;
}

ConsolidationPlan makeConsolidationPlan(const Decomposition& dec, int nEngines) {
    if (nEngines < 1 || nEngines > dec.nRanks)
        throw std::invalid_argument("makeConsolidationPlan: need 1 <= nEngines <= nRanks");
    ConsolidationPlan p;
    p.nEngines = nEngines;
    p.rankToEngine.resize(dec.nRanks);
    p.engineRowOffset.resize(dec.nRanks);
    std::vector<int> rows(nEngines, 0);
    for (int r = 0; r < dec.nRanks; ++r) {
        const int e = static_cast<int>((static_cast<long long>(r) * nEngines) / dec.nRanks);
        p.rankToEngine[r] = e;
        p.engineRowOffset[r] = rows[e];
        rows[e] += dec.nLocalRows(r);
    }
    return p;
}

std::vector<Partition> consolidate(const std::vector<Partition>& parts, const ConsolidationPlan& plan,
                                   const Decomposition& dec) {
    std::vector<Partition> eng(plan.nEngines);
    for (int e = 0; e < plan.nEngines; ++e) {
        eng[e].id = e;
        eng[e].rowStart = INT32_MAX;
        eng[e].rowEnd = 0;
    }
    for (int r = 0; r < dec.nRanks; ++r) {
        Partition& e = eng[plan.rankToEngine[r]];
        e.rowStart = std::min(e.rowStart, dec.rankRowOffset[r]);
        e.rowEnd = std::max(e.rowEnd, dec.rankRowOffset[r + 1]);
        e.memberRanks.push_back(r);
    }
    auto engineOfRow = [&](int g) { return plan.rankToEngine[dec.rankOfRow(g)]; };
    std::vector<std::vector<Trip>> trip(plan.nEngines);
    std::vector<std::vector<Halo>> halo(plan.nEngines);
    for (const Partition& p : parts) {
        const int e = plan.rankToEngine[p.id];
        Partition& E = eng[e];
        const int shift = p.rowStart - E.rowStart;
        for (int row = 0; row + 1 < static_cast<int>(p.ro.size()); ++row)
            for (int k = p.ro[row]; k < p.ro[row + 1]; ++k) trip[e].push_back({row + shift, p.ci[k] + shift, p.src[k]});
        for (size_t h = 0; h < p.haloRow.size(); ++h) {
            const int ec = engineOfRow(p.haloCol[h]);
            if (ec == e) {
                trip[e].push_back({p.haloRow[h] + shift, p.haloCol[h] - E.rowStart, p.haloSrc[h]});
            } else {
                halo[e].push_back({p.haloRow[h] + shift, p.haloCol[h], ec, p.haloSrc[h]});
                eng[ec].sendPlan.emplace_back(e, p.haloCol[h] - eng[ec].rowStart);
            }
        }
    }
    for (int e = 0; e < plan.nEngines; ++e) {
        assemble(trip[e], eng[e].nLocalRows(), eng[e]);
        finalize(halo[e], eng[e]);
    }
    return eng;
}

ExchangePlan makeExchangePlan(const std::vector<Partition>& engines, int me) {
    const int G = static_cast<int>(engines.size());
    if (me < 0 || me >= G) throw std::invalid_argument("makeExchangePlan: engine out of range");
    ExchangePlan x;
    x.sendCount.assign(G, 0);
    x.recvCount.assign(G, 0);
    for (const auto& [peer, row] : engines[me].sendPlan) {  // sorted (peer, row)
        x.sendRows.push_back(row);
        ++x.sendCount[peer];
    }
    std::vector<std::pair<int, int>> where;  // (global row, recv index)
    for (int q = 0; q < G; ++q) {
        if (q == me) continue;
        for (const auto& [peer, row] : engines[q].sendPlan)
            if (peer == me) {
                const int g = engines[q].rowStart + row;
                where.emplace_back(g, static_cast<int>(x.recvGlobalRow.size()));
                x.recvGlobalRow.push_back(g);
                ++x.recvCount[q];
            }
    }
    std::sort(where.begin(), where.end());
    const Partition& p = engines[me];
    x.haloRecvIdx.resize(p.haloCol.size());
    for (size_t h = 0; h < p.haloCol.size(); ++h) {
        const auto it = std::lower_bound(where.begin(), where.end(), std::make_pair(p.haloCol[h], -1));
        if (it == where.end() || it->first != p.haloCol[h])
            throw std::logic_error("makeExchangePlan: halo column without a sender");
        x.haloRecvIdx[h] = it->second;
    }
    return x;
}

namespace {
void gatherBlocks(const std::vector<int>& src, int nCells, int nFaces, size_t nn, const double* diag,
                  const double* upper, const double* lower, double* out, int threads) {
    const size_t cnt = src.size();
    if (!cnt) return;
    auto work = [&](size_t b, size_t e) {
        for (size_t k = b; k < e; ++k) {
            const int id = src[k];
            const double* from = id < nCells ? diag + static_cast<size_t>(id) * nn
                                 : id < nCells + nFaces ? upper + static_cast<size_t>(id - nCells) * nn
                                                        : lower + static_cast<size_t>(id - nCells - nFaces) * nn;
            std::memcpy(out + k * nn, from, nn * sizeof(double));
        }
    };
    const int T = std::max(1, std::min<int>(threads, static_cast<int>(cnt / 4096 + 1)));
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(work, cnt * t / T, cnt * (t + 1) / T);
    work(0, cnt / T);
    for (auto& th : pool) th.join();
}
}  // namespace

void gatherPartValues(const Partition& p, int nCells, int nFaces, int n, const double* diag, const double* upper,
                      const double* lower, double* localVals, double* haloVals, int threads) {
    const size_t nn = static_cast<size_t>(n) * n;
    if (localVals) gatherBlocks(p.src, nCells, nFaces, nn, diag, upper, lower, localVals, threads);
    if (haloVals) gatherBlocks(p.haloSrc, nCells, nFaces, nn, diag, upper, lower, haloVals, threads);
}

}  // namespace bcs
