// Domain decomposition for Mode R (the reference's distributed semantics,
// proj/core/src/partition.cpp): RCB on centroids with rank-major renumbering,
// per-rank local BSR + halo couplings + send plans, consolidation of ranks
// onto engines.  Integer work, bit-exact with the reference (pinned by
// tests/test_partition.py).  Values are not copied here: every local slot and
// halo entry carries the id of its LDU source block (c, nc+f, nc+nf+f) so a
// value replace is a device gather.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

namespace bcs {

struct Decomposition {
    int nRanks = 0;
    std::vector<int> cellToRank;     // by original cell
    std::vector<int> rankRowOffset;  // nRanks + 1
    std::vector<int> oldToNew, newToOld;
    int rankOfRow(int globalRow) const;
    int nLocalRows(int r) const { return rankRowOffset[r + 1] - rankRowOffset[r]; }
};

// partition.cpp:21-85
Decomposition decompose(int nCells, const double* centroids, int nRanks);

struct Partition {
    int id = 0;
    int rowStart = 0, rowEnd = 0;                 // owned global rows (new numbering)
    std::vector<int> ro, ci, src;                 // local BSR (local numbering) + LDU source ids
    std::vector<int> haloRow, haloCol, haloPeer;  // sorted by (localRow, globalCol)
    std::vector<int> haloSrc;
    std::vector<std::pair<int, int>> sendPlan;    // (peer, localRow), sorted unique
    std::vector<int> memberRanks;                 // engines only
    int nLocalRows() const { return rowEnd - rowStart; }
};

// partition.cpp:123-165 (values by source id)
std::vector<Partition> buildPartitioned(int nCells, int nFaces, const int32_t* owner, const int32_t* neigh,
                                        const Decomposition& dec);

struct ConsolidationPlan {
    int nEngines = 0;
    std::vector<int> rankToEngine, engineRowOffset;
};
// partition.cpp:184-199
ConsolidationPlan makeConsolidationPlan(const Decomposition& dec, int nEngines);
// partition.cpp:201-248
std::vector<Partition> consolidate(const std::vector<Partition>& parts, const ConsolidationPlan& plan,
                                   const Decomposition& dec);

// Multi-process Mode R: what engine `me` sends to and receives from every
// peer per halo exchange, and where each of its halo entries finds its value.
// Send: the engine's sendPlan grouped by peer (peers ascending, local rows
// ascending) -> sendRows, sendCount[peer].  Receive: every other engine's
// sendPlan entries addressed to `me`, in that engine's order -> recvGlobalRow
// (renumbered global rows), recvCount[peer]; peers ascending.  haloRecvIdx[h]
// = position of haloCol[h] in the concatenated receive buffer.
struct ExchangePlan {
    std::vector<int> sendRows, sendCount, recvGlobalRow, recvCount, haloRecvIdx;
};
ExchangePlan makeExchangePlan(const std::vector<Partition>& engines, int me);

// The reference's per-rank "upload" (partition.cpp:384-407, the paper's
// per-partition NExternalNZ arrays) on the host: the LDU
// blocks of one engine's local slots (slot order) and halo entries (entry
// order), n*n doubles each, gathered from the caller's face-addressed arrays
// by `threads` host threads over contiguous slot ranges.  Only these bytes
// cross PCIe to that engine's GPU (about 1/G of the system).
void gatherPartValues(const Partition& p, int nCells, int nFaces, int n, const double* diag, const double* upper,
                      const double* lower, double* localVals, double* haloVals, int threads);

}  // namespace bcs
