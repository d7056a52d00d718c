// Link-time interposition of fvb::SolvePipeline::solve (TEST INFRASTRUCTURE
// and the zero-source-change integration recipe of INTEGRATION.md).
//
// Linked with -Wl,--wrap=<mangled fvb::SolvePipeline::solve> next to the
// reference's objects, every call another reference object makes to
// SolvePipeline::solve (engine.cpp:47-120) -- LinearDispatch's serial branch
// in runCase (case_runner.cpp:333) above all -- lands here and runs on the
// B200 pipeline (include/bcs.hpp); one bcs::SolvePipeline per reference
// pipeline object keeps its setup-vs-replace state.  fvb::backendSolve (the
// one-shot wrapper, engine.cpp:123-129) is interposed the same way on one
// shared pipeline, and fvb::distributedSolve (partition.cpp:370-479,
// LinearDispatch's multi-rank branch) runs the one-device Mode R on the
// caller's partitions (bcs_dist_solve_parts).
//   bcs_interpose_route: -1 the reference's own solve (__real_), else the
//   BCS_MODE_* of the B200 solve; initialised from $BCS_INTERPOSE
//   (off | parity | exact; default parity).
#include "blockfv/engine.hpp"
#include "blockfv/partition.hpp"

#include "../../include/bcs.hpp"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>

using SolveResult = std::pair<fvb::BlockVector, fvb::SolveReport>;

extern "C" SolveResult
__real__ZN3fvb13SolvePipeline5solveERKNS_14BlockLduMatrixERKNS_11BlockVectorES6_NS_7BackendERKNS_12SolverConfigE(
    fvb::SolvePipeline* self, const fvb::BlockLduMatrix& A, const fvb::BlockVector& b, const fvb::BlockVector& x0,
    fvb::Backend backend, const fvb::SolverConfig& cfg);

static int route_from_env() {
    const char* e = std::getenv("BCS_INTERPOSE");
    if (!e || !std::strcmp(e, "parity")) return BCS_MODE_PARITY;
    if (!std::strcmp(e, "exact")) return BCS_MODE_EXACT;
    if (!std::strcmp(e, "off")) return -1;
    return BCS_MODE_PARITY;
}

extern "C" {
int bcs_interpose_route = route_from_env();
long bcs_interpose_calls = 0;  // solves that ran on the B200
}

// the count goes to stderr at exit, so a caller can tell the B200 really ran
static struct ReportAtExit {
    ~ReportAtExit() { std::fprintf(stderr, "bcs interpose: %ld solves on the B200\n", bcs_interpose_calls); }
} g_report_at_exit;

extern "C" SolveResult
__wrap__ZN3fvb13SolvePipeline5solveERKNS_14BlockLduMatrixERKNS_11BlockVectorES6_NS_7BackendERKNS_12SolverConfigE(
    fvb::SolvePipeline* self, const fvb::BlockLduMatrix& A, const fvb::BlockVector& b, const fvb::BlockVector& x0,
    fvb::Backend backend, const fvb::SolverConfig& cfg) {
    if (bcs_interpose_route < 0)
        return __real__ZN3fvb13SolvePipeline5solveERKNS_14BlockLduMatrixERKNS_11BlockVectorES6_NS_7BackendERKNS_12SolverConfigE(
            self, A, b, x0, backend, cfg);
    static std::map<const fvb::SolvePipeline*, std::unique_ptr<bcs::SolvePipeline>> pipes;
    auto& p = pipes[self];
    if (!p) p = std::make_unique<bcs::SolvePipeline>(0);
    p->setMode(bcs_interpose_route);
    ++bcs_interpose_calls;
    return p->solve<fvb::SolveReport>(A, b, x0, backend, cfg);
}

extern "C" SolveResult
__real__ZN3fvb12backendSolveERKNS_14BlockLduMatrixERKNS_11BlockVectorES5_NS_7BackendERKNS_12SolverConfigE(
    const fvb::BlockLduMatrix& A, const fvb::BlockVector& b, const fvb::BlockVector& x0, fvb::Backend backend,
    const fvb::SolverConfig& cfg);

extern "C" SolveResult
__wrap__ZN3fvb12backendSolveERKNS_14BlockLduMatrixERKNS_11BlockVectorES5_NS_7BackendERKNS_12SolverConfigE(
    const fvb::BlockLduMatrix& A, const fvb::BlockVector& b, const fvb::BlockVector& x0, fvb::Backend backend,
    const fvb::SolverConfig& cfg) {
    if (bcs_interpose_route < 0)
        return __real__ZN3fvb12backendSolveERKNS_14BlockLduMatrixERKNS_11BlockVectorES5_NS_7BackendERKNS_12SolverConfigE(
            A, b, x0, backend, cfg);
    // one context for every one-shot call: the results do not depend on the
    // setup-vs-replace branch (bit-identical either way), and a context per
    // call would cost more than a small solve
    static std::unique_ptr<bcs::SolvePipeline> p;
    if (!p) p = std::make_unique<bcs::SolvePipeline>(0);
    p->setMode(bcs_interpose_route);
    ++bcs_interpose_calls;
    return p->solve<fvb::SolveReport>(A, b, x0, backend, cfg);
}

using DistResult = std::pair<fvb::DistributedVector, fvb::SolveReport>;
#define BCS_DIST_SOLVE                                                                                              \
    _ZN3fvb16distributedSolveERKSt6vectorINS_15MatrixPartitionESaIS1_EERKS0_IS0_IdSaIdEESaIS7_EESB_RKNS_12SolverConfigERKNS_17ConsolidationPlanERKNS_13DecompositionERNS_14MailboxNetworkE
#define BCS_CAT2(a, b) a##b
#define BCS_CAT(a, b) BCS_CAT2(a, b)

extern "C" DistResult BCS_CAT(__real_, BCS_DIST_SOLVE)(const std::vector<fvb::MatrixPartition>& parts,
                                                       const fvb::DistributedVector& b, const fvb::DistributedVector& x0,
                                                       const fvb::SolverConfig& cfg, const fvb::ConsolidationPlan& plan,
                                                       const fvb::Decomposition& dec, fvb::MailboxNetwork& net);

extern "C" DistResult BCS_CAT(__wrap_, BCS_DIST_SOLVE)(const std::vector<fvb::MatrixPartition>& parts,
                                                       const fvb::DistributedVector& b, const fvb::DistributedVector& x0,
                                                       const fvb::SolverConfig& cfg, const fvb::ConsolidationPlan& plan,
                                                       const fvb::Decomposition& dec, fvb::MailboxNetwork& net) {
    if (bcs_interpose_route < 0) return BCS_CAT(__real_, BCS_DIST_SOLVE)(parts, b, x0, cfg, plan, dec, net);
    static std::unique_ptr<bcs::SolvePipeline> p;
    if (!p) p = std::make_unique<bcs::SolvePipeline>(0);
    p->setMode(bcs_interpose_route);
    ++bcs_interpose_calls;
    return p->distributedSolve<fvb::SolveReport>(parts, b, x0, cfg, plan, dec);
}
