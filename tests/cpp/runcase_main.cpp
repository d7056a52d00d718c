// runCase drop-in check (TEST INFRASTRUCTURE).
//
// The reference's own case runner -- fvb::runCase (case_runner.cpp:389-495)
// with its LinearDispatch (case_runner.cpp:322-353) -- runs unchanged; only
// the serial branch's call into fvb::SolvePipeline::solve (case_runner.cpp:333)
// is routed to the B200 pipeline, by link-time interposition
// (-Wl,--wrap=<that symbol> + tests/cpp/pipeline_interpose.cpp, oracle/Makefile):
// no reference source is touched,
// which is exactly the one-symbol swap INTEGRATION.md describes.
//
// Checks, in the style of the reference's acceptance criterion 2
// (acceptance_main.cpp:105-134; configurations as cavityConfig(32, 200) and
// sodImplicitConfig(100, 200), acceptance_main.cpp:76-101), 200 nonlinear
// iterations each, B200 EngineCsr/AMG against the reference EngineCsr/AMG:
//   * EXACT mode: every nonlinear residual of the history bit-identical
//     (compareRuns' maxResidualDelta == 0), coefficients identical;
//   * default (PARITY) mode: compareRuns' maxResidualRelDelta <= 1e-6 and the
//     coefficients within 1e-6 (the criterion's bar);
// and the same two cases through LinearDispatch's multi-rank branch (4 ranks
// on 2 engines, 3 ranks on 3 engines), whose fvb::distributedSolve runs the
// B200's one-device Mode R on the reference's own partitions.
// Prints one "ok"/"FAIL" line per check and a summary line with the measured
// deltas; exit code = number of failures.  Run by tests/test_gpu_dropin.py.
#include "blockfv/case_runner.hpp"
#include "blockfv/engine.hpp"

#include "../../include/bcs.hpp"

#include <cmath>
#include <cstdio>
#include <string>

using namespace fvb;

// tests/cpp/pipeline_interpose.cpp: the __wrap_ of fvb::SolvePipeline::solve
extern "C" int bcs_interpose_route;
extern "C" long bcs_interpose_calls;

static int g_fail = 0;
static void check(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "ok  " : "FAIL", what.c_str());
    if (!ok) ++g_fail;
}

static CaseConfig cavity(int n, int iters) {
    return CaseConfig::fromJson(R"({"name": "cavity)" + std::to_string(n) + R"(",
      "mesh": {"generator": "structured2d", "nx": )" + std::to_string(n) + R"(, "ny": )" + std::to_string(n) + R"(},
      "solver": "pressureCoupled",
      "physics": {"nu": 0.01, "boundaries": {
        "left": {"kind": "wall"}, "right": {"kind": "wall"},
        "bottom": {"kind": "wall"}, "top": {"kind": "movingWall", "u": [1.0, 0.0, 0.0]}}},
      "linear": {"method": "gmres", "relTol": 1e-10, "absTol": 1e-14, "maxIters": 4000, "restart": 60},
      "run": {"maxIters": )" + std::to_string(iters) + R"(, "convergenceTol": 1e-30}})");
}

static CaseConfig sod(int n, int iters) {
    return CaseConfig::fromJson(R"({"name": "sod)" + std::to_string(n) + R"(",
      "mesh": {"generator": "tube1d", "n": )" + std::to_string(n) + R"(},
      "solver": "density",
      "physics": {"flux": "roe", "firstOrder": true, "init": "sod",
                  "cfl": {"start": 1.0, "end": 20.0, "rampIters": 100}},
      "linear": {"method": "gmres", "relTol": 1e-10, "absTol": 1e-14, "maxIters": 4000, "restart": 60},
      "run": {"maxIters": )" + std::to_string(iters) + R"(, "convergenceTol": 1e-30}})");
}

// the acceptance criterion's engine run: EngineCsr backend, AMG (acceptance_main.cpp:110-112)
static CaseConfig engineAmg(CaseConfig c) {
    c.backend = Backend::EngineCsr;
    c.linear.preconditioner = PrecondKind::AMG;
    return c;
}

static RunReport run(const CaseConfig& cfg, int route) {
    bcs_interpose_route = route;
    const long before = bcs_interpose_calls;
    RunReport r = runCase(cfg);
    if (route >= 0)
        check(bcs_interpose_calls - before >= cfg.run.maxIters,
              cfg.name + ": runCase's linear solves went through the B200 pipeline");
    bcs_interpose_route = -1;
    return r;
}

// LinearDispatch's multi-rank branch (case_runner.cpp:329-343): buildPartitioned
// + distributedSolve over simulated ranks consolidated onto engines
static CaseConfig ranks(CaseConfig c, int nRanks, int nEngines, int iters) {
    c.partitioning.ranks = nRanks;
    c.partitioning.engines = nEngines;
    c.run.maxIters = iters;
    c.name += "/ranks" + std::to_string(nRanks) + "x" + std::to_string(nEngines);
    return c;
}

int main() {
    for (const CaseConfig& cfg : {engineAmg(cavity(32, 200)), engineAmg(sod(100, 200)),
                                  ranks(engineAmg(cavity(32, 200)), 4, 2, 200),
                                  ranks(engineAmg(sod(100, 200)), 3, 3, 200)}) {
        const RunReport ref = run(cfg, -1);
        check(ref.iterations == cfg.run.maxIters && static_cast<int>(ref.history.size()) == cfg.run.maxIters,
              cfg.name + ": reference run has all its iterations");
        // EXACT: bit-identical nonlinear history
        const RunReport ex = run(cfg, BCS_MODE_EXACT);
        const ComparisonSummary se = compareRuns(ref, ex);
        bool same = ex.history.size() == ref.history.size();
        for (std::size_t k = 0; same && k < ref.history.size(); ++k)
            same = ex.history[k].residuals == ref.history[k].residuals;
        check(se.overlapIters == cfg.run.maxIters && same && se.maxResidualDelta == 0.0,
              cfg.name + ": EXACT mode, 200 nonlinear residuals bit-identical to the reference through runCase");
        bool coefSame = ex.coefficients == ref.coefficients;
        check(coefSame, cfg.name + ": EXACT mode, final coefficients identical");
        // default mode: the acceptance bar
        const RunReport pa = run(cfg, BCS_MODE_PARITY);
        const ComparisonSummary sp = compareRuns(ref, pa);
        check(sp.overlapIters == cfg.run.maxIters && sp.maxResidualRelDelta <= 1e-6,
              cfg.name + ": PARITY mode, residual histories within 1e-6 relative over 200 iterations");
        double worstCoef = 0.0;
        for (const auto& [k, d] : sp.coefficientDeltas) {
            const double scale = std::max(std::fabs(ref.coefficients.at(k)), std::fabs(pa.coefficients.at(k)));
            if (scale <= 1e-9) continue;  // rounding noise in both runs (acceptance_main.cpp:121-124)
            worstCoef = std::max(worstCoef, d);
        }
        check(worstCoef <= 1e-6, cfg.name + ": PARITY mode, coefficients within 1e-6");
        std::printf("summary %s: exact maxResidualDelta %.3e | parity maxResidualRelDelta %.3e maxResidualDelta %.3e "
                    "worst coefficient delta %.3e\n",
                    cfg.name.c_str(), se.maxResidualDelta, sp.maxResidualRelDelta, sp.maxResidualDelta, worstCoef);
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "PASSED", g_fail);
    return g_fail;
}
