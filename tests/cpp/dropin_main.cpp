// Drop-in check with the reference's OWN types (TEST INFRASTRUCTURE).
//
// Built by oracle/Makefile against the read-only reference sources (its
// headers, objects and test fixtures) and the product libbcs.so, into
// oracle/_ref/dropin_test; run on the GPU box by tests/test_gpu_dropin.py.
// It mirrors the reference's own tests with bcs::SolvePipeline (include/bcs.hpp)
// substituted for fvb::SolvePipeline:
//   * test_engine.cpp:13-38   host vs engine backends agree (1e-8)
//   * test_engine.cpp:40-56   host backend rejects DILU/AMG (invalid_argument)
//   * test_engine.cpp:58-93   setup branch then replace branch; same answer
//   * test_engine.cpp:95-102  dimension mismatch -> invalid_argument
//   * acceptance_main.cpp:105-134 (criterion 2): nonlinear residual histories of
//     the coupled cavity (4x4) and the implicit Sod tube (5x5) over 200 outer
//     iterations, reference EngineCsr/AMG vs B200 EngineCsr/AMG, <= 1e-6 rel.
//   * euler.cpp:390-470 device assembly: bcs::SolvePipeline::assembleJacobian
//     on the reference's own meshes (generateStructured2d: inlet/outlet/wall,
//     generate1dTube: inlet/outlet/slip), every flux x reconstruction, plus
//     patchOverride: right-hand side bit-identical to fvb::assembleJacobian and
//     solves bit-identical to uploading the reference's matrix; and a 100-step
//     second-order (HLLC + MUSCL/Barth-Jespersen) implicit Sod run whose
//     LinearSolveFn assembles on the device, checked bit for bit every step.
#include "blockfv/case_runner.hpp"
#include "blockfv/engine.hpp"
#include "blockfv/euler.hpp"
#include "blockfv/incompressible.hpp"
#include "blockfv/partition.hpp"
#include "support/test_helpers.hpp"

#include "../../include/bcs.hpp"

#include <cmath>
#include <cstring>
#include <cstdio>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>

using namespace fvb;

static int g_fail = 0;
#define CHECK(cond, what)                                                  \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__);    \
            ++g_fail;                                                      \
        } else {                                                           \
            std::printf("ok   %s\n", what);                                \
        }                                                                  \
    } while (0)

static double maxAbsDiff(const BlockVector& a, const BlockVector& b, double* scale) {
    double s = 0.0, e = 0.0;
    for (std::size_t i = 0; i < a.values.size(); ++i) {
        s = std::max(s, std::fabs(a.values[i]));
        e = std::max(e, std::fabs(a.values[i] - b.values[i]));
    }
    *scale = s;
    return e;
}

int main() {
    bcs::SolvePipeline gpu(0);

    // --- test_engine.cpp:13-38 analog on the B200
    {
        std::mt19937 rng(51);
        bool all = true;
        for (int trial = 0; trial < 4; ++trial) {
            const Mesh m = testsup::randomMesh(rng, 200);
            BlockLduMatrix A(m, testsup::variablesFor(4));
            testsup::randomize(A, rng);
            const BlockVector b = testsup::randomVector(m.nCells(), 4, rng);
            BlockVector x0(m.nCells(), 4);
            SolverConfig cfg;
            cfg.relTol = 1e-12;
            cfg.maxIters = 2000;
            bcs::SolvePipeline fresh(0);
            const auto [xh, rh] = fresh.solve<SolveReport>(A, b, x0, Backend::HostLdu, cfg);
            const auto [xe, re] = gpu.solve<SolveReport>(A, b, x0, Backend::EngineCsr, cfg);
            const auto [xr, rr] = backendSolve(A, b, x0, Backend::EngineCsr, cfg);  // the reference itself
            double sc;
            all = all && rh.converged && re.converged && maxAbsDiff(xh, xe, &sc) <= 1e-8 * sc &&
                  maxAbsDiff(xr, xe, &sc) <= 1e-8 * sc && std::abs(re.iterations - rr.iterations) <= 1;
        }
        CHECK(all, "host and engine backends agree to solver tolerance (and match the reference)");
    }
    // --- test_engine.cpp:40-56
    {
        const Mesh m = generate1dTube(4, 1.0);
        BlockLduMatrix A(m, testsup::variablesFor(1));
        std::mt19937 rng(1);
        testsup::randomize(A, rng);
        const BlockVector b = testsup::randomVector(m.nCells(), 1, rng);
        const BlockVector x0(m.nCells(), 1);
        SolverConfig cfg;
        bool threw = false;
        cfg.preconditioner = PrecondKind::DILU;
        try {
            gpu.solve<SolveReport>(A, b, x0, Backend::HostLdu, cfg);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw, "host backend rejects DILU with std::invalid_argument");
        threw = false;
        cfg.preconditioner = PrecondKind::AMG;
        try {
            gpu.solve<SolveReport>(A, b, x0, Backend::HostLdu, cfg);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw, "host backend rejects AMG with std::invalid_argument");
        cfg.preconditioner = PrecondKind::DILU;
        CHECK(gpu.solve<SolveReport>(A, b, x0, Backend::EngineCsr, cfg).second.converged,
              "engine path accepts DILU");
    }
    // --- test_engine.cpp:58-93 (setup then replace)
    {
        std::mt19937 rng(61);
        const Mesh m = generateStructured2d(6, 6, {1, 1, 1});
        BlockLduMatrix A(m, testsup::variablesFor(4));
        testsup::randomize(A, rng);
        const BlockVector b = testsup::randomVector(m.nCells(), 4, rng);
        BlockVector x0(m.nCells(), 4);
        SolverConfig cfg;
        cfg.relTol = 1e-10;
        cfg.preconditioner = PrecondKind::AMG;
        bcs::SolvePipeline p(0);
        const auto [x1, r1] = p.solve<SolveReport>(A, b, x0, Backend::EngineCsr, cfg);
        CHECK(r1.timings.at("setup") > 0.0 && r1.timings.at("replace") == 0.0, "first call takes the setup branch");
        const auto [x2, r2] = p.solve<SolveReport>(A, b, x0, Backend::EngineCsr, cfg);
        CHECK(r2.timings.at("replace") > 0.0 && r2.timings.at("setup") == 0.0, "second call takes the replace branch");
        double sc;
        CHECK(maxAbsDiff(x1, x2, &sc) <= 1e-9 * sc, "replace result equals setup result");
    }
    // --- test_engine.cpp:95-102
    {
        const Mesh m = generate1dTube(4, 1.0);
        BlockLduMatrix A(m, testsup::variablesFor(4));
        const BlockVector b(3, 4), x0(4, 4);
        bool threw = false;
        try {
            gpu.solve<SolveReport>(A, b, x0, Backend::EngineCsr, SolverConfig{});
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()).find("dimension mismatch") != std::string::npos;
        }
        CHECK(threw, "dimension mismatch -> std::invalid_argument");
    }
    // --- Mode R: LinearDispatch's multi-rank branch (case_runner.cpp:329-343)
    {
        std::mt19937 rng(71);
        const Mesh m = generateStructured2d(24, 20, {1, 1, 1});
        BlockLduMatrix A(m, testsup::variablesFor(4));
        testsup::randomize(A, rng);
        const BlockVector b = testsup::randomVector(m.nCells(), 4, rng);
        BlockVector x0(m.nCells(), 4);
        SolverConfig cfg;
        cfg.relTol = 1e-10;
        cfg.preconditioner = PrecondKind::AMG;
        bool all = true;
        for (const auto& re : std::vector<std::pair<int, int>>{{2, 1}, {4, 2}, {6, 3}}) {
            const Decomposition dec = decompose(m, re.first);
            const ConsolidationPlan plan = makeConsolidationPlan(dec, re.second);
            const std::vector<MatrixPartition> parts = buildPartitioned(A, dec);
            MailboxNetwork net;
            auto [dx, rr] = distributedSolve(parts, scatterVector(b, dec, 4), scatterVector(x0, dec, 4), cfg, plan,
                                             dec, net);
            const BlockVector xr = gatherVector(dx, dec, 4);
            const auto [xg, rg] = gpu.distributedSolve<SolveReport>(A, b, x0, cfg, re.first, re.second);
            double sc;
            const double e = maxAbsDiff(xr, xg, &sc);
            std::printf("     ranks %d engines %d: iters ref %d gpu %d, max |dx| %.3e (scale %.3e)\n", re.first,
                        re.second, rr.iterations, rg.iterations, e, sc);
            all = all && rg.converged && std::abs(rr.iterations - rg.iterations) <= 1 && e <= 1e-8 * sc;
        }
        CHECK(all, "Mode R distributedSolve matches the reference (ranks/engines 2/1, 4/2, 6/3)");
    }
    // --- acceptance criterion 2 analog: nonlinear residual histories, 200 outer iterations
    // histories are compared with the reference's own compareRuns
    // (case_runner.cpp:631-676), exactly as acceptance criterion 2 does
    auto record = [](RunReport& rr, int iter, const double* res, int n) {
        IterationRecord rec;
        rec.iter = iter;
        rec.residuals.assign(res, res + n);
        rr.history.push_back(std::move(rec));
    };
    SolverConfig lin;
    lin.method = KrylovMethod::GMRES;
    lin.preconditioner = PrecondKind::AMG;
    lin.relTol = 1e-10;
    lin.absTol = 1e-14;
    lin.maxIters = 4000;
    lin.gmresRestart = 60;
    {
        // lid-driven cavity 32x32, coupled p-U (4x4): acceptance_main.cpp:75-88
        const Mesh m = generateStructured2d(32, 32, {1, 1, 1});
        BcMap bcs;
        bcs["left"] = {IncompressibleBc::Kind::wall, {}, 0.0};
        bcs["right"] = {IncompressibleBc::Kind::wall, {}, 0.0};
        bcs["bottom"] = {IncompressibleBc::Kind::wall, {}, 0.0};
        bcs["top"] = {IncompressibleBc::Kind::movingWall, {1.0, 0.0, 0.0}, 0.0};
        BlockVector sRef(m.nCells(), 4), sGpu(m.nCells(), 4);
        FaceFluxField pRef(m.nInternalFaces(), 0.0), pGpu(m.nInternalFaces(), 0.0);
        SolvePipeline refPipe;
        CoupledSolveFn refSolve = [&](const BlockLduMatrix& A, const BlockVector& b, const BlockVector& x0) {
            return refPipe.solve(A, b, x0, Backend::EngineCsr, lin);
        };
        CoupledSolveFn gpuSolve = [&](const BlockLduMatrix& A, const BlockVector& b, const BlockVector& x0) {
            return gpu.solve<SolveReport>(A, b, x0, Backend::EngineCsr, lin);
        };
        RunReport ra, rg;
        ra.residualNames = rg.residualNames = {"Ux", "Uy", "Uz", "p"};
        for (int it = 0; it < 200; ++it) {
            const IterateResult a = coupledIterate(sRef, pRef, m, 0.01, bcs, refSolve);
            const IterateResult g = coupledIterate(sGpu, pGpu, m, 0.01, bcs, gpuSolve);
            record(ra, it + 1, a.residuals.data(), 4);
            record(rg, it + 1, g.residuals.data(), 4);
        }
        const ComparisonSummary cs = compareRuns(ra, rg);
        const double worst = cs.maxResidualRelDelta;
        std::printf("     cavity32 worst residual rel delta %.3e (overlap %d)\n", worst, cs.overlapIters);
        CHECK(worst <= 1e-6, "cavity 32^2 coupled (4x4): 200 nonlinear iterations match the reference (<=1e-6)");
    }
    {
        // implicit Sod tube, 100 cells, first-order Roe, cfl ramp 1->20 over 100: acceptance_main.cpp:90-102
        const Mesh m = generate1dTube(100, 1.0);
        EulerCase ec;
        ec.flux = FluxScheme::Roe;
        ec.recon.firstOrder = true;
        std::vector<PrimState> qRef(m.nCells()), qGpu(m.nCells());
        for (int i = 0; i < m.nCells(); ++i) {
            const bool left = m.cellCentroids()[i].x < 0.5;
            qRef[i] = left ? PrimState{1.0, 0.0, 0.0, 0.0, 1.0} : PrimState{0.125, 0.0, 0.0, 0.0, 0.1};
        }
        qGpu = qRef;
        PseudoTimeControl ctl;
        ctl.startCfl = 1.0;
        ctl.endCfl = 20.0;
        ctl.rampIters = 100;
        SolvePipeline refPipe;
        LinearSolveFn refSolve = [&](const BlockLduMatrix& A, const BlockVector& b, const BlockVector& x0) {
            return refPipe.solve(A, b, x0, Backend::EngineCsr, lin);
        };
        LinearSolveFn gpuSolve = [&](const BlockLduMatrix& A, const BlockVector& b, const BlockVector& x0) {
            return gpu.solve<SolveReport>(A, b, x0, Backend::EngineCsr, lin);
        };
        RunReport ra, rg;
        ra.residualNames = rg.residualNames = {"rho", "rhoUx", "rhoUy", "rhoUz", "rhoE"};
        for (int it = 0; it < 200; ++it) {
            const EulerStepResult a = implicitStep(qRef, m, ec, ctl.cfl(it), refSolve);
            const EulerStepResult g = implicitStep(qGpu, m, ec, ctl.cfl(it), gpuSolve);
            record(ra, it + 1, a.residualNorms.data(), 5);
            record(rg, it + 1, g.residualNorms.data(), 5);
        }
        const ComparisonSummary cs = compareRuns(ra, rg);
        const double worst = cs.maxResidualRelDelta;
        std::printf("     sod100 worst residual rel delta %.3e (overlap %d)\n", worst, cs.overlapIters);
        CHECK(worst <= 1e-6, "Sod tube implicit (5x5): 200 nonlinear iterations match the reference (<=1e-6)");
    }
    // --- device assembly with the reference's own types (euler.cpp:390-455)
    {
        auto sameBits = [](const BlockVector& a, const BlockVector& b) {
            return a.values.size() == b.values.size() &&
                   std::memcmp(a.values.data(), b.values.data(), sizeof(double) * a.values.size()) == 0;
        };
        const Mesh meshes[2] = {generateStructured2d(12, 9, {1.0, 0.75, 0.1}), generate1dTube(60, 1.0)};
        const char* names[2] = {"structured 12x9", "tube 60"};
        std::mt19937 rng(5);
        std::uniform_real_distribution<double> U(-0.05, 0.05);
        SolverConfig cfgA;
        cfgA.method = KrylovMethod::GMRES;
        cfgA.preconditioner = PrecondKind::DILU;
        cfgA.relTol = 1e-10;
        bool allRhs = true, allSolve = true;
        int cases = 0;
        for (int mi = 0; mi < 2; ++mi) {
            const Mesh& m = meshes[mi];
            std::vector<PrimState> q(m.nCells());
            for (auto& st : q) st = {1.0 + U(rng), 0.4 + U(rng), 0.1 + U(rng), U(rng), (1.0 / 1.4) * (1.0 + U(rng))};
            for (int fl = 0; fl < 3; ++fl)
                for (int rc = 0; rc < 3; ++rc)
                    for (int ov = 0; ov < 2; ++ov) {
                        EulerCase ec;
                        ec.flux = static_cast<FluxScheme>(fl);
                        ec.recon.firstOrder = rc == 0;
                        ec.recon.limiter = rc == 1 ? Limiter::none : Limiter::BarthJespersen;
                        ec.freestream = {1.0, 0.5, 0.1, 0.0, 1.0 / 1.4};
                        if (ov) {  // the reference's patchOverride hook (euler.cpp:345-348)
                            ec.patchOverride["left"] = PatchKind::farfield;
                            ec.patchOverride["right"] = PatchKind::symmetry;
                        }
                        auto [A, rhs] = fvb::assembleJacobian(q, m, ec, 20.0);
                        const BlockVector rhsG = gpu.assembleJacobian<BlockVector>(q, m, ec, 20.0);
                        const bool okR = sameBits(rhs, rhsG);
                        const BlockVector x0(m.nCells(), 5);
                        auto [xa, ra] = gpu.solveAssembled<SolveReport>(rhsG, x0, cfgA);
                        auto [xu, ru] = gpu.solve<SolveReport>(A, rhs, x0, Backend::EngineCsr, cfgA);
                        const bool okS = sameBits(xa, xu) && ra.iterations == ru.iterations;
                        if (!okR || !okS)
                            std::printf("     mismatch: %s flux %d recon %d override %d (rhs %d solve %d)\n",
                                        names[mi], fl, rc, ov, okR, okS);
                        allRhs = allRhs && okR;
                        allSolve = allSolve && okS;
                        ++cases;
                    }
        }
        std::printf("     %d assembly cases\n", cases);
        CHECK(allRhs, "device assembleJacobian: right-hand side bit-identical on reference meshes (all fluxes, "
                      "recon, patchOverride)");
        CHECK(allSolve, "device assembleJacobian: solve bit-identical to uploading the reference matrix");

        // a second-order implicit Sod run whose solve assembles on the device
        const Mesh m = generate1dTube(100, 1.0);
        EulerCase ec;
        ec.flux = FluxScheme::HLLC;
        ec.recon.firstOrder = false;
        ec.recon.limiter = Limiter::BarthJespersen;
        std::vector<PrimState> qs(m.nCells());
        for (int i = 0; i < m.nCells(); ++i)
            qs[i] = m.cellCentroids()[i].x < 0.5 ? PrimState{1.0, 0.0, 0.0, 0.0, 1.0}
                                                 : PrimState{0.125, 0.0, 0.0, 0.0, 0.1};
        PseudoTimeControl ctl;
        ctl.startCfl = 1.0;
        ctl.endCfl = 20.0;
        ctl.rampIters = 50;
        double cflNow = 0.0;
        bool everyStep = true;
        LinearSolveFn devSolve = [&](const BlockLduMatrix& A, const BlockVector& b, const BlockVector& x0) {
            (void)A;  // the matrix is assembled on the device from the same state
            const BlockVector rhsG = gpu.assembleJacobian<BlockVector>(qs, m, ec, cflNow);
            everyStep = everyStep && sameBits(rhsG, b);
            return gpu.solveAssembled<SolveReport>(rhsG, x0, lin);
        };
        for (int it = 0; it < 100; ++it) {
            cflNow = ctl.cfl(it);
            implicitStep(qs, m, ec, cflNow, devSolve);
        }
        CHECK(everyStep, "implicit Sod, HLLC + MUSCL/Barth-Jespersen: device assembly bit-identical in all 100 steps");
    }
    // --- coupled device assembly inside the reference's coupledIterate
    //     (incompressible.cpp:324-341): cavity (walls + moving lid, pinned
    //     pressure) and a channel (inlet, outlet, walls: pressure level fixed)
    {
        auto sameBits = [](const BlockVector& a, const BlockVector& b) {
            return a.values.size() == b.values.size() &&
                   std::memcmp(a.values.data(), b.values.data(), sizeof(double) * a.values.size()) == 0;
        };
        for (int cs = 0; cs < 2; ++cs) {
            const Mesh m = generateStructured2d(cs ? 24 : 16, cs ? 8 : 16, {cs ? 3.0 : 1.0, 1.0, 1.0});
            BcMap bcs;
            if (cs == 0) {
                for (const char* nm : {"left", "right", "bottom"}) bcs[nm] = {IncompressibleBc::Kind::wall, {}, 0.0};
                bcs["top"] = {IncompressibleBc::Kind::movingWall, {1.0, 0.0, 0.0}, 0.0};
            } else {
                bcs["left"] = {IncompressibleBc::Kind::inlet, {1.0, 0.0, 0.0}, 0.0};
                bcs["right"] = {IncompressibleBc::Kind::outlet, {}, 0.0};
                bcs["bottom"] = {IncompressibleBc::Kind::wall, {}, 0.0};
                bcs["top"] = {IncompressibleBc::Kind::wall, {}, 0.0};
            }
            BlockVector st(m.nCells(), 4);
            FaceFluxField ph(m.nInternalFaces(), 0.0);
            const int pin = fixesPressureLevel(bcs) ? -1 : 0;
            bool every = true;
            CoupledSolveFn devSolve = [&](const BlockLduMatrix& A, const BlockVector& b, const BlockVector& x0) {
                (void)A;  // assembled on the device from the same state and fluxes
                const BlockVector rhsG = gpu.assembleCoupled<BlockVector>(st, ph, m, 0.01, bcs, pin);
                every = every && sameBits(rhsG, b);
                return gpu.solveAssembled<SolveReport>(rhsG, x0, lin);
            };
            for (int it = 0; it < 40; ++it) coupledIterate(st, ph, m, 0.01, bcs, devSolve);
            CHECK(every, cs ? "coupled channel (inlet/outlet/walls): device assembly bit-identical in 40 coupledIterate steps"
                            : "coupled cavity: device assembly bit-identical in 40 coupledIterate steps");
        }
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "PASSED", g_fail);
    return g_fail ? 1 : 0;
}
