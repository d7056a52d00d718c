// bcs.hpp — header-only C++ drop-in over the C ABI (bcs.h).
//
// bcs::SolvePipeline has the reference's signature
//     std::pair<BlockVector, SolveReport>
//     fvb::SolvePipeline::solve(const BlockLduMatrix&, const BlockVector&,
//                               const BlockVector&, Backend, const SolverConfig&)
// (proj/core/include/blockfv/engine.hpp:28-38, engine.cpp:47-120) and accepts
// the reference's own types (or any types with the same members), so a
// LinearSolveFn (euler.hpp:116-117 / incompressible.hpp:68-69) can switch to
// the B200 by changing one line.  Errors are rethrown with
// the reference's exception types and message text.
#pragma once

#include "bcs.h"

#include <algorithm>
#include <cstdint>
#include <map>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace bcs {

inline void throwStatus(bcs_status st, const char* msg) {
    const std::string m = msg ? msg : "";
    switch (st) {
        case BCS_OK: return;
        case BCS_INVALID_ARGUMENT: throw std::invalid_argument(m);
        case BCS_OUT_OF_MEMORY: throw std::bad_alloc();
        default: throw std::runtime_error(m);
    }
}

// Reference enums are mapped by value: KrylovMethod{GMRES, PBiCGStab},
// PrecondKind{none, LUSGS, DILU, AMG}, Backend{HostLdu, EngineCsr}.
template <class Config>
bcs_solver_config toC(const Config& cfg) {
    bcs_solver_config c;
    bcs_default_config(&c);
    c.method = static_cast<int>(cfg.method);
    c.precond = static_cast<int>(cfg.preconditioner);
    c.rel_tol = cfg.relTol;
    c.abs_tol = cfg.absTol;
    c.max_iters = cfg.maxIters;
    c.gmres_restart = cfg.gmresRestart;
    c.amg_max_levels = cfg.amg.maxLevels;
    c.amg_min_coarse_rows = cfg.amg.minCoarseRows;
    c.amg_pre_sweeps = cfg.amg.preSweeps;
    c.amg_post_sweeps = cfg.amg.postSweeps;
    return c;
}

// Fills a reference-shaped SolveReport (krylov.hpp:39-50).
template <class Report>
Report fromC(const bcs_report& r, bool hostBackend) {
    Report out;
    out.iterations = r.iterations;
    out.initialResidual = r.initial_residual;
    out.finalResidual = r.final_residual;
    out.converged = r.converged != 0;
    out.breakdown = r.breakdown != 0;
    out.timings["convert"] = r.t_convert;
    out.timings["setup"] = r.t_setup;
    if (!hostBackend) out.timings["replace"] = r.t_replace;
    out.timings["solve"] = r.t_solve;
    out.timings["retrieve"] = r.t_retrieve;
    return out;
}

class SolvePipeline {
public:
    explicit SolvePipeline(int device = 0) {
        const bcs_status st = bcs_create(&ctx_, device);
        if (st != BCS_OK) throwStatus(st, bcs_last_error(nullptr));
    }
    ~SolvePipeline() { bcs_destroy(ctx_); }
    SolvePipeline(const SolvePipeline&) = delete;
    SolvePipeline& operator=(const SolvePipeline&) = delete;

    // execution mode of the following solves (bcs_solver_config.mode:
    // BCS_MODE_PARITY default, BCS_MODE_EXACT, BCS_MODE_PERF, BCS_MODE_PERF_JACOBI);
    // the reference's SolverConfig has no such field
    void setMode(int mode) { mode_ = mode; }
    int mode() const { return mode_; }

    template <class Report, class Matrix, class Vector, class Backend, class Config>
    std::pair<Vector, Report> solve(const Matrix& A, const Vector& b, const Vector& x0, Backend backend,
                                    const Config& cfg) {
        if (b.blockSize != A.blockSize() || x0.blockSize != A.blockSize() || b.nCells() != A.nCells() ||
            x0.nCells() != A.nCells())
            throw std::invalid_argument("SolvePipeline::solve: dimension mismatch");
        // the mesh is immutable (block_matrix.hpp:81): addressing is refreshed
        // only when the matrix refers to a different mesh object
        const void* mesh = &A.mesh();
        if (mesh != mesh_ || static_cast<int>(owner_.size()) != A.nFaces()) {
            const auto& faces = A.mesh().faces();
            owner_.resize(faces.size());
            neigh_.resize(faces.size());
            for (std::size_t f = 0; f < faces.size(); ++f) {
                owner_[f] = faces[f].owner;
                neigh_[f] = faces[f].neighbour;
            }
            mesh_ = mesh;
        }
        Vector x(A.nCells(), A.blockSize());
        bcs_solver_config c = toC(cfg);
        c.mode = mode_;
        bcs_report r{};
        const int be = static_cast<int>(backend);
        const bcs_status st = bcs_pipeline_solve(
            ctx_, A.nCells(), A.nFaces(), A.blockSize(), owner_.data(), neigh_.data(), A.diagValues().data(),
            A.upperValues().data(), A.lowerValues().data(), b.values.data(), b.values.size(), x0.values.data(),
            x0.values.size(), x.values.data(), be, &c, &r);
        if (st != BCS_OK) throwStatus(st, bcs_last_error(ctx_));
        return {std::move(x), fromC<Report>(r, be == BCS_BACKEND_HOST_LDU)};
    }

    // distributedSolve itself (partition.hpp, partition.cpp:370-479) over the
    // reference's own partition types: rank partitions as buildPartitioned
    // returns them (rowStart/rowEnd, BlockCsrMatrix `local`, HaloCoefficients
    // `halo`), DistributedVector b/x0 (rank slices), its ConsolidationPlan and
    // Decomposition.  The MailboxNetwork of the reference's simulated ranks is
    // not needed (the engines share this device).  Returns x as rank slices.
    template <class Report, class Parts, class DVec, class Config, class Plan, class Dec>
    std::pair<DVec, Report> distributedSolve(const Parts& parts, const DVec& b, const DVec& x0, const Config& cfg,
                                             const Plan& plan, const Dec& dec) {
        const int R = static_cast<int>(parts.size());
        if (R < 1 || static_cast<int>(b.size()) != R || static_cast<int>(x0.size()) != R)
            throw std::invalid_argument("distributedSolve: dimension mismatch");
        const int n = parts[0].local.blockSize;
        const size_t nn = static_cast<size_t>(n) * n;
        std::vector<int32_t> rro(R + 1, 0), hcnt(R);
        std::vector<const int32_t*> lro(R), lci(R), hrow(R), hcol(R), hpeer(R);
        std::vector<const double*> lv(R), hv(R);
        std::vector<std::vector<int32_t>> hr(R), hc(R), hp(R);
        std::vector<std::vector<double>> hb(R);
        for (int r = 0; r < R; ++r) {
            const auto& p = parts[r];
            if (p.id != r || p.local.blockSize != n) throw std::invalid_argument("distributedSolve: bad partition list");
            rro[r] = p.rowStart;
            rro[r + 1] = p.rowEnd;
            lro[r] = p.local.rowOffsets.data();
            lci[r] = p.local.colIndices.data();
            lv[r] = p.local.values.data();
            const auto& E = p.halo.entries;
            hcnt[r] = static_cast<int32_t>(E.size());
            hr[r].resize(E.size());
            hc[r].resize(E.size());
            hp[r].resize(E.size());
            hb[r].resize(E.size() * nn);
            for (size_t h = 0; h < E.size(); ++h) {
                hr[r][h] = E[h].localRow;
                hc[r][h] = E[h].globalCol;
                hp[r][h] = E[h].peerRank;
                std::copy(E[h].block.begin(), E[h].block.end(), hb[r].begin() + h * nn);
            }
            hrow[r] = hr[r].data();
            hcol[r] = hc[r].data();
            hpeer[r] = hp[r].data();
            hv[r] = hb[r].data();
            if (b[r].size() != static_cast<size_t>(p.rowEnd - p.rowStart) * n || x0[r].size() != b[r].size())
                throw std::invalid_argument("distributedSolve: dimension mismatch");
        }
        (void)dec;  // rank row ranges travel with the partitions
        std::vector<double> gb, gx0;
        for (int r = 0; r < R; ++r) {
            gb.insert(gb.end(), b[r].begin(), b[r].end());
            gx0.insert(gx0.end(), x0[r].begin(), x0[r].end());
        }
        std::vector<double> gx(gb.size());
        std::vector<int32_t> r2e(plan.rankToEngine.begin(), plan.rankToEngine.end()),
            ero(plan.engineRowOffset.begin(), plan.engineRowOffset.end());
        bcs_solver_config c = toC(cfg);
        c.mode = mode_;
        bcs_report rep{};
        const bcs_status st = bcs_dist_solve_parts(ctx_, R, n, rro.data(), lro.data(), lci.data(), lv.data(),
                                                   hcnt.data(), hrow.data(), hcol.data(), hpeer.data(), hv.data(),
                                                   plan.nEngines, r2e.data(), ero.data(), gb.data(), gx0.data(),
                                                   gx.data(), &c, &rep);
        if (st != BCS_OK) throwStatus(st, bcs_last_error(ctx_));
        DVec x(R);
        size_t off = 0;
        for (int r = 0; r < R; ++r) {
            x[r].assign(gx.begin() + off, gx.begin() + off + b[r].size());
            off += b[r].size();
        }
        Report out;
        out.iterations = rep.iterations;
        out.initialResidual = rep.initial_residual;
        out.finalResidual = rep.final_residual;
        out.converged = rep.converged != 0;
        out.breakdown = rep.breakdown != 0;
        out.timings["convert"] = rep.t_convert;
        out.timings["setup"] = rep.t_setup;
        out.timings["solve"] = rep.t_solve;
        out.timings["retrieve"] = rep.t_retrieve;
        return {std::move(x), std::move(out)};
    }

    // Mode R: the multi-rank branch of LinearDispatch::solve
    // (case_runner.cpp:329-343) — decompose + buildPartitioned +
    // makeConsolidationPlan + distributedSolve + gatherVector in one call.
    // b, x0 and the returned x are in the original cell order.
    template <class Report, class Matrix, class Vector, class Config>
    std::pair<Vector, Report> distributedSolve(const Matrix& A, const Vector& b, const Vector& x0,
                                               const Config& cfg, int nRanks, int nEngines) {
        if (b.blockSize != A.blockSize() || x0.blockSize != A.blockSize() || b.nCells() != A.nCells() ||
            x0.nCells() != A.nCells())
            throw std::invalid_argument("distributedSolve: dimension mismatch");
        const auto& faces = A.mesh().faces();
        const int nf = A.nFaces();
        std::vector<int32_t> own(nf), nei(nf);
        for (int f = 0; f < nf; ++f) {
            own[f] = faces[f].owner;
            nei[f] = faces[f].neighbour;
        }
        const auto& cen = A.mesh().cellCentroids();
        std::vector<double> c(3 * cen.size());
        for (std::size_t i = 0; i < cen.size(); ++i) {
            c[3 * i] = cen[i].x;
            c[3 * i + 1] = cen[i].y;
            c[3 * i + 2] = cen[i].z;
        }
        Vector x(A.nCells(), A.blockSize());
        bcs_solver_config cc = toC(cfg);
        cc.mode = mode_;
        bcs_report r{};
        const bcs_status st = bcs_dist_solve(ctx_, A.nCells(), nf, A.blockSize(), own.data(), nei.data(), c.data(),
                                             A.diagValues().data(), A.upperValues().data(), A.lowerValues().data(),
                                             b.values.data(), x0.values.data(), x.values.data(), nRanks, nEngines,
                                             &cc, &r);
        if (st != BCS_OK) throwStatus(st, bcs_last_error(ctx_));
        Report out = fromC<Report>(r, true);
        return {std::move(x), std::move(out)};
    }

    // Device assembleJacobian + computeResidual (euler.cpp:361-455) over the
    // reference's own Mesh / EulerCase / PrimState types: patchOverride is
    // resolved per patch (:345-348), the flux scheme and the reconstruction
    // are passed through (bcs_assemble_euler_ex).  The matrix stays in this
    // pipeline's context for solveAssembled; the right-hand side (vector-first
    // order, like the reference's) is returned.  The device kernels carry the
    // reference's default gas (gamma 1.4).
    template <class Vector, class States, class Mesh, class Case>
    Vector assembleJacobian(const States& q, const Mesh& mesh, const Case& ec, double cfl) {
        if (ec.gas.gamma != 1.4) throw std::invalid_argument("device assembly: only gamma = 1.4 is compiled in");
        const auto& faces = mesh.faces();
        const int nf = static_cast<int>(faces.size()), nc = mesh.nCells();
        if (static_cast<int>(q.size()) != nc) throw std::invalid_argument("assembleJacobian: state size mismatch");
        std::vector<int32_t> own(nf), nei(nf), bcell, bkind;
        std::vector<double> area(3 * static_cast<size_t>(nf)), fx(nf), cen(3 * static_cast<size_t>(nc)), barea, qv;
        for (int f = 0; f < nf; ++f) {
            own[f] = faces[f].owner;
            nei[f] = faces[f].neighbour;
            area[3 * f] = faces[f].areaVector.x;
            area[3 * f + 1] = faces[f].areaVector.y;
            area[3 * f + 2] = faces[f].areaVector.z;
            fx[f] = faces[f].fx;
        }
        const auto& cc = mesh.cellCentroids();
        for (int i = 0; i < nc; ++i) {
            cen[3 * i] = cc[i].x;
            cen[3 * i + 1] = cc[i].y;
            cen[3 * i + 2] = cc[i].z;
        }
        for (const auto& patch : mesh.patches()) {
            const auto it = ec.patchOverride.find(patch.name);
            const int kind = static_cast<int>(it == ec.patchOverride.end() ? patch.kind : it->second);
            for (const auto& bf : patch.faces) {
                bcell.push_back(bf.cell);
                bkind.push_back(kind);
                barea.push_back(bf.areaVector.x);
                barea.push_back(bf.areaVector.y);
                barea.push_back(bf.areaVector.z);
            }
        }
        qv.resize(5 * static_cast<size_t>(nc));
        for (int i = 0; i < nc; ++i)
            for (int k = 0; k < 5; ++k) qv[5 * static_cast<size_t>(i) + k] = q[i][k];
        double qinf[5];
        for (int k = 0; k < 5; ++k) qinf[k] = ec.freestream[k];
        const int recon = ec.recon.firstOrder ? 0 : (static_cast<int>(ec.recon.limiter) == 0 ? 1 : 2);
        Vector rhs(nc, 5);
        const bcs_status st = bcs_assemble_euler_ex(
            ctx_, nc, nf, own.data(), nei.data(), area.data(), fx.data(), cen.data(), static_cast<int>(bcell.size()),
            bcell.data(), barea.data(), bkind.data(), qv.data(), qinf, recon, static_cast<int>(ec.flux), cfl,
            rhs.values.data());
        if (st != BCS_OK) throwStatus(st, bcs_last_error(ctx_));
        return rhs;
    }

    // Device assembleCoupled (incompressible.cpp:143-250) followed by
    // pinPressure(pinCell, pinValue) (:252-264; pinCell < 0: none) over the
    // reference's own state / face fluxes / Mesh / BcMap (every
    // IncompressibleBc kind).  The matrix stays in this context for
    // solveAssembled; the right-hand side is returned.
    template <class Vector, class Flux, class Mesh, class Bcs>
    Vector assembleCoupled(const Vector& state, const Flux& phi, const Mesh& mesh, double nu, const Bcs& bcs,
                           int pinCell, double pinValue = 0.0) {
        const auto& faces = mesh.faces();
        const int nf = static_cast<int>(faces.size()), nc = mesh.nCells();
        if (state.nCells() != nc || state.blockSize != 4 || static_cast<int>(phi.size()) != nf)
            throw std::invalid_argument("assembleCoupled: size mismatch");
        std::vector<int32_t> own(nf), nei(nf), bcell, bkind;
        std::vector<double> area(3 * static_cast<size_t>(nf)), fx(nf), cen(3 * static_cast<size_t>(nc)), barea, bu, bp;
        for (int f = 0; f < nf; ++f) {
            own[f] = faces[f].owner;
            nei[f] = faces[f].neighbour;
            area[3 * f] = faces[f].areaVector.x;
            area[3 * f + 1] = faces[f].areaVector.y;
            area[3 * f + 2] = faces[f].areaVector.z;
            fx[f] = faces[f].fx;
        }
        const auto& cc = mesh.cellCentroids();
        for (int i = 0; i < nc; ++i) {
            cen[3 * i] = cc[i].x;
            cen[3 * i + 1] = cc[i].y;
            cen[3 * i + 2] = cc[i].z;
        }
        for (const auto& patch : mesh.patches()) {
            const auto it = bcs.find(patch.name);
            if (it == bcs.end())  // bcFor (incompressible.cpp:43-48)
                throw std::invalid_argument("no boundary condition for patch '" + patch.name + "'");
            const auto& bc = it->second;
            for (const auto& bf : patch.faces) {
                bcell.push_back(bf.cell);
                bkind.push_back(static_cast<int32_t>(bc.kind));
                barea.push_back(bf.areaVector.x);
                barea.push_back(bf.areaVector.y);
                barea.push_back(bf.areaVector.z);
                bu.push_back(bc.u.x);
                bu.push_back(bc.u.y);
                bu.push_back(bc.u.z);
                bp.push_back(bc.p);
            }
        }
        Vector rhs(nc, 4);
        const bcs_status st = bcs_assemble_coupled_ex(
            ctx_, nc, nf, own.data(), nei.data(), area.data(), fx.data(), mesh.cellVolumes().data(), cen.data(),
            static_cast<int>(bcell.size()), bcell.data(), barea.data(), bkind.data(), bu.data(), bp.data(),
            state.values.data(), phi.data(), nu, pinCell, pinValue, rhs.values.data());
        if (st != BCS_OK) throwStatus(st, bcs_last_error(ctx_));
        return rhs;
    }

    // Krylov + preconditioner on the matrix assembled in this context
    // (bcs_solve: the reference's solveCsr, engine.cpp:31-45).
    template <class Report, class Vector, class Config>
    std::pair<Vector, Report> solveAssembled(const Vector& b, const Vector& x0, const Config& cfg) {
        Vector x = x0;
        bcs_solver_config c = toC(cfg);
        c.mode = mode_;
        bcs_report r{};
        const bcs_status st = bcs_solve(ctx_, b.values.data(), x.values.data(), &c, &r);
        if (st != BCS_OK) throwStatus(st, bcs_last_error(ctx_));
        return {std::move(x), fromC<Report>(r, false)};
    }

    bcs_ctx* handle() const { return ctx_; }

private:
    bcs_ctx* ctx_ = nullptr;
    int mode_ = BCS_MODE_PARITY;
    const void* mesh_ = nullptr;
    std::vector<int32_t> owner_, neigh_;
};

}  // namespace bcs
