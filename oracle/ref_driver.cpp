// TEST INFRASTRUCTURE ONLY — never linked into the product (libbcs.so).
//
// C-ABI shim around the *unmodified* reference implementation (blockfv,
// /root/reference/proj/core), compiled from its own sources by
// oracle/Makefile into oracle/_ref/libbcs_ref.so.  Used by tests/ to pin the
// C restatement (oracle/bcs_oracle.c) and the synthetic generator, by
// oracle/make_golden.py to produce tests/golden/*, and by bench.py's
// cpu_baseline / --impl reference leg to time the reference CPU path.
//
// Nothing here re-implements reference arithmetic: every number comes from a
// reference call (SolvePipeline::solve, lduToBlockCsr, AmgHierarchy,
// CsrDiluPrecond, decompose, buildPartitioned, distributedSolve, ...).
// The only arithmetic of our own is the residual-history replay, which
// re-runs the reference's Givens recurrence (krylov.cpp:104-117) on the dot
// stream recorded through the KrylovOps::dot hook (krylov.hpp:53-58).

#include "blockfv/amg.hpp"
#include "blockfv/block_csr.hpp"
#include "blockfv/block_matrix.hpp"
#include "blockfv/engine.hpp"
#include "blockfv/euler.hpp"
#include "blockfv/incompressible.hpp"
#include "blockfv/krylov.hpp"
#include "blockfv/mesh.hpp"
#include "blockfv/partition.hpp"
#include "blockfv/preconditioner.hpp"

// the reference test suite's own fixtures (tests/support/test_helpers.hpp)
#include "support/test_helpers.hpp"

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

using namespace fvb;

namespace {

thread_local std::string g_err;

struct RefCfg {  // mirrors bcs_solver_config field order (include/bcs.h)
    int method;         // 0 GMRES, 1 BiCGStab
    int precond;        // 0 none, 1 LUSGS, 2 DILU, 3 AMG
    double relTol;
    double absTol;
    int maxIters;
    int gmresRestart;
    int amgMaxLevels;
    int amgMinCoarseRows;
    int amgPreSweeps;
    int amgPostSweeps;
};

struct RefReport {
    int iterations;
    int converged;
    int breakdown;
    int setupBranch;  // 1 when the pipeline took the setup branch
    double initialResidual;
    double finalResidual;
    double tConvert, tSetup, tReplace, tSolve, tRetrieve;
};

SolverConfig toCfg(const RefCfg* c) {
    SolverConfig s;
    s.method = c->method == 0 ? KrylovMethod::GMRES : KrylovMethod::PBiCGStab;
    s.preconditioner = static_cast<PrecondKind>(c->precond);
    s.relTol = c->relTol;
    s.absTol = c->absTol;
    s.maxIters = c->maxIters;
    s.gmresRestart = c->gmresRestart;
    s.amg.maxLevels = c->amgMaxLevels;
    s.amg.minCoarseRows = c->amgMinCoarseRows;
    s.amg.preSweeps = c->amgPreSweeps;
    s.amg.postSweeps = c->amgPostSweeps;
    return s;
}

// Topology-only mesh (owner < neighbour already) so a BlockLduMatrix can be
// built around caller-provided face addressing.
std::unique_ptr<Mesh> topoMesh(int nc, int nf, const int* owner, const int* neigh,
                               const double* centroids) {
    std::vector<double> vol(nc, 1.0);
    std::vector<Vec3> cen(nc);
    if (centroids)
        for (int c = 0; c < nc; ++c) cen[c] = {centroids[3 * c], centroids[3 * c + 1], centroids[3 * c + 2]};
    std::vector<InternalFace> faces(nf);
    for (int f = 0; f < nf; ++f) faces[f] = {owner[f], neigh[f], {1.0, 0.0, 0.0}, 0.5};
    return std::make_unique<Mesh>(Mesh::fromComponents(std::move(vol), std::move(cen), std::move(faces), {}, false));
}

std::vector<VariableDescriptor> varsFor(int n) {
    switch (n) {
        case 1: return {{"s", 1}};
        case 3: return {{"U", 3}};
        case 4: return {{"U", 3}, {"p", 1}};
        case 5: return {{"rhoU", 3}, {"rho", 1}, {"rhoE", 1}};
        default: break;
    }
    std::vector<VariableDescriptor> v;
    for (int i = 0; i < n; ++i) v.push_back({"s" + std::to_string(i), 1});
    return v;
}

void fillLdu(BlockLduMatrix& A, const double* diag, const double* upper, const double* lower) {
    const std::size_t nn = static_cast<std::size_t>(A.blockSize()) * A.blockSize();
    std::memcpy(A.diag(0), diag, sizeof(double) * nn * A.nCells());
    if (A.nFaces() > 0) {
        std::memcpy(A.upper(0), upper, sizeof(double) * nn * A.nFaces());
        std::memcpy(A.lower(0), lower, sizeof(double) * nn * A.nFaces());
    }
}

// --- synthetic hex mesh built with the reference Mesh type ---
// polySeed >= 0: the generator's polyhedral augmentation (csrc/gen/bcs_gen.cpp
// buildHex): a seeded 30% of the cells get a face to (i+1, j+1, k).
Mesh hexMesh(int nx, int ny, int nz, double aspect, long long scrambleSeed, PatchKind kind, long long polySeed = -1) {
    const double lx = 1.0, ly = 1.0 * ny / nx;
    const double hx = lx / nx, hy = ly / ny;
    const double hz = hx / aspect;
    const int nc = nx * ny * nz;
    std::vector<int> perm(nc);
    for (int c = 0; c < nc; ++c) perm[c] = c;
    if (scrambleSeed >= 0) {
        std::mt19937_64 rng(static_cast<std::uint64_t>(scrambleSeed));
        for (int i = nc - 1; i > 0; --i) {
            const int j = static_cast<int>(rng() % static_cast<std::uint64_t>(i + 1));
            std::swap(perm[i], perm[j]);
        }
    }
    auto id = [&](int i, int j, int k) { return perm[(k * ny + j) * nx + i]; };
    std::vector<double> vol(nc, hx * hy * hz);
    std::vector<Vec3> cen(nc);
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) cen[id(i, j, k)] = {(i + 0.5) * hx, (j + 0.5) * hy, (k + 0.5) * hz};
    std::vector<InternalFace> faces;
    std::mt19937_64 prng(static_cast<std::uint64_t>(polySeed >= 0 ? polySeed : 0));
    const double dl = std::sqrt(hx * hx + hy * hy);
    const double ds = 0.25 * hx * hz / dl;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                if (i + 1 < nx) faces.push_back({id(i, j, k), id(i + 1, j, k), {hy * hz, 0.0, 0.0}, 0.5});
                if (j + 1 < ny) faces.push_back({id(i, j, k), id(i, j + 1, k), {0.0, hx * hz, 0.0}, 0.5});
                if (k + 1 < nz) faces.push_back({id(i, j, k), id(i, j, k + 1), {0.0, 0.0, hx * hy}, 0.5});
                if (polySeed >= 0 && i + 1 < nx && j + 1 < ny && prng() % 10 < 3)
                    faces.push_back({id(i, j, k), id(i + 1, j + 1, k), {hx * ds, hy * ds, 0.0}, 0.5});
            }
    std::vector<BoundaryPatch> patches;
    BoundaryPatch p;
    p = {"xmin", kind, {}};
    for (int k = 0; k < nz; ++k) for (int j = 0; j < ny; ++j) p.faces.push_back({id(0, j, k), {-hy * hz, 0.0, 0.0}});
    patches.push_back(p);
    p = {"xmax", kind, {}};
    for (int k = 0; k < nz; ++k) for (int j = 0; j < ny; ++j) p.faces.push_back({id(nx - 1, j, k), {hy * hz, 0.0, 0.0}});
    patches.push_back(p);
    p = {"ymin", kind, {}};
    for (int k = 0; k < nz; ++k) for (int i = 0; i < nx; ++i) p.faces.push_back({id(i, 0, k), {0.0, -hx * hz, 0.0}});
    patches.push_back(p);
    p = {"ymax", kind, {}};
    for (int k = 0; k < nz; ++k) for (int i = 0; i < nx; ++i) p.faces.push_back({id(i, ny - 1, k), {0.0, hx * hz, 0.0}});
    patches.push_back(p);
    p = {"zmin", kind, {}};
    for (int j = 0; j < ny; ++j) for (int i = 0; i < nx; ++i) p.faces.push_back({id(i, j, 0), {0.0, 0.0, -hx * hy}});
    patches.push_back(p);
    p = {"zmax", kind, {}};
    for (int j = 0; j < ny; ++j) for (int i = 0; i < nx; ++i) p.faces.push_back({id(i, j, nz - 1), {0.0, 0.0, hx * hy}});
    patches.push_back(p);
    return Mesh::fromComponents(std::move(vol), std::move(cen), std::move(faces), std::move(patches), false);
}

void exportLdu(const BlockLduMatrix& A, const BlockVector& rhs, int* owner, int* neigh, double* diag,
               double* upper, double* lower, double* b, double* centroids) {
    const auto& m = A.mesh();
    for (int f = 0; f < A.nFaces(); ++f) {
        owner[f] = m.faces()[f].owner;
        neigh[f] = m.faces()[f].neighbour;
    }
    const std::size_t nn = static_cast<std::size_t>(A.blockSize()) * A.blockSize();
    std::memcpy(diag, A.diagValues().data(), sizeof(double) * nn * A.nCells());
    std::memcpy(upper, A.upperValues().data(), sizeof(double) * nn * A.nFaces());
    std::memcpy(lower, A.lowerValues().data(), sizeof(double) * nn * A.nFaces());
    std::memcpy(b, rhs.values.data(), sizeof(double) * rhs.values.size());
    if (centroids)
        for (int c = 0; c < A.nCells(); ++c) {
            centroids[3 * c] = m.cellCentroids()[c].x;
            centroids[3 * c + 1] = m.cellCentroids()[c].y;
            centroids[3 * c + 2] = m.cellCentroids()[c].z;
        }
}

// Replays the reference GMRES / BiCGStab residual recurrences on the dot
// stream: returns relative residuals per Arnoldi step.
struct DotTape {
    std::vector<double> v;
};

void replayGmres(const std::vector<double>& d, const SolverConfig& cfg, std::vector<double>& hist) {
    // d[0] = ||r0||^2; then per Arnoldi step j: (j+1) dots <w,v_i>, then ||w||^2;
    // at every restart/exit one ||b-Ax||^2.
    std::size_t p = 0;
    const double beta0 = std::sqrt(d[p++]);
    const double tol = std::max(cfg.relTol * beta0, cfg.absTol);
    if (beta0 <= tol) return;
    const int m = cfg.gmresRestart;
    double beta = beta0;
    int total = 0;
    while (p < d.size() && total < cfg.maxIters) {
        std::vector<std::vector<double>> H(m + 1, std::vector<double>(m, 0.0));
        std::vector<double> cs(m), sn(m), g(m + 1, 0.0);
        g[0] = beta;
        int j = 0;
        for (; j < m && total < cfg.maxIters; ++j, ++total) {
            for (int i = 0; i <= j; ++i) H[i][j] = d[p++];
            H[j + 1][j] = std::sqrt(d[p++]);
            const bool happy = !(H[j + 1][j] > 1e-290);
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * H[i][j] + sn[i] * H[i + 1][j];
                H[i + 1][j] = -sn[i] * H[i][j] + cs[i] * H[i + 1][j];
                H[i][j] = t;
            }
            const double den = std::hypot(H[j][j], H[j + 1][j]);
            cs[j] = den > 0.0 ? H[j][j] / den : 1.0;
            sn[j] = den > 0.0 ? H[j + 1][j] / den : 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            hist.push_back(std::fabs(g[j + 1]) / beta0);
            if (std::fabs(g[j + 1]) <= tol || happy) { ++j; ++total; break; }
        }
        if (p >= d.size()) break;
        beta = std::sqrt(d[p++]);  // true residual at restart / exit
        hist.back() = beta / beta0;  // the reference reports the true residual here
        if (beta <= tol) break;
    }
}

void replayBicgstab(const std::vector<double>& d, const SolverConfig& cfg, std::vector<double>& hist) {
    std::size_t p = 0;
    const double beta0 = std::sqrt(d[p++]);
    const double tol = std::max(cfg.relTol * beta0, cfg.absTol);
    if (beta0 <= tol) return;
    // per iteration: rhat.r, rhat.v, s.s, [t.t, (t.s), r.r]; the tape ends with
    // the final ||b-Ax||^2, so every read is bounds-checked.
    while (p + 3 < d.size()) {
        p += 2;  // rho, rhat.v
        const double ns = std::sqrt(d[p++]);
        if (ns <= tol) { hist.push_back(ns / beta0); break; }
        const double tt = d[p++];
        if (tt > 0.0) ++p;
        if (p + 1 >= d.size()) break;
        const double nr = std::sqrt(d[p++]);
        hist.push_back(nr / beta0);
        if (nr <= tol) break;
    }
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

struct AmgDump {
    std::vector<BlockCsrMatrix> A;
    std::vector<std::vector<int>> agg;
};

} // namespace

void fillReport(const SolveReport& r, RefReport* rep) {
    auto t = [&](const char* k) {
        const auto it = r.timings.find(k);
        return it == r.timings.end() ? 0.0 : it->second;
    };
    rep->iterations = r.iterations;
    rep->converged = r.converged;
    rep->breakdown = r.breakdown;
    rep->initialResidual = r.initialResidual;
    rep->finalResidual = r.finalResidual;
    rep->tConvert = t("convert");
    rep->tSetup = t("setup");
    rep->tReplace = t("replace");
    rep->tSolve = t("solve");
    rep->tRetrieve = t("retrieve");
    rep->setupBranch = (r.timings.count("setup") && r.timings.at("setup") > 0.0) ? 1 : 0;
}

// A persistent SolvePipeline over one system (bench: per-call wall times of
// the setup branch, then of replace-branch calls, engine.cpp:85-98)
struct PipeHandle {
    std::unique_ptr<Mesh> mesh;
    std::unique_ptr<BlockLduMatrix> A;
    BlockVector b, x0;
    SolvePipeline pipe;
    PipeHandle(int nc, int n) : b(nc, n), x0(nc, n) {}
};

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_hex_sizes(int nx, int ny, int nz, int* nCells, int* nFaces, int* nBoundary) {
    *nCells = nx * ny * nz;
    *nFaces = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1);
    *nBoundary = 2 * (ny * nz + nx * nz + nx * ny);
}

// 5x5 density-based system: assembleJacobian (euler.cpp:390-455) on the
// synthetic hex mesh, Roe, cfl 50; patchKinds (6 ints in the PatchKind
// order, for xmin xmax ymin ymax zmin zmax) go through
// EulerCase::patchOverride, nullptr = all farfield; recon 0 first order,
// 1 MUSCL without limiter, 2 MUSCL + Barth-Jespersen; flux in FluxScheme order.
int ref_gen_euler_kinds(int nx, int ny, int nz, double aspect, long long scrambleSeed, long long polySeed,
                        const int* patchKinds, int recon, int flux, int* owner, int* neigh, double* diag, double* upper, double* lower,
                        double* rhs, double* centroids) {
    return guard([&] {
        const Mesh mesh = hexMesh(nx, ny, nz, aspect, scrambleSeed, PatchKind::farfield, polySeed);
        EulerCase ec;
        if (patchKinds) {
            const char* names[6] = {"xmin", "xmax", "ymin", "ymax", "zmin", "zmax"};
            for (int p = 0; p < 6; ++p) ec.patchOverride[names[p]] = static_cast<PatchKind>(patchKinds[p]);
        }
        ec.flux = static_cast<FluxScheme>(flux);
        ec.recon.firstOrder = recon == 0;
        ec.recon.limiter = recon == 1 ? Limiter::none : Limiter::BarthJespersen;
        ec.freestream = {1.0, 0.5, 0.1, 0.0, 1.0 / 1.4};
        std::mt19937 gen(2);
        std::uniform_real_distribution<double> U(-0.05, 0.05);
        std::vector<PrimState> q(mesh.nCells());
        for (auto& s : q) {
            const double d0 = U(gen);
            const double d1 = U(gen);
            const double d2 = U(gen);
            const double d4 = U(gen);
            s = {1.0 * (1.0 + d0), 0.5 + d1, 0.1 + d2, 0.0, (1.0 / 1.4) * (1.0 + d4)};
        }
        auto [A, b] = assembleJacobian(q, mesh, ec, 50.0);
        exportLdu(A, b, owner, neigh, diag, upper, lower, rhs, centroids);
    });
}

int ref_gen_euler_poly(int nx, int ny, int nz, double aspect, long long scrambleSeed, long long polySeed, int* owner,
                       int* neigh, double* diag, double* upper, double* lower, double* rhs, double* centroids) {
    return ref_gen_euler_kinds(nx, ny, nz, aspect, scrambleSeed, polySeed, nullptr, 0, 0, owner, neigh, diag, upper, lower,
                               rhs, centroids);
}

// 4x4 pressure-based coupled system (incompressible.cpp:143-264): lid-driven
// box, nu 0.01, zmax moving wall u=(1,0,0), pressure pinned in cell 0.
int ref_gen_coupled_poly(int nx, int ny, int nz, double aspect, long long scrambleSeed, long long polySeed,
                         int* owner, int* neigh, double* diag, double* upper, double* lower, double* rhs, double* x0,
                         double* centroids) {
    return guard([&] {
        const Mesh mesh = hexMesh(nx, ny, nz, aspect, scrambleSeed, PatchKind::wall, polySeed);
        BcMap bcs;
        for (const char* nm : {"xmin", "xmax", "ymin", "ymax", "zmin"}) bcs[nm] = {IncompressibleBc::Kind::wall, {}, 0.0};
        bcs["zmax"] = {IncompressibleBc::Kind::movingWall, {1.0, 0.0, 0.0}, 0.0};
        BlockVector state(mesh.nCells(), 4);
        std::mt19937 gen(1);
        std::uniform_real_distribution<double> U(-0.1, 0.1);
        for (double& v : state.values) v = U(gen);
        const FaceFluxField phi0(mesh.nInternalFaces(), 0.0);
        const std::vector<double> a = momentumDiagCoeff(state, phi0, mesh, 0.01, bcs);
        std::vector<double> D(mesh.nCells());
        for (int i = 0; i < mesh.nCells(); ++i) D[i] = mesh.cellVolumes()[i] / a[i];
        const FaceFluxField phi = rhieChowFlux(state, mesh, D);
        auto [A, b] = assembleCoupled(state, phi, mesh, 0.01, bcs);
        pinPressure(A, b, 0, 0.0);
        exportLdu(A, b, owner, neigh, diag, upper, lower, rhs, centroids);
        std::memcpy(x0, state.values.data(), sizeof(double) * state.values.size());
    });
}

// the same coupled system with one IncompressibleBc per hex patch (xmin xmax
// ymin ymax zmin zmax): kinds (Kind order), u (3 per patch), p (per patch);
// pinCell < 0: no pinPressure; phiOut: the Rhie-Chow face fluxes assembled with.
int ref_gen_coupled_bcs(int nx, int ny, int nz, double aspect, long long scrambleSeed, long long polySeed,
                        const int* kinds, const double* u, const double* p, int pinCell, int* owner, int* neigh,
                        double* diag, double* upper, double* lower, double* rhs, double* x0, double* centroids,
                        double* phiOut) {
    return guard([&] {
        const Mesh mesh = hexMesh(nx, ny, nz, aspect, scrambleSeed, PatchKind::wall, polySeed);
        BcMap bcs;
        const char* names[6] = {"xmin", "xmax", "ymin", "ymax", "zmin", "zmax"};
        for (int q = 0; q < 6; ++q)
            bcs[names[q]] = {static_cast<IncompressibleBc::Kind>(kinds[q]), {u[3 * q], u[3 * q + 1], u[3 * q + 2]}, p[q]};
        BlockVector state(mesh.nCells(), 4);
        std::mt19937 gen(1);
        std::uniform_real_distribution<double> U(-0.1, 0.1);
        for (double& v : state.values) v = U(gen);
        const FaceFluxField phi0(mesh.nInternalFaces(), 0.0);
        const std::vector<double> a = momentumDiagCoeff(state, phi0, mesh, 0.01, bcs);
        std::vector<double> D(mesh.nCells());
        for (int i = 0; i < mesh.nCells(); ++i) D[i] = mesh.cellVolumes()[i] / a[i];
        const FaceFluxField phi = rhieChowFlux(state, mesh, D);
        auto [A, b] = assembleCoupled(state, phi, mesh, 0.01, bcs);
        if (pinCell >= 0) pinPressure(A, b, pinCell, 0.0);
        exportLdu(A, b, owner, neigh, diag, upper, lower, rhs, centroids);
        std::memcpy(x0, state.values.data(), sizeof(double) * state.values.size());
        std::memcpy(phiOut, phi.data(), sizeof(double) * phi.size());
    });
}

int ref_gen_euler(int nx, int ny, int nz, double aspect, long long scrambleSeed, int* owner, int* neigh,
                  double* diag, double* upper, double* lower, double* rhs, double* centroids) {
    return ref_gen_euler_poly(nx, ny, nz, aspect, scrambleSeed, -1, owner, neigh, diag, upper, lower, rhs, centroids);
}
int ref_gen_coupled(int nx, int ny, int nz, double aspect, long long scrambleSeed, int* owner, int* neigh,
                    double* diag, double* upper, double* lower, double* rhs, double* x0, double* centroids) {
    return ref_gen_coupled_poly(nx, ny, nz, aspect, scrambleSeed, -1, owner, neigh, diag, upper, lower, rhs, x0,
                                centroids);
}

// testsup::randomize (tests/support/test_helpers.hpp:47-70) on caller topology.
int ref_randomize(int nc, int nf, int n, const int* owner, const int* neigh, unsigned seed, double diagBoost,
                  double* diag, double* upper, double* lower) {
    return guard([&] {
        const auto mesh = topoMesh(nc, nf, owner, neigh, nullptr);
        BlockLduMatrix A(*mesh, varsFor(n));
        std::mt19937 rng(seed);
        testsup::randomize(A, rng, diagBoost);
        const std::size_t nn = static_cast<std::size_t>(n) * n;
        std::memcpy(diag, A.diagValues().data(), sizeof(double) * nn * nc);
        if (nf) {
            std::memcpy(upper, A.upperValues().data(), sizeof(double) * nn * nf);
            std::memcpy(lower, A.lowerValues().data(), sizeof(double) * nn * nf);
        }
    });
}

// testsup::randomVector (tests/support/test_helpers.hpp:72-77)
void ref_random_vector(int nc, int n, unsigned seed, double* out) {
    std::mt19937 rng(seed);
    const BlockVector v = testsup::randomVector(nc, n, rng);
    std::memcpy(out, v.values.data(), sizeof(double) * v.values.size());
}

// Reference mesh generators (mesh.cpp:99-165): sizes first, then addressing.
int ref_mesh_2d(int nx, int ny, double lx, double ly, int* nCells, int* nFaces, int* owner, int* neigh,
                double* centroids) {
    return guard([&] {
        const Mesh m = generateStructured2d(nx, ny, {lx, ly, 1.0});
        *nCells = m.nCells();
        *nFaces = m.nInternalFaces();
        if (owner)
            for (int f = 0; f < m.nInternalFaces(); ++f) {
                owner[f] = m.faces()[f].owner;
                neigh[f] = m.faces()[f].neighbour;
            }
        if (centroids)
            for (int c = 0; c < m.nCells(); ++c) {
                centroids[3 * c] = m.cellCentroids()[c].x;
                centroids[3 * c + 1] = m.cellCentroids()[c].y;
                centroids[3 * c + 2] = m.cellCentroids()[c].z;
            }
    });
}
int ref_mesh_tube(int n, double length, int* nCells, int* nFaces, int* owner, int* neigh, double* centroids) {
    return guard([&] {
        const Mesh m = generate1dTube(n, length);
        *nCells = m.nCells();
        *nFaces = m.nInternalFaces();
        if (owner)
            for (int f = 0; f < m.nInternalFaces(); ++f) {
                owner[f] = m.faces()[f].owner;
                neigh[f] = m.faces()[f].neighbour;
            }
        if (centroids)
            for (int c = 0; c < m.nCells(); ++c) {
                centroids[3 * c] = m.cellCentroids()[c].x;
                centroids[3 * c + 1] = m.cellCentroids()[c].y;
                centroids[3 * c + 2] = m.cellCentroids()[c].z;
            }
    });
}

unsigned long long ref_signature(int nc, int nf, const int* owner, const int* neigh) {
    const auto mesh = topoMesh(nc, nf, owner, neigh, nullptr);
    BlockLduMatrix A(*mesh, varsFor(1));
    return topologySignature(A);
}

// lduToBlockCsr (block_csr.cpp:97-109). cols/vals sized by nnz = nc + 2 nf.
int ref_csr(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag, const double* upper,
            const double* lower, int* rowOffsets, int* cols, double* vals) {
    return guard([&] {
        const auto mesh = topoMesh(nc, nf, owner, neigh, nullptr);
        BlockLduMatrix A(*mesh, varsFor(n));
        fillLdu(A, diag, upper, lower);
        const BlockCsrMatrix csr = lduToBlockCsr(A);
        std::memcpy(rowOffsets, csr.rowOffsets.data(), sizeof(int) * (nc + 1));
        std::memcpy(cols, csr.colIndices.data(), sizeof(int) * csr.nnz());
        std::memcpy(vals, csr.values.data(), sizeof(double) * csr.values.size());
    });
}

// y = A x via csrMatvec (block_csr.cpp:129-137) and via blockMatvec (LDU).
int ref_matvec(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag, const double* upper,
               const double* lower, const double* x, double* yCsr, double* yLdu) {
    return guard([&] {
        const auto mesh = topoMesh(nc, nf, owner, neigh, nullptr);
        BlockLduMatrix A(*mesh, varsFor(n));
        fillLdu(A, diag, upper, lower);
        const BlockCsrMatrix csr = lduToBlockCsr(A);
        csrMatvec(csr, x, yCsr);
        if (yLdu) blockMatvec(A, x, yLdu);
    });
}

// One application z = M^{-1} r of the reference preconditioner (engine.cpp:21-29).
int ref_precond_apply(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
                      const double* upper, const double* lower, const RefCfg* cfg, const double* r, double* z) {
    return guard([&] {
        const auto mesh = topoMesh(nc, nf, owner, neigh, nullptr);
        BlockLduMatrix A(*mesh, varsFor(n));
        fillLdu(A, diag, upper, lower);
        const BlockCsrMatrix csr = lduToBlockCsr(A);
        const auto M = makeCsrPreconditioner(csr, toCfg(cfg));
        M->apply(r, z);
    });
}

// SolvePipeline::solve (engine.cpp:47-120), EngineCsr backend (backend=1) or
// HostLdu (backend=0). `calls` >= 1 repeats the call on one pipeline (first
// call = setup branch, later calls = replace branch); the report is the last.
// hist (optional): per-iteration relative residual replayed from the dot
// stream of an equivalent solveCsr-style run.
int ref_solve(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
              const double* upper, const double* lower, const double* b, const double* x0, int backend,
              const RefCfg* cfg, int calls, double* x, RefReport* rep, double* hist, int histCap, int* histN) {
    return guard([&] {
        const auto mesh = topoMesh(nc, nf, owner, neigh, nullptr);
        BlockLduMatrix A(*mesh, varsFor(n));
        fillLdu(A, diag, upper, lower);
        BlockVector bv(nc, n), xv(nc, n);
        std::memcpy(bv.values.data(), b, sizeof(double) * bv.values.size());
        std::memcpy(xv.values.data(), x0, sizeof(double) * xv.values.size());
        const SolverConfig scfg = toCfg(cfg);
        // calls == 0 (with a history buffer): only the instrumented run below,
        // which is solveCsr (engine.cpp:31-45) with a recording dot; its
        // report and solution are returned (halves the cost at 128^3)
        if (calls > 0) {
            SolvePipeline pipe;
            std::pair<BlockVector, SolveReport> out;
            for (int c = 0; c < calls; ++c)
                out = pipe.solve(A, bv, xv, backend == 0 ? Backend::HostLdu : Backend::EngineCsr, scfg);
            std::memcpy(x, out.first.values.data(), sizeof(double) * out.first.values.size());
            fillReport(out.second, rep);
        } else if (!(hist && histN)) {
            throw std::invalid_argument("ref_solve: calls == 0 needs a history buffer");
        }
        if (hist && histN) {
            // the operators of the requested backend: EngineCsr = solveCsr's
            // (engine.cpp:31-45), HostLdu = blockMatvec + LduLusgsPrecond (:54-72)
            const BlockCsrMatrix csr = lduToBlockCsr(A);
            std::unique_ptr<Preconditioner> M;
            if (backend == 0) {
                if (scfg.preconditioner == PrecondKind::LUSGS) M = std::make_unique<LduLusgsPrecond>(A);
            } else {
                M = makeCsrPreconditioner(csr, scfg);
            }
            DotTape tape;
            KrylovOps ops;
            ops.size = static_cast<std::size_t>(nc) * n;
            if (backend == 0) ops.applyA = [&A](const double* in, double* o) { blockMatvec(A, in, o); };
            else ops.applyA = [&csr](const double* in, double* o) { csrMatvec(csr, in, o); };
            if (M) ops.applyM = [&M](const double* rr, double* zz) { M->apply(rr, zz); };
            ops.dot = [&tape, &ops](const double* a, const double* bb) {
                double s = 0.0;
                for (std::size_t i = 0; i < ops.size; ++i) s += a[i] * bb[i];
                tape.v.push_back(s);
                return s;
            };
            std::vector<double> xx(x0, x0 + ops.size);
            try {
                const SolveReport r = krylovSolve(ops, b, xx.data(), scfg);
                if (calls == 0) {
                    fillReport(r, rep);
                    std::memcpy(x, xx.data(), sizeof(double) * xx.size());
                }
            } catch (const std::runtime_error&) {
                if (calls == 0) throw;
            }
            std::vector<double> h;
            if (scfg.method == KrylovMethod::GMRES) replayGmres(tape.v, scfg, h);
            else replayBicgstab(tape.v, scfg, h);
            *histN = static_cast<int>(h.size());
            for (int i = 0; i < std::min(histCap, *histN); ++i) hist[i] = h[i];
        }
    });
}

void* ref_pipe_new(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
                   const double* upper, const double* lower, const double* b, const double* x0) {
    try {
        auto h = std::make_unique<PipeHandle>(nc, n);
        h->mesh = topoMesh(nc, nf, owner, neigh, nullptr);
        h->A = std::make_unique<BlockLduMatrix>(*h->mesh, varsFor(n));
        fillLdu(*h->A, diag, upper, lower);
        std::memcpy(h->b.values.data(), b, sizeof(double) * h->b.values.size());
        std::memcpy(h->x0.values.data(), x0, sizeof(double) * h->x0.values.size());
        return h.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// one SolvePipeline::solve call; *wall = its wall time (seconds)
int ref_pipe_solve(void* hp, int backend, const RefCfg* cfg, double* x, RefReport* rep, double* wall) {
    return guard([&] {
        auto* h = static_cast<PipeHandle*>(hp);
        const SolverConfig scfg = toCfg(cfg);
        const auto t0 = std::chrono::steady_clock::now();
        auto out = h->pipe.solve(*h->A, h->b, h->x0, backend == 0 ? Backend::HostLdu : Backend::EngineCsr, scfg);
        *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (x) std::memcpy(x, out.first.values.data(), sizeof(double) * out.first.values.size());
        fillReport(out.second, rep);
    });
}

void ref_pipe_free(void* h) { delete static_cast<PipeHandle*>(h); }

// AMG hierarchy dump (amg.cpp:73-105): handle API.
void* ref_amg_build(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
                    const double* upper, const double* lower, int maxLevels, int minCoarseRows) {
    AmgDump* d = nullptr;
    const int rc = guard([&] {
        const auto mesh = topoMesh(nc, nf, owner, neigh, nullptr);
        BlockLduMatrix A(*mesh, varsFor(n));
        fillLdu(A, diag, upper, lower);
        const BlockCsrMatrix csr = lduToBlockCsr(A);
        AmgConfig cfg;
        cfg.maxLevels = maxLevels;
        cfg.minCoarseRows = minCoarseRows;
        AmgHierarchy h(csr, cfg);
        auto* out = new AmgDump;
        for (int l = 0; l < h.depth(); ++l) {
            out->A.push_back(h.level(l).A);
            out->agg.push_back(h.level(l).aggregate);
        }
        d = out;
    });
    return rc == 0 ? d : nullptr;
}
int ref_amg_depth(void* h) { return static_cast<int>(static_cast<AmgDump*>(h)->A.size()); }
void ref_amg_level_sizes(void* h, int l, int* rows, int* nnz, int* aggLen) {
    auto* d = static_cast<AmgDump*>(h);
    *rows = d->A[l].nRows;
    *nnz = d->A[l].nnz();
    *aggLen = static_cast<int>(d->agg[l].size());
}
void ref_amg_level_get(void* h, int l, int* rowOffsets, int* cols, double* vals, int* agg) {
    auto* d = static_cast<AmgDump*>(h);
    const BlockCsrMatrix& A = d->A[l];
    if (rowOffsets) std::memcpy(rowOffsets, A.rowOffsets.data(), sizeof(int) * (A.nRows + 1));
    if (cols) std::memcpy(cols, A.colIndices.data(), sizeof(int) * A.nnz());
    if (vals) std::memcpy(vals, A.values.data(), sizeof(double) * A.values.size());
    if (agg && !d->agg[l].empty()) std::memcpy(agg, d->agg[l].data(), sizeof(int) * d->agg[l].size());
}
void ref_amg_free(void* h) { delete static_cast<AmgDump*>(h); }

// pairwiseAggregate on a BSR matrix given directly (amg.cpp:10-37).
int ref_aggregate_csr(int rows, int n, const int* rowOffsets, const int* cols, const double* vals, int* agg,
                      int* nCoarse) {
    return guard([&] {
        BlockCsrMatrix A;
        A.nRows = rows;
        A.blockSize = n;
        A.rowOffsets.assign(rowOffsets, rowOffsets + rows + 1);
        A.colIndices.assign(cols, cols + rowOffsets[rows]);
        A.values.assign(vals, vals + static_cast<std::size_t>(rowOffsets[rows]) * n * n);
        const std::vector<int> a = pairwiseAggregate(A, *nCoarse);
        std::memcpy(agg, a.data(), sizeof(int) * rows);
    });
}

// --- partition layer (partition.cpp) -------------------------------------
int ref_decompose(int nc, const double* centroids, int nRanks, int* cellToRank, int* rankRowOffset,
                  int* oldToNew) {
    return guard([&] {
        std::vector<double> vol(nc, 1.0);
        std::vector<Vec3> cen(nc);
        for (int c = 0; c < nc; ++c) cen[c] = {centroids[3 * c], centroids[3 * c + 1], centroids[3 * c + 2]};
        const Mesh m = Mesh::fromComponents(std::move(vol), std::move(cen), {}, {}, false);
        const Decomposition d = decompose(m, nRanks);
        std::memcpy(cellToRank, d.cellToRank.data(), sizeof(int) * nc);
        std::memcpy(rankRowOffset, d.rankRowOffset.data(), sizeof(int) * (nRanks + 1));
        std::memcpy(oldToNew, d.oldToNewRow.data(), sizeof(int) * nc);
    });
}

// Partition + consolidation dump. Returns per-engine local BSR sizes and halo
// entries through a handle.
struct PartDump {
    std::vector<MatrixPartition> parts;
};
void* ref_partition(int nc, int nf, int n, const int* owner, const int* neigh, const double* centroids,
                    const double* diag, const double* upper, const double* lower, int nRanks, int nEngines) {
    PartDump* out = nullptr;
    guard([&] {
        auto mesh = topoMesh(nc, nf, owner, neigh, centroids);
        BlockLduMatrix A(*mesh, varsFor(n));
        fillLdu(A, diag, upper, lower);
        const Decomposition dec = decompose(*mesh, nRanks);
        auto parts = buildPartitioned(A, dec);
        auto* d = new PartDump;
        if (nEngines > 0) {
            const ConsolidationPlan plan = makeConsolidationPlan(dec, nEngines);
            d->parts = consolidate(parts, plan, dec);
        } else {
            d->parts = std::move(parts);
        }
        out = d;
    });
    return out;
}
int ref_part_count(void* h) { return static_cast<int>(static_cast<PartDump*>(h)->parts.size()); }
void ref_part_sizes(void* h, int p, int* rowStart, int* rowEnd, int* nnz, int* nHalo, int* nSend) {
    const MatrixPartition& m = static_cast<PartDump*>(h)->parts[p];
    *rowStart = m.rowStart;
    *rowEnd = m.rowEnd;
    *nnz = m.local.nnz();
    *nHalo = m.halo.count();
    *nSend = static_cast<int>(m.sendPlan.size());
}
void ref_part_get(void* h, int p, int* rowOffsets, int* cols, double* vals, int* haloRow, int* haloCol,
                  int* haloPeer, double* haloVals, int* sendPeer, int* sendRow) {
    const MatrixPartition& m = static_cast<PartDump*>(h)->parts[p];
    std::memcpy(rowOffsets, m.local.rowOffsets.data(), sizeof(int) * (m.local.nRows + 1));
    std::memcpy(cols, m.local.colIndices.data(), sizeof(int) * m.local.nnz());
    std::memcpy(vals, m.local.values.data(), sizeof(double) * m.local.values.size());
    const int nb = m.local.blockSize * m.local.blockSize;
    for (int i = 0; i < m.halo.count(); ++i) {
        haloRow[i] = m.halo.entries[i].localRow;
        haloCol[i] = m.halo.entries[i].globalCol;
        haloPeer[i] = m.halo.entries[i].peerRank;
        std::memcpy(haloVals + static_cast<std::size_t>(i) * nb, m.halo.entries[i].block.data(), sizeof(double) * nb);
    }
    for (std::size_t i = 0; i < m.sendPlan.size(); ++i) {
        sendPeer[i] = m.sendPlan[i].first;
        sendRow[i] = m.sendPlan[i].second;
    }
}
void ref_part_free(void* h) { delete static_cast<PartDump*>(h); }

// distributedSolve (partition.cpp:370-479) with ranks = nRanks, engines = nEngines.
// b, x0, x are in the ORIGINAL cell order.
int ref_distributed_solve(int nc, int nf, int n, const int* owner, const int* neigh, const double* centroids,
                          const double* diag, const double* upper, const double* lower, const double* b,
                          const double* x0, int nRanks, int nEngines, const RefCfg* cfg, double* x,
                          RefReport* rep) {
    return guard([&] {
        auto mesh = topoMesh(nc, nf, owner, neigh, centroids);
        BlockLduMatrix A(*mesh, varsFor(n));
        fillLdu(A, diag, upper, lower);
        const Decomposition dec = decompose(*mesh, nRanks);
        const auto parts = buildPartitioned(A, dec);
        const ConsolidationPlan plan = makeConsolidationPlan(dec, nEngines);
        BlockVector bv(nc, n), xv(nc, n);
        std::memcpy(bv.values.data(), b, sizeof(double) * bv.values.size());
        std::memcpy(xv.values.data(), x0, sizeof(double) * xv.values.size());
        MailboxNetwork net;
        auto [xs, r] = distributedSolve(parts, scatterVector(bv, dec, n), scatterVector(xv, dec, n), toCfg(cfg),
                                        plan, dec, net);
        const BlockVector xo = gatherVector(xs, dec, n);
        std::memcpy(x, xo.values.data(), sizeof(double) * xo.values.size());
        rep->iterations = r.iterations;
        rep->converged = r.converged;
        rep->breakdown = r.breakdown;
        rep->initialResidual = r.initialResidual;
        rep->finalResidual = r.finalResidual;
        rep->tConvert = r.timings["convert"];
        rep->tSetup = r.timings["setup"];
        rep->tSolve = r.timings["solve"];
        rep->tRetrieve = r.timings["retrieve"];
    });
}

} // extern "C"
