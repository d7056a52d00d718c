// Synthetic workload generator: 3-D hex meshes (natural,
// scrambled, anisotropic) and the two block systems the hot path solves.
//
//   * 5x5 density-based Jacobian  — restates euler.cpp:390-455
//     (assembleJacobian: first-order approximate Jacobian, Roe-averaged
//     spectral radius, pseudo-time diagonal) and its RHS, the steady residual
//     euler.cpp:361-389 with the Roe flux euler.cpp:116-150.
//   * 4x4 pressure-based coupled p-U system — restates incompressible.cpp:
//     momentumDiagCoeff :57-89, pressureGradients :91-126, rhieChowFlux
//     :128-141, assembleCoupled :143-250, pinPressure :252-264.
//
// This is NOT the hot path (the matrix producers are out of scope);
// it is the input side of the benchmark.  It reproduces the reference
// producers bit for bit (same operation order, no FMA contraction: built with
// -ffp-contract=off), which tests/test_generator.py checks against the
// reference compiled in oracle/_ref.  Layouts are the reference's: int32
// owner/neighbour per internal face (owner < neighbour), row-major n x n
// blocks per cell/face, AoS vectors.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "../euler_jac.cuh"

namespace {

using namespace bcs_euler;

struct BFace {
    int cell;
    V3 area;  // outward
};

// Hex box: cells (k*ny + j)*nx + i before the optional scramble permutation.
struct Hex {
    int nc = 0;
    std::vector<int> owner, neigh;
    std::vector<V3> area;
    std::vector<double> fx;
    std::vector<double> vol;
    std::vector<V3> cen;
    std::vector<std::vector<BFace>> patches;  // xmin xmax ymin ymax zmin zmax
};

// Polyhedral augmentation: with polySeed >= 0 a seeded 30%
// of the cells (i, j, k) with i + 1 < nx, j + 1 < ny also get a face to their
// edge-diagonal neighbour (i+1, j+1, k), area h_x h_z / 4 along the centroid
// delta, emitted after the cell's +z face.  Draw: mt19937_64(polySeed)() % 10 < 3.
inline bool polyPick(std::mt19937_64& prng) { return prng() % 10 < 3; }

Hex buildHex(int nx, int ny, int nz, double aspect, long long scrambleSeed, long long polySeed = -1) {
    Hex h;
    const double lx = 1.0, ly = 1.0 * ny / nx;
    const double hx = lx / nx, hy = ly / ny, hz = hx / aspect;
    h.nc = nx * ny * nz;
    std::vector<int> perm(h.nc);
    for (int c = 0; c < h.nc; ++c) perm[c] = c;
    if (scrambleSeed >= 0) {  // seeded Fisher-Yates on mt19937_64
        std::mt19937_64 rng(static_cast<std::uint64_t>(scrambleSeed));
        for (int i = h.nc - 1; i > 0; --i) {
            const int j = static_cast<int>(rng() % static_cast<std::uint64_t>(i + 1));
            std::swap(perm[i], perm[j]);
        }
    }
    auto id = [&](int i, int j, int k) { return perm[(k * ny + j) * nx + i]; };
    h.vol.assign(h.nc, hx * hy * hz);
    h.cen.resize(h.nc);
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) h.cen[id(i, j, k)] = {(i + 0.5) * hx, (j + 0.5) * hy, (k + 0.5) * hz};
    auto face = [&](int a, int b, V3 s) {
        if (a > b) {  // owner < neighbour convention (mesh.cpp:84-89)
            std::swap(a, b);
            s = {-s.x, -s.y, -s.z};
            h.fx.push_back(1.0 - 0.5);
        } else {
            h.fx.push_back(0.5);
        }
        h.owner.push_back(a);
        h.neigh.push_back(b);
        h.area.push_back(s);
    };
    std::mt19937_64 prng(static_cast<std::uint64_t>(polySeed >= 0 ? polySeed : 0));
    const double dl = std::sqrt(hx * hx + hy * hy);
    const double ds = 0.25 * hx * hz / dl;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                if (i + 1 < nx) face(id(i, j, k), id(i + 1, j, k), {hy * hz, 0.0, 0.0});
                if (j + 1 < ny) face(id(i, j, k), id(i, j + 1, k), {0.0, hx * hz, 0.0});
                if (k + 1 < nz) face(id(i, j, k), id(i, j, k + 1), {0.0, 0.0, hx * hy});
                if (polySeed >= 0 && i + 1 < nx && j + 1 < ny && polyPick(prng))
                    face(id(i, j, k), id(i + 1, j + 1, k), {hx * ds, hy * ds, 0.0});
            }
    h.patches.resize(6);
    for (int k = 0; k < nz; ++k) for (int j = 0; j < ny; ++j) h.patches[0].push_back({id(0, j, k), {-hy * hz, 0.0, 0.0}});
    for (int k = 0; k < nz; ++k) for (int j = 0; j < ny; ++j) h.patches[1].push_back({id(nx - 1, j, k), {hy * hz, 0.0, 0.0}});
    for (int k = 0; k < nz; ++k) for (int i = 0; i < nx; ++i) h.patches[2].push_back({id(i, 0, k), {0.0, -hx * hz, 0.0}});
    for (int k = 0; k < nz; ++k) for (int i = 0; i < nx; ++i) h.patches[3].push_back({id(i, ny - 1, k), {0.0, hx * hz, 0.0}});
    for (int j = 0; j < ny; ++j) for (int i = 0; i < nx; ++i) h.patches[4].push_back({id(i, j, 0), {0.0, 0.0, -hx * hy}});
    for (int j = 0; j < ny; ++j) for (int i = 0; i < nx; ++i) h.patches[5].push_back({id(i, j, nz - 1), {0.0, 0.0, hx * hy}});
    return h;
}

// dst(block order) += scale * J + lamScale * I
void accumulate(double* dst, double scale, const double* J, double lamScale) {
    for (int r = 0; r < 5; ++r)
        for (int c = 0; c < 5; ++c) dst[kSlot[r] * 5 + kSlot[c]] += scale * J[r * 5 + c] + (r == c ? lamScale : 0.0);
}

// the seeded primitive state of the 5x5 workload
std::vector<Prim> eulerState(int nc) {
    std::mt19937 gen(2);
    std::uniform_real_distribution<double> U(-0.05, 0.05);
    std::vector<Prim> q(nc);
    for (int c = 0; c < nc; ++c) {
        const double d0 = U(gen);
        const double d1 = U(gen);
        const double d2 = U(gen);
        const double d4 = U(gen);
        q[c] = {{1.0 * (1.0 + d0), 0.5 + d1, 0.1 + d2, 0.0, (1.0 / 1.4) * (1.0 + d4)}};
    }
    return q;
}

void euler(const Hex& h, double* diag, double* upper, double* lower, double* rhs) {
    const int nc = h.nc;
    const int nf = static_cast<int>(h.owner.size());
    const std::vector<Prim> q = eulerState(nc);
    const Prim farfield{{1.0, 0.5, 0.1, 0.0, 1.0 / 1.4}};
    std::memset(diag, 0, sizeof(double) * 25 * nc);
    std::memset(upper, 0, sizeof(double) * 25 * nf);
    std::memset(lower, 0, sizeof(double) * 25 * nf);
    std::vector<double> lamSum(nc, 0.0);
    double J[25];
    for (int f = 0; f < nf; ++f) {
        const int o = h.owner[f], nb = h.neigh[f];
        const double S = len3(h.area[f]);
        const V3 n = dvd(h.area[f], S);
        const RoeAvg a = roeAvg(q[o], q[nb]);
        const double lam = std::fabs(dot3(a.u, n)) + a.c;
        convJac(q[o], n, J);
        accumulate(diag + 25 * static_cast<std::size_t>(o), 0.5 * S, J, 0.5 * S * lam);
        accumulate(lower + 25 * static_cast<std::size_t>(f), -0.5 * S, J, -0.5 * S * lam);
        convJac(q[nb], n, J);
        accumulate(upper + 25 * static_cast<std::size_t>(f), 0.5 * S, J, -0.5 * S * lam);
        accumulate(diag + 25 * static_cast<std::size_t>(nb), -0.5 * S, J, 0.5 * S * lam);
        lamSum[o] += lam * S;
        lamSum[nb] += lam * S;
    }
    for (const auto& patch : h.patches)
        for (const BFace& bf : patch) {
            const double S = len3(bf.area);
            const V3 n = dvd(bf.area, S);
            const RoeAvg a = roeAvg(q[bf.cell], farfield);
            const double lam = std::fabs(dot3(a.u, n)) + a.c;
            convJac(q[bf.cell], n, J);
            accumulate(diag + 25 * static_cast<std::size_t>(bf.cell), 0.5 * S, J, 0.5 * S * lam);
            lamSum[bf.cell] += lam * S;
        }
    const double cfl = 50.0;
    for (int c = 0; c < nc; ++c) {
        const double vOverDtau = lamSum[c] / cfl;
        for (int r = 0; r < 5; ++r) diag[25 * static_cast<std::size_t>(c) + r * 5 + r] += vOverDtau;
    }
    // steady residual, natural component order, then permuted into the RHS
    std::vector<double> res(5 * static_cast<std::size_t>(nc), 0.0);
    double fl[5];
    for (int f = 0; f < nf; ++f) {
        const int o = h.owner[f], nb = h.neigh[f];
        const double S = len3(h.area[f]);
        const V3 n = dvd(h.area[f], S);
        roe(q[o], q[nb], n, fl);
        for (int k = 0; k < 5; ++k) {
            res[5 * static_cast<std::size_t>(o) + k] -= S * fl[k];
            res[5 * static_cast<std::size_t>(nb) + k] += S * fl[k];
        }
    }
    for (const auto& patch : h.patches)
        for (const BFace& bf : patch) {
            const double S = len3(bf.area);
            const V3 n = dvd(bf.area, S);
            roe(q[bf.cell], farfield, n, fl);
            for (int k = 0; k < 5; ++k) res[5 * static_cast<std::size_t>(bf.cell) + k] -= S * fl[k];
        }
    for (int c = 0; c < nc; ++c)
        for (int k = 0; k < 5; ++k) rhs[5 * static_cast<std::size_t>(c) + kSlot[k]] = res[5 * static_cast<std::size_t>(c) + k];
}

// -------------------------------------------------------- coupled p-U 4x4
std::vector<V3> lsqPressureGrad(const Hex& h, const std::vector<double>& s) {
    const int nc = h.nc;
    std::vector<double> G(9 * static_cast<std::size_t>(nc), 0.0);
    std::vector<V3> b(nc, V3{0.0, 0.0, 0.0});
    auto acc = [&](int i, int j) {
        lsqAccumulate(sub(h.cen[j], h.cen[i]), s[4 * static_cast<std::size_t>(j) + 3] - s[4 * static_cast<std::size_t>(i) + 3],
                      &G[9 * static_cast<std::size_t>(i)], b[i]);
    };
    for (std::size_t f = 0; f < h.owner.size(); ++f) {
        acc(h.owner[f], h.neigh[f]);
        acc(h.neigh[f], h.owner[f]);
    }
    std::vector<V3> g(nc);
    for (int i = 0; i < nc; ++i) g[i] = lsqFinish(&G[9 * static_cast<std::size_t>(i)], b[i]);
    return g;
}

// seeded coupled state (u, v, w, p per cell) and the Rhie-Chow face fluxes the
// workload assembles with: rhieChowFlux(state, D(momentumDiagCoeff(phi = 0)))
std::vector<double> coupledState(int nc) {
    std::vector<double> s(4 * static_cast<std::size_t>(nc));
    std::mt19937 gen(1);
    std::uniform_real_distribution<double> U(-0.1, 0.1);
    for (double& v : s) v = U(gen);
    return s;
}

struct Geo {
    double S, nd;
};
std::vector<Geo> faceGeo(const Hex& h) {
    std::vector<Geo> geo(h.owner.size());
    for (std::size_t f = 0; f < h.owner.size(); ++f) {
        const double S = len3(h.area[f]);
        const V3 n = dvd(h.area[f], S);
        geo[f] = {S, dot3(n, sub(h.cen[h.neigh[f]], h.cen[h.owner[f]]))};
    }
    return geo;
}

std::vector<double> coupledPhi(const Hex& h, const std::vector<double>& s, double nu) {
    const int nc = h.nc;
    const int nf = static_cast<int>(h.owner.size());
    const std::vector<Geo> geo = faceGeo(h);
    auto wallDist = [&](const BFace& bf) { return h.vol[bf.cell] / (2.0 * len3(bf.area)); };
    // momentum diagonal with phi = 0 (moving/static walls only contribute diffusion)
    std::vector<double> aP(nc, 0.0);
    for (int f = 0; f < nf; ++f) {
        const double gDiff = nu * geo[f].S / geo[f].nd;
        aP[h.owner[f]] += std::max(0.0, 0.0) + gDiff;
        aP[h.neigh[f]] += -std::min(0.0, 0.0) + gDiff;
    }
    for (const auto& patch : h.patches)
        for (const BFace& bf : patch) aP[bf.cell] += nu * len3(bf.area) / wallDist(bf);
    std::vector<double> D(nc);
    for (int i = 0; i < nc; ++i) D[i] = h.vol[i] / aP[i];
    const std::vector<V3> gp = lsqPressureGrad(h, s);
    auto Ucell = [&](int c) { return V3{s[4 * static_cast<std::size_t>(c)], s[4 * static_cast<std::size_t>(c) + 1], s[4 * static_cast<std::size_t>(c) + 2]}; };
    std::vector<double> phi(nf);
    for (int f = 0; f < nf; ++f) {
        const int o = h.owner[f], nb = h.neigh[f];
        const double fx = h.fx[f];
        const V3 uBar = add(scl(Ucell(o), fx), scl(Ucell(nb), 1.0 - fx));
        const double dBar = fx * D[o] + (1.0 - fx) * D[nb];
        const double dpc = (s[4 * static_cast<std::size_t>(nb) + 3] - s[4 * static_cast<std::size_t>(o) + 3]) / geo[f].nd;
        const V3 gpBar = add(scl(gp[o], fx), scl(gp[nb], 1.0 - fx));
        phi[f] = dot3(h.area[f], uBar) - dBar * (geo[f].S * dpc - dot3(h.area[f], gpBar));
    }
    return phi;
}

void coupled(const Hex& h, double* diag, double* upper, double* lower, double* rhs, double* x0) {
    const int nc = h.nc;
    const int nf = static_cast<int>(h.owner.size());
    const double nu = 0.01;
    const std::vector<double> s = coupledState(nc);
    std::memcpy(x0, s.data(), sizeof(double) * s.size());
    const std::vector<Geo> geo = faceGeo(h);
    auto wallDist = [&](const BFace& bf) { return h.vol[bf.cell] / (2.0 * len3(bf.area)); };
    const std::vector<double> phi = coupledPhi(h, s, nu);
    const std::vector<V3> gp = lsqPressureGrad(h, s);
    std::vector<double> D(nc);
    // assembleCoupled recomputes aP from the new fluxes
    std::vector<double> aP2(nc, 0.0);
    for (int f = 0; f < nf; ++f) {
        const double gDiff = nu * geo[f].S / geo[f].nd;
        aP2[h.owner[f]] += std::max(phi[f], 0.0) + gDiff;
        aP2[h.neigh[f]] += -std::min(phi[f], 0.0) + gDiff;
    }
    for (const auto& patch : h.patches)
        for (const BFace& bf : patch) aP2[bf.cell] += nu * len3(bf.area) / wallDist(bf);
    for (int i = 0; i < nc; ++i) D[i] = h.vol[i] / aP2[i];
    // (pressure gradients of the unchanged state are recomputed identically)
    std::memset(diag, 0, sizeof(double) * 16 * nc);
    std::memset(upper, 0, sizeof(double) * 16 * nf);
    std::memset(lower, 0, sizeof(double) * 16 * nf);
    std::memset(rhs, 0, sizeof(double) * 4 * nc);
    constexpr int P = 3;
    for (int f = 0; f < nf; ++f) {
        const int o = h.owner[f], nb = h.neigh[f];
        const double fx = h.fx[f];
        const double gDiff = nu * geo[f].S / geo[f].nd;
        const V3 Sf = h.area[f];
        const double dBar = fx * D[o] + (1.0 - fx) * D[nb];
        const double cc = dBar * geo[f].S / geo[f].nd;
        double* dO = diag + 16 * static_cast<std::size_t>(o);
        double* dN = diag + 16 * static_cast<std::size_t>(nb);
        double* up = upper + 16 * static_cast<std::size_t>(f);
        double* lo = lower + 16 * static_cast<std::size_t>(f);
        for (int r = 0; r < 3; ++r) {
            const double sr = comp(Sf, r);
            dO[r * 4 + r] += std::max(phi[f], 0.0) + gDiff;
            up[r * 4 + r] += std::min(phi[f], 0.0) - gDiff;
            dN[r * 4 + r] += -std::min(phi[f], 0.0) + gDiff;
            lo[r * 4 + r] += -std::max(phi[f], 0.0) - gDiff;
            dO[r * 4 + P] += fx * sr;
            up[r * 4 + P] += (1.0 - fx) * sr;
            dN[r * 4 + P] -= (1.0 - fx) * sr;
            lo[r * 4 + P] -= fx * sr;
            dO[P * 4 + r] -= fx * sr;
            up[P * 4 + r] -= (1.0 - fx) * sr;
            dN[P * 4 + r] += (1.0 - fx) * sr;
            lo[P * 4 + r] += fx * sr;
        }
        dO[P * 4 + P] -= cc;
        up[P * 4 + P] += cc;
        dN[P * 4 + P] -= cc;
        lo[P * 4 + P] += cc;
        const V3 gpBar = add(scl(gp[o], fx), scl(gp[nb], 1.0 - fx));
        const double e = dBar * dot3(Sf, gpBar);
        rhs[4 * static_cast<std::size_t>(o) + P] += e;
        rhs[4 * static_cast<std::size_t>(nb) + P] -= e;
    }
    const V3 lid{1.0, 0.0, 0.0}, still{0.0, 0.0, 0.0};
    for (int p = 0; p < 6; ++p) {
        const V3 ub = p == 5 ? lid : still;
        for (const BFace& bf : h.patches[p]) {
            const double S = len3(bf.area);
            const double gb = nu * S / wallDist(bf);
            double* dP = diag + 16 * static_cast<std::size_t>(bf.cell);
            for (int r = 0; r < 3; ++r) {
                dP[r * 4 + r] += gb;
                rhs[4 * static_cast<std::size_t>(bf.cell) + r] += gb * comp(ub, r);
                dP[r * 4 + P] += comp(bf.area, r);
            }
        }
    }
    // pin p in cell 0
    double* d0 = diag;
    for (int c = 0; c < 4; ++c) d0[P * 4 + c] = 0.0;
    d0[P * 4 + P] = 1.0;
    for (int f = 0; f < nf; ++f) {
        if (h.owner[f] == 0)
            for (int c = 0; c < 4; ++c) upper[16 * static_cast<std::size_t>(f) + P * 4 + c] = 0.0;
        if (h.neigh[f] == 0)
            for (int c = 0; c < 4; ++c) lower[16 * static_cast<std::size_t>(f) + P * 4 + c] = 0.0;
    }
    rhs[P] = 0.0;
}

void exportTopo(const Hex& h, int* owner, int* neigh, double* centroids) {
    std::memcpy(owner, h.owner.data(), sizeof(int) * h.owner.size());
    std::memcpy(neigh, h.neigh.data(), sizeof(int) * h.neigh.size());
    if (centroids)
        for (int c = 0; c < h.nc; ++c) {
            centroids[3 * c] = h.cen[c].x;
            centroids[3 * c + 1] = h.cen[c].y;
            centroids[3 * c + 2] = h.cen[c].z;
        }
}

} // namespace

extern "C" {

void bcsgen_hex_sizes(int nx, int ny, int nz, int* nCells, int* nFaces) {
    *nCells = nx * ny * nz;
    *nFaces = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1);
}

// sizes with the polyhedral augmentation of polySeed (< 0: plain hex)
void bcsgen_hex_sizes_poly(int nx, int ny, int nz, long long polySeed, int* nCells, int* nFaces) {
    bcsgen_hex_sizes(nx, ny, nz, nCells, nFaces);
    if (polySeed < 0) return;
    std::mt19937_64 prng(static_cast<std::uint64_t>(polySeed));
    int extra = 0;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i)
                if (i + 1 < nx && j + 1 < ny && polyPick(prng)) ++extra;
    *nFaces += extra;
}

// 5x5 density-based system. scrambleSeed < 0 keeps natural order; polySeed < 0: plain hex.
int bcsgen_hex_euler_poly(int nx, int ny, int nz, double aspect, long long scrambleSeed, long long polySeed,
                          int* owner, int* neigh, double* diag, double* upper, double* lower, double* rhs,
                          double* centroids) {
    if (nx < 1 || ny < 1 || nz < 1 || !(aspect > 0.0)) return 1;
    const Hex h = buildHex(nx, ny, nz, aspect, scrambleSeed, polySeed);
    exportTopo(h, owner, neigh, centroids);
    euler(h, diag, upper, lower, rhs);
    return 0;
}

// 4x4 pressure-based coupled system; x0 = the seeded state.
int bcsgen_hex_coupled_poly(int nx, int ny, int nz, double aspect, long long scrambleSeed, long long polySeed,
                            int* owner, int* neigh, double* diag, double* upper, double* lower, double* rhs,
                            double* x0, double* centroids) {
    if (nx < 1 || ny < 1 || nz < 1 || !(aspect > 0.0)) return 1;
    const Hex h = buildHex(nx, ny, nz, aspect, scrambleSeed, polySeed);
    exportTopo(h, owner, neigh, centroids);
    coupled(h, diag, upper, lower, rhs, x0);
    return 0;
}

// inputs of the 5x5 assembly on the same mesh: face area vectors (3 per
// internal face), boundary faces in patch order (cell, area vector; all
// farfield), the seeded primitive state q (5 per cell: rho, u, v, w, p)
void bcsgen_hex_boundary_count(int nx, int ny, int nz, int* nb) { *nb = 2 * (ny * nz + nx * nz + nx * ny); }
int bcsgen_hex_euler_inputs(int nx, int ny, int nz, double aspect, long long scrambleSeed, long long polySeed,
                            double* faceArea, int* bcell, double* barea, double* q) {
    if (nx < 1 || ny < 1 || nz < 1 || !(aspect > 0.0)) return 1;
    const Hex h = buildHex(nx, ny, nz, aspect, scrambleSeed, polySeed);
    for (std::size_t f = 0; f < h.area.size(); ++f) {
        faceArea[3 * f] = h.area[f].x;
        faceArea[3 * f + 1] = h.area[f].y;
        faceArea[3 * f + 2] = h.area[f].z;
    }
    std::size_t b = 0;
    for (const auto& patch : h.patches)
        for (const BFace& bf : patch) {
            bcell[b] = bf.cell;
            barea[3 * b] = bf.area.x;
            barea[3 * b + 1] = bf.area.y;
            barea[3 * b + 2] = bf.area.z;
            ++b;
        }
    const std::vector<Prim> st = eulerState(h.nc);
    for (int c = 0; c < h.nc; ++c)
        for (int k = 0; k < 5; ++k) q[5 * static_cast<std::size_t>(c) + k] = st[c].v[k];
    return 0;
}

// inputs of the 4x4 assembleCoupled on the same mesh: face area vectors and
// interpolation weights, cell volumes and centroids, boundary faces in patch
// order (cell, area, kind 0 wall / 1 moving wall, wall velocity), the seeded
// state (u, v, w, p per cell) and the Rhie-Chow face fluxes phi
int bcsgen_hex_coupled_inputs(int nx, int ny, int nz, double aspect, long long scrambleSeed, long long polySeed,
                              double* faceArea, double* fx, double* vol, double* cen, int* bcell, double* barea,
                              int* bkind, double* bu, double* state, double* phi) {
    if (nx < 1 || ny < 1 || nz < 1 || !(aspect > 0.0)) return 1;
    const Hex h = buildHex(nx, ny, nz, aspect, scrambleSeed, polySeed);
    for (std::size_t f = 0; f < h.area.size(); ++f) {
        faceArea[3 * f] = h.area[f].x;
        faceArea[3 * f + 1] = h.area[f].y;
        faceArea[3 * f + 2] = h.area[f].z;
        fx[f] = h.fx[f];
    }
    for (int c = 0; c < h.nc; ++c) {
        vol[c] = h.vol[c];
        cen[3 * c] = h.cen[c].x;
        cen[3 * c + 1] = h.cen[c].y;
        cen[3 * c + 2] = h.cen[c].z;
    }
    std::size_t b = 0;
    for (int p = 0; p < 6; ++p)
        for (const BFace& bf : h.patches[p]) {
            bcell[b] = bf.cell;
            barea[3 * b] = bf.area.x;
            barea[3 * b + 1] = bf.area.y;
            barea[3 * b + 2] = bf.area.z;
            bkind[b] = p == 5 ? 1 : 0;  // zmax: the moving lid
            bu[3 * b] = p == 5 ? 1.0 : 0.0;
            bu[3 * b + 1] = 0.0;
            bu[3 * b + 2] = 0.0;
            ++b;
        }
    const std::vector<double> s = coupledState(h.nc);
    std::memcpy(state, s.data(), sizeof(double) * s.size());
    const std::vector<double> ph = coupledPhi(h, s, 0.01);
    std::memcpy(phi, ph.data(), sizeof(double) * ph.size());
    return 0;
}

int bcsgen_hex_euler(int nx, int ny, int nz, double aspect, long long scrambleSeed, int* owner, int* neigh,
                     double* diag, double* upper, double* lower, double* rhs, double* centroids) {
    return bcsgen_hex_euler_poly(nx, ny, nz, aspect, scrambleSeed, -1, owner, neigh, diag, upper, lower, rhs,
                                 centroids);
}

int bcsgen_hex_coupled(int nx, int ny, int nz, double aspect, long long scrambleSeed, int* owner, int* neigh,
                       double* diag, double* upper, double* lower, double* rhs, double* x0, double* centroids) {
    return bcsgen_hex_coupled_poly(nx, ny, nz, aspect, scrambleSeed, -1, owner, neigh, diag, upper, lower, rhs, x0,
                                   centroids);
}

} // extern "C"
