// Device-side assembly of the 5x5 density-based system:
// assembleJacobian (euler.cpp:390-455: first-order approximate Jacobian,
// Roe-averaged spectral radius, pseudo-time diagonal) and its right-hand side,
// the steady residual (computeResidual, euler.cpp:361-389, Roe flux :103-150)
// for first-order reconstruction and every boundary patch kind of the
// reference (ghostState, euler.cpp:320-341: wall/slip/symmetry reflect the
// velocity, inlet/farfield take the freestream, outlet the interior), written
// straight into the engine's block-CSR slots.  A caller then uploads the
// primitive state (5 doubles per cell) instead of the LDU values (50 doubles
// per face + 25 per cell).
//
// Same arithmetic as the reference: the face kernel writes the two
// off-diagonal blocks of a face (each is one contribution onto 0.0); the cell
// kernel accumulates a cell's diagonal block, spectral-radius sum and residual
// over its faces in face-index order, then its boundary faces in patch order,
// then V/dtau -- the order of the reference's loops.  The flux, Jacobian and
// Roe-average routines are the ones the host generator uses (euler_jac.cuh),
// compiled without FMA contraction, so the values are bit-identical.
#include "device.cuh"
#include "euler_jac.cuh"
#include "kernels.hpp"

namespace bcs {

namespace {

using bcs_euler::Prim;
using bcs_euler::RoeAvg;
using bcs_euler::V3;

// natural component [rho, m, E] -> block slot in the vector-first layout (euler.cpp:15)
__device__ __forceinline__ int kslot(int r) { return r == 0 ? 3 : (r == 4 ? 4 : r - 1); }

__device__ __forceinline__ Prim load_prim(const double* q, int c) {
    const double* p = q + 5 * static_cast<size_t>(c);
    return Prim{{p[0], p[1], p[2], p[3], p[4]}};
}
__device__ __forceinline__ V3 load_v3(const double* a, int i) {
    const double* p = a + 3 * static_cast<size_t>(i);
    return V3{p[0], p[1], p[2]};
}

__device__ __forceinline__ double maxd(double a, double b) { return a < b ? b : a; }  // std::max
__device__ __forceinline__ double mind(double a, double b) { return b < a ? b : a; }  // std::min

// ghost state across a boundary face (ghostState, euler.cpp:320-341); kind =
// the reference's PatchKind (0 wall, 1 inlet, 2 outlet, 3 farfield, 4 slip,
// 5 symmetry), validated on the host
__device__ __forceinline__ Prim ghost_state(const Prim& in, V3 n, int kind, const Prim& far) {
    if (kind == 1 || kind == 3) return far;
    if (kind == 2) return in;
    const V3 u{in.v[1], in.v[2], in.v[3]};
    const double s = 2.0 * bcs_euler::dot3(u, n);  // u - n * (2 dot(u, n))
    Prim g = in;
    g.v[1] = u.x - n.x * s;
    g.v[2] = u.y - n.y * s;
    g.v[3] = u.z - n.z * s;
    return g;
}

__global__ void k_inverse_src(int nnzb, const int* __restrict__ src, int* inv) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nnzb) inv[src[k]] = k;
}

// off-diagonal blocks of face f: lower (neighbour row, owner column) =
// -0.5 S J(q_o) - 0.5 S lam I, upper (owner row, neighbour column) =
// 0.5 S J(q_n) - 0.5 S lam I (euler.cpp:418-423)
constexpr int kAsmT = 128;  // threads (faces / cells) per assembly CTA

// Blocks staged in shared memory (already in the vector-first slot order)
// go out one 200-byte block per 25 consecutive lanes: coalesced stores of
// whole sectors instead of 32 scattered 8-byte stores per instruction
// (which cost ~30% extra DRAM write and read-for-ownership traffic).
template <int NN = 25>
__device__ __forceinline__ void flush_blocks(const double* st, const int* slot, int count, double* vals) {
    for (int e = threadIdx.x; e < NN * count; e += kAsmT) {
        const int b = e / NN;
        vals[NN * static_cast<size_t>(slot[b]) + (e - NN * b)] = st[e];
    }
}

__global__ void __launch_bounds__(kAsmT) k_asm_faces(int nc, int nf, const int* __restrict__ owner,
                                                     const int* __restrict__ neigh, const double* __restrict__ area,
                                                     const double* __restrict__ q, const int* __restrict__ inv,
                                                     double* vals) {
    __shared__ double st[25 * kAsmT];
    __shared__ int slot[kAsmT];
    const int f0 = blockIdx.x * kAsmT;
    const int f = f0 + threadIdx.x;
    const int count = min(kAsmT, nf - f0);
    const bool on = f < nf;
    double* my = st + 25 * threadIdx.x;
    Prim qo{}, qn{};
    V3 n{};
    double S = 0.0, lam = 0.0;
    double J[25];
    if (on) {
        const int o = owner[f], nb = neigh[f];
        const V3 A = load_v3(area, f);
        S = bcs_euler::len3(A);
        n = bcs_euler::dvd(A, S);
        qo = load_prim(q, o);
        qn = load_prim(q, nb);
        const RoeAvg a = bcs_euler::roeAvg(qo, qn);
        lam = fabs(bcs_euler::dot3(a.u, n)) + a.c;
        bcs_euler::convJac(qo, n, J);
        const double scale = -0.5 * S, lamScale = -0.5 * S * lam;
#pragma unroll
        for (int r = 0; r < 5; ++r)
#pragma unroll
            for (int c = 0; c < 5; ++c)
                my[kslot(r) * 5 + kslot(c)] = __dadd_rn(0.0, __dadd_rn(__dmul_rn(scale, J[r * 5 + c]), r == c ? lamScale : 0.0));
        slot[threadIdx.x] = inv[nc + nf + f];
    }
    __syncthreads();
    flush_blocks(st, slot, count, vals);
    __syncthreads();
    if (on) {
        bcs_euler::convJac(qn, n, J);
        const double scale = 0.5 * S, lamScale = -0.5 * S * lam;
#pragma unroll
        for (int r = 0; r < 5; ++r)
#pragma unroll
            for (int c = 0; c < 5; ++c)
                my[kslot(r) * 5 + kslot(c)] = __dadd_rn(0.0, __dadd_rn(__dmul_rn(scale, J[r * 5 + c]), r == c ? lamScale : 0.0));
        slot[threadIdx.x] = inv[nc + f];
    }
    __syncthreads();
    flush_blocks(st, slot, count, vals);
}

// ---- MUSCL reconstruction of the residual's face states (musclReconstruct,
// euler.cpp:236-312; primitiveGradients :205-234).  Per cell: least-squares
// gradients of the five primitives (G and the five right-hand sides summed
// over the cell's faces in face order, the order of the reference's
// accumulate loop), then the Barth-Jespersen factor (min/max are
// order-free).  Per face: the limited linear extrapolation from both sides,
// first order where the result is non-physical.  The Jacobian stays first
// order (assembleJacobian uses q itself); only computeResidual sees these.
__device__ __forceinline__ V3 face_centre(const double* cen, const double* fx, int f, int o, int nb) {
    const V3 co = load_v3(cen, o), cn = load_v3(cen, nb);  // Mesh::faceCentre (mesh.hpp:55-59)
    const double w = fx[f];
    return bcs_euler::add(bcs_euler::scl(co, w), bcs_euler::scl(cn, 1.0 - w));
}

__device__ __forceinline__ void mu_cell(int c, const int* __restrict__ owner, const int* __restrict__ neigh,
                                        const int* __restrict__ cfo, const int* __restrict__ cfl,
                                        const double* __restrict__ cen, const double* __restrict__ fx,
                                        const double* __restrict__ q, int limiter, double* grad, double* psi) {
    const Prim qc = load_prim(q, c);
    const V3 cc = load_v3(cen, c);
    double G[9];
    V3 b[5];
    Prim qmin = qc, qmax = qc;
#pragma unroll
    for (int e = 0; e < 9; ++e) G[e] = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) b[k] = V3{0.0, 0.0, 0.0};
    for (int e = cfo[c]; e < cfo[c + 1]; ++e) {
        const int f = cfl[e];
        const int j = owner[f] == c ? neigh[f] : owner[f];
        const Prim qj = load_prim(q, j);
        const V3 d = bcs_euler::sub(load_v3(cen, j), cc);
        const double w = 1.0 / bcs_euler::dot3(d, d);
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int cl = 0; cl < 3; ++cl) G[r * 3 + cl] += w * bcs_euler::comp(d, r) * bcs_euler::comp(d, cl);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            b[k] = bcs_euler::add(b[k], bcs_euler::scl(d, w * (qj.v[k] - qc.v[k])));
            qmin.v[k] = mind(qmin.v[k], qj.v[k]);
            qmax.v[k] = maxd(qmax.v[k], qj.v[k]);
        }
    }
    V3 g[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        double Gk[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) Gk[e] = G[e];
        g[k] = bcs_euler::lsqFinish(Gk, b[k]);  // same regularisation and LU for every component
        grad[3 * k] = g[k].x;
        grad[3 * k + 1] = g[k].y;
        grad[3 * k + 2] = g[k].z;
    }
    double ps[5] = {1.0, 1.0, 1.0, 1.0, 1.0};
    if (limiter == 1) {  // Barth-Jespersen (euler.cpp:262-283)
        for (int e = cfo[c]; e < cfo[c + 1]; ++e) {
            const int f = cfl[e];
            const V3 dx = bcs_euler::sub(face_centre(cen, fx, f, owner[f], neigh[f]), cc);
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const double d = bcs_euler::dot3(g[k], dx);
                double r = 1.0;
                if (d > 1e-300) r = (qmax.v[k] - qc.v[k]) / d;
                else if (d < -1e-300) r = (qmin.v[k] - qc.v[k]) / d;
                ps[k] = mind(ps[k], mind(1.0, r));
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) psi[k] = ps[k];
}

// gradients (15 per cell) and limiter factors (5 per cell) of kAsmT cells,
// staged in shared memory and stored as two contiguous runs
__global__ void __launch_bounds__(kAsmT, 4) k_mu_cells(int nc, const int* __restrict__ owner,
                                                    const int* __restrict__ neigh, const int* __restrict__ cfo,
                                                    const int* __restrict__ cfl, const double* __restrict__ cen,
                                                    const double* __restrict__ fx, const double* __restrict__ q,
                                                    int limiter, double* grad, double* psi) {
    __shared__ double sg[15 * kAsmT], sp[5 * kAsmT];
    const int c0 = blockIdx.x * kAsmT;
    const int c = c0 + threadIdx.x;
    const int count = min(kAsmT, nc - c0);
    if (c < nc) mu_cell(c, owner, neigh, cfo, cfl, cen, fx, q, limiter, sg + 15 * threadIdx.x, sp + 5 * threadIdx.x);
    __syncthreads();
    for (int e = threadIdx.x; e < 15 * count; e += kAsmT) grad[15 * static_cast<size_t>(c0) + e] = sg[e];
    for (int e = threadIdx.x; e < 5 * count; e += kAsmT) psi[5 * static_cast<size_t>(c0) + e] = sp[e];
}

__global__ void k_mu_faces(int nf, const int* __restrict__ owner, const int* __restrict__ neigh,
                           const double* __restrict__ cen, const double* __restrict__ fx, const double* __restrict__ q,
                           const double* __restrict__ grad, const double* __restrict__ psi, double* fsL, double* fsR) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const int o = owner[f], nb = neigh[f];
    const V3 xf = face_centre(cen, fx, f, o, nb);
    const V3 dL = bcs_euler::sub(xf, load_v3(cen, o)), dR = bcs_euler::sub(xf, load_v3(cen, nb));
    Prim L = load_prim(q, o), R = load_prim(q, nb);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        L.v[k] += psi[5 * static_cast<size_t>(o) + k] * bcs_euler::dot3(load_v3(grad, 5 * o + k), dL);
        R.v[k] += psi[5 * static_cast<size_t>(nb) + k] * bcs_euler::dot3(load_v3(grad, 5 * nb + k), dR);
    }
    if (!(L.v[0] > 0.0 && L.v[4] > 0.0) || !(R.v[0] > 0.0 && R.v[4] > 0.0)) {  // physical() (euler.hpp:29)
        L = load_prim(q, o);
        R = load_prim(q, nb);
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        fsL[5 * static_cast<size_t>(f) + k] = L.v[k];
        fsR[5 * static_cast<size_t>(f) + k] = R.v[k];
    }
}

// diagonal block, spectral-radius sum and residual of cell c
__device__ __forceinline__ void asm_cell(int c, int nf, const int* __restrict__ owner,
                                         const int* __restrict__ neigh, const double* __restrict__ area,
                                         const int* __restrict__ cfo, const int* __restrict__ cfl,
                                         const int* __restrict__ bco, const double* __restrict__ barea,
                                         const int* __restrict__ bkind, const double* __restrict__ fsL,
                                         const double* __restrict__ fsR, int scheme, const double* __restrict__ q,
                                         const double* __restrict__ qinf, double cfl_num, double* dst, double* rdst,
                                         int* firstBad) {
    const Prim qc = load_prim(q, c);
    if (!(qc.v[0] > 0.0 && qc.v[4] > 0.0)) atomicMin(firstBad, c);  // assembleJacobian's physical() check (euler.cpp:393-395)
    const Prim far = load_prim(qinf, 0);
    double D[25], res[5], J[25], fl[5];
#pragma unroll
    for (int e = 0; e < 25; ++e) D[e] = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) res[k] = 0.0;
    double lamSum = 0.0;
    for (int e = cfo[c]; e < cfo[c + 1]; ++e) {
        const int f = cfl[e];
        const int o = owner[f], nb = neigh[f];
        const bool own = o == c;
        const V3 A = load_v3(area, f);
        const double S = bcs_euler::len3(A);
        const V3 n = bcs_euler::dvd(A, S);
        const Prim qo = own ? qc : load_prim(q, o);
        const Prim qn = own ? load_prim(q, nb) : qc;
        const RoeAvg a = bcs_euler::roeAvg(qo, qn);
        const double lam = fabs(bcs_euler::dot3(a.u, n)) + a.c;
        // owner side: += 0.5 S J(q_o) + 0.5 S lam I; neighbour side: += -0.5 S J(q_n) + 0.5 S lam I
        bcs_euler::convJac(own ? qo : qn, n, J);
        const double scale = own ? 0.5 * S : -0.5 * S, lamScale = 0.5 * S * lam;
#pragma unroll
        for (int r = 0; r < 5; ++r)
#pragma unroll
            for (int cc = 0; cc < 5; ++cc)
                D[r * 5 + cc] = __dadd_rn(D[r * 5 + cc], __dadd_rn(__dmul_rn(scale, J[r * 5 + cc]), r == cc ? lamScale : 0.0));
        lamSum = __dadd_rn(lamSum, __dmul_rn(lam, S));
        if (fsL)  // second order: the reconstructed face states (computeResidual, euler.cpp:364-374)
            bcs_euler::riemann(scheme, load_prim(fsL, f), load_prim(fsR, f), n, fl);
        else
            bcs_euler::riemann(scheme, qo, qn, n, fl);
#pragma unroll
        for (int k = 0; k < 5; ++k) res[k] = own ? __dsub_rn(res[k], __dmul_rn(S, fl[k])) : __dadd_rn(res[k], __dmul_rn(S, fl[k]));
    }
    // boundary faces: ghost state frozen, only the interior half enters (euler.cpp:426-441)
    for (int b = bco[c]; b < bco[c + 1]; ++b) {
        const V3 A = load_v3(barea, b);
        const double S = bcs_euler::len3(A);
        const V3 n = bcs_euler::dvd(A, S);
        const Prim g = ghost_state(qc, n, bkind ? bkind[b] : 3, far);
        const RoeAvg a = bcs_euler::roeAvg(qc, g);
        const double lam = fabs(bcs_euler::dot3(a.u, n)) + a.c;
        bcs_euler::convJac(qc, n, J);
        const double scale = 0.5 * S, lamScale = 0.5 * S * lam;
#pragma unroll
        for (int r = 0; r < 5; ++r)
#pragma unroll
            for (int cc = 0; cc < 5; ++cc)
                D[r * 5 + cc] = __dadd_rn(D[r * 5 + cc], __dadd_rn(__dmul_rn(scale, J[r * 5 + cc]), r == cc ? lamScale : 0.0));
        lamSum = __dadd_rn(lamSum, __dmul_rn(lam, S));
        bcs_euler::riemann(scheme, qc, g, n, fl);
#pragma unroll
        for (int k = 0; k < 5; ++k) res[k] = __dsub_rn(res[k], __dmul_rn(S, fl[k]));
    }
    if (cfl_num > 0.0) {
        const double vOverDtau = __ddiv_rn(lamSum, cfl_num);  // V/dtau with dtau = cfl V / sum (euler.cpp:444-448)
#pragma unroll
        for (int r = 0; r < 5; ++r) D[r * 5 + r] = __dadd_rn(D[r * 5 + r], vOverDtau);
    }
#pragma unroll
    for (int r = 0; r < 5; ++r)
#pragma unroll
        for (int cc = 0; cc < 5; ++cc) dst[kslot(r) * 5 + kslot(cc)] = D[r * 5 + cc];
#pragma unroll
    for (int k = 0; k < 5; ++k) rdst[kslot(k)] = res[k];
}

// diagonal blocks and right-hand side of kAsmT consecutive cells, staged in
// shared memory and stored coalesced (the rhs of the CTA is one contiguous run)
__global__ void __launch_bounds__(kAsmT, 3) k_asm_cells(int nc, int nf, const int* __restrict__ owner,
                                                     const int* __restrict__ neigh, const double* __restrict__ area,
                                                     const int* __restrict__ cfo, const int* __restrict__ cfl,
                                                     const int* __restrict__ bco, const double* __restrict__ barea,
                                                     const int* __restrict__ bkind, const double* __restrict__ fsL,
                                                     const double* __restrict__ fsR, int scheme,
                                                     const double* __restrict__ q, const double* __restrict__ qinf,
                                                     double cfl_num, const int* __restrict__ inv, double* vals,
                                                     double* rhs, int* firstBad) {
    __shared__ double st[25 * kAsmT];
    __shared__ double rst[5 * kAsmT];
    __shared__ int slot[kAsmT];
    const int c0 = blockIdx.x * kAsmT;
    const int c = c0 + threadIdx.x;
    const int count = min(kAsmT, nc - c0);
    if (c < nc) {
        asm_cell(c, nf, owner, neigh, area, cfo, cfl, bco, barea, bkind, fsL, fsR, scheme, q, qinf, cfl_num,
                 st + 25 * threadIdx.x, rst + 5 * threadIdx.x, firstBad);
        slot[threadIdx.x] = inv[c];
    }
    __syncthreads();
    flush_blocks(st, slot, count, vals);
    for (int e = threadIdx.x; e < 5 * count; e += kAsmT) rhs[5 * static_cast<size_t>(c0) + e] = rst[e];
}


// ---- 4x4 pressure-based coupled p-U system (assembleCoupled,
// incompressible.cpp:143-250, + pinPressure :252-264) for wall / moving-wall
// patches: D = V / momentumDiagCoeff(state, phi) and the least-squares
// pressure gradient per cell, then the face blocks and the cell blocks.
constexpr int kP = 3;

struct CoupledGeom {
    const int *owner, *neigh, *cfo, *cf, *bco;
    const double *area, *fx, *vol, *cen, *barea, *bu;
    const int* bkind;   // IncompressibleBc::Kind per boundary face: 0 wall, 1 moving wall, 2 inlet, 3 outlet
    const double* bp;   // outlet pressure per boundary face
};

__global__ void k_cp_cellpre(int nc, CoupledGeom g, const double* __restrict__ phi, const double* __restrict__ state,
                             double nu, double* D, double* grad) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    double aP = 0.0, G[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) G[e] = 0.0;
    V3 b{0.0, 0.0, 0.0};
    const V3 cc = load_v3(g.cen, c);
    const double pc = state[4 * static_cast<size_t>(c) + kP];
    for (int e = g.cfo[c]; e < g.cfo[c + 1]; ++e) {
        const int f = g.cf[e];
        const int o = g.owner[f], nb = g.neigh[f];
        const bool own = o == c;
        const V3 A = load_v3(g.area, f);
        const double S = bcs_euler::len3(A);
        const V3 n = bcs_euler::dvd(A, S);
        const double nd = bcs_euler::dot3(n, bcs_euler::sub(load_v3(g.cen, nb), load_v3(g.cen, o)));
        const double gDiff = nu * S / nd;
        aP = __dadd_rn(aP, own ? __dadd_rn(maxd(phi[f], 0.0), gDiff) : __dadd_rn(-mind(phi[f], 0.0), gDiff));
        const int j = own ? nb : o;
        bcs_euler::lsqAccumulate(bcs_euler::sub(load_v3(g.cen, j), cc), state[4 * static_cast<size_t>(j) + kP] - pc, G, b);
    }
    for (int k = g.bco[c]; k < g.bco[c + 1]; ++k) {  // momentumDiagCoeff's patch terms (incompressible.cpp:70-86)
        const V3 A = load_v3(g.barea, k);
        const double S = bcs_euler::len3(A);
        const double db = g.vol[c] / (2.0 * bcs_euler::len3(A));
        const int kind = g.bkind[k];
        if (kind == 3) {  // outlet: outflow through the face
            const V3 uc{state[4 * static_cast<size_t>(c)], state[4 * static_cast<size_t>(c) + 1],
                        state[4 * static_cast<size_t>(c) + 2]};
            aP = __dadd_rn(aP, maxd(bcs_euler::dot3(A, uc), 0.0));
        } else if (kind == 2) {  // inlet: diffusion + inflow
            aP = __dadd_rn(aP, nu * S / db + maxd(bcs_euler::dot3(A, load_v3(g.bu, k)), 0.0));
        } else {  // walls: nu S / wallDistance
            aP = __dadd_rn(aP, nu * S / db);
        }
    }
    D[c] = g.vol[c] / aP;
    const V3 gr = bcs_euler::lsqFinish(G, b);
    grad[3 * static_cast<size_t>(c)] = gr.x;
    grad[3 * static_cast<size_t>(c) + 1] = gr.y;
    grad[3 * static_cast<size_t>(c) + 2] = gr.z;
}

__device__ __forceinline__ void cp_face(int f, CoupledGeom g, const double* __restrict__ phi,
                                        const double* __restrict__ D, double nu, int pin, double* up, double* lo) {
    const int o = g.owner[f], nb = g.neigh[f];
    const V3 A = load_v3(g.area, f);
    const double S = bcs_euler::len3(A);
    const V3 n = bcs_euler::dvd(A, S);
    const double nd = bcs_euler::dot3(n, bcs_euler::sub(load_v3(g.cen, nb), load_v3(g.cen, o)));
    const double gDiff = nu * S / nd;
    const double fx = g.fx[f];
    const double dBar = fx * D[o] + (1.0 - fx) * D[nb];
    const double c = dBar * S / nd;
#pragma unroll
    for (int e = 0; e < 16; ++e) up[e] = lo[e] = 0.0;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const double sr = bcs_euler::comp(A, r);
        up[r * 4 + r] += mind(phi[f], 0.0) - gDiff;
        lo[r * 4 + r] += -maxd(phi[f], 0.0) - gDiff;
        up[r * 4 + kP] += (1.0 - fx) * sr;
        lo[r * 4 + kP] -= fx * sr;
        up[kP * 4 + r] -= (1.0 - fx) * sr;
        lo[kP * 4 + r] += fx * sr;
    }
    up[kP * 4 + kP] += c;
    lo[kP * 4 + kP] += c;
    if (o == pin)
#pragma unroll
        for (int q = 0; q < 4; ++q) up[kP * 4 + q] = 0.0;
    if (nb == pin)
#pragma unroll
        for (int q = 0; q < 4; ++q) lo[kP * 4 + q] = 0.0;
}

// the two off-diagonal 4x4 blocks of kAsmT faces, staged and stored coalesced (flush_blocks)
__global__ void __launch_bounds__(kAsmT) k_cp_faces(int nc, int nf, CoupledGeom g, const double* __restrict__ phi,
                                                    const double* __restrict__ D, double nu, int pin,
                                                    const int* __restrict__ inv, double* vals) {
    __shared__ double su[16 * kAsmT], sl[16 * kAsmT];
    __shared__ int slotU[kAsmT], slotL[kAsmT];
    const int f0 = blockIdx.x * kAsmT;
    const int f = f0 + threadIdx.x;
    const int count = min(kAsmT, nf - f0);
    if (f < nf) {
        double up[16], lo[16];
        cp_face(f, g, phi, D, nu, pin, up, lo);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            su[16 * threadIdx.x + e] = up[e];
            sl[16 * threadIdx.x + e] = lo[e];
        }
        slotU[threadIdx.x] = inv[nc + f];
        slotL[threadIdx.x] = inv[nc + nf + f];
    }
    __syncthreads();
    flush_blocks<16>(su, slotU, count, vals);
    flush_blocks<16>(sl, slotL, count, vals);
}

__device__ __forceinline__ void cp_cell(int c, CoupledGeom g, const double* __restrict__ phi,
                                        const double* __restrict__ D, const double* __restrict__ grad,
                                        const double* __restrict__ state, double nu, int pin, double pinValue,
                                        double* dst, double* rdst) {
    double Dm[16], rr[4];
#pragma unroll
    for (int e = 0; e < 16; ++e) Dm[e] = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) rr[q] = 0.0;
    for (int e = g.cfo[c]; e < g.cfo[c + 1]; ++e) {
        const int f = g.cf[e];
        const int o = g.owner[f], nb = g.neigh[f];
        const bool own = o == c;
        const V3 A = load_v3(g.area, f);
        const double S = bcs_euler::len3(A);
        const V3 n = bcs_euler::dvd(A, S);
        const double nd = bcs_euler::dot3(n, bcs_euler::sub(load_v3(g.cen, nb), load_v3(g.cen, o)));
        const double gDiff = nu * S / nd;
        const double fx = g.fx[f];
        const double dBar = fx * D[o] + (1.0 - fx) * D[nb];
        const double cc = dBar * S / nd;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const double sr = bcs_euler::comp(A, r);
            if (own) {
                Dm[r * 4 + r] += maxd(phi[f], 0.0) + gDiff;
                Dm[r * 4 + kP] += fx * sr;
                Dm[kP * 4 + r] -= fx * sr;
            } else {
                Dm[r * 4 + r] += -mind(phi[f], 0.0) + gDiff;
                Dm[r * 4 + kP] -= (1.0 - fx) * sr;
                Dm[kP * 4 + r] += (1.0 - fx) * sr;
            }
        }
        Dm[kP * 4 + kP] -= cc;
        const V3 gpBar = bcs_euler::add(bcs_euler::scl(load_v3(grad, o), fx), bcs_euler::scl(load_v3(grad, nb), 1.0 - fx));
        const double ev = dBar * bcs_euler::dot3(A, gpBar);
        if (own) rr[kP] += ev;
        else rr[kP] -= ev;
    }
    for (int k = g.bco[c]; k < g.bco[c + 1]; ++k) {  // boundary patches (incompressible.cpp:203-247)
        const V3 A = load_v3(g.barea, k);
        const double S = bcs_euler::len3(A);
        const double db = g.vol[c] / (2.0 * bcs_euler::len3(A));
        const int kind = g.bkind[k];
        if (kind <= 1) {  // wall / moving wall
            const double gb = nu * S / db;
            const V3 u = load_v3(g.bu, k);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                Dm[r * 4 + r] += gb;
                rr[r] += gb * bcs_euler::comp(u, r);
                Dm[r * 4 + kP] += bcs_euler::comp(A, r);  // zero-gradient p
            }
        } else if (kind == 2) {  // inlet: fixed velocity, known flux
            const double gb = nu * S / db;
            const V3 u = load_v3(g.bu, k);
            const double phiB = bcs_euler::dot3(A, u);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                Dm[r * 4 + r] += gb + maxd(phiB, 0.0);
                rr[r] += gb * bcs_euler::comp(u, r) - mind(phiB, 0.0) * bcs_euler::comp(u, r);
                Dm[r * 4 + kP] += bcs_euler::comp(A, r);
            }
            rr[kP] += phiB;  // known flux, negated row
        } else {  // outlet: zero-gradient u, fixed pressure
            const V3 uc{state[4 * static_cast<size_t>(c)], state[4 * static_cast<size_t>(c) + 1],
                        state[4 * static_cast<size_t>(c) + 2]};
            const double phiB = bcs_euler::dot3(A, uc);
            const double cb = D[c] * S / db;
            const double pb = g.bp[k];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                Dm[r * 4 + r] += maxd(phiB, 0.0);
                rr[r] -= bcs_euler::comp(A, r) * pb;
                Dm[kP * 4 + r] -= bcs_euler::comp(A, r);
            }
            Dm[kP * 4 + kP] -= cb;
            rr[kP] -= cb * pb;
        }
    }
    if (c == pin) {
#pragma unroll
        for (int q = 0; q < 4; ++q) Dm[kP * 4 + q] = 0.0;
        Dm[kP * 4 + kP] = 1.0;
        rr[kP] = pinValue;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) dst[e] = Dm[e];
#pragma unroll
    for (int q = 0; q < 4; ++q) rdst[q] = rr[q];
}

// diagonal 4x4 blocks and right-hand side of kAsmT cells, staged and stored coalesced
__global__ void __launch_bounds__(kAsmT) k_cp_cells(int nc, CoupledGeom g, const double* __restrict__ phi,
                                                    const double* __restrict__ D, const double* __restrict__ grad,
                                                    const double* __restrict__ state, double nu, int pin, double pinValue, const int* __restrict__ inv,
                                                    double* vals, double* rhs) {
    __shared__ double st[16 * kAsmT], rst[4 * kAsmT];
    __shared__ int slot[kAsmT];
    const int c0 = blockIdx.x * kAsmT;
    const int c = c0 + threadIdx.x;
    const int count = min(kAsmT, nc - c0);
    if (c < nc) {
        cp_cell(c, g, phi, D, grad, state, nu, pin, pinValue, st + 16 * threadIdx.x, rst + 4 * threadIdx.x);
        slot[threadIdx.x] = inv[c];
    }
    __syncthreads();
    flush_blocks<16>(st, slot, count, vals);
    for (int e = threadIdx.x; e < 4 * count; e += kAsmT) rhs[4 * static_cast<size_t>(c0) + e] = rst[e];
}

}  // namespace

void assemble_inverse_src(int nnzb, const int* src, int* inv, cudaStream_t s) {
    if (nnzb <= 0) return;
    k_inverse_src<<<(nnzb + 255) / 256, 256, 0, s>>>(nnzb, src, inv);
    count_launch();
}

void assemble_euler_muscl(int nc, int nf, const int* owner, const int* neigh, const int* cfo, const int* cfl,
                          const double* cen, const double* fx, const double* q, int limiter, double* grad, double* psi,
                          double* fsL, double* fsR, cudaStream_t s) {
    k_mu_cells<<<(nc + kAsmT - 1) / kAsmT, kAsmT, 0, s>>>(nc, owner, neigh, cfo, cfl, cen, fx, q, limiter, grad, psi);
    if (nf > 0) k_mu_faces<<<(nf + 255) / 256, 256, 0, s>>>(nf, owner, neigh, cen, fx, q, grad, psi, fsL, fsR);
    count_launch(nf > 0 ? 2 : 1);
}

void assemble_euler(int nc, int nf, const int* owner, const int* neigh, const double* area, const int* cfo,
                    const int* cfl, const int* bco, const double* barea, const int* bkind, const double* fsL,
                    const double* fsR, int scheme, const double* q, const double* qinf, double cfl_num,
                    const int* inv, double* vals, double* rhs, int* firstBad, cudaStream_t s) {
    if (nf > 0) k_asm_faces<<<(nf + kAsmT - 1) / kAsmT, kAsmT, 0, s>>>(nc, nf, owner, neigh, area, q, inv, vals);
    k_asm_cells<<<(nc + kAsmT - 1) / kAsmT, kAsmT, 0, s>>>(nc, nf, owner, neigh, area, cfo, cfl, bco, barea, bkind, fsL, fsR,
                                                 scheme, q, qinf, cfl_num, inv, vals, rhs, firstBad);
    count_launch(nf > 0 ? 2 : 1);
}

void assemble_coupled(int nc, int nf, const int* owner, const int* neigh, const double* area, const double* fx,
                      const double* vol, const double* cen, const int* cfo, const int* cf, const int* bco,
                      const double* barea, const double* bu, const int* bkind, const double* bp,
                      const double* state, const double* phi, double nu, int pin, double pinValue, const int* inv,
                      double* D, double* grad, double* vals, double* rhs, cudaStream_t s) {
    const CoupledGeom g{owner, neigh, cfo, cf, bco, area, fx, vol, cen, barea, bu, bkind, bp};
    k_cp_cellpre<<<(nc + 127) / 128, 128, 0, s>>>(nc, g, phi, state, nu, D, grad);
    if (nf > 0) k_cp_faces<<<(nf + kAsmT - 1) / kAsmT, kAsmT, 0, s>>>(nc, nf, g, phi, D, nu, pin, inv, vals);
    k_cp_cells<<<(nc + kAsmT - 1) / kAsmT, kAsmT, 0, s>>>(nc, g, phi, D, grad, state, nu, pin, pinValue, inv, vals,
                                                        rhs);
    count_launch(nf > 0 ? 3 : 2);
}

}  // namespace bcs
