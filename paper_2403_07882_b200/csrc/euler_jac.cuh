// Euler 5x5 building blocks shared by the host workload generator
// (csrc/gen/bcs_gen.cpp) and the device assembly (k_assemble.cu), so both
// evaluate the same expression trees: Roe average, physical flux, convective
// Jacobian and Roe flux of the reference (euler.cpp:44-150), restated.
// Compile without FMA contraction (host -ffp-contract=off, device
// -fmad=false): sqrt and division are IEEE on both sides.
#pragma once
#include <cmath>

#ifdef __CUDACC__
#define BCS_HD __host__ __device__ __forceinline__
#else
#define BCS_HD inline
#endif

namespace bcs_euler {

struct V3 {
    double x, y, z;
};
BCS_HD V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
BCS_HD V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
BCS_HD V3 scl(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
BCS_HD V3 dvd(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
BCS_HD double dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
BCS_HD double len3(V3 a) { return sqrt(dot3(a, a)); }
BCS_HD double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

// ---------------------------------------------------------------- Euler 5x5
constexpr double kGamma = 1.4;
// natural component [rho, m, E] -> block slot in the vector-first layout
constexpr int kSlot[5] = {3, 0, 1, 2, 4};

struct Prim {
    double v[5];  // rho, ux, uy, uz, p
};
BCS_HD V3 vel(const Prim& q) { return {q.v[1], q.v[2], q.v[3]}; }

struct RoeAvg {
    double rho;
    V3 u;
    double H, c;
};

BCS_HD RoeAvg roeAvg(const Prim& L, const Prim& R) {
    const double sL = sqrt(L.v[0]), sR = sqrt(R.v[0]);
    const double w = 1.0 / (sL + sR);
    RoeAvg a;
    a.rho = sL * sR;
    a.u = scl(add(scl(vel(L), sL), scl(vel(R), sR)), w);
    const double HL = kGamma / (kGamma - 1.0) * L.v[4] / L.v[0] + 0.5 * dot3(vel(L), vel(L));
    const double HR = kGamma / (kGamma - 1.0) * R.v[4] / R.v[0] + 0.5 * dot3(vel(R), vel(R));
    a.H = (sL * HL + sR * HR) * w;
    a.c = sqrt((kGamma - 1.0) * (a.H - 0.5 * dot3(a.u, a.u)));
    return a;
}

BCS_HD void physFlux(const Prim& q, V3 n, double* f) {
    const V3 u = vel(q);
    const double un = dot3(u, n);
    const double rhoE = q.v[4] / (kGamma - 1.0) + 0.5 * q.v[0] * dot3(u, u);
    f[0] = q.v[0] * un;
    f[1] = q.v[0] * u.x * un + q.v[4] * n.x;
    f[2] = q.v[0] * u.y * un + q.v[4] * n.y;
    f[3] = q.v[0] * u.z * un + q.v[4] * n.z;
    f[4] = (rhoE + q.v[4]) * un;
}

// convective Jacobian d(F.n)/dQ in [rho, m, E] order
BCS_HD void convJac(const Prim& q, V3 n, double* J) {
    const V3 u = vel(q);
    const double un = dot3(u, n);
    const double g1 = kGamma - 1.0;
    const double ek = 0.5 * dot3(u, u);
    const double c = sqrt(kGamma * q.v[4] / q.v[0]);
    const double H = c * c / g1 + ek;
    const double nv[3] = {n.x, n.y, n.z};
    const double uv[3] = {u.x, u.y, u.z};
    J[0] = 0.0;
    J[1] = nv[0];
    J[2] = nv[1];
    J[3] = nv[2];
    J[4] = 0.0;
    for (int i = 0; i < 3; ++i) {
        double* row = J + 5 * (i + 1);
        row[0] = g1 * ek * nv[i] - uv[i] * un;
        for (int j = 0; j < 3; ++j) row[1 + j] = uv[i] * nv[j] - g1 * uv[j] * nv[i] + (i == j ? un : 0.0);
        row[4] = g1 * nv[i];
    }
    double* e = J + 20;
    e[0] = (g1 * ek - H) * un;
    for (int j = 0; j < 3; ++j) e[1 + j] = H * nv[j] - g1 * uv[j] * un;
    e[4] = kGamma * un;
}

BCS_HD void roe(const Prim& L, const Prim& R, V3 n, double* flux) {
    double fL[5], fR[5];
    physFlux(L, n, fL);
    physFlux(R, n, fR);
    const RoeAvg a = roeAvg(L, R);
    const double un = dot3(a.u, n);
    const double c = a.c;
    const double dRho = R.v[0] - L.v[0];
    const V3 dU = sub(vel(R), vel(L));
    const double dUn = dot3(dU, n);
    const double dP = R.v[4] - L.v[4];
    const double a1 = (dP - a.rho * c * dUn) / (2.0 * c * c);
    const double a5 = (dP + a.rho * c * dUn) / (2.0 * c * c);
    const double a2 = dRho - dP / (c * c);
    const double delta = 0.1 * (fabs(un) + c);
    auto entropyFix = [delta](double lam) {
        const double m = fabs(lam);
        return m < delta ? (lam * lam + delta * delta) / (2.0 * delta) : m;
    };
    const double l1 = entropyFix(un - c);
    const double l2 = fabs(un);
    const double l5 = entropyFix(un + c);
    double diss[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    auto wave = [&](double strength, double lam, double k0, V3 kU, double kE) {
        const double w = strength * lam;
        diss[0] += w * k0;
        diss[1] += w * kU.x;
        diss[2] += w * kU.y;
        diss[3] += w * kU.z;
        diss[4] += w * kE;
    };
    wave(a1, l1, 1.0, sub(a.u, scl(n, c)), a.H - c * un);
    wave(a2, l2, 1.0, a.u, 0.5 * dot3(a.u, a.u));
    wave(a5, l5, 1.0, add(a.u, scl(n, c)), a.H + c * un);
    const V3 dUt = sub(dU, scl(n, dUn));
    wave(a.rho, l2, 0.0, dUt, dot3(a.u, dU) - un * dUn);
    for (int i = 0; i < 5; ++i) flux[i] = 0.5 * (fL[i] + fR[i]) - 0.5 * diss[i];
}


// ---- HLLC and Rusanov fluxes (euler.cpp:150-193), for FluxScheme::HLLC / Rusanov
BCS_HD double soundSpeed(const Prim& q) { return sqrt(kGamma * q.v[4] / q.v[0]); }

BCS_HD void primToCons(const Prim& q, double* Q) {
    const V3 u = vel(q);
    Q[0] = q.v[0];
    Q[1] = q.v[0] * u.x;
    Q[2] = q.v[0] * u.y;
    Q[3] = q.v[0] * u.z;
    Q[4] = q.v[4] / (kGamma - 1.0) + 0.5 * q.v[0] * dot3(u, u);
}

BCS_HD void hllc(const Prim& L, const Prim& R, V3 n, double* flux) {
    const double unL = dot3(vel(L), n), unR = dot3(vel(R), n);
    const double cL = soundSpeed(L), cR = soundSpeed(R);
    const RoeAvg a = roeAvg(L, R);
    const double unTilde = dot3(a.u, n);
    const double x1 = unL - cL, y1 = unTilde - a.c;
    const double sL = y1 < x1 ? y1 : x1;  // std::min
    const double x2 = unR + cR, y2 = unTilde + a.c;
    const double sR = x2 < y2 ? y2 : x2;  // std::max
    if (sL >= 0.0) { physFlux(L, n, flux); return; }
    if (sR <= 0.0) { physFlux(R, n, flux); return; }
    const double sStar = (R.v[4] - L.v[4] + L.v[0] * unL * (sL - unL) - R.v[0] * unR * (sR - unR)) /
                         (L.v[0] * (sL - unL) - R.v[0] * (sR - unR));
    const Prim& K = sStar >= 0.0 ? L : R;
    const double sK = sStar >= 0.0 ? sL : sR;
    const double unK = sStar >= 0.0 ? unL : unR;
    double QK[5], FK[5];
    primToCons(K, QK);
    physFlux(K, n, FK);
    const double fac = K.v[0] * (sK - unK) / (sK - sStar);
    double Qs[5];
    Qs[0] = fac;
    const V3 uStar = add(vel(K), scl(n, sStar - unK));
    Qs[1] = fac * uStar.x;
    Qs[2] = fac * uStar.y;
    Qs[3] = fac * uStar.z;
    Qs[4] = fac * (QK[4] / K.v[0] + (sStar - unK) * (sStar + K.v[4] / (K.v[0] * (sK - unK))));
    for (int i = 0; i < 5; ++i) flux[i] = FK[i] + sK * (Qs[i] - QK[i]);
}

BCS_HD void rusanov(const Prim& L, const Prim& R, V3 n, double* flux) {
    double fL[5], fR[5], QL[5], QR[5];
    physFlux(L, n, fL);
    physFlux(R, n, fR);
    primToCons(L, QL);
    primToCons(R, QR);
    const RoeAvg a = roeAvg(L, R);
    const double lam = fabs(dot3(a.u, n)) + a.c;
    for (int i = 0; i < 5; ++i) flux[i] = 0.5 * (fL[i] + fR[i]) - 0.5 * lam * (QR[i] - QL[i]);
}

// riemannFlux (euler.cpp:195-203): scheme 0 Roe, 1 HLLC, 2 Rusanov (FluxScheme order)
BCS_HD void riemann(int scheme, const Prim& L, const Prim& R, V3 n, double* flux) {
    if (scheme == 1) hllc(L, R, n, flux);
    else if (scheme == 2) rusanov(L, R, n, flux);
    else roe(L, R, n, flux);
}


// ---- coupled p-U building blocks (incompressible.cpp:91-126) --------------
// smallmat::luFactor + luSolve for a 3x3 (first max by strict >, no singular
// check: the caller regularises), in place
BCS_HD void lu3Solve(double* a, double* x) {
    int piv[3];
    for (int k = 0; k < 3; ++k) {
        int p = k;
        double best = fabs(a[k * 3 + k]);
        for (int i = k + 1; i < 3; ++i)
            if (fabs(a[i * 3 + k]) > best) {
                best = fabs(a[i * 3 + k]);
                p = i;
            }
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < 3; ++j) {
                const double t = a[k * 3 + j];
                a[k * 3 + j] = a[p * 3 + j];
                a[p * 3 + j] = t;
            }
        const double d = a[k * 3 + k];
        for (int i = k + 1; i < 3; ++i) {
            a[i * 3 + k] /= d;
            for (int j = k + 1; j < 3; ++j) a[i * 3 + j] -= a[i * 3 + k] * a[k * 3 + j];
        }
    }
    for (int k = 0; k < 3; ++k)
        if (piv[k] != k) {
            const double t = x[k];
            x[k] = x[piv[k]];
            x[piv[k]] = t;
        }
    for (int i = 1; i < 3; ++i)
        for (int j = 0; j < i; ++j) x[i] -= a[i * 3 + j] * x[j];
    for (int i = 2; i >= 0; --i) {
        for (int j = i + 1; j < 3; ++j) x[i] -= a[i * 3 + j] * x[j];
        x[i] /= a[i * 3 + i];
    }
}

// least-squares gradient term of neighbour j seen from cell i
// (pressureGradients' accumulate: G += w d d^T, b += d (w (p_j - p_i)))
BCS_HD void lsqAccumulate(V3 d, double pj_minus_pi, double* G, V3& b) {
    const double w = 1.0 / dot3(d, d);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) G[r * 3 + c] += w * comp(d, r) * comp(d, c);
    const double t = w * pj_minus_pi;
    b = add(b, scl(d, t));
}

// regularise degenerate directions and solve G g = b (pressureGradients' tail)
BCS_HD V3 lsqFinish(double* G, V3 b) {
    double rv[3] = {b.x, b.y, b.z};
    double scale = 0.0;
    for (int r = 0; r < 3; ++r) scale = scale < G[r * 3 + r] ? G[r * 3 + r] : scale;  // std::max
    for (int r = 0; r < 3; ++r)
        if (G[r * 3 + r] <= 1e-12 * scale) {
            for (int c = 0; c < 3; ++c) G[r * 3 + c] = G[c * 3 + r] = 0.0;
            G[r * 3 + r] = 1.0;
            rv[r] = 0.0;
        }
    lu3Solve(G, rv);
    return V3{rv[0], rv[1], rv[2]};
}

}  // namespace bcs_euler
