// K11 for large coarsest levels: blocked dense LU and solve, bit-identical to
// smallmat::denseFactor / denseSolve (smallmat.hpp:134-174).
//
// Scrambled (randomly permuted) inputs stall the pairwise aggregation and hit
// the 30-level cap with a coarsest level of ~5e-4 R rows:
// m = 5,000+ at 128^3.  The reference's right-looking LU updates every element
// with one rounded multiply and one rounded subtraction per elimination step,
// in step order.  A blocked schedule keeps that per-element sequence:
//   panel   columns [k0, k0+b): the reference steps k0..k0+b-1 restricted to the
//           panel (pivot search, row swap, multipliers, panel update);
//   laswp   the panel's row swaps applied, in order, to the other columns;
//   trsm    rows [k0, k0+b) right of the panel: a_ij -= l_ik u_kj, k ascending;
//   update  the trailing matrix: a_ij -= l_ik u_kj for k in the panel, ascending,
//           one rounded product and one rounded subtraction each.
// Every element therefore sees exactly the reference's operations in the
// reference's order; only the schedule across elements differs.
//
// Solve: forward substitution in the reference order has an O(m) critical
// path (the last subtraction of row i needs x_{i-1}); the backward one does
// not: x_i's first subtraction uses x_{i+1}, so its chain of m-i-1 rounded
// subtractions can only start when row i+1 is done — O(m^2/2) dependent FP64
// operations, inherent to the reference's order.  One thread runs that chain
// while the other warps of the CTA stage the next U rows in shared memory.
#include "device.cuh"
#include "kernels.hpp"

#include <cooperative_groups.h>
#include <cstdlib>
#include <stdexcept>
#include <string>

namespace bcs {

constexpr int kDB = 64;  // panel width

// panel factorisation: one CTA, columns [k0, k0+nb), rows [k0, m)
__global__ void __launch_bounds__(1024) k_dense_panel(int m, int k0, int nb, double* a, int* piv, int* err) {
    __shared__ double sv[32];
    __shared__ int si[32];
    __shared__ int sp;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    const int k1 = k0 + nb;
    for (int k = k0; k < k1; ++k) {
        double best = -1.0;
        int bi = 0x7fffffff;
        for (int i = k + tid; i < m; i += nt) {
            const double v = fabs(a[static_cast<size_t>(i) * m + k]);
            if (v > best || (v == best && i < bi)) {
                best = v;
                bi = i;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, best, o);
            const int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) {
                best = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            sv[wid] = best;
            si[wid] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            double bb = sv[0];
            int ii = si[0];
            for (int w = 1; w < (nt >> 5); ++w)
                if (sv[w] > bb || (sv[w] == bb && si[w] < ii)) {
                    bb = sv[w];
                    ii = si[w];
                }
            const double akk = fabs(a[static_cast<size_t>(k) * m + k]);
            if (!(bb > akk)) ii = k, bb = akk;  // the reference starts from p = k; ties keep k
            if (bb < 1e-300) atomicExch(err, 1);
            piv[k] = ii;
            sp = ii;
        }
        __syncthreads();
        const int p = sp;
        if (p != k)
            for (int j = k0 + tid; j < k1; j += nt) {
                const double t = a[static_cast<size_t>(k) * m + j];
                a[static_cast<size_t>(k) * m + j] = a[static_cast<size_t>(p) * m + j];
                a[static_cast<size_t>(p) * m + j] = t;
            }
        __syncthreads();
        const double d = a[static_cast<size_t>(k) * m + k];
        for (int i = k + 1 + tid; i < m; i += nt) a[static_cast<size_t>(i) * m + k] = __ddiv_rn(a[static_cast<size_t>(i) * m + k], d);
        __syncthreads();
        // panel columns right of k: thread (row group tid/64, column k0 + tid%64)
        {
            const int j = k0 + (tid & 63);
            if (j > k && j < k1) {
                const double ukj = a[static_cast<size_t>(k) * m + j];
                for (int i = k + 1 + (tid >> 6); i < m; i += nt >> 6)
                    a[static_cast<size_t>(i) * m + j] =
                        __dsub_rn(a[static_cast<size_t>(i) * m + j], __dmul_rn(a[static_cast<size_t>(i) * m + k], ukj));
            }
        }
        __syncthreads();
    }
}

// panel factorisation spread over a cooperative grid: CTA c keeps rows
// [k0 + c*per, ...) of the panel in shared memory; per step one grid-wide
// argmax (first maximum, ties to the smaller row, the reference's p = k start
// included), the row swap through global scratch, then the local multipliers
// and panel update — the reference's per-element operation sequence.
__global__ void __launch_bounds__(256) k_dense_panel_coop(int m, int k0, int nb, int per, double* a, int* piv,
                                                          int* err, double* cand_v, int* cand_i, double* rowbuf) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sp[];  // per x kDB
    __shared__ double sv[8];
    __shared__ int si[8];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int r0 = k0 + c * per;
    const int r1 = min(m, r0 + per);
    const int k1 = k0 + nb;
    for (int t = tid; t < per * nb; t += nt) {
        const int rr = t / nb, j = t % nb;
        sp[rr * kDB + j] = r0 + rr < r1 ? a[static_cast<size_t>(r0 + rr) * m + k0 + j] : 0.0;
    }
    __syncthreads();
    for (int k = k0; k < k1; ++k) {
        const int kc = k - k0;
        // scratch double-buffered by step parity: two grid barriers per step
        double* cv = cand_v + (k & 1) * G;
        int* ci = cand_i + (k & 1) * G;
        double* rb = rowbuf + (k & 1) * 2 * kDB;
        // local first maximum of |a_ik|, i >= k
        double best = -1.0;
        int bi = 0x7fffffff;
        for (int i = max(r0, k) + tid; i < r1; i += nt) {
            const double v = fabs(sp[(i - r0) * kDB + kc]);
            if (v > best || (v == best && i < bi)) {
                best = v;
                bi = i;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, best, o);
            const int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) {
                best = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            sv[wid] = best;
            si[wid] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < (nt >> 5); ++w)
                if (sv[w] > sv[0] || (sv[w] == sv[0] && si[w] < si[0])) {
                    sv[0] = sv[w];
                    si[0] = si[w];
                }
            cv[c] = sv[0];
            ci[c] = si[0];
        }
        grid.sync();
        // every CTA reduces the candidates the same way
        if (wid == 0) {
            double b2 = -1.0;
            int i2 = 0x7fffffff;
            for (int q = lane; q < G; q += 32) {
                const double v = cv[q];
                const int ii = ci[q];
                if (v > b2 || (v == b2 && ii < i2)) {
                    b2 = v;
                    i2 = ii;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_down_sync(0xffffffffu, b2, o);
                const int oi = __shfl_down_sync(0xffffffffu, i2, o);
                if (ov > b2 || (ov == b2 && oi < i2)) {
                    b2 = ov;
                    i2 = oi;
                }
            }
            if (lane == 0) {
                si[0] = i2;
                sv[0] = b2;
            }
        }
        __syncthreads();
        const int p = si[0];
        if (c == 0 && tid == 0) {
            piv[k] = p;
            if (sv[0] < 1e-300) atomicExch(err, 1);
        }
        // swap rows k and p of the panel through global scratch:
        // rb[0..nb) = old row p (the new row k), rb[kDB..) = old row k
        if (p >= r0 && p < r1)
            for (int j = tid; j < nb; j += nt) rb[j] = sp[(p - r0) * kDB + j];
        if (k >= r0 && k < r1)
            for (int j = tid; j < nb; j += nt) rb[kDB + j] = sp[(k - r0) * kDB + j];
        grid.sync();
        if (k >= r0 && k < r1)
            for (int j = tid; j < nb; j += nt) sp[(k - r0) * kDB + j] = rb[j];
        if (p != k && p >= r0 && p < r1)
            for (int j = tid; j < nb; j += nt) sp[(p - r0) * kDB + j] = rb[kDB + j];
        __syncthreads();
        // multipliers and the panel update on the owned rows below k
        const double d = rb[kc];
        for (int i = max(r0, k + 1) + tid; i < r1; i += nt) {
            double* row = sp + (i - r0) * kDB;
            const double l = __ddiv_rn(row[kc], d);
            row[kc] = l;
            for (int j = kc + 1; j < nb; ++j) row[j] = __dsub_rn(row[j], __dmul_rn(l, rb[j]));
        }
        __syncthreads();
    }
    for (int t = tid; t < per * nb; t += nt) {
        const int rr = t / nb, j = t % nb;
        if (r0 + rr < r1) a[static_cast<size_t>(r0 + rr) * m + k0 + j] = sp[rr * kDB + j];
    }
}

// The same panel on ONE thread-block cluster of kPanelCl CTAs: the panel's
// rows live in the cluster's distributed shared memory (CTA c owns rows
// [k0 + c*per, ...)), a step's candidates and the pivot / swapped rows are
// read from peer CTAs' shared memory, and the two grid barriers per step
// become cluster barriers (~0.5 us instead of a few us over the whole grid).
// Same pivot rule and per-element operation sequence as k_dense_panel_coop.
constexpr int kPanelCl = 16;
__device__ __forceinline__ unsigned dsm_map(const void* p, unsigned cta) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))), "r"(cta));
    return r;
}
__device__ __forceinline__ double dsm_ld(unsigned addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ int dsm_ld_int(unsigned addr) {
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void cl_barrier() {
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}

__global__ void __launch_bounds__(512, 1) k_dense_panel_cl(int m, int k0, int nb, int per, double* a, int* piv,
                                                           int* err) {
    extern __shared__ double sp[];  // per x kDB rows of the panel
    __shared__ double cand_v, rb[kDB], rk[kDB];
    __shared__ int cand_i;
    __shared__ double sv[16];
    __shared__ int si[16];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    unsigned c;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(c));
    const int r0 = k0 + static_cast<int>(c) * per;
    const int r1 = min(m, r0 + per);
    const int k1 = k0 + nb;
    for (int t = tid; t < per * nb; t += nt) {
        const int rr = t / nb, j = t % nb;
        sp[rr * kDB + j] = r0 + rr < r1 ? a[static_cast<size_t>(r0 + rr) * m + k0 + j] : 0.0;
    }
    __syncthreads();
    cl_barrier();  // every CTA's rows are loaded before any peer reads them
    for (int k = k0; k < k1; ++k) {
        const int kc = k - k0;
        double best = -1.0;
        int bi = 0x7fffffff;
        for (int i = max(r0, k) + tid; i < r1; i += nt) {
            const double v = fabs(sp[(i - r0) * kDB + kc]);
            if (v > best || (v == best && i < bi)) {
                best = v;
                bi = i;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, best, o);
            const int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) {
                best = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            sv[wid] = best;
            si[wid] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < (nt >> 5); ++w)
                if (sv[w] > sv[0] || (sv[w] == sv[0] && si[w] < si[0])) {
                    sv[0] = sv[w];
                    si[0] = si[w];
                }
            cand_v = sv[0];
            cand_i = si[0];
        }
        cl_barrier();  // A: candidates visible cluster-wide
        // every CTA reduces the kPanelCl candidates in CTA order (same result everywhere)
        __shared__ int s_p;
        __shared__ double s_pv;
        if (wid == 0) {
            double b2 = -1.0;
            int i2 = 0x7fffffff;
            if (lane < kPanelCl) {
                b2 = dsm_ld(dsm_map(&cand_v, lane));
                i2 = dsm_ld_int(dsm_map(&cand_i, lane));
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_down_sync(0xffffffffu, b2, o);
                const int oi = __shfl_down_sync(0xffffffffu, i2, o);
                if (ov > b2 || (ov == b2 && oi < i2)) {
                    b2 = ov;
                    i2 = oi;
                }
            }
            if (lane == 0) {
                s_p = i2;
                s_pv = b2;
            }
        }
        __syncthreads();
        const int p = s_p;
        if (c == 0 && tid == 0) {
            piv[k] = p;
            if (s_pv < 1e-300) atomicExch(err, 1);
        }
        // the pivot row (old row p) into every CTA; its owner also takes old row k
        const unsigned op = static_cast<unsigned>((p - k0) / per), ok = static_cast<unsigned>((k - k0) / per);
        for (int j = tid; j < nb; j += nt) {
            rb[j] = dsm_ld(dsm_map(&sp[(p - (k0 + static_cast<int>(op) * per)) * kDB + j], op));
            if (c == op && p != k) rk[j] = dsm_ld(dsm_map(&sp[(k - (k0 + static_cast<int>(ok) * per)) * kDB + j], ok));
        }
        cl_barrier();  // B: every read of rows p and k done before they are overwritten
        if (k >= r0 && k < r1)
            for (int j = tid; j < nb; j += nt) sp[(k - r0) * kDB + j] = rb[j];
        if (p != k && p >= r0 && p < r1)
            for (int j = tid; j < nb; j += nt) sp[(p - r0) * kDB + j] = rk[j];
        __syncthreads();
        const double d = rb[kc];
        for (int i = max(r0, k + 1) + tid; i < r1; i += nt) {
            double* row = sp + (i - r0) * kDB;
            const double l = __ddiv_rn(row[kc], d);
            row[kc] = l;
            for (int j = kc + 1; j < nb; ++j) row[j] = __dsub_rn(row[j], __dmul_rn(l, rb[j]));
        }
        __syncthreads();
    }
    for (int t = tid; t < per * nb; t += nt) {
        const int rr = t / nb, j = t % nb;
        if (r0 + rr < r1) a[static_cast<size_t>(r0 + rr) * m + k0 + j] = sp[rr * kDB + j];
    }
    cl_barrier();  // no CTA exits while a peer may still read its shared memory
}

static bool panel_cl_ok(size_t smem) {
    static int ok = -1;
    if (ok < 0) {
        ok = 0;
        if (cudaFuncSetAttribute(k_dense_panel_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ==
                cudaSuccess &&
            cudaFuncSetAttribute(k_dense_panel_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = kPanelCl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(kPanelCl);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = 200 * 1024;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, k_dense_panel_cl, &cfg) == cudaSuccess && nc >= 1) ok = 1;
        }
        cudaGetLastError();
    }
    return ok == 1 && smem <= 200 * 1024;
}

// the panel's row swaps, in order, on every column outside the panel
__global__ void k_dense_laswp(int m, int k0, int nb, double* a, const int* piv) {
    const int j0 = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = j0 < k0 ? j0 : j0 + nb;
    if (j0 >= m - nb) return;
    for (int k = k0; k < k0 + nb; ++k) {
        const int p = piv[k];
        if (p != k) {
            const double t = a[static_cast<size_t>(k) * m + j];
            a[static_cast<size_t>(k) * m + j] = a[static_cast<size_t>(p) * m + j];
            a[static_cast<size_t>(p) * m + j] = t;
        }
    }
}

// rows [k0, k0+nb), columns [k0+nb, m): a_ij -= l_ik u_kj, k ascending (unit L11)
__global__ void __launch_bounds__(128) k_dense_trsm(int m, int k0, int nb, double* a) {
    __shared__ double L[kDB][kDB + 1];
    for (int t = threadIdx.x; t < nb * nb; t += blockDim.x) {
        const int i = t / nb, k = t % nb;
        L[i][k] = a[static_cast<size_t>(k0 + i) * m + k0 + k];
    }
    __syncthreads();
    const int j = k0 + nb + blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    double x[kDB];
#pragma unroll
    for (int i = 0; i < kDB; ++i) x[i] = i < nb ? a[static_cast<size_t>(k0 + i) * m + j] : 0.0;
#pragma unroll
    for (int k = 0; k < kDB; ++k) {
#pragma unroll
        for (int i = k + 1; i < kDB; ++i)
            if (i < nb && k < nb) x[i] = __dsub_rn(x[i], __dmul_rn(L[i][k], x[k]));
    }
#pragma unroll
    for (int i = 0; i < kDB; ++i)
        if (i < nb) a[static_cast<size_t>(k0 + i) * m + j] = x[i];
}

// trailing update, 64x64 tiles of 256 threads (4x4 elements each):
// a_ij -= l_ik u_kj for k = k0 .. k0+nb-1 in order, one rounded mul + sub each
__global__ void __launch_bounds__(256) k_dense_update(int m, int k0, int nb, double* a) {
    extern __shared__ double sm[];
    double* Lt = sm;                 // [kDB][64]: Lt[k][r] = a[i0+r][k0+k]
    double* U = sm + kDB * 64;       // [kDB][64]: U[k][c] = a[k0+k][j0+c]
    const int k1 = k0 + nb;
    const int i0 = k1 + blockIdx.y * 64, j0 = k1 + blockIdx.x * 64;
    for (int t = threadIdx.x; t < nb * 64; t += blockDim.x) {
        const int r = t / nb, k = t % nb;  // coalesced along k for L
        const int i = i0 + r;
        Lt[k * 64 + r] = i < m ? a[static_cast<size_t>(i) * m + k0 + k] : 0.0;
    }
    for (int t = threadIdx.x; t < nb * 64; t += blockDim.x) {
        const int k = t / 64, c = t % 64;
        const int j = j0 + c;
        U[k * 64 + c] = j < m ? a[static_cast<size_t>(k0 + k) * m + j] : 0.0;
    }
    __syncthreads();
    const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int i = i0 + ty + 16 * r, j = j0 + tx + 16 * c;
            acc[r][c] = (i < m && j < m) ? a[static_cast<size_t>(i) * m + j] : 0.0;
        }
    for (int k = 0; k < nb; ++k) {
        double l[4], u[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) l[r] = Lt[k * 64 + ty + 16 * r];
#pragma unroll
        for (int c = 0; c < 4; ++c) u[c] = U[k * 64 + tx + 16 * c];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = __dsub_rn(acc[r][c], __dmul_rn(l[r], u[c]));
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int i = i0 + ty + 16 * r, j = j0 + tx + 16 * c;
            if (i < m && j < m) a[static_cast<size_t>(i) * m + j] = acc[r][c];
        }
}

// composed permutation of the swap sequence: x_perm[i] = x[perm[i]]
__global__ void k_dense_perm(int m, const int* piv, int* perm) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int i = 0; i < m; ++i) perm[i] = i;
    for (int k = 0; k < m; ++k) {
        const int p = piv[k];
        if (p != k) {
            const int t = perm[k];
            perm[k] = perm[p];
            perm[p] = t;
        }
    }
}

// BCS_DENSE_PANEL_CL=0: the grid-cooperative panel only
static int g_panel_cl = [] {
    const char* e = std::getenv("BCS_DENSE_PANEL_CL");
    return e ? std::atoi(e) : 1;
}();

void dense_factor_blocked(int m, double* a, int* piv, int* err, cudaStream_t s) {
    static bool attr = false;
    const int smem = 2 * kDB * 64 * static_cast<int>(sizeof(double));
    if (!attr) {
        cudaFuncSetAttribute(k_dense_update, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    // cooperative panel: one CTA per SM at most, rows split evenly
    static int G = 0;
    static double* scratch = nullptr;
    if (!G) {
        G = num_sms();
        cudaMalloc(&scratch, sizeof(double) * (4 * G + 4 * kDB));
    }
    double* cand_v = scratch;                                   // 2G
    int* cand_i = reinterpret_cast<int*>(scratch + 2 * G);      // 2G ints
    double* rowbuf = scratch + 4 * G;                           // 2 x 2kDB
    int launches = 0;
    for (int k0 = 0; k0 < m; k0 += kDB) {
        const int nb = m - k0 < kDB ? m - k0 : kDB;
        const int rows = m - k0;
        int g = G < rows ? G : rows;
        int per = (rows + g - 1) / g;
        g = (rows + per - 1) / per;
        const size_t psmem = sizeof(double) * static_cast<size_t>(per) * kDB;
        const int pcl = (rows + kPanelCl - 1) / kPanelCl;
        const size_t clsmem = sizeof(double) * static_cast<size_t>(pcl) * kDB;
        if (g_panel_cl && rows >= 4 * kPanelCl && panel_cl_ok(clsmem)) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = kPanelCl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(kPanelCl);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = clsmem;
            cfg.stream = s;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            const cudaError_t e = cudaLaunchKernelEx(&cfg, k_dense_panel_cl, m, k0, nb, pcl, a, piv, err);
            if (e != cudaSuccess) throw std::runtime_error(std::string("dense cluster panel: ") + cudaGetErrorString(e));
        } else if (psmem <= 200 * 1024) {
            static size_t attr_p = 0;
            if (psmem > attr_p) {
                cudaFuncSetAttribute(k_dense_panel_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                attr_p = 200 * 1024;
            }
            void* args[] = {(void*)&m, (void*)&k0, (void*)&nb, (void*)&per, (void*)&a, (void*)&piv, (void*)&err,
                            (void*)&cand_v, (void*)&cand_i, (void*)&rowbuf};
            const cudaError_t e = cudaLaunchCooperativeKernel((void*)k_dense_panel_coop, dim3(g), dim3(256), args,
                                                              psmem, s);
            if (e != cudaSuccess) throw std::runtime_error(std::string("dense panel: ") + cudaGetErrorString(e));
        } else {
            k_dense_panel<<<1, 1024, 0, s>>>(m, k0, nb, a, piv, err);
        }
        if (m - nb > 0) k_dense_laswp<<<(m - nb + 255) / 256, 256, 0, s>>>(m, k0, nb, a, piv);
        const int rest = m - k0 - nb;
        launches += 2;
        if (rest > 0) {
            k_dense_trsm<<<(rest + 127) / 128, 128, 0, s>>>(m, k0, nb, a);
            const int t = (rest + 63) / 64;
            k_dense_update<<<dim3(t, t), 256, smem, s>>>(m, k0, nb, a);
            launches += 2;
        }
    }
    k_dense_perm<<<1, 1, 0, s>>>(m, piv, piv + m);
    count_launch(launches + 1);
}

// forward + backward substitution, one CTA (reference order, see header).
// SX: x and the staged U rows in shared memory (m up to ~9,000); otherwise
// x lives in z (global) and U rows are read in place.
template <bool SX>
__global__ void __launch_bounds__(1024) k_dense_solve_big(int m, const double* __restrict__ lu,
                                                          const int* __restrict__ perm, const double* r, double* z) {
    extern __shared__ double sm[];
    double* tile = sm;                          // 32 x 33: the in-tile block of L
    double* x = SX ? sm + 32 * 33 : z;
    double* ub = sm + 32 * 33 + m;              // SX: two staged U rows
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < m; i += nt) {
        const double v = r[perm[i]];
        if (SX) x[i] = v;
        else z[i] = v;  // (r and z never alias)
    }
    __syncthreads();
    // forward, unit lower: column tiles of 32; warp 0 finalises a tile's x
    // (in-tile chain on the staged tile), then every thread folds the tile
    // into the rows below, each row's subtractions in ascending column order
    for (int j0 = 0; j0 < m; j0 += 32) {
        const int j1 = j0 + 32 < m ? j0 + 32 : m;
        for (int t = tid; t < 32 * 32; t += nt) {
            const int i = j0 + t / 32, j = j0 + t % 32;
            tile[(t / 32) * 33 + t % 32] = (i < j1 && j < i) ? lu[static_cast<size_t>(i) * m + j] : 0.0;
        }
        __syncthreads();
        if (wid == 0) {
            const int i = j0 + lane;
            double xi = i < j1 ? x[i] : 0.0;
            for (int j = j0; j < j1 - 1; ++j) {
                const double xj = __shfl_sync(0xffffffffu, xi, j - j0);
                if (i > j && i < j1) xi = __dsub_rn(xi, __dmul_rn(tile[lane * 33 + (j - j0)], xj));
            }
            if (i < j1) x[i] = xi;
        }
        __syncthreads();
        for (int i = j1 + tid; i < m; i += nt) {
            double xi = x[i];
            const double* row = lu + static_cast<size_t>(i) * m;
#pragma unroll 8
            for (int j = j0; j < j1; ++j) xi = __dsub_rn(xi, __dmul_rn(row[j], x[j]));
            x[i] = xi;
        }
        __syncthreads();
    }
    // backward: thread 0 runs the subtraction chain; with SX the other warps
    // precompute row i-1's products t_q = RN(U_{i-1,i-1+q} x_{i-1+q}) for
    // q >= 2 (those x are final) while row i is processed, so the chain is
    // one rounded subtraction per step read from shared memory
    // (zero padding to the next multiple of 16 plus one block: x - (+0) == x
    // exactly, so the chain runs in whole blocks)
    auto stage = [&](int i, double* dst) {
        const double* row = lu + static_cast<size_t>(i) * m;
        if (tid - 32 == 0) dst[0] = row[i];
        const int pad = ((m - i + 15) & ~15) + 48;  // every index the chain loads
        for (int q = 2 + (tid - 32); q < pad; q += nt - 32) dst[q] = i + q < m ? __dmul_rn(row[i + q], x[i + q]) : 0.0;
    };
    if (SX && wid > 0) stage(m - 1, ub);  // two buffers of m + 64
    __syncthreads();
    for (int i = m - 1; i >= 0; --i) {
        double* nxt = ub + ((m - i) & 1) * (m + 64);
        if (tid == 0) {
            double xi = x[i];
            const int len = m - i;
            if (SX) {
                const double* t = ub + ((m - 1 - i) & 1) * (m + 64);  // t[0] = U_ii, t[q >= 2] = products
                if (len > 1) xi = __dsub_rn(xi, __dmul_rn(lu[static_cast<size_t>(i) * m + i + 1], x[i + 1]));
                // blocks of 16: the next block's loads are in flight while
                // the current one is folded
                double A[16], B[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) A[q] = q >= 2 ? t[q] : 0.0;
                for (int q0 = 16; q0 < len + 16; q0 += 32) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) B[q] = t[q0 + q];
#pragma unroll
                    for (int q = 0; q < 16; ++q) xi = __dsub_rn(xi, A[q]);
#pragma unroll
                    for (int q = 0; q < 16; ++q) A[q] = t[q0 + 16 + q];
#pragma unroll
                    for (int q = 0; q < 16; ++q) xi = __dsub_rn(xi, B[q]);
                }
                x[i] = __ddiv_rn(xi, t[0]);
            } else {
                const double* cur = lu + static_cast<size_t>(i) * m + i;
#pragma unroll 8
                for (int q = 1; q < len; ++q) xi = __dsub_rn(xi, __dmul_rn(cur[q], x[i + q]));
                x[i] = __ddiv_rn(xi, cur[0]);
            }
        } else if (SX && wid > 0 && i > 0) {
            stage(i - 1, nxt);
        }
        __syncthreads();
    }
    if (SX)
        for (int i = tid; i < m; i += nt) z[i] = x[i];
}

// Tolerance-level solve for large coarsest levels (the
// scrambled inputs' aggregation stall leaves m in the thousands): the forward
// substitution is k_dense_solve_big's (reference order, bit-exact); the
// backward one runs by column tiles of 32 from the right -- warp 0 finishes a
// tile's x (in-tile chain), then every thread folds the tile into the rows
// above -- so the critical path is m/32 tiles, not the reference's m^2/2
// dependent subtractions (whose order it does not keep: rounding differs).
__global__ void __launch_bounds__(1024) k_dense_solve_tiled(int m, const double* __restrict__ lu,
                                                            const int* __restrict__ perm, const double* r, double* z,
                                                            int sx) {
    extern __shared__ double sm[];
    double* tile = sm;                     // 32 x 33
    double* x = sx ? sm + 32 * 33 : z;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < m; i += nt) x[i] = r[perm[i]];
    __syncthreads();
    for (int j0 = 0; j0 < m; j0 += 32) {  // forward (unit lower), reference order per row
        const int j1 = j0 + 32 < m ? j0 + 32 : m;
        for (int t = tid; t < 32 * 32; t += nt) {
            const int i = j0 + t / 32, j = j0 + t % 32;
            tile[(t / 32) * 33 + t % 32] = (i < j1 && j < i) ? lu[static_cast<size_t>(i) * m + j] : 0.0;
        }
        __syncthreads();
        if (wid == 0) {
            const int i = j0 + lane;
            double xi = i < j1 ? x[i] : 0.0;
            for (int j = j0; j < j1 - 1; ++j) {
                const double xj = __shfl_sync(0xffffffffu, xi, j - j0);
                if (i > j && i < j1) xi = __dsub_rn(xi, __dmul_rn(tile[lane * 33 + (j - j0)], xj));
            }
            if (i < j1) x[i] = xi;
        }
        __syncthreads();
        for (int i = j1 + tid; i < m; i += nt) {
            double xi = x[i];
            const double* row = lu + static_cast<size_t>(i) * m;
#pragma unroll 8
            for (int j = j0; j < j1; ++j) xi = __dsub_rn(xi, __dmul_rn(row[j], x[j]));
            x[i] = xi;
        }
        __syncthreads();
    }
    for (int j1 = m; j1 > 0; j1 -= 32) {  // backward (upper), tiles from the right
        const int j0 = j1 - 32 > 0 ? j1 - 32 : 0;
        for (int t = tid; t < 32 * 32; t += nt) {
            const int i = j0 + t / 32, j = j0 + t % 32;
            tile[(t / 32) * 33 + t % 32] = (i < j1 && j < j1 && j >= i) ? lu[static_cast<size_t>(i) * m + j] : 0.0;
        }
        __syncthreads();
        if (wid == 0) {
            const int i = j0 + lane;
            double xi = i < j1 ? x[i] : 0.0;
            for (int j = j1 - 1; j >= j0; --j) {
                if (i == j) xi = __ddiv_rn(xi, tile[lane * 33 + (j - j0)]);
                const double xj = __shfl_sync(0xffffffffu, xi, j - j0);
                if (i < j && i >= j0) xi = __dsub_rn(xi, __dmul_rn(tile[lane * 33 + (j - j0)], xj));
            }
            if (i < j1) x[i] = xi;
        }
        __syncthreads();
        for (int i = tid; i < j0; i += nt) {
            double xi = x[i];
            const double* row = lu + static_cast<size_t>(i) * m;
#pragma unroll 8
            for (int j = j0; j < j1; ++j) xi = __dsub_rn(xi, __dmul_rn(row[j], x[j]));
            x[i] = xi;
        }
        __syncthreads();
    }
    if (sx)
        for (int i = tid; i < m; i += nt) z[i] = x[i];
}

constexpr size_t kDenseSmemMax = 200 * 1024;

void dense_solve_tiled(int m, const double* lu, const int* piv, const double* r, double* z, cudaStream_t s) {
    const size_t full = (static_cast<size_t>(32) * 33 + static_cast<size_t>(m)) * sizeof(double);
    const int sx = full <= kDenseSmemMax ? 1 : 0;
    const size_t smem = sx ? full : static_cast<size_t>(32) * 33 * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_dense_solve_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kDenseSmemMax));
        attr = true;
    }
    k_dense_solve_tiled<<<1, 1024, smem, s>>>(m, lu, piv + m, r, z, sx);
    count_launch();
}

void dense_solve_big(int m, const double* lu, const int* piv, const double* r, double* z, cudaStream_t s) {
    const size_t full = (static_cast<size_t>(32) * 33 + 3 * static_cast<size_t>(m) + 128) * sizeof(double);
    const bool sx = full <= kDenseSmemMax;
    const size_t smem = sx ? full : static_cast<size_t>(32) * 33 * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_dense_solve_big<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kDenseSmemMax));
        attr = true;
    }
    if (sx) k_dense_solve_big<true><<<1, 1024, smem, s>>>(m, lu, piv + m, r, z);
    else k_dense_solve_big<false><<<1, 1024, smem, s>>>(m, lu, piv + m, r, z);
    count_launch();
}

}  // namespace bcs
