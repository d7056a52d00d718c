// The coarse tail of the V-cycle (amg.cpp:111-158) in one CTA.
//
// Below a few thousand rows a level's smoothing is a short dependency chain
// of tiny rows: as separate launches every hop pays a cross-SM handoff through
// L2 and every operation a launch.  Here one CTA runs the whole tail — the
// down path (pre-smoothing, residual, restriction) of every tail level, then,
// after the coarsest dense solve, the up path (prolongation, residual,
// post-smoothing) — with the sweeps' outputs in shared memory, so a dependency
// handoff is a shared-memory store and poll.  Arithmetic and its order are
// exactly those of k_sweep / k_spmv / k_restrict / k_prolong.
#include "device.cuh"
#include "kernels.hpp"

#include <stdexcept>
#include <string>

namespace bcs {

namespace {

__device__ __forceinline__ double lds_v(const double* p) { return *reinterpret_cast<const volatile double*>(p); }
__device__ __forceinline__ void sts_v(double* p, double v) { *reinterpret_cast<volatile double*>(p) = v; }

template <int N>
__device__ __forceinline__ double pick_t(const double* x, int lane) {
    double o = x[0];
#pragma unroll
    for (int q = 1; q < N; ++q) o = (lane == q) ? x[q] : o;
    return o;
}

constexpr unsigned kAll = 0xffffffffu;
constexpr unsigned kTailSpin = 1u << 26;

// one sweep of one level, rows in level order on the CTA's warps (warp w:
// tickets w, w+W, ...; co-resident, so deadlock-free).  FWD: y = (D~+L)^-1 rin
// into ys; BWD: zb = y - D~^-1 U zb into zbs and z (accumulate 1: 0 + zb,
// 2: z + zb).
template <int N, bool FWD>
__device__ void tail_sweep(const TailLevelDev& L, const double* rin, double* ys, double* zbs, double* z, int accumulate,
                           int* err) {
    constexpr int NN = N * N;
    constexpr int DPP = 32 / N < 12 ? 32 / N : 12;
    const int lane = threadIdx.x & 31, W = blockDim.x >> 5;
    const int dd = lane / N, qq = lane - (lane / N) * N;
    double* outs = FWD ? ys : zbs;
    for (int t = threadIdx.x >> 5; t < L.rows; t += W) {
        const int i = FWD ? __ldg(&L.order[t]) : __ldg(&L.order[L.rows - 1 - t]);
        const int kf = FWD ? __ldg(&L.ro[i]) : __ldg(&L.ro[i + 1]) - 1;
        const int d = __ldg(&L.dg[i]);
        const int cnt = FWD ? d - kf : kf - d;
        double lf[NN], rcf[N];
        int pmf[N];
#pragma unroll
        for (int e = 0; e < NN; ++e) lf[e] = __ldg(&L.lu[static_cast<size_t>(i) * NN + e]);
#pragma unroll
        for (int q = 0; q < N; ++q) {
            rcf[q] = __ldg(&L.rcp[static_cast<size_t>(i) * N + q]);
            pmf[q] = __ldg(&L.perm[static_cast<size_t>(i) * N + q]);
        }
        const double ri = lane < N ? (FWD ? rin[static_cast<size_t>(i) * N + lane] : lds_v(&ys[i * N + lane])) : 0.0;
        double acc = FWD ? ri : 0.0;
        for (int c0 = 0; c0 < cnt; c0 += DPP) {
            const int c = c0 + dd;
            const bool has = lane < DPP * N && c < cnt;
            const int k = FWD ? kf + c : kf - c;
            const int j = has ? __ldg(&L.ci[k]) : 0;
            double arow[N];
#pragma unroll
            for (int p = 0; p < N; ++p) arow[p] = has ? __ldg(&L.v[static_cast<size_t>(k) * NN + qq * N + p]) : 0.0;
            double yq = has ? __longlong_as_double(-1ll) : 0.0;
            for (unsigned spins = 0;; ++spins) {
                if (has && is_pending(yq)) yq = lds_v(&outs[j * N + qq]);
                if (__all_sync(kAll, !is_pending(yq))) break;
                if (spins > kTailSpin) {
                    if (lane == 0) atomicExch(err, 1);
                    yq = is_pending(yq) ? 0.0 : yq;
                    break;
                }
            }
            double sblk = 0.0;
#pragma unroll
            for (int p = 0; p < N; ++p) sblk = __dadd_rn(sblk, __dmul_rn(arow[p], __shfl_sync(kAll, yq, dd * N + p)));
            const int ne = cnt - c0 < DPP ? cnt - c0 : DPP;
            double sg[DPP];
#pragma unroll
            for (int e = 0; e < DPP; ++e) sg[e] = __shfl_sync(kAll, sblk, e * N + (lane < N ? lane : 0));
#pragma unroll
            for (int e = 0; e < DPP; ++e) {
                if (e >= ne) break;  // a branch, not a select chain: ne FP steps on the critical path, not DPP
                acc = FWD ? __dsub_rn(acc, sg[e]) : __dadd_rn(acc, sg[e]);
            }
        }
        double x[N];
#pragma unroll
        for (int p = 0; p < N; ++p) x[p] = __shfl_sync(kAll, acc, pmf[p]);
        DVec<N> xin;
#pragma unroll
        for (int p = 0; p < N; ++p) xin.v[p] = x[p];
        if (__builtin_expect(!lu_solve_perm_fast<N>(lf, rcf, x), 0)) {
            const DVec<N> xe = lu_solve_perm_exact<N>(L.lu + static_cast<size_t>(i) * NN, xin);
#pragma unroll
            for (int p = 0; p < N; ++p) x[p] = xe.v[p];
        }
        if (lane < N) {
            const double res = FWD ? pick_t<N>(x, lane) : __dsub_rn(ri, pick_t<N>(x, lane));
            sts_v(&outs[i * N + lane], res);
            if (!FWD) {
                const size_t o = static_cast<size_t>(i) * N + lane;
                if (accumulate == 1) z[o] = __dadd_rn(0.0, res);
                else if (accumulate == 2) z[o] = __dadd_rn(z[o], res);
            }
        }
        __syncwarp();
    }
}

template <int N>
__device__ void tail_smooth(const TailLevelDev& L, const double* rin, double* z, int accumulate, double* ys, double* zbs,
                            int* err) {
    const int n = L.rows * N;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        ys[t] = __longlong_as_double(-1ll);
        zbs[t] = __longlong_as_double(-1ll);
    }
    __syncthreads();
    tail_sweep<N, true>(L, rin, ys, zbs, z, accumulate, err);
    __syncthreads();
    tail_sweep<N, false>(L, rin, ys, zbs, z, accumulate, err);
    __syncthreads();
}

// res = r - A z  (k_spmv with `sub`)
template <int N>
__device__ void tail_residual(const TailLevelDev& L, const double* r, const double* z, double* res) {
    constexpr int NN = N * N;
    const int n = L.rows * N;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const int row = t / N, q = t - (t / N) * N;
        const int b = __ldg(&L.ro[row]), e = __ldg(&L.ro[row + 1]);
        double acc = 0.0;
#pragma unroll 4
        for (int k = b; k < e; ++k) {
            const int c = __ldg(&L.ci[k]);
            const double* a = L.v + static_cast<size_t>(k) * NN + q * N;
            double sblk = 0.0;
#pragma unroll
            for (int p = 0; p < N; ++p) sblk = __dadd_rn(sblk, __dmul_rn(__ldg(&a[p]), z[static_cast<size_t>(c) * N + p]));
            acc = __dadd_rn(acc, sblk);
        }
        res[t] = __dsub_rn(r[t], acc);
    }
    __syncthreads();
}

}  // namespace

template <int N>
__global__ void __launch_bounds__(512, 1) k_vcycle_tail(int nl, const TailLevelDev* __restrict__ lv, const double* rtop,
                                                        double* ztop, int pre, int post, int phase, int* err) {
    extern __shared__ double tsm[];  // ys | zbs, rows_max * N each
    const int half = lv[0].rows * N;  // the top tail level is the largest
    double* ys = tsm;
    double* zbs = tsm + half;
    if (phase == 0) {
        for (int l = 0; l + 1 < nl; ++l) {
            const TailLevelDev& L = lv[l];
            const double* r = l == 0 ? rtop : L.r;
            double* z = l == 0 ? ztop : L.z;
            for (int s = 0; s < pre; ++s) {
                const double* rin = r;  // z == 0 on the first sweep: r - A*0 == r exactly
                if (s > 0) {
                    tail_residual<N>(L, r, z, L.res);
                    rin = L.res;
                }
                tail_smooth<N>(L, rin, z, s == 0 ? 1 : 2, ys, zbs, err);
            }
            const double* res = r;
            if (pre > 0) {
                tail_residual<N>(L, r, z, L.res);
                res = L.res;
            } else {
                for (int t = threadIdx.x; t < L.rows * N; t += blockDim.x) z[t] = 0.0;
                __syncthreads();
            }
            const TailLevelDev& C = lv[l + 1];
            for (int t = threadIdx.x; t < L.ncoarse * N; t += blockDim.x) {  // k_restrict
                const int c = t / N, q = t - (t / N) * N;
                const int r1 = L.members[2 * c], r2 = L.members[2 * c + 1];
                double v = __dadd_rn(0.0, res[static_cast<size_t>(r1) * N + q]);
                if (r2 >= 0) v = __dadd_rn(v, res[static_cast<size_t>(r2) * N + q]);
                C.r[t] = v;
            }
            __syncthreads();
        }
    } else {
        for (int l = nl - 2; l >= 0; --l) {
            const TailLevelDev& L = lv[l];
            const TailLevelDev& C = lv[l + 1];
            const double* r = l == 0 ? rtop : L.r;
            double* z = l == 0 ? ztop : L.z;
            for (int t = threadIdx.x; t < L.rows * N; t += blockDim.x) {  // k_prolong
                const int row = t / N, q = t - (t / N) * N;
                z[t] = __dadd_rn(z[t], C.z[static_cast<size_t>(L.agg[row]) * N + q]);
            }
            __syncthreads();
            for (int s = 0; s < post; ++s) {
                tail_residual<N>(L, r, z, L.res);
                tail_smooth<N>(L, L.res, z, 2, ys, zbs, err);
            }
        }
    }
}

size_t tail_smem_bytes(int n, int rows) { return static_cast<size_t>(2) * rows * n * sizeof(double); }

template <int N>
static void launch_tail(int nl, const TailLevelDev* lv, size_t smem, const double* rtop, double* ztop, int pre,
                        int post, int phase, int* err, cudaStream_t s) {
    static size_t set = 0;  // per block size: the attribute belongs to the instantiation
    {
        std::lock_guard<std::recursive_mutex> lazy_lk(lazy_init_mutex());
        if (smem > set) {
            const cudaError_t e = cudaFuncSetAttribute(k_vcycle_tail<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       static_cast<int>(smem));
            if (e != cudaSuccess) throw std::runtime_error(std::string("V-cycle tail: ") + cudaGetErrorString(e));
            set = smem;
        }
    }
    k_vcycle_tail<N><<<1, 512, smem, s>>>(nl, lv, rtop, ztop, pre, post, phase, err);
}

void vcycle_tail(int n, int nl, const TailLevelDev* lv, int top_rows, const double* rtop, double* ztop, int pre,
                 int post, int phase, int* err, cudaStream_t s) {
    const size_t smem = tail_smem_bytes(n, top_rows);
    switch (n) {
        case 1: launch_tail<1>(nl, lv, smem, rtop, ztop, pre, post, phase, err, s); break;
        case 2: launch_tail<2>(nl, lv, smem, rtop, ztop, pre, post, phase, err, s); break;
        case 3: launch_tail<3>(nl, lv, smem, rtop, ztop, pre, post, phase, err, s); break;
        case 4: launch_tail<4>(nl, lv, smem, rtop, ztop, pre, post, phase, err, s); break;
        case 5: launch_tail<5>(nl, lv, smem, rtop, ztop, pre, post, phase, err, s); break;
        default: throw std::invalid_argument("block size must be 1..5 on the device");
    }
    count_launch();
}

}  // namespace bcs
