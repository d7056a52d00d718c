// Performance mode (BCS_MODE_PERF): multicolour block DILU smoothing, the
// north_star's "multicolour block-Gauss-Seidel/DILU smoothing" (AmgX's
// MULTICOLOR_DILU).  The reference orders its DILU/LUSGS sweeps naturally
// (preconditioner.cpp:101-156), whose dependency DAG is hundreds of levels
// deep on a hex mesh; here every smoothed AMG level is coloured (no two
// coupled rows share a colour) and the smoother runs on the level's matrix
// symmetrically permuted by colour.  On that matrix a row's lower neighbours
// all carry smaller colours, so the natural-order machinery (sync-free DILU
// setup, sync-free sweeps, k_sweep.cu) sees a DAG only #colours deep, and the
// big levels run one streaming launch per colour (k_mc_colour): the sweeps
// become throughput (HBM) bound.  The hierarchy itself, the SpMVs and
// the Krylov method are unchanged; the smoother is a different operator, so
// iteration counts differ from the reference and are reported as such.
//
// Colouring: Jones-Plassmann with hashed priorities, first-fit colours, one
// kernel per round reading the previous round's colours (double buffered), so
// the colouring is deterministic (a function of the pattern only).
#include "device.cuh"
#include "kernels.hpp"

#include <cooperative_groups.h>

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

namespace bcs {

__device__ __forceinline__ unsigned mc_hash(unsigned x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}
// strict total order of the priorities: (hash, index)
__device__ __forceinline__ bool mc_above(unsigned hj, int j, unsigned hi, int i) {
    return hj > hi || (hj == hi && j > i);
}

constexpr int kMaxColors = 64;

__global__ void k_jp_round(int rows, const int* __restrict__ ro, const int* __restrict__ ci, const int* __restrict__ cin,
                           int* cout, int* left, int* overflow) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool wait = false, over = false;
    if (i < rows) {
        const int ci0 = cin[i];
        int out = ci0;
        if (ci0 < 0) {
            const unsigned hi = mc_hash(static_cast<unsigned>(i));
            unsigned long long used = 0ull;
            for (int k = ro[i]; k < ro[i + 1]; ++k) {
                const int j = ci[k];
                if (j == i) continue;
                const int cj = cin[j];
                if (cj < 0) {
                    if (mc_above(mc_hash(static_cast<unsigned>(j)), j, hi, i)) {  // an uncoloured neighbour goes first
                        wait = true;
                        break;
                    }
                } else if (cj < kMaxColors) {
                    used |= 1ull << cj;
                }
            }
            if (!wait) {
                const unsigned long long freeMask = ~used;
                if (!freeMask) {
                    over = true;
                    out = kMaxColors;  // colour count overflow: reported, level falls back
                } else {
                    out = __ffsll(static_cast<long long>(freeMask)) - 1;
                }
            }
        }
        cout[i] = out;
    }
    // one atomic per warp (a single counter would serialise millions of rows)
    const unsigned wm = __ballot_sync(0xffffffffu, wait), om = __ballot_sync(0xffffffffu, over);
    if ((threadIdx.x & 31) == 0) {
        if (wm) atomicAdd(left, __popc(wm));
        if (om) atomicExch(overflow, 1);
    }
}

__global__ void k_color_hist(int rows, const int* __restrict__ color, int* cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows) atomicAdd(&cnt[color[i]], 1);
}

// stable counting sort by colour: warp-cooperative over contiguous row chunks
// would be faster; rows are placed by (colour, index) with one pass per colour
// block of 1024 rows (ranks within a colour from a per-block prefix)
__global__ void k_color_rank(int rows, const int* __restrict__ color, int ncol, int* blockCnt) {
    // blockCnt[b * ncol + c] = rows of colour c in block b
    __shared__ int cnt[kMaxColors];
    for (int c = threadIdx.x; c < ncol; c += blockDim.x) cnt[c] = 0;
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows) atomicAdd(&cnt[color[i]], 1);
    __syncthreads();
    for (int c = threadIdx.x; c < ncol; c += blockDim.x) blockCnt[blockIdx.x * ncol + c] = cnt[c];
}
__global__ void k_color_place(int rows, const int* __restrict__ color, int ncol, const int* __restrict__ base,
                              int* perm, int* inv) {
    // base[b * ncol + c]: first new index of colour c rows in block b; within
    // a block rows keep their index order: rank = rows of the same colour in
    // earlier warps (shared counts) + earlier lanes of this warp (match mask)
    __shared__ int wcnt[32][kMaxColors + 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int c = i < rows ? color[i] : kMaxColors;
    for (int e = threadIdx.x; e < 32 * (kMaxColors + 1); e += blockDim.x) (&wcnt[0][0])[e] = 0;
    __syncthreads();
    const unsigned m = __match_any_sync(0xffffffffu, c);
    const int rw = __popc(m & ((1u << lane) - 1u));
    if (rw == 0) wcnt[w][c] = __popc(m);
    __syncthreads();
    if (i >= rows) return;
    int pre = 0;
    for (int q = 0; q < w; ++q) pre += wcnt[q][c];
    const int ni = base[blockIdx.x * ncol + c] + pre + rw;
    perm[ni] = i;
    inv[i] = ni;
}

// permuted BSR: new row i' = perm[i'] keeps its blocks; columns renumbered
// (inv) and the row sorted by new column (insertion sort of slot indices,
// rows are short); sv[k'] = the source slot of new slot k'
__global__ void k_perm_rows(int rows, const int* __restrict__ ro, const int* __restrict__ ci,
                            const int* __restrict__ perm, const int* __restrict__ inv, const int* __restrict__ nro,
                            int* nci, int* sv) {
    const int ip = blockIdx.x * blockDim.x + threadIdx.x;
    if (ip >= rows) return;
    const int i = perm[ip];
    const int b = ro[i], e = ro[i + 1], o = nro[ip];
    for (int k = b; k < e; ++k) {
        const int c = inv[ci[k]];
        int p = o + (k - b);
        while (p > o && nci[p - 1] > c) {
            nci[p] = nci[p - 1];
            sv[p] = sv[p - 1];
            --p;
        }
        nci[p] = c;
        sv[p] = k;
    }
}
__global__ void k_row_len_perm(int rows, const int* __restrict__ ro, const int* __restrict__ perm, int* len) {
    const int ip = blockIdx.x * blockDim.x + threadIdx.x;
    if (ip < rows) len[ip] = ro[perm[ip] + 1] - ro[perm[ip]];
}
template <int NN>
__global__ void k_gather_blocks(size_t nnz, const int* __restrict__ sv, const double* __restrict__ v, double* nv) {
    const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (t >= nnz * NN) return;
    const size_t k = t / NN, e = t - k * NN;
    nv[t] = v[static_cast<size_t>(sv[k]) * NN + e];
}

int mc_color(int rows, const int* ro, const int* ci, int* colA, int* colB, int* counters, int* hostCounters,
             cudaStream_t s) {
    cudaMemsetAsync(colA, 0xFF, sizeof(int) * static_cast<size_t>(rows), s);
    int* cur = colA;
    int* nxt = colB;
    for (int round = 0; round < 4096; ++round) {
        cudaMemsetAsync(counters, 0, 2 * sizeof(int), s);
        k_jp_round<<<(rows + 255) / 256, 256, 0, s>>>(rows, ro, ci, cur, nxt, counters, counters + 1);
        count_launch();
        cudaMemcpyAsync(hostCounters, counters, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        std::swap(cur, nxt);
        if (hostCounters[1]) return -1;
        if (hostCounters[0] == 0) {
            if (cur != colA) cudaMemcpyAsync(colA, cur, sizeof(int) * static_cast<size_t>(rows), cudaMemcpyDeviceToDevice, s);
            return round + 1;
        }
    }
    throw std::runtime_error("bcs: multicolouring did not finish");
}

int mc_permutation(int rows, const int* color, int* perm, int* inv, int* scratch, size_t scratchInts, int* hostBuf,
                   cudaStream_t s) {
    // colours used
    int* cnt = scratch;
    cudaMemsetAsync(cnt, 0, sizeof(int) * (kMaxColors + 1), s);
    k_color_hist<<<(rows + 255) / 256, 256, 0, s>>>(rows, color, cnt);
    count_launch();
    cudaMemcpyAsync(hostBuf, cnt, sizeof(int) * (kMaxColors + 1), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    int ncol = 0;
    for (int c = 0; c < kMaxColors; ++c)
        if (hostBuf[c]) ncol = c + 1;
    const int nb = (rows + 1023) / 1024;
    const size_t need = static_cast<size_t>(nb) * ncol + 1;
    if (need + kMaxColors + 1 > scratchInts) throw std::logic_error("bcs: multicolour scratch too small");
    int* bc = scratch + kMaxColors + 1;
    k_color_rank<<<nb, 1024, 0, s>>>(rows, color, ncol, bc);
    count_launch();
    // exclusive scan in (colour, block) order: transpose on the host (nb*ncol is small)
    std::vector<int> hb(static_cast<size_t>(nb) * ncol);
    cudaMemcpyAsync(hb.data(), bc, sizeof(int) * hb.size(), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    std::vector<int> base(hb.size());
    int run = 0;
    for (int c = 0; c < ncol; ++c)
        for (int b = 0; b < nb; ++b) {
            base[static_cast<size_t>(b) * ncol + c] = run;
            run += hb[static_cast<size_t>(b) * ncol + c];
        }
    cudaMemcpyAsync(bc, base.data(), sizeof(int) * base.size(), cudaMemcpyHostToDevice, s);
    k_color_place<<<nb, 1024, 0, s>>>(rows, color, ncol, bc, perm, inv);
    count_launch();
    cudaStreamSynchronize(s);  // base dies here
    return ncol;
}

void mc_permute_pattern(int rows, const int* ro, const int* ci, const int* perm, const int* inv, int* nro, int* nci,
                        int* sv, int* scanTmp, int* dTotal, cudaStream_t s) {
    k_row_len_perm<<<(rows + 255) / 256, 256, 0, s>>>(rows, ro, perm, nro);
    cudaMemsetAsync(nro + rows, 0, sizeof(int), s);
    exclusive_scan(nro, rows + 1, dTotal, scanTmp, s);
    k_perm_rows<<<(rows + 127) / 128, 128, 0, s>>>(rows, ro, ci, perm, inv, nro, nci, sv);
    count_launch(2);
}

void mc_permute_values(int n, size_t nnz, const int* sv, const double* v, double* nv, cudaStream_t s) {
    const size_t tot = nnz * static_cast<size_t>(n) * n;
    const unsigned g = static_cast<unsigned>((tot + 255) / 256);
    switch (n) {
        case 1: k_gather_blocks<1><<<g, 256, 0, s>>>(nnz, sv, v, nv); break;
        case 2: k_gather_blocks<4><<<g, 256, 0, s>>>(nnz, sv, v, nv); break;
        case 3: k_gather_blocks<9><<<g, 256, 0, s>>>(nnz, sv, v, nv); break;
        case 4: k_gather_blocks<16><<<g, 256, 0, s>>>(nnz, sv, v, nv); break;
        default: k_gather_blocks<25><<<g, 256, 0, s>>>(nnz, sv, v, nv); break;
    }
    count_launch();
}

// vectors: xp[i'] = x[perm[i']] ; z[perm[i']] = (acc == 2 ? z : 0) + s[i'] (acc 1: 0 + s, acc 0: s)
__global__ void k_vec_gather(int n, int rows, const int* __restrict__ perm, const double* __restrict__ x, double* xp) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * n) return;
    const int ip = t / n, q = t - ip * n;
    xp[t] = x[static_cast<size_t>(perm[ip]) * n + q];
}
__global__ void k_vec_scatter(int n, int rows, const int* __restrict__ perm, const double* __restrict__ sp, double* z,
                              int acc) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * n) return;
    const int ip = t / n, q = t - ip * n;
    const size_t o = static_cast<size_t>(perm[ip]) * n + q;
    const double v = sp[t];
    z[o] = acc == 2 ? __dadd_rn(z[o], v) : acc == 1 ? __dadd_rn(0.0, v) : v;
}
void mc_vec_gather(int n, int rows, const int* perm, const double* x, double* xp, cudaStream_t s) {
    k_vec_gather<<<(rows * n + 255) / 256, 256, 0, s>>>(n, rows, perm, x, xp);
    count_launch();
}
void mc_vec_scatter(int n, int rows, const int* perm, const double* sp, double* z, int acc, cudaStream_t s) {
    k_vec_scatter<<<(rows * n + 255) / 256, 256, 0, s>>>(n, rows, perm, sp, z, acc);
    count_launch();
}


// ---- colour-synchronous sweeps of a coloured level --------------------------
// On the colour-permuted matrix every dependency of a row of colour c has a
// smaller colour (forward) / larger colour (backward), so the sweep is c
// rounds of independent rows: one cooperative kernel, grid barrier between
// colours, no per-row dependency polling and no staging -- an HBM stream over
// the level's triangle like an SpMV.  N lanes per row (lane q = component q),
// 32/N rows per warp; the arithmetic is k_sweep's (k_sweep.cu) operation for
// operation: acc = r_i - sum_k (A_ik y_k) per block in slot order (backward:
// 0 + sum over the upper slots from the last one down), the composed pivot
// permutation, the reciprocal-based LU solve with the exact IEEE fallback --
// so the result is bit-identical to the sync-free sweeps on the same matrix.
template <int N, bool FWD>
__global__ void __launch_bounds__(256) k_mc_sweep(int ncol, const int* __restrict__ coff, const int* __restrict__ ro,
                                                  const int* __restrict__ dg, const int* __restrict__ ci,
                                                  const double* __restrict__ v, const double* __restrict__ lu,
                                                  const double* __restrict__ rcp, const int* __restrict__ perm,
                                                  const double* __restrict__ rin, double* out) {
    namespace cg = cooperative_groups;
    constexpr int NN = N * N, G = 32 / N;
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, g = lane / N, q = lane - (lane / N) * N;
    const int warp = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int W = static_cast<int>((gridDim.x * blockDim.x) >> 5);
    for (int cc = 0; cc < ncol; ++cc) {
        const int c = FWD ? cc : ncol - 1 - cc;
        const int b = __ldg(&coff[c]), e = __ldg(&coff[c + 1]);
        for (int i0 = b + warp * G; i0 < e; i0 += W * G) {
            const int i = i0 + g;
            const bool row = g < G && i < e;
            double ri = 0.0, acc = 0.0;
            if (row) {
                ri = __ldg(&rin[static_cast<size_t>(i) * N + q]);
                acc = FWD ? ri : 0.0;
                const int k0 = __ldg(&ro[i]), kd = __ldg(&dg[i]), k1 = __ldg(&ro[i + 1]);
                if (FWD) {
                    for (int k = k0; k < kd; ++k) {
                        const double* a = v + static_cast<size_t>(k) * NN + q * N;
                        const double* y = out + static_cast<size_t>(__ldg(&ci[k])) * N;
                        double s = 0.0;
#pragma unroll
                        for (int p = 0; p < N; ++p) s = __dadd_rn(s, __dmul_rn(__ldg(&a[p]), __ldcg(&y[p])));
                        acc = __dsub_rn(acc, s);
                    }
                } else {
                    for (int k = k1 - 1; k > kd; --k) {
                        const double* a = v + static_cast<size_t>(k) * NN + q * N;
                        const double* y = out + static_cast<size_t>(__ldg(&ci[k])) * N;
                        double s = 0.0;
#pragma unroll
                        for (int p = 0; p < N; ++p) s = __dadd_rn(s, __dmul_rn(__ldg(&a[p]), __ldcg(&y[p])));
                        acc = __dadd_rn(acc, s);
                    }
                }
            }
            // composed pivot permutation: x[p] = acc of component perm[p] of this row
            const size_t ib = static_cast<size_t>(row ? i : 0);
            double x[N];
#pragma unroll
            for (int p = 0; p < N; ++p) {
                const int src = row ? g * N + __ldg(&perm[ib * N + p]) : lane;
                x[p] = __shfl_sync(0xffffffffu, acc, src);
            }
            if (row) {
                double lf[NN], rc[N];
#pragma unroll
                for (int t = 0; t < NN; ++t) lf[t] = __ldg(&lu[ib * NN + t]);
#pragma unroll
                for (int p = 0; p < N; ++p) rc[p] = __ldg(&rcp[ib * N + p]);
                DVec<N> xin;
#pragma unroll
                for (int p = 0; p < N; ++p) xin.v[p] = x[p];
                if (__builtin_expect(!lu_solve_perm_fast<N>(lf, rc, x), 0)) {
                    const DVec<N> xe = lu_solve_perm_exact<N>(lu + ib * NN, xin);
#pragma unroll
                    for (int p = 0; p < N; ++p) x[p] = xe.v[p];
                }
                double mine = x[0];
#pragma unroll
                for (int p = 1; p < N; ++p) mine = (q == p) ? x[p] : mine;
                out[ib * N + q] = FWD ? mine : __dsub_rn(ri, mine);
            }
        }
        if (cc + 1 < ncol) grid.sync();
    }
}

// ---- performance mode: one colour per launch -------------------------------
// Rows of one colour are independent, so a colour is a streaming pass: warps
// take G = 32/N rows (N lanes each, lane q = component q), issue the loads of
// up to kMcDeps dependency rows at once (block row q of A_ij from HBM, y_j[q]
// from the earlier colours' results), then fold them in slot order and solve
// with the row's LU -- the operation sequence of the sync-free sweeps, so the
// result is bit-identical to them.  Kernel boundaries order the colours.
constexpr int kMcDeps = 4;
constexpr int kMcWarps = 8;  // warps per CTA

__device__ __forceinline__ unsigned mc_smem(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// TMA bulk copy of [src, src + bytes) widened to 16-byte bounds into dst;
// returns the byte offset of src inside dst.  Caller counts the bytes.
__device__ __forceinline__ unsigned mc_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                            unsigned* tx) {
    const unsigned long long s0 = reinterpret_cast<unsigned long long>(src);
    const unsigned long long lo = s0 & ~15ull, hi = (s0 + bytes + 15ull) & ~15ull;
    const unsigned len = static_cast<unsigned>(hi - lo);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(mc_smem(dst)),
        "l"(lo), "r"(len), "r"(mc_smem(bar))
        : "memory");
    *tx += len;
    return static_cast<unsigned>(s0 - lo);
}

// rowmap (the coloured level's new -> original row map), when given: the
// forward reads its input r in the original numbering (the gather into the
// coloured order fused), the backward also writes its result to zfinal in the
// original numbering with k_vec_scatter's accumulate semantics (zacc; the
// scatter fused).
template <int N, bool FWD>
__global__ void __launch_bounds__(256, 4) k_mc_colour(int i0, int i1, const int* __restrict__ ro,
                                                   const int* __restrict__ dg, const int* __restrict__ ci,
                                                   const double* __restrict__ v, const double* __restrict__ lu,
                                                   const double* __restrict__ rcp, const int* __restrict__ perm,
                                                   const double* __restrict__ rin, double* out,
                                                   const int* __restrict__ rowmap, double* zfinal, int zacc) {
    constexpr int NN = N * N, G = 32 / N, RB = kMcWarps * G;  // rows per CTA
    // the CTA's rows' factors, reciprocals and permutations (contiguous in the
    // colour-ordered level) arrive by TMA while the warps fold their dependencies
    __shared__ alignas(16) double slu[RB * NN + 2];
    __shared__ alignas(16) double src_[RB * N + 2];
    __shared__ alignas(16) int spm[RB * N + 4];
    __shared__ alignas(8) unsigned long long bar;
    __shared__ unsigned offs[3];
    const int lane = threadIdx.x & 31, g = lane / N, q = lane - (lane / N) * N;
    const int wib = threadIdx.x >> 5;
    const int c0row = i0 + blockIdx.x * RB;
    const int nrow = i1 - c0row < RB ? i1 - c0row : RB;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mc_smem(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        unsigned tx = 0;
        const size_t r0 = static_cast<size_t>(c0row);
        // expect_tx after the byte count is known: arrive once with the total
        offs[0] = mc_bulk(slu, lu + r0 * NN, nrow * NN * 8, &bar, &tx);
        offs[1] = mc_bulk(src_, rcp + r0 * N, nrow * N * 8, &bar, &tx);
        offs[2] = mc_bulk(spm, perm + r0 * N, nrow * N * 4, &bar, &tx);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mc_smem(&bar)), "r"(tx) : "memory");
    }
    const int li = wib * G + g;  // row within the CTA
    const int i = c0row + li;
    const bool row = g < G && li < nrow;
    const size_t ib = static_cast<size_t>(row ? i : c0row);
    double ri = 0.0;
    int kb = 0, cnt = 0;
    const size_t orig = rowmap && row ? static_cast<size_t>(__ldg(&rowmap[ib])) : ib;  // original row
    if (row) {
        ri = FWD && rowmap ? __ldg(&rin[orig * N + q]) : __ldg(&rin[ib * N + q]);
        const int k0 = __ldg(&ro[ib]), kd = __ldg(&dg[ib]), k1 = __ldg(&ro[ib + 1]);
        kb = FWD ? k0 : k1 - 1;
        cnt = FWD ? kd - k0 : k1 - 1 - kd;
    }
    double acc = FWD ? ri : 0.0;
    const int cmax = __reduce_max_sync(0xffffffffu, cnt);
    for (int cc = 0; cc < cmax; cc += kMcDeps) {
        double aq[kMcDeps][N], yq[kMcDeps];
#pragma unroll
        for (int d = 0; d < kMcDeps; ++d) {
            const int c = cc + d;
            const int k = FWD ? kb + c : kb - c;
            if (c < cnt) {
                const double* a = v + static_cast<size_t>(k) * NN + q * N;
#pragma unroll
                for (int p = 0; p < N; ++p) aq[d][p] = __ldcs(&a[p]);
                yq[d] = __ldcg(&out[static_cast<size_t>(__ldg(&ci[k])) * N + q]);
            } else {
#pragma unroll
                for (int p = 0; p < N; ++p) aq[d][p] = 0.0;
                yq[d] = 0.0;
            }
        }
#pragma unroll
        for (int d = 0; d < kMcDeps; ++d) {
            double sblk = 0.0;
#pragma unroll
            for (int p = 0; p < N; ++p)
                sblk = __dadd_rn(sblk, __dmul_rn(aq[d][p], __shfl_sync(0xffffffffu, yq[d], g * N + p)));
            if (cc + d < cnt) acc = FWD ? __dsub_rn(acc, sblk) : __dadd_rn(acc, sblk);
        }
    }
    __syncthreads();  // barrier initialised and offsets published
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra W;\n\t}" ::"r"(mc_smem(&bar))
        : "memory");
    const double* L = reinterpret_cast<const double*>(reinterpret_cast<const unsigned char*>(slu) + offs[0]) +
                      (row ? li : 0) * NN;
    const double* rc = reinterpret_cast<const double*>(reinterpret_cast<const unsigned char*>(src_) + offs[1]) +
                       (row ? li : 0) * N;
    const int* pm = reinterpret_cast<const int*>(reinterpret_cast<const unsigned char*>(spm) + offs[2]) +
                    (row ? li : 0) * N;
    // composed pivot permutation, then the row's LU solve (every lane of the row)
    double x[N];
#pragma unroll
    for (int p = 0; p < N; ++p) {
        const int sl = row ? g * N + pm[p] : lane;
        x[p] = __shfl_sync(0xffffffffu, acc, sl);
    }
    if (!row) return;
    DVec<N> xin;
#pragma unroll
    for (int p = 0; p < N; ++p) xin.v[p] = x[p];
    if (__builtin_expect(!lu_solve_perm_fast<N>(L, rc, x), 0)) {
        const DVec<N> xe = lu_solve_perm_exact<N>(lu + ib * NN, xin);
#pragma unroll
        for (int p = 0; p < N; ++p) x[p] = xe.v[p];
    }
    double mine = x[0];
#pragma unroll
    for (int p = 1; p < N; ++p) mine = (q == p) ? x[p] : mine;
    const double res = FWD ? mine : __dsub_rn(ri, mine);
    out[ib * N + q] = res;
    if (!FWD && zfinal) {
        const size_t o = orig * N + q;
        zfinal[o] = zacc == 2 ? __dadd_rn(zfinal[o], res) : zacc == 1 ? __dadd_rn(0.0, res) : res;
    }
}

void mc_colour_sweep(int n, bool fwd, int i0, int i1, const int* ro, const int* dg, const int* ci, const double* v,
                     const double* lu, const double* rcp, const int* perm, const double* rin, double* out,
                     const int* rowmap, double* zfinal, int acc, cudaStream_t s) {
    if (i1 <= i0) return;
    const long long rb = static_cast<long long>(kMcWarps) * (32 / n);  // rows per CTA
    const unsigned g = static_cast<unsigned>((static_cast<long long>(i1 - i0) + rb - 1) / rb);
    switch (n) {
#define BCS_MCC_CASE(NV)                                                                                        \
    case NV:                                                                                                    \
        if (fwd) k_mc_colour<NV, true><<<g, 256, 0, s>>>(i0, i1, ro, dg, ci, v, lu, rcp, perm, rin, out, rowmap,  \
                                                         zfinal, acc);                                         \
        else k_mc_colour<NV, false><<<g, 256, 0, s>>>(i0, i1, ro, dg, ci, v, lu, rcp, perm, rin, out, rowmap,  \
                                                      zfinal, acc);                                            \
        break;
        BCS_MCC_CASE(1)
        BCS_MCC_CASE(2)
        BCS_MCC_CASE(3)
        BCS_MCC_CASE(4)
        BCS_MCC_CASE(5)
#undef BCS_MCC_CASE
        default: throw std::invalid_argument("block size must be 1..5 on the device");
    }
    count_launch();
}

// ---- performance mode, block-Jacobi smoothing ------------------------------
// out_i = omega * D_i^-1 r_i per block row (the diagonal block's LU with the
// composed pivot permutation and reciprocal-based division, as the sweeps),
// z = out | 0 + out | z + out by `acc` (the V-cycle's pre/post-smoothing
// forms).  No dependencies: one pass over the factors, HBM-bound.  Every
// per-row array (factors, reciprocals, permutation, r, z) moves between HBM
// and shared memory with coalesced 16-byte streaming accesses; a thread then
// solves one row out of shared memory.
constexpr int kJacRows = 128;

// fallback copy (unaligned tails): 4-byte words
__device__ __forceinline__ void jac_load_words(void* dst, const void* src, int bytes) {
    const int* s1 = reinterpret_cast<const int*>(src);
    int* d1 = reinterpret_cast<int*>(dst);
    for (int e = threadIdx.x; e < bytes / 4; e += blockDim.x) d1[e] = __ldcs(&s1[e]);
}
__device__ __forceinline__ unsigned jac_smem(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// one TMA bulk copy global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void jac_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(jac_smem(dst)),
        "l"(src), "r"(bytes), "r"(jac_smem(bar))
        : "memory");
}

template <int N>
__global__ void __launch_bounds__(kJacRows) k_block_jacobi(int rows, const double* __restrict__ lu,
                                                          const double* __restrict__ rcp, const int* __restrict__ perm,
                                                          const double* __restrict__ r, double* z, int acc,
                                                          double omega) {
    constexpr int NN = N * N;
    __shared__ alignas(16) double sl[kJacRows * NN];
    __shared__ alignas(16) double sr[kJacRows * N];
    __shared__ alignas(16) double sc[kJacRows * N];
    __shared__ alignas(16) double sz[kJacRows * N];
    __shared__ alignas(16) int sp[kJacRows * N];
    __shared__ alignas(8) unsigned long long bar;
    const int r0 = blockIdx.x * kJacRows;
    const int nrow = rows - r0 < kJacRows ? rows - r0 : kJacRows;
    const size_t b0 = static_cast<size_t>(r0) * N;
    // the block's rows arrive by TMA bulk copies (one thread issues them, no
    // register round trip); sizes and addresses are 16-byte multiples except
    // possibly in the last block, which copies word by word
    const unsigned bl = nrow * NN * 8, bv = nrow * N * 8, bp = nrow * N * 4;
    const bool bulk = ((reinterpret_cast<unsigned long long>(lu + b0 * N) | reinterpret_cast<unsigned long long>(r + b0) |
                        reinterpret_cast<unsigned long long>(rcp + b0) | reinterpret_cast<unsigned long long>(perm + b0) |
                        reinterpret_cast<unsigned long long>(z + b0) | bl | bv | bp) & 15) == 0;
    if (bulk) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(jac_smem(&bar)) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            const unsigned tx = bl + 2 * bv + bp + (acc == 2 ? bv : 0);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(jac_smem(&bar)), "r"(tx)
                         : "memory");
            jac_bulk(sl, lu + b0 * N, bl, &bar);
            jac_bulk(sr, r + b0, bv, &bar);
            jac_bulk(sc, rcp + b0, bv, &bar);
            jac_bulk(sp, perm + b0, bp, &bar);
            if (acc == 2) jac_bulk(sz, z + b0, bv, &bar);
        }
        __syncthreads();  // barrier initialised before anyone waits on it
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra W;\n\t}" ::"r"(jac_smem(&bar))
            : "memory");
    } else {
        jac_load_words(sl, lu + b0 * N, bl);
        jac_load_words(sr, r + b0, bv);
        jac_load_words(sc, rcp + b0, bv);
        jac_load_words(sp, perm + b0, bp);
        if (acc == 2) jac_load_words(sz, z + b0, bv);
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t < nrow) {
        double rv[N], x[N], rc[N];
#pragma unroll
        for (int q = 0; q < N; ++q) {
            rv[q] = sr[t * N + q];
            rc[q] = sc[t * N + q];
        }
#pragma unroll
        for (int p = 0; p < N; ++p) {
            const int spp = sp[t * N + p];
            double v = rv[0];
#pragma unroll
            for (int q = 1; q < N; ++q) v = (spp == q) ? rv[q] : v;
            x[p] = v;
        }
        DVec<N> xin;
#pragma unroll
        for (int p = 0; p < N; ++p) xin.v[p] = x[p];
        const double* L = sl + t * NN;
        if (__builtin_expect(!lu_solve_perm_fast<N>(L, rc, x), 0)) {
            const DVec<N> xe = lu_solve_perm_exact<N>(L, xin);
#pragma unroll
            for (int p = 0; p < N; ++p) x[p] = xe.v[p];
        }
#pragma unroll
        for (int q = 0; q < N; ++q) {
            const double o = __dmul_rn(omega, x[q]);
            sz[t * N + q] = acc == 2 ? __dadd_rn(sz[t * N + q], o) : acc == 1 ? __dadd_rn(0.0, o) : o;
        }
    }
    __syncthreads();
    // coalesced store of the block's results
    double* dz = z + b0;
    const int nd = nrow * N;
    if ((reinterpret_cast<unsigned long long>(dz) & 15) == 0 && (nd & 1) == 0) {
        const double2* s2 = reinterpret_cast<const double2*>(sz);
        double2* d2 = reinterpret_cast<double2*>(dz);
        for (int e = threadIdx.x; e < nd / 2; e += blockDim.x) __stcs(&d2[e], s2[e]);
    } else {
        for (int e = threadIdx.x; e < nd; e += blockDim.x) __stcs(&dz[e], sz[e]);
    }
}

void block_jacobi(int n, int rows, const double* lu, const double* rcp, const int* perm, const double* r, double* z,
                  int acc, double omega, cudaStream_t s) {
    if (rows <= 0) return;
    const unsigned g = static_cast<unsigned>((rows + kJacRows - 1) / kJacRows);
    switch (n) {
        case 1: k_block_jacobi<1><<<g, kJacRows, 0, s>>>(rows, lu, rcp, perm, r, z, acc, omega); break;
        case 2: k_block_jacobi<2><<<g, kJacRows, 0, s>>>(rows, lu, rcp, perm, r, z, acc, omega); break;
        case 3: k_block_jacobi<3><<<g, kJacRows, 0, s>>>(rows, lu, rcp, perm, r, z, acc, omega); break;
        case 4: k_block_jacobi<4><<<g, kJacRows, 0, s>>>(rows, lu, rcp, perm, r, z, acc, omega); break;
        default: k_block_jacobi<5><<<g, kJacRows, 0, s>>>(rows, lu, rcp, perm, r, z, acc, omega); break;
    }
    count_launch();
}

template <int N, bool FWD>
static void launch_mc_sweep(int rows, int ncol, const int* coff, const int* ro, const int* dg, const int* ci,
                            const double* v, const double* lu, const double* rcp, const int* perm, const double* rin,
                            double* out, cudaStream_t s) {
    static int cap = 0;
    {
        std::lock_guard<std::recursive_mutex> lazy_lk(lazy_init_mutex());
        if (!cap) {
            int bps = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_mc_sweep<N, FWD>, 256, 0);
            cap = num_sms() * (bps < 1 ? 1 : bps);
        }
    }
    constexpr int G = 32 / N;
    long long want = (static_cast<long long>(rows) / G + 63) / 64;  // ~8 row groups per warp per pass over the level
    int g = static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
    void* args[] = {(void*)&ncol, (void*)&coff, (void*)&ro, (void*)&dg, (void*)&ci, (void*)&v,
                    (void*)&lu, (void*)&rcp, (void*)&perm, (void*)&rin, (void*)&out};
    const cudaError_t e = cudaLaunchCooperativeKernel((void*)k_mc_sweep<N, FWD>, dim3(g), dim3(256), args, 0, s);
    if (e != cudaSuccess) throw std::runtime_error(std::string("colour sweep launch failed: ") + cudaGetErrorString(e));
    count_launch();
}

void mc_sweep(int n, bool fwd, int rows, int ncol, const int* coff, const int* ro, const int* dg, const int* ci,
              const double* v, const double* lu, const double* rcp, const int* perm, const double* rin, double* out,
              cudaStream_t s) {
    if (rows <= 0) return;
    switch (n) {
#define BCS_MC_CASE(NV)                                                                                            \
    case NV:                                                                                                       \
        if (fwd) launch_mc_sweep<NV, true>(rows, ncol, coff, ro, dg, ci, v, lu, rcp, perm, rin, out, s);           \
        else launch_mc_sweep<NV, false>(rows, ncol, coff, ro, dg, ci, v, lu, rcp, perm, rin, out, s);              \
        break;
        BCS_MC_CASE(1)
        BCS_MC_CASE(2)
        BCS_MC_CASE(3)
        BCS_MC_CASE(4)
        BCS_MC_CASE(5)
#undef BCS_MC_CASE
        default: throw std::invalid_argument("block size must be 1..5 on the device");
    }
}

}  // namespace bcs
