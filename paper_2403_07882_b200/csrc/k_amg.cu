// K9-K12: pairwise-aggregation AMG setup and transfer operators.
//
// Reference: pairwiseAggregate (amg.cpp:10-37), galerkinCoarse (:39-71),
// hierarchy/dense coarsest (:73-105), V-cycle transfers (:111-158).
//
// Aggregation is a sequential greedy matching in row order.  Its exact
// parallel form: row r's decision depends only on (a) its lower neighbours
// (was r already taken?) and (b) the lower-than-r neighbours of each upper
// neighbour j (is j still free?).  k_agg_syncfree resolves that DAG
// sync-free: rows are taken in index order by co-resident warps (cooperative
// launch), each polls the decisions it depends on and decides as soon as they
// are known, which equals the sequential decision (the round-synchronous Kahn
// form, k_agg_rounds, is kept behind BCS_AGG_MODE=1).  Strengths are computed with the reference's operation
// order (sequential Frobenius sums, IEEE sqrt/div, no FMA), so the integer
// aggregates are bit-identical.  Galerkin sums are taken per coarse block in
// (fine row ascending, slot ascending) order from +0.0 — also bit-identical.
#include "device.cuh"
#include "kernels.hpp"

#include <cooperative_groups.h>
#include <stdexcept>
#include <string>

namespace cg = cooperative_groups;

namespace bcs {

#define BCS_DISPATCH_N(n, ...)                                                        \
    switch (n) {                                                                      \
        case 1: { constexpr int N = 1; __VA_ARGS__; } break;                          \
        case 2: { constexpr int N = 2; __VA_ARGS__; } break;                          \
        case 3: { constexpr int N = 3; __VA_ARGS__; } break;                          \
        case 4: { constexpr int N = 4; __VA_ARGS__; } break;                          \
        case 5: { constexpr int N = 5; __VA_ARGS__; } break;                          \
        default: throw std::invalid_argument("block size must be 1..5 on the device"); \
    }

// ------------------------------------------------------------- strengths
template <int N>
__global__ void k_diag_norm(int rows, const int* __restrict__ dg, const double* __restrict__ v, double* dn) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int d = dg[r];
    dn[r] = d >= 0 ? frob<N>(v + static_cast<size_t>(d) * N * N) : 0.0;
}

// str[k] = ||A_k||_F / sqrt(max(dn_r dn_j, 1e-300))   (amg.cpp:27-28).
// Same values, block-parallel: a CTA stages 256 consecutive blocks through
// shared memory with coalesced 16-byte loads (a thread per row would read
// 200-byte blocks 8 bytes at a time from 32 rows at once), then thread t
// takes block k0 + t: row by binary search, sequential Frobenius sum.
constexpr int kStrChunk = 256;
template <int N>
__global__ void __launch_bounds__(kStrChunk) k_strength_blk(int rows, int nnz, const int* __restrict__ ro,
                                                            const int* __restrict__ ci,
                                                            const double* __restrict__ v,
                                                            const double* __restrict__ dn, double* str) {
    constexpr int NN = N * N;
    extern __shared__ __align__(16) double sblk[];
    const int k0 = blockIdx.x * kStrChunk;
    const int cnt = nnz - k0 < kStrChunk ? nnz - k0 : kStrChunk;
    const double* src = v + static_cast<size_t>(k0) * NN;
    const int tot = cnt * NN;
    if ((NN & 1) == 0 || (k0 & 1) == 0) {  // 16-byte aligned source (k0 is a multiple of 256)
        const int t2 = tot >> 1;
        for (int e = threadIdx.x; e < t2; e += blockDim.x)
            reinterpret_cast<double2*>(sblk)[e] = __ldcs(reinterpret_cast<const double2*>(src) + e);
        if ((tot & 1) && threadIdx.x == 0) sblk[tot - 1] = __ldcs(src + tot - 1);
    } else {
        for (int e = threadIdx.x; e < tot; e += blockDim.x) sblk[e] = __ldcs(src + e);
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t >= cnt) return;
    const int k = k0 + t;
    int lo = 0, hi = rows - 1;  // last row with ro[row] <= k
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(&ro[mid]) <= k) lo = mid;
        else hi = mid - 1;
    }
    const double prod = __dmul_rn(__ldg(&dn[lo]), __ldg(&dn[__ldg(&ci[k])]));
    const double den = __dsqrt_rn(prod < 1e-300 ? 1e-300 : prod);  // std::max(prod, 1e-300)
    str[k] = __ddiv_rn(frob<N>(sblk + t * NN), den);
}

void strengths(int n, int rows, const int* ro, const int* ci, const int* dg, const double* v, double* dn,
               double* str, int nnz, cudaStream_t s) {
    const unsigned g = (rows + 255) / 256;
    if (!g) return;
    const unsigned gb = (nnz + kStrChunk - 1) / kStrChunk;
    BCS_DISPATCH_N(n, {
        static bool attr = false;
        {
            std::lock_guard<std::recursive_mutex> lazy_lk(lazy_init_mutex());
            if (!attr) {
                cudaFuncSetAttribute(k_strength_blk<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sizeof(double) * kStrChunk * N * N));
                attr = true;
            }
        }
        k_diag_norm<N><<<g, 256, 0, s>>>(rows, dg, v, dn);
        k_strength_blk<N><<<gb, kStrChunk, sizeof(double) * kStrChunk * N * N, s>>>(rows, nnz, ro, ci, v, dn, str);
    });
    count_launch(2);
}

// ------------------------------------------------------------ aggregation
constexpr int kTaken = -2;
constexpr int kSingle = -1;
int last_agg_rounds = 0;

// Exact parallel greedy (lazy readiness).  A row becomes *active* once all
// its lower neighbours are decided (1-hop Kahn counter).  An active row then
// tries to decide with the decisions visible so far:
//   * taken   iff a lower neighbour chose it (all of them are decided);
//   * else it walks its upper neighbours in the reference's preference order
//     (strength descending, column ascending == the first max of the
//     sequential scan) and for each inspects the lower-than-r entries of that
//     neighbour's row: if one of them chose it, it is taken (skip); if one is
//     still undecided, the outcome is unknown and the row retries next round;
//     otherwise it is free and becomes the partner.
// Every conclusion drawn is one the sequential algorithm draws at time r, so
// the result is bit-identical; the smallest undecided row always decides, so
// the rounds terminate.  choice[r]: -3 undecided, -2 taken, -1 singleton,
// >= 0 partner.
constexpr int kUndecided = -3;

__global__ void k_agg_init(int rows, const int* __restrict__ ro, const int* __restrict__ dg, int* cnt, int* choice,
                           int* act, int* push) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int c = dg[r] - ro[r];
    cnt[r] = c;
    choice[r] = kUndecided;
    if (c == 0) act[atomicAdd(&push[2], 1)] = r;
}

constexpr unsigned kAll = 0xffffffffu;

// (s, k) is preferred over (s2, k2): larger strength, ties by smaller slot
__device__ __forceinline__ bool preferred(double s, int k, double s2, int k2) {
    return k2 < 0 || (k >= 0 && (s > s2 || (s == s2 && k < k2)));
}

// One warp decides row r (lane-parallel scans; see the comment above).
__device__ __forceinline__ int agg_try_warp(int r, int lane, const int* __restrict__ ro, const int* __restrict__ ci,
                                            const int* __restrict__ dg, const int* __restrict__ tpos,
                                            const double* __restrict__ str, const int* choice) {
    const int b = __ldg(&ro[r]), d = __ldg(&dg[r]), e = __ldg(&ro[r + 1]);
    bool taken = false;
    for (int k = b + lane; k < d; k += 32) taken |= __ldcg(&choice[__ldg(&ci[k])]) == r;
    if (__any_sync(kAll, taken)) return kTaken;
    double lastS = 0.0;
    int lastK = -1;  // -1: nothing excluded yet
    while (true) {
        double bs = 0.0;
        int bk = -1;
        for (int k = d + 1 + lane; k < e; k += 32) {
            const double sv = __ldg(&str[k]);
            if (!(sv > -1.0)) continue;  // NaN never wins (reference: s > best)
            if (lastK >= 0 && !(sv < lastS || (sv == lastS && k > lastK))) continue;
            if (preferred(sv, k, bs, bk)) {
                bs = sv;
                bk = k;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double os = __shfl_xor_sync(kAll, bs, o);
            const int ok = __shfl_xor_sync(kAll, bk, o);
            if (preferred(os, ok, bs, bk)) {
                bs = os;
                bk = ok;
            }
        }
        if (bk < 0) return kSingle;
        lastS = bs;
        lastK = bk;
        const int j = __ldg(&ci[bk]);
        const int tp = __ldg(&tpos[bk]);
        bool tk = false, unk = false;
        for (int kk = __ldg(&ro[j]) + lane; kk < tp; kk += 32) {
            const int c = __ldcg(&choice[__ldg(&ci[kk])]);
            tk |= c == j;
            unk |= c == kUndecided;
        }
        if (__any_sync(kAll, tk)) continue;
        if (__any_sync(kAll, unk)) return kUndecided;
        return j;
    }
}

template <bool GRID>
__global__ void __launch_bounds__(256) k_agg_rounds(int rows, const int* __restrict__ ro, const int* __restrict__ ci,
                                                    const int* __restrict__ dg, const int* __restrict__ tpos,
                                                    const double* __restrict__ str, int* choice, int* cnt,
                                                    int* actA, int* actB, int* push, int* out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    int round = 0;
    int* cur = actA;
    int* nxt = actB;
    while (true) {
        const int c = __ldcg(&push[(round + 2) % 3]);
        if (c == 0) break;
        if (blockIdx.x == 0 && threadIdx.x == 0) push[(round + 1) % 3] = 0;
        int* pc = &push[round % 3];
        for (int t = warp; t < c; t += nw) {
            const int r = __ldcg(&cur[t]);
            const int dec = agg_try_warp(r, lane, ro, ci, dg, tpos, str, choice);
            if (dec == kUndecided) {
                if (lane == 0) nxt[atomicAdd(pc, 1)] = r;
                continue;
            }
            if (lane == 0) atomicExch(&choice[r], dec);
            const int ub = __ldg(&dg[r]) + 1, ue = __ldg(&ro[r + 1]);
            for (int kb = ub; kb < ue; kb += 32) {
                const int k = kb + lane;
                bool ready = false;
                int j = 0;
                if (k < ue) {
                    j = __ldg(&ci[k]);
                    ready = atomicSub(&cnt[j], 1) == 1;
                }
                const unsigned m = __ballot_sync(kAll, ready);
                if (m) {
                    int base = 0;
                    if (lane == 0) base = atomicAdd(pc, __popc(m));
                    base = __shfl_sync(kAll, base, 0);
                    if (ready) nxt[base + __popc(m & ((1u << lane) - 1u))] = j;
                }
            }
        }
        int* tmp = cur;
        cur = nxt;
        nxt = tmp;
        ++round;
        if (GRID) {
            cg::this_grid().sync();
        } else {
            __syncthreads();
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = round;
}

// ---- sync-free variant: thread per row, rows statically in index order.
// Each warp loops until all of its lanes have decided; an undecided lane
// re-evaluates with the decisions visible so far (relaxed loads).  Deadlock
// freedom: the globally smallest undecided row sits in the current batch of
// its (co-resident) warp and all its dependencies are decided.
__device__ __forceinline__ int ld_choice(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ int agg_try_thread(int r, const int* __restrict__ ro, const int* __restrict__ ci,
                                              const int* __restrict__ dg, const int* __restrict__ tpos,
                                              const double* __restrict__ str, const int* choice) {
    const int b = __ldg(&ro[r]), d = __ldg(&dg[r]), e = __ldg(&ro[r + 1]);
    bool lowUndecided = false;
    for (int k = b; k < d; ++k) {
        const int c = ld_choice(&choice[__ldg(&ci[k])]);
        if (c == r) return kTaken;
        lowUndecided |= c == kUndecided;
    }
    if (lowUndecided) return kUndecided;
    double lastS = 0.0;
    int lastK = -1;
    while (true) {
        double bs = 0.0;
        int bk = -1;
        for (int k = d + 1; k < e; ++k) {
            const double sv = __ldg(&str[k]);
            if (!(sv > -1.0)) continue;
            if (lastK >= 0 && !(sv < lastS || (sv == lastS && k > lastK))) continue;
            if (bk < 0 || sv > bs) {
                bs = sv;
                bk = k;
            }
        }
        if (bk < 0) return kSingle;
        lastS = bs;
        lastK = bk;
        const int j = __ldg(&ci[bk]);
        const int tp = __ldg(&tpos[bk]);
        bool tk = false, unk = false;
        for (int kk = __ldg(&ro[j]); kk < tp; ++kk) {
            const int c = ld_choice(&choice[__ldg(&ci[kk])]);
            if (c == j) {
                tk = true;
                break;
            }
            unk |= c == kUndecided;
        }
        if (tk) continue;
        if (unk) return kUndecided;
        return j;
    }
}

__global__ void k_agg_fill(int rows, int* choice) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < rows) choice[r] = kUndecided;
}

// Resumable per-row state of the lazy greedy decision: every attempt
// continues from the first input that was still undecided, so a row issues
// one dependent load chain over its whole lifetime instead of one per attempt.
template <int AL>
__global__ void __launch_bounds__(256) k_agg_syncfree(int rows, const int* __restrict__ ro, const int* __restrict__ ci,
                                                      const int* __restrict__ dg, const int* __restrict__ tpos,
                                                      const double* __restrict__ str, int* choice, int* err) {
    const int T = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int base0 = tid - (threadIdx.x & 31);
    for (int base = base0; base < rows; base += T) {
        const int r = base + (threadIdx.x & 31);
        bool done = r >= rows;
        // phase A: lower neighbours of r (was r taken by one of them?)
        int k = done ? 0 : __ldg(&ro[r]);
        const int d = done ? 0 : __ldg(&dg[r]);
        const int e = done ? 0 : __ldg(&ro[r + 1]);
        bool phaseB = false;
        // phase B: current candidate (preference order: strength desc, slot asc)
        double lastS = 0.0;
        int lastK = -1, j = -1, kk = 0, tp = 0;
        // fast path: the row's lower columns and its two preferred candidates
        // (with their lower-than-r columns) are static, so every input of a
        // decision is loaded in one round of independent loads
        constexpr int AJ = AL;  // AL: static lower / candidate columns kept per row
        int lc[AL], jc0[AJ], jc1[AJ];
        int c0 = -1, c1 = -1, j0 = -1, j1 = -1, n0 = 0, n1 = 0;
        double s0 = 0.0, s1 = 0.0;
        bool fast = false;
        if (!done) {
            const int nl = d - k;
            double bs0 = 0.0, bs1 = 0.0;
            for (int q = d + 1; q < e; ++q) {
                const double sv = __ldg(&str[q]);
                if (!(sv > -1.0)) continue;
                if (c0 < 0 || sv > bs0) {
                    bs1 = bs0;
                    c1 = c0;
                    bs0 = sv;
                    c0 = q;
                } else if (c1 < 0 || sv > bs1) {
                    bs1 = sv;
                    c1 = q;
                }
            }
            s0 = bs0;
            s1 = bs1;
            int t0 = 0, t1 = 0;
            if (c0 >= 0) {
                j0 = __ldg(&ci[c0]);
                t0 = __ldg(&tpos[c0]);
                n0 = t0 - __ldg(&ro[j0]);
            }
            if (c1 >= 0) {
                j1 = __ldg(&ci[c1]);
                t1 = __ldg(&tpos[c1]);
                n1 = t1 - __ldg(&ro[j1]);
            }
            fast = nl <= AL && n0 <= AJ && n1 <= AJ;
            if (fast) {
#pragma unroll
                for (int q = 0; q < AL; ++q) lc[q] = q < nl ? __ldg(&ci[k + q]) : -1;
#pragma unroll
                for (int q = 0; q < AJ; ++q) {
                    jc0[q] = q < n0 ? __ldg(&ci[t0 - n0 + q]) : -1;
                    jc1[q] = q < n1 ? __ldg(&ci[t1 - n1 + q]) : -1;
                }
            }
        }
        unsigned spins = 0;
        while (!__all_sync(0xffffffffu, done)) {
            if (!done && fast) {
                int a[AL], b0[AJ], b1[AJ];
#pragma unroll
                for (int q = 0; q < AL; ++q) a[q] = lc[q] >= 0 ? ld_choice(&choice[lc[q]]) : kSingle;
#pragma unroll
                for (int q = 0; q < AJ; ++q) {
                    b0[q] = jc0[q] >= 0 ? ld_choice(&choice[jc0[q]]) : kSingle;
                    b1[q] = jc1[q] >= 0 ? ld_choice(&choice[jc1[q]]) : kSingle;
                }
                bool tk = false, un = false;
#pragma unroll
                for (int q = 0; q < AL; ++q) {
                    tk |= a[q] == r;
                    un |= a[q] == kUndecided;
                }
                int dec = kUndecided;
                if (tk) {
                    dec = kTaken;
                } else if (!un) {
                    if (c0 < 0) {
                        dec = kSingle;
                    } else {
                        bool t0k = false, u0 = false;
#pragma unroll
                        for (int q = 0; q < AJ; ++q) {
                            t0k |= b0[q] == j0;
                            u0 |= b0[q] == kUndecided;
                        }
                        if (!t0k) {
                            if (!u0) dec = j0;
                        } else if (c1 < 0) {
                            dec = kSingle;
                        } else {
                            bool t1k = false, u1 = false;
#pragma unroll
                            for (int q = 0; q < AJ; ++q) {
                                t1k |= b1[q] == j1;
                                u1 |= b1[q] == kUndecided;
                            }
                            if (!t1k) {
                                if (!u1) dec = j1;
                            } else {
                                // both preferred candidates taken: continue in the
                                // general walk after the second one
                                fast = false;
                                phaseB = true;
                                k = d;
                                lastS = s1;
                                lastK = c1;
                                j = -1;
                            }
                        }
                    }
                }
                if (dec != kUndecided) {
                    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(&choice[r]), "r"(dec) : "memory");
                    done = true;
                }
            } else if (!done) {
                int dec = kUndecided;
                if (!phaseB) {
                    for (; k < d; ++k) {
                        const int c = ld_choice(&choice[__ldg(&ci[k])]);
                        if (c == kUndecided) break;
                        if (c == r) {
                            dec = kTaken;
                            break;
                        }
                    }
                    if (dec == kUndecided && k == d) phaseB = true;
                }
                while (phaseB && dec == kUndecided) {
                    if (j < 0) {  // next candidate after (lastS, lastK)
                        double bs = 0.0;
                        int bk = -1;
                        for (int q = d + 1; q < e; ++q) {
                            const double sv = __ldg(&str[q]);
                            if (!(sv > -1.0)) continue;
                            if (lastK >= 0 && !(sv < lastS || (sv == lastS && q > lastK))) continue;
                            if (bk < 0 || sv > bs) {
                                bs = sv;
                                bk = q;
                            }
                        }
                        if (bk < 0) {
                            dec = kSingle;
                            break;
                        }
                        lastS = bs;
                        lastK = bk;
                        j = __ldg(&ci[bk]);
                        tp = __ldg(&tpos[bk]);
                        kk = __ldg(&ro[j]);
                    }
                    // was j taken by one of its lower neighbours below r?
                    bool taken = false, wait = false;
                    for (; kk < tp; ++kk) {
                        const int c = ld_choice(&choice[__ldg(&ci[kk])]);
                        if (c == kUndecided) {
                            wait = true;
                            break;
                        }
                        if (c == j) {
                            taken = true;
                            break;
                        }
                    }
                    if (wait) break;
                    if (taken) {
                        j = -1;
                        continue;
                    }
                    dec = j;
                }
                if (dec != kUndecided) {
                    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(&choice[r]), "r"(dec) : "memory");
                    done = true;
                }
            }
            if (++spins > (1u << 24)) {
                if (!done) atomicExch(err, 1);
                break;
            }
        }
    }
}

void aggregate_syncfree(int rows, const int* ro, const int* ci, const int* dg, const int* tpos, const double* str,
                        int* choice, int* err, cudaStream_t s) {
    if (rows <= 0) return;
    k_agg_fill<<<(rows + 255) / 256, 256, 0, s>>>(rows, choice);
    // big fine levels (low degree): the lean variant, more threads in flight;
    // coarse levels (higher degree): more columns kept per row
    const bool lean = rows >= (1 << 20);
    static int cap[2] = {0, 0};
    std::unique_lock<std::recursive_mutex> lazy_lk(lazy_init_mutex());
    if (!cap[0]) {
        int bps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_agg_syncfree<6>, 256, 0);
        cap[0] = num_sms() * (bps < 1 ? 1 : bps);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_agg_syncfree<10>, 256, 0);
        cap[1] = num_sms() * (bps < 1 ? 1 : bps);
    }
    lazy_lk.unlock();
    int g = (rows + 255) / 256;
    const int c = cap[lean ? 0 : 1];
    if (g > c) g = c;
    void* args[] = {(void*)&rows, (void*)&ro, (void*)&ci, (void*)&dg, (void*)&tpos, (void*)&str, (void*)&choice,
                    (void*)&err};
    const cudaError_t e = cudaLaunchCooperativeKernel(lean ? (void*)k_agg_syncfree<6> : (void*)k_agg_syncfree<10>,
                                                      dim3(g), dim3(256), args, 0, s);
    if (e != cudaSuccess) throw std::runtime_error(std::string("aggregation launch failed: ") + cudaGetErrorString(e));
    count_launch(2);
}

__global__ void k_agg_check(int rows, const int* choice, int* out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < rows && choice[r] == kUndecided) atomicAdd(&out[1], 1);
}

void aggregate_kahn(int rows, const int* ro, const int* ci, const int* dg, const int* tpos, const double* str,
                    int* choice, KahnWork w, int* err, cudaStream_t s) {
    (void)err;
    if (rows <= 0) return;
    int* push = w.tail;  // push[3] + out[2]
    cudaMemsetAsync(push, 0, 5 * sizeof(int), s);
    int* actA = w.lvl;
    int* actB = w.lvl2;
    k_agg_init<<<(rows + 255) / 256, 256, 0, s>>>(rows, ro, dg, w.cnt, choice, actA, push);
    count_launch();
    int* out = push + 3;
    if (rows <= 8192) {
        k_agg_rounds<false><<<1, 256, 0, s>>>(rows, ro, ci, dg, tpos, str, choice, w.cnt, actA, actB, push, out);
    } else {
        static int bps = 0;
        {
            std::lock_guard<std::recursive_mutex> lazy_lk(lazy_init_mutex());
            if (!bps) {
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_agg_rounds<true>, 256, 0);
                if (bps < 1) bps = 1;
            }
        }
        int grid = num_sms() * bps;
        const int need = (rows + 7) / 8;
        if (grid > need) grid = need;
        void* args[] = {(void*)&rows, (void*)&ro,   (void*)&ci,   (void*)&dg,   (void*)&tpos, (void*)&str,
                        (void*)&choice, (void*)&w.cnt, (void*)&actA, (void*)&actB, (void*)&push, (void*)&out};
        cudaError_t e = cudaLaunchCooperativeKernel((void*)k_agg_rounds<true>, dim3(grid), dim3(256), args, 0, s);
        if (e != cudaSuccess)
            throw std::runtime_error(std::string("cooperative launch failed: ") + cudaGetErrorString(e));
    }
    count_launch();
    k_agg_check<<<(rows + 255) / 256, 256, 0, s>>>(rows, choice, out);
    count_launch();
    int h[2] = {0, 0};
    cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (h[1] != 0) throw std::runtime_error("aggregation: rows left undecided (broken pattern)");
    last_agg_rounds = h[0];
}

__global__ void k_init_flag(int rows, const int* choice, int* flag) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < rows) flag[r] = choice[r] != kTaken ? 1 : 0;
}
__global__ void k_number(int rows, const int* choice, const int* cid, int* agg, int* members) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int ch = choice[r];
    if (ch == kTaken) return;
    const int c = cid[r];
    agg[r] = c;
    members[2 * c] = r;
    members[2 * c + 1] = ch >= 0 ? ch : -1;
    if (ch >= 0) agg[ch] = c;
}

int aggregate_number(int rows, const int* choice, int* flag_tmp, int* agg, int* members, int* d_total,
                     int* scan_tmp, cudaStream_t s) {
    const unsigned g = (rows + 255) / 256;
    k_init_flag<<<g, 256, 0, s>>>(rows, choice, flag_tmp);
    count_launch();
    exclusive_scan(flag_tmp, rows, d_total, scan_tmp, s);
    k_number<<<g, 256, 0, s>>>(rows, choice, flag_tmp, agg, members);
    count_launch();
    int nc = 0;
    cudaMemcpyAsync(&nc, d_total, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return nc;
}

// -------------------------------------------------------------- Galerkin
__global__ void k_seg_len(int nC, const int* ro, const int* members, int* seg) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nC) return;
    const int r1 = members[2 * c], r2 = members[2 * c + 1];
    seg[c] = (ro[r1 + 1] - ro[r1]) + (r2 >= 0 ? ro[r2 + 1] - ro[r2] : 0) + 1;
}
void galerkin_seg_len(int nCoarse, const int* ro, const int* members, int* seg_off, cudaStream_t s) {
    k_seg_len<<<(nCoarse + 255) / 256, 256, 0, s>>>(nCoarse, ro, members, seg_off);
    count_launch();
}

// key = (coarse column << 32) | position in the (r1 entries, r2 entries) list;
// the forced diagonal is (c << 32) | 0xFFFFFFFF (sorts after real entries).
__global__ void k_keys(int nC, const int* ro, const int* ci, const int* agg, const int* members, const int* seg,
                       unsigned long long* keys) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nC) return;
    const int r1 = members[2 * c], r2 = members[2 * c + 1];
    unsigned long long* out = keys + seg[c];
    unsigned p = 0;
    for (int k = ro[r1]; k < ro[r1 + 1]; ++k, ++p)
        out[p] = (static_cast<unsigned long long>(agg[ci[k]]) << 32) | p;
    if (r2 >= 0)
        for (int k = ro[r2]; k < ro[r2 + 1]; ++k, ++p)
            out[p] = (static_cast<unsigned long long>(agg[ci[k]]) << 32) | p;
    out[p] = (static_cast<unsigned long long>(c) << 32) | 0xFFFFFFFFull;
}
void galerkin_keys(int nCoarse, const int* ro, const int* ci, const int* agg, const int* members,
                   const int* seg_off, unsigned long long* keys, cudaStream_t s) {
    k_keys<<<(nCoarse + 127) / 128, 128, 0, s>>>(nCoarse, ro, ci, agg, members, seg_off, keys);
    count_launch();
}

constexpr int kWarpSeg = 256;    // segments up to this size: one warp, rank sort in smem
constexpr int kBlockSeg = 12288; // larger: one CTA, rank sort in 96 KB smem

__global__ void __launch_bounds__(256) k_sort_small(int nC, const int* seg, const unsigned long long* keys,
                                                    unsigned long long* sorted, int* big, int* nbig) {
    __shared__ unsigned long long sh[8][kWarpSeg];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = blockIdx.x * 8 + w;
    if (c >= nC) return;
    const int b = seg[c], len = seg[c + 1] - b;
    if (len > kWarpSeg) {
        if (lane == 0) big[atomicAdd(nbig, 1)] = c;
        return;
    }
    for (int i = lane; i < len; i += 32) sh[w][i] = keys[b + i];
    __syncwarp();
    for (int i = lane; i < len; i += 32) {
        const unsigned long long k = sh[w][i];
        int rank = 0;
        for (int q = 0; q < len; ++q) rank += sh[w][q] < k ? 1 : 0;
        sorted[b + rank] = k;
    }
}

__global__ void __launch_bounds__(1024) k_sort_big(const int* seg, const unsigned long long* keys,
                                                   unsigned long long* sorted, const int* big, int* err) {
    extern __shared__ unsigned long long shb[];
    const int c = big[blockIdx.x];
    const int b = seg[c], len = seg[c + 1] - b;
    if (len > kBlockSeg) {
        if (threadIdx.x == 0) atomicExch(err, 1);
        return;
    }
    for (int i = threadIdx.x; i < len; i += blockDim.x) shb[i] = keys[b + i];
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        const unsigned long long k = shb[i];
        int rank = 0;
        for (int q = 0; q < len; ++q) rank += shb[q] < k ? 1 : 0;
        sorted[b + rank] = k;
    }
}

void galerkin_sort(int nCoarse, const int* seg_off, const unsigned long long* keys, unsigned long long* sorted,
                   int* big, int* nbig, int* err, cudaStream_t s) {
    cudaMemsetAsync(nbig, 0, sizeof(int), s);
    k_sort_small<<<(nCoarse + 7) / 8, 256, 0, s>>>(nCoarse, seg_off, keys, sorted, big, nbig);
    count_launch();
    int nb = 0;
    cudaMemcpyAsync(&nb, nbig, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (nb > 0) {
        static bool attr = false;
        {
            std::lock_guard<std::recursive_mutex> lazy_lk(lazy_init_mutex());
            if (!attr) {
                cudaFuncSetAttribute(k_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kBlockSeg * static_cast<int>(sizeof(unsigned long long)));
                attr = true;
            }
        }
        k_sort_big<<<nb, 1024, kBlockSeg * sizeof(unsigned long long), s>>>(seg_off, keys, sorted, big, err);
        count_launch();
    }
}

__global__ void k_count(int nC, const int* seg, const unsigned long long* sorted, int* cro) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nC) return;
    const int b = seg[c], e = seg[c + 1];
    int u = 0;
    unsigned prev = 0xFFFFFFFFu;
    for (int i = b; i < e; ++i) {
        const unsigned J = static_cast<unsigned>(sorted[i] >> 32);
        if (i == b || J != prev) ++u;
        prev = J;
    }
    cro[c] = u;
}
void galerkin_count(int nCoarse, const int* seg_off, const unsigned long long* sorted, int* cro, cudaStream_t s) {
    k_count<<<(nCoarse + 255) / 256, 256, 0, s>>>(nCoarse, seg_off, sorted, cro);
    count_launch();
}

// one warp per coarse row; lane e accumulates block element e of each slot.
// Keys are read 8 at a time and their fine blocks loaded before the
// (sequential, reference-order) accumulation, so a warp keeps 8 block loads
// in flight instead of one dependent key -> block round trip per term.
template <int N>
__global__ void __launch_bounds__(256) k_fill(int nC, const int* __restrict__ ro, const int* __restrict__ members,
                                              const int* __restrict__ seg, const unsigned long long* __restrict__ sorted,
                                              const double* __restrict__ v, const int* __restrict__ cro, int* cci,
                                              double* cv) {
    constexpr int NN = N * N;
    constexpr int KB = 8;
    const int lane = threadIdx.x & 31;
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= nC) return;
    const int r1 = members[2 * c], r2 = members[2 * c + 1];
    const int b1 = ro[r1], len1 = ro[r1 + 1] - b1;
    const int b2 = r2 >= 0 ? ro[r2] : 0;
    const int sb = seg[c], se = seg[c + 1];
    int slot = cro[c] - 1;
    unsigned prev = 0;
    double acc = 0.0;
    for (int i0 = sb; i0 < se; i0 += KB) {
        const int nk = se - i0 < KB ? se - i0 : KB;  // warp-uniform
        const unsigned long long mine = lane < nk ? __ldg(&sorted[i0 + lane]) : 0ull;
        unsigned Js[KB], ps[KB];
        double vals[KB];
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const unsigned long long key = __shfl_sync(0xffffffffu, mine, e);
            Js[e] = static_cast<unsigned>(key >> 32);
            ps[e] = static_cast<unsigned>(key & 0xFFFFFFFFull);
            vals[e] = 0.0;
            if (e < nk && ps[e] != 0xFFFFFFFFu && lane < NN) {
                const int k = ps[e] < static_cast<unsigned>(len1) ? b1 + static_cast<int>(ps[e])
                                                                  : b2 + static_cast<int>(ps[e]) - len1;
                vals[e] = __ldg(&v[static_cast<size_t>(k) * NN + lane]);
            }
        }
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            if (e >= nk) break;
            const int i = i0 + e;
            if (i == sb || Js[e] != prev) {
                if (i != sb && lane < NN) cv[static_cast<size_t>(slot) * NN + lane] = acc;
                ++slot;
                if (lane == 0) cci[slot] = static_cast<int>(Js[e]);
                acc = 0.0;
                prev = Js[e];
            }
            if (ps[e] != 0xFFFFFFFFu && lane < NN) acc = __dadd_rn(acc, vals[e]);
        }
    }
    if (lane < NN) cv[static_cast<size_t>(slot) * NN + lane] = acc;
}
void galerkin_fill(int n, int nCoarse, const int* ro, const int* members, const int* seg_off,
                   const unsigned long long* sorted, const double* v, const int* cro, int* cci, double* cv,
                   cudaStream_t s) {
    const unsigned g = (nCoarse + 7) / 8;
    BCS_DISPATCH_N(n, k_fill<N><<<g, 256, 0, s>>>(nCoarse, ro, members, seg_off, sorted, v, cro, cci, cv));
    count_launch();
}

// ------------------------------------------------------------- transfers
__global__ void k_restrict(int n, int nC, const int* members, const double* res, double* rc) {
    const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<size_t>(nC) * n) return;
    const int c = static_cast<int>(t / n), q = static_cast<int>(t - static_cast<size_t>(c) * n);
    const int r1 = members[2 * c], r2 = members[2 * c + 1];
    double v = __dadd_rn(0.0, res[static_cast<size_t>(r1) * n + q]);
    if (r2 >= 0) v = __dadd_rn(v, res[static_cast<size_t>(r2) * n + q]);
    rc[t] = v;
}
void restrict_vec(int n, int nCoarse, const int* members, const double* res, double* rc, cudaStream_t s) {
    const size_t w = static_cast<size_t>(nCoarse) * n;
    k_restrict<<<static_cast<unsigned>((w + 255) / 256), 256, 0, s>>>(n, nCoarse, members, res, rc);
    count_launch();
}
__global__ void k_prolong(int n, int rows, const int* agg, const double* zc, double* z) {
    const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<size_t>(rows) * n) return;
    const int r = static_cast<int>(t / n), q = static_cast<int>(t - static_cast<size_t>(r) * n);
    z[t] = __dadd_rn(z[t], zc[static_cast<size_t>(agg[r]) * n + q]);
}
void prolong_vec(int n, int rows, const int* agg, const double* zc, double* z, cudaStream_t s) {
    const size_t w = static_cast<size_t>(rows) * n;
    k_prolong<<<static_cast<unsigned>((w + 255) / 256), 256, 0, s>>>(n, rows, agg, zc, z);
    count_launch();
}

// ------------------------------------------------------- dense coarsest
__global__ void k_dense_build(int n, int rows, const int* ro, const int* ci, const double* v, double* dense) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const size_t m = static_cast<size_t>(rows) * n;
    for (int k = ro[r]; k < ro[r + 1]; ++k) {
        const int c = ci[k];
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                dense[(static_cast<size_t>(r) * n + i) * m + (static_cast<size_t>(c) * n + j)] =
                    v[static_cast<size_t>(k) * n * n + i * n + j];
    }
}
void dense_build(int n, int rows, const int* ro, const int* ci, const double* v, double* dense, cudaStream_t s) {
    const size_t m = static_cast<size_t>(rows) * n;
    cudaMemsetAsync(dense, 0, m * m * sizeof(double), s);
    k_dense_build<<<(rows + 127) / 128, 128, 0, s>>>(n, rows, ro, ci, v, dense);
    count_launch();
}

// denseFactor (smallmat.hpp:134-161): one CTA, right-looking, reference order
__global__ void __launch_bounds__(1024) k_dense_factor(int m, double* a, int* piv, int* err) {
    __shared__ double sv[32];
    __shared__ int si[32];
    __shared__ int sp;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    for (int k = 0; k < m; ++k) {
        // first max of |a_ik|, i >= k (strict >: smallest index among maxima)
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
            // the reference starts from |a_kk| with p = k; ties keep k
            const double akk = fabs(a[static_cast<size_t>(k) * m + k]);
            if (!(bb > akk)) ii = k, bb = akk;
            if (bb < 1e-300) atomicExch(err, 1);
            piv[k] = ii;
            sp = ii;
        }
        __syncthreads();
        const int p = sp;
        if (p != k)
            for (int j = tid; j < m; j += nt) {
                const double t = a[static_cast<size_t>(k) * m + j];
                a[static_cast<size_t>(k) * m + j] = a[static_cast<size_t>(p) * m + j];
                a[static_cast<size_t>(p) * m + j] = t;
            }
        __syncthreads();
        const double d = a[static_cast<size_t>(k) * m + k];
        for (int i = k + 1 + tid; i < m; i += nt) a[static_cast<size_t>(i) * m + k] = __ddiv_rn(a[static_cast<size_t>(i) * m + k], d);
        __syncthreads();
        const int w = m - k - 1;
        for (long long t = tid; t < static_cast<long long>(w) * w; t += nt) {
            const int i = k + 1 + static_cast<int>(t / w), j = k + 1 + static_cast<int>(t % w);
            a[static_cast<size_t>(i) * m + j] =
                __dsub_rn(a[static_cast<size_t>(i) * m + j], __dmul_rn(a[static_cast<size_t>(i) * m + k], a[static_cast<size_t>(k) * m + j]));
        }
        __syncthreads();
    }
}
void dense_factor(int m, double* a, int* piv, int* err, cudaStream_t s) {
    k_dense_factor<<<1, 1024, 0, s>>>(m, a, piv, err);
    count_launch();
}

// denseSolve (smallmat.hpp:163-174), sequential reference order
// denseSolve (smallmat.hpp:163-174) for small m: the factor and the vector
// are staged in shared memory by the whole warp, then lane 0 runs the
// reference's chains (swaps, forward, backward) on shared-memory operands
// (a chain of global loads cost ~90 us at m = 35)
constexpr int kDenseSmallMax = 72;  // m <= kDenseSmallMax: staged (m^2 doubles, <= 41 KB of shared memory)
__global__ void k_dense_solve(int m, const double* lu, const int* piv, const double* r, double* z) {
    __shared__ double sl[kDenseSmallMax * kDenseSmallMax];
    __shared__ double sz[kDenseSmallMax];
    const bool staged = m <= kDenseSmallMax;
    if (staged) {
        for (int e = threadIdx.x; e < m * m; e += blockDim.x) sl[e] = lu[e];
        for (int e = threadIdx.x; e < m; e += blockDim.x) sz[e] = r[e];
        __syncwarp();
    }
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double* L = staged ? sl : lu;
    double* x = staged ? sz : z;
    if (!staged)
        for (int i = 0; i < m; ++i) x[i] = r[i];
    for (int k = 0; k < m; ++k) {
        const int p = piv[k];
        if (p != k) {
            const double t = x[k];
            x[k] = x[p];
            x[p] = t;
        }
    }
    for (int i = 1; i < m; ++i) {
        double v = x[i];
        for (int j = 0; j < i; ++j) v = __dsub_rn(v, __dmul_rn(L[static_cast<size_t>(i) * m + j], x[j]));
        x[i] = v;
    }
    for (int i = m - 1; i >= 0; --i) {
        double v = x[i];
        for (int j = i + 1; j < m; ++j) v = __dsub_rn(v, __dmul_rn(L[static_cast<size_t>(i) * m + j], x[j]));
        x[i] = __ddiv_rn(v, L[static_cast<size_t>(i) * m + i]);
    }
    if (staged)
        for (int i = 0; i < m; ++i) z[i] = x[i];
}

void dense_solve(int m, const double* lu, const int* piv, const double* r, double* z, cudaStream_t s) {
    k_dense_solve<<<1, 32, 0, s>>>(m, lu, piv, r, z);
    count_launch();
}

}  // namespace bcs
