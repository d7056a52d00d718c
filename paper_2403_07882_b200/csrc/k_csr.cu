// K1-K3: LDU -> block-CSR plan and value permutation, BSR SpMV, prefix scan.
//
// Reference: buildPlan / lduToBlockCsr / replaceValues / csrMatvec
// (proj/core/src/block_csr.cpp:56-80, 97-109, 120-137).  The plan is integer
// work and bit-exact: per row the diagonal, upper faces and lower faces,
// ordered by column (columns are distinct, so the order is unique).  The
// value copy is a pure permutation of 8 n^2-byte blocks.  SpMV computes each
// output scalar as the reference does: y_i = 0; per block s = sum_j a_ij x_j
// (j ascending), y_i += s  — bit-identical under -fmad=false.
#include "device.cuh"
#include "kernels.hpp"

#include <stdexcept>

namespace bcs {

std::recursive_mutex& lazy_init_mutex() {
    static std::recursive_mutex m;
    return m;
}


thread_local LaunchCounter* g_launches = nullptr;

int num_sms() {
    static int sms = 0;
    {
        std::lock_guard<std::recursive_mutex> lazy_lk(lazy_init_mutex());
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (sms <= 0) sms = 148;
        }
    }
    return sms;
}

static inline unsigned grid_for(size_t work, int threads, size_t cap = 1u << 20) {
    size_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

// ------------------------------------------------------------------ scan
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_exclusive_scan(int v, int* sh, int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int w = lane < (blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        sh[lane] = w;
    }
    __syncthreads();
    const int before = (wid > 0 ? sh[wid - 1] : 0) + x - v;
    if (total) *total = sh[(blockDim.x >> 5) - 1];
    __syncthreads();
    return before;
}

__global__ void scan_tiles(int* data, int n, int* tile_sums) {
    __shared__ int sh[32];
    const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    int v[kScanItems];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = (base + i < static_cast<size_t>(n)) ? data[base + i] : 0;
        sum += v[i];
    }
    int total;
    int run = block_exclusive_scan(sum, sh, &total);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < static_cast<size_t>(n)) data[base + i] = run;
        run += v[i];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void scan_single(int* data, int n, int* d_total) {
    __shared__ int sh[32];
    int carry = 0;
    for (int base = 0; base < n; base += kScanTile) {
        const int b = base + threadIdx.x * kScanItems;
        int v[kScanItems];
        int sum = 0;
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            v[i] = (b + i < n) ? data[b + i] : 0;
            sum += v[i];
        }
        int total;
        int run = block_exclusive_scan(sum, sh, &total) + carry;
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            if (b + i < n) data[b + i] = run;
            run += v[i];
        }
        carry += total;
    }
    if (threadIdx.x == 0 && d_total) *d_total = carry;
}

__global__ void scan_add(int* data, int n, const int* tile_offsets) {
    const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile;
    const int add = tile_offsets[blockIdx.x];
    for (int i = threadIdx.x; i < kScanTile; i += blockDim.x)
        if (base + i < static_cast<size_t>(n)) data[base + i] += add;
}

size_t scan_tmp_ints(size_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

void exclusive_scan(int* data, int n, int* d_total, int* tmp, cudaStream_t s) {
    if (n <= kScanTile * 8) {
        scan_single<<<1, kScanThreads, 0, s>>>(data, n, d_total);
        count_launch();
        return;
    }
    const int tiles = (n + kScanTile - 1) / kScanTile;
    scan_tiles<<<tiles, kScanThreads, 0, s>>>(data, n, tmp);
    scan_single<<<1, kScanThreads, 0, s>>>(tmp, tiles, d_total);
    scan_add<<<tiles, 256, 0, s>>>(data, n, tmp);
    count_launch(3);
}

// ------------------------------------------------------------------ plan
__global__ void k_plan_count(int nc, int nf, const int* owner, const int* neigh, int* cnt) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < static_cast<size_t>(nc) + nf;
         i += stride) {
        if (i < static_cast<size_t>(nc)) {
            atomicAdd(&cnt[i], 1);
        } else {
            const size_t f = i - nc;
            atomicAdd(&cnt[owner[f]], 1);
            atomicAdd(&cnt[neigh[f]], 1);
        }
    }
}
void plan_count(int nc, int nf, const int* owner, const int* neigh, int* rowcnt, cudaStream_t s) {
    k_plan_count<<<grid_for(static_cast<size_t>(nc) + nf, 256, 8 * 148 * 8), 256, 0, s>>>(nc, nf, owner, neigh,
                                                                                       rowcnt);
    count_launch();
}

// slot sources: c (diag), nc + f (upper of f), nc + nf + f (lower of f)
__global__ void k_plan_fill(int nc, int nf, const int* owner, const int* neigh, const int* ro, int* fillc, int* ci,
                            int* src) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < static_cast<size_t>(nc) + nf;
         i += stride) {
        if (i < static_cast<size_t>(nc)) {
            const int c = static_cast<int>(i);
            const int k = ro[c] + atomicAdd(&fillc[c], 1);
            ci[k] = c;
            src[k] = c;
        } else {
            const int f = static_cast<int>(i - nc);
            const int o = owner[f], nb = neigh[f];
            int k = ro[o] + atomicAdd(&fillc[o], 1);
            ci[k] = nb;
            src[k] = nc + f;
            k = ro[nb] + atomicAdd(&fillc[nb], 1);
            ci[k] = o;
            src[k] = nc + nf + f;
        }
    }
}
void plan_fill(int nc, int nf, const int* owner, const int* neigh, const int* ro, int* fillc, int* ci, int* src,
               cudaStream_t s) {
    k_plan_fill<<<grid_for(static_cast<size_t>(nc) + nf, 256, 8 * 148 * 8), 256, 0, s>>>(nc, nf, owner, neigh, ro,
                                                                                      fillc, ci, src);
    count_launch();
}

// per-row insertion sort by column (rows are short: <= a few dozen entries)
__global__ void k_plan_sort(int nc, const int* ro, int* ci, int* src) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nc) return;
    const int b = ro[r], e = ro[r + 1];
    for (int k = b + 1; k < e; ++k) {
        const int c = ci[k], sv = src[k];
        int q = k - 1;
        while (q >= b && ci[q] > c) {
            ci[q + 1] = ci[q];
            src[q + 1] = src[q];
            --q;
        }
        ci[q + 1] = c;
        src[q + 1] = sv;
    }
}
void plan_sort_rows(int nc, const int* ro, int* ci, int* src, cudaStream_t s) {
    k_plan_sort<<<grid_for(nc, 128), 128, 0, s>>>(nc, ro, ci, src);
    count_launch();
}

__device__ __forceinline__ int row_find(const int* ci, int b, int e, int col) {
    while (b < e) {
        const int mid = b + ((e - b) >> 1);
        if (ci[mid] < col) b = mid + 1;
        else e = mid;
    }
    return b;
}

__global__ void k_find_diag(int rows, const int* ro, const int* ci, int* dg) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int e = ro[r + 1];
    const int k = row_find(ci, ro[r], e, r);
    dg[r] = (k < e && ci[k] == r) ? k : -1;
}
void find_diag(int rows, const int* ro, const int* ci, int* dg, cudaStream_t s) {
    k_find_diag<<<grid_for(rows, 256), 256, 0, s>>>(rows, ro, ci, dg);
    count_launch();
}

// tpos[k] = slot of the transposed entry (c, r) of entry k = (r, c), or -1.
__global__ void k_tpos(int rows, const int* ro, const int* ci, int* tpos, int* asym) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    for (int k = ro[r]; k < ro[r + 1]; ++k) {
        const int c = ci[k];
        const int e = ro[c + 1];
        const int t = row_find(ci, ro[c], e, r);
        const bool ok = t < e && ci[t] == r;
        tpos[k] = ok ? t : -1;
        if (!ok) atomicExch(asym, 1);
    }
}
void transpose_pos(int rows, const int* ro, const int* ci, int* tpos, int* asym_flag, cudaStream_t s) {
    k_tpos<<<grid_for(rows, 256), 256, 0, s>>>(rows, ro, ci, tpos, asym_flag);
    count_launch();
}

// value permutation: one thread per double, coalesced writes
// 4 doubles per thread (a CTA covers 1024 consecutive ones, coalesced per
// instruction); NN compile-time so the slot index is a constant division;
// the grid covers the array once (no grid-stride loop)
template <int NN>
__global__ void __launch_bounds__(256) k_gather(size_t total, int nc, int nf, const int* __restrict__ src,
                                                const double* __restrict__ diag, const double* __restrict__ upper,
                                                const double* __restrict__ lower, double* __restrict__ vals) {
    const size_t i0 = 4 * blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const size_t i = i0 + static_cast<size_t>(u) * blockDim.x;  // coalesced per instruction
        if (i >= total) return;
        const size_t k = i / NN;
        const int e = static_cast<int>(i - k * NN);
        const int sidx = __ldg(&src[k]);
        const double* from = sidx < nc ? diag + static_cast<size_t>(sidx) * NN
                             : sidx < nc + nf ? upper + static_cast<size_t>(sidx - nc) * NN
                                              : lower + static_cast<size_t>(sidx - nc - nf) * NN;
        __stcs(&vals[i], __ldcs(&from[e]));
    }
}

void gather_values(int n, int nnz, int nc, int nf, const int* src, const double* diag, const double* upper,
                   const double* lower, double* vals, cudaStream_t s) {
    const size_t total = static_cast<size_t>(nnz) * n * n;
    if (!total) return;
    const unsigned g = static_cast<unsigned>((total + 1023) / 1024);
    switch (n) {
        case 1: k_gather<1><<<g, 256, 0, s>>>(total, nc, nf, src, diag, upper, lower, vals); break;
        case 2: k_gather<4><<<g, 256, 0, s>>>(total, nc, nf, src, diag, upper, lower, vals); break;
        case 3: k_gather<9><<<g, 256, 0, s>>>(total, nc, nf, src, diag, upper, lower, vals); break;
        case 4: k_gather<16><<<g, 256, 0, s>>>(total, nc, nf, src, diag, upper, lower, vals); break;
        default: k_gather<25><<<g, 256, 0, s>>>(total, nc, nf, src, diag, upper, lower, vals); break;
    }
    count_launch();
}

// ------------------------------------------------------------------ SpMV
// One thread per output scalar (row, q).  N threads of a row read the row's
// contiguous block segment (40-byte row slices); x gathers go through L1/L2.
template <int N>
__global__ void __launch_bounds__(256) k_spmv(int rows, const int* __restrict__ ro, const int* __restrict__ ci,
                                              const double* __restrict__ v, const double* __restrict__ x,
                                              const double* __restrict__ sub, double* __restrict__ y) {
    const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<size_t>(rows) * N) return;
    const int r = static_cast<int>(t / N);
    const int q = static_cast<int>(t - static_cast<size_t>(r) * N);
    const int b = __ldg(&ro[r]), e = __ldg(&ro[r + 1]);
    double acc = 0.0;
    for (int k = b; k < e; ++k) {
        const int c = __ldg(&ci[k]);
        const double* a = v + static_cast<size_t>(k) * (N * N) + q * N;
        const double* xc = x + static_cast<size_t>(c) * N;
        double sblk = 0.0;
#pragma unroll
        for (int p = 0; p < N; ++p) sblk = __dadd_rn(sblk, __dmul_rn(__ldg(&a[p]), __ldg(&xc[p])));
        acc = __dadd_rn(acc, sblk);
    }
    y[t] = sub ? __dsub_rn(sub[t], acc) : acc;
}

void spmv(int n, int rows, const int* ro, const int* ci, const double* v, const double* x, const double* sub,
          double* y, cudaStream_t s) {
    const size_t work = static_cast<size_t>(rows) * n;
    const unsigned g = static_cast<unsigned>((work + 255) / 256);
    if (!g) return;
    switch (n) {
        case 1: k_spmv<1><<<g, 256, 0, s>>>(rows, ro, ci, v, x, sub, y); break;
        case 2: k_spmv<2><<<g, 256, 0, s>>>(rows, ro, ci, v, x, sub, y); break;
        case 3: k_spmv<3><<<g, 256, 0, s>>>(rows, ro, ci, v, x, sub, y); break;
        case 4: k_spmv<4><<<g, 256, 0, s>>>(rows, ro, ci, v, x, sub, y); break;
        case 5: k_spmv<5><<<g, 256, 0, s>>>(rows, ro, ci, v, x, sub, y); break;
        default: throw std::invalid_argument("block size must be 1..5 on the device");
    }
    count_launch();
}

}  // namespace bcs
