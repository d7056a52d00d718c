// K13-K15: Krylov vector kernels (gmresSolve / bicgstabSolve,
// proj/core/src/krylov.cpp:59-214).
//
// Element-wise updates use the reference expressions verbatim (bit-identical
// under -fmad=false).  Reductions are deterministic two-level trees (fixed
// grid, fixed per-block order, the last block to finish sums the partials in
// block order) — the only place where the association order differs from the
// reference's sequential sum.  MGS orthogonalisation fuses each axpy with the
// next dot product; the Hessenberg/Givens scalars never leave the device
// except the one |g_{j+1}| the host needs for the convergence test.
#include "device.cuh"
#include "kernels.hpp"

namespace bcs {

constexpr int kRedThreads = 256;

int reduce_blocks() { return 2 * num_sms(); }

// Segmented deterministic reduction.  The vector is split into nseg
// contiguous segments (Mode-R engines; 1 for a serial solve); B blocks reduce
// each segment (fixed per-block order), the last block to finish sums every
// segment's block partials in block order and folds the segment sums with
// the reference's pairwise tree in engine order (partition.cpp:433-450).
__device__ __forceinline__ void finish_reduction(double part, int nseg, double* partials, int* ticket, double* out,
                                                 bool sqrt_out) {
    __shared__ double sh[32];
    __shared__ bool last;
    __shared__ double segsum[64];
    const double s = block_sum<kRedThreads>(part, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = s;
        __threadfence();
        last = atomicAdd(ticket, 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int B = gridDim.x / nseg;
    for (int e = 0; e < nseg; ++e) {
        double t = 0.0;
        for (int i = threadIdx.x; i < B; i += blockDim.x) t += __ldcg(&partials[e * B + i]);
        t = block_sum<kRedThreads>(t, sh);
        if (threadIdx.x == 0) segsum[e] = t;
    }
    if (threadIdx.x == 0) {
        int m = nseg;
        while (m > 1) {  // pairwise tree, engine order
            int w = 0;
            for (int i = 0; i + 1 < m; i += 2) segsum[w++] = segsum[i] + segsum[i + 1];
            if (m % 2) segsum[w++] = segsum[m - 1];
            m = w;
        }
        const double t = segsum[0];
        out[0] = sqrt_out ? sqrt(t) : t;
        *ticket = 0;
    }
}

struct SegRange {
    size_t b, e, i0, stride;
};
__device__ __forceinline__ SegRange seg_range(const long long* seg, int nseg) {
    const int B = gridDim.x / nseg;
    const int e = blockIdx.x / B, bi = blockIdx.x - e * B;
    SegRange r;
    r.b = static_cast<size_t>(seg[e]);
    r.e = static_cast<size_t>(seg[e + 1]);
    r.i0 = r.b + static_cast<size_t>(bi) * blockDim.x + threadIdx.x;
    r.stride = static_cast<size_t>(B) * blockDim.x;
    return r;
}

__global__ void __launch_bounds__(kRedThreads) k_dot(const double* __restrict__ a, const double* __restrict__ b,
                                                     const long long* __restrict__ seg, int nseg, double* out,
                                                     int sqrt_out, double* partials, int* ticket) {
    const SegRange R = seg_range(seg, nseg);
    double s = 0.0;
#pragma unroll 4
    for (size_t i = R.i0; i < R.e; i += R.stride) s += a[i] * b[i];  // (unrolled: loads in flight, same order)
    finish_reduction(s, nseg, partials, ticket, out, sqrt_out != 0);
}

// Exact mode (BCS_MODE_EXACT): the reference's own association order.
// defaultDot (krylov.cpp:38-42) is `s += a[i] * b[i]` from s = 0 in index
// order, i.e. a serial chain of rounded additions; one CTA per segment
// (engine) runs it: threads 32.. stage the rounded products of the next chunk
// in shared memory while thread 0 adds the current chunk in order.  The
// engine partials are then folded with the pairwise tree (partition.cpp:433-450).
// Throughput is one dependent FP64 add per element (~4.3 ns): diagnostic /
// proof speed, not the default.
constexpr int kSeqChunk = 2048;
__global__ void __launch_bounds__(256) k_dot_seq(const double* __restrict__ a, const double* __restrict__ b,
                                                 const long long* __restrict__ seg, double* part) {
    __shared__ double buf[2][kSeqChunk];
    const size_t s0 = static_cast<size_t>(seg[blockIdx.x]);
    const size_t n = static_cast<size_t>(seg[blockIdx.x + 1]) - s0;
    const int nch = static_cast<int>((n + kSeqChunk - 1) / kSeqChunk);
    const double* pa = a + s0;
    const double* pb = b + s0;
    auto fill = [&](int c, int t0, int nt) {
        const size_t base = static_cast<size_t>(c) * kSeqChunk;
        const int len = static_cast<int>(n - base < static_cast<size_t>(kSeqChunk) ? n - base : kSeqChunk);
        for (int k = threadIdx.x - t0; k < len; k += nt) buf[c & 1][k] = __dmul_rn(pa[base + k], pb[base + k]);
    };
    if (nch > 0) fill(0, 0, blockDim.x);
    __syncthreads();
    double s = 0.0;
    for (int c = 0; c < nch; ++c) {
        if (threadIdx.x >= 32 && c + 1 < nch) fill(c + 1, 32, blockDim.x - 32);
        if (threadIdx.x == 0) {
            const size_t base = static_cast<size_t>(c) * kSeqChunk;
            const int len = static_cast<int>(n - base < static_cast<size_t>(kSeqChunk) ? n - base : kSeqChunk);
            const double* bc = buf[c & 1];
#pragma unroll 16
            for (int k = 0; k < len; ++k) s = __dadd_rn(s, bc[k]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_axpy(double* __restrict__ w, const double* __restrict__ h, const double* __restrict__ v, size_t N) {
    const double hv = *h;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < N; i += stride) w[i] = w[i] - hv * v[i];
}

void dot_seq(const double* a, const double* b, const long long* seg, int nseg, double* out, bool sqrt_out,
             double* partials, cudaStream_t s) {
    k_dot_seq<<<nseg, 256, 0, s>>>(a, b, seg, partials);
    count_launch();
    fold_engines(partials, nseg, out, sqrt_out, s);
}
void axpy_dot_seq(double* w, const double* h, const double* v, const double* nextv, size_t N, const long long* seg,
                  int nseg, double* out, double* partials, bool sqrt_out, cudaStream_t s) {
    k_axpy<<<4 * num_sms(), 256, 0, s>>>(w, h, v, N);
    count_launch();
    dot_seq(w, nextv ? nextv : w, seg, nseg, out, sqrt_out, partials, s);
}

static int seg_grid(int nseg) {
    int B = reduce_blocks() / nseg;
    if (B < 4) B = 4;
    return B * nseg;
}

int seg_blocks(int nseg) { return seg_grid(nseg) / nseg; }

void dot(const double* a, const double* b, const long long* seg, int nseg, double* out, bool sqrt_out,
         double* partials, int* ticket, cudaStream_t s, int bps) {
    const int g = bps > 0 ? bps * nseg : seg_grid(nseg);
    k_dot<<<g, kRedThreads, 0, s>>>(a, b, seg, nseg, out, sqrt_out ? 1 : 0, partials, ticket);
    count_launch();
}

// per-engine partials (one per process, all-gathered) folded with the
// reference's pairwise tree in engine order (partition.cpp:433-450)
__global__ void k_fold_engines(const double* __restrict__ parts, int G, double* out, int sqrt_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double t[64];
    for (int i = 0; i < G; ++i) t[i] = parts[i];
    int m = G;
    while (m > 1) {
        int w = 0;
        for (int i = 0; i + 1 < m; i += 2) t[w++] = t[i] + t[i + 1];
        if (m % 2) t[w++] = t[m - 1];
        m = w;
    }
    out[0] = sqrt_out ? sqrt(t[0]) : t[0];
}
void fold_engines(const double* parts, int G, double* out, bool sqrt_out, cudaStream_t s) {
    k_fold_engines<<<1, 32, 0, s>>>(parts, G, out, sqrt_out ? 1 : 0);
    count_launch();
}

__global__ void k_pack_rows(int n, int cnt, const int* __restrict__ idx, const double* __restrict__ x, double* out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt * n) return;
    const int r = t / n, q = t - r * n;
    out[t] = x[static_cast<size_t>(idx[r]) * n + q];
}
void pack_rows(int n, int cnt, const int* idx, const double* x, double* out, cudaStream_t s) {
    if (cnt <= 0) return;
    k_pack_rows<<<(cnt * n + 255) / 256, 256, 0, s>>>(n, cnt, idx, x, out);
    count_launch();
}

// w -= h v ; dot(w, nextv) or ||w||
__global__ void __launch_bounds__(kRedThreads) k_axpy_dot(double* __restrict__ w, const double* __restrict__ h,
                                                          const double* __restrict__ v,
                                                          const double* __restrict__ nextv,
                                                          const long long* __restrict__ seg, int nseg, double* out,
                                                          double* partials, int* ticket, int sq) {
    const double hv = *h;
    const SegRange R = seg_range(seg, nseg);
    double s = 0.0;
#pragma unroll 4
    for (size_t i = R.i0; i < R.e; i += R.stride) {
        const double wn = w[i] - hv * v[i];
        w[i] = wn;
        s += nextv ? wn * nextv[i] : wn * wn;
    }
    finish_reduction(s, nseg, partials, ticket, out, sq != 0);
}

void axpy_dot(double* w, const double* h, const double* v, const double* nextv, const long long* seg, int nseg,
              double* out, double* partials, int* ticket, cudaStream_t s, int bps, int sqrt_mode) {
    const int g = bps > 0 ? bps * nseg : seg_grid(nseg);
    const int sq = sqrt_mode < 0 ? (nextv == nullptr ? 1 : 0) : sqrt_mode;
    k_axpy_dot<<<g, kRedThreads, 0, s>>>(w, h, v, nextv, seg, nseg, out, partials, ticket, sq);
    count_launch();
}

// Mode-R halo couplings (partitionedMatvec, partition.cpp:335-350): after the
// local product, y[row] += sum over the row's halo entries in (localRow,
// globalCol) order of matvecAdd(block, x[globalCol]).
__global__ void k_halo(int n, int nhr, const int* __restrict__ hrow, const int* __restrict__ hoff,
                       const int* __restrict__ hcol, const double* __restrict__ hv, const double* __restrict__ x,
                       double* __restrict__ y, int rowStart) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nhr * n) return;
    const int hr = t / n, q = t - hr * n;
    const size_t o = static_cast<size_t>(rowStart + hrow[hr]) * n + q;
    double acc = y[o];
    for (int h = hoff[hr]; h < hoff[hr + 1]; ++h) {
        const double* blk = hv + static_cast<size_t>(h) * n * n + q * n;
        const double* xc = x + static_cast<size_t>(hcol[h]) * n;
        double sb = 0.0;
        for (int p = 0; p < n; ++p) sb = __dadd_rn(sb, __dmul_rn(blk[p], xc[p]));
        acc = __dadd_rn(acc, sb);
    }
    y[o] = acc;
}
void halo_spmv(int n, int nhr, const int* hrow, const int* hoff, const int* hcol, const double* hv, const double* x,
               double* y, int rowStart, cudaStream_t s) {
    if (nhr <= 0) return;
    k_halo<<<(nhr * n + 127) / 128, 128, 0, s>>>(n, nhr, hrow, hoff, hcol, hv, x, y, rowStart);
    count_launch();
}

__global__ void k_scale_by(const double* __restrict__ x, const double* __restrict__ den, double thr,
                           double* __restrict__ y, size_t N) {
    const double d = *den;
    if (!(d > thr)) return;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < N; i += stride) y[i] = x[i] / d;
}
void scale_by(const double* x, const double* den, double thr, double* y, size_t N, cudaStream_t s) {
    k_scale_by<<<4 * num_sms(), 256, 0, s>>>(x, den, thr, y, N);
    count_launch();
}

__global__ void k_sub(const double* __restrict__ b, const double* __restrict__ y, double* __restrict__ r, size_t N) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < N; i += stride) r[i] = b[i] - y[i];
}
void sub_vec(const double* b, const double* y, double* r, size_t N, cudaStream_t s) {
    k_sub<<<4 * num_sms(), 256, 0, s>>>(b, y, r, N);
    count_launch();
}
void copy_vec(const double* x, double* y, size_t N, cudaStream_t s) {
    cudaMemcpyAsync(y, x, N * sizeof(double), cudaMemcpyDeviceToDevice, s);
}
__global__ void k_add_to(double* __restrict__ x, const double* __restrict__ z, size_t N) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < N; i += stride) x[i] += z[i];
}
void add_to(double* x, const double* z, size_t N, cudaStream_t s) {
    k_add_to<<<4 * num_sms(), 256, 0, s>>>(x, z, N);
    count_launch();
}

// w = sum_{i<j} y_i V_i with the reference's accumulation order (krylov.cpp:127-129)
__global__ void k_lincomb(const double* __restrict__ V, size_t ld, const double* __restrict__ y, int j,
                          double* __restrict__ w, size_t N) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < N; q += stride) {
        double acc = 0.0;
        for (int i = 0; i < j; ++i) acc += y[i] * V[static_cast<size_t>(i) * ld + q];
        w[q] = acc;
    }
}
void lincomb(const double* V, size_t ld, const double* y, int j, double* w, size_t N, cudaStream_t s) {
    k_lincomb<<<4 * num_sms(), 256, 0, s>>>(V, ld, y, j, w, N);
    count_launch();
}

// std::hypot of the reference's libm (glibc 2.35+ e_hypot.c: Borges' "An
// Improved Algorithm for hypot(a,b)", the non-FMA kernel with its scaling
// thresholds 2^511 / 2^-459 / 2^-54 and scale 2^-600), restated operation by
// operation so the Givens rotation of krylov.cpp:106-117 rounds as the
// reference's does.  Pinned against the host libm bit for bit
// (tests/test_oracle.py::test_glibc_hypot_restatement, bcs_selftest_hypot).
__device__ __forceinline__ double glibc_hypot_kernel(double ax, double ay) {
    double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    double t1, t2;
    if (h <= __dmul_rn(2.0, ay)) {
        const double delta = __dsub_rn(h, ay);
        t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
        t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
    } else {
        const double delta = __dsub_rn(h, ax);
        t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
        t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
    }
    return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}
__device__ double glibc_hypot(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000ll);
        return __dadd_rn(x, y);
    }
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x, ay = x < y ? x : y;
    constexpr double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-459, kEps = 0x1p-54;
    if (ax > kLarge) {
        if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
        return __ddiv_rn(glibc_hypot_kernel(__dmul_rn(ax, kScale), __dmul_rn(ay, kScale)), kScale);
    }
    if (ay < kTiny) {
        if (ax >= __ddiv_rn(ay, kEps)) return __dadd_rn(ax, ay);
        return __dmul_rn(glibc_hypot_kernel(__ddiv_rn(ax, kScale), __ddiv_rn(ay, kScale)), kScale);
    }
    if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
    return glibc_hypot_kernel(ax, ay);
}
__global__ void k_hypot_eval(const double* x, const double* y, double* out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = glibc_hypot(x[i], y[i]);
}
void hypot_eval(const double* x, const double* y, double* out, int n, cudaStream_t s) {
    if (n <= 0) return;
    k_hypot_eval<<<(n + 255) / 256, 256, 0, s>>>(x, y, out, n);
    count_launch();
}

// Givens update of column j (krylov.cpp:104-117); H is (m+1) x m row-major
__global__ void k_givens(double* H, int m, int j, double* cs, double* sn, double* g, double* status) {
    if (threadIdx.x != 0) return;
    const double hh = H[(j + 1) * m + j];
    for (int i = 0; i < j; ++i) {
        const double t = cs[i] * H[i * m + j] + sn[i] * H[(i + 1) * m + j];
        H[(i + 1) * m + j] = -sn[i] * H[i * m + j] + cs[i] * H[(i + 1) * m + j];
        H[i * m + j] = t;
    }
    const double den = glibc_hypot(H[j * m + j], H[(j + 1) * m + j]);
    cs[j] = den > 0.0 ? H[j * m + j] / den : 1.0;
    sn[j] = den > 0.0 ? H[(j + 1) * m + j] / den : 0.0;
    H[j * m + j] = den;
    H[(j + 1) * m + j] = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    status[0] = fabs(g[j + 1]);
    status[1] = (hh > 1e-290) ? 0.0 : 1.0;
}
void givens_step(double* H, int m, int j, double* cs, double* sn, double* g, double* status, cudaStream_t s) {
    k_givens<<<1, 32, 0, s>>>(H, m, j, cs, sn, g, status);
    count_launch();
}

__global__ void k_back_subst(const double* H, int m, int j, const double* g, double* y) {
    if (threadIdx.x != 0) return;
    for (int i = j - 1; i >= 0; --i) {
        double sacc = g[i];
        for (int q = i + 1; q < j; ++q) sacc -= H[i * m + q] * y[q];
        y[i] = sacc / H[i * m + i];
    }
}
void back_subst(const double* H, int m, int j, const double* g, double* y, cudaStream_t s) {
    k_back_subst<<<1, 32, 0, s>>>(H, m, j, g, y);
    count_launch();
}

// ---- BiCGStab (krylov.cpp:174-200)
__global__ void k_bicg_p(double* p, const double* r, const double* v, double bf, double omega, size_t N) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < N; i += stride)
        p[i] = r[i] + bf * (p[i] - omega * v[i]);
}
void bicg_p(double* p, const double* r, const double* v, double bf, double omega, size_t N, cudaStream_t s) {
    k_bicg_p<<<4 * num_sms(), 256, 0, s>>>(p, r, v, bf, omega, N);
    count_launch();
}
__global__ void k_bicg_s(double* sv, const double* r, const double* v, double alpha, size_t N) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < N; i += stride)
        sv[i] = r[i] - alpha * v[i];
}
void bicg_s(double* sv, const double* r, const double* v, double alpha, size_t N, cudaStream_t s) {
    k_bicg_s<<<4 * num_sms(), 256, 0, s>>>(sv, r, v, alpha, N);
    count_launch();
}
__global__ void k_bicg_xh(double* x, const double* ph, double alpha, size_t N) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < N; i += stride)
        x[i] += alpha * ph[i];
}
void bicg_x_half(double* x, const double* ph, double alpha, size_t N, cudaStream_t s) {
    k_bicg_xh<<<4 * num_sms(), 256, 0, s>>>(x, ph, alpha, N);
    count_launch();
}
__global__ void k_bicg_xr(double* x, double* r, const double* ph, const double* sh, const double* sv,
                          const double* t, double alpha, double omega, size_t N) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < N; i += stride) {
        x[i] += alpha * ph[i] + omega * sh[i];
        r[i] = sv[i] - omega * t[i];
    }
}
void bicg_x_r(double* x, double* r, const double* ph, const double* sh, const double* sv, const double* t,
              double alpha, double omega, size_t N, cudaStream_t s) {
    k_bicg_xr<<<4 * num_sms(), 256, 0, s>>>(x, r, ph, sh, sv, t, alpha, omega, N);
    count_launch();
}

}  // namespace bcs
