// C ABI (include/bcs.h) over bcs::Engine.  Exceptions never cross the ABI:
// std::invalid_argument -> BCS_INVALID_ARGUMENT, std::bad_alloc ->
// BCS_OUT_OF_MEMORY, CudaError -> BCS_CUDA_ERROR, any other std::exception
// (the reference's std::runtime_error cases) -> BCS_RUNTIME_ERROR; the message
// is kept per context (or thread-locally for context-free calls).
#include "../../include/bcs.h"
#include "engine.hpp"

#include <algorithm>
#include <map>
#include <mutex>
#include <cstring>
#include <new>
#include <string>

struct bcs_partition {
    bcs::Decomposition dec;
    std::vector<bcs::Partition> parts;
};

struct bcs_ctx {
    bcs::Engine* eng = nullptr;
    std::string err;
};

namespace {
thread_local std::string g_err;

template <class F>
bcs_status guarded(bcs_ctx* ctx, F&& f) {
    std::string& msg = ctx ? ctx->err : g_err;
    try {
        f();
        msg.clear();
        return BCS_OK;
    } catch (const std::invalid_argument& e) {
        msg = e.what();
        return BCS_INVALID_ARGUMENT;
    } catch (const std::bad_alloc&) {
        msg = "out of device or host memory";
        return BCS_OUT_OF_MEMORY;
    } catch (const bcs::CudaError& e) {
        msg = e.what();
        return BCS_CUDA_ERROR;
    } catch (const std::exception& e) {
        msg = e.what();
        return BCS_RUNTIME_ERROR;
    } catch (...) {
        msg = "unknown error";
        return BCS_RUNTIME_ERROR;
    }
}

bcs::Engine& eng(bcs_ctx* ctx) {
    if (!ctx || !ctx->eng) throw std::invalid_argument("bcs: null context");
    return *ctx->eng;
}
const bcs_solver_config& cfgOf(const bcs_solver_config* c) {
    if (!c) throw std::invalid_argument("bcs: null solver config");
    return *c;
}
}  // namespace

namespace bcs {
uint64_t topologySignatureHost(int nc, int nf, const int32_t* owner, const int32_t* neigh);
}

extern "C" {

void bcs_default_config(bcs_solver_config* c) {
    if (!c) return;
    c->method = BCS_GMRES;
    c->precond = BCS_PRECOND_LUSGS;
    c->rel_tol = 1e-6;
    c->abs_tol = 1e-300;
    c->max_iters = 500;
    c->gmres_restart = 30;
    c->amg_max_levels = 10;
    c->amg_min_coarse_rows = 8;
    c->amg_pre_sweeps = 1;
    c->amg_post_sweeps = 1;
    c->mode = 0;
}

const char* bcs_version(void) { return "bcs 0.1 (sm_100a)"; }

// pinned host-buffer cache: size class -> free blocks; live block -> class
namespace {
std::mutex g_host_mu;
std::multimap<size_t, void*> g_host_free;
std::map<void*, size_t> g_host_live;
size_t host_class(size_t bytes) {
    size_t c = 4096;
    while (c < bytes) c <<= 1;
    return c;
}
}  // namespace

bcs_status bcs_host_alloc(size_t bytes, void** out) {
    if (!out) return BCS_INVALID_ARGUMENT;
    *out = nullptr;
    const size_t cls = host_class(bytes ? bytes : 1);
    {
        std::lock_guard<std::mutex> g(g_host_mu);
        auto it = g_host_free.find(cls);
        if (it != g_host_free.end()) {
            *out = it->second;
            g_host_free.erase(it);
            g_host_live[*out] = cls;
            return BCS_OK;
        }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, cls, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return BCS_OUT_OF_MEMORY;
    }
    std::lock_guard<std::mutex> g(g_host_mu);
    g_host_live[p] = cls;
    *out = p;
    return BCS_OK;
}

void bcs_host_free(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> g(g_host_mu);
    auto it = g_host_live.find(p);
    if (it == g_host_live.end()) return;
    g_host_free.emplace(it->second, p);
    g_host_live.erase(it);
}

bcs_status bcs_create(bcs_ctx** out, int device) {
    if (!out) return BCS_INVALID_ARGUMENT;
    *out = nullptr;
    auto* c = new (std::nothrow) bcs_ctx;
    if (!c) return BCS_OUT_OF_MEMORY;
    const bcs_status st = guarded(nullptr, [&] { c->eng = new bcs::Engine(device); });
    if (st != BCS_OK) {
        delete c;
        return st;
    }
    *out = c;
    return BCS_OK;
}

bcs_status bcs_destroy(bcs_ctx* ctx) {
    if (!ctx) return BCS_OK;
    delete ctx->eng;
    delete ctx;
    return BCS_OK;
}

const char* bcs_last_error(const bcs_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

bcs_status bcs_set_stream(bcs_ctx* ctx, void* stream) {
    return guarded(ctx, [&] { eng(ctx).setStream(static_cast<cudaStream_t>(stream)); });
}

bcs_status bcs_set_kernel_timing(bcs_ctx* ctx, int enable) {
    return guarded(ctx, [&] { eng(ctx).setKernelTiming(enable != 0); });
}

uint64_t bcs_topology_signature(int n_cells, int n_faces, const int32_t* owner, const int32_t* neighbour) {
    return bcs::topologySignatureHost(n_cells, n_faces, owner, neighbour);
}

bcs_status bcs_pipeline_solve(bcs_ctx* ctx, int n_cells, int n_faces, int block_size, const int32_t* owner,
                              const int32_t* neighbour, const double* diag, const double* upper,
                              const double* lower, const double* b, size_t b_len, const double* x0,
                              size_t x0_len, double* x, int backend, const bcs_solver_config* cfg,
                              bcs_report* report) {
    return guarded(ctx, [&] {
        bcs_report rep{};
        eng(ctx).pipelineSolve(n_cells, n_faces, block_size, owner, neighbour, diag, upper, lower, b, b_len, x0,
                               x0_len, x, backend, cfgOf(cfg), rep);
        if (report) *report = rep;
    });
}

bcs_status bcs_dist_solve(bcs_ctx* ctx, int n_cells, int n_faces, int block_size, const int32_t* owner,
                          const int32_t* neighbour, const double* centroids, const double* diag, const double* upper,
                          const double* lower, const double* b, const double* x0, double* x, int n_ranks,
                          int n_engines, const bcs_solver_config* cfg, bcs_report* report) {
    return guarded(ctx, [&] {
        bcs_report rep{};
        eng(ctx).distSolve(n_cells, n_faces, block_size, owner, neighbour, centroids, diag, upper, lower, b, x0, x,
                           n_ranks, n_engines, cfgOf(cfg), rep);
        if (report) *report = rep;
    });
}

bcs_status bcs_partition_create(bcs_partition** out, int n_cells, int n_faces, const int32_t* owner,
                                const int32_t* neighbour, const double* centroids, int n_ranks, int n_engines) {
    return guarded(nullptr, [&] {
        if (!out) throw std::invalid_argument("bcs_partition_create: null output");
        auto* p = new bcs_partition;
        try {
            p->dec = bcs::decompose(n_cells, centroids, n_ranks);
            p->parts = bcs::buildPartitioned(n_cells, n_faces, owner, neighbour, p->dec);
            if (n_engines > 0)
                p->parts = bcs::consolidate(p->parts, bcs::makeConsolidationPlan(p->dec, n_engines), p->dec);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}
void bcs_partition_destroy(bcs_partition* p) { delete p; }
int bcs_partition_count(const bcs_partition* p) { return p ? static_cast<int>(p->parts.size()) : 0; }
bcs_status bcs_partition_decomposition(const bcs_partition* p, int32_t* c2r, int32_t* rro, int32_t* o2n) {
    return guarded(nullptr, [&] {
        if (!p) throw std::invalid_argument("null partition");
        if (c2r) std::copy(p->dec.cellToRank.begin(), p->dec.cellToRank.end(), c2r);
        if (rro) std::copy(p->dec.rankRowOffset.begin(), p->dec.rankRowOffset.end(), rro);
        if (o2n) std::copy(p->dec.oldToNew.begin(), p->dec.oldToNew.end(), o2n);
    });
}
bcs_status bcs_partition_sizes(const bcs_partition* p, int part, int* rs, int* re, int* nnz, int* nh, int* ns) {
    return guarded(nullptr, [&] {
        if (!p || part < 0 || part >= static_cast<int>(p->parts.size())) throw std::invalid_argument("bad partition index");
        const auto& q = p->parts[part];
        if (rs) *rs = q.rowStart;
        if (re) *re = q.rowEnd;
        if (nnz) *nnz = static_cast<int>(q.ci.size());
        if (nh) *nh = static_cast<int>(q.haloRow.size());
        if (ns) *ns = static_cast<int>(q.sendPlan.size());
    });
}
bcs_status bcs_partition_get(const bcs_partition* p, int part, int32_t* ro, int32_t* ci, int32_t* src, int32_t* hr,
                             int32_t* hc, int32_t* hp, int32_t* hs, int32_t* sp, int32_t* sr) {
    return guarded(nullptr, [&] {
        if (!p || part < 0 || part >= static_cast<int>(p->parts.size())) throw std::invalid_argument("bad partition index");
        const auto& q = p->parts[part];
        if (ro) std::copy(q.ro.begin(), q.ro.end(), ro);
        if (ci) std::copy(q.ci.begin(), q.ci.end(), ci);
        if (src) std::copy(q.src.begin(), q.src.end(), src);
        if (hr) std::copy(q.haloRow.begin(), q.haloRow.end(), hr);
        if (hc) std::copy(q.haloCol.begin(), q.haloCol.end(), hc);
        if (hp) std::copy(q.haloPeer.begin(), q.haloPeer.end(), hp);
        if (hs) std::copy(q.haloSrc.begin(), q.haloSrc.end(), hs);
        for (size_t i = 0; i < q.sendPlan.size(); ++i) {
            if (sp) sp[i] = q.sendPlan[i].first;
            if (sr) sr[i] = q.sendPlan[i].second;
        }
    });
}

bcs_status bcs_partition_exchange_sizes(const bcs_partition* p, int part, int* n_send, int* n_recv) {
    return guarded(nullptr, [&] {
        if (!p || part < 0 || part >= static_cast<int>(p->parts.size())) throw std::invalid_argument("bad partition index");
        const bcs::ExchangePlan x = bcs::makeExchangePlan(p->parts, part);
        if (n_send) *n_send = static_cast<int>(x.sendRows.size());
        if (n_recv) *n_recv = static_cast<int>(x.recvGlobalRow.size());
    });
}
bcs_status bcs_partition_exchange_get(const bcs_partition* p, int part, int32_t* send_row, int32_t* send_count,
                                      int32_t* recv_global_row, int32_t* recv_count, int32_t* halo_recv_idx) {
    return guarded(nullptr, [&] {
        if (!p || part < 0 || part >= static_cast<int>(p->parts.size())) throw std::invalid_argument("bad partition index");
        const bcs::ExchangePlan x = bcs::makeExchangePlan(p->parts, part);
        if (send_row) std::copy(x.sendRows.begin(), x.sendRows.end(), send_row);
        if (send_count) std::copy(x.sendCount.begin(), x.sendCount.end(), send_count);
        if (recv_global_row) std::copy(x.recvGlobalRow.begin(), x.recvGlobalRow.end(), recv_global_row);
        if (recv_count) std::copy(x.recvCount.begin(), x.recvCount.end(), recv_count);
        if (halo_recv_idx) std::copy(x.haloRecvIdx.begin(), x.haloRecvIdx.end(), halo_recv_idx);
    });
}

bcs_status bcs_comm_unique_id(unsigned char id[128]) {
    return guarded(nullptr, [&] { bcs::Engine::commUniqueId(id); });
}
bcs_status bcs_comm_init(bcs_ctx* ctx, int rank, int n_ranks_total, const unsigned char id[128]) {
    return guarded(ctx, [&] { eng(ctx).commInit(rank, n_ranks_total, id); });
}
bcs_status bcs_dist_solve_mp(bcs_ctx* ctx, int n_cells, int n_faces, int block_size, const int32_t* owner,
                             const int32_t* neighbour, const double* centroids, const double* diag,
                             const double* upper, const double* lower, const double* b, const double* x0, double* x,
                             int n_ranks, const bcs_solver_config* cfg, bcs_report* report) {
    return guarded(ctx, [&] {
        bcs_report rep{};
        eng(ctx).distSolveMP(n_cells, n_faces, block_size, owner, neighbour, centroids, diag, upper, lower, b, x0, x,
                             n_ranks, cfgOf(cfg), rep);
        if (report) *report = rep;
    });
}

bcs_status bcs_set_topology(bcs_ctx* ctx, int n_cells, int n_faces, int block_size, const int32_t* owner,
                            const int32_t* neighbour) {
    return guarded(ctx, [&] { eng(ctx).setTopology(n_cells, n_faces, block_size, owner, neighbour); });
}

bcs_status bcs_upload_ldu(bcs_ctx* ctx, const double* diag, const double* upper, const double* lower) {
    return guarded(ctx, [&] {
        eng(ctx).uploadLdu(diag, upper, lower, false);
        cudaStreamSynchronize(eng(ctx).stream());
    });
}

bcs_status bcs_upload_ldu_device(bcs_ctx* ctx, const double* d_diag, const double* d_upper, const double* d_lower) {
    return guarded(ctx, [&] { eng(ctx).uploadLdu(d_diag, d_upper, d_lower, true); });
}

bcs_status bcs_assemble_euler(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner, const int32_t* neighbour,
                              const double* face_area, int n_bfaces, const int32_t* bface_cell,
                              const double* bface_area, const double* q, const double* q_inf, double cfl,
                              double* rhs) {
    return guarded(ctx, [&] {
        if (n_cells < 1 || n_faces < 0 || !q || !q_inf || !rhs || (n_faces && (!owner || !neighbour || !face_area)) ||
            (n_bfaces && (!bface_cell || !bface_area)))
            throw std::invalid_argument("bcs_assemble_euler: bad arguments");
        eng(ctx).assembleEuler(n_cells, n_faces, owner, neighbour, face_area, n_bfaces, bface_cell, bface_area, q,
                               q_inf, cfl, rhs);
    });
}

bcs_status bcs_solve(bcs_ctx* ctx, const double* b, double* x, const bcs_solver_config* cfg, bcs_report* report) {
    return guarded(ctx, [&] {
        bcs_report rep{};
        eng(ctx).solveHost(b, x, cfgOf(cfg), rep);
        if (report) *report = rep;
    });
}

bcs_status bcs_solve_device(bcs_ctx* ctx, const double* d_b, double* d_x, const bcs_solver_config* cfg,
                            bcs_report* report) {
    return guarded(ctx, [&] {
        bcs_report rep{};
        eng(ctx).solveDevice(d_b, d_x, cfgOf(cfg), rep);
        if (report) *report = rep;
    });
}

bcs_status bcs_residual(bcs_ctx* ctx, const double* b, const double* x, double* norm) {
    return guarded(ctx, [&] {
        const double v = eng(ctx).residualNorm(b, x);
        if (norm) *norm = v;
    });
}

bcs_status bcs_residual_history(bcs_ctx* ctx, double* out, int cap, int* n) {
    return guarded(ctx, [&] {
        const auto& h = eng(ctx).history();
        const int cnt = static_cast<int>(h.size());
        if (n) *n = cnt;
        if (out)
            for (int i = 0; i < cnt && i < cap; ++i) out[i] = h[i];
    });
}

bcs_status bcs_spmv(bcs_ctx* ctx, const double* x, double* y) {
    return guarded(ctx, [&] { eng(ctx).spmvHost(x, y); });
}

bcs_status bcs_spmv_device(bcs_ctx* ctx, const double* d_x, double* d_y) {
    return guarded(ctx, [&] { eng(ctx).spmvDevice(d_x, d_y); });
}

bcs_status bcs_csr_get(bcs_ctx* ctx, int32_t* row_offsets, int32_t* cols, double* values) {
    return guarded(ctx, [&] { eng(ctx).csrGet(row_offsets, cols, values); });
}

bcs_status bcs_precond_setup(bcs_ctx* ctx, const bcs_solver_config* cfg) {
    return guarded(ctx, [&] { eng(ctx).precondSetup(cfgOf(cfg)); });
}

bcs_status bcs_precond_apply(bcs_ctx* ctx, const double* r, double* z) {
    return guarded(ctx, [&] { eng(ctx).precondApplyHost(r, z); });
}

bcs_status bcs_amg_depth(bcs_ctx* ctx, int* depth) {
    return guarded(ctx, [&] {
        if (depth) *depth = eng(ctx).amgDepth();
    });
}

bcs_status bcs_amg_level_sizes(bcs_ctx* ctx, int level, int* rows, int* nnz) {
    return guarded(ctx, [&] { eng(ctx).amgLevelSizes(level, rows, nnz); });
}

bcs_status bcs_amg_level_get(bcs_ctx* ctx, int level, int32_t* row_offsets, int32_t* cols, double* values,
                             int32_t* aggregate) {
    return guarded(ctx, [&] { eng(ctx).amgLevelGet(level, row_offsets, cols, values, aggregate); });
}

bcs_status bcs_level_schedule_depth(bcs_ctx* ctx, int level, int* depth) {
    return guarded(ctx, [&] {
        if (depth) *depth = eng(ctx).scheduleDepth(level);
    });
}

bcs_status bcs_selftest(int what, unsigned long long n, unsigned long long seed, unsigned long long* result) {
    return guarded(nullptr, [&] {
        if (what >= 10 && what <= 14) {  // ping-pong latency, flavour what-10
            const unsigned long long ns = bcs::selftest_pingpong(what - 10, static_cast<int>(n));
            bcs::check(cudaDeviceSynchronize(), "selftest");
            if (result) *result = ns;
            return;
        }
        if (what >= 40 && what <= 44) {  // dependent-op latency: cycles of n ops
            const unsigned long long c = bcs::selftest_latency(what - 40, static_cast<int>(n));
            if (result) *result = c;
            return;
        }
        if (what == 30 || what == 31) {  // minimal chain: n = steps, seed = warps
            const unsigned long long ns = bcs::selftest_chain(what - 30, static_cast<int>(n), static_cast<int>(seed));
            bcs::check(cudaDeviceSynchronize(), "selftest");
            if (result) *result = ns;
            return;
        }
        if (what == 20) {  // install (n != 0: device buffer address in seed; n > 1: only sweeps with rows*2+fwd == n) / remove
            bcs::set_sweep_trace(n ? reinterpret_cast<unsigned long long*>(seed) : nullptr, n > 1 ? static_cast<long long>(n) : 0);
            return;
        }
        if (what != 0) throw std::invalid_argument("bcs_selftest: unknown test");
        const unsigned long long bad = bcs::selftest_division(n, seed);
        bcs::check(cudaDeviceSynchronize(), "selftest");
        if (result) *result = bad;
    });
}

}  // extern "C"
