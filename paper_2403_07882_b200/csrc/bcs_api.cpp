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
#include <cstdio>
#include <cstring>
#include <vector>
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

// ---- binary LDU dump (bcs.h) ----------------------------------------------
namespace {
constexpr char kLduMagic[8] = {'B', 'C', 'S', 'L', 'D', 'U', '0', '1'};
struct LduHeader {
    char magic[8];
    int32_t version, n_cells, n_faces, block_size, flags;
    uint64_t checksum;
    char pad[24];
};
static_assert(sizeof(LduHeader) == 64, "LDU header is 64 bytes");
uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
        h ^= c[i];
        h *= 1099511628211ull;
    }
    return h;
}
struct Section {
    void* p;
    size_t bytes;
};
std::vector<Section> lduSections(const LduHeader& h, const void* owner, const void* neigh, const void* diag,
                                 const void* upper, const void* lower, const void* b, const void* x0) {
    const size_t nn = static_cast<size_t>(h.block_size) * h.block_size, nf = h.n_faces, nc = h.n_cells;
    std::vector<Section> v = {{const_cast<void*>(owner), 4 * nf},          {const_cast<void*>(neigh), 4 * nf},
                              {const_cast<void*>(diag), 8 * nc * nn},     {const_cast<void*>(upper), 8 * nf * nn},
                              {const_cast<void*>(lower), 8 * nf * nn}};
    if (h.flags & 1) v.push_back({const_cast<void*>(b), 8 * nc * h.block_size});
    if (h.flags & 2) v.push_back({const_cast<void*>(x0), 8 * nc * h.block_size});
    return v;
}
LduHeader readHeader(std::FILE* f, const char* path) {
    LduHeader h{};
    if (std::fread(&h, sizeof h, 1, f) != 1 || std::memcmp(h.magic, kLduMagic, 8) != 0 || h.version != 1 ||
        h.n_cells < 1 || h.n_faces < 0 || h.block_size < 1 || h.block_size > 16)
        throw std::runtime_error(std::string("bcs_ldu_load: not a BCSLDU01 file: ") + path);
    return h;
}
}  // namespace

bcs_status bcs_ldu_save(const char* path, int n_cells, int n_faces, int block_size, const int32_t* owner,
                        const int32_t* neighbour, const double* diag, const double* upper, const double* lower,
                        const double* b, const double* x0) {
    return guarded(nullptr, [&] {
        if (!path || n_cells < 1 || n_faces < 0 || block_size < 1 || block_size > 16 || !diag ||
            (n_faces && (!owner || !neighbour || !upper || !lower)))
            throw std::invalid_argument("bcs_ldu_save: bad arguments");
        LduHeader h{};
        std::memcpy(h.magic, kLduMagic, 8);
        h.version = 1;
        h.n_cells = n_cells;
        h.n_faces = n_faces;
        h.block_size = block_size;
        h.flags = (b ? 1 : 0) | (x0 ? 2 : 0);
        const auto sec = lduSections(h, owner, neighbour, diag, upper, lower, b, x0);
        uint64_t sum = 1469598103934665603ull;
        for (const auto& x : sec) sum = fnv1a(sum, x.p, x.bytes);
        h.checksum = sum;
        std::FILE* f = std::fopen(path, "wb");
        if (!f) throw std::runtime_error(std::string("bcs_ldu_save: cannot open ") + path);
        bool ok = std::fwrite(&h, sizeof h, 1, f) == 1;
        for (const auto& x : sec) ok = ok && (x.bytes == 0 || std::fwrite(x.p, 1, x.bytes, f) == x.bytes);
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) throw std::runtime_error(std::string("bcs_ldu_save: write failed: ") + path);
    });
}

bcs_status bcs_ldu_load_sizes(const char* path, int* n_cells, int* n_faces, int* block_size, int* has_b,
                              int* has_x0) {
    return guarded(nullptr, [&] {
        std::FILE* f = path ? std::fopen(path, "rb") : nullptr;
        if (!f) throw std::runtime_error(std::string("bcs_ldu_load: cannot open ") + (path ? path : "(null)"));
        LduHeader h{};
        try {
            h = readHeader(f, path);
        } catch (...) {
            std::fclose(f);
            throw;
        }
        std::fclose(f);
        if (n_cells) *n_cells = h.n_cells;
        if (n_faces) *n_faces = h.n_faces;
        if (block_size) *block_size = h.block_size;
        if (has_b) *has_b = h.flags & 1;
        if (has_x0) *has_x0 = (h.flags >> 1) & 1;
    });
}

bcs_status bcs_ldu_load(const char* path, int32_t* owner, int32_t* neighbour, double* diag, double* upper,
                        double* lower, double* b, double* x0) {
    return guarded(nullptr, [&] {
        std::FILE* f = path ? std::fopen(path, "rb") : nullptr;
        if (!f) throw std::runtime_error(std::string("bcs_ldu_load: cannot open ") + (path ? path : "(null)"));
        std::vector<unsigned char> skip;
        try {
            const LduHeader h = readHeader(f, path);
            auto sec = lduSections(h, owner, neighbour, diag, upper, lower, b, x0);
            uint64_t sum = 1469598103934665603ull;
            for (auto& x : sec) {
                if (!x.p) {  // caller skips this section: read into scratch for the checksum
                    skip.resize(x.bytes);
                    x.p = skip.data();
                }
                if (x.bytes && std::fread(x.p, 1, x.bytes, f) != x.bytes)
                    throw std::runtime_error(std::string("bcs_ldu_load: truncated file: ") + path);
                sum = fnv1a(sum, x.p, x.bytes);
            }
            if (sum != h.checksum) throw std::runtime_error(std::string("bcs_ldu_load: checksum mismatch: ") + path);
        } catch (...) {
            std::fclose(f);
            throw;
        }
        std::fclose(f);
    });
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

bcs_status bcs_dist_solve_parts(bcs_ctx* ctx, int n_ranks, int block_size, const int32_t* rank_row_offset,
                                const int32_t* const* local_row_offsets, const int32_t* const* local_cols,
                                const double* const* local_values, const int32_t* halo_counts,
                                const int32_t* const* halo_rows, const int32_t* const* halo_cols,
                                const int32_t* const* halo_peers, const double* const* halo_values, int n_engines,
                                const int32_t* rank_to_engine, const int32_t* engine_row_offset, const double* b,
                                const double* x0, double* x, const bcs_solver_config* cfg, bcs_report* report) {
    return guarded(ctx, [&] {
        if (!rank_row_offset || !local_row_offsets || !local_cols || !local_values || !halo_counts || !rank_to_engine ||
            !engine_row_offset || !b || !x0 || !x)
            throw std::invalid_argument("bcs_dist_solve_parts: null argument");
        bcs_report rep{};
        eng(ctx).distSolveParts(n_ranks, block_size, rank_row_offset, local_row_offsets, local_cols, local_values,
                                halo_counts, halo_rows, halo_cols, halo_peers, halo_values, n_engines, rank_to_engine,
                                engine_row_offset, b, x0, x, cfgOf(cfg), rep);
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

bcs_status bcs_partition_gather_values(const bcs_partition* p, int part, int n_cells, int n_faces, int block_size,
                                       const double* diag, const double* upper, const double* lower,
                                       double* local_values, double* halo_values) {
    return guarded(nullptr, [&] {
        if (!p || part < 0 || part >= static_cast<int>(p->parts.size())) throw std::invalid_argument("bad partition index");
        if (block_size < 1 || block_size > 5) throw std::invalid_argument("bcs: block size must be 1..5");
        bcs::gatherPartValues(p->parts[part], n_cells, n_faces, block_size, diag, upper, lower, local_values,
                              halo_values, 8);
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

bcs_status bcs_assemble_euler_patches(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner,
                                      const int32_t* neighbour, const double* face_area, int n_bfaces,
                                      const int32_t* bface_cell, const double* bface_area, const int32_t* bface_kind,
                                      const double* q, const double* q_inf, double cfl, double* rhs) {
    return guarded(ctx, [&] {
        if (n_cells < 1 || n_faces < 0 || !q || !q_inf || !rhs || (n_faces && (!owner || !neighbour || !face_area)) ||
            (n_bfaces && (!bface_cell || !bface_area)))
            throw std::invalid_argument("bcs_assemble_euler: bad arguments");
        eng(ctx).assembleEuler(n_cells, n_faces, owner, neighbour, face_area, n_bfaces, bface_cell, bface_area,
                               bface_kind, q, q_inf, cfl, rhs);
    });
}

bcs_status bcs_assemble_euler_ex(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner,
                                 const int32_t* neighbour, const double* face_area, const double* face_fx,
                                 const double* cell_centroid, int n_bfaces, const int32_t* bface_cell,
                                 const double* bface_area, const int32_t* bface_kind, const double* q,
                                 const double* q_inf, int recon, int flux, double cfl, double* rhs) {
    return guarded(ctx, [&] {
        if (n_cells < 1 || n_faces < 0 || !q || !q_inf || !rhs || (n_faces && (!owner || !neighbour || !face_area)) ||
            (n_bfaces && (!bface_cell || !bface_area)) || recon < 0 || recon > 2 ||
            (recon && (!cell_centroid || (n_faces && !face_fx))))
            throw std::invalid_argument("bcs_assemble_euler_ex: bad arguments");
        eng(ctx).assembleEuler(n_cells, n_faces, owner, neighbour, face_area, n_bfaces, bface_cell, bface_area,
                               bface_kind, q, q_inf, cfl, rhs, recon, face_fx, cell_centroid, flux);
    });
}

bcs_status bcs_assemble_euler(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner, const int32_t* neighbour,
                              const double* face_area, int n_bfaces, const int32_t* bface_cell,
                              const double* bface_area, const double* q, const double* q_inf, double cfl,
                              double* rhs) {
    return bcs_assemble_euler_patches(ctx, n_cells, n_faces, owner, neighbour, face_area, n_bfaces, bface_cell,
                                      bface_area, nullptr, q, q_inf, cfl, rhs);
}

bcs_status bcs_assemble_coupled_ex(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner,
                                   const int32_t* neighbour, const double* face_area, const double* face_fx,
                                   const double* cell_vol, const double* cell_centroid, int n_bfaces,
                                   const int32_t* bface_cell, const double* bface_area, const int32_t* bface_kind,
                                   const double* bface_u, const double* bface_p, const double* state,
                                   const double* phi, double nu, int pin_cell, double pin_value, double* rhs) {
    return guarded(ctx, [&] {
        if (n_cells < 1 || n_faces < 0 || !cell_vol || !cell_centroid || !state || !rhs ||
            (n_faces && (!owner || !neighbour || !face_area || !face_fx || !phi)) ||
            (n_bfaces && (!bface_cell || !bface_area || !bface_kind || !bface_u)))
            throw std::invalid_argument("bcs_assemble_coupled: bad arguments");
        eng(ctx).assembleCoupled(n_cells, n_faces, owner, neighbour, face_area, face_fx, cell_vol, cell_centroid,
                                 n_bfaces, bface_cell, bface_area, bface_kind, bface_u, bface_p, state, phi, nu,
                                 pin_cell, pin_value, rhs);
    });
}

bcs_status bcs_assemble_coupled(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner,
                                const int32_t* neighbour, const double* face_area, const double* face_fx,
                                const double* cell_vol, const double* cell_centroid, int n_bfaces,
                                const int32_t* bface_cell, const double* bface_area, const int32_t* bface_kind,
                                const double* bface_u, const double* state, const double* phi, double nu,
                                int pin_cell, double pin_value, double* rhs) {
    return bcs_assemble_coupled_ex(ctx, n_cells, n_faces, owner, neighbour, face_area, face_fx, cell_vol,
                                   cell_centroid, n_bfaces, bface_cell, bface_area, bface_kind, bface_u, nullptr,
                                   state, phi, nu, pin_cell, pin_value, rhs);
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

bcs_status bcs_selftest_hypot(const double* x, const double* y, double* out, int n) {
    return guarded(nullptr, [&] {
        if (n <= 0) return;
        double *dx = nullptr, *dy = nullptr, *dz = nullptr;
        const size_t b = sizeof(double) * static_cast<size_t>(n);
        bcs::check(cudaMalloc(&dx, b), "cudaMalloc");
        bcs::check(cudaMalloc(&dy, b), "cudaMalloc");
        bcs::check(cudaMalloc(&dz, b), "cudaMalloc");
        cudaMemcpy(dx, x, b, cudaMemcpyHostToDevice);
        cudaMemcpy(dy, y, b, cudaMemcpyHostToDevice);
        bcs::hypot_eval(dx, dy, dz, n, nullptr);
        const cudaError_t e = cudaMemcpy(out, dz, b, cudaMemcpyDeviceToHost);
        cudaFree(dx);
        cudaFree(dy);
        cudaFree(dz);
        bcs::check(e, "hypot selftest");
    });
}

bcs_status bcs_memory_report(bcs_ctx* ctx, char* buf, size_t cap, size_t* needed) {
    return guarded(ctx, [&] {
        const std::string r = eng(ctx).memoryReport();
        if (needed) *needed = r.size() + 1;
        if (buf && cap) {
            const size_t k = std::min(cap - 1, r.size());
            std::memcpy(buf, r.data(), k);
            buf[k] = 0;
        }
    });
}

bcs_status bcs_level_coloring(bcs_ctx* ctx, int level, int* n_colors, int32_t* perm, int32_t* color_offsets) {
    return guarded(ctx, [&] {
        const int c = eng(ctx).levelColoring(level, perm, color_offsets);
        if (n_colors) *n_colors = c;
    });
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
