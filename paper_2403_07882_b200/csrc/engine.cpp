// bcs::Engine implementation — host orchestration of the device path.
//
// Mirrors the reference control flow line by line where it matters for
// parity: SolvePipeline::solve (engine.cpp:47-120), makeCsrPreconditioner
// (engine.cpp:21-29), AmgHierarchy ctor / vcycle (amg.cpp:73-158),
// gmresSolve / bicgstabSolve (krylov.cpp:59-214).  All numerical work is on
// the device; the host only sequences kernels and reads the few scalars the
// reference's control flow branches on.
#include "engine.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <thread>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <map>

namespace bcs {

// ------------------------------------------------------------------ NCCL
// Loaded at run time (dlopen) so libbcs.so has no link-time dependency on
// it: only the multi-process Mode R entry points need it, and they fail with
// a clear error when it is missing.  Search: $BCS_NCCL_LIB, the soname (the
// copy torch already loaded), the venv's nvidia-nccl wheel.
namespace nccl {
struct Api {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
};
const Api& api() {
    static Api a;
    static bool tried = false;
    if (!tried) {
        tried = true;
        std::vector<std::string> names;
        if (const char* e = std::getenv("BCS_NCCL_LIB")) names.emplace_back(e);
        names.emplace_back("libnccl.so.2");
        names.emplace_back("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2");
        void* h = nullptr;
        for (const auto& n : names)
            if ((h = dlopen(n.c_str(), RTLD_NOW | RTLD_GLOBAL))) break;
        if (h) {
            a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
            a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
            a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
            a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(h, "ncclAllGather"));
            a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
            a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
            a.groupStart = reinterpret_cast<decltype(a.groupStart)>(dlsym(h, "ncclGroupStart"));
            a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(dlsym(h, "ncclGroupEnd"));
            a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(h, "ncclGetErrorString"));
        }
    }
    if (!a.getUniqueId || !a.commInitRank || !a.allGather || !a.send || !a.recv || !a.groupStart || !a.groupEnd)
        throw std::runtime_error("bcs: NCCL (libnccl.so.2) not found; set BCS_NCCL_LIB");
    return a;
}
// NCCL failures surface as the reference's distributed-failure runtime_error
// (MailboxNetwork::receive / partitionedMatvec, partition.cpp:254-267, 345-347),
// naming this rank (and the peer for point-to-point operations)
int g_rank = 0;
void ck(ncclResult_t r, const char* what, int peer = -1) {
    if (r != ncclSuccess)
        throw std::runtime_error("distributed failure: rank " + std::to_string(g_rank) + " NCCL " + what +
                                 (peer >= 0 ? " with rank " + std::to_string(peer) : std::string()) + ": " +
                                 (api().errorString ? api().errorString(r) : "error"));
}
}  // namespace nccl

void check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) throw std::bad_alloc();
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {
using clk = std::chrono::steady_clock;
double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

uint64_t hashCombine(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}

// RAII: count launches of one API call into the report
struct LaunchScope {
    LaunchCounter* prev;
    explicit LaunchScope(LaunchCounter* c) : prev(g_launches) { g_launches = c; }
    ~LaunchScope() { g_launches = prev; }
};
}  // namespace

// f(i) for i in [0, n) over up to T host threads (contiguous ranges)
template <class F>
static void parallelFor(int n, int T, F&& f) {
    const int parts = n < (1 << 16) ? 1 : std::max(1, T);
    auto work = [&](int p) {
        const int b = static_cast<int>(static_cast<long long>(n) * p / parts);
        const int e = static_cast<int>(static_cast<long long>(n) * (p + 1) / parts);
        for (int i = b; i < e; ++i) f(i);
    };
    std::vector<std::thread> th;
    for (int p = 1; p < parts; ++p) th.emplace_back(work, p);
    work(0);
    for (auto& t : th) t.join();
}

// element-wise equality of two host arrays in parallel chunks
template <class T>
static bool parallelEqual(const T* a, const T* b, size_t n) {
    const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    const size_t parts = n < (1u << 20) ? 1 : hw;
    std::vector<char> eq(parts, 1);
    auto work = [&](size_t p) { eq[p] = std::equal(a + n * p / parts, a + n * (p + 1) / parts, b + n * p / parts); };
    std::vector<std::thread> th;
    for (size_t p = 1; p < parts; ++p) th.emplace_back(work, p);
    work(0);
    for (auto& t : th) t.join();
    return std::all_of(eq.begin(), eq.end(), [](char c) { return c != 0; });
}

// topologySignature (block_csr.cpp:146-160) — exact, host side
uint64_t topologySignatureHost(int nc, int nf, const int32_t* owner, const int32_t* neigh) {
    uint64_t h = hashCombine(0, static_cast<uint64_t>(static_cast<int64_t>(nc)));
    std::vector<uint64_t> keys(static_cast<size_t>(nf));
    bool sorted = true;
    for (int f = 0; f < nf; ++f) {
        keys[f] = (static_cast<uint64_t>(static_cast<uint32_t>(owner[f])) << 32) | static_cast<uint32_t>(neigh[f]);
        if (f && keys[f] < keys[f - 1]) sorted = false;
    }
    // (owner, neighbour) are non-negative, so unsigned packing preserves the order
    if (!sorted) std::sort(keys.begin(), keys.end());
    for (uint64_t k : keys) {
        h = hashCombine(h, static_cast<uint64_t>(static_cast<int64_t>(static_cast<int32_t>(k >> 32))));
        h = hashCombine(h, static_cast<uint64_t>(static_cast<int64_t>(static_cast<int32_t>(k & 0xffffffffu))));
    }
    return h;
}

void Engine::profMark(const std::string& what) {
    if (!prof_) return;
    sync();
    const auto now = clk::now();
    profRec_.emplace_back(what, secs(profT_, now));
    profT_ = now;
}

void Engine::profDump() {
    if (!prof_ || profRec_.empty()) return;
    std::map<std::string, double> agg;
    std::map<std::string, int> cnt;
    for (auto& [k, v] : profRec_) {
        agg[k] += v;
        cnt[k]++;
    }
    std::fprintf(stderr, "[bcs-profile] %zu marks\n", profRec_.size());
    for (auto& [k, v] : agg) std::fprintf(stderr, "[bcs-profile] %-28s %10.3f ms  (x%d)\n", k.c_str(), v * 1e3, cnt[k]);
    profRec_.clear();
}

Engine::Engine(int device) : device_(device) {
    prof_ = std::getenv("BCS_PROFILE") != nullptr;
    if (const char* m = std::getenv("BCS_AGG_MODE")) aggMode_ = std::atoi(m);    // 1: barrier rounds
    if (const char* m = std::getenv("BCS_DILU_MODE")) diluMode_ = std::atoi(m);  // 1: Kahn levels
    if (const char* m = std::getenv("BCS_DENSE_BLOCKED_MIN")) denseBlockedMin_ = std::atoi(m);
    if (const char* m = std::getenv("BCS_TAIL_ROWS")) tailMaxRows_ = std::atoi(m);
    if (const char* m = std::getenv("BCS_DENSE_TILED_MIN")) denseTiledMin_ = std::atoi(m);
    if (const char* m = std::getenv("BCS_MC_SWEEP")) mcSweep_ = std::atoi(m) != 0;
    if (const char* m = std::getenv("BCS_MC_LAUNCH_MIN")) mcLaunchMin_ = std::atoi(m);
    if (const char* m = std::getenv("BCS_JACOBI_OMEGA")) jacobiOmega_ = std::atof(m);
    check(cudaSetDevice(device), "cudaSetDevice");
    check(cudaStreamCreateWithFlags(&own_, cudaStreamNonBlocking), "cudaStreamCreate");
    stream_ = own_;
    cudaMemPool_t pool;
    check(cudaDeviceGetDefaultMemPool(&pool, device), "cudaDeviceGetDefaultMemPool");
    uint64_t thr = std::numeric_limits<uint64_t>::max();
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    check(cudaMallocHost(reinterpret_cast<void**>(&hStatus_), 8 * sizeof(double)), "cudaMallocHost");
    check(cudaMallocHost(reinterpret_cast<void**>(&hTot_), 2 * 64 * sizeof(int)), "cudaMallocHost");
    check(cudaEventCreate(&ev0_), "cudaEventCreate");
    check(cudaEventCreate(&ev1_), "cudaEventCreate");
    err_.ensure(4, stream_);
    ctr_.ensure(4, stream_);
    ticket_.ensure(4, stream_);
    push_.ensure(64, stream_);
    cudaMemsetAsync(ctr_.p, 0, 4 * sizeof(int), stream_);
    cudaMemsetAsync(ticket_.p, 0, 4 * sizeof(int), stream_);
    partials_.ensure(static_cast<size_t>(reduce_blocks()) + 512, stream_);
    seg_.ensure(65, stream_);
    scal_.ensure(16, stream_);
    sync();
}

Engine::~Engine() {
    cudaSetDevice(device_);
    cudaStreamSynchronize(stream_);
    // device arrays are released with the pool when the context goes away;
    // free explicitly to keep long-lived processes lean
    auto rel = [&](auto& a) { a.release(stream_); };
    for (auto& L : main_.levels) {
        if (L.mc) {
            Level& M = *L.mc;
            rel(M.o_ro); rel(M.o_ci); rel(M.o_dg); rel(M.o_tpos); rel(M.o_v); rel(M.lu); rel(M.rcp); rel(M.perm);
            rel(M.recf); rel(M.recb); rel(M.dlev); rel(M.offf); rel(M.offb); rel(M.piv); rel(M.order);
            rel(M.r); rel(M.y); rel(M.zb);
        }
        rel(L.mcPerm);
        rel(L.mcColorOffD);
        rel(L.o_ro); rel(L.o_ci); rel(L.o_dg); rel(L.o_tpos); rel(L.o_v); rel(L.lu); rel(L.rcp); rel(L.perm); rel(L.recf); rel(L.recb); rel(L.dlev); rel(L.offf); rel(L.offb); rel(L.pkf); rel(L.pkb); rel(L.piv); rel(L.order);
        rel(L.woff); rel(L.woffb);
        rel(L.agg); rel(L.members); rel(L.r); rel(L.z); rel(L.res); rel(L.y); rel(L.zb);
    }
    rel(dOwner_); rel(dNeigh_); rel(ro_); rel(ci_); rel(dg_); rel(tpos_); rel(src_); rel(fill_); rel(vals_);
    rel(ldu_diag_); rel(ldu_upper_); rel(ldu_lower_); rel(main_.dense); rel(main_.dpiv); rel(main_.tailDesc); rel(cnt_); rel(lvl_); rel(push_);
    rel(scanTmp_); rel(dkeys_); rel(dorder_); rel(ddesc_); rel(act2_); rel(flag_); rel(err_); rel(ctr_); rel(choice_); rel(segOff_); rel(cro_); rel(big_); rel(dn_); rel(tblk_);
    rel(str_); rel(keys_); rel(sorted_); rel(V_); rel(w_); rel(zk_); rel(rk_); rel(Hm_); rel(cs_); rel(sn_); rel(g_);
    rel(y_); rel(scal_); rel(partials_); rel(kb_); rel(kx_); rel(bp_); rel(bv_); rel(bs_); rel(bt_); rel(bph_);
    rel(bsh_); rel(brh_); rel(ticket_); rel(seg_); rel(distTmp_); rel(mcSv_); rel(chunkOrd_); rel(chainCnt_); rel(partOrd_);
    for (auto& P : dist_) {
        rel(P.ro); rel(P.ci); rel(P.src); rel(P.dg); rel(P.tpos); rel(P.vals); rel(P.hrow); rel(P.hoff);
        rel(P.hcol); rel(P.hsrc); rel(P.hvals);
        for (auto& L : P.H.levels) {
            rel(L.o_ro); rel(L.o_ci); rel(L.o_dg); rel(L.o_tpos); rel(L.o_v); rel(L.lu); rel(L.rcp); rel(L.perm); rel(L.recf);
            rel(L.recb); rel(L.dlev); rel(L.offf); rel(L.offb); rel(L.pkf); rel(L.pkb); rel(L.piv); rel(L.order); rel(L.agg); rel(L.members); rel(L.r); rel(L.z); rel(L.res);
            rel(L.y); rel(L.zb); rel(L.woff); rel(L.woffb);
        }
        rel(P.H.dense); rel(P.H.dpiv);
        P.H.arena.release(stream_);
    }
    main_.arena.release(stream_);
    cudaStreamSynchronize(stream_);
    for (void* p : stage_) cudaFreeHost(p);
    if (mpStage_) cudaFreeHost(mpStage_);
    if (mpEvPack_) cudaEventDestroy(mpEvPack_);
    if (mpEvComm_) cudaEventDestroy(mpEvComm_);
    if (commStream_) cudaStreamDestroy(commStream_);
    for (cudaEvent_t e : stageEv_) cudaEventDestroy(e);
    if (hStatus_) cudaFreeHost(hStatus_);
    if (hTot_) cudaFreeHost(hTot_);
    if (ev0_) cudaEventDestroy(ev0_);
    if (ev1_) cudaEventDestroy(ev1_);
    for (auto& e : evPool_) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    if (own_) cudaStreamDestroy(own_);
}

void Engine::setStream(cudaStream_t s) {
    sync();
    stream_ = s ? s : own_;
}

void Engine::sync() { check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize"); }

void Engine::checkErr(const char* where) {
    check(cudaGetLastError(), where);
}

int Engine::readErrCell() {
    int v = 0;
    check(cudaMemcpyAsync(&v, err_.p, sizeof(int), cudaMemcpyDeviceToHost, stream_), "read err");
    sync();
    return v;
}

// --------------------------------------------------------------- topology
void Engine::setTopology(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh) {
    LaunchScope ls(&launches_);
    if (n < 1 || n > 5) throw std::invalid_argument("bcs: block size must be 1..5 on the device");
    if (nc < 1 || nf < 0) throw std::invalid_argument("bcs: need n_cells >= 1 and n_faces >= 0");
    for (int f = 0; f < nf; ++f)
        if (owner[f] < 0 || neigh[f] >= nc || owner[f] >= neigh[f])
            throw std::invalid_argument("bcs: face " + std::to_string(f) +
                                        " violates 0 <= owner < neighbour < n_cells");
    // nothing of the previous topology stays usable if this call throws (e.g.
    // out of memory): sizes and host face copies are committed at the end
    hasTopo_ = false;
    hasValues_ = false;
    asmTopo_ = false;
    hlTopo_ = false;
    H_->pcKind = -1;
    const size_t nnz = static_cast<size_t>(nc) + 2 * static_cast<size_t>(nf);
    if (nnz > static_cast<size_t>(std::numeric_limits<int>::max()))
        throw std::invalid_argument("bcs: more than 2^31-1 blocks");
    dOwner_.ensure(nf, stream_);
    dNeigh_.ensure(nf, stream_);
    ro_.ensure(nc + 1, stream_);
    ci_.ensure(nnz, stream_);
    src_.ensure(nnz, stream_);
    dg_.ensure(nc, stream_);
    tpos_.ensure(nnz, stream_);
    fill_.ensure(nc + 1, stream_);
    scanTmp_.ensure(scan_tmp_ints(nnz) + 16, stream_);
    if (nf) {
        check(cudaMemcpyAsync(dOwner_.p, owner, sizeof(int) * nf, cudaMemcpyHostToDevice, stream_), "H2D owner");
        check(cudaMemcpyAsync(dNeigh_.p, neigh, sizeof(int) * nf, cudaMemcpyHostToDevice, stream_), "H2D neigh");
    }
    // K1: row counts -> offsets -> unordered fill -> per-row sort by column
    cudaMemsetAsync(ro_.p, 0, sizeof(int) * (nc + 1), stream_);
    plan_count(nc, nf, dOwner_, dNeigh_, ro_.p, stream_);
    exclusive_scan(ro_.p, nc + 1, push_.p, scanTmp_.p, stream_);
    cudaMemsetAsync(fill_.p, 0, sizeof(int) * (nc + 1), stream_);
    plan_fill(nc, nf, dOwner_, dNeigh_, ro_, fill_.p, ci_.p, src_.p, stream_);
    plan_sort_rows(nc, ro_, ci_.p, src_.p, stream_);
    find_diag(nc, ro_, ci_, dg_.p, stream_);
    cudaMemsetAsync(err_.p, 0, sizeof(int), stream_);
    transpose_pos(nc, ro_, ci_, tpos_.p, err_.p, stream_);
    vals_.ensure(nnz * n * n, stream_);
    checkErr("setTopology");
    if (readErrCell()) throw std::runtime_error("bcs: structurally asymmetric block pattern");
    nc_ = nc;
    nf_ = nf;
    n_ = n;
    hOwner_.assign(owner, owner + nf);
    hNeigh_.assign(neigh, neigh + nf);
    hasTopo_ = true;
}

// assembleJacobian + computeResidual (euler.cpp:361-455; first order, Roe,
// farfield patches) on the device, straight into the BSR slots
void Engine::assemblyTopology(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh) {
    if (!(hasTopo_ && nc == nc_ && nf == nf_ && n_ == n && sameFaces(owner, neigh, nf)))
        setTopology(nc, nf, n, owner, neigh);
    if (asmTopo_) return;
    // cell -> its faces in face order (the reference's accumulation order)
    std::vector<int> cfo(static_cast<size_t>(nc) + 1, 0), cf(2 * static_cast<size_t>(nf));
    for (int f = 0; f < nf; ++f) {
        ++cfo[owner[f] + 1];
        ++cfo[neigh[f] + 1];
    }
    for (int c = 0; c < nc; ++c) cfo[c + 1] += cfo[c];
    std::vector<int> pos(cfo.begin(), cfo.end() - 1);
    for (int f = 0; f < nf; ++f) {
        cf[pos[owner[f]]++] = f;
        cf[pos[neigh[f]]++] = f;
    }
    asmCfo_.ensure(cfo.size(), stream_);
    asmCf_.ensure(cf.size() + 1, stream_);
    check(cudaMemcpyAsync(asmCfo_.p, cfo.data(), sizeof(int) * cfo.size(), cudaMemcpyHostToDevice, stream_), "H2D cfo");
    if (nf) check(cudaMemcpyAsync(asmCf_.p, cf.data(), sizeof(int) * cf.size(), cudaMemcpyHostToDevice, stream_), "H2D cf");
    const size_t nnz = static_cast<size_t>(nc) + 2 * static_cast<size_t>(nf);
    asmInv_.ensure(nnz, stream_);
    assemble_inverse_src(static_cast<int>(nnz), src_, asmInv_.p, stream_);
    sync();  // the host tables are released on return
    asmTopo_ = true;
}

void Engine::assemblyBoundary(int nc, int nb, const int32_t* bcell, std::vector<int>& order) {
    std::vector<int> bco(static_cast<size_t>(nc) + 1, 0);
    order.assign(static_cast<size_t>(nb), 0);
    for (int b = 0; b < nb; ++b) {
        if (bcell[b] < 0 || bcell[b] >= nc) throw std::invalid_argument("bcs_assemble: boundary face cell out of range");
        ++bco[bcell[b] + 1];
    }
    for (int c = 0; c < nc; ++c) bco[c + 1] += bco[c];
    std::vector<int> pos(bco.begin(), bco.end() - 1);
    for (int b = 0; b < nb; ++b) order[pos[bcell[b]]++] = b;
    asmBco_.ensure(bco.size(), stream_);
    check(cudaMemcpyAsync(asmBco_.p, bco.data(), sizeof(int) * bco.size(), cudaMemcpyHostToDevice, stream_), "H2D bco");
    sync();  // bco is a stack temporary
}

// assembleJacobian + computeResidual (euler.cpp:361-455; first order, Roe,
// any patch kinds, ghostState :320-341) on the device, straight into the BSR slots
void Engine::assembleEuler(int nc, int nf, const int32_t* owner, const int32_t* neigh, const double* faceArea,
                           int nb, const int32_t* bcell, const double* barea, const int32_t* bkind, const double* q,
                           const double* qinf, double cfl, double* rhs, int recon, const double* faceFx,
                           const double* cellCen, int flux) {
    LaunchScope ls(&launches_);
    if (nb < 0) throw std::invalid_argument("bcs_assemble_euler: n_bfaces < 0");
    if (recon < 0 || recon > 2) throw std::invalid_argument("bcs_assemble_euler: unknown reconstruction");
    if (flux < 0 || flux > 2) throw std::invalid_argument("unknown flux scheme");  // euler.cpp:202
    if (recon && (!cellCen || (nf && !faceFx)))
        throw std::invalid_argument("bcs_assemble_euler: MUSCL needs face_fx and cell_centroid");
    if (bkind)
        for (int b = 0; b < nb; ++b)
            if (bkind[b] < 0 || bkind[b] > 5) throw std::invalid_argument("unknown patch kind");  // euler.cpp:340
    assemblyTopology(nc, nf, 5, owner, neigh);
    std::vector<int> border;
    assemblyBoundary(nc, nb, bcell, border);
    std::vector<double> bsorted(3 * static_cast<size_t>(nb));
    std::vector<int> ksorted(bkind ? static_cast<size_t>(nb) : 0);
    for (int k = 0; k < nb; ++k) {
        for (int d = 0; d < 3; ++d) bsorted[3 * static_cast<size_t>(k) + d] = barea[3 * static_cast<size_t>(border[k]) + d];
        if (bkind) ksorted[k] = bkind[border[k]];
    }
    if (bkind) {
        asmBkind_.ensure(ksorted.size() + 1, stream_);
        if (nb)
            check(cudaMemcpyAsync(asmBkind_.p, ksorted.data(), sizeof(int) * ksorted.size(), cudaMemcpyHostToDevice,
                                  stream_),
                  "H2D bkind");
    }
    const size_t N = static_cast<size_t>(nc) * 5;
    asmArea_.ensure(3 * static_cast<size_t>(nf) + 3, stream_);
    asmBarea_.ensure(bsorted.size() + 3, stream_);
    asmQ_.ensure(N + 5, stream_);
    asmRhs_.ensure(N, stream_);
    if (nf)
        h2d(asmArea_.p, faceArea, sizeof(double) * 3 * nf, "H2D area");
    if (nb)
        check(cudaMemcpyAsync(asmBarea_.p, bsorted.data(), sizeof(double) * bsorted.size(), cudaMemcpyHostToDevice, stream_),
              "H2D barea");
    h2d(asmQ_.p, q, sizeof(double) * N, "H2D q");
    check(cudaMemcpyAsync(asmQ_.p + N, qinf, sizeof(double) * 5, cudaMemcpyHostToDevice, stream_), "H2D qinf");
    asmBad_.ensure(1, stream_);
    check(cudaMemsetAsync(asmBad_.p, 0x7f, sizeof(int), stream_), "memset bad");  // 0x7f7f7f7f > any cell index
    const double *fsL = nullptr, *fsR = nullptr;
    if (recon) {  // musclReconstruct on the device (euler.cpp:236-312)
        asmFx_.ensure(static_cast<size_t>(nf) + 1, stream_);
        asmCen_.ensure(3 * static_cast<size_t>(nc), stream_);
        asmMuGrad_.ensure(15 * static_cast<size_t>(nc), stream_);
        asmPsi_.ensure(5 * static_cast<size_t>(nc), stream_);
        asmFs_.ensure(10 * static_cast<size_t>(nf) + 1, stream_);
        if (nf)
            h2d(asmFx_.p, faceFx, sizeof(double) * nf, "H2D fx");
        h2d(asmCen_.p, cellCen, sizeof(double) * 3 * nc, "H2D cen");
        fsL = asmFs_.p;
        fsR = asmFs_.p + 5 * static_cast<size_t>(nf);
        assemble_euler_muscl(nc, nf, dOwner_, dNeigh_, asmCfo_, asmCf_, asmCen_, asmFx_, asmQ_, recon == 2 ? 1 : 0,
                             asmMuGrad_, asmPsi_, asmFs_.p, asmFs_.p + 5 * static_cast<size_t>(nf), stream_);
    }
    assemble_euler(nc, nf, dOwner_, dNeigh_, asmArea_, asmCfo_, asmCf_, asmBco_, asmBarea_,
                   bkind ? asmBkind_.p : nullptr, fsL, fsR, flux, asmQ_, asmQ_.p + N, cfl, asmInv_, vals_.p, asmRhs_.p,
                   asmBad_.p, stream_);
    int firstBad = 0;
    check(cudaMemcpyAsync(&firstBad, asmBad_.p, sizeof(int), cudaMemcpyDeviceToHost, stream_), "D2H bad");
    d2h(rhs, asmRhs_.p, sizeof(double) * N, "D2H rhs");  // synchronous
    checkErr("assembleEuler");
    if (firstBad < nc) {  // the values written are not a valid system
        hasValues_ = false;
        H_->pcKind = -1;
        throw std::runtime_error("non-physical state in cell " + std::to_string(firstBad));
    }
    hasValues_ = true;
    H_->pcKind = -1;  // any preconditioner built on old values is stale
}

// assembleCoupled + pinPressure (incompressible.cpp:143-264) on the device:
// IncompressibleBc kinds per boundary face (0 wall, 1 moving wall, 2 inlet,
// 3 outlet), velocity bu (moving wall / inlet), pressure bp (outlet)
void Engine::assembleCoupled(int nc, int nf, const int32_t* owner, const int32_t* neigh, const double* faceArea,
                             const double* fx, const double* vol, const double* cen, int nb, const int32_t* bcell,
                             const double* barea, const int32_t* bkind, const double* bu, const double* bp,
                             const double* state, const double* phi, double nu, int pinCell, double pinValue,
                             double* rhs) {
    LaunchScope ls(&launches_);
    if (nb < 0) throw std::invalid_argument("bcs_assemble_coupled: n_bfaces < 0");
    for (int b = 0; b < nb; ++b) {
        if (bkind[b] < 0 || bkind[b] > 3)
            throw std::invalid_argument("bcs_assemble_coupled: unknown boundary kind " + std::to_string(bkind[b]));
        if (bkind[b] == 3 && !bp) throw std::invalid_argument("bcs_assemble_coupled: outlet patches need bface_p");
    }
    if (pinCell >= nc) throw std::invalid_argument("bcs_assemble_coupled: pin cell out of range");
    assemblyTopology(nc, nf, 4, owner, neigh);
    std::vector<int> border;
    assemblyBoundary(nc, nb, bcell, border);
    std::vector<double> ba(3 * static_cast<size_t>(nb)), bv(3 * static_cast<size_t>(nb)), bps(nb, 0.0);
    std::vector<int> bks(nb);
    for (int k = 0; k < nb; ++k) {
        for (int d = 0; d < 3; ++d) {
            ba[3 * static_cast<size_t>(k) + d] = barea[3 * static_cast<size_t>(border[k]) + d];
            bv[3 * static_cast<size_t>(k) + d] = bu[3 * static_cast<size_t>(border[k]) + d];
        }
        bks[k] = bkind[border[k]];
        if (bp) bps[k] = bp[border[k]];
    }
    const size_t N = static_cast<size_t>(nc) * 4;
    asmArea_.ensure(3 * static_cast<size_t>(nf) + 3, stream_);
    asmFx_.ensure(static_cast<size_t>(nf) + 1, stream_);
    asmPhi_.ensure(static_cast<size_t>(nf) + 1, stream_);
    asmVol_.ensure(nc, stream_);
    asmCen_.ensure(3 * static_cast<size_t>(nc), stream_);
    asmBarea_.ensure(ba.size() + 3, stream_);
    asmBu_.ensure(bv.size() + 3, stream_);
    asmBkind_.ensure(bks.size() + 1, stream_);
    asmBp_.ensure(bps.size() + 1, stream_);
    asmQ_.ensure(N, stream_);
    asmD_.ensure(nc, stream_);
    asmGrad_.ensure(3 * static_cast<size_t>(nc), stream_);
    asmRhs_.ensure(N, stream_);
    if (nf) {
        h2d(asmArea_.p, faceArea, sizeof(double) * 3 * nf, "H2D area");
        h2d(asmFx_.p, fx, sizeof(double) * nf, "H2D fx");
        h2d(asmPhi_.p, phi, sizeof(double) * nf, "H2D phi");
    }
    check(cudaMemcpyAsync(asmVol_.p, vol, sizeof(double) * nc, cudaMemcpyHostToDevice, stream_), "H2D vol");
    h2d(asmCen_.p, cen, sizeof(double) * 3 * nc, "H2D cen");
    if (nb) {
        check(cudaMemcpyAsync(asmBarea_.p, ba.data(), sizeof(double) * ba.size(), cudaMemcpyHostToDevice, stream_),
              "H2D barea");
        check(cudaMemcpyAsync(asmBu_.p, bv.data(), sizeof(double) * bv.size(), cudaMemcpyHostToDevice, stream_), "H2D bu");
        check(cudaMemcpyAsync(asmBkind_.p, bks.data(), sizeof(int) * bks.size(), cudaMemcpyHostToDevice, stream_),
              "H2D bkind");
        check(cudaMemcpyAsync(asmBp_.p, bps.data(), sizeof(double) * bps.size(), cudaMemcpyHostToDevice, stream_),
              "H2D bp");
    }
    h2d(asmQ_.p, state, sizeof(double) * N, "H2D state");
    assemble_coupled(nc, nf, dOwner_, dNeigh_, asmArea_, asmFx_, asmVol_, asmCen_, asmCfo_, asmCf_, asmBco_, asmBarea_,
                     asmBu_, asmBkind_, asmBp_, asmQ_, asmPhi_, nu, pinCell, pinValue, asmInv_, asmD_.p, asmGrad_.p, vals_.p, asmRhs_.p,
                     stream_);
    d2h(rhs, asmRhs_.p, sizeof(double) * N, "D2H rhs");  // synchronous
    checkErr("assembleCoupled");
    hasValues_ = true;
    H_->pcKind = -1;
}

// Staged H2D (pinned streaming upload): kWorkers host
// threads each own two pinned kChunk slots; worker w copies chunks w, w + W,
// w + 2W, ... of the source into its next free slot (waiting for that slot's
// previous DMA through its event) and enqueues the DMA on the engine stream.
// Chunks land at disjoint offsets, so their order on the stream is free; work
// enqueued after h2d returns sees every chunk.
namespace {
constexpr size_t kStageChunk = size_t(32) << 20;  // slot size (measured: 32 MB beats 8 MB)
// copies up to one slot go straight from pageable memory; spreading 84 MB
// vectors over smaller chunks measured no better than whole 32 MB slots
constexpr size_t kStageDirect = kStageChunk;
inline size_t stageChunk(size_t) { return kStageChunk; }
constexpr int kStageWorkers = 8, kStageSlots = 2;
}  // namespace

bool Engine::hostPinned(const void* p) const {
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();  // a pageable pointer is not an error worth keeping
    return pinned;
}

void Engine::ensureStaging() {
    if (!stage_.empty()) return;
    for (int k = 0; k < kStageWorkers * kStageSlots; ++k) {
        void* p = nullptr;
        check(cudaHostAlloc(&p, kStageChunk, cudaHostAllocPortable), "cudaHostAlloc staging");
        stage_.push_back(p);
        cudaEvent_t e;
        check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate staging");
        stageEv_.push_back(e);
    }
}

void Engine::h2d(void* dst, const void* src, size_t bytes, const char* what) {
    if (!bytes) return;
    const size_t kChunk = stageChunk(bytes);
    constexpr int kWorkers = kStageWorkers, kSlots = kStageSlots;
    if (bytes <= kStageDirect || hostPinned(src)) {
        check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream_), what);
        return;
    }
    ensureStaging();
    const size_t nChunks = (bytes + kChunk - 1) / kChunk;
    const int workers = static_cast<int>(std::min<size_t>(kWorkers, nChunks));
    std::vector<cudaError_t> errs(workers, cudaSuccess);
    auto work = [&](int w) {
        cudaSetDevice(device_);
        int j = 0;
        for (size_t i = w; i < nChunks; i += workers, ++j) {
            const int k = w * kSlots + (j % kSlots);
            if (j >= kSlots) {
                const cudaError_t e = cudaEventSynchronize(stageEv_[k]);
                if (e != cudaSuccess) { errs[w] = e; return; }
            }
            const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
            std::memcpy(stage_[k], static_cast<const char*>(src) + off, len);
            cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + off, stage_[k], len, cudaMemcpyHostToDevice,
                                            stream_);
            if (e == cudaSuccess) e = cudaEventRecord(stageEv_[k], stream_);
            if (e != cudaSuccess) { errs[w] = e; return; }
        }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < workers; ++w) pool.emplace_back(work, w);
    work(0);
    for (auto& t : pool) t.join();
    for (cudaError_t e : errs) check(e, what);
    // the staging slots are reused by the next call: drain this call's DMAs first
    for (int k = 0; k < workers * kSlots; ++k) check(cudaEventSynchronize(stageEv_[k]), what);
}

// D2H into a pageable buffer: each worker DMAs its chunks into its pinned
// slots (in stream order after the work that produced src) and copies them
// out as they land.
void Engine::d2h(void* dst, const void* src, size_t bytes, const char* what) {
    if (!bytes) return;
    if (bytes <= kStageDirect || hostPinned(dst)) {
        check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream_), what);
        sync();
        return;
    }
    ensureStaging();
    const size_t kChunk = stageChunk(bytes);
    const size_t nChunks = (bytes + kChunk - 1) / kChunk;
    const int workers = static_cast<int>(std::min<size_t>(kStageWorkers, nChunks));
    std::vector<cudaError_t> errs(workers, cudaSuccess);
    auto work = [&](int w) {
        cudaSetDevice(device_);
        for (size_t i = w; i < nChunks; i += workers) {
            const int k = w * kStageSlots;
            const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
            cudaError_t e = cudaMemcpyAsync(stage_[k], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost,
                                            stream_);
            if (e == cudaSuccess) e = cudaEventRecord(stageEv_[k], stream_);
            if (e == cudaSuccess) e = cudaEventSynchronize(stageEv_[k]);
            if (e != cudaSuccess) { errs[w] = e; return; }
            std::memcpy(static_cast<char*>(dst) + off, stage_[k], len);
        }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < workers; ++w) pool.emplace_back(work, w);
    work(0);
    for (auto& t : pool) t.join();
    for (cudaError_t e : errs) check(e, what);
}

void Engine::uploadLdu(const double* diag, const double* upper, const double* lower, bool device_ptrs) {
    LaunchScope ls(&launches_);
    if (!hasTopo_) throw std::invalid_argument("bcs: set the topology before uploading values");
    const size_t nn = static_cast<size_t>(n_) * n_;
    const double *dd = diag, *du = upper, *dl = lower;
    if (!device_ptrs) {
        ldu_diag_.ensure(nc_ * nn, stream_);
        ldu_upper_.ensure(nf_ * nn, stream_);
        ldu_lower_.ensure(nf_ * nn, stream_);
        h2d(ldu_diag_.p, diag, sizeof(double) * nc_ * nn, "H2D diag");
        if (nf_) {
            h2d(ldu_upper_.p, upper, sizeof(double) * nf_ * nn, "H2D upper");
            h2d(ldu_lower_.p, lower, sizeof(double) * nf_ * nn, "H2D lower");
        }
        dd = ldu_diag_;
        du = ldu_upper_;
        dl = ldu_lower_;
    }
    // K2: replaceValues permutation
    gather_values(n_, nc_ + 2 * nf_, nc_, nf_, src_, dd, du, dl, vals_.p, stream_);
    checkErr("uploadLdu");
    hasValues_ = true;
    H_->pcKind = -1;  // any preconditioner built on old values is stale
}

void Engine::requireMatrix() const {
    if (!hasTopo_ || !hasValues_) throw std::invalid_argument("bcs: no matrix uploaded");
}

// Fine-level SpMV launches are bracketed by CUDA events on the launching
// stream when kernel timing is on; the pairs are read after the solve's final
// synchronisation, so timing never adds a host sync inside the solve.
void Engine::spmvLevel(const Level& L, const double* x, const double* sub, double* y) {
    const bool timed = kernelTiming_ && &L == &H_->levels[0];
    if (timed) timerBegin();
    spmv(n_, L.rows, L.ro, L.ci, L.v, x, sub, y, stream_);
    if (timed) timerEnd(0, 0.0);
}

void Engine::timerBegin() {
    if (evUsed_ == evPool_.size()) {
        cudaEvent_t a, b;
        check(cudaEventCreate(&a), "cudaEventCreate");
        check(cudaEventCreate(&b), "cudaEventCreate");
        evPool_.push_back({a, b});
        evKind_.push_back(0);
        evBytes_.push_back(0.0);
    }
    cudaEventRecord(evPool_[evUsed_].first, stream_);
}

void Engine::timerEnd(int kind, double bytes) {
    cudaEventRecord(evPool_[evUsed_].second, stream_);
    evKind_[evUsed_] = kind;
    evBytes_[evUsed_] = bytes;
    ++evUsed_;
}

void Engine::collectSpmvTimes() {
    for (size_t i = 0; i < evUsed_; ++i) {
        float ms = 0.f;
        check(cudaEventElapsedTime(&ms, evPool_[i].first, evPool_[i].second), "cudaEventElapsedTime");
        if (evKind_[i] == 0) {
            spmvMs_ += ms;
            ++spmvCount_;
        } else {
            sweepMs_ += ms;
            sweepBytes_ += evBytes_[i];
            ++sweepCount_;
        }
    }
    evUsed_ = 0;
}

// ------------------------------------------------------------ config/setup
void Engine::validateConfig(const bcs_solver_config& c) const {
    // SolverConfig::validate (krylov.cpp:10-18)
    if (!(c.rel_tol > 0.0) || !(c.abs_tol > 0.0)) throw std::invalid_argument("SolverConfig: tolerances must be positive");
    if (c.max_iters < 1) throw std::invalid_argument("SolverConfig: maxIters must be >= 1");
    if (c.gmres_restart < 1) throw std::invalid_argument("SolverConfig: gmresRestart must be >= 1");
    if (c.amg_max_levels < 1) throw std::invalid_argument("SolverConfig: amg.maxLevels must be >= 1");
    if (c.amg_pre_sweeps < 0 || c.amg_post_sweeps < 0) throw std::invalid_argument("SolverConfig: amg sweeps must be >= 0");
    if (c.method != BCS_GMRES && c.method != BCS_BICGSTAB && c.method != BCS_FGMRES) throw std::invalid_argument("unknown Krylov method");
    if (c.precond < 0 || c.precond > 3) throw std::invalid_argument("unknown preconditioner kind");
    if (c.mode != BCS_MODE_PARITY && c.mode != BCS_MODE_PERF && c.mode != BCS_MODE_EXACT &&
        c.mode != BCS_MODE_PERF_JACOBI)
        throw std::invalid_argument("bcs: unknown mode");
}

void Engine::setupLevelPattern(Level& L) {
    L.o_dg.ensure(L.rows, stream_);
    L.o_tpos.ensure(L.nnz, stream_);
    find_diag(L.rows, L.ro, L.ci, L.o_dg.p, stream_);
    cudaMemsetAsync(err_.p, 0, sizeof(int), stream_);
    transpose_pos(L.rows, L.ro, L.ci, L.o_tpos.p, err_.p, stream_);
    L.dg = L.o_dg;
    L.tpos = L.o_tpos;
    if (readErrCell()) throw std::runtime_error("bcs: structurally asymmetric coarse pattern");
}

static KahnWork kahnWork(DArray<int>& cnt, DArray<int>& push, DArray<int>& lvl, int* lvl2 = nullptr) {
    return KahnWork{cnt.p, push.p, lvl.p, lvl2};
}

// DILU smoothers of the levels lv (preconditioner.cpp:101-126): dependency
// levels per matrix, then ONE sync-free factorisation over all of them
// (tickets ordered by dependency level, then matrix), then the sweeps' data.
void Engine::diluSetupAll(const std::vector<Level*>& lv, const bcs_solver_config* cfg) {
    const int nl = static_cast<int>(lv.size());
    const size_t nn = static_cast<size_t>(n_) * n_;
    const int big = std::numeric_limits<int>::max();
    if (diluMode_ != 0) {  // Kahn-rounds variant (BCS_DILU_MODE=1), level by level
        for (int l = 0; l < nl; ++l) {
            Level& L = *lv[l];
            L.lu.ensure(L.rows * nn, stream_);
            L.piv.ensure(static_cast<size_t>(L.rows) * n_, stream_);
            L.order.ensure(L.rows, stream_);
            cnt_.ensure(static_cast<size_t>(L.rows) + 2, stream_);
            lvl_.ensure(static_cast<size_t>(L.rows) + 1, stream_);
            tblk_.ensure(static_cast<size_t>(L.nnz) * nn, stream_);
            check(cudaMemcpyAsync(err_.p, &big, sizeof(int), cudaMemcpyHostToDevice, stream_), "err init");
            L.depth = kahn_schedule(n_, L.rows, L.ro, L.ci, L.dg, L.tpos, L.v, true, L.lu.p, L.piv.p, tblk_.p,
                                    L.order.p, kahnWork(cnt_, push_, lvl_), err_.p, stream_);
            const int cell = readErrCell();
            if (cell != big)
                throw std::runtime_error("DILU setup: singular modified diagonal in cell " + std::to_string(cell));
            L.dlevOk = false;
        }
        finishSmoothers(lv, nullptr);
        return;
    }
    size_t totalRows = 0, totalT = 0, maxRows = 0;
    int maxdepth = 0;
    cudaMemsetAsync(err_.p + 2, 0, sizeof(int), stream_);
    std::vector<LevelsHost> lh(nl);
    for (int l = 0; l < nl; ++l) {
        Level& L = *lv[l];
        L.lu.ensure(L.rows * nn, stream_);
        L.piv.ensure(static_cast<size_t>(L.rows) * n_, stream_);
        L.order.ensure(L.rows, stream_);
        L.dlev.ensure(L.rows, stream_);
        L.dlevOk = true;
        lh[l] = {L.rows, L.ro, L.ci, L.dg, L.dlev.p, L.order.p};
        totalRows += L.rows;
        maxRows = std::max(maxRows, static_cast<size_t>(L.rows));
    }
    cnt_.ensure(maxRows + 2, stream_);
    scanTmp_.ensure(scan_tmp_ints(maxRows + 2) + 16, stream_);
    ddesc_.ensure(dilu_desc_bytes(), stream_);
    std::vector<int> depth(nl, 0);
    level_schedule_multi(nl, lh.data(), depth.data(), cnt_.p, scanTmp_.p, push_.p, ddesc_.p, err_.p + 2, stream_);
    for (int l = 0; l < nl; ++l) {
        lv[l]->depth = depth[l];
        maxdepth = std::max(maxdepth, depth[l]);
    }
    profMark("dilu:levels");
    // T (D~_j^-1 A_ji per lower slot) is setup-phase memory: compact (lower
    // slots only) and released when the factorisation is done
    std::vector<DiluLevelHost> desc(nl);
    size_t toff = 0;
    {
        // setup phase of the arena: tc + lpre per level and T (lower slots:
        // (nnz - rows) / 2 blocks, the patterns being structurally symmetric)
        size_t bytes = 0;
        for (int l = 0; l < nl; ++l) {
            const Level& L = *lv[l];
            bytes += PhaseArena::al(sizeof(int) * (static_cast<size_t>(L.rows) + 1)) +
                     PhaseArena::al(sizeof(int) * static_cast<size_t>(L.nnz));
            totalT += (static_cast<size_t>(L.nnz) - L.rows) / 2 * nn;
        }
        dropArenaViews();
        H_->arena.reserve(bytes + PhaseArena::al(sizeof(double) * (totalT + 1)), stream_);
        for (int l = 0; l < nl; ++l) {
            Level& L = *lv[l];
            L.lpre.borrow(H_->arena.take<int>(static_cast<size_t>(L.rows) + 1), static_cast<size_t>(L.rows) + 1, stream_);
            L.tc.borrow(H_->arena.take<int>(L.nnz), L.nnz, stream_);
        }
        tblk_.borrow(H_->arena.take<double>(totalT + 1), totalT + 1, stream_);
    }
    for (int l = 0; l < nl; ++l) {
        Level& L = *lv[l];
        scanTmp_.ensure(scan_tmp_ints(static_cast<size_t>(L.rows) + 1) + 16, stream_);
        const size_t lower = dilu_compact_index(L.rows, L.ro, L.dg, L.ci, L.tpos, L.lpre.p, L.tc.p, push_.p + 9,
                                                scanTmp_.p, stream_);
        desc[l] = {L.rows, L.ro, L.dg, L.tpos, L.tc.p, L.lpre.p, L.dlev.p, L.v, L.lu.p, L.piv.p, toff};
        toff += lower * nn;
    }
    if (toff > totalT) throw std::logic_error("bcs: DILU scratch larger than its lower-slot bound");
    totalT = toff;
    const size_t buckets = static_cast<size_t>(maxdepth) * nl + 1;
    dkeys_.ensure(totalRows, stream_);
    dorder_.ensure(totalRows, stream_);
    cnt_.ensure(buckets + 1, stream_);
    scanTmp_.ensure(scan_tmp_ints(buckets + 1) + 16, stream_);
    ddesc_.ensure(dilu_desc_bytes(), stream_);
    check(cudaMemcpyAsync(err_.p, &big, sizeof(int), cudaMemcpyHostToDevice, stream_), "err init");
    dilu_setup_multi(n_, nl, desc.data(), maxdepth, dkeys_.p, dorder_.p, cnt_.p, scanTmp_.p, push_.p + 8, ddesc_.p,
                     tblk_.p, totalT, err_.p, err_.p + 2, stream_);
    int e2 = 0;
    check(cudaMemcpyAsync(&e2, err_.p + 2, sizeof(int), cudaMemcpyDeviceToHost, stream_), "err");
    const int cell = readErrCell();  // syncs
    if (e2) throw std::runtime_error("bcs: DILU setup dependency wait timed out");
    if (cell != big)
        throw std::runtime_error("DILU setup: singular modified diagonal in cell " + std::to_string(cell & ((1 << 26) - 1)));
    profMark("dilu:factor");
    finishSmoothers(lv, cfg);
}

// Engine-level arrays that borrow arena memory (the serial Krylov basis, the
// DILU scratch T) are views of the phase they were taken in: a new reserve
// recycles that memory, so the views are dropped first and the next ensure()
// allocates (e.g. a LUSGS setup after an AMG solve on the same context).
void Engine::dropArenaViews() {
    for (auto* a : {&V_, &Z_, &tblk_})
        if (!a->owned) a->release(stream_);
}

// reciprocals, composed permutations, ticket records and packed slots of
// the levels lv; the sweep programs (and, for a serial GMRES solve, the
// Krylov basis) are the solve phase of the hierarchy's arena.  cfg == nullptr:
// no Krylov basis reserved (preconditioner-only setups).
void Engine::finishSmoothers(const std::vector<Level*>& lv, const bcs_solver_config* cfg) {
    const int nl = static_cast<int>(lv.size());
    if (nl > 64) throw std::logic_error("bcs: more than 64 smoothed levels");
    // chain schedules (opt-in, BCS_CHAIN=1) for wide levels whose rows mostly
    // chain to the previous row (natural-order meshes): see k_chain_starts.
    // Measured at 128^3 it loses to the level order (0.310 vs 0.2935 s/step):
    // every y/z coupling is a cross-warp hop between lines in flight at the
    // same time, so the rows advance at the hop rate.
    static const bool chainOn = [] {
        const char* e = std::getenv("BCS_CHAIN");
        return e && std::atoi(e) != 0;
    }();
    static const int chainMinWidth = [] {  // rows per dependency level
        const char* e = std::getenv("BCS_CHAIN_MIN_WIDTH");
        return e ? std::atoi(e) : 4096;
    }();
    auto candidate = [&](const Level& L) {
        return chainOn && !L.colourSweep && L.dlevOk && L.depth > 0 && L.rows / L.depth >= chainMinWidth;
    };
    int chains[2 * 64];
    bool anyCand = false;
    chainCnt_.ensure(2 * 64, stream_);
    cudaMemsetAsync(chainCnt_.p, 0, 2 * 64 * sizeof(int), stream_);
    for (int l = 0; l < nl; ++l) {
        Level& L = *lv[l];
        L.chain = false;
        if (candidate(L)) {
            chain_count(L.rows, L.ro, L.dg, L.ci, chainCnt_.p + l, stream_);
            anyCand = true;
        }
    }
    if (anyCand) {
        check(cudaMemcpyAsync(chains, chainCnt_.p, nl * sizeof(int), cudaMemcpyDeviceToHost, stream_), "chains");
        sync();
        size_t need = 0;
        for (int l = 0; l < nl; ++l) {
            Level& L = *lv[l];
            L.chain = candidate(L) && 2LL * chains[l] >= L.rows;
            if (L.chain) need += 2 * static_cast<size_t>(L.rows);
        }
        // the schedules (orders in chunkOrd_, checked before use)
        chunkOrd_.ensure(need, stream_);
        size_t at = 0;
        for (int l = 0; l < nl; ++l) {
            Level& L = *lv[l];
            if (!L.chain) continue;
            const int Wf = sweep_chunk_warps(n_, true), Wb = sweep_chunk_warps(n_, false);
            L.woff.ensure(static_cast<size_t>(Wf) + 1, stream_);
            L.woffb.ensure(static_cast<size_t>(Wb) + 1, stream_);
            chain_schedule(L.rows, true, L.depth, L.ro, L.dg, L.ci, L.dlev, Wf, chunkOrd_.p + at, L.woff.p,
                           chainCnt_.p + 64 + l, stream_);
            chain_schedule(L.rows, false, L.depth, L.ro, L.dg, L.ci, L.dlev, Wb, chunkOrd_.p + at + L.rows,
                           L.woffb.p, chainCnt_.p + 64 + l, stream_);
            at += 2 * static_cast<size_t>(L.rows);
        }
        check(cudaMemcpyAsync(chains + 64, chainCnt_.p + 64, nl * sizeof(int), cudaMemcpyDeviceToHost, stream_),
              "chain check");
        sync();
        static const bool verbose = std::getenv("BCS_CHAIN_VERBOSE") != nullptr;
        for (int l = 0; l < nl; ++l) {
            if (lv[l]->chain && chains[64 + l]) lv[l]->chain = false;  // progress check failed: level order
            if (verbose && candidate(*lv[l]))
                std::fprintf(stderr, "bcs chain: level rows %d depth %d chained %d -> %s\n", lv[l]->rows,
                             lv[l]->depth, chains[l], lv[l]->chain ? "chain schedule" : "level order");
        }
    }
    for (int l = 0; l < nl; ++l) {
        Level& L = *lv[l];
        L.rcp.ensure(static_cast<size_t>(L.rows) * n_, stream_);
        L.perm.ensure(static_cast<size_t>(L.rows) * n_, stream_);
        make_reciprocals(n_, L.rows, L.lu, L.piv, L.rcp.p, L.perm.p, stream_);
        if (L.colourSweep) {  // no sweep programs
            hTot_[2 * l] = hTot_[2 * l + 1] = 0;
            continue;
        }
        L.recf.ensure(4 * static_cast<size_t>(L.rows), stream_);
        L.recb.ensure(4 * static_cast<size_t>(L.rows), stream_);
        if (L.chain) {
            size_t at = 0;  // this level's schedules in chunkOrd_
            for (int k = 0; k < l; ++k)
                if (lv[k]->chain) at += 2 * static_cast<size_t>(lv[k]->rows);
            sweep_records(L.rows, chunkOrd_.p + at, chunkOrd_.p + at + L.rows, L.ro, L.dg, L.recf.p, L.recb.p,
                          stream_);
        } else if (const int G = sweep_cluster_parts(n_, L.rows, L.depth); G > 1) {
            // several clusters: tickets range-major (each cluster's rows in level order)
            partOrd_.ensure(static_cast<size_t>(L.rows), stream_);
            cluster_part_order(L.rows, G, L.order, partOrd_.p, stream_);
            sweep_records(L.rows, partOrd_.p, nullptr, L.ro, L.dg, L.recf.p, L.recb.p, stream_);
        } else {
            sweep_records(L.rows, L.order, nullptr, L.ro, L.dg, L.recf.p, L.recb.p, stream_);
        }
        const size_t n1 = static_cast<size_t>(L.rows) + 1;
        scanTmp_.ensure(scan_tmp_ints(n1) + 16, stream_);
        for (int d = 0; d < 2; ++d) {
            DArray<int>& off = d == 0 ? L.offf : L.offb;
            off.ensure(n1, stream_);
            sweep_slot_sizes(n_, d == 0, L.rows, L.sweepDepth(), d == 0 ? L.recf : L.recb, off.p, stream_);
            exclusive_scan(off.p, L.rows, off.p + L.rows, scanTmp_.p, stream_);
            check(cudaMemcpyAsync(hTot_ + 2 * l + d, off.p + L.rows, sizeof(int), cudaMemcpyDeviceToHost, stream_),
                  "slot total");
        }
    }
    sync();
    profMark("dilu:rcp+records");
    size_t bytes = 0;
    for (int l = 0; l < 2 * nl; ++l) bytes += PhaseArena::al(16 * static_cast<size_t>(hTot_[l]) + 16);
    // a serial GMRES solve's basis V (and FGMRES's Z) share the phase
    const bool basis = cfg && H_ == &main_ && !distActive_ &&
                       (cfg->method == BCS_GMRES || cfg->method == BCS_FGMRES);
    const size_t N = static_cast<size_t>(H_->levels[0].rows) * n_;
    const size_t nV = basis ? static_cast<size_t>(cfg->gmres_restart + 1) * N : 0;
    const size_t nZ = basis && cfg->method == BCS_FGMRES ? static_cast<size_t>(cfg->gmres_restart) * N : 0;
    if (basis) bytes += PhaseArena::al(nV * sizeof(double)) + (nZ ? PhaseArena::al(nZ * sizeof(double)) : 0);
    dropArenaViews();
    H_->arena.reserve(bytes, stream_);
    if (basis) {
        V_.borrow(H_->arena.take<double>(nV), nV, stream_);
        if (nZ) Z_.borrow(H_->arena.take<double>(nZ), nZ, stream_);
    }
    for (int l = 0; l < nl; ++l) {
        Level& L = *lv[l];
        if (L.colourSweep) continue;
        for (int d = 0; d < 2; ++d) {
            DArray<unsigned char>& pk = d == 0 ? L.pkf : L.pkb;
            const size_t b = 16 * static_cast<size_t>(hTot_[2 * l + d]) + 16;
            pk.borrow(H_->arena.take<unsigned char>(b), b, stream_);
            sweep_pack(n_, d == 0, L.rows, L.sweepDepth(), d == 0 ? L.recf : L.recb, L.ci, L.v, L.lu, L.perm, L.rcp,
                       d == 0 ? L.offf : L.offb, pk.p, stream_);
        }
    }
    profMark("dilu:pack");
}

// performance mode, block Jacobi: the diagonal blocks' LU (luFactor order,
// smallmat.hpp:67-94), reciprocals and composed permutations
void Engine::jacobiSetup(Level& L) {
    const size_t nn = static_cast<size_t>(n_) * n_;
    L.lu.ensure(L.rows * nn, stream_);
    L.piv.ensure(static_cast<size_t>(L.rows) * n_, stream_);
    L.rcp.ensure(static_cast<size_t>(L.rows) * n_, stream_);
    L.perm.ensure(static_cast<size_t>(L.rows) * n_, stream_);
    const int big = std::numeric_limits<int>::max();
    check(cudaMemcpyAsync(err_.p, &big, sizeof(int), cudaMemcpyHostToDevice, stream_), "err init");
    factor_diag_blocks(n_, L.rows, L.dg, L.v, L.lu.p, L.piv.p, err_.p, stream_);
    make_reciprocals(n_, L.rows, L.lu, L.piv, L.rcp.p, L.perm.p, stream_);
    const int cell = readErrCell();
    if (cell != big)
        throw std::runtime_error("preconditioner setup: singular diagonal block in cell " + std::to_string(cell));
    L.jacobi = true;
}

void Engine::lusgsSetup(Level& L) {
    const size_t nn = static_cast<size_t>(n_) * n_;
    L.lu.ensure(L.rows * nn, stream_);
    L.piv.ensure(static_cast<size_t>(L.rows) * n_, stream_);
    L.order.ensure(L.rows, stream_);
    cnt_.ensure(L.rows, stream_);
    lvl_.ensure(static_cast<size_t>(L.rows) + 1, stream_);
    const int big = std::numeric_limits<int>::max();
    check(cudaMemcpyAsync(err_.p, &big, sizeof(int), cudaMemcpyHostToDevice, stream_), "err init");
    factor_diag_blocks(n_, L.rows, L.dg, L.v, L.lu.p, L.piv.p, err_.p, stream_);
    const int cell = readErrCell();
    if (cell != big)
        throw std::runtime_error((hostLdu_ ? "LUSGS setup: singular diagonal block in cell "  // preconditioner.cpp:66
                                           : "preconditioner setup: singular diagonal block in cell ") +
                                 std::to_string(cell));
    cnt_.ensure(static_cast<size_t>(L.rows) + 2, stream_);
    scanTmp_.ensure(scan_tmp_ints(static_cast<size_t>(L.rows) + 2) + 16, stream_);
    cudaMemsetAsync(err_.p + 2, 0, sizeof(int), stream_);
    L.dlev.ensure(static_cast<size_t>(L.rows) + 1, stream_);
    L.depth = level_schedule(L.rows, L.ro, L.ci, L.dg, L.order.p, L.dlev.p, cnt_.p, scanTmp_.p, push_.p,
                             err_.p + 2, stream_);
    L.dlevOk = true;
    finishSmoothers({&L}, nullptr);
}

void Engine::buildHierarchy(const bcs_solver_config& cfg) {
    const size_t nn = static_cast<size_t>(n_) * n_;
    H_->nlev = 1;
    // coarsening loop (amg.cpp:75-84)
    while (H_->nlev < cfg.amg_max_levels && H_->levels[H_->nlev - 1].rows > cfg.amg_min_coarse_rows) {
        const int l = H_->nlev - 1;
        {
            Level& L = H_->levels[l];
            dn_.ensure(L.rows, stream_);
            str_.ensure(L.nnz, stream_);
            profMark("setup:other");
            strengths(n_, L.rows, L.ro, L.ci, L.dg, L.v, dn_.p, str_.p, L.nnz, stream_);
            profMark("setup:strength");
            choice_.ensure(L.rows, stream_);
            cnt_.ensure(L.rows, stream_);
            lvl_.ensure(static_cast<size_t>(L.rows) + 1, stream_);
            if (aggMode_ == 0) {
                cudaMemsetAsync(err_.p, 0, sizeof(int), stream_);
                aggregate_syncfree(L.rows, L.ro, L.ci, L.dg, L.tpos, str_, choice_.p, err_.p, stream_);
                if (readErrCell()) throw std::runtime_error("aggregation: rows left undecided (broken pattern)");
                profMark("setup:aggregate L" + std::to_string(l));
            } else {
                act2_.ensure(static_cast<size_t>(L.rows) + 1, stream_);
                aggregate_kahn(L.rows, L.ro, L.ci, L.dg, L.tpos, str_, choice_.p,
                               kahnWork(cnt_, push_, lvl_, act2_.p), err_.p, stream_);
                profMark("setup:aggregate L" + std::to_string(l) + " rounds " + std::to_string(last_agg_rounds));
            }
            L.agg.ensure(L.rows, stream_);
            L.members.ensure(2 * static_cast<size_t>(L.rows), stream_);
            flag_.ensure(L.rows, stream_);
            scanTmp_.ensure(scan_tmp_ints(static_cast<size_t>(L.nnz) * 2 + L.rows) + 16, stream_);
            const int nC = aggregate_number(L.rows, choice_, flag_.p, L.agg.p, L.members.p, push_.p + 6,
                                            scanTmp_.p, stream_);
            profMark("setup:aggregate_number");
            if (nC == L.rows) break;  // no coarsening possible (amg.cpp:80)
            L.ncoarse = nC;
        }
        if (static_cast<int>(H_->levels.size()) < H_->nlev + 1) H_->levels.emplace_back();
        ++H_->nlev;
        Level& L = H_->levels[l];
        Level& C = H_->levels[l + 1];
        const int nC = L.ncoarse;
        // Galerkin (amg.cpp:39-71): segmented keys, per-segment rank sort, runs -> slots
        segOff_.ensure(static_cast<size_t>(nC) + 1, stream_);
        galerkin_seg_len(nC, L.ro, L.members, segOff_.p, stream_);
        cudaMemsetAsync(segOff_.p + nC, 0, sizeof(int), stream_);
        exclusive_scan(segOff_.p, nC + 1, push_.p + 6, scanTmp_.p, stream_);
        int total = 0;
        check(cudaMemcpyAsync(&total, push_.p + 6, sizeof(int), cudaMemcpyDeviceToHost, stream_), "seg total");
        sync();
        keys_.ensure(total, stream_);
        sorted_.ensure(total, stream_);
        profMark("galerkin:seglen+scan");
        galerkin_keys(nC, L.ro, L.ci, L.agg, L.members, segOff_, keys_.p, stream_);
        profMark("galerkin:keys");
        big_.ensure(static_cast<size_t>(nC) + 1, stream_);
        cudaMemsetAsync(err_.p, 0, sizeof(int), stream_);
        galerkin_sort(nC, segOff_, keys_, sorted_.p, big_.p, push_.p + 7, err_.p, stream_);
        if (readErrCell()) throw std::runtime_error("bcs: Galerkin coarse row exceeds the 12288-entry sort limit");
        profMark("galerkin:sort");
        C.o_ro.ensure(static_cast<size_t>(nC) + 1, stream_);
        galerkin_count(nC, segOff_, sorted_, C.o_ro.p, stream_);
        cudaMemsetAsync(C.o_ro.p + nC, 0, sizeof(int), stream_);
        exclusive_scan(C.o_ro.p, nC + 1, push_.p + 6, scanTmp_.p, stream_);
        int cnnz = 0;
        check(cudaMemcpyAsync(&cnnz, push_.p + 6, sizeof(int), cudaMemcpyDeviceToHost, stream_), "coarse nnz");
        sync();
        C.rows = nC;
        C.nnz = cnnz;
        profMark("galerkin:count+scan");
        C.o_ci.ensure(cnnz, stream_);
        C.o_v.ensure(static_cast<size_t>(cnnz) * nn, stream_);
        galerkin_fill(n_, nC, L.ro, L.members, segOff_, sorted_, L.v, C.o_ro, C.o_ci.p, C.o_v.p, stream_);
        C.ro = C.o_ro;
        C.ci = C.o_ci;
        C.v = C.o_v;
        profMark("galerkin:fill");
        setupLevelPattern(C);
        profMark("setup:pattern");
    }
    H_->levels[H_->nlev - 1].ncoarse = 0;

    // DILU smoother on all but the coarsest level (amg.cpp:86-88); the block-Jacobi
    // performance mode smooths the levels above the one-CTA tail with omega D^-1
    if (cfg.mode == BCS_MODE_PERF_JACOBI) {
        const int t = tailStart();
        std::vector<Level*> tail;
        for (int l = 0; l + 1 < H_->nlev; ++l) {
            if (l < t) jacobiSetup(H_->levels[l]);
            else tail.push_back(&H_->levels[l]);
        }
        if (!tail.empty()) diluSetupAll(tail, &cfg);
        profMark("perf:jacobi");
    } else {
        diluSetupAll(smoothedLevels(cfg), &cfg);
    }
    // dense factorisation of the coarsest level (amg.cpp:90-104)
    const Level& Cl = H_->levels[H_->nlev - 1];
    H_->m = Cl.rows * n_;
    H_->dense.ensure(static_cast<size_t>(H_->m) * H_->m, stream_);
    H_->dpiv.ensure(2 * static_cast<size_t>(H_->m), stream_);
    dense_build(n_, Cl.rows, Cl.ro, Cl.ci, Cl.v, H_->dense.p, stream_);
    cudaMemsetAsync(err_.p, 0, sizeof(int), stream_);
    if (H_->m >= denseBlockedMin_) dense_factor_blocked(H_->m, H_->dense.p, H_->dpiv.p, err_.p, stream_);
    else dense_factor(H_->m, H_->dense.p, H_->dpiv.p, err_.p, stream_);
    if (readErrCell()) throw std::runtime_error("singular coarse-level matrix");
    profMark("setup:dense");
    // V-cycle vectors
    for (int l = 0; l < H_->nlev; ++l) {
        Level& L = H_->levels[l];
        const size_t N = static_cast<size_t>(L.rows) * n_;
        if (l > 0) {
            L.r.ensure(N, stream_);
            L.z.ensure(N, stream_);
        }
        if (l + 1 < H_->nlev) {
            L.res.ensure(N, stream_);
            L.y.ensure(N, stream_);
            L.zb.ensure(N, stream_);
        }
    }
    setupTail();
}

// the first level of the one-CTA coarse tail (nlev - 1: none)
int Engine::tailStart() const {
    if (tailMaxRows_ <= 0 || H_->nlev < 2) return H_->nlev - 1;
    int t = H_->nlev - 1;
    while (t > 0 && H_->levels[t - 1].rows <= tailMaxRows_) --t;
    return t;
}

std::vector<Level*> Engine::smoothedLevels(const bcs_solver_config& cfg) {
    std::vector<Level*> lv;
    const int t = cfg.mode == BCS_MODE_PERF ? tailStart() : 0;
    for (int l = 0; l + 1 < H_->nlev; ++l) lv.push_back(l < t ? perfLevel(H_->levels[l], cfg) : &H_->levels[l]);
    for (int l = t; l + 1 < H_->nlev; ++l) H_->levels[l].mcValid = false;
    return lv;
}

Level* Engine::perfLevel(Level& L, const bcs_solver_config& cfg) {
    L.mcValid = false;
    if (cfg.mode != BCS_MODE_PERF) return &L;
    if (!buildColoured(L)) return &L;  // more than 64 colours: natural-order smoother on this level
    L.mcValid = true;
    return L.mc.get();
}

// the colour-permuted copy of L (k_color.cu): rows ordered by (colour, row),
// columns renumbered and sorted, blocks gathered; the smoother's DILU is then
// built on it by the natural-order machinery (a DAG #colours deep)
bool Engine::buildColoured(Level& L) {
    const size_t nn = static_cast<size_t>(n_) * n_;
    if (!L.mc) L.mc = std::make_unique<Level>();
    Level& M = *L.mc;
    const int R = L.rows;
    cnt_.ensure(static_cast<size_t>(R) + 2, stream_);
    lvl_.ensure(static_cast<size_t>(R) + 1, stream_);
    const int rounds = mc_color(R, L.ro, L.ci, cnt_.p, lvl_.p, ctr_.p, hTot_, stream_);
    if (rounds < 0) return false;
    L.mcPerm.ensure(R, stream_);
    act2_.ensure(static_cast<size_t>(R) + 1, stream_);  // inverse permutation
    const size_t scratch = static_cast<size_t>((R + 1023) / 1024) * 64 + 256;
    flag_.ensure(std::max<size_t>(scratch, R), stream_);
    L.ncolors = mc_permutation(R, cnt_.p, L.mcPerm.p, act2_.p, flag_.p, flag_.cap, hTot_, stream_);
    L.mcColorOff.assign(1, 0);  // hTot_[c] = rows of colour c (mc_permutation)
    for (int c = 0; c < L.ncolors; ++c) L.mcColorOff.push_back(L.mcColorOff.back() + hTot_[c]);
    L.mcColorOffD.ensure(L.mcColorOff.size(), stream_);
    check(cudaMemcpyAsync(L.mcColorOffD.p, L.mcColorOff.data(), sizeof(int) * L.mcColorOff.size(),
                          cudaMemcpyHostToDevice, stream_), "H2D colour offsets");
    // big levels: one streaming launch per colour (k_mc_colour); small ones
    // keep the sync-free sweeps (a DAG #colours deep) in one launch each way
    M.colourSweep = mcSweep_ || (mcLaunchMin_ > 0 && R >= static_cast<long long>(mcLaunchMin_) * L.ncolors);
    M.rows = R;
    M.nnz = L.nnz;
    M.o_ro.ensure(static_cast<size_t>(R) + 1, stream_);
    M.o_ci.ensure(L.nnz, stream_);
    mcSv_.ensure(L.nnz, stream_);
    scanTmp_.ensure(scan_tmp_ints(static_cast<size_t>(R) + 1) + 16, stream_);
    mc_permute_pattern(R, L.ro, L.ci, L.mcPerm.p, act2_.p, M.o_ro.p, M.o_ci.p, mcSv_.p, scanTmp_.p, push_.p + 10,
                       stream_);
    M.o_v.ensure(static_cast<size_t>(L.nnz) * nn, stream_);
    mc_permute_values(n_, static_cast<size_t>(L.nnz), mcSv_.p, L.v, M.o_v.p, stream_);
    M.ro = M.o_ro;
    M.ci = M.o_ci;
    M.v = M.o_v;
    setupLevelPattern(M);
    const size_t N = static_cast<size_t>(R) * n_;
    M.r.ensure(N, stream_);
    M.y.ensure(N, stream_);
    M.zb.ensure(N, stream_);
    profMark("perf:colour");
    return true;
}

// the one-CTA coarse tail: the first level from which every smoothed level
// has at most tailMaxRows_ rows (the coarsest is solved densely in between)
void Engine::setupTail() {
    H_->tail = -1;
    if (tailMaxRows_ <= 0 || H_->nlev < 2) return;
    const int t = tailStart();
    if (t >= H_->nlev - 1) return;  // no smoothed level small enough
    const int nl = H_->nlev - t;
    std::vector<TailLevelDev> d(nl);
    for (int q = 0; q < nl; ++q) {
        Level& L = H_->levels[t + q];
        TailLevelDev& x = d[q];
        x.rows = L.rows;
        x.ncoarse = L.ncoarse;
        x.ro = L.ro;
        x.ci = L.ci;
        x.dg = L.dg;
        x.order = L.order.p;
        x.agg = L.agg.p;
        x.members = L.members.p;
        x.v = L.v;
        x.lu = L.lu.p;
        x.rcp = L.rcp.p;
        x.perm = L.perm.p;
        x.r = L.r.p;
        x.z = L.z.p;
        x.res = L.res.p;
    }
    H_->tailDesc.ensure(sizeof(TailLevelDev) * nl, stream_);
    check(cudaMemcpyAsync(H_->tailDesc.p, d.data(), sizeof(TailLevelDev) * nl, cudaMemcpyHostToDevice, stream_),
          "H2D tail");
    sync();  // d dies here
    H_->tail = t;
}

FineMatrix Engine::serialFine() const {
    FineMatrix F;
    F.rows = nc_;
    F.nnz = nc_ + 2 * nf_;
    F.ro = ro_;
    F.ci = ci_;
    F.dg = dg_;
    F.tpos = tpos_;
    F.v = vals_;
    return F;
}

// makeCsrPreconditioner (engine.cpp:21-29)
void Engine::buildPrecond(const bcs_solver_config& cfg) {
    requireMatrix();
    buildPrecondOn(serialFine(), cfg);
}

void Engine::buildPrecondOn(const FineMatrix& F, const bcs_solver_config& cfg) {
    H_->pcKind = -1;
    for (auto& L : H_->levels) L.mcValid = L.jacobi = false;

    if (H_->levels.empty()) H_->levels.emplace_back();
    H_->nlev = 1;
    Level& L0 = H_->levels[0];
    L0.rows = F.rows;
    L0.nnz = F.nnz;
    L0.ro = F.ro;
    L0.ci = F.ci;
    L0.dg = F.dg;
    L0.tpos = F.tpos;
    L0.v = F.v;
    const size_t N = static_cast<size_t>(F.rows) * n_;
    switch (cfg.precond) {
        case BCS_PRECOND_NONE: break;
        case BCS_PRECOND_LUSGS:
            lusgsSetup(L0);
            L0.y.ensure(N, stream_);
            break;
        case BCS_PRECOND_DILU:
            diluSetupAll({perfLevel(L0, cfg)}, &cfg);
            L0.y.ensure(N, stream_);
            break;
        case BCS_PRECOND_AMG: buildHierarchy(cfg); break;
        default: throw std::invalid_argument("unknown preconditioner kind");
    }
    checkErr("buildPrecond");
    H_->pcKind = cfg.precond;
    H_->pcCfg = cfg;
}

// DILU/LUSGS sweep pair: z = (D+U)^{-1} D (D+L)^{-1} r  (accumulate: see sweep_backward)
void Engine::smootherApply(Level& L, const double* r, double* z, int accumulate) {
    if (L.jacobi && H_->pcCfg.mode == BCS_MODE_PERF_JACOBI) {
        const double nb = static_cast<double>(n_), R = static_cast<double>(L.rows);
        const double per = R * (8.0 * nb * nb + 8.0 * nb + 4.0 * nb + 16.0 * nb) + (accumulate == 2 ? R * 8.0 * nb : 0.0);
        if (kernelTiming_) timerBegin();
        block_jacobi(n_, L.rows, L.lu, L.rcp, L.perm, r, z, accumulate, jacobiOmega_, stream_);
        if (kernelTiming_) timerEnd(1, per);
        return;
    }
    if (L.mcValid && H_->pcCfg.mode == BCS_MODE_PERF) {
        // performance mode: the multicolour DILU on the colour-permuted copy;
        // r in, result scattered back (and accumulated) in the level's numbering
        Level& M = *L.mc;
        // one launch per colour: the gather of r and the scatter of z are fused
        // into the first-colour forward and the backward colour kernels
        static const bool fuseOn = [] {
            const char* e = std::getenv("BCS_MC_FUSE");
            return !e || std::atoi(e) != 0;
        }();
        const bool fused = M.colourSweep && !mcSweep_ && fuseOn;
        if (!fused) mc_vec_gather(n_, L.rows, L.mcPerm, r, M.r.p, stream_);
        if (M.colourSweep) {
            // colour-synchronous sweeps: the forward reads the lower triangle,
            // the backward the upper one, each with the row's LU, input, output
            const double nb = static_cast<double>(n_), R = static_cast<double>(M.rows);
            const double per = 0.5 * (static_cast<double>(M.nnz) - R) * (8.0 * nb * nb + 4.0) +
                               R * (8.0 * nb * nb + 8.0 * nb + 4.0 * nb + 12.0) + 2.0 * R * 8.0 * nb;
            if (mcSweep_) {  // opt-in: one cooperative kernel, a grid barrier per colour
                if (kernelTiming_) timerBegin();
                mc_sweep(n_, true, M.rows, L.ncolors, L.mcColorOffD, M.ro, M.dg, M.ci, M.v, M.lu, M.rcp, M.perm, M.r,
                         M.y.p, stream_);
                if (kernelTiming_) timerEnd(1, per);
                if (kernelTiming_) timerBegin();
                mc_sweep(n_, false, M.rows, L.ncolors, L.mcColorOffD, M.ro, M.dg, M.ci, M.v, M.lu, M.rcp, M.perm, M.y,
                         M.zb.p, stream_);
                if (kernelTiming_) timerEnd(1, per);
            } else {  // one streaming launch per colour
                const auto& co = L.mcColorOff;
                if (kernelTiming_) timerBegin();
                for (int c = 0; c < L.ncolors; ++c)
                    mc_colour_sweep(n_, true, co[c], co[c + 1], M.ro, M.dg, M.ci, M.v, M.lu, M.rcp, M.perm,
                                    fused ? r : M.r.p, M.y.p, fused ? L.mcPerm.p : nullptr, nullptr, 0, stream_);
                if (kernelTiming_) timerEnd(1, per);
                if (kernelTiming_) timerBegin();
                for (int c = L.ncolors - 1; c >= 0; --c)
                    mc_colour_sweep(n_, false, co[c], co[c + 1], M.ro, M.dg, M.ci, M.v, M.lu, M.rcp, M.perm, M.y,
                                    M.zb.p, fused ? L.mcPerm.p : nullptr, fused ? z : nullptr, accumulate, stream_);
                if (kernelTiming_) timerEnd(1, per);
            }
        } else {
            smootherApply(M, M.r, M.zb.p, 0);
        }
        if (!fused) mc_vec_scatter(n_, L.rows, L.mcPerm, M.zb, z, accumulate, stream_);
        return;
    }
    const size_t N = static_cast<size_t>(L.rows) * n_;
    double* zb = accumulate ? L.zb.p : z;
    cudaMemsetAsync(L.y.p, 0xFF, N * sizeof(double), stream_);
    cudaMemsetAsync(zb, 0xFF, N * sizeof(double), stream_);
    // algorithmic bytes of one sweep: the dependency blocks
    // + column ids of its triangle, the row's LU/reciprocals/permutation and
    // record, the input vector read and the output written (+ z update)
    const double nb = static_cast<double>(n_), R = static_cast<double>(L.rows);
    const double tri = 0.5 * (static_cast<double>(L.nnz) - R) * (8.0 * nb * nb + 4.0);
    const double per = tri + R * (8.0 * nb * nb + 8.0 * nb + 4.0 * nb + 16.0) + 2.0 * R * 8.0 * nb;
    const bool timed = kernelTiming_;
    if (timed) timerBegin();
    sweep_forward(n_, L.rows, L.sweepDepth(), L.offf, L.pkf, L.recf, L.woff, L.ci, L.v, r, L.y.p, err_.p + 1, stream_);
    if (timed) timerEnd(1, per);
    if (timed) timerBegin();
    sweep_backward(n_, L.rows, L.sweepDepth(), L.offb, L.pkb, L.recb, L.woffb, L.ci, L.v, L.y, zb, z, accumulate, err_.p + 1, stream_);
    if (timed) timerEnd(1, per + (accumulate == 2 ? 2.0 : accumulate == 1 ? 1.0 : 0.0) * R * 8.0 * nb);
}

// coarsest level: denseSolve (smallmat.hpp:163-174) in the reference's order;
// from m >= denseTiledMin_ (scrambled inputs' stalled aggregation) the
// backward substitution runs tiled (tolerance-level) unless the
// EXACT mode asks for the reference's order throughout
void Engine::denseSolve(const double* r, double* z) {
    const int m = H_->m;
    if (m >= denseTiledMin_ && !exactDots_) dense_solve_tiled(m, H_->dense, H_->dpiv, r, z, stream_);
    else if (m >= denseBlockedMin_) dense_solve_big(m, H_->dense, H_->dpiv, r, z, stream_);
    else dense_solve(m, H_->dense, H_->dpiv, r, z, stream_);
}

// AmgHierarchy::vcycle (amg.cpp:111-158)
void Engine::vcycle(int l, const double* r, double* z) {
    Level& L = H_->levels[l];
    const size_t N = static_cast<size_t>(L.rows) * n_;
    if (l == H_->tail) {  // the whole coarse tail: one CTA down, dense coarsest, one CTA up
        const int nl = H_->nlev - l;
        const auto* td = reinterpret_cast<const TailLevelDev*>(H_->tailDesc.p);
        const int pre = H_->pcCfg.amg_pre_sweeps, post = H_->pcCfg.amg_post_sweeps;
        vcycle_tail(n_, nl, td, L.rows, r, z, pre, post, 0, err_.p + 1, stream_);
        const Level& Cl = H_->levels[H_->nlev - 1];
        denseSolve(Cl.r, Cl.z.p);
        vcycle_tail(n_, nl, td, L.rows, r, z, pre, post, 1, err_.p + 1, stream_);
        profMark("vcycle:tail L" + std::to_string(l) + "+");
        return;
    }
    if (l == H_->nlev - 1) {
        denseSolve(r, z);
        profMark("vcycle:dense_solve");
        return;
    }
    const int pre = H_->pcCfg.amg_pre_sweeps, post = H_->pcCfg.amg_post_sweeps;
    for (int s = 0; s < pre; ++s) {
        const double* rin = r;  // z == 0 on the first sweep: r - A*0 == r exactly
        if (s > 0) {
            spmvLevel(L, z, r, L.res.p);
            rin = L.res;
        }
        smootherApply(L, rin, z, s == 0 ? 1 : 2);
        profMark("vcycle:presmooth L" + std::to_string(l));
    }
    const double* res = r;
    if (pre > 0) {
        spmvLevel(L, z, r, L.res.p);
        res = L.res;
    } else {
        cudaMemsetAsync(z, 0, N * sizeof(double), stream_);
    }
    Level& C = H_->levels[l + 1];
    restrict_vec(n_, L.ncoarse, L.members, res, C.r.p, stream_);
    profMark("vcycle:residual+restrict");
    vcycle(l + 1, C.r, C.z.p);
    prolong_vec(n_, L.rows, L.agg, C.z, z, stream_);
    profMark("vcycle:prolong");
    for (int s = 0; s < post; ++s) {
        spmvLevel(L, z, r, L.res.p);
        profMark("vcycle:post-spmv");
        smootherApply(L, L.res, z, 2);
        profMark("vcycle:postsmooth L" + std::to_string(l));
    }
}

void Engine::applyPrecond(const double* r, double* z) {
    const size_t N = static_cast<size_t>(H_->levels[0].rows) * n_;
    switch (H_->pcKind) {
        case BCS_PRECOND_NONE: copy_vec(r, z, N, stream_); break;
        case BCS_PRECOND_LUSGS:
        case BCS_PRECOND_DILU: smootherApply(H_->levels[0], r, z, 0); break;
        case BCS_PRECOND_AMG: vcycle(0, r, z); break;
        default: throw std::logic_error("preconditioner not built");
    }
}

// ------------------------------------------------------------------ Krylov
double Engine::dotHost(const double* a, const double* b, size_t N, bool sqrt_out) {
    (void)N;
    opDot(a, b, scal_.p + 2, sqrt_out);
    check(cudaMemcpyAsync(hStatus_ + 2, scal_.p + 2, sizeof(double), cudaMemcpyDeviceToHost, stream_), "D2H scalar");
    sync();
    return hStatus_[2];
}

// gmresSolve (krylov.cpp:59-150)
void Engine::gmres(const double* b, double* x, const bcs_solver_config& cfg, bcs_report& rep) {
    const size_t N = static_cast<size_t>(nc_) * n_;
    const int m = cfg.gmres_restart;
    rk_.ensure(N, stream_);
    w_.ensure(N, stream_);
    zk_.ensure(N, stream_);
    opResidual(x, b, rk_.p);
    double beta = dotHost(rk_, rk_, N, true);
    rep.initial_residual = beta;
    const double beta0 = beta;
    const double tol = std::max(cfg.rel_tol * beta, cfg.abs_tol);
    if (beta <= tol) {
        rep.final_residual = beta;
        rep.converged = 1;
        return;
    }
    V_.ensure(static_cast<size_t>(m + 1) * N, stream_);
    const bool flexible = cfg.method == BCS_FGMRES;
    if (flexible) Z_.ensure(static_cast<size_t>(m) * N, stream_);
    Hm_.ensure(static_cast<size_t>(m + 1) * m, stream_);
    cs_.ensure(m, stream_);
    sn_.ensure(m, stream_);
    g_.ensure(static_cast<size_t>(m) + 1, stream_);
    y_.ensure(m, stream_);
    double* beta_d = scal_.p + 2;  // holds ||r|| from dotHost
    int total = 0;
    while (total < cfg.max_iters) {
        scale_by(rk_, beta_d, -1.0, V_.p, N, stream_);
        cudaMemsetAsync(g_.p, 0, sizeof(double) * (m + 1), stream_);
        cudaMemsetAsync(Hm_.p, 0, sizeof(double) * (m + 1) * m, stream_);
        cudaMemcpyAsync(g_.p, beta_d, sizeof(double), cudaMemcpyDeviceToDevice, stream_);
        int j = 0;
        bool happy = false;
        for (; j < m && total < cfg.max_iters; ++j, ++total) {
            double* vj = V_.p + static_cast<size_t>(j) * N;
            double* zj = flexible ? Z_.p + static_cast<size_t>(j) * N : zk_.p;
            opPrecond(vj, zj);
            opSpmv(zj, w_.p);
            opDot(w_, V_.p, Hm_.p + j, false);
            for (int i = 0; i < j; ++i)
                opAxpyDot(w_.p, Hm_.p + static_cast<size_t>(i) * m + j, V_.p + static_cast<size_t>(i) * N,
                          V_.p + static_cast<size_t>(i + 1) * N, Hm_.p + static_cast<size_t>(i + 1) * m + j);
            opAxpyDot(w_.p, Hm_.p + static_cast<size_t>(j) * m + j, vj, nullptr,
                      Hm_.p + static_cast<size_t>(j + 1) * m + j);
            scale_by(w_, Hm_.p + static_cast<size_t>(j + 1) * m + j, 1e-290, V_.p + static_cast<size_t>(j + 1) * N, N,
                     stream_);
            givens_step(Hm_.p, m, j, cs_.p, sn_.p, g_.p, scal_.p + 4, stream_);
            check(cudaMemcpyAsync(hStatus_ + 4, scal_.p + 4, 2 * sizeof(double), cudaMemcpyDeviceToHost, stream_),
                  "D2H status");
            sync();
            const double gabs = hStatus_[4];
            happy = hStatus_[5] != 0.0;
            hist_.push_back(gabs / beta0);
            if (gabs <= tol || happy) {
                ++j;
                ++total;
                break;
            }
        }
        // back substitution, x += M^{-1}(V y)   (FGMRES: x += Z y)
        back_subst(Hm_, m, j, g_, y_.p, stream_);
        if (flexible) {
            lincomb(Z_, N, y_, j, w_.p, N, stream_);
            add_to(x, w_, N, stream_);
        } else {
            lincomb(V_, N, y_, j, w_.p, N, stream_);
            opPrecond(w_, zk_.p);
            add_to(x, zk_, N, stream_);
        }
        opResidual(x, b, rk_.p);
        beta = dotHost(rk_, rk_, N, true);
        if (!hist_.empty()) hist_.back() = beta / beta0;
        rep.iterations = total;
        rep.final_residual = beta;
        if (beta <= tol) {
            rep.converged = 1;
            return;
        }
        if (happy && beta <= tol * 1.0000001) {
            rep.converged = 1;
            return;
        }
    }
    rep.iterations = total;
    rep.converged = rep.final_residual <= tol;
}

// bicgstabSolve (krylov.cpp:152-214)
void Engine::bicgstab(const double* b, double* x, const bcs_solver_config& cfg, bcs_report& rep) {
    const size_t N = static_cast<size_t>(nc_) * n_;
    rk_.ensure(N, stream_);
    brh_.ensure(N, stream_);
    bp_.ensure(N, stream_);
    bv_.ensure(N, stream_);
    bs_.ensure(N, stream_);
    bt_.ensure(N, stream_);
    bph_.ensure(N, stream_);
    bsh_.ensure(N, stream_);
    opResidual(x, b, rk_.p);
    const double beta0 = dotHost(rk_, rk_, N, true);
    rep.initial_residual = beta0;
    const double tol = std::max(cfg.rel_tol * beta0, cfg.abs_tol);
    if (beta0 <= tol) {
        rep.final_residual = beta0;
        rep.converged = 1;
        return;
    }
    copy_vec(rk_, brh_.p, N, stream_);
    double rhoPrev = 1.0, alpha = 1.0, omega = 1.0;
    for (int it = 0; it < cfg.max_iters; ++it) {
        const double rho = dotHost(brh_, rk_, N, false);
        if (std::fabs(rho) < 1e-30) {
            rep.breakdown = 1;
            break;
        }
        if (it == 0) copy_vec(rk_, bp_.p, N, stream_);
        else bicg_p(bp_.p, rk_, bv_, (rho / rhoPrev) * (alpha / omega), omega, N, stream_);
        opPrecond(bp_, bph_.p);
        opSpmv(bph_, bv_.p);
        const double rhatv = dotHost(brh_, bv_, N, false);
        if (std::fabs(rhatv) < 1e-300) {
            rep.breakdown = 1;
            break;
        }
        alpha = rho / rhatv;
        bicg_s(bs_.p, rk_, bv_, alpha, N, stream_);
        const double ns = dotHost(bs_, bs_, N, true);
        if (ns <= tol) {
            bicg_x_half(x, bph_, alpha, N, stream_);
            rep.iterations = it + 1;
            hist_.push_back(ns / beta0);
            break;
        }
        opPrecond(bs_, bsh_.p);
        opSpmv(bsh_, bt_.p);
        const double tt = dotHost(bt_, bt_, N, false);
        omega = tt > 0.0 ? dotHost(bt_, bs_, N, false) / tt : 0.0;
        bicg_x_r(x, rk_.p, bph_, bsh_, bs_, bt_, alpha, omega, N, stream_);
        rep.iterations = it + 1;
        if (std::fabs(omega) < 1e-30) {
            rep.breakdown = 1;
            break;
        }
        rhoPrev = rho;
        const double nr = dotHost(rk_, rk_, N, true);
        hist_.push_back(nr / beta0);
        if (nr <= tol) break;
    }
    opResidual(x, b, rk_.p);
    rep.final_residual = dotHost(rk_, rk_, N, true);
    rep.converged = rep.final_residual <= tol;
    if (rep.converged) rep.breakdown = 0;
    if (rep.breakdown)
        throw std::runtime_error("BiCGStab breakdown at iteration " + std::to_string(rep.iterations) + ", residual " +
                                 std::to_string(rep.final_residual));
}

void Engine::solveDevice(const double* d_b, double* d_x, const bcs_solver_config& cfg, bcs_report& rep) {
    LaunchScope ls(&launches_);
    requireMatrix();
    validateConfig(cfg);
    distActive_ = false;
    H_ = &main_;
    nseg_ = 1;
    const long long segh[2] = {0, static_cast<long long>(nc_) * n_};
    check(cudaMemcpyAsync(seg_.p, segh, sizeof segh, cudaMemcpyHostToDevice, stream_), "seg");
    const long long l0 = launches_.launches;
    spmvMs_ = 0.0;
    spmvCount_ = 0;
    sweepMs_ = 0.0;
    sweepBytes_ = 0.0;
    sweepCount_ = 0;
    evUsed_ = 0;
    hist_.clear();
    cudaMemsetAsync(err_.p + 1, 0, sizeof(int), stream_);
    const auto t0 = clk::now();
    profT_ = t0;
    buildPrecond(cfg);
    sync();
    const auto t1 = clk::now();
    solveKrylov(d_b, d_x, cfg, rep);
    const auto t2 = clk::now();
    rep.t_amg_setup = secs(t0, t1);
    rep.t_krylov = secs(t1, t2);
    rep.amg_levels = H_->pcKind == BCS_PRECOND_AMG ? H_->nlev : 0;
    rep.coarse_rows = H_->pcKind == BCS_PRECOND_AMG ? H_->levels[H_->nlev - 1].rows : 0;
    rep.spmv_launches = spmvCount_;
    rep.spmv_ms = spmvMs_;
    rep.sweep_launches = sweepCount_;
    rep.sweep_ms = sweepMs_;
    rep.sweep_bytes = sweepBytes_;
    rep.kernel_launches = static_cast<int>(launches_.launches - l0);
    lastSolveLaunches_ = rep.kernel_launches;
}

void Engine::solveKrylov(const double* d_b, double* d_x, const bcs_solver_config& cfg, bcs_report& rep) {
    exactDots_ = cfg.mode == BCS_MODE_EXACT;
    struct Reset {
        bool& f;
        ~Reset() { f = false; }
    } reset{exactDots_};
    if (cfg.method == BCS_GMRES || cfg.method == BCS_FGMRES) gmres(d_b, d_x, cfg, rep);
    else bicgstab(d_b, d_x, cfg, rep);
    sync();
    collectSpmvTimes();
    profDump();
    int spinErr = 0;
    check(cudaMemcpy(&spinErr, err_.p + 1, sizeof(int), cudaMemcpyDeviceToHost), "spin flag");
    if (spinErr) throw std::runtime_error("bcs: sweep dependency wait timed out (corrupt schedule)");
    checkErr("solve");
}

// ------------------------------------------------------- Krylov operators
void Engine::opResidual(const double* x, const double* b, double* r) {
    if (hostLdu_) {
        spmv(n_, nc_, hlMvRo_, hlMvCi_, hlMvV_, x, b, r, stream_);
        return;
    }
    if (!distActive_) {
        spmvLevel(H_->levels[0], x, b, r);
        return;
    }
    opSpmv(x, distTmp_.p);
    sub_vec(b, distTmp_, r, static_cast<size_t>(mpActive_ ? mpRows_ : nc_) * n_, stream_);  // nc_: the global rows of this Mode R call
}

// halo exchange of the multi-process Mode R: pack the rows peers need, one
// grouped NCCL send/recv per peer (peers ascending), values land in mpRecv_
// The exchange runs on its own stream: pack (engine stream) -> event ->
// grouped send/recv (comm stream) -> event; the caller's local product runs
// meanwhile and waits for the event only before the halo couplings, which the
// reference adds after the local product anyway (partition.cpp:335-350).
void Engine::mpExchange(const double* x) {
    const auto& A = nccl::api();
    nccl::g_rank = mpRank_;
    pack_rows(n_, mpSendRows_, mpSendIdx_, x, mpSend_.p, stream_);
    check(cudaEventRecord(mpEvPack_, stream_), "record pack");
    check(cudaStreamWaitEvent(commStream_, mpEvPack_, 0), "wait pack");
    nccl::ck(A.groupStart(), "group start");
    size_t so = 0, ro = 0;
    for (int q = 0; q < mpSize_; ++q) {
        if (mpSendCnt_[q])
            nccl::ck(A.send(mpSend_.p + so * n_, static_cast<size_t>(mpSendCnt_[q]) * n_, ncclDouble, q,
                            static_cast<ncclComm_t>(comm_), commStream_), "send", q);
        if (mpRecvCnt_[q])
            nccl::ck(A.recv(mpRecv_.p + ro * n_, static_cast<size_t>(mpRecvCnt_[q]) * n_, ncclDouble, q,
                            static_cast<ncclComm_t>(comm_), commStream_), "recv", q);
        so += mpSendCnt_[q];
        ro += mpRecvCnt_[q];
    }
    nccl::ck(A.groupEnd(), "group end");
    check(cudaEventRecord(mpEvComm_, commStream_), "record comm");
}

// partitionedMatvec (partition.cpp:298-352): every engine's local product on
// its row slice, then its halo couplings (the exchange is implicit: all engine
// slices live in one device vector on this GPU)
void Engine::opSpmv(const double* x, double* y) {
    if (hostLdu_) {
        spmv(n_, nc_, hlMvRo_, hlMvCi_, hlMvV_, x, nullptr, y, stream_);
        return;
    }
    if (!distActive_) {
        spmvLevel(H_->levels[0], x, nullptr, y);
        return;
    }
    if (mpActive_) {  // this process's engine; halo columns index the receive buffer
        DistPart& P = dist_[0];
        mpExchange(x);
        spmv(n_, P.rows, P.ro, P.ci, P.vals, x, nullptr, y, stream_);  // overlaps the exchange
        check(cudaStreamWaitEvent(stream_, mpEvComm_, 0), "wait comm");
        halo_spmv(n_, P.nhr, P.hrow, P.hoff, P.hcol, P.hvals, mpRecv_, y, 0, stream_);
        return;
    }
    for (auto& P : dist_) {
        const size_t off = static_cast<size_t>(P.rowStart) * n_;
        spmv(n_, P.rows, P.ro, P.ci, P.vals, x + off, nullptr, y + off, stream_);
        halo_spmv(n_, P.nhr, P.hrow, P.hoff, P.hcol, P.hvals, x, y, P.rowStart, stream_);
    }
}

// per-engine local preconditioners (partition.cpp:427-431), block Jacobi across engines
void Engine::opPrecond(const double* r, double* z) {
    if (!distActive_) {
        applyPrecond(r, z);
        return;
    }
    for (auto& P : dist_) {
        H_ = &P.H;
        const size_t off = static_cast<size_t>(P.rowStart) * n_;
        applyPrecond(r + off, z + off);
    }
    H_ = &main_;
}

// multi-process: this engine's partial with the block layout the one-device
// Mode R uses for an engine segment, all-gathered, folded in engine order
void Engine::opDot(const double* a, const double* b, double* out, bool sqrt_out) {
    if (exactDots_) {  // BCS_MODE_EXACT: the reference's sequential order (krylov.cpp:38-42)
        if (mpActive_) {
            dot_seq(a, b, seg_, 1, mpPart_.p, false, partials_.p, stream_);
            nccl::ck(nccl::api().allGather(mpPart_.p, mpGath_.p, 1, ncclDouble, static_cast<ncclComm_t>(comm_), stream_),
                     "allgather");
            fold_engines(mpGath_, mpSize_, out, sqrt_out, stream_);
            return;
        }
        dot_seq(a, b, seg_, nseg_, out, sqrt_out, partials_.p, stream_);
        return;
    }
    if (mpActive_) {
        dot(a, b, seg_, 1, mpPart_.p, false, partials_.p, ticket_.p, stream_, mpBps_);
        nccl::ck(nccl::api().allGather(mpPart_.p, mpGath_.p, 1, ncclDouble, static_cast<ncclComm_t>(comm_), stream_),
                 "allgather");
        fold_engines(mpGath_, mpSize_, out, sqrt_out, stream_);
        return;
    }
    dot(a, b, seg_, nseg_, out, sqrt_out, partials_.p, ticket_.p, stream_);
}

void Engine::opAxpyDot(double* w, const double* h, const double* v, const double* nextv, double* out) {
    if (exactDots_) {
        const size_t N = static_cast<size_t>(nc_) * n_;
        if (mpActive_) {
            axpy_dot_seq(w, h, v, nextv, N, seg_, 1, mpPart_.p, partials_.p, false, stream_);  // sqrt after the fold
            nccl::ck(nccl::api().allGather(mpPart_.p, mpGath_.p, 1, ncclDouble, static_cast<ncclComm_t>(comm_), stream_),
                     "allgather");
            fold_engines(mpGath_, mpSize_, out, nextv == nullptr, stream_);
            return;
        }
        axpy_dot_seq(w, h, v, nextv, N, seg_, nseg_, out, partials_.p, nextv == nullptr, stream_);
        return;
    }
    if (mpActive_) {
        axpy_dot(w, h, v, nextv, seg_, 1, mpPart_.p, partials_.p, ticket_.p, stream_, mpBps_, 0);
        nccl::ck(nccl::api().allGather(mpPart_.p, mpGath_.p, 1, ncclDouble, static_cast<ncclComm_t>(comm_), stream_),
                 "allgather");
        fold_engines(mpGath_, mpSize_, out, nextv == nullptr, stream_);
        return;
    }
    axpy_dot(w, h, v, nextv, seg_, nseg_, out, partials_.p, ticket_.p, stream_);
}

// ------------------------------------------------------------------ Mode R
// one engine's local BSR, LDU source ids, diagonal/transpose positions and
// halo CSR (halo columns: global rows, or hcolOverride = receive-buffer rows)
void Engine::uploadEnginePart(DistPart& P, const Partition& p, int n, const std::vector<int>* hcolOverride) {
    P.rowStart = 0;
    P.rows = p.nLocalRows();
    P.nnz = static_cast<int>(p.ci.size());
    P.nh = static_cast<int>(p.haloRow.size());
    P.ro.ensure(p.ro.size(), stream_);
    P.ci.ensure(p.ci.size(), stream_);
    P.src.ensure(p.src.size(), stream_);
    P.dg.ensure(P.rows, stream_);
    P.tpos.ensure(p.ci.size(), stream_);
    P.vals.ensure(static_cast<size_t>(P.nnz) * n * n, stream_);
    check(cudaMemcpyAsync(P.ro.p, p.ro.data(), sizeof(int) * p.ro.size(), cudaMemcpyHostToDevice, stream_), "H2D");
    check(cudaMemcpyAsync(P.ci.p, p.ci.data(), sizeof(int) * p.ci.size(), cudaMemcpyHostToDevice, stream_), "H2D");
    check(cudaMemcpyAsync(P.src.p, p.src.data(), sizeof(int) * p.src.size(), cudaMemcpyHostToDevice, stream_), "H2D");
    find_diag(P.rows, P.ro, P.ci, P.dg.p, stream_);
    cudaMemsetAsync(err_.p, 0, sizeof(int), stream_);
    transpose_pos(P.rows, P.ro, P.ci, P.tpos.p, err_.p, stream_);
    if (readErrCell()) throw std::runtime_error("bcs: structurally asymmetric engine pattern");
    // halo rows: distinct local rows of the (row, col)-sorted entries
    std::vector<int> hrow, hoff;
    for (int h = 0; h < P.nh; ++h)
        if (h == 0 || p.haloRow[h] != p.haloRow[h - 1]) {
            hrow.push_back(p.haloRow[h]);
            hoff.push_back(h);
        }
    hoff.push_back(P.nh);
    P.nhr = static_cast<int>(hrow.size());
    P.hrow.ensure(hrow.size(), stream_);
    P.hoff.ensure(hoff.size(), stream_);
    P.hcol.ensure(P.nh, stream_);
    P.hsrc.ensure(P.nh, stream_);
    P.hvals.ensure(static_cast<size_t>(P.nh) * n * n, stream_);
    const std::vector<int>& hc = hcolOverride ? *hcolOverride : p.haloCol;
    if (P.nh) {
        check(cudaMemcpyAsync(P.hrow.p, hrow.data(), sizeof(int) * hrow.size(), cudaMemcpyHostToDevice, stream_), "H2D");
        check(cudaMemcpyAsync(P.hoff.p, hoff.data(), sizeof(int) * hoff.size(), cudaMemcpyHostToDevice, stream_), "H2D");
        check(cudaMemcpyAsync(P.hcol.p, hc.data(), sizeof(int) * P.nh, cudaMemcpyHostToDevice, stream_), "H2D");
        check(cudaMemcpyAsync(P.hsrc.p, p.haloSrc.data(), sizeof(int) * P.nh, cudaMemcpyHostToDevice, stream_), "H2D");
    }
    sync();  // host vectors die with the caller's iteration
}

void Engine::distSetupTopology(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh,
                               const double* centroids, int nRanks, int nEngines) {
    if (nEngines > 64) throw std::invalid_argument("bcs: at most 64 engines per device");
    const Decomposition dec = decompose(nc, centroids, nRanks);
    const std::vector<Partition> parts = buildPartitioned(nc, nf, owner, neigh, dec);
    const ConsolidationPlan plan = makeConsolidationPlan(dec, nEngines);
    const std::vector<Partition> eng = consolidate(parts, plan, dec);
    dist_.resize(eng.size());
    std::vector<long long> segh(eng.size() + 1, 0);
    for (size_t e = 0; e < eng.size(); ++e) {
        const Partition& p = eng[e];
        uploadEnginePart(dist_[e], p, n, nullptr);
        dist_[e].rowStart = p.rowStart;
        segh[e + 1] = static_cast<long long>(p.rowEnd) * n;
        segh[e] = static_cast<long long>(p.rowStart) * n;
    }
    distSegh_ = segh;
    distNewToOld_ = dec.newToOld;
    distOwner_.assign(owner, owner + nf);
    distNeigh_.assign(neigh, neigh + nf);
    distCen_.assign(centroids, centroids + 3 * static_cast<size_t>(nc));
    distRanks_ = nRanks;
    distEngines_ = nEngines;
    distNc_ = nc;
    distNf_ = nf;
    distN_ = n;
    sync();
}

// Mode R on this device over dist_'s engines (partition.cpp:411-471): the
// engines' dot segments, one local preconditioner per engine, global Krylov
// on kb_/kx_ (new numbering); returns the time the preconditioners were ready
std::chrono::steady_clock::time_point Engine::distSolveCore(const bcs_solver_config& cfg, bcs_report& rep) {
    // dot-product segments of the engines (a serial call in between rewrites seg_)
    nseg_ = static_cast<int>(dist_.size());
    seg_.ensure(distSegh_.size(), stream_);
    check(cudaMemcpyAsync(seg_.p, distSegh_.data(), sizeof(long long) * distSegh_.size(), cudaMemcpyHostToDevice,
                          stream_), "H2D seg");
    // per-engine preconditioners (partition.cpp:411-412)
    hist_.clear();
    spmvMs_ = 0.0;
    spmvCount_ = 0;
    sweepMs_ = 0.0;
    sweepBytes_ = 0.0;
    sweepCount_ = 0;
    evUsed_ = 0;
    cudaMemsetAsync(err_.p + 1, 0, sizeof(int), stream_);
    for (auto& P : dist_) {
        H_ = &P.H;
        FineMatrix F;
        F.rows = P.rows;
        F.nnz = P.nnz;
        F.ro = P.ro;
        F.ci = P.ci;
        F.dg = P.dg;
        F.tpos = P.tpos;
        F.v = P.vals;
        buildPrecondOn(F, cfg);
    }
    H_ = &main_;
    sync();
    const auto t2 = clk::now();
    distActive_ = true;
    solveKrylov(kb_, kx_.p, cfg, rep);
    distActive_ = false;
    return t2;
}

void Engine::distSolve(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh, const double* centroids,
                       const double* diag, const double* upper, const double* lower, const double* b,
                       const double* x0, double* x, int nRanks, int nEngines, const bcs_solver_config& cfg,
                       bcs_report& rep) {
    LaunchScope ls(&launches_);
    if (n < 1 || n > 5) throw std::invalid_argument("bcs: block size must be 1..5 on the device");
    if (nEngines < 1 || nEngines > nRanks) throw std::invalid_argument("makeConsolidationPlan: need 1 <= nEngines <= nRanks");
    validateConfig(cfg);
    const auto t0 = clk::now();
    const bool same = distNc_ == nc && distNf_ == nf && distN_ == n && distRanks_ == nRanks && distEngines_ == nEngines &&
                      std::equal(owner, owner + nf, distOwner_.begin()) && std::equal(neigh, neigh + nf, distNeigh_.begin()) &&
                      std::equal(centroids, centroids + 3 * static_cast<size_t>(nc), distCen_.begin());
    // the serial system's sizes (n_, nc_) are borrowed for the Krylov operators of
    // this call and restored on every exit, with H_ and the operator switches
    SerialStateGuard guard(*this);
    if (!same) distSetupTopology(nc, nf, n, owner, neigh, centroids, nRanks, nEngines);
    n_ = n;
    // upload: LDU values -> engine slots and halo blocks (replace semantics)
    const size_t nn = static_cast<size_t>(n) * n;
    ldu_diag_.ensure(nc * nn, stream_);
    ldu_upper_.ensure(nf * nn, stream_);
    ldu_lower_.ensure(nf * nn, stream_);
    h2d(ldu_diag_.p, diag, sizeof(double) * nc * nn, "H2D");
    if (nf) {
        h2d(ldu_upper_.p, upper, sizeof(double) * nf * nn, "H2D");
        h2d(ldu_lower_.p, lower, sizeof(double) * nf * nn, "H2D");
    }
    for (auto& P : dist_) {
        gather_values(n, P.nnz, nc, nf, P.src, ldu_diag_, ldu_upper_, ldu_lower_, P.vals.p, stream_);
        if (P.nh) gather_values(n, P.nh, nc, nf, P.hsrc, ldu_diag_, ldu_upper_, ldu_lower_, P.hvals.p, stream_);
    }
    // scatterVector: rank-major renumbering (partition.cpp:269-280)
    const size_t N = static_cast<size_t>(nc) * n;
    std::vector<double> hb(N), hx(N);
    for (int g = 0; g < nc; ++g) {
        const int old = distNewToOld_[g];
        std::copy(b + static_cast<size_t>(old) * n, b + static_cast<size_t>(old + 1) * n, hb.begin() + static_cast<size_t>(g) * n);
        std::copy(x0 + static_cast<size_t>(old) * n, x0 + static_cast<size_t>(old + 1) * n, hx.begin() + static_cast<size_t>(g) * n);
    }
    kb_.ensure(N, stream_);
    kx_.ensure(N, stream_);
    distTmp_.ensure(N, stream_);
    check(cudaMemcpyAsync(kb_.p, hb.data(), N * sizeof(double), cudaMemcpyHostToDevice, stream_), "H2D b");
    check(cudaMemcpyAsync(kx_.p, hx.data(), N * sizeof(double), cudaMemcpyHostToDevice, stream_), "H2D x0");
    sync();
    const auto t1 = clk::now();
    nc_ = nc;
    const auto t2 = distSolveCore(cfg, rep);
    const auto t3 = clk::now();
    check(cudaMemcpyAsync(hx.data(), kx_.p, N * sizeof(double), cudaMemcpyDeviceToHost, stream_), "D2H x");
    sync();
    for (int g = 0; g < nc; ++g) {  // gatherVector (partition.cpp:282-296)
        const int old = distNewToOld_[g];
        std::copy(hx.begin() + static_cast<size_t>(g) * n, hx.begin() + static_cast<size_t>(g + 1) * n,
                  x + static_cast<size_t>(old) * n);
    }
    const auto t4 = clk::now();
    rep.t_convert = secs(t0, t1);  // partition.cpp:474-477 keys
    rep.t_setup = secs(t1, t2);
    rep.t_solve = secs(t2, t3);
    rep.t_retrieve = secs(t3, t4);
    rep.t_amg_setup = rep.t_setup;
    rep.t_krylov = rep.t_solve;
    rep.amg_levels = static_cast<int>(dist_.size());
}

// distributedSolve (partition.cpp:370-479) on partitions the caller already
// built (the reference's buildPartitioned output): rank r owns global rows
// [rank_row_offset[r], rank_row_offset[r+1]) with a local BSR (local columns)
// and halo entries (local row, global column, peer rank, block).  The ranks
// are consolidated onto engines by the caller's plan (consolidate,
// partition.cpp:201-248, restated bit-exact) with every block carried by the
// id of its position in one concatenated value array [all local blocks in
// rank order | all halo blocks in rank order], which is then gathered on the
// device.  b, x0 and x are global vectors in the new (rank-major) numbering.
void Engine::distSolveParts(int nRanks, int n, const int* rankRowOffset, const int* const* localRo,
                            const int* const* localCi, const double* const* localVals, const int* haloCount,
                            const int* const* haloRow, const int* const* haloCol, const int* const* haloPeer,
                            const double* const* haloVals, int nEngines, const int* rankToEngine,
                            const int* engineRowOffset, const double* b, const double* x0, double* x,
                            const bcs_solver_config& cfg, bcs_report& rep) {
    LaunchScope ls(&launches_);
    if (n < 1 || n > 5) throw std::invalid_argument("bcs: block size must be 1..5 on the device");
    if (nRanks < 1) throw std::invalid_argument("distributedSolve: no partitions");
    if (nEngines < 1 || nEngines > nRanks) throw std::invalid_argument("makeConsolidationPlan: need 1 <= nEngines <= nRanks");
    if (nEngines > 64) throw std::invalid_argument("bcs: at most 64 engines per device");
    validateConfig(cfg);
    const auto t0 = clk::now();
    SerialStateGuard guard(*this);
    const size_t nn = static_cast<size_t>(n) * n;
    Decomposition dec;
    dec.nRanks = nRanks;
    dec.rankRowOffset.assign(rankRowOffset, rankRowOffset + nRanks + 1);
    for (int r = 0; r < nRanks; ++r)
        if (dec.rankRowOffset[r + 1] < dec.rankRowOffset[r]) throw std::invalid_argument("distributedSolve: bad row ranges");
    const int nc = dec.rankRowOffset[nRanks];
    // partitions with value ids into the concatenated array
    std::vector<Partition> parts(nRanks);
    size_t localTotal = 0, haloTotal = 0;
    for (int r = 0; r < nRanks; ++r) localTotal += static_cast<size_t>(localRo[r][dec.nLocalRows(r)]);
    for (int r = 0; r < nRanks; ++r) haloTotal += static_cast<size_t>(haloCount[r]);
    if (localTotal + haloTotal > static_cast<size_t>(INT32_MAX)) throw std::invalid_argument("distributedSolve: too many blocks");
    size_t lb = 0, hb = localTotal;
    for (int r = 0; r < nRanks; ++r) {
        Partition& p = parts[r];
        const int rows = dec.nLocalRows(r);
        p.id = r;
        p.rowStart = dec.rankRowOffset[r];
        p.rowEnd = dec.rankRowOffset[r + 1];
        p.ro.assign(localRo[r], localRo[r] + rows + 1);
        const int nnz = p.ro[rows];
        p.ci.assign(localCi[r], localCi[r] + nnz);
        p.src.resize(nnz);
        for (int k = 0; k < nnz; ++k) p.src[k] = static_cast<int>(lb + k);
        lb += nnz;
        const int nh = haloCount[r];
        p.haloRow.assign(haloRow[r], haloRow[r] + nh);
        p.haloCol.assign(haloCol[r], haloCol[r] + nh);
        p.haloPeer.assign(haloPeer[r], haloPeer[r] + nh);
        p.haloSrc.resize(nh);
        for (int h = 0; h < nh; ++h) p.haloSrc[h] = static_cast<int>(hb + h);
        hb += nh;
    }
    ConsolidationPlan plan;
    plan.nEngines = nEngines;
    plan.rankToEngine.assign(rankToEngine, rankToEngine + nRanks);
    plan.engineRowOffset.assign(engineRowOffset, engineRowOffset + nRanks);
    for (int r = 0; r < nRanks; ++r)
        if (plan.rankToEngine[r] < 0 || plan.rankToEngine[r] >= nEngines)
            throw std::invalid_argument("distributedSolve: rank mapped to no engine");
    const std::vector<Partition> engs = consolidate(parts, plan, dec);
    // the concatenated values on the device (staged), then the engines' slots
    const size_t total = localTotal + haloTotal;
    ldu_diag_.ensure(std::max<size_t>(total, 1) * nn, stream_);
    lb = 0;
    for (int r = 0; r < nRanks; ++r) {
        const size_t cnt = static_cast<size_t>(parts[r].ro.back());
        if (cnt) h2d(ldu_diag_.p + lb * nn, localVals[r], cnt * nn * sizeof(double), "H2D local blocks");
        lb += cnt;
    }
    for (int r = 0; r < nRanks; ++r) {
        const size_t cnt = static_cast<size_t>(haloCount[r]);
        if (cnt) h2d(ldu_diag_.p + lb * nn, haloVals[r], cnt * nn * sizeof(double), "H2D halo blocks");
        lb += cnt;
    }
    dist_.resize(engs.size());
    std::vector<long long> segh(engs.size() + 1, 0);
    for (size_t e = 0; e < engs.size(); ++e) {
        uploadEnginePart(dist_[e], engs[e], n, nullptr);
        dist_[e].rowStart = engs[e].rowStart;
        segh[e] = static_cast<long long>(engs[e].rowStart) * n;
        segh[e + 1] = static_cast<long long>(engs[e].rowEnd) * n;
        DistPart& P = dist_[e];
        gather_values(n, P.nnz, static_cast<int>(total), 0, P.src, ldu_diag_, nullptr, nullptr, P.vals.p, stream_);
        if (P.nh) gather_values(n, P.nh, static_cast<int>(total), 0, P.hsrc, ldu_diag_, nullptr, nullptr, P.hvals.p, stream_);
    }
    distSegh_ = segh;
    distNc_ = -1;  // the LDU-based Mode R cache no longer describes dist_
    n_ = n;
    const size_t N = static_cast<size_t>(nc) * n;
    kb_.ensure(N, stream_);
    kx_.ensure(N, stream_);
    distTmp_.ensure(N, stream_);
    h2d(kb_.p, b, N * sizeof(double), "H2D b");
    h2d(kx_.p, x0, N * sizeof(double), "H2D x0");
    sync();
    const auto t1 = clk::now();
    nc_ = nc;
    const auto t2 = distSolveCore(cfg, rep);
    const auto t3 = clk::now();
    d2h(x, kx_.p, N * sizeof(double), "D2H x");
    const auto t4 = clk::now();
    rep.t_convert = secs(t0, t1);  // partition.cpp:474-477 keys
    rep.t_setup = secs(t1, t2);
    rep.t_solve = secs(t2, t3);
    rep.t_retrieve = secs(t3, t4);
    rep.t_amg_setup = rep.t_setup;
    rep.t_krylov = rep.t_solve;
    rep.amg_levels = static_cast<int>(dist_.size());
}

// ------------------------------------------------- Mode R, one process per GPU
void Engine::commUniqueId(unsigned char id[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId u;
    nccl::ck(nccl::api().getUniqueId(&u), "unique id");
    std::memcpy(id, &u, sizeof u);
}

void Engine::commInit(int rank, int size, const unsigned char id[128]) {
    if (size < 1 || rank < 0 || rank >= size) throw std::invalid_argument("bcs_comm_init: bad rank / size");
    if (size > 64) throw std::invalid_argument("bcs_comm_init: at most 64 processes");
    const auto& A = nccl::api();
    cudaSetDevice(device_);
    if (comm_ && A.commDestroy) A.commDestroy(static_cast<ncclComm_t>(comm_));
    comm_ = nullptr;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    ncclComm_t c = nullptr;
    nccl::g_rank = rank;
    nccl::ck(A.commInitRank(&c, size, u, rank), "comm init");
    comm_ = c;
    if (!commStream_) {
        check(cudaStreamCreateWithFlags(&commStream_, cudaStreamNonBlocking), "cudaStreamCreate comm");
        check(cudaEventCreateWithFlags(&mpEvPack_, cudaEventDisableTiming), "cudaEventCreate");
        check(cudaEventCreateWithFlags(&mpEvComm_, cudaEventDisableTiming), "cudaEventCreate");
    }
    mpRank_ = rank;
    mpSize_ = size;
    mpNc_ = -1;  // topology cache belongs to the previous communicator
}

// this process's engine of the consolidated decomposition (engines = processes)
void Engine::mpSetupTopology(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh,
                             const double* centroids, int nRanks) {
    const Decomposition dec = decompose(nc, centroids, nRanks);
    const std::vector<Partition> parts = buildPartitioned(nc, nf, owner, neigh, dec);
    const ConsolidationPlan plan = makeConsolidationPlan(dec, mpSize_);
    const std::vector<Partition> eng = consolidate(parts, plan, dec);
    const ExchangePlan xp = makeExchangePlan(eng, mpRank_);
    mpPart = eng[mpRank_];  // host slot sources for the per-rank upload
    dist_.resize(1);
    uploadEnginePart(dist_[0], eng[mpRank_], n, &xp.haloRecvIdx);
    mpRows_ = dist_[0].rows;
    mpSendCnt_ = xp.sendCount;
    mpRecvCnt_ = xp.recvCount;
    mpSendRows_ = static_cast<int>(xp.sendRows.size());
    mpRecvRows_ = static_cast<int>(xp.recvGlobalRow.size());
    mpSendIdx_.ensure(std::max(1, mpSendRows_), stream_);
    if (mpSendRows_)
        check(cudaMemcpyAsync(mpSendIdx_.p, xp.sendRows.data(), sizeof(int) * mpSendRows_, cudaMemcpyHostToDevice,
                              stream_), "H2D");
    mpSend_.ensure(static_cast<size_t>(std::max(1, mpSendRows_)) * n, stream_);
    mpRecv_.ensure(static_cast<size_t>(std::max(1, mpRecvRows_)) * n, stream_);
    mpPart_.ensure(1, stream_);
    mpGath_.ensure(mpSize_, stream_);
    mpEngStart_.assign(mpSize_, 0);
    mpEngRows_.assign(mpSize_, 0);
    mpMaxRows_ = 0;
    for (int e = 0; e < mpSize_; ++e) {
        mpEngStart_[e] = eng[e].rowStart;
        mpEngRows_[e] = eng[e].nLocalRows();
        mpMaxRows_ = std::max(mpMaxRows_, mpEngRows_[e]);
    }
    mpXall_.ensure(static_cast<size_t>(mpMaxRows_) * n * (mpSize_ + 1), stream_);
    // reductions: the block layout of an engine segment in the one-device Mode R
    mpBps_ = seg_blocks(mpSize_);

    mpNewToOld_ = dec.newToOld;
    mpOwner_.assign(owner, owner + nf);
    mpNeigh_.assign(neigh, neigh + nf);
    mpCen_.assign(centroids, centroids + 3 * static_cast<size_t>(nc));
    mpRanks_ = nRanks;
    mpNc_ = nc;
    mpNf_ = nf;
    mpN_ = n;
    distNc_ = -1;  // the one-device Mode R cache no longer describes dist_
    sync();
}

void Engine::distSolveMP(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh, const double* centroids,
                         const double* diag, const double* upper, const double* lower, const double* b,
                         const double* x0, double* x, int nRanks, const bcs_solver_config& cfg, bcs_report& rep) {
    LaunchScope ls(&launches_);
    const long long l0 = launches_.launches;
    if (!comm_) throw std::invalid_argument("bcs_dist_solve_mp: call bcs_comm_init first");
    if (n < 1 || n > 5) throw std::invalid_argument("bcs: block size must be 1..5 on the device");
    if (mpSize_ < 1 || mpSize_ > nRanks) throw std::invalid_argument("makeConsolidationPlan: need 1 <= nEngines <= nRanks");
    validateConfig(cfg);
    const auto t0 = clk::now();
    const bool same = mpNc_ == nc && mpNf_ == nf && mpN_ == n && mpRanks_ == nRanks &&
                      parallelEqual(owner, mpOwner_.data(), static_cast<size_t>(nf)) &&
                      parallelEqual(neigh, mpNeigh_.data(), static_cast<size_t>(nf)) &&
                      parallelEqual(centroids, mpCen_.data(), 3 * static_cast<size_t>(nc));
    SerialStateGuard guard(*this);
    if (!same) mpSetupTopology(nc, nf, n, owner, neigh, centroids, nRanks);
    n_ = n;
    DistPart& P = dist_[0];
    const size_t nn = static_cast<size_t>(n) * n;
    // upload (partition.cpp:384-407): only this engine's local and halo blocks
    // cross PCIe, gathered on the host into page-locked staging in slot order.
    // An engine that needs most of the system (one or two processes) takes the
    // whole LDU at full DMA rate and gathers on the device instead.
    const size_t nnzAll = static_cast<size_t>(nc) + 2 * static_cast<size_t>(nf);
    const int hw = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    if (2 * (static_cast<size_t>(P.nnz) + P.nh) > nnzAll) {
        ldu_diag_.ensure(nc * nn, stream_);
        ldu_upper_.ensure(nf * nn, stream_);
        ldu_lower_.ensure(nf * nn, stream_);
        h2d(ldu_diag_.p, diag, sizeof(double) * nc * nn, "H2D");
        if (nf) {
            h2d(ldu_upper_.p, upper, sizeof(double) * nf * nn, "H2D");
            h2d(ldu_lower_.p, lower, sizeof(double) * nf * nn, "H2D");
        }
        gather_values(n, P.nnz, nc, nf, P.src, ldu_diag_, ldu_upper_, ldu_lower_, P.vals.p, stream_);
        if (P.nh) gather_values(n, P.nh, nc, nf, P.hsrc, ldu_diag_, ldu_upper_, ldu_lower_, P.hvals.p, stream_);
    } else {
        const size_t cnt = (static_cast<size_t>(P.nnz) + P.nh) * nn;
        if (mpStageCap_ < cnt) {
            if (mpStage_) cudaFreeHost(mpStage_);
            mpStage_ = nullptr;
            mpStageCap_ = 0;
            check(cudaHostAlloc(reinterpret_cast<void**>(&mpStage_), cnt * sizeof(double), cudaHostAllocPortable),
                  "cudaHostAlloc upload staging");
            mpStageCap_ = cnt;
        }
        sync();  // the previous call's copies out of the staging buffer are done
        gatherPartValues(mpPart, nc, nf, n, diag, upper, lower, mpStage_, mpStage_ + static_cast<size_t>(P.nnz) * nn,
                         hw);
        check(cudaMemcpyAsync(P.vals.p, mpStage_, sizeof(double) * P.nnz * nn, cudaMemcpyHostToDevice, stream_), "H2D");
        if (P.nh)
            check(cudaMemcpyAsync(P.hvals.p, mpStage_ + static_cast<size_t>(P.nnz) * nn, sizeof(double) * P.nh * nn,
                                  cudaMemcpyHostToDevice, stream_), "H2D halo");
    }
    // this engine's slice of scatterVector (partition.cpp:269-280)
    const size_t Nl = static_cast<size_t>(mpRows_) * n;
    std::vector<double> hb(Nl), hx(Nl);
    const int g0 = mpEngStart_[mpRank_];
    parallelFor(mpRows_, hw, [&](int r) {
        const int old = mpNewToOld_[g0 + r];
        std::copy(b + static_cast<size_t>(old) * n, b + static_cast<size_t>(old + 1) * n, hb.begin() + static_cast<size_t>(r) * n);
        std::copy(x0 + static_cast<size_t>(old) * n, x0 + static_cast<size_t>(old + 1) * n, hx.begin() + static_cast<size_t>(r) * n);
    });
    kb_.ensure(Nl, stream_);
    kx_.ensure(Nl, stream_);
    distTmp_.ensure(Nl, stream_);
    check(cudaMemcpyAsync(kb_.p, hb.data(), Nl * sizeof(double), cudaMemcpyHostToDevice, stream_), "H2D b");
    check(cudaMemcpyAsync(kx_.p, hx.data(), Nl * sizeof(double), cudaMemcpyHostToDevice, stream_), "H2D x0");
    sync();
    const auto t1 = clk::now();
    hist_.clear();
    spmvMs_ = 0.0;
    spmvCount_ = 0;
    sweepMs_ = 0.0;
    sweepBytes_ = 0.0;
    sweepCount_ = 0;
    evUsed_ = 0;
    cudaMemsetAsync(err_.p + 1, 0, sizeof(int), stream_);
    nc_ = mpRows_;
    H_ = &P.H;
    FineMatrix F;
    F.rows = P.rows;
    F.nnz = P.nnz;
    F.ro = P.ro;
    F.ci = P.ci;
    F.dg = P.dg;
    F.tpos = P.tpos;
    F.v = P.vals;
    buildPrecondOn(F, cfg);
    H_ = &main_;
    sync();
    const auto t2 = clk::now();
    distActive_ = true;
    mpActive_ = true;
    nseg_ = 1;
    {
        const long long segh[2] = {0, static_cast<long long>(mpRows_) * n};
        check(cudaMemcpyAsync(seg_.p, segh, sizeof segh, cudaMemcpyHostToDevice, stream_), "H2D seg");
    }
    solveKrylov(kb_, kx_.p, cfg, rep);
    distActive_ = mpActive_ = false;
    const auto t3 = clk::now();
    // gatherVector (partition.cpp:282-296): padded all-gather of the slices
    const size_t pad = static_cast<size_t>(mpMaxRows_) * n;
    double* mine = mpXall_.p + pad * mpSize_;
    check(cudaMemsetAsync(mine, 0, pad * sizeof(double), stream_), "memset");
    check(cudaMemcpyAsync(mine, kx_.p, Nl * sizeof(double), cudaMemcpyDeviceToDevice, stream_), "D2D");
    nccl::ck(nccl::api().allGather(mine, mpXall_.p, pad, ncclDouble, static_cast<ncclComm_t>(comm_), stream_),
             "allgather x");
    std::vector<double> all(pad * mpSize_);
    check(cudaMemcpyAsync(all.data(), mpXall_.p, all.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_), "D2H x");
    sync();
    for (int e = 0; e < mpSize_; ++e)
        parallelFor(mpEngRows_[e], hw, [&](int r) {
            const int old = mpNewToOld_[mpEngStart_[e] + r];
            std::copy(all.begin() + pad * e + static_cast<size_t>(r) * n, all.begin() + pad * e + static_cast<size_t>(r + 1) * n,
                      x + static_cast<size_t>(old) * n);
        });
    const auto t4 = clk::now();
    rep.t_convert = secs(t0, t1);  // partition.cpp:474-477 keys
    rep.t_setup = secs(t1, t2);
    rep.t_solve = secs(t2, t3);
    rep.t_retrieve = secs(t3, t4);
    rep.t_amg_setup = rep.t_setup;
    rep.t_krylov = rep.t_solve;
    rep.amg_levels = P.H.pcKind == BCS_PRECOND_AMG ? P.H.nlev : 0;
    rep.kernel_launches = static_cast<int>(launches_.launches - l0);
}

void Engine::solveHost(const double* b, double* x, const bcs_solver_config& cfg, bcs_report& rep) {
    requireMatrix();
    const size_t N = static_cast<size_t>(nc_) * n_;
    kb_.ensure(N, stream_);
    kx_.ensure(N, stream_);
    h2d(kb_.p, b, N * sizeof(double), "H2D b");
    h2d(kx_.p, x, N * sizeof(double), "H2D x");
    solveDevice(kb_, kx_, cfg, rep);
    d2h(x, kx_.p, N * sizeof(double), "D2H x");  // synchronous
}

// Backend::HostLdu's two slot orders of the LDU blocks (ids: cell c, upper
// of face f = nc + f, lower of face f = nc + nf + f), built on the host:
//   matvec row c: diag, then every face touching c in face order (upper when c
//     owns it, column = neighbour; lower otherwise, column = owner) -- the
//     accumulation order of blockMatvec (block_matrix.cpp:104-119);
//   LUSGS row c: lower faces (c = neighbour) in face order, diag, upper faces
//     (c = owner) in DESCENDING face order -- the sweep kernels walk the upper
//     part backwards, so LduLusgsPrecond::apply's face order results
//     (preconditioner.cpp:81-99).
void Engine::hostLduTopology() {
    if (hlTopo_) return;
    const int nc = nc_, nf = nf_;
    const size_t nnz = static_cast<size_t>(nc) + 2 * static_cast<size_t>(nf);
    std::vector<int> deg(static_cast<size_t>(nc) + 1, 0);
    for (int f = 0; f < nf; ++f) {
        ++deg[hOwner_[f] + 1];
        ++deg[hNeigh_[f] + 1];
    }
    std::vector<int> cfo(static_cast<size_t>(nc) + 1, 0);  // cell -> faces (face order)
    for (int c = 0; c < nc; ++c) cfo[c + 1] = cfo[c] + deg[c + 1];
    std::vector<int> cf(2 * static_cast<size_t>(nf)), pos(cfo.begin(), cfo.end() - 1);
    for (int f = 0; f < nf; ++f) {
        cf[pos[hOwner_[f]]++] = f;
        cf[pos[hNeigh_[f]]++] = f;
    }
    std::vector<int> ro(static_cast<size_t>(nc) + 1), mci(nnz), msrc(nnz), gci(nnz), gsrc(nnz), gdg(nc);
    for (int c = 0; c < nc; ++c) ro[c + 1] = ro[c] + 1 + (cfo[c + 1] - cfo[c]);
    for (int c = 0; c < nc; ++c) {
        int k = ro[c];
        mci[k] = c;
        msrc[k] = c;
        ++k;
        for (int q = cfo[c]; q < cfo[c + 1]; ++q) {
            const int f = cf[q];
            const bool own = hOwner_[f] == c;
            mci[k] = own ? hNeigh_[f] : hOwner_[f];
            msrc[k] = own ? nc + f : nc + nf + f;
            ++k;
        }
        k = ro[c];
        for (int q = cfo[c]; q < cfo[c + 1]; ++q)  // lower faces ascending
            if (hNeigh_[cf[q]] == c) {
                gci[k] = hOwner_[cf[q]];
                gsrc[k] = nc + nf + cf[q];
                ++k;
            }
        gdg[c] = k;
        gci[k] = c;
        gsrc[k] = c;
        ++k;
        for (int q = cfo[c + 1] - 1; q >= cfo[c]; --q)  // upper faces descending
            if (hOwner_[cf[q]] == c) {
                gci[k] = hNeigh_[cf[q]];
                gsrc[k] = nc + cf[q];
                ++k;
            }
    }
    auto up = [&](DArray<int>& d, const std::vector<int>& h) {
        d.ensure(h.size() + 1, stream_);
        check(cudaMemcpyAsync(d.p, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, stream_), "H2D host-LDU");
    };
    up(hlMvRo_, ro);
    up(hlMvCi_, mci);
    up(hlMvSrc_, msrc);
    up(hlGsRo_, ro);
    up(hlGsCi_, gci);
    up(hlGsSrc_, gsrc);
    up(hlGsDg_, gdg);
    const size_t nn = static_cast<size_t>(n_) * n_;
    hlMvV_.ensure(nnz * nn, stream_);
    hlGsV_.ensure(nnz * nn, stream_);
    sync();  // the host vectors die here
    hlTopo_ = true;
}

// krylovSolve with the HostLdu operators (engine.cpp:54-72): blockMatvec and
// LduLusgsPrecond arithmetic, on the device
void Engine::solveHostLdu(const double* b, double* x, const bcs_solver_config& cfg, bcs_report& rep) {
    LaunchScope ls(&launches_);
    const size_t N = static_cast<size_t>(nc_) * n_;
    kb_.ensure(N, stream_);
    kx_.ensure(N, stream_);
    h2d(kb_.p, b, N * sizeof(double), "H2D b");
    h2d(kx_.p, x, N * sizeof(double), "H2D x");
    distActive_ = false;
    H_ = &main_;
    nseg_ = 1;
    const long long segh[2] = {0, static_cast<long long>(N)};
    check(cudaMemcpyAsync(seg_.p, segh, sizeof segh, cudaMemcpyHostToDevice, stream_), "seg");
    hist_.clear();
    evUsed_ = 0;
    spmvMs_ = sweepMs_ = sweepBytes_ = 0.0;
    spmvCount_ = sweepCount_ = 0;
    cudaMemsetAsync(err_.p + 1, 0, sizeof(int), stream_);
    struct Flag {
        bool& f;
        ~Flag() { f = false; }
    } flag{hostLdu_};
    hostLdu_ = true;
    FineMatrix F;  // the LUSGS slot order
    F.rows = nc_;
    F.nnz = nc_ + 2 * nf_;
    F.ro = hlGsRo_;
    F.ci = hlGsCi_;
    F.dg = hlGsDg_;
    F.tpos = nullptr;
    F.v = hlGsV_;
    const auto t0 = clk::now();
    buildPrecondOn(F, cfg);
    sync();
    const auto t1 = clk::now();
    solveKrylov(kb_, kx_.p, cfg, rep);
    rep.t_amg_setup = secs(t0, t1);
    rep.t_krylov = secs(t1, clk::now());
    d2h(x, kx_.p, N * sizeof(double), "D2H x");
    // the serial preconditioner now describes the host-LDU matrix, not vals_
    main_.pcKind = -1;
}

// SolvePipeline::solve (engine.cpp:47-120)
// The face lists of this call equal the stored topology's (the exact test the
// reference's signature comparison stands for, engine.cpp:85), compared in
// parallel chunks: 2 x 25 MB at 128^3 would otherwise cost ~5 ms of one core.
bool Engine::sameFaces(const int32_t* owner, const int32_t* neigh, int nf) const {
    const size_t n = static_cast<size_t>(nf);
    const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    const size_t parts = n < (1u << 20) ? 1 : hw;
    std::vector<char> eq(parts, 1);
    auto work = [&](size_t p) {
        const size_t b = n * p / parts, e = n * (p + 1) / parts;
        eq[p] = std::equal(owner + b, owner + e, hOwner_.begin() + b) && std::equal(neigh + b, neigh + e, hNeigh_.begin() + b);
    };
    std::vector<std::thread> th;
    for (size_t p = 1; p < parts; ++p) th.emplace_back(work, p);
    work(0);
    for (auto& t : th) t.join();
    return std::all_of(eq.begin(), eq.end(), [](char c) { return c != 0; });
}

void Engine::pipelineSolve(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh, const double* diag,
                           const double* upper, const double* lower, const double* b, size_t b_len,
                           const double* x0, size_t x0_len, double* x, int backend, const bcs_solver_config& cfg,
                           bcs_report& rep) {
    const size_t N = static_cast<size_t>(nc) * n;
    if (b_len != N || x0_len != N) throw std::invalid_argument("SolvePipeline::solve: dimension mismatch");
    if (backend != BCS_BACKEND_HOST_LDU && backend != BCS_BACKEND_ENGINE_CSR)
        throw std::invalid_argument("unknown backend");
    const bool sameTopo = hasTopo_ && nc == nc_ && nf == nf_ && n == n_ && sameFaces(owner, neigh, nf);
    if (backend == BCS_BACKEND_HOST_LDU) {
        if (cfg.precond != BCS_PRECOND_NONE && cfg.precond != BCS_PRECOND_LUSGS)
            throw std::invalid_argument("host backend supports only none/LUSGS preconditioning");
        validateConfig(cfg);
        const auto t0 = clk::now();
        if (!sameTopo) setTopology(nc, nf, n, owner, neigh);
        hostLduTopology();
        // the LDU values in the two face-addressed slot orders
        const size_t nn = static_cast<size_t>(n_) * n_;
        ldu_diag_.ensure(nc_ * nn, stream_);
        ldu_upper_.ensure(nf_ * nn, stream_);
        ldu_lower_.ensure(nf_ * nn, stream_);
        h2d(ldu_diag_.p, diag, sizeof(double) * nc_ * nn, "H2D diag");
        if (nf_) {
            h2d(ldu_upper_.p, upper, sizeof(double) * nf_ * nn, "H2D upper");
            h2d(ldu_lower_.p, lower, sizeof(double) * nf_ * nn, "H2D lower");
        }
        const int nnz = nc_ + 2 * nf_;
        gather_values(n_, nnz, nc_, nf_, hlMvSrc_, ldu_diag_, ldu_upper_, ldu_lower_, hlMvV_.p, stream_);
        gather_values(n_, nnz, nc_, nf_, hlGsSrc_, ldu_diag_, ldu_upper_, ldu_lower_, hlGsV_.p, stream_);
        std::memcpy(x, x0, N * sizeof(double));
        solveHostLdu(b, x, cfg, rep);
        rep.t_solve = secs(t0, clk::now());
        rep.t_convert = rep.t_setup = rep.t_retrieve = rep.t_replace = 0.0;
        rep.setup_branch = 0;
        return;
    }
    const size_t nn = static_cast<size_t>(n) * n;
    (void)nn;
    // "convert": stage b and x0 on the device
    auto t = clk::now();
    kb_.ensure(N, stream_);
    kx_.ensure(N, stream_);
    h2d(kb_.p, b, N * sizeof(double), "H2D b");
    h2d(kx_.p, x0, N * sizeof(double), "H2D x0");
    sync();
    rep.t_convert = secs(t, clk::now());
    // setup-or-replace by topology signature (engine.cpp:85-98)
    bool takeSetup = !pipeHasSetup_;
    if (!takeSetup && !sameTopo) {
        if (!pipeSigValid_ && hasTopo_) {
            pipeSig_ = topologySignatureHost(nc_, nf_, hOwner_.data(), hNeigh_.data());
            pipeSigValid_ = true;
        }
        const uint64_t sig = topologySignatureHost(nc, nf, owner, neigh);
        takeSetup = sig != pipeSig_;
    }
    t = clk::now();
    if (takeSetup || !sameTopo) {
        try {
            setTopology(nc, nf, n, owner, neigh);
        } catch (...) {
            pipeHasSetup_ = false;  // the next call takes the setup branch again
            pipeSigValid_ = false;
            throw;
        }
    }
    uploadLdu(diag, upper, lower, false);
    sync();
    const double tsr = secs(t, clk::now());
    if (takeSetup) {
        rep.t_setup = tsr;
        rep.t_replace = 0.0;
        rep.setup_branch = 1;
        pipeSigValid_ = false;  // computed lazily on the next topology change
        pipeHasSetup_ = true;
    } else {
        rep.t_replace = tsr;
        rep.t_setup = 0.0;
        rep.setup_branch = 0;
    }
    // "solve": preconditioner + Krylov
    t = clk::now();
    solveDevice(kb_, kx_, cfg, rep);
    rep.t_solve = secs(t, clk::now());
    // "retrieve"
    t = clk::now();
    d2h(x, kx_.p, N * sizeof(double), "D2H x");  // synchronous
    rep.t_retrieve = secs(t, clk::now());
}

// ------------------------------------------------------------ query paths
double Engine::residualNorm(const double* b, const double* x) {
    LaunchScope ls(&launches_);
    requireMatrix();
    nseg_ = 1;
    const long long segh[2] = {0, static_cast<long long>(nc_) * n_};
    check(cudaMemcpyAsync(seg_.p, segh, sizeof segh, cudaMemcpyHostToDevice, stream_), "seg");
    const size_t N = static_cast<size_t>(nc_) * n_;
    kb_.ensure(N, stream_);
    kx_.ensure(N, stream_);
    rk_.ensure(N, stream_);
    h2d(kb_.p, b, N * sizeof(double), "H2D b");
    h2d(kx_.p, x, N * sizeof(double), "H2D x");
    spmv(n_, nc_, ro_, ci_, vals_, kx_, kb_, rk_.p, stream_);
    return dotHost(rk_, rk_, N, true);
}

void Engine::spmvDevice(const double* d_x, double* d_y) {
    LaunchScope ls(&launches_);
    requireMatrix();
    spmv(n_, nc_, ro_, ci_, vals_, d_x, nullptr, d_y, stream_);
    checkErr("spmv");
}

void Engine::spmvHost(const double* x, double* y) {
    const size_t N = static_cast<size_t>(nc_) * n_;
    requireMatrix();
    kb_.ensure(N, stream_);
    kx_.ensure(N, stream_);
    check(cudaMemcpyAsync(kx_.p, x, N * sizeof(double), cudaMemcpyHostToDevice, stream_), "H2D x");
    spmvDevice(kx_, kb_.p);
    check(cudaMemcpyAsync(y, kb_.p, N * sizeof(double), cudaMemcpyDeviceToHost, stream_), "D2H y");
    sync();
}

void Engine::csrGet(int32_t* ro, int32_t* ci, double* v) {
    requireMatrix();
    const size_t nnz = static_cast<size_t>(nc_) + 2 * static_cast<size_t>(nf_);
    if (ro) check(cudaMemcpyAsync(ro, ro_.p, sizeof(int) * (nc_ + 1), cudaMemcpyDeviceToHost, stream_), "D2H ro");
    if (ci) check(cudaMemcpyAsync(ci, ci_.p, sizeof(int) * nnz, cudaMemcpyDeviceToHost, stream_), "D2H ci");
    if (v) check(cudaMemcpyAsync(v, vals_.p, sizeof(double) * nnz * n_ * n_, cudaMemcpyDeviceToHost, stream_), "D2H v");
    sync();
}

void Engine::precondSetup(const bcs_solver_config& cfg) {
    LaunchScope ls(&launches_);
    validateConfig(cfg);
    buildPrecond(cfg);
    sync();
}

void Engine::precondApplyHost(const double* r, double* z) {
    LaunchScope ls(&launches_);
    if (H_->pcKind < 0) throw std::invalid_argument("bcs: call bcs_precond_setup first");
    const size_t N = static_cast<size_t>(nc_) * n_;
    kb_.ensure(N, stream_);
    kx_.ensure(N, stream_);
    cudaMemsetAsync(err_.p + 1, 0, sizeof(int), stream_);
    check(cudaMemcpyAsync(kb_.p, r, N * sizeof(double), cudaMemcpyHostToDevice, stream_), "H2D r");
    applyPrecond(kb_, kx_.p);
    check(cudaMemcpyAsync(z, kx_.p, N * sizeof(double), cudaMemcpyDeviceToHost, stream_), "D2H z");
    sync();
    checkErr("precond apply");
    int spinErr = 0;
    check(cudaMemcpy(&spinErr, err_.p + 1, sizeof(int), cudaMemcpyDeviceToHost), "spin flag");
    if (spinErr) throw std::runtime_error("bcs: sweep dependency wait timed out (corrupt schedule)");
}

void Engine::amgLevelSizes(int l, int* rows, int* nnz) const {
    if (l < 0 || l >= H_->nlev) throw std::invalid_argument("bcs: level out of range");
    *rows = H_->levels[l].rows;
    *nnz = H_->levels[l].nnz;
}

void Engine::amgLevelGet(int l, int32_t* ro, int32_t* ci, double* v, int32_t* agg) {
    if (l < 0 || l >= H_->nlev) throw std::invalid_argument("bcs: level out of range");
    const Level& L = H_->levels[l];
    const size_t nn = static_cast<size_t>(n_) * n_;
    if (ro) check(cudaMemcpyAsync(ro, L.ro, sizeof(int) * (L.rows + 1), cudaMemcpyDeviceToHost, stream_), "D2H");
    if (ci) check(cudaMemcpyAsync(ci, L.ci, sizeof(int) * L.nnz, cudaMemcpyDeviceToHost, stream_), "D2H");
    if (v) check(cudaMemcpyAsync(v, L.v, sizeof(double) * L.nnz * nn, cudaMemcpyDeviceToHost, stream_), "D2H");
    if (agg && l + 1 < H_->nlev)
        check(cudaMemcpyAsync(agg, L.agg.p, sizeof(int) * L.rows, cudaMemcpyDeviceToHost, stream_), "D2H");
    sync();
}

std::string Engine::memoryReport() const {
    std::map<std::string, double> m;
    // owned arrays only; arena views are counted once, as the arena
    auto add = [&](const char* k, const auto& a) {
        if (a.owned) m[k] += static_cast<double>(a.cap) * sizeof(*a.p);
    };
    auto hier = [&](const Hier& H, bool fine) {
        for (size_t l = 0; l < H.levels.size(); ++l) {
            const Level& L = H.levels[l];
            add("bsr_coarse", L.o_v);
            add("pattern", L.o_ro); add("pattern", L.o_ci); add("pattern", L.o_dg); add("pattern", L.o_tpos);
            add("smoother_factors", L.lu); add("smoother_factors", L.rcp); add("smoother_factors", L.piv);
            add("smoother_factors", L.perm);
            add("schedule", L.order); add("schedule", L.recf); add("schedule", L.recb); add("schedule", L.offf);
            add("schedule", L.offb); add("schedule", L.dlev); add("schedule", L.woff); add("schedule", L.woffb);
            add("sweep_programs", L.pkf); add("sweep_programs", L.pkb);
            add("aggregates", L.agg); add("aggregates", L.members);
            add("vcycle_vectors", L.r); add("vcycle_vectors", L.z); add("vcycle_vectors", L.res);
            add("vcycle_vectors", L.y); add("vcycle_vectors", L.zb);
            if (L.mc) {  // performance mode: the colour-permuted copy and its smoother
                const Level& M = *L.mc;
                add("perf_coloured_copies", M.o_v); add("perf_coloured_copies", M.o_ro); add("perf_coloured_copies", M.o_ci);
                add("perf_coloured_copies", M.o_dg); add("perf_coloured_copies", M.o_tpos); add("perf_coloured_copies", M.lu);
                add("perf_coloured_copies", M.rcp); add("perf_coloured_copies", M.piv); add("perf_coloured_copies", M.perm);
                add("perf_coloured_copies", M.order); add("perf_coloured_copies", M.recf); add("perf_coloured_copies", M.recb);
                add("perf_coloured_copies", M.offf); add("perf_coloured_copies", M.offb); add("perf_coloured_copies", M.dlev);
                add("perf_coloured_copies", M.r); add("perf_coloured_copies", M.y); add("perf_coloured_copies", M.zb);
                add("perf_coloured_copies", L.mcPerm); add("perf_coloured_copies", L.mcColorOffD);
            }
        }
        add("dense_coarsest", H.dense); add("dense_coarsest", H.dpiv); add("schedule", H.tailDesc);
        m["phase_arena (DILU scratch | sweep programs + Krylov basis)"] += static_cast<double>(H.arena.cap);
        (void)fine;
    };
    hier(main_, true);
    for (const auto& P : dist_) {
        add("mode_r_engines", P.vals); add("mode_r_engines", P.hvals); add("mode_r_engines", P.ro);
        add("mode_r_engines", P.ci); add("mode_r_engines", P.src); add("mode_r_engines", P.dg);
        add("mode_r_engines", P.tpos); add("mode_r_engines", P.hrow); add("mode_r_engines", P.hoff);
        add("mode_r_engines", P.hcol); add("mode_r_engines", P.hsrc);
        hier(P.H, false);
    }
    add("bsr_fine", vals_);
    add("pattern", ro_); add("pattern", ci_); add("pattern", dg_); add("pattern", tpos_); add("pattern", src_);
    add("pattern", fill_); add("pattern", dOwner_); add("pattern", dNeigh_);
    add("ldu_staging", ldu_diag_); add("ldu_staging", ldu_upper_); add("ldu_staging", ldu_lower_);
    add("dilu_setup_scratch", tblk_);
    for (const auto* a : {&V_, &Z_, &w_, &zk_, &rk_, &kb_, &kx_, &bp_, &bv_, &bs_, &bt_, &bph_, &bsh_, &brh_, &distTmp_})
        add("krylov", *a);
    for (const auto* a : {&asmMuGrad_, &asmPsi_, &asmFs_, &asmBp_, &asmArea_, &asmBarea_, &asmQ_, &asmRhs_, &asmFx_,
                          &asmVol_, &asmCen_, &asmBu_, &asmPhi_, &asmD_, &asmGrad_})
        add("assembly", *a);
    for (const auto* a : {&asmInv_, &asmCfo_, &asmCf_, &asmBco_, &asmBkind_, &asmBad_}) add("assembly", *a);
    for (const auto* a : {&cnt_, &lvl_, &act2_, &push_, &scanTmp_, &flag_, &err_, &ctr_, &choice_, &segOff_, &cro_,
                          &big_, &dkeys_, &dorder_, &ticket_, &chunkOrd_, &chainCnt_, &partOrd_})
        add("setup_scratch", *a);
    add("setup_scratch", dn_); add("setup_scratch", str_); add("setup_scratch", keys_); add("setup_scratch", sorted_);
    add("setup_scratch", ddesc_);
    double total = 0.0;
    std::string out = "{";
    for (const auto& [k, v] : m) {
        total += v;
        out += "\"" + k + "\": " + std::to_string(static_cast<long long>(v)) + ", ";
    }
    out += "\"total\": " + std::to_string(static_cast<long long>(total)) + "}";
    return out;
}

int Engine::levelColoring(int l, int32_t* perm, int32_t* colorOff) {
    if (l < 0 || l >= H_->nlev) throw std::invalid_argument("bcs: level out of range");
    Level& L = H_->levels[l];
    if (!L.mcValid) return 0;
    if (colorOff) std::copy(L.mcColorOff.begin(), L.mcColorOff.end(), colorOff);
    if (perm) {
        check(cudaMemcpyAsync(perm, L.mcPerm.p, sizeof(int) * L.rows, cudaMemcpyDeviceToHost, stream_), "D2H perm");
        sync();
    }
    return L.ncolors;
}

int Engine::scheduleDepth(int l) const {
    if (l < 0 || l >= H_->nlev) throw std::invalid_argument("bcs: level out of range");
    return H_->levels[l].depth;
}

}  // namespace bcs
