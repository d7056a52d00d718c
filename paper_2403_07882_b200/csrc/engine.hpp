// bcs::Engine — the device-side state behind one bcs_ctx: the BSR plan of
// the current topology, the AMG hierarchy / smoother factors rebuilt on every
// solve (engine.cpp:100-107 semantics), and the Krylov workspace.
#pragma once

#include "../../include/bcs.h"
#include "kernels.hpp"
#include "partition.hpp"

#include <chrono>
#include <memory>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace bcs {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void check(cudaError_t e, const char* what);

// Stream-ordered device array (cudaMallocAsync from the device pool, whose
// release threshold is raised so that steady-state solves never return memory
// to the driver).  Grows by capacity; contents are not preserved on growth.
template <class T>
struct DArray {
    T* p = nullptr;
    size_t cap = 0;
    bool owned = true;  // false: a view into a PhaseArena (never freed here)
    void ensure(size_t n, cudaStream_t s) {
        if (n <= cap && p) return;
        if (p && owned) check(cudaFreeAsync(p, s), "cudaFreeAsync");
        p = nullptr;
        cap = 0;
        owned = true;
        // + 64 bytes: the 16-byte-widened copies (cp.async / TMA bulk ranges
        // rounded out to 16-byte bounds) may touch up to 15 bytes past the end
        const size_t bytes = (n ? n : 1) * sizeof(T) + 64;
        check(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, s), "cudaMallocAsync");
        cap = n ? n : 1;
    }
    // point at n elements of arena memory (valid until the arena's next phase)
    void borrow(T* q, size_t n, cudaStream_t s) {
        if (p && owned) cudaFreeAsync(p, s);
        p = q;
        cap = n;
        owned = false;
    }
    void release(cudaStream_t s) {
        if (p && owned) cudaFreeAsync(p, s);
        p = nullptr;
        cap = 0;
        owned = true;
    }
    operator T*() const { return p; }
};

// Memory whose lifetime is one phase of a solve: the DILU factorisation's
// scratch (T, setup phase) and the sweep programs + Krylov basis (solve
// phase) never coexist, so they share one buffer (peak = max of the phases,
// not their sum).  reserve() starts a phase: it re-allocates only when the
// phase needs more than the buffer holds (first solve / bigger system); in
// steady state no allocator call happens.
struct PhaseArena {
    char* base = nullptr;
    size_t cap = 0, off = 0;
    static size_t al(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }
    void reserve(size_t bytes, cudaStream_t s) {
        off = 0;
        if (bytes <= cap) return;
        if (base) check(cudaFreeAsync(base, s), "cudaFreeAsync arena");
        base = nullptr;
        cap = 0;
        check(cudaMallocAsync(reinterpret_cast<void**>(&base), bytes + 64, s), "cudaMallocAsync arena");  // widened-copy slack
        cap = bytes;
    }
    template <class T>
    T* take(size_t n) {
        const size_t b = al(n * sizeof(T));
        if (off + b > cap) throw std::logic_error("bcs: phase arena overflow");
        T* q = reinterpret_cast<T*>(base + off);
        off += b;
        return q;
    }
    void release(cudaStream_t s) {
        if (base) cudaFreeAsync(base, s);
        base = nullptr;
        cap = off = 0;
    }
};

struct Level {
    int rows = 0, nnz = 0;
    // pattern/values: level 0 aliases the engine's plan arrays
    const int* ro = nullptr;
    const int* ci = nullptr;
    const int* dg = nullptr;
    const int* tpos = nullptr;
    const double* v = nullptr;
    DArray<int> o_ro, o_ci, o_dg, o_tpos;
    DArray<double> o_v;
    // smoother (DILU or LUSGS) factors + level-sorted schedule
    DArray<double> lu, rcp;
    DArray<int> piv, perm, order, recf, recb;  // perm: composed pivot permutation; recf/recb: int4 records
    DArray<int> offf, offb;                    // per-ticket slot offsets (16-byte units), rows + 1
    DArray<int> dlev;                          // dependency level of every row
    DArray<int> tc, lpre;                      // DILU setup only: compact T indices (released after)
    DArray<unsigned char> pkf, pkb;            // packed per-ticket slots of the two sweeps
    int depth = 0;
    bool dlevOk = false;     // dlev holds the dependency levels of the current factorisation
    bool chain = false;      // chain schedule (k_sweep_chain), launched with depth -1
    DArray<int> woff, woffb;  // chain schedule: warp ticket ranges of the two sweeps
    int sweepDepth() const { return chain ? -1 : depth; }
    // aggregation to level+1
    DArray<int> agg, members;
    int ncoarse = 0;
    // V-cycle vectors
    DArray<double> r, z, res, y, zb;
    // performance mode (BCS_MODE_PERF): colour-permuted copy for the smoother
    std::unique_ptr<Level> mc;
    DArray<int> mcPerm;  // new (colour-ordered) row -> row
    DArray<int> mcColorOffD;  // device copy of mcColorOff
    bool colourSweep = false; // this is a coloured copy: colour-synchronous sweeps, no sweep programs
    bool jacobi = false;      // performance mode, block Jacobi: smoothed by omega * D^-1 (no DILU)
    int ncolors = 0;
    std::vector<int> mcColorOff;  // colour c = new rows [off[c], off[c+1])
    bool mcValid = false;  // mc built for the current values
};

// Preconditioner state of one matrix (the serial system or one Mode-R engine)
struct Hier {
    std::vector<Level> levels;  // storage persists across solves; nlev active
    int nlev = 0;
    DArray<double> dense;
    DArray<int> dpiv;
    int m = 0;
    int pcKind = -1;  // 0 none, 1 LUSGS, 2 DILU, 3 AMG
    int tail = -1;    // first level of the one-CTA coarse tail (-1: none)
    DArray<unsigned char> tailDesc;  // TailLevelDev[nlev - tail]
    bcs_solver_config pcCfg{};
    PhaseArena arena;  // DILU scratch (setup phase) / sweep programs + Krylov basis (solve phase)
};

// One Mode-R engine on the device: its consolidated local BSR (local
// numbering, LDU source ids), halo couplings and its own preconditioner.
struct DistPart {
    int rowStart = 0, rows = 0, nnz = 0, nh = 0, nhr = 0;
    DArray<int> ro, ci, src, dg, tpos;
    DArray<double> vals;
    DArray<int> hrow, hoff, hcol, hsrc;  // halo rows (local), CSR offsets, global cols, LDU source ids
    DArray<double> hvals;
    Hier H;
};

// Fine-level matrix a preconditioner is built on
struct FineMatrix {
    int rows = 0, nnz = 0;
    const int *ro = nullptr, *ci = nullptr, *dg = nullptr, *tpos = nullptr;
    const double* v = nullptr;
};

class Engine {
    // Mode R calls borrow n_/nc_/H_ and the operator switches for their Krylov
    // run; this restores the serial system's view on every exit (incl. throws)
    friend struct SerialStateGuard;

public:
    explicit Engine(int device);
    ~Engine();

    void setStream(cudaStream_t s);
    void setKernelTiming(bool on) { kernelTiming_ = on; }

    // topology / values
    void setTopology(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh);
    void uploadLdu(const double* diag, const double* upper, const double* lower, bool device_ptrs);
    // device assembly of the 5x5 density-based system (k_assemble.cu); rhs: host, 5 per cell
    // bkind: PatchKind per boundary face (0 wall .. 5 symmetry) or nullptr (all farfield);
    // recon 0 first order, 1 MUSCL without limiter, 2 MUSCL + Barth-Jespersen (needs faceFx, cellCen);
    // flux: the residual's riemannFlux, 0 Roe, 1 HLLC, 2 Rusanov
    void assembleEuler(int nc, int nf, const int32_t* owner, const int32_t* neigh, const double* faceArea, int nb,
                       const int32_t* bcell, const double* barea, const int32_t* bkind, const double* q,
                       const double* qinf, double cfl, double* rhs, int recon = 0, const double* faceFx = nullptr,
                       const double* cellCen = nullptr, int flux = 0);
    // device assembleCoupled + pinPressure (wall / moving-wall patches); rhs: host, 4 per cell
    void assembleCoupled(int nc, int nf, const int32_t* owner, const int32_t* neigh, const double* faceArea,
                         const double* fx, const double* vol, const double* cen, int nb, const int32_t* bcell,
                         const double* barea, const int32_t* bkind, const double* bu, const double* bp,
                         const double* state, const double* phi, double nu, int pinCell, double pinValue,
                         double* rhs);
    void assemblyTopology(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh);
    // boundary faces grouped per cell (patch order kept): offsets and the permutation
    void assemblyBoundary(int nc, int nb, const int32_t* bcell, std::vector<int>& order);

    // drop-in pipeline (engine.cpp:47-120)
    void pipelineSolve(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh, const double* diag,
                       const double* upper, const double* lower, const double* b, size_t b_len, const double* x0,
                       size_t x0_len, double* x, int backend, const bcs_solver_config& cfg, bcs_report& rep);

    // Mode R: the reference's distributedSolve semantics (partition.cpp:370-479)
    // on this device — ranks decomposed by RCB, consolidated onto engines, one
    // local preconditioner per engine, global Krylov with halo couplings and
    // the fixed engine-order tree for dot products.
    // Mode R with one process per GPU (NCCL, loaded at run time)
    static void commUniqueId(unsigned char id[128]);
    void commInit(int rank, int size, const unsigned char id[128]);
    void distSolveMP(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh, const double* centroids,
                     const double* diag, const double* upper, const double* lower, const double* b, const double* x0,
                     double* x, int nRanks, const bcs_solver_config& cfg, bcs_report& rep);
    // distributedSolve on caller-built rank partitions (bcs_dist_solve_parts)
    void distSolveParts(int nRanks, int n, const int* rankRowOffset, const int* const* localRo,
                        const int* const* localCi, const double* const* localVals, const int* haloCount,
                        const int* const* haloRow, const int* const* haloCol, const int* const* haloPeer,
                        const double* const* haloVals, int nEngines, const int* rankToEngine,
                        const int* engineRowOffset, const double* b, const double* x0, double* x,
                        const bcs_solver_config& cfg, bcs_report& rep);
    void distSolve(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh, const double* centroids,
                   const double* diag, const double* upper, const double* lower, const double* b, const double* x0,
                   double* x, int nRanks, int nEngines, const bcs_solver_config& cfg, bcs_report& rep);

    // staged
    void solveDevice(const double* d_b, double* d_x, const bcs_solver_config& cfg, bcs_report& rep);
    void solveHost(const double* b, double* x, const bcs_solver_config& cfg, bcs_report& rep);

    // queries / kernels
    double residualNorm(const double* b, const double* x);  // host arrays
    const std::vector<double>& history() const { return hist_; }
    void spmvDevice(const double* d_x, double* d_y);
    void spmvHost(const double* x, double* y);
    void csrGet(int32_t* ro, int32_t* ci, double* v);
    void precondSetup(const bcs_solver_config& cfg);
    void precondApplyHost(const double* r, double* z);
    int amgDepth() const { return H_->nlev; }
    void amgLevelSizes(int l, int* rows, int* nnz) const;
    void amgLevelGet(int l, int32_t* ro, int32_t* ci, double* v, int32_t* agg);
    int scheduleDepth(int l) const;
    // performance mode: colours of level l's smoother and its row order
    // (perm[new] = row), 0 when the level is smoothed in natural order
    int levelColoring(int l, int32_t* perm, int32_t* colorOff);

    // device bytes held by this context, per category (JSON object)
    std::string memoryReport() const;

    cudaStream_t stream() const { return stream_; }
    long long totalLaunches() const { return launches_.launches; }
    int blockSize() const { return n_; }
    int nCells() const { return nc_; }

private:
    void requireMatrix() const;
    void validateConfig(const bcs_solver_config& cfg) const;
    void buildPrecond(const bcs_solver_config& cfg);
    void buildPrecondOn(const FineMatrix& F, const bcs_solver_config& cfg);
    FineMatrix serialFine() const;
    void buildHierarchy(const bcs_solver_config& cfg);
    void setupLevelPattern(Level& L);
    void diluSetupAll(const std::vector<Level*>& lv, const bcs_solver_config* cfg);
    void dropArenaViews();
    void finishSmoothers(const std::vector<Level*>& lv, const bcs_solver_config* cfg);
    // performance mode: the colour-permuted copy of L the smoother runs on
    // (k_color.cu), or L itself when the colouring is not possible
    Level* perfLevel(Level& L, const bcs_solver_config& cfg);
    bool buildColoured(Level& L);
    // the levels whose DILU is built: every level but the coarsest, coloured
    // copies in performance mode above the one-CTA tail
    std::vector<Level*> smoothedLevels(const bcs_solver_config& cfg);
    int tailStart() const;
    void jacobiSetup(Level& L);
    void lusgsSetup(Level& L);

    void applyPrecond(const double* r, double* z);
    void smootherApply(Level& L, const double* r, double* z, int accumulate);
    void vcycle(int l, const double* r, double* z);
    void gmres(const double* b, double* x, const bcs_solver_config& cfg, bcs_report& rep);
    void bicgstab(const double* b, double* x, const bcs_solver_config& cfg, bcs_report& rep);
    void spmvLevel(const Level& L, const double* x, const double* sub, double* y);
    // Krylov operators: serial system or Mode-R engines (distActive_)
    void opResidual(const double* x, const double* b, double* r);  // r = b - A x
    void opSpmv(const double* x, double* y);
    void opPrecond(const double* r, double* z);
    void opDot(const double* a, const double* b, double* out, bool sqrt_out);
    void opAxpyDot(double* w, const double* h, const double* v, const double* nextv, double* out);
    std::chrono::steady_clock::time_point distSolveCore(const bcs_solver_config& cfg, bcs_report& rep);
    void distSetupTopology(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh,
                           const double* centroids, int nRanks, int nEngines);
    void mpSetupTopology(int nc, int nf, int n, const int32_t* owner, const int32_t* neigh, const double* centroids,
                         int nRanks);
    void uploadEnginePart(DistPart& P, const Partition& p, int n, const std::vector<int>* hcolOverride);
    void solveKrylov(const double* d_b, double* d_x, const bcs_solver_config& cfg, bcs_report& rep);
    double dotHost(const double* a, const double* b, size_t N, bool sqrt_out);
    void sync();
    void checkErr(const char* where);
    int readErrCell();

    int device_ = 0;
    cudaStream_t own_ = nullptr, stream_ = nullptr;
    bool kernelTiming_ = false;
    bool exactDots_ = false;  // BCS_MODE_EXACT for the current Krylov run
    LaunchCounter launches_;

    // topology
    int nc_ = 0, nf_ = 0, n_ = 0;
    bool hasTopo_ = false, hasValues_ = false;
    std::vector<int32_t> hOwner_, hNeigh_;
    DArray<int> dOwner_, dNeigh_, ro_, ci_, dg_, tpos_, src_, fill_;
    DArray<double> vals_;
    DArray<double> ldu_diag_, ldu_upper_, ldu_lower_;
    // host->device copy of a caller's buffer: straight DMA when it is
    // page-locked, else streamed through a ring of pinned staging chunks filled
    // by several host threads (pageable cudaMemcpyAsync runs at ~11 GB/s)
    void h2d(void* dst, const void* src, size_t bytes, const char* what);
    // device->host counterpart (synchronous: dst is complete on return)
    void d2h(void* dst, const void* src, size_t bytes, const char* what);
    bool hostPinned(const void* p) const;
    void ensureStaging();
    std::vector<void*> stage_;
    std::vector<cudaEvent_t> stageEv_;
    // device assembly: slot of every LDU block, cell -> faces (face order), cell -> boundary faces
    bool asmTopo_ = false;
    DArray<int> asmInv_, asmCfo_, asmCf_, asmBco_, asmBkind_, asmBad_;
    DArray<double> asmMuGrad_, asmPsi_, asmFs_, asmBp_;
    DArray<double> asmArea_, asmBarea_, asmQ_, asmRhs_, asmFx_, asmVol_, asmCen_, asmBu_, asmPhi_, asmD_, asmGrad_;
    // Backend::HostLdu (engine.cpp:54-72): the reference's face-addressed
    // arithmetic on the device -- blockMatvec's order (block_matrix.cpp:104-119:
    // diagonal, then the faces of a row in face order) and LduLusgsPrecond's
    // (preconditioner.cpp:59-99: lower faces in face order forward, upper faces
    // in face order backward) as two slot orders of the same blocks
    bool hlTopo_ = false, hostLdu_ = false;
    DArray<int> hlMvRo_, hlMvCi_, hlMvSrc_, hlGsRo_, hlGsCi_, hlGsSrc_, hlGsDg_;
    DArray<double> hlMvV_, hlGsV_;
    void hostLduTopology();
    void solveHostLdu(const double* b, double* x, const bcs_solver_config& cfg, bcs_report& rep);
    // SolvePipeline state (engine.hpp:35-37): only the EngineCsr branch updates it
    bool pipeHasSetup_ = false;
    uint64_t pipeSig_ = 0;
    bool pipeSigValid_ = false;

    // preconditioner of the serial system; H_ points at the hierarchy being
    // built/applied (the serial one or a Mode-R engine's)
    Hier main_;
    Hier* H_ = &main_;
    // scratch
    DArray<int> chunkOrd_, chainCnt_;  // chain schedules: orders, chain counts / check flags
    DArray<int> partOrd_;              // cluster variant over several clusters: range-major order
    DArray<int> cnt_, lvl_, act2_, push_, scanTmp_, flag_, err_, ctr_, choice_, segOff_, cro_, big_;
    DArray<double> dn_, str_, tblk_;
    DArray<int> dkeys_, dorder_;       // combined DILU tickets
    DArray<int> mcSv_;                 // performance mode: source slot of every permuted slot
    DArray<unsigned char> ddesc_;      // device level descriptors of the combined DILU setup
    DArray<unsigned long long> keys_, sorted_;

    // Krylov workspace
    DArray<double> V_, Z_, w_, zk_, rk_, Hm_, cs_, sn_, g_, y_, scal_, partials_;
    DArray<double> kb_, kx_;  // staging for host-array entry points
    DArray<double> bp_, bv_, bs_, bt_, bph_, bsh_, brh_;
    DArray<int> ticket_;
    double* hStatus_ = nullptr;  // pinned
    std::vector<double> hist_;

    // SpMV event timing (fine level)
    void collectSpmvTimes();
    // Mode R state
    bool distActive_ = false;
    // multi-process Mode R
    void* comm_ = nullptr;  // ncclComm_t
    int mpRank_ = 0, mpSize_ = 1;
    bool mpActive_ = false;
    int mpBps_ = 0, mpRows_ = 0, mpSendRows_ = 0, mpRecvRows_ = 0, mpMaxRows_ = 0;
    std::vector<int> mpSendCnt_, mpRecvCnt_, mpEngStart_, mpEngRows_;
    DArray<int> mpSendIdx_;
    DArray<double> mpSend_, mpRecv_, mpPart_, mpGath_, mpXall_;
    int mpRanks_ = 0, mpNc_ = 0, mpNf_ = 0, mpN_ = 0;
    std::vector<int32_t> mpOwner_, mpNeigh_;
    std::vector<double> mpCen_;
    std::vector<int> mpNewToOld_;
    void mpExchange(const double* x);
    Partition mpPart;                  // this process's engine (host slot sources)
    double* mpStage_ = nullptr;        // pinned per-rank upload staging
    size_t mpStageCap_ = 0;
    cudaStream_t commStream_ = nullptr;
    cudaEvent_t mpEvPack_ = nullptr, mpEvComm_ = nullptr;
    std::vector<DistPart> dist_;
    std::vector<int32_t> distOwner_, distNeigh_;
    std::vector<double> distCen_;
    int distRanks_ = 0, distEngines_ = 0, distNc_ = 0, distNf_ = 0, distN_ = 0;
    std::vector<int> distNewToOld_;
    DArray<long long> seg_;  // segment offsets for reductions (1 segment serial, E for Mode R)
    std::vector<long long> distSegh_;  // the one-device Mode R engines' segments
    int nseg_ = 1;
    DArray<double> distTmp_;
    // BCS_PROFILE=1: per-phase / per-level wall times (with syncs) to stderr
    bool prof_ = false;
    int aggMode_ = 0;   // 0 sync-free aggregation, 1 cooperative rounds
    int diluMode_ = 0;  // 0 sync-free level-ordered DILU setup, 1 Kahn levels
    int denseBlockedMin_ = kDenseBlockedMin;  // coarsest m from which the blocked dense LU/solve run
    int tailMaxRows_ = kTailMaxRows;          // levels at most this big run in the one-CTA tail (0: off)
    int denseTiledMin_ = 2048;                // coarsest m from which the backward solve is tiled (non-EXACT)
    bool mcSweep_ = false;                    // perf mode: colour-synchronous sweeps (BCS_MC_SWEEP=1; measured slower)
    int mcLaunchMin_ = 16384;  // performance mode: rows per colour (mean) for one launch per colour
    double jacobiOmega_ = 0.8;                // block-Jacobi damping (of 0.8 / 0.9 / 1.0: 18 / 22 / 94 its at 128^3); BCS_JACOBI_OMEGA
    void denseSolve(const double* r, double* z);
    int* hTot_ = nullptr;                     // pinned: per-level sweep program sizes
    void setupTail();
    std::vector<std::pair<std::string, double>> profRec_;
    std::chrono::steady_clock::time_point profT_;
    void profMark(const std::string& what);
    bool sameFaces(const int32_t* owner, const int32_t* neigh, int nf) const;
    void profDump();
    cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evPool_;
    size_t evUsed_ = 0;
    int lastSolveLaunches_ = 0;
    double spmvMs_ = 0.0;
    int spmvCount_ = 0;
    std::vector<int> evKind_;      // 0: fine-level SpMV, 1: sweep (any level)
    std::vector<double> evBytes_;  // algorithmic bytes of the timed launch
    double sweepMs_ = 0.0, sweepBytes_ = 0.0;
    int sweepCount_ = 0;
    void timerBegin();
    void timerEnd(int kind, double bytes);
};

struct SerialStateGuard {
    Engine& e;
    int nc, n, nseg;
    explicit SerialStateGuard(Engine& en) : e(en), nc(en.nc_), n(en.n_), nseg(en.nseg_) {}
    ~SerialStateGuard() {
        e.nc_ = nc;
        e.n_ = n;
        e.nseg_ = nseg;
        e.H_ = &e.main_;
        e.distActive_ = false;
        e.mpActive_ = false;
    }
};

}  // namespace bcs
