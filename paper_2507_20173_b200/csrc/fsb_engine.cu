// fsb_engine.cu -- host runtime behind the C-ABI (include/fsb_b200.h).
//
// One engine owns one shard of the school on one GPU: SoA state in HBM, a
// non-blocking stream, the reduction workspace, cached CUDA graphs of the
// fused step loop, and (world_size > 1) an NCCL communicator used for the one
// per-step exchange of {max(prev-cur), sum x*f, sum y*f, sum f}.
//
// Replaces, for this path, the reference's parfor::Executor dispatch
// (executor.hpp:63-103, 130-159): no host thread touches fish state.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <cstdlib>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/fsb_b200.h"
#include "fsb_kernels.cuh"

using fsb_dev::Partial;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    const int code = (e == cudaErrorMemoryAllocation) ? FSB_ERR_OUT_OF_MEMORY : FSB_ERR_CUDA;
    g_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    cudaGetLastError();  // clear sticky-free errors
    return code;
}

#define CU(call)                                          \
    do {                                                  \
        cudaError_t _e = (call);                          \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

#define TRY(call)                 \
    do {                          \
        int _rc = (call);         \
        if (_rc != FSB_OK) return _rc; \
    } while (0)

// ---- NCCL, loaded on demand (only world_size > 1 needs it) -----------------
struct NcclApi {
    bool tried = false;
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

std::mutex g_nccl_mu;
NcclApi g_nccl;

int nccl_load() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.handle) return FSB_OK;
    if (g_nccl.tried) return fail(FSB_ERR_NCCL, "libnccl.so.2 could not be loaded");
    g_nccl.tried = true;
    // FSB_NCCL_LIB names the library explicitly.  The Python layer points it
    // at the NCCL torch itself links, so whichever of the two loads first,
    // both resolve libnccl.so.2 to the same file; otherwise an already-loaded
    // NCCL is reused through its soname, else the system one is loaded.
    void* h = nullptr;
    const char* path = std::getenv("FSB_NCCL_LIB");
    if (path && *path) {
        h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
        if (!h) return fail(FSB_ERR_NCCL, std::string("dlopen FSB_NCCL_LIB failed: ") + dlerror());
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return fail(FSB_ERR_NCCL, std::string("dlopen libnccl.so.2 failed: ") + dlerror());
    g_nccl.GetUniqueId = reinterpret_cast<decltype(g_nccl.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    g_nccl.CommInitRank = reinterpret_cast<decltype(g_nccl.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    g_nccl.CommDestroy = reinterpret_cast<decltype(g_nccl.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    g_nccl.AllGather = reinterpret_cast<decltype(g_nccl.AllGather)>(dlsym(h, "ncclAllGather"));
    g_nccl.GetErrorString =
        reinterpret_cast<decltype(g_nccl.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.CommDestroy || !g_nccl.AllGather ||
        !g_nccl.GetErrorString)
        return fail(FSB_ERR_NCCL, "libnccl.so.2 lacks a required symbol");
    g_nccl.handle = h;
    return FSB_OK;
}

int nccl_fail(ncclResult_t r, const char* what) {
    return fail(FSB_ERR_NCCL, std::string(what) + ": " +
                                  (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error"));
}

constexpr uint64_t kStagingFish = 1ull << 22;  // 160 MB AoS staging per chunk
// Shards from this size take step_kernel_dyn.  Round 1 measured it ahead of
// the static chunks only from 3e6 fish; with the unguarded full-group loop it
// is 8-20 % faster at every size from 2e4 to 3e6 as well (1e6: 16.9 vs 21.0 us,
// 2.75e6: 33.4 vs 39.8; profiles/round2_ab_dyn_vs_static.jsonl), so it is the
// stream strategy's kernel at every size; FSB_FLAG_STATIC_TILES pins the other.
constexpr uint64_t kDynamicMinFish = 0;

struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    double* d_trace = nullptr;
    double* d_bary = nullptr;
    uint64_t launches = 0;
};

}  // namespace

struct fsb_engine {
    fsb_sim_config cfg{};
    int device = 0;
    int rank = 0;
    int world = 1;
    bool host_xchg = false;   // FSB_FLAG_HOST_EXCHANGE: the caller gathers the rank partials
    bool xchg_ready = true;   // host exchange: every rank's partial of the current state is set
    int strategy = FSB_STRATEGY_AUTO;
    unsigned flags = 0;
    bool use_nccl = false;
    uint64_t first = 0;  // global index of local fish 0
    uint64_t count = 0;  // local fish

    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    fsb_dev::SoA s{};       // s.c stays nullptr in the engine's canonical state
    double* c_buf = nullptr;  // explicit current_objective (only after an inconsistent upload)
    bool cur_explicit = false;
    bool cfg_in_range = false;  // configuration inside the in-range mode's bounds
    bool state_sane = false;    // ... and the state too (set by init / upload, kept by every step)
    bool max_valid = false;  // part_all[cur_buf] holds the partials of the current state
    bool sums_valid = true;  // ... including the barycentre sums (not after a max-only run)
    int cur_buf = 0;

    Partial* part_all = nullptr;  // [2][world]
    Partial* block_part = nullptr;
    // split fold of one-rank graph chains (fsb_kernels.cuh FastFold): three rotating key slots and
    // two CTA-partial buffers of block_cap entries each
    unsigned long long* ff_keys = nullptr;
    Partial* ff_part = nullptr;
    bool ff_enabled = true;  // off with FSB_FLAG_LAST_CTA_FOLD (or FSB_NO_SPLIT_FOLD=1 in the environment: A/B runs)
    unsigned* counter = nullptr;
    uint64_t* d_step0 = nullptr;  // [2]: first step of the launched graph, exchange epoch base
    uint64_t* h_step0 = nullptr;  // pinned [2], copied by each graph's first node
    double* d_scalar = nullptr;   // [4]
    int* d_mismatch = nullptr;
    int grid = 0;            // grid of the compact-state step kernel in use
    int grid_auto = 0;       // ... as chosen at creation (SMs x occupancy)
    int block_cap = 0;       // capacity of block_part (CTA partials)
    int grid_explicit = 0;   // grid of the explicit-cur step kernel
    int grid_aux = 0;        // grid of the eat / reduce kernels (SMs x occupancy, 256 threads)
    bool use_dyn = false;    // compact LDG step: step_kernel_dyn (one CTA per SM, claimed tiles)
    bool use_ws = false;     // compact step: step_kernel_ws (TMA producer warp, 31 consumer warps per SM)
    unsigned tile_groups = 0;  // claimed-tile kernel: minimum groups per tile (0 = the kernel's default)
    int grid_coop = 0;       // grid of the cooperative persistent grid kernel
    unsigned long long* d_gen = nullptr;     // grid-kernel arrival counter
    int cgrid_nc = 0;                        // co-resident clusters of the cluster-reduced grid kernel (0: none)
    double* d_cl_slots = nullptr;            // [kSlotRing][cgrid_nc][kSlotWords]
    bool use_bulk = false;   // compact step streams through the cp.async.bulk ring
    unsigned sg_cap = 0;     // shared-memory-resident grid: fish pairs per CTA (0: unavailable)
    int sg_grid = 0;         // ... its CTAs (one per SM)
    unsigned long long* d_sg_keys = nullptr;  // [3] per-step max keys of the shared-memory grid

    void* staging = nullptr;  // device AoS staging (two halves of kStagingFish / 2 fish: double-buffered transfers)
    cudaStream_t xfer = nullptr;        // copy stream of upload / download (overlaps the transposes)
    cudaEvent_t ev_half[2][2] = {};     // per staging half: [0] copy done, [1] transpose done
    void* pinned = nullptr;   // host pinned staging (checksum)
    double* d_cl_trace = nullptr;  // persistent-kernel trace buffers
    double* d_cl_bary = nullptr;
    uint64_t cl_cap = 0;
    uint64_t last_launches = 0;
    int last_strategy = FSB_STRATEGY_AUTO;  // strategy the last run executed
    std::string fallback;                   // why the last AUTO run left its first choice ("" = it did not)
    fsb_dev::EatClock* eclk = nullptr;      // eat-region clock (device)
    double last_eat_s = 0.0;                // eat region of the last run / eat call

    std::map<std::pair<uint64_t, int>, GraphEntry> graphs;  // (T, explicit_first | sane << 1)
    ncclComm_t comm = nullptr;

    // peer exchange (FSB_FLAG_PEER_EXCHANGE)
    bool peer_mode = false;
    bool peer_connected = false;
    fsb_dev::PeerWindow* window = nullptr;   // this rank's window (IPC-exported)
    fsb_dev::PeerWindow** d_peers = nullptr;  // [world] device array of mapped windows
    std::vector<void*> opened;               // IPC mappings to close
    uint64_t xseq = 0;                       // exchanges completed (epoch of the latest)
    unsigned long long peer_timeout_ns = 60000000000ull;  // a kernel's wait for the other ranks' partials
};

namespace {

fsb_dev::Scalars scalars_of(const fsb_sim_config& c) {
    fsb_dev::Scalars k;
    k.pond = c.pond_size;
    k.half_pond = c.pond_size / 2.0;
    k.step_base = c.step_base;
    k.w_max = 2.0 * c.weight_scale;  // SimConfig::weight_max (sim.hpp:42)
    k.seed = c.seed;
    k.zero = 0;
    return k;
}

fsb_dev::SoA canonical(const fsb_engine* e) {
    fsb_dev::SoA s = e->s;
    s.c = e->cur_explicit ? e->c_buf : nullptr;
    return s;
}

Partial* local_part(fsb_engine* e, int buf) { return e->part_all + buf * e->world + e->rank; }
Partial* all_part(fsb_engine* e, int buf) { return e->part_all + buf * e->world; }

int exchange(fsb_engine* e, int buf) {
    if (!e->use_nccl) return FSB_OK;
    // in place: send = recv + rank * count
    ncclResult_t r = g_nccl.AllGather(local_part(e, buf), all_part(e, buf), 4, ncclFloat64, e->comm,
                                      e->stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
    return FSB_OK;
}

// Eat-region clock links (fsb_kernels.cuh EatClock).
fsb_dev::EatLink ec_link(const fsb_engine* e, int out_slot, int in_slot, int phase) {
    fsb_dev::EatLink l{};
    l.out = out_slot >= 0 ? &e->eclk->s[out_slot] : nullptr;
    l.in = in_slot >= 0 ? &e->eclk->s[in_slot] : nullptr;
    l.ns = &e->eclk->ns;
    l.phase = phase;
    return l;
}

int read_eat_ns(fsb_engine* e, double divisor, double* seconds) {
    unsigned long long ns = 0;
    CU(cudaMemcpyAsync(&ns, &e->eclk->ns, sizeof ns, cudaMemcpyDeviceToHost, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    *seconds = (double)ns * 1e-9 / (divisor > 0 ? divisor : 1.0);
    return FSB_OK;
}

// Persistent kernels: per-CTA SM cycles summed in ns, CTA 0's globaltimer /
// clock64 brackets convert them; mean over the `ctas` CTAs.
int read_eat_cycles(fsb_engine* e, double ctas, double* seconds) {
    fsb_dev::EatClock c{};
    CU(cudaMemcpyAsync(&c, e->eclk, sizeof c, cudaMemcpyDeviceToHost, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    const double ns_per_cycle =
        (c.c1 > c.c0 && c.g1 > c.g0) ? (double)(c.g1 - c.g0) / (double)(c.c1 - c.c0) : 0.0;
    *seconds = (double)c.ns * ns_per_cycle * 1e-9 / (ctas > 0 ? ctas : 1.0);
    return FSB_OK;
}

// Fault injection for the AUTO fallback tests: FSB_FAULT_INJECT names the
// launches that should be refused as if the device could not co-schedule them
// ("grid", "persistent"; comma-separated).  Read at every launch.
bool fault_injected(const char* what) {
    const char* v = std::getenv("FSB_FAULT_INJECT");
    return v && *v && std::strstr(v, what) != nullptr;
}

// Launch errors that mean "this device cannot co-schedule the persistent
// grid / cluster right now" (a profiler replay, MPS, a shared or partitioned
// device): AUTO then runs the graph of step kernels instead.
bool co_schedule_refused(cudaError_t ce) {
    return ce == cudaErrorCooperativeLaunchTooLarge || ce == cudaErrorNotSupported ||
           ce == cudaErrorInvalidClusterSize || ce == cudaErrorLaunchOutOfResources ||
           ce == cudaErrorNotPermitted;
}

// NVTX ranges around every public entry point (tracing): an
// nsys / ncu --nvtx timeline shows init / upload / run / move / eat / download
// per rank.  Header-only NVTX v3: without an attached tool a range is one
// predicted branch.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define FSB_NVTX(name) NvtxRange fsb_nvtx_range_(name)

int guard(fsb_engine* e) {
    if (!e) return fail(FSB_ERR_INVALID_ARGUMENT, "null engine");
    CU(cudaSetDevice(e->device));
    return FSB_OK;
}

int ensure_staging(fsb_engine* e) {
    if (!e->staging) CU(cudaMalloc(&e->staging, kStagingFish * sizeof(fsb_fish)));
    if (!e->xfer) {
        CU(cudaStreamCreateWithFlags(&e->xfer, cudaStreamNonBlocking));
        for (auto& h : e->ev_half)
            for (auto& v : h) CU(cudaEventCreateWithFlags(&v, cudaEventDisableTiming));
    }
    return FSB_OK;
}

int elapsed(fsb_engine* e, double* seconds) {
    CU(cudaEventSynchronize(e->ev1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    if (seconds) *seconds = ms * 1e-3;
    return FSB_OK;
}

// The kernels' view of the peer exchange: epochs base + in_add / base + out_add
// with base = *seq_ptr (graph) or 0 (eager launches pass absolute epochs).
fsb_dev::PeerXchg px_of(const fsb_engine* e, const uint64_t* seq_ptr, uint64_t in_add, uint64_t out_add) {
    fsb_dev::PeerXchg px{};
    if (!e->peer_mode) return px;
    px.peers = e->d_peers;
    px.local = e->window;
    px.rank = e->rank;
    px.seq_ptr = seq_ptr;
    px.in_add = in_add;
    px.out_add = out_add;
    px.timeout_ns = e->peer_timeout_ns;
    return px;
}

int need_peers(const fsb_engine* e) {
    if (e->peer_mode && !e->peer_connected)
        return fail(FSB_ERR_INVALID_ARGUMENT, "peer exchange not connected (fsb_engine_peer_connect)");
    return FSB_OK;
}

// Host exchange with more than one rank: the caller's partials must be in place.
bool host_multi(const fsb_engine* e) { return e->host_xchg && e->world > 1; }

// Peer exchange failure detection: a kernel that waited longer than the
// device-side timeout for another rank's partial marked its window (the call's
// results are void).  Checked after every call that consumes partials.
int peer_fault(fsb_engine* e) {
    if (!e->peer_mode || !e->window) return FSB_OK;
    unsigned long long f = 0;
    CU(cudaMemcpy(&f, &e->window->fault, sizeof f, cudaMemcpyDeviceToHost));
    if (!f) return FSB_OK;
    CU(cudaMemset(&e->window->fault, 0, sizeof f));
    return fail(FSB_ERR_NCCL, "peer exchange: the partials of epoch " + std::to_string(f) +
                                  " did not all arrive (a rank stopped publishing); results void");
}

int need_partials(const fsb_engine* e) {
    if (host_multi(e) && !e->xchg_ready)
        return fail(FSB_ERR_INVALID_ARGUMENT, "host exchange: fsb_engine_set_partials before eat/barycentre");
    return FSB_OK;
}

int phase_only(const fsb_engine* e, const char* what) {
    if (host_multi(e))
        return fail(FSB_ERR_UNSUPPORTED, std::string("host exchange: ") + what +
                                             " needs a per-step exchange (NCCL or peer); use move/eat");
    return FSB_OK;
}

bool want_persistent(const fsb_engine* e) {
    if (e->world != 1 || e->use_nccl || e->peer_mode) return false;
    if (e->strategy == FSB_STRATEGY_PERSISTENT) return true;
    if (e->strategy == FSB_STRATEGY_STREAM) return false;
    return e->count > 0 && e->count <= 16384;
}

// FSB_STRATEGY_GRID, and AUTO for single-rank schools that fit in shared memory
// (fits_sgrid: about 1.06e6 fish).  Above that AUTO runs the graph of step
// kernels: in round 1 the L2 cluster grid was 3-13 % faster than the graph up to
// 2e6 fish (profiles/r03_ab_grid.jsonl); with the split fold and the pre-wait
// prologue the graph is 0.5-7 % faster from 1.1e6 to 2.5e6
// (profiles/round2_ab_graph_vs_l2_grid.jsonl).  With FSB_FLAG_L2_GRID or
// FSB_FLAG_FLAT_GRID, AUTO still takes the grid up to this size.
constexpr uint64_t kGridAutoMaxFish = 2500000;

// The shared-memory-resident grid kernel holds the school on chip: every CTA's
// pair range must fit its shared memory (about 1.06e6 fish on 148 SMs).
bool fits_sgrid(const fsb_engine* e) {
    if (!e->sg_cap || (e->flags & (FSB_FLAG_L2_GRID | FSB_FLAG_FLAT_GRID))) return false;
    const uint64_t npairs = e->count >> 1;
    const uint64_t per_cta = (npairs + e->sg_grid - 1) / e->sg_grid;
    return per_cta <= e->sg_cap;
}

// Nsight Compute (and other CUDA tool injections) cannot replay a cooperative
// launch of thread-block clusters: it terminates the process instead of
// returning an error.  With a tool injected, that launch is treated as refused.
bool tool_injected() {
    const char* v = std::getenv("CUDA_INJECTION64_PATH");
    return v && *v;
}

bool want_grid(const fsb_engine* e) {
    if (e->cur_explicit || e->world != 1 || e->use_nccl || e->peer_mode) return false;
    if (e->strategy == FSB_STRATEGY_GRID) return true;
    const bool asked_l2 = (e->flags & (FSB_FLAG_L2_GRID | FSB_FLAG_FLAT_GRID)) && e->count <= kGridAutoMaxFish;
    return e->strategy == FSB_STRATEGY_AUTO && e->cgrid_nc > 0 && e->count > 16384 && (fits_sgrid(e) || asked_l2) &&
           !(e->flags & (FSB_FLAG_FORCE_BULK | FSB_FLAG_DYNAMIC_TILES | FSB_FLAG_STATIC_TILES));
}

void free_graphs(fsb_engine* e) {
    for (auto& kv : e->graphs) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        if (kv.second.d_trace) cudaFree(kv.second.d_trace);
        if (kv.second.d_bary) cudaFree(kv.second.d_bary);
    }
    e->graphs.clear();
}

// In-range mode (fsb_math.cuh): the step kernels skip the fp64 operand guards.
// The bounds hold for every state init produces and are preserved by every
// step; an upload re-establishes them by check.
bool config_in_range(const fsb_sim_config& c) {
    return c.pond_size >= 0x1p-400 && c.pond_size <= 0x1p500 && c.step_base >= 0x1p-400 &&
           c.step_base <= 0x1p500 && c.weight_scale <= 0x1p500;
}

bool in_range(const fsb_engine* e) { return e->state_sane && !(e->flags & FSB_FLAG_CHECKED); }

fsb_dev::StepArgs step_args(fsb_engine* e, const fsb_dev::SoA& s) {
    fsb_dev::StepArgs a{};
    a.s = s;
    a.k = scalars_of(e->cfg);
    a.n = e->count;
    a.gfirst = e->first;
    a.world = e->world;
    a.ws.block_part = e->block_part;
    a.ws.counter = e->counter;
    a.ws.cap = (unsigned)e->block_cap;
    a.alternate = (e->flags & FSB_FLAG_NO_ALTERNATE) ? 0 : 1;
    a.bulk = e->use_bulk ? 1 : 0;
    a.dyn = e->use_dyn ? 1 : 0;
    a.wspec = e->use_ws ? 1 : 0;
    a.tile_groups = e->tile_groups;
    a.sane = in_range(e) ? 1 : 0;
    return a;
}

// Capture: step kernel k (k = 0..T-1) applies the deferred eat of step k-1,
// moves step first+k and publishes its partial; NCCL allgathers it; a final
// eat kernel applies step T-1's eat.  The first step index is read at run time
// from d_step0 (filled by the graph's first node from pinned memory), so one
// graph serves every first_step.
// Programmatic Dependent Launch between consecutive step kernels of a graph:
// not across an NCCL exchange (its kernel does not release dependents early).
bool use_pdl(const fsb_engine* e) { return !e->use_nccl && !(e->flags & FSB_FLAG_NO_PDL); }

int build_graph(fsb_engine* e, uint64_t T, bool explicit_first, GraphEntry* out) {
    GraphEntry g;
    CU(cudaMalloc(&g.d_trace, T * sizeof(double)));
    CU(cudaMalloc(&g.d_bary, 3 * T * sizeof(double)));
    CU(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
    int rc = FSB_OK;
    cudaError_t ce = cudaMemcpyAsync(e->d_step0, e->h_step0, 2 * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                     e->stream);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(&e->eclk->ns, 0, sizeof(unsigned long long), e->stream);
    // One rank, the claimed-tile kernel, no peer / host exchange: the split fold (FastFold).
    const bool split = e->ff_enabled && T >= 1 && e->world == 1 && !e->use_nccl && !e->peer_mode && !e->host_xchg &&
                       e->use_dyn && !e->use_ws && !e->use_bulk;
    if (split && ce == cudaSuccess) ce = cudaMemsetAsync(e->ff_keys, 0, 3 * sizeof(unsigned long long), e->stream);
    auto grid_of = [&](uint64_t k) { return (k == 0 && explicit_first) ? e->grid_explicit : e->grid; };
    auto consume = [&](fsb_dev::FastFold& ff, uint64_t k) {  // the consumer of step k's partials
        ff.key_in = e->ff_keys + k % 3;
        ff.bp_in = e->ff_part + (k & 1) * (size_t)e->block_cap;
        ff.bp_in_count = (unsigned)grid_of(k);
        ff.fold_out = local_part(e, (int)(k & 1));
    };
    uint64_t launches = 0;
    for (uint64_t k = 0; k < T && ce == cudaSuccess && rc == FSB_OK; ++k) {
        fsb_dev::SoA s = e->s;
        s.c = (k == 0 && explicit_first) ? e->c_buf : nullptr;
        fsb_dev::StepArgs a = step_args(e, s);
        a.step_ptr = e->d_step0;
        a.step_add = k;
        a.part_in = k ? all_part(e, (int)((k - 1) & 1)) : nullptr;
        a.trace_out = k ? g.d_trace + (k - 1) : nullptr;
        a.bary_out = k ? g.d_bary + 3 * (k - 1) : nullptr;
        a.part_out = local_part(e, (int)(k & 1));
        a.px = px_of(e, e->d_step0 + 1, k, k + 1);  // consumes epoch base+k, produces base+k+1
        a.pdl = (k > 0 && use_pdl(e)) ? 1 : 0;  // kernel -> kernel edges only
        a.ec = ec_link(e, (int)(k & 1), k ? (int)((k - 1) & 1) : -1, 0);
        if (split) {
            a.ff.key_out = e->ff_keys + k % 3;
            a.ff.bp_out = e->ff_part + (k & 1) * (size_t)e->block_cap;
            if (k) {
                consume(a.ff, k - 1);
                a.ff.key_reset = e->ff_keys + (k + 1) % 3;
            }
        }
        ce = fsb_dev::launch_step(a, (k == 0 && explicit_first) ? e->grid_explicit : e->grid, e->stream);
        ++launches;
        if (ce == cudaSuccess) rc = exchange(e, (int)(k & 1));
    }
    if (ce == cudaSuccess && rc == FSB_OK) {
        fsb_dev::EatArgs ea{};
        ea.s = e->s;
        ea.s.c = (T == 0 && explicit_first) ? e->c_buf : nullptr;
        ea.k = scalars_of(e->cfg);
        ea.n = e->count;
        ea.part_in = all_part(e, (int)((T - 1) & 1));
        ea.world = e->world;
        ea.trace_out = g.d_trace + (T - 1);
        ea.bary_out = g.d_bary + 3 * (T - 1);
        ea.px = px_of(e, e->d_step0 + 1, T, 0);
        ea.pdl = use_pdl(e) ? 1 : 0;
        ea.ec = ec_link(e, -1, (int)((T - 1) & 1), 0);
        if (split) consume(ea.ff, T - 1);
        ce = fsb_dev::launch_eat(ea, e->grid_aux, e->stream);
        ++launches;
    }
    cudaGraph_t graph = nullptr;
    cudaError_t ee = cudaStreamEndCapture(e->stream, &graph);
    if (ce != cudaSuccess) return cuda_fail(ce, "capture step loop");
    if (rc != FSB_OK) return rc;
    if (ee != cudaSuccess) return cuda_fail(ee, "cudaStreamEndCapture");
    ee = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ee != cudaSuccess) return cuda_fail(ee, "cudaGraphInstantiate");
    // upload the executable graph now, not as part of its first (timed) launch
    ee = cudaGraphUpload(g.exec, e->stream);
    if (ee != cudaSuccess) return cuda_fail(ee, "cudaGraphUpload");
    g.launches = launches;
    *out = g;
    return FSB_OK;
}

int run_stream(fsb_engine* e, uint64_t first_step, uint64_t T, double* trace, double* bary,
               double* seconds) {
    FSB_NVTX("run_stream: graph of fused step kernels");
    const auto key = std::make_pair(T, (e->cur_explicit ? 1 : 0) | (in_range(e) ? 2 : 0));
    auto it = e->graphs.find(key);
    if (it == e->graphs.end()) {
        if (e->graphs.size() >= 16) free_graphs(e);  // bound the cache (distinct step counts)
        GraphEntry g;
        TRY(build_graph(e, T, e->cur_explicit, &g));
        it = e->graphs.emplace(key, g).first;
    }
    e->h_step0[0] = first_step;
    e->h_step0[1] = e->xseq;  // exchange epoch base of this launch
    CU(cudaEventRecord(e->ev0, e->stream));
    CU(cudaGraphLaunch(it->second.exec, e->stream));
    CU(cudaEventRecord(e->ev1, e->stream));
    if (trace) CU(cudaMemcpyAsync(trace, it->second.d_trace, T * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    if (bary) CU(cudaMemcpyAsync(bary, it->second.d_bary, 3 * T * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    TRY(peer_fault(e));
    TRY(elapsed(e, seconds));
    TRY(read_eat_ns(e, 1.0, &e->last_eat_s));
    e->cur_explicit = false;
    e->max_valid = e->sums_valid = true;
    e->cur_buf = (int)((T - 1) & 1);
    e->last_launches = it->second.launches;
    e->xseq += T;  // one exchange per step kernel
    return FSB_OK;
}

int ensure_run_buffers(fsb_engine* e, uint64_t T) {
    if (T <= e->cl_cap) return FSB_OK;
    if (e->d_cl_trace) cudaFree(e->d_cl_trace);
    if (e->d_cl_bary) cudaFree(e->d_cl_bary);
    e->d_cl_trace = e->d_cl_bary = nullptr;
    e->cl_cap = 0;
    CU(cudaMalloc(&e->d_cl_trace, T * sizeof(double)));
    CU(cudaMalloc(&e->d_cl_bary, 3 * T * sizeof(double)));
    e->cl_cap = T;
    return FSB_OK;
}

// FSB_STRATEGY_GRID: one cooperative launch runs all T steps (compact state,
// single rank), then the trace comes back.
size_t cl_slot_bytes(const fsb_engine* e) {
    return (size_t)fsb_dev::kSlotRing * e->cgrid_nc * fsb_dev::kSlotWords * sizeof(double);
}

int run_grid(fsb_engine* e, uint64_t first_step, uint64_t T, double* trace, double* bary, double* seconds) {
    FSB_NVTX("run_grid: cooperative grid kernel");
    if (e->cur_explicit || e->world != 1 || e->use_nccl || e->peer_mode)
        return fail(FSB_ERR_UNSUPPORTED, "grid strategy: single rank, compact state only");
    TRY(ensure_run_buffers(e, T));
    fsb_dev::StepArgs base = step_args(e, canonical(e));
    base.part_out = local_part(e, 0);
    CU(cudaMemsetAsync(e->eclk, 0, sizeof(fsb_dev::EatClock), e->stream));
    int ctas = 0;
    bool sums = true;  // the run leaves the barycentre sums of the last step in part_out
    cudaError_t ce = cudaSuccess;
    if (fits_sgrid(e)) {
        // the school on chip: one CTA per SM holds its pairs in shared memory for all T steps
        fsb_dev::SGridArgs g{};
        g.base = base;
        g.first_step = first_step;
        g.num_steps = T;
        g.trace = e->d_cl_trace;
        g.bary = bary ? e->d_cl_bary : nullptr;
        g.pair_cap = e->sg_cap;
        g.eclk = e->eclk;
        g.gen = e->d_gen;
        g.parts = e->block_part;  // block_cap >= 2 x grid_coop >= 2 x SMs
        g.keys = e->d_sg_keys;
        CU(cudaMemsetAsync(e->d_gen, 0, sizeof(unsigned long long), e->stream));
        CU(cudaMemsetAsync(e->d_sg_keys, 0, 3 * sizeof(unsigned long long), e->stream));
        CU(cudaEventRecord(e->ev0, e->stream));
        ce = fault_injected("grid") ? cudaErrorCooperativeLaunchTooLarge
                                    : fsb_dev::launch_sgrid_run(g, e->sg_grid, e->stream);
        ctas = e->sg_grid;
        sums = bary != nullptr;  // max-only reduction unless the barycentre trace is wanted
    } else if (e->cgrid_nc > 0) {
        // clusters of 8 CTAs reduce over DSMEM; leaders meet through sentinel slots
        fsb_dev::CGridArgs g{};
        g.base = base;
        g.first_step = first_step;
        g.num_steps = T;
        g.trace = e->d_cl_trace;
        g.bary = bary ? e->d_cl_bary : nullptr;
        g.cl_slots = e->d_cl_slots;
        g.eclk = e->eclk;
        CU(cudaMemsetAsync(e->d_cl_slots, 0xFF, cl_slot_bytes(e), e->stream));  // every word the sentinel
        CU(cudaEventRecord(e->ev0, e->stream));
        ce = (fault_injected("grid") || tool_injected()) ? cudaErrorNotSupported
                                                         : fsb_dev::launch_cgrid_run(g, e->cgrid_nc, e->stream);
        ctas = e->cgrid_nc * fsb_dev::kCGridCluster;
    } else {
        fsb_dev::GridArgs g{};
        g.base = base;
        g.first_step = first_step;
        g.num_steps = T;
        g.trace = e->d_cl_trace;
        g.bary = bary ? e->d_cl_bary : nullptr;
        g.gen = e->d_gen;
        g.eclk = e->eclk;
        CU(cudaMemsetAsync(e->d_gen, 0, sizeof(unsigned long long), e->stream));
        CU(cudaEventRecord(e->ev0, e->stream));
        ce = fault_injected("grid") ? cudaErrorCooperativeLaunchTooLarge
                                    : fsb_dev::launch_grid_run(g, e->grid_coop, e->stream);
        ctas = e->grid_coop;
    }
    if (ce != cudaSuccess) {
        cudaGetLastError();  // launch-configuration errors are not sticky
        const int code = co_schedule_refused(ce) ? FSB_ERR_UNSUPPORTED : FSB_ERR_CUDA;
        return fail(code, std::string("grid strategy: cooperative launch refused: ") + cudaGetErrorName(ce));
    }
    CU(cudaEventRecord(e->ev1, e->stream));
    if (trace) CU(cudaMemcpyAsync(trace, e->d_cl_trace, T * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    if (bary) CU(cudaMemcpyAsync(bary, e->d_cl_bary, 3 * T * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    TRY(elapsed(e, seconds));
    TRY(read_eat_cycles(e, (double)ctas, &e->last_eat_s));
    e->max_valid = true;
    e->sums_valid = sums;
    e->cur_buf = 0;
    e->last_launches = 1;
    e->last_strategy = FSB_STRATEGY_GRID;
    return FSB_OK;
}

int run_persistent(fsb_engine* e, uint64_t first_step, uint64_t T, double* trace, double* bary,
                   double* seconds) {
    FSB_NVTX("run_persistent: persistent cluster kernel");
    if (T > e->cl_cap) {
        if (e->d_cl_trace) cudaFree(e->d_cl_trace);
        if (e->d_cl_bary) cudaFree(e->d_cl_bary);
        e->d_cl_trace = e->d_cl_bary = nullptr;
        e->cl_cap = 0;
        CU(cudaMalloc(&e->d_cl_trace, T * sizeof(double)));
        CU(cudaMalloc(&e->d_cl_bary, 3 * T * sizeof(double)));
        e->cl_cap = T;
    }
    fsb_dev::ClusterArgs a{};
    a.s = canonical(e);
    a.k = scalars_of(e->cfg);
    a.n = e->count;
    a.gfirst = e->first;
    a.first_step = first_step;
    a.num_steps = T;
    a.trace = e->d_cl_trace;
    a.bary = bary ? e->d_cl_bary : nullptr;  // max-only reduction unless sums are wanted
    a.part_out = local_part(e, 0);
    a.eclk = std::getenv("FSB_NO_EAT_CLOCK") ? nullptr : e->eclk;  // (A/B of the clock's cost)
    a.sane = in_range(e) ? 1 : 0;
    CU(cudaMemsetAsync(e->eclk, 0, sizeof(fsb_dev::EatClock), e->stream));
    CU(cudaEventRecord(e->ev0, e->stream));
    int ctas = 0;
    cudaError_t ce = fault_injected("persistent") ? cudaErrorInvalidClusterSize
                                                  : fsb_dev::launch_cluster_run(a, e->stream, &ctas);
    if (ce == cudaErrorNotSupported)
        return fail(FSB_ERR_UNSUPPORTED, "school does not fit the persistent cluster kernel");
    if (ce != cudaSuccess) {
        cudaGetLastError();
        if (co_schedule_refused(ce))
            return fail(FSB_ERR_UNSUPPORTED, std::string("persistent strategy: cluster launch refused: ") +
                                                 cudaGetErrorName(ce));
        return cuda_fail(ce, "cluster kernel launch");
    }
    CU(cudaEventRecord(e->ev1, e->stream));
    if (trace) CU(cudaMemcpyAsync(trace, e->d_cl_trace, T * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    if (bary) CU(cudaMemcpyAsync(bary, e->d_cl_bary, 3 * T * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    TRY(elapsed(e, seconds));
    TRY(read_eat_cycles(e, (double)ctas, &e->last_eat_s));
    e->cur_explicit = false;
    e->max_valid = true;
    e->sums_valid = bary != nullptr;
    e->cur_buf = 0;
    e->last_launches = 1;
    e->last_strategy = FSB_STRATEGY_PERSISTENT;
    return FSB_OK;
}

int reduce_current(fsb_engine* e) {
    fsb_dev::ReduceArgs a{};
    a.s = canonical(e);
    a.k = scalars_of(e->cfg);
    a.n = e->count;
    a.ws.block_part = e->block_part;
    a.ws.counter = e->counter;
    a.ws.cap = (unsigned)e->block_cap;
    a.part_out = local_part(e, 0);
    a.world = e->world;
    a.px = px_of(e, nullptr, 0, e->xseq + 1);
    a.ec = ec_link(e, 0, -1, 1);
    // launched even for an empty shard: it publishes the identity partial (and,
    // with a peer exchange, pushes it so the other ranks are not kept waiting)
    CU(fsb_dev::launch_reduce(a, e->grid_aux, e->stream));
    TRY(exchange(e, 0));
    e->cur_buf = 0;
    e->max_valid = e->sums_valid = true;
    e->xchg_ready = !host_multi(e);
    e->xseq += 1;
    return FSB_OK;
}

int host_combine(fsb_engine* e, Partial* out) {
    std::vector<Partial> parts(e->world);
    if (e->peer_mode) {
        // the latest epoch's slots, once every rank's flag shows it has landed
        const int b = (int)(e->xseq & 1);
        std::vector<unsigned long long> flags(e->world);
        for (int spins = 0;; ++spins) {
            CU(cudaMemcpy(flags.data(), &e->window->flags[b][0], e->world * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost));
            bool all = true;
            for (unsigned long long f : flags) all = all && f == e->xseq;
            if (all) break;
            if (spins > 20000000) return fail(FSB_ERR_NCCL, "peer exchange: timed out waiting for ranks");
        }
        CU(cudaMemcpy(parts.data(), &e->window->slots[b][0], e->world * sizeof(Partial), cudaMemcpyDeviceToHost));
    } else {
        CU(cudaMemcpyAsync(parts.data(), all_part(e, e->cur_buf), e->world * sizeof(Partial),
                           cudaMemcpyDeviceToHost, e->stream));
        CU(cudaStreamSynchronize(e->stream));
    }
    // rank order, same operators as the device combine (no contraction: adds only)
    Partial r{-INFINITY, 0.0, 0.0, 0.0};
    for (const Partial& p : parts) {
        r.best = (p.best > r.best) ? p.best : r.best;
        r.sx += p.sx;
        r.sy += p.sy;
        r.sf += p.sf;
    }
    *out = r;
    return FSB_OK;
}

}  // namespace

// ============================================================================
extern "C" {

int fsb_abi_version(void) { return FSB_B200_ABI_VERSION; }

const char* fsb_last_error(void) { return g_err.c_str(); }

int fsb_config_validate(const fsb_sim_config* cfg) {
    if (!cfg) return fail(FSB_ERR_INVALID_ARGUMENT, "null config");
    // sim.hpp:44-49, same order and messages
    if (!(cfg->pond_size > 0.0)) return fail(FSB_ERR_INVALID_CONFIG, "SimConfig: pond_size must be > 0");
    if (!(cfg->weight_scale >= 1.0))
        return fail(FSB_ERR_INVALID_CONFIG, "SimConfig: weight_scale must be >= 1");
    if (!(cfg->step_base > 0.0)) return fail(FSB_ERR_INVALID_CONFIG, "SimConfig: step_base must be > 0");
    return FSB_OK;
}

int fsb_shard_range(uint64_t n, int world, int rank, uint64_t* first, uint64_t* count) {
    if (world < 1 || rank < 0 || rank >= world || !first || !count)
        return fail(FSB_ERR_INVALID_ARGUMENT, "fsb_shard_range: bad world/rank");
    // floor(r*N/G) without 128-bit overflow concerns for N < 2^57, G <= 128
    const unsigned __int128 lo = (unsigned __int128)n * (unsigned)rank / (unsigned)world;
    const unsigned __int128 hi = (unsigned __int128)n * (unsigned)(rank + 1) / (unsigned)world;
    *first = (uint64_t)lo;
    *count = (uint64_t)(hi - lo);
    return FSB_OK;
}

uint64_t fsb_checksum_update(uint64_t h, const fsb_fish* fish, uint64_t n) {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(fish);
    const uint64_t bytes = n * sizeof(fsb_fish);
    for (uint64_t k = 0; k < bytes; ++k) {
        h ^= p[k];
        h *= 0x100000001b3ull;
    }
    return h;
}

int fsb_device_count(int* count) {
    if (!count) return fail(FSB_ERR_INVALID_ARGUMENT, "null count");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    *count = n;
    return FSB_OK;
}

int fsb_host_alloc(void** ptr, size_t bytes) {
    if (!ptr) return fail(FSB_ERR_INVALID_ARGUMENT, "null ptr");
    CU(cudaMallocHost(ptr, bytes ? bytes : 1));
    return FSB_OK;
}

int fsb_host_free(void* ptr) {
    if (ptr) CU(cudaFreeHost(ptr));
    return FSB_OK;
}

int fsb_nccl_unique_id(void* out, size_t len) {
    if (!out || len < sizeof(ncclUniqueId)) return fail(FSB_ERR_INVALID_ARGUMENT, "need 128 bytes");
    TRY(nccl_load());
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof id);
    return FSB_OK;
}

int fsb_engine_destroy(fsb_engine* e) {
    if (!e) return FSB_OK;
    cudaSetDevice(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    free_graphs(e);
    if (e->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(e->comm);
    for (void* p : e->opened) cudaIpcCloseMemHandle(p);
    if (e->window) cudaFree(e->window);
    if (e->d_peers) cudaFree(e->d_peers);
    if (e->d_gen) cudaFree(e->d_gen);
    if (e->d_cl_slots) cudaFree(e->d_cl_slots);
    if (e->d_sg_keys) cudaFree(e->d_sg_keys);
    for (void* p : {(void*)e->s.x, (void*)e->s.y, (void*)e->s.w, (void*)e->s.p, (void*)e->c_buf,
                    (void*)e->part_all, (void*)e->block_part, (void*)e->counter, (void*)e->d_step0,
                    (void*)e->d_scalar, (void*)e->d_mismatch, e->staging, (void*)e->d_cl_trace,
                    (void*)e->d_cl_bary, (void*)e->eclk, (void*)e->ff_keys, (void*)e->ff_part})
        if (p) cudaFree(p);
    if (e->h_step0) cudaFreeHost(e->h_step0);
    if (e->pinned) cudaFreeHost(e->pinned);
    if (e->ev0) cudaEventDestroy(e->ev0);
    if (e->ev1) cudaEventDestroy(e->ev1);
    for (auto& h : e->ev_half)
        for (auto& v : h)
            if (v) cudaEventDestroy(v);
    if (e->xfer) {
        cudaStreamSynchronize(e->xfer);
        cudaStreamDestroy(e->xfer);
    }
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
    return FSB_OK;
}

int fsb_engine_create(const fsb_sim_config* cfg, const fsb_engine_options* opts, fsb_engine** out) {
    if (!cfg || !out) return fail(FSB_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    TRY(fsb_config_validate(cfg));
    fsb_engine_options o{};
    o.world_size = 1;
    if (opts) o = *opts;
    if (o.world_size < 1 || o.rank < 0 || o.rank >= o.world_size)
        return fail(FSB_ERR_INVALID_ARGUMENT, "bad rank/world_size");
    if (o.strategy < FSB_STRATEGY_AUTO || o.strategy > FSB_STRATEGY_GRID)
        return fail(FSB_ERR_INVALID_ARGUMENT, "bad strategy");

    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    if (ce != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(FSB_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
    }
    if (o.device < 0 || o.device >= ndev) return fail(FSB_ERR_INVALID_ARGUMENT, "bad device ordinal");
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, o.device));
    if (prop.major < 10)
        return fail(FSB_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100 (built for sm_100a only)");

    fsb_engine* e = new (std::nothrow) fsb_engine();
    if (!e) return fail(FSB_ERR_OUT_OF_MEMORY, "host allocation");
    e->cfg = *cfg;
    e->cfg_in_range = config_in_range(*cfg);
    e->device = o.device;
    e->rank = o.rank;
    e->world = o.world_size;
    e->strategy = o.strategy;
    e->flags = o.flags;
    e->peer_mode = (o.flags & FSB_FLAG_PEER_EXCHANGE) != 0;
    e->host_xchg = !e->peer_mode && (o.flags & FSB_FLAG_HOST_EXCHANGE) != 0;
    e->use_nccl = !e->peer_mode && !e->host_xchg && (o.world_size > 1 || (o.flags & FSB_FLAG_FORCE_NCCL));
    fsb_shard_range(cfg->num_fish, e->world, e->rank, &e->first, &e->count);

    auto bail = [&](int rc) {
        const std::string msg = g_err;
        fsb_engine_destroy(e);
        g_err = msg;
        return rc;
    };
#define CB(call)                                                 \
    do {                                                         \
        cudaError_t _e = (call);                                 \
        if (_e != cudaSuccess) return bail(cuda_fail(_e, #call)); \
    } while (0)

    CB(cudaSetDevice(e->device));
    CB(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    CB(cudaEventCreate(&e->ev0));
    CB(cudaEventCreate(&e->ev1));
    const size_t bytes = (e->count ? e->count : 1) * sizeof(double);
    CB(cudaMalloc(&e->s.x, bytes));
    CB(cudaMalloc(&e->s.y, bytes));
    CB(cudaMalloc(&e->s.w, bytes));
    CB(cudaMalloc(&e->s.p, bytes));
    e->s.c = nullptr;
    // The LDG step kernel is the default: in in-range mode it measured 2-3%
    // faster than the cp.async.bulk ring at 1e7 and 1e8 fish and 25% faster at
    // 1e6 (profiles/r03_ab_bulk_ldg.jsonl); the ring stays available for A/B.
    e->use_bulk = (e->flags & FSB_FLAG_FORCE_BULK) && !(e->flags & FSB_FLAG_NO_BULK);
    // claimed tiles at every size (see kDynamicMinFish)
    e->use_dyn = !e->use_bulk && !(e->flags & FSB_FLAG_STATIC_TILES) &&
                 ((e->flags & FSB_FLAG_DYNAMIC_TILES) || e->count >= kDynamicMinFish);
    // the warp-specialised kernel replaces the claimed-tile one for the
    // compact state (the explicit-cur first step after an upload stays on
    // step_kernel_dyn, with the same one-CTA-per-SM grid)
    if ((e->flags & FSB_FLAG_WS_TILES) && !e->use_bulk && !(e->flags & FSB_FLAG_STATIC_TILES)) {
        const int wsg = fsb_dev::step_ws_blocks(e->device);
        e->use_ws = wsg > 0 && wsg == fsb_dev::step_dyn_blocks(e->device);
        if (e->use_ws) e->use_dyn = true;
    }
    e->grid_aux = fsb_dev::step_grid_blocks(e->device, false, false);
    e->grid = e->use_dyn ? fsb_dev::step_dyn_blocks(e->device)
                         : fsb_dev::step_grid_blocks(e->device, false, e->use_bulk);
    e->grid_explicit = e->use_dyn ? e->grid : fsb_dev::step_grid_blocks(e->device, true, false);
    e->grid_coop = fsb_dev::grid_kernel_blocks(e->device);
    e->grid_auto = e->grid;
    int maxgrid = e->grid > e->grid_explicit ? e->grid : e->grid_explicit;
    if (e->grid_aux > maxgrid) maxgrid = e->grid_aux;
    if (e->grid_coop > maxgrid) maxgrid = e->grid_coop;
    if (2 * e->grid_coop > maxgrid) maxgrid = 2 * e->grid_coop;  // grid kernel: two slot sets
    e->block_cap = maxgrid;
    CB(cudaMalloc(&e->d_gen, sizeof(unsigned long long)));
    e->cgrid_nc = (e->flags & FSB_FLAG_FLAT_GRID) ? 0 : fsb_dev::cgrid_clusters(e->device);
    if (e->cgrid_nc > 0) {
        CB(cudaMalloc(&e->d_cl_slots, cl_slot_bytes(e)));
    }
    if (e->world == 1 && !(e->flags & (FSB_FLAG_L2_GRID | FSB_FLAG_FLAT_GRID))) {
        e->sg_cap = fsb_dev::sgrid_pair_capacity(e->device, &e->sg_grid);
        if (e->sg_cap > 0 && 2ull * e->sg_cap * e->sg_grid >= e->count && e->count > 0 &&
            2 * e->sg_grid <= e->block_cap)
            CB(cudaMalloc(&e->d_sg_keys, 3 * sizeof(unsigned long long)));
        else
            e->sg_cap = 0;
    }
    CB(cudaMalloc(&e->part_all, 2 * e->world * sizeof(Partial)));
    CB(cudaMalloc(&e->block_part, maxgrid * sizeof(Partial)));
    CB(cudaMalloc(&e->ff_keys, 3 * sizeof(unsigned long long)));
    CB(cudaMalloc(&e->ff_part, 2 * (size_t)maxgrid * sizeof(Partial)));
    {
        const char* off = std::getenv("FSB_NO_SPLIT_FOLD");
        e->ff_enabled = !(off && *off && *off != '0') && !(e->flags & FSB_FLAG_LAST_CTA_FOLD);
    }
    CB(cudaMalloc(&e->counter, sizeof(unsigned)));
    CB(cudaMemset(e->counter, 0, sizeof(unsigned)));
    CB(cudaMalloc(&e->d_step0, 2 * sizeof(uint64_t)));
    CB(cudaMallocHost(&e->h_step0, 2 * sizeof(uint64_t)));
    if (e->peer_mode) {
        if (e->world > fsb_dev::kMaxRanks) return bail(fail(FSB_ERR_UNSUPPORTED, "peer exchange: too many ranks"));
        if (const char* v = std::getenv("FSB_PEER_TIMEOUT_S")) {  // failure-detection horizon (default 60 s)
            const double sec = std::atof(v);
            if (sec > 0) e->peer_timeout_ns = (unsigned long long)(sec * 1e9);
        }
        CB(cudaMalloc(&e->window, sizeof(fsb_dev::PeerWindow)));
        CB(cudaMemset(e->window, 0, sizeof(fsb_dev::PeerWindow)));
        CB(cudaMalloc(&e->d_peers, e->world * sizeof(fsb_dev::PeerWindow*)));
        if (e->world == 1) {  // a single rank exchanges with itself
            CB(cudaMemcpy(e->d_peers, &e->window, sizeof(fsb_dev::PeerWindow*), cudaMemcpyHostToDevice));
            e->peer_connected = true;
        }
    }
    CB(cudaMalloc(&e->d_scalar, 4 * sizeof(double)));
    CB(cudaMalloc(&e->eclk, sizeof(fsb_dev::EatClock)));
    CB(cudaMemset(e->eclk, 0, sizeof(fsb_dev::EatClock)));
    CB(cudaMalloc(&e->d_mismatch, sizeof(int)));

    if (e->use_nccl) {
        if (!o.nccl_unique_id) return bail(fail(FSB_ERR_INVALID_ARGUMENT, "world_size > 1 needs nccl_unique_id"));
        int rc = nccl_load();
        if (rc != FSB_OK) return bail(rc);
        ncclUniqueId id;
        std::memcpy(&id, o.nccl_unique_id, sizeof id);
        ncclResult_t r = g_nccl.CommInitRank(&e->comm, e->world, id, e->rank);
        if (r != ncclSuccess) return bail(nccl_fail(r, "ncclCommInitRank"));
        // One eager exchange so NCCL sets up its (lazily established) connections
        // outside any CUDA-graph capture.
        CB(cudaMemsetAsync(e->part_all, 0, 2 * e->world * sizeof(Partial), e->stream));
        rc = exchange(e, 0);
        if (rc != FSB_OK) return bail(rc);
        CB(cudaStreamSynchronize(e->stream));
    }
#undef CB
    *out = e;
    return FSB_OK;
}

int fsb_engine_shard(const fsb_engine* e, uint64_t* first, uint64_t* count) {
    if (!e) return fail(FSB_ERR_INVALID_ARGUMENT, "null engine");
    if (first) *first = e->first;
    if (count) *count = e->count;
    return FSB_OK;
}

int fsb_engine_init(fsb_engine* e) {
    FSB_NVTX("fsb_engine_init");
    TRY(guard(e));
    fsb_dev::InitArgs a{};
    a.s = e->s;
    a.k = scalars_of(e->cfg);
    a.n = e->count;
    a.gfirst = e->first;
    a.w0 = e->cfg.weight_scale;
    CU(fsb_dev::launch_init(a, 0, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    e->cur_explicit = false;
    e->state_sane = e->cfg_in_range;
    e->max_valid = false;
    return FSB_OK;
}

int fsb_engine_upload(fsb_engine* e, const fsb_fish* fish, uint64_t count) {
    FSB_NVTX("fsb_engine_upload");
    TRY(guard(e));
    if (count != e->count) return fail(FSB_ERR_INVALID_ARGUMENT, "upload count != shard count");
    if (count && !fish) return fail(FSB_ERR_INVALID_ARGUMENT, "null fish");
    if (!e->c_buf) CU(cudaMalloc(&e->c_buf, (e->count ? e->count : 1) * sizeof(double)));
    TRY(ensure_staging(e));
    // until the upload completes the state is unknown: checked kernels, explicit cur
    e->state_sane = false;
    e->cur_explicit = true;
    e->max_valid = false;
    fsb_dev::SoA s = e->s;
    s.c = e->c_buf;
    CU(cudaMemsetAsync(e->d_mismatch, 0, sizeof(int), e->stream));
    // chunk i: H2D into staging half i&1 on the copy stream, transpose on the
    // engine stream; the copy of chunk i+1 runs while chunk i is transposed.
    // On any error both streams are drained before returning (no copy may
    // still read the caller's buffer).
    struct Drain {
        fsb_engine* e;
        ~Drain() {
            cudaStreamSynchronize(e->xfer);
            cudaStreamSynchronize(e->stream);
        }
    } drain{e};
    constexpr uint64_t kHalf = kStagingFish / 2;
    CU(cudaEventRecord(e->ev_half[0][1], e->stream));  // both halves free, ordered after prior work
    CU(cudaEventRecord(e->ev_half[1][1], e->stream));
    uint64_t i = 0;
    for (uint64_t lo = 0; lo < count; lo += kHalf, ++i) {
        const int h = (int)(i & 1);
        const uint64_t cnt = (count - lo < kHalf) ? count - lo : kHalf;
        fsb_fish* half = static_cast<fsb_fish*>(e->staging) + h * kHalf;
        CU(cudaStreamWaitEvent(e->xfer, e->ev_half[h][1], 0));
        CU(cudaMemcpyAsync(half, fish + lo, cnt * sizeof(fsb_fish), cudaMemcpyHostToDevice, e->xfer));
        CU(cudaEventRecord(e->ev_half[h][0], e->xfer));
        CU(cudaStreamWaitEvent(e->stream, e->ev_half[h][0], 0));
        CU(fsb_dev::launch_aos_to_soa(half, s, e->cfg.pond_size / 2.0, lo, cnt, e->d_mismatch, e->stream));
        CU(cudaEventRecord(e->ev_half[h][1], e->stream));
    }
    int mismatch = 0;
    CU(cudaMemcpyAsync(&mismatch, e->d_mismatch, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    e->cur_explicit = (mismatch & 1) != 0;
    e->state_sane = e->cfg_in_range && !(mismatch & 2);
    e->max_valid = false;
    return FSB_OK;
}

int fsb_engine_download(fsb_engine* e, fsb_fish* fish, uint64_t count) {
    FSB_NVTX("fsb_engine_download");
    TRY(guard(e));
    if (count != e->count) return fail(FSB_ERR_INVALID_ARGUMENT, "download count != shard count");
    if (count && !fish) return fail(FSB_ERR_INVALID_ARGUMENT, "null fish");
    TRY(ensure_staging(e));
    const fsb_dev::SoA s = canonical(e);
    // chunk i: transpose into staging half i&1 on the engine stream, D2H on the
    // copy stream; the transpose of chunk i+1 runs while chunk i is copied.
    // Both streams are drained on every return path.
    struct Drain {
        fsb_engine* e;
        ~Drain() {
            cudaStreamSynchronize(e->xfer);
            cudaStreamSynchronize(e->stream);
        }
    } drain{e};
    constexpr uint64_t kHalf = kStagingFish / 2;
    CU(cudaEventRecord(e->ev_half[0][0], e->xfer));  // both halves free
    CU(cudaEventRecord(e->ev_half[1][0], e->xfer));
    uint64_t i = 0;
    for (uint64_t lo = 0; lo < count; lo += kHalf, ++i) {
        const int h = (int)(i & 1);
        const uint64_t cnt = (count - lo < kHalf) ? count - lo : kHalf;
        fsb_fish* half = static_cast<fsb_fish*>(e->staging) + h * kHalf;
        CU(cudaStreamWaitEvent(e->stream, e->ev_half[h][0], 0));
        CU(fsb_dev::launch_soa_to_aos(s, e->cfg.pond_size / 2.0, lo, cnt, half, e->stream));
        CU(cudaEventRecord(e->ev_half[h][1], e->stream));
        CU(cudaStreamWaitEvent(e->xfer, e->ev_half[h][1], 0));
        CU(cudaMemcpyAsync(fish + lo, half, cnt * sizeof(fsb_fish), cudaMemcpyDeviceToHost, e->xfer));
        CU(cudaEventRecord(e->ev_half[h][0], e->xfer));
    }
    CU(cudaStreamSynchronize(e->xfer));
    CU(cudaStreamSynchronize(e->stream));
    return FSB_OK;  // (drain: already idle)
}

int fsb_engine_move(fsb_engine* e, uint64_t step, double* seconds) {
    FSB_NVTX("fsb_engine_move");
    TRY(guard(e));
    TRY(need_peers(e));
    CU(cudaEventRecord(e->ev0, e->stream));
    if (e->count || e->peer_mode) {  // an empty shard still publishes (and pushes) its identity partial
        fsb_dev::StepArgs a = step_args(e, canonical(e));
        a.step_ptr = nullptr;
        a.step_add = step;
        a.part_in = nullptr;  // no pending eat: phases are applied eagerly
        a.part_out = local_part(e, 0);
        a.px = px_of(e, nullptr, 0, e->xseq + 1);
        a.ec = ec_link(e, 0, -1, 1);  // the fused max: producer side of the eat region
        CU(fsb_dev::launch_step(a, e->cur_explicit ? e->grid_explicit : e->grid, e->stream));
    } else {
        const Partial id{-INFINITY, 0.0, 0.0, 0.0};
        CU(cudaMemcpyAsync(local_part(e, 0), &id, sizeof(Partial), cudaMemcpyHostToDevice, e->stream));
    }
    TRY(exchange(e, 0));
    CU(cudaEventRecord(e->ev1, e->stream));
    TRY(elapsed(e, seconds));
    e->cur_explicit = false;
    e->max_valid = e->sums_valid = true;
    e->xchg_ready = !host_multi(e);
    e->cur_buf = 0;
    e->xseq += 1;
    return FSB_OK;
}

int fsb_engine_eat(fsb_engine* e, double* max_diff, double* seconds) {
    FSB_NVTX("fsb_engine_eat");
    TRY(guard(e));
    TRY(need_peers(e));
    CU(cudaMemsetAsync(&e->eclk->ns, 0, sizeof(unsigned long long), e->stream));
    if (!e->max_valid) TRY(reduce_current(e));
    TRY(need_partials(e));
    fsb_dev::EatArgs a{};
    a.s = canonical(e);
    a.k = scalars_of(e->cfg);
    a.n = e->count;
    a.part_in = all_part(e, e->cur_buf);
    a.world = e->world;
    a.px = px_of(e, nullptr, e->xseq, 0);
    a.trace_out = e->d_scalar;
    a.ec = ec_link(e, -1, 0, 1);  // consumer side: the producer's reduction tail + this combine
    CU(fsb_dev::launch_eat(a, e->grid_aux, e->stream));
    double m = 0.0;
    CU(cudaMemcpyAsync(&m, e->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    TRY(peer_fault(e));
    // EatResult::seconds (sim.hpp:103): the max only, not the weight update
    TRY(read_eat_ns(e, 1.0, &e->last_eat_s));
    if (seconds) *seconds = e->last_eat_s;
    if (max_diff) *max_diff = m;
    return FSB_OK;
}

// Long runs are cut into graphs of at most kMaxGraphSteps steps (each a
// complete run: its own trailing eat), so graph size stays bounded.
int run_stream_chunked(fsb_engine* e, uint64_t first_step, uint64_t T, double* trace, double* bary,
                       double* seconds) {
    constexpr uint64_t kMaxGraphSteps = 1024;
    double total = 0.0, eat = 0.0;
    uint64_t launches = 0;
    for (uint64_t off = 0; off < T; off += kMaxGraphSteps) {
        const uint64_t len = (T - off < kMaxGraphSteps) ? T - off : kMaxGraphSteps;
        double s = 0.0;
        TRY(run_stream(e, first_step + off, len, trace ? trace + off : nullptr, bary ? bary + 3 * off : nullptr,
                       &s));
        total += s;
        eat += e->last_eat_s;
        launches += e->last_launches;
    }
    *seconds = total;
    e->last_eat_s = eat;
    e->last_launches = launches;
    e->last_strategy = FSB_STRATEGY_STREAM;
    return FSB_OK;
}

int fsb_engine_run(fsb_engine* e, uint64_t first_step, uint64_t num_steps, double* trace, double* bary,
                   fsb_timing* timing) {
    FSB_NVTX("fsb_engine_run");
    TRY(guard(e));
    TRY(need_peers(e));
    TRY(phase_only(e, "fsb_engine_run"));
    if (timing) *timing = fsb_timing{0.0, 0.0, 0.0, 0.0};
    e->fallback.clear();
    e->last_eat_s = 0.0;
    if (num_steps == 0) return FSB_OK;
    double secs = 0.0;
    if (e->count == 0 && !e->use_nccl && !e->peer_mode) {
        // empty school: every max is -inf (executor.hpp:86), sums are 0
        for (uint64_t k = 0; k < num_steps; ++k) {
            if (trace) trace[k] = -INFINITY;
            if (bary) bary[3 * k] = bary[3 * k + 1] = bary[3 * k + 2] = 0.0;
        }
        const Partial id{-INFINITY, 0.0, 0.0, 0.0};
        CU(cudaMemcpy(local_part(e, 0), &id, sizeof(Partial), cudaMemcpyHostToDevice));
        e->max_valid = e->sums_valid = true;
        e->cur_buf = 0;
        e->last_launches = 0;
        e->last_strategy = FSB_STRATEGY_STREAM;
    } else if (want_grid(e)) {
        // (the first run after an inconsistent upload takes the stream path below)
        int rc = run_grid(e, first_step, num_steps, trace, bary, &secs);
        if (rc == FSB_ERR_UNSUPPORTED && e->strategy == FSB_STRATEGY_AUTO) {
            e->fallback = g_err;  // the device refused the co-resident grid: graph of step kernels
            rc = run_stream_chunked(e, first_step, num_steps, trace, bary, &secs);
        }
        TRY(rc);
    } else if (want_persistent(e)) {
        int rc = run_persistent(e, first_step, num_steps, trace, bary, &secs);
        if (rc == FSB_ERR_UNSUPPORTED && e->strategy == FSB_STRATEGY_AUTO) {
            e->fallback = g_err;
            rc = run_stream_chunked(e, first_step, num_steps, trace, bary, &secs);
        }
        TRY(rc);
    } else {
        TRY(run_stream_chunked(e, first_step, num_steps, trace, bary, &secs));
    }
    if (timing) {
        // SimResult (sim.hpp:125-131): seconds_eat = the max region only, seconds_move = the rest of the loop
        timing->seconds_total = secs;
        timing->seconds_eat = e->last_eat_s < secs ? e->last_eat_s : secs;
        timing->seconds_move = secs - timing->seconds_eat;
        timing->seconds_loop = secs;
    }
    return FSB_OK;
}

int fsb_engine_simulate(fsb_engine* e, double* trace, double* bary, fsb_timing* timing) {
    FSB_NVTX("fsb_engine_simulate");
    TRY(guard(e));
    TRY(phase_only(e, "fsb_engine_simulate"));
    CU(cudaEventRecord(e->ev0, e->stream));
    TRY(fsb_engine_init(e));
    CU(cudaEventRecord(e->ev1, e->stream));
    double init_s = 0.0;
    TRY(elapsed(e, &init_s));
    TRY(fsb_engine_run(e, 0, e->cfg.num_steps, trace, bary, timing));
    if (timing) timing->seconds_total += init_s;
    return FSB_OK;
}

int fsb_engine_barycentre(fsb_engine* e, double sums[3], double xy[2]) {
    FSB_NVTX("fsb_engine_barycentre");
    TRY(guard(e));
    TRY(need_peers(e));
    if (!e->max_valid || !e->sums_valid) TRY(reduce_current(e));
    TRY(need_partials(e));
    Partial r;
    TRY(host_combine(e, &r));
    if (sums) {
        sums[0] = r.sx;
        sums[1] = r.sy;
        sums[2] = r.sf;
    }
    if (xy) {
        xy[0] = r.sx / r.sf;
        xy[1] = r.sy / r.sf;
    }
    return FSB_OK;
}

int fsb_engine_partial(fsb_engine* e, double out[5]) {
    FSB_NVTX("fsb_engine_partial");
    TRY(guard(e));
    TRY(need_peers(e));
    if (!out) return fail(FSB_ERR_INVALID_ARGUMENT, "null out");
    if (!e->max_valid || !e->sums_valid) TRY(reduce_current(e));
    Partial p;
    CU(cudaMemcpyAsync(&p, local_part(e, e->cur_buf), sizeof p, cudaMemcpyDeviceToHost, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    out[0] = p.best;
    out[1] = p.sx;
    out[2] = p.sy;
    out[3] = p.sf;
    out[4] = (double)e->xseq;  // exchange epoch: identical on every rank at the same step
    return FSB_OK;
}

int fsb_engine_set_partials(fsb_engine* e, const double* parts, size_t count) {
    FSB_NVTX("fsb_engine_set_partials");
    TRY(guard(e));
    if (!e->host_xchg) return fail(FSB_ERR_INVALID_ARGUMENT, "set_partials needs FSB_FLAG_HOST_EXCHANGE");
    if (!parts || count != 5 * (size_t)e->world)
        return fail(FSB_ERR_INVALID_ARGUMENT, "set_partials: need 5 * world_size doubles");
    if (!e->max_valid || !e->sums_valid)
        return fail(FSB_ERR_INVALID_ARGUMENT, "set_partials: no partial of the current state (fsb_engine_partial)");
    // this rank's own entry must be its partial, bit for bit: catches partials out of rank order
    double mine[5];
    TRY(fsb_engine_partial(e, mine));
    if (std::memcmp(mine, parts + 5 * (size_t)e->rank, sizeof mine) != 0)
        return fail(FSB_ERR_INVALID_ARGUMENT, "set_partials: entry [rank] is not this rank's partial");
    // every rank's partial must be of the same step (exchange epoch): catches a
    // rank that moved twice or skipped a move
    std::vector<Partial> packed(e->world);
    for (int q = 0; q < e->world; ++q) {
        const double* v = parts + 5 * (size_t)q;
        if (std::memcmp(&v[4], &mine[4], sizeof(double)) != 0)
            return fail(FSB_ERR_INVALID_ARGUMENT, "set_partials: entry [" + std::to_string(q) +
                                                      "] is from another step (exchange epoch differs)");
        packed[q] = Partial{v[0], v[1], v[2], v[3]};
    }
    CU(cudaMemcpyAsync(all_part(e, e->cur_buf), packed.data(), (size_t)e->world * sizeof(Partial),
                       cudaMemcpyHostToDevice, e->stream));
    CU(cudaStreamSynchronize(e->stream));
    e->xchg_ready = true;
    return FSB_OK;
}

int fsb_engine_gather(fsb_engine* e, const uint64_t* local_idx, uint64_t n, fsb_fish* out) {
    FSB_NVTX("fsb_engine_gather");
    TRY(guard(e));
    if (n && (!local_idx || !out)) return fail(FSB_ERR_INVALID_ARGUMENT, "null argument");
    for (uint64_t k = 0; k < n; ++k)
        if (local_idx[k] >= e->count) return fail(FSB_ERR_INVALID_ARGUMENT, "gather index out of range");
    TRY(ensure_staging(e));
    const fsb_dev::SoA s = canonical(e);
    // indices ride in the tail of the staging buffer: kStagingFish/6 per chunk
    const uint64_t chunk = kStagingFish / 6;
    uint64_t* d_idx = reinterpret_cast<uint64_t*>(static_cast<char*>(e->staging) +
                                                  chunk * sizeof(fsb_fish));
    for (uint64_t lo = 0; lo < n; lo += chunk) {
        const uint64_t cnt = (n - lo < chunk) ? n - lo : chunk;
        CU(cudaMemcpyAsync(d_idx, local_idx + lo, cnt * sizeof(uint64_t), cudaMemcpyHostToDevice, e->stream));
        CU(fsb_dev::launch_gather(s, e->cfg.pond_size / 2.0, d_idx, cnt, e->staging, e->stream));
        CU(cudaMemcpyAsync(out + lo, e->staging, cnt * sizeof(fsb_fish), cudaMemcpyDeviceToHost, e->stream));
        CU(cudaStreamSynchronize(e->stream));
    }
    return FSB_OK;
}

int fsb_engine_checksum(fsb_engine* e, uint64_t h_in, uint64_t* h_out) {
    FSB_NVTX("fsb_engine_checksum");
    TRY(guard(e));
    if (!h_out) return fail(FSB_ERR_INVALID_ARGUMENT, "null h_out");
    TRY(ensure_staging(e));
    if (!e->pinned) CU(cudaMallocHost(&e->pinned, kStagingFish * sizeof(fsb_fish)));
    const fsb_dev::SoA s = canonical(e);
    uint64_t h = h_in;
    for (uint64_t lo = 0; lo < e->count; lo += kStagingFish) {
        const uint64_t cnt = (e->count - lo < kStagingFish) ? e->count - lo : kStagingFish;
        CU(fsb_dev::launch_soa_to_aos(s, e->cfg.pond_size / 2.0, lo, cnt, e->staging, e->stream));
        CU(cudaMemcpyAsync(e->pinned, e->staging, cnt * sizeof(fsb_fish), cudaMemcpyDeviceToHost, e->stream));
        CU(cudaStreamSynchronize(e->stream));
        h = fsb_checksum_update(h, static_cast<const fsb_fish*>(e->pinned), cnt);
    }
    *h_out = h;
    return FSB_OK;
}

int fsb_engine_synchronize(fsb_engine* e) {
    TRY(guard(e));
    CU(cudaStreamSynchronize(e->stream));
    return FSB_OK;
}

int fsb_engine_stream(fsb_engine* e, void** stream) {
    if (!e || !stream) return fail(FSB_ERR_INVALID_ARGUMENT, "null argument");
    *stream = e->stream;
    return FSB_OK;
}

int fsb_engine_time_step_kernels(fsb_engine* e, uint64_t first_step, uint64_t num_steps, double* kernel_ms) {
    TRY(guard(e));
    TRY(need_peers(e));
    TRY(phase_only(e, "fsb_engine_time_step_kernels"));
    if (!kernel_ms && num_steps) return fail(FSB_ERR_INVALID_ARGUMENT, "null kernel_ms");
    if (e->count == 0 && e->world == 1) {
        for (uint64_t k = 0; k < num_steps; ++k) kernel_ms[k] = 0.0;
        return FSB_OK;
    }
    struct Events {  // destroyed on every return path
        std::vector<cudaEvent_t> v;
        ~Events() {
            for (cudaEvent_t x : v)
                if (x) cudaEventDestroy(x);
        }
    } events;
    events.v.assign(num_steps + 1, nullptr);
    std::vector<cudaEvent_t>& ev = events.v;
    for (auto& v : ev) CU(cudaEventCreate(&v));
    CU(cudaEventRecord(ev[0], e->stream));
    const uint64_t x0 = e->xseq;
    for (uint64_t k = 0; k < num_steps; ++k) {
        fsb_dev::StepArgs a = step_args(e, canonical(e));
        a.step_add = first_step + k;
        a.part_in = (k == 0) ? nullptr : all_part(e, (int)((k - 1) & 1));
        a.part_out = local_part(e, (int)(k & 1));
        a.px = px_of(e, nullptr, k ? x0 + k : 0, x0 + k + 1);
        CU(fsb_dev::launch_step(a, e->cur_explicit ? e->grid_explicit : e->grid, e->stream));
        e->cur_explicit = false;
        CU(cudaEventRecord(ev[k + 1], e->stream));
        TRY(exchange(e, (int)(k & 1)));
    }
    // materialise the last step's eat so the school is a valid end-of-step state
    if (num_steps) {
        fsb_dev::EatArgs ea{};
        ea.s = canonical(e);
        ea.k = scalars_of(e->cfg);
        ea.n = e->count;
        ea.part_in = all_part(e, (int)((num_steps - 1) & 1));
        ea.world = e->world;
        ea.px = px_of(e, nullptr, x0 + num_steps, 0);
        CU(fsb_dev::launch_eat(ea, e->grid_aux, e->stream));
        e->cur_buf = (int)((num_steps - 1) & 1);
        e->max_valid = e->sums_valid = true;
        e->xseq = x0 + num_steps;
    }
    CU(cudaStreamSynchronize(e->stream));
    for (uint64_t k = 0; k < num_steps; ++k) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
        kernel_ms[k] = ms;
    }
    return FSB_OK;
}

int fsb_engine_set_grid(fsb_engine* e, int ctas) {
    TRY(guard(e));
    if (ctas < 0 || ctas > 65536) return fail(FSB_ERR_INVALID_ARGUMENT, "ctas must be in [0, 65536]");
    const int g = ctas ? ctas : e->grid_auto;
    if (g > e->block_cap) {
        CU(cudaStreamSynchronize(e->stream));
        Partial* nb = nullptr;
        CU(cudaMalloc(&nb, g * sizeof(Partial)));
        Partial* nf = nullptr;
        CU(cudaMalloc(&nf, 2 * (size_t)g * sizeof(Partial)));
        cudaFree(e->block_part);
        cudaFree(e->ff_part);
        e->block_part = nb;
        e->ff_part = nf;
        e->block_cap = g;
        free_graphs(e);  // captured launches carry the old buffers
    }
    if (g != e->grid) free_graphs(e);  // captured launches carry the old grid
    e->grid = g;
    return FSB_OK;
}

int fsb_engine_set_tile_groups(fsb_engine* e, int groups) {
    TRY(guard(e));
    if (groups < 0 || groups > 4096) return fail(FSB_ERR_INVALID_ARGUMENT, "groups must be in [0, 4096]");
    if ((unsigned)groups != e->tile_groups) free_graphs(e);  // captured launches carry the old value
    e->tile_groups = (unsigned)groups;
    return FSB_OK;
}

int fsb_engine_grid(const fsb_engine* e, int* ctas, int* threads_per_cta) {
    if (!e) return fail(FSB_ERR_INVALID_ARGUMENT, "null engine");
    if (ctas) *ctas = e->grid;
    if (threads_per_cta)
        *threads_per_cta = e->use_bulk ? fsb_dev::kBulkThreads : e->use_dyn ? fsb_dev::kDynThreads : fsb_dev::kStepThreads;
    return FSB_OK;
}

int fsb_engine_last_launches(const fsb_engine* e, uint64_t* launches) {
    if (!e || !launches) return fail(FSB_ERR_INVALID_ARGUMENT, "null argument");
    *launches = e->last_launches;
    return FSB_OK;
}

int fsb_engine_last_strategy(const fsb_engine* e, int* strategy, const char** fallback_reason) {
    if (!e || !strategy) return fail(FSB_ERR_INVALID_ARGUMENT, "null argument");
    *strategy = e->last_strategy;
    if (fallback_reason) *fallback_reason = e->fallback.c_str();
    return FSB_OK;
}

}  // extern "C"

extern "C" int fsb_selftest_fast_math(int device, uint64_t n, uint64_t seed, uint64_t out[4]) {
    if (!out) return fail(FSB_ERR_INVALID_ARGUMENT, "null out");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(FSB_ERR_CUDA, "no CUDA device available");
    }
    CU(cudaSetDevice(device));
    unsigned long long* d = nullptr;
    CU(cudaMalloc(&d, 4 * sizeof *d));
    cudaError_t e = cudaMemset(d, 0, 4 * sizeof *d);
    if (e == cudaSuccess) e = fsb_dev::launch_selftest_fast_math(n, seed, d, 0);
    unsigned long long h[4] = {0, 0, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "selftest fast math");
    for (int k = 0; k < 4; ++k) out[k] = h[k];
    return FSB_OK;
}

extern "C" int fsb_engine_peer_handle(fsb_engine* e, void* out, size_t len) {
    TRY(guard(e));
    if (!e->peer_mode) return fail(FSB_ERR_INVALID_ARGUMENT, "engine not created with FSB_FLAG_PEER_EXCHANGE");
    if (!out || len < sizeof(cudaIpcMemHandle_t)) return fail(FSB_ERR_INVALID_ARGUMENT, "need 64 bytes");
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, e->window));
    std::memcpy(out, &h, sizeof h);
    return FSB_OK;
}

extern "C" int fsb_engine_peer_connect_local(fsb_engine* e, fsb_engine* const* ranks, int n) {
    TRY(guard(e));
    if (!e->peer_mode) return fail(FSB_ERR_INVALID_ARGUMENT, "engine not created with FSB_FLAG_PEER_EXCHANGE");
    if (!ranks || n != e->world) return fail(FSB_ERR_INVALID_ARGUMENT, "need world_size engines");
    if (ranks[e->rank] != e) return fail(FSB_ERR_INVALID_ARGUMENT, "ranks[rank] must be this engine");
    std::vector<fsb_dev::PeerWindow*> peers(e->world);
    for (int q = 0; q < e->world; ++q) {
        const fsb_engine* r = ranks[q];
        if (!r || !r->peer_mode || r->world != e->world || r->rank != q)
            return fail(FSB_ERR_INVALID_ARGUMENT, "ranks[q] must be rank q's peer-exchange engine");
        if (r->device != e->device) {
            int ok = 0;
            CU(cudaDeviceCanAccessPeer(&ok, e->device, r->device));
            if (!ok) return fail(FSB_ERR_UNSUPPORTED, "no peer access between the ranks' devices");
            // guard() made this engine's device current: enable access from it
            const cudaError_t pe = cudaDeviceEnablePeerAccess(r->device, 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(pe, "peer access");
            cudaGetLastError();
        }
        peers[q] = r->window;
    }
    CU(cudaMemcpy(e->d_peers, peers.data(), e->world * sizeof(fsb_dev::PeerWindow*), cudaMemcpyHostToDevice));
    e->peer_connected = true;
    return FSB_OK;
}

extern "C" int fsb_engine_peer_connect(fsb_engine* e, const void* handles, size_t len) {
    TRY(guard(e));
    if (!e->peer_mode) return fail(FSB_ERR_INVALID_ARGUMENT, "engine not created with FSB_FLAG_PEER_EXCHANGE");
    const size_t hs = sizeof(cudaIpcMemHandle_t);
    if (!handles || len < hs * (size_t)e->world) return fail(FSB_ERR_INVALID_ARGUMENT, "need world_size handles");
    std::vector<fsb_dev::PeerWindow*> peers(e->world);
    for (int q = 0; q < e->world; ++q) {
        if (q == e->rank) {
            peers[q] = e->window;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char*>(handles) + hs * q, hs);
        void* p = nullptr;
        CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        e->opened.push_back(p);
        peers[q] = static_cast<fsb_dev::PeerWindow*>(p);
    }
    CU(cudaMemcpy(e->d_peers, peers.data(), e->world * sizeof(fsb_dev::PeerWindow*), cudaMemcpyHostToDevice));
    e->peer_connected = true;
    return FSB_OK;
}
