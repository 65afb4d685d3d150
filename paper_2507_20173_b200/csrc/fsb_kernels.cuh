// fsb_kernels.cuh -- device kernels of the B200 FSB engine and their host
// launchers (implemented in fsb_kernels.cu, called by fsb_engine.cu).
//
// Fish state lives in HBM as structure-of-arrays of fp64:
//   x[n], y[n], w[n]  position and weight                (Fish::x,y,weight)
//   p[n]              prev_objective                      (Fish::prev_objective)
//   c[n]              current_objective -- only materialised after an upload
//                     whose current_objective is not objective(x, y); in every
//                     state the engine produces itself cur == objective(x, y)
//                     bit-for-bit, so it is recomputed instead of stored.
// One fused step therefore reads 32 B and writes 32 B per fish.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// Debug builds (tools/variants.py "debug"): device-side bounds checks that trap
// with a message -- the substitute for compute-sanitizer, which this GPU pool
// does not offer.  Compiled out otherwise.
#ifndef FSB_DEBUG_CHECKS
#define FSB_DEBUG_CHECKS 0
#endif
#if FSB_DEBUG_CHECKS
#include <cstdio>
#define FSB_CHECK(c)                                                                   \
    do {                                                                               \
        if (!(c)) {                                                                    \
            printf("FSB_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x, #c);                             \
            __trap();                                                                  \
        }                                                                              \
    } while (0)
#else
#define FSB_CHECK(c) \
    do {             \
    } while (0)
#endif

namespace fsb_dev {

// Tuning knobs (compile-time; tools/variants.py builds alternatives for A/B runs).
#ifndef FSB_PAIRS
#define FSB_PAIRS 1
#endif
#ifndef FSB_MIN_BLOCKS
#define FSB_MIN_BLOCKS 4
#endif

#ifndef FSB_CLUSTER_MIN_FISH
#define FSB_CLUSTER_MIN_FISH 256  // persistent kernel: fish per CTA before adding CTAs
#endif

#ifndef FSB_BULK_STAGES
#define FSB_BULK_STAGES 4
#endif
#ifndef FSB_BULK_MIN_BLOCKS
#define FSB_BULK_MIN_BLOCKS 3
#endif
#ifndef FSB_BULK_PAIRS
#define FSB_BULK_PAIRS 1
#endif

#ifndef FSB_STEP_THREADS
#define FSB_STEP_THREADS 256
#endif

constexpr int kThreads = 256;     // threads per CTA of the streaming kernels
constexpr int kStepThreads = FSB_STEP_THREADS;  // ... of the LDG step kernel and the grid kernel
constexpr int kPairsPerThread = FSB_PAIRS;  // double2 loads per array per thread per tile
constexpr int kTilePairs = kStepThreads * kPairsPerThread;

// step_kernel_dyn: one CTA per SM, warps claim tiles of its chunk.
#ifndef FSB_DYN_THREADS
#define FSB_DYN_THREADS 1024
#endif
#ifndef FSB_DYN_MIN_BLOCKS
#define FSB_DYN_MIN_BLOCKS 1
#endif
constexpr int kDynThreads = FSB_DYN_THREADS;
constexpr int kDynTiles = 1024;   // tile-partial slots per CTA (32 KB of shared memory)
#ifndef FSB_DYN_MIN_GROUPS
#define FSB_DYN_MIN_GROUPS 4
#endif
constexpr unsigned kDynMinGroups = FSB_DYN_MIN_GROUPS;  // minimum 32-pair groups per claimed tile
constexpr int kTileFish = 2 * kTilePairs;

// step_kernel_bulk: 8 compute warps x kBulkPairsPerThread pairs per sub-tile,
// plus one producer warp; a kBulkStages-deep ring of sub-tiles in smem.
#ifndef FSB_BULK_COMPUTE
#define FSB_BULK_COMPUTE 256
#endif
constexpr int kBulkCompute = FSB_BULK_COMPUTE;  // compute threads per bulk-ring CTA (+ one producer warp)
constexpr int kBulkThreads = kBulkCompute + 32;
constexpr int kBulkPairsPerThread = FSB_BULK_PAIRS;
constexpr int kBulkTilePairs = kBulkCompute * kBulkPairsPerThread;
constexpr int kBulkStages = FSB_BULK_STAGES;
constexpr int kBulkStageBytes = kBulkTilePairs * 16 * 4;  // x, y, w, p as double2
constexpr int kBulkSmemBytes = kBulkStages * kBulkStageBytes;

// Global partials of one step: max(prev-cur) and the barycentre sums
// sum x*f, sum y*f, sum f.  One per rank; combined in rank order.
struct alignas(32) Partial {
    double best;
    double sx;
    double sy;
    double sf;
};

struct SoA {
    double* x;
    double* y;
    double* w;
    double* p;
    double* c;  // nullptr unless current_objective is explicit
};

struct Scalars {
    double pond;
    double half_pond;
    double step_base;
    double w_max;
    uint64_t seed;
    uint64_t zero;  // always 0; opaque to the compiler (the RNG-first scheduling fence)
};

// Reduction workspace of one launch.
struct ReduceWs {
    Partial* block_part;  // [cap] (>= grid; the grid kernel uses 2 x grid)
    unsigned* counter;    // zero between launches
    unsigned cap;         // capacity of block_part (checked by FSB_DEBUG_CHECKS builds)
};

// Peer exchange (FSB_FLAG_PEER_EXCHANGE): every rank owns one window in its
// HBM, exported with CUDA IPC and mapped by every peer.  The last CTA of a
// rank's step kernel stores the rank partial straight into slot [epoch&1][rank]
// of every peer's window over NVLink and then releases flag [epoch&1][rank] =
// epoch (system scope); the next kernel on each rank acquires all flags of the
// epoch from its own window and combines the slots in rank order.  Epochs are a
// per-engine exchange sequence number, identical on all ranks.
constexpr int kMaxRanks = 64;

struct PeerWindow {
    Partial slots[2][kMaxRanks];
    unsigned long long flags[2][kMaxRanks];
    unsigned long long fault;  // nonzero: an epoch whose partials did not all arrive in time
};

struct PeerXchg {
    PeerWindow* const* peers;  // device array [world]: peer windows as mapped here (nullptr = off)
    PeerWindow* local;         // this rank's window
    int rank;
    const uint64_t* seq_ptr;   // epoch base = (seq_ptr ? *seq_ptr : 0) ...
    uint64_t in_add;           // ... + in_add: epoch of the partials consumed (0 = none)
    uint64_t out_add;          // ... + out_add: epoch of the partial produced (0 = none)
    unsigned long long timeout_ns;  // give up waiting for a rank after this long (window.fault)
};

// Eat-region clock: the GPU counterpart of SimResult::seconds_eat, which the
// reference times around the max only (sim.hpp:103,112,130).  On the GPU the
// max is fused into the step kernels, so its cost is measured where it sits on
// the critical path, with %globaltimer (ns, one clock for every SM):
//  * stream path: from the moment the last CTA of step t has updated its fish
//    (t_done, max over CTAs by red.max) to the moment step t+1's kernel (or the
//    trailing eat kernel) holds the combined global max -- the block and grid
//    reductions, the kernel boundary that is the grid-wide barrier, and any
//    NCCL / peer exchange in between;
//  * phase API (move, then eat as separate calls): the producer's reduction
//    tail (t_done -> t_pub, rank partial published) plus the eat kernel's own
//    combine, without the host gap between the two calls;
//  * persistent kernels: every CTA's time from its own fish done to holding the
//    step's global max, summed, divided by the CTA count by the host.
struct EatStamp {
    unsigned long long t_done;  // max over CTAs: all fish of the step updated
    unsigned long long t_pub;   // the step's rank partial published (last CTA)
};
struct EatClock {
    EatStamp s[2];              // by step parity (graph) / slot 0 (eager launches)
    unsigned long long ns;      // accumulated eat-region nanoseconds (persistent kernels: SM cycles)
    unsigned long long pad;
    // persistent kernels count SM cycles (clock64: a globaltimer read per step
    // costs ~0.1 us on the 0.9 us C4 step); CTA 0 brackets the kernel with both
    // clocks so the host converts cycles to ns
    unsigned long long g0, c0, g1, c1;
};
struct EatLink {
    EatStamp* out;              // producer: this step's stamp (nullptr: off)
    EatStamp* in;               // consumer: the stamp of the step whose max is combined (nullptr: none)
    unsigned long long* ns;     // accumulator (nullptr: off)
    int phase;                  // consumer mode: 1 = phase API (tail + own combine), 0 = graph chain
};

// Split fold of a one-rank graph chain (fsb_engine.cu build_graph): the next
// step needs only the MAX of this step, so every CTA red.max's its max -- as an
// order-preserving key -- into the step's key slot and stores its partial
// without meeting the other CTAs (no arrival counter, no last-CTA fold inside
// this kernel: two dependent L2 round trips and a block reduction off the
// per-step chain).  The consumer (the next step kernel, or the trailing eat)
// reads the key; one warp of its CTA 0 folds the CTA partials in index order
// for the outputs (barycentre sums, the cached rank partial) after its own run.
// Key slots rotate over three steps (CTA 0 of step k zeroes step k+1's slot,
// last read by step k-1's consumers), CTA-partial buffers over two.
struct FastFold {
    unsigned long long* key_out;       // this step's key slot (nullptr: the last-CTA fold)
    Partial* bp_out;                   // this step's CTA partials [gridDim.x]
    const unsigned long long* key_in;  // the previous step's key slot (nullptr: nothing to consume this way)
    const Partial* bp_in;              // the previous step's CTA partials
    unsigned bp_in_count;              // CTAs of the kernel that produced them
    Partial* fold_out;                 // where the folded partial of the previous step goes (the rank partial)
    unsigned long long* key_reset;     // the next step's key slot, zeroed here (nullptr: none)
};

struct StepArgs {
    SoA s;
    Scalars k;
    uint64_t n;           // local fish
    uint64_t gfirst;      // global index of local fish 0 (RNG key, rng.hpp:35)
    const uint64_t* step_ptr;  // step = (step_ptr ? *step_ptr : 0) + step_add
    uint64_t step_add;
    const Partial* part_in;  // [world] previous step's partials, or nullptr (no pending eat)
    int world;
    double* trace_out;    // if non-null, CTA 0 stores the previous step's max here
    double* bary_out;     // if non-null, CTA 0 stores the previous step's 3 sums here
    ReduceWs ws;
    Partial* part_out;    // this rank's partial of this step
    int alternate;        // reverse tile order on odd steps (L2 reuse across steps)
    int bulk;             // stream through shared memory with cp.async.bulk (compact state)
    int pdl;              // launched as a programmatic dependent of the previous step
    PeerXchg px;          // peer exchange instead of part_in/part_out (px.peers != nullptr)
    int sane;             // state and config in range: guards elided (fsb_math.cuh "In-range mode")
    int dyn;              // compact LDG path: step_kernel_dyn (one CTA per SM, claimed tiles)
    int wspec;            // compact path: step_kernel_ws (TMA producer warp + 31 consumer warps per SM)
    unsigned tile_groups; // step_kernel_dyn: minimum 32-pair groups per claimed tile (0 = kDynMinGroups)
    EatLink ec;           // eat-region clock
    FastFold ff;          // split fold (step_kernel_dyn in a one-rank graph), all null otherwise
};

// Persistent cooperative-grid run (FSB_STRATEGY_GRID): `base` supplies the
// state, scalars and reduction workspace; all num_steps steps in one launch.
struct GridArgs {
    StepArgs base;
    uint64_t first_step;
    uint64_t num_steps;
    double* trace;              // [num_steps]
    double* bary;               // [3*num_steps] or nullptr
    unsigned long long* gen;    // arrival counter, zero at launch; base.ws.block_part holds 2 x grid slots
    EatClock* eclk;             // eat-region clock (nullptr: off)
};

// Cluster-reduced persistent run (FSB_STRATEGY_GRID when cluster launch is
// available): clusters of kCGridCluster CTAs reduce over DSMEM, cluster
// leaders meet through self-validating slots (one 128-B line per cluster).
#ifndef FSB_CGRID_CLUSTER
#define FSB_CGRID_CLUSTER 8
#endif
constexpr int kCGridCluster = FSB_CGRID_CLUSTER;
constexpr int kSlotRing = 3;     // cluster-partial slot sets (step k uses k % 3)
constexpr int kSlotWords = 16;   // doubles per cluster slot: one 128-B line each (no polling storm on a line)
constexpr unsigned long long kSlotSentinel = ~0ull;  // "not yet written" (a NaN pattern arithmetic never yields)

struct CGridArgs {
    StepArgs base;
    uint64_t first_step;
    uint64_t num_steps;
    double* trace;                // [num_steps]
    double* bary;                 // [3*num_steps] or nullptr
    double* cl_slots;             // [kSlotRing][clusters][kSlotWords], all bytes 0xFF (sentinel) at launch
    EatClock* eclk;               // eat-region clock (nullptr: off)
};

// Shared-memory-resident persistent run (FSB_STRATEGY_GRID for schools that
// fit on chip, ~1.06e6 fish on 148 SMs): one 512-thread CTA per SM, the CTA's
// contiguous range of fish pairs held in shared memory for all num_steps steps,
// one cooperative launch (no clusters: Nsight Compute can replay it); the CTAs
// meet at a counter barrier each step.
#ifndef FSB_SGRID_THREADS
#define FSB_SGRID_THREADS 512
#endif
constexpr int kSGridThreads = FSB_SGRID_THREADS;
struct SGridArgs {
    StepArgs base;                // state (read at launch, written back at the end), scalars, n, gfirst
    uint64_t first_step;
    uint64_t num_steps;
    double* trace;                // [num_steps]
    double* bary;                 // [3*num_steps] or nullptr
    unsigned pair_cap;            // pairs of shared-memory state per CTA (dynamic smem = 64 B each)
    EatClock* eclk;               // eat-region clock (nullptr: off)
    unsigned long long* gen;      // arrival counter, zero at launch
    Partial* parts;               // [2][grid] CTA partials (barycentre runs)
    unsigned long long* keys;     // [3] per-step max keys (max-only runs), zero at launch
};

struct EatArgs {
    SoA s;
    Scalars k;
    uint64_t n;
    const Partial* part_in;
    int world;
    double* trace_out;
    double* bary_out;
    int pdl;
    PeerXchg px;
    EatLink ec;
    FastFold ff;  // consumer side only (key_in, bp_in, bp_in_count, fold_out)
};

struct ReduceArgs {
    SoA s;
    Scalars k;
    uint64_t n;
    ReduceWs ws;
    Partial* part_out;
    PeerXchg px;
    int world;
    EatLink ec;           // producer only; t_done = kernel start (the whole pass is the max region)
};

struct InitArgs {
    SoA s;
    Scalars k;
    uint64_t n;
    uint64_t gfirst;
    double w0;  // weight_scale
};

// Small-swarm persistent kernel (one thread-block cluster, state on chip).
struct ClusterArgs {
    SoA s;
    Scalars k;
    uint64_t n;
    uint64_t gfirst;
    uint64_t first_step;
    uint64_t num_steps;
    double* trace;        // [num_steps]
    double* bary;         // [3*num_steps] or nullptr
    Partial* part_out;    // final step partial (for a later eat())
    EatClock* eclk;       // eat-region clock: per-CTA cycles summed in ns, brackets in g/c (nullptr: off)
    int sane;             // in-range state: unguarded fast paths (fsb_math.cuh "In-range mode")
};

int step_grid_blocks(int device, bool explicit_cur, bool bulk);
int step_dyn_blocks(int device);
int step_ws_blocks(int device);  // 0: the warp-specialised kernel cannot be resident
cudaError_t launch_init(const InitArgs& a, int grid, cudaStream_t st);
cudaError_t launch_step(const StepArgs& a, int grid, cudaStream_t st);
cudaError_t launch_eat(const EatArgs& a, int grid, cudaStream_t st);
cudaError_t launch_reduce(const ReduceArgs& a, int grid, cudaStream_t st);
cudaError_t launch_soa_to_aos(const SoA& s, double half_pond, uint64_t lo, uint64_t cnt, void* aos,
                              cudaStream_t st);
cudaError_t launch_aos_to_soa(const void* aos, SoA s, double half_pond, uint64_t lo, uint64_t cnt,
                              int* mismatch, cudaStream_t st);
cudaError_t launch_gather(const SoA& s, double half_pond, const uint64_t* idx, uint64_t cnt, void* aos,
                          cudaStream_t st);

// Persistent cooperative-grid run; grid = SMs x occupancy of grid_kernel.
int grid_kernel_blocks(int device);
// Co-resident clusters of the cluster-reduced grid kernel (0: not available).
int cgrid_clusters(int device);
cudaError_t launch_cgrid_run(const CGridArgs& g, int clusters, cudaStream_t st);
cudaError_t launch_grid_run(const GridArgs& g, int grid, cudaStream_t st);
// Shared-memory-resident grid: the largest number of fish pairs one CTA can
// hold (0: not available) for a grid of `grid` CTAs (one per SM).
unsigned sgrid_pair_capacity(int device, int* grid);
cudaError_t launch_sgrid_run(const SGridArgs& g, int grid, cudaStream_t st);

// Cluster kernel: returns cudaErrorNotSupported when n does not fit.
int cluster_capacity(int device, int* cluster_ctas, int* threads_per_cta);
// *ctas (may be null) receives the CTA count launched.
cudaError_t launch_cluster_run(const ClusterArgs& a, cudaStream_t st, int* ctas = nullptr);

// Self-test of the guarded fast fp64 paths vs __ddiv_rn / __dsqrt_rn on n
// generated operands; out[4] (device) accumulates the counts (see .cu).
cudaError_t launch_selftest_fast_math(uint64_t n, uint64_t seed, unsigned long long* out, cudaStream_t st);

}  // namespace fsb_dev
