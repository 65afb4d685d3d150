/*
 * fsb_b200.h -- C-ABI of the B200-native Fish School Behaviour step engine.
 *
 * Plain C: POD structs, pointers, sizes and int status codes; no CUDA, torch
 * or C++ types cross this boundary.  Implemented by
 * paper_2507_20173_b200/libfsb_b200.so (sm_100a kernels + host runtime).
 *
 * The reference has no FFI of its own: its seam for this path is the
 * parfor::Executor& parameter of the fsb phase functions
 * (/root/reference/proj/include/fsb/sim.hpp:84,110,133).  Each
 * entry point below names the reference function it replaces.  A C++ drop-in
 * that restores the reference's own types and call shapes on top of this ABI
 * is include/fsb/gpu.hpp; the ctypes binding is paper_2507_20173_b200/_native.py.
 *
 * Semantics follow the reference bit-for-bit (positions, weights, objectives
 * and the max_diff trace), computed in IEEE binary64 without FMA contraction.
 * There is no CPU fallback: every compute entry point fails with
 * FSB_ERR_CUDA when no usable sm_100 device is present.
 */
#ifndef FSB_B200_H
#define FSB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSB_B200_ABI_VERSION 2

/* Status codes.  fsb_last_error() holds a message for the calling thread. */
enum fsb_status {
    FSB_OK = 0,
    FSB_ERR_INVALID_CONFIG = 1,   /* SimConfig::validate would throw std::invalid_argument (sim.hpp:44-49) */
    FSB_ERR_INVALID_ARGUMENT = 2, /* bad pointer / size / rank */
    FSB_ERR_CUDA = 3,             /* CUDA runtime or device error (incl. no GPU) */
    FSB_ERR_NCCL = 4,             /* NCCL unavailable or failed */
    FSB_ERR_OUT_OF_MEMORY = 5,
    FSB_ERR_UNSUPPORTED = 6       /* e.g. persistent strategy for a school that does not fit */
};

/* fsb::SimConfig (sim.hpp:34-50), same field order and meaning. */
typedef struct fsb_sim_config {
    uint64_t num_fish;
    double pond_size;
    double weight_scale; /* W0: init weights uniform in [1, W0]; band [1, 2*W0] */
    uint64_t num_steps;
    uint64_t seed;
    double step_base;    /* per-axis displacement bound at unit weight */
} fsb_sim_config;

/* fsb::Fish (sim.hpp:26-32): 40 bytes, the byte layout fsb::checksum hashes. */
typedef struct fsb_fish {
    double x;
    double y;
    double weight;
    double prev_objective;
    double current_objective;
} fsb_fish;

/* fsb::SimResult timing fields (sim.hpp:125-131), device-timed.
 * seconds_eat is the reference's eat-region time: the global max only
 * (sim.hpp:103,112 -- the weight update is not timed there either).  The max
 * is fused into the step kernels, so it is measured on the device with
 * %globaltimer where it sits on the critical path: per step, from the moment
 * every fish of the step has been updated to the moment the kernel that
 * needs the global max holds it (CTA and grid reductions, the kernel boundary
 * or in-kernel grid barrier, the NCCL / peer exchange).  For the persistent
 * strategies it is the mean over CTAs of each CTA's time from its own fish
 * done to holding the max.  seconds_move = seconds_loop - seconds_eat. */
typedef struct fsb_timing {
    double seconds_total; /* init + step loop (simulate) or the step loop (run), cudaEvent */
    double seconds_move;  /* the step loop outside the eat region                        */
    double seconds_eat;   /* the eat region: the global max only (see above)             */
    double seconds_loop;  /* the step loop, cudaEvent (what the bench divides by)        */
} fsb_timing;

/* Step-loop strategies. */
enum fsb_strategy {
    FSB_STRATEGY_AUTO = 0,       /* single GPU: persistent cluster up to 16384 fish, grid while the school fits
                                    in shared memory (~1.06e6 fish), else stream; several ranks: stream */
    FSB_STRATEGY_STREAM = 1,     /* one fused step kernel per step, CUDA-graph replayed  */
    FSB_STRATEGY_PERSISTENT = 2, /* one thread-block cluster runs all steps on chip       */
    FSB_STRATEGY_GRID = 3        /* one cooperative launch of the whole grid runs all steps (single GPU,
                                    mid-size schools): up to ~1.06e6 fish the school lives in shared
                                    memory (one CTA per SM, the CTAs meet at one arrival counter per
                                    step; AUTO falls back to stream if the device refuses the
                                    co-resident launch); larger
                                    schools stay in L2, CTAs reduce inside thread-block clusters and
                                    cluster leaders meet through one global slot each */
};

/* Engine flags. */
#define FSB_FLAG_NO_ALTERNATE 0x1u /* keep tile order fixed (default reverses odd steps for L2 reuse) */
#define FSB_FLAG_FORCE_NCCL 0x2u   /* use the NCCL exchange even when world_size == 1 (testing) */
#define FSB_FLAG_NO_BULK 0x4u      /* LDG step kernel (the default; overrides FSB_FLAG_FORCE_BULK) */
#define FSB_FLAG_FORCE_BULK 0x8u   /* step kernel streams through the cp.async.bulk shared-memory ring
                                      (measured 2-3% slower than LDG in in-range mode; A/B) */
#define FSB_FLAG_NO_PDL 0x10u      /* no Programmatic Dependent Launch between graph step kernels */
#define FSB_FLAG_PEER_EXCHANGE 0x20u /* per-step exchange by NVLink peer stores from the step kernel
                                        itself (CUDA IPC windows) instead of an NCCL allgather */
#define FSB_FLAG_STATIC_TILES 0x80u  /* LDG step kernel: one static chunk per 256-thread CTA, 4 CTAs per SM */
#define FSB_FLAG_DYNAMIC_TILES 0x100u /* LDG step kernel: one 1024-thread CTA per SM whose warps claim tiles
                                        (default: dynamic at every shard size) */
#define FSB_FLAG_FLAT_GRID 0x200u   /* FSB_STRATEGY_GRID without thread-block clusters (one counter barrier) */
#define FSB_FLAG_HOST_EXCHANGE 0x400u /* world_size > 1 without NCCL: the caller moves the 4-scalar rank
                                        partials between move and eat (fsb_engine_partial /
                                        fsb_engine_set_partials), e.g. over its own MPI or gloo
                                        communicator; phase API only (run/simulate need NCCL or peers) */
#define FSB_FLAG_L2_GRID 0x800u     /* FSB_STRATEGY_GRID: keep the school in L2/HBM (cluster-reduced grid)
                                      even when it fits in shared memory (default: on chip up to ~1.06e6
                                      fish, one CTA per SM holding its pairs for all steps) */
#define FSB_FLAG_WS_TILES 0x1000u   /* compact step kernel warp-specialised: per SM one producer warp streams
                                      the state HBM -> shared memory with cp.async.bulk through a deep
                                      mbarrier ring, 31 consumer warps compute from it and store to HBM */
#define FSB_FLAG_LAST_CTA_FOLD 0x2000u /* one-rank graphs: reduce each step inside its kernel (arrival counter,
                                        the last CTA folds every CTA partial) instead of the default split fold,
                                        where every CTA red.max's its max into the step's key slot and the next
                                        kernel folds the sums beside its run (2-2.5 us per step faster) */
#define FSB_FLAG_CHECKED 0x40u     /* always evaluate the fp64 fast-path operand guards (default: elided
                                      while config and state are provably in range; results identical) */

typedef struct fsb_engine_options {
    int device;                  /* CUDA device ordinal of this shard */
    int rank;                    /* shard index in [0, world_size) */
    int world_size;              /* number of shards (one process or thread per GPU) */
    const void* nccl_unique_id;  /* 128-byte ncclUniqueId shared by all ranks (world_size > 1) */
    int strategy;                /* enum fsb_strategy */
    unsigned flags;              /* FSB_FLAG_* */
} fsb_engine_options;

typedef struct fsb_engine fsb_engine;

int fsb_abi_version(void);
const char* fsb_last_error(void);

/* SimConfig::validate (sim.hpp:44-49): FSB_OK or FSB_ERR_INVALID_CONFIG with
 * the reference's exception text in fsb_last_error(). Host-only. */
int fsb_config_validate(const fsb_sim_config* cfg);

/* Contiguous partition: rank r owns global fish [floor(rN/G), floor((r+1)N/G)). Host-only. */
int fsb_shard_range(uint64_t num_fish, int world_size, int rank, uint64_t* first, uint64_t* count);

/* FNV-1a 64 over fsb_fish bytes, continuing from h (kChecksumEmpty =
 * 0xcbf29ce484222325 to start): fsb::checksum (sim.hpp:158-176). Host-only
 * verification helper. */
uint64_t fsb_checksum_update(uint64_t h, const fsb_fish* fish, uint64_t n);

/* Number of visible CUDA devices (0 when none). */
int fsb_device_count(int* count);

/* Page-locked host buffers for fast upload/download. */
int fsb_host_alloc(void** ptr, size_t bytes);
int fsb_host_free(void* ptr);

/* 128-byte ncclUniqueId for a world_size > 1 engine (call on rank 0, broadcast). */
int fsb_nccl_unique_id(void* out, size_t len);

/* Create the engine for one shard.  Replaces constructing parfor::Executor
 * (executor.hpp:30-41) for this path.  opts may be NULL (device 0, 1 rank). */
int fsb_engine_create(const fsb_sim_config* cfg, const fsb_engine_options* opts, fsb_engine** out);
int fsb_engine_destroy(fsb_engine* e);

/* This shard's global index range. */
int fsb_engine_shard(const fsb_engine* e, uint64_t* first, uint64_t* count);

/* init_school (sim.hpp:65-79) on the device. */
int fsb_engine_init(fsb_engine* e);

/* Replace / read the shard's school (count == shard count) in fsb::Fish layout. */
int fsb_engine_upload(fsb_engine* e, const fsb_fish* fish, uint64_t count);
int fsb_engine_download(fsb_engine* e, fsb_fish* fish, uint64_t count);

/* move_phase(school, cfg, step, exec) (sim.hpp:84-99).  seconds: device time. */
int fsb_engine_move(fsb_engine* e, uint64_t step, double* seconds);

/* eat_phase(school, cfg, exec) (sim.hpp:110-123): global max of prev-cur
 * (-inf for an empty school) and the weight update when it is > 0.
 * seconds: EatResult::seconds, the max only (sim.hpp:103): the reduction tail
 * of the preceding move kernel plus this call's combine, device-timed. */
int fsb_engine_eat(fsb_engine* e, double* max_diff, double* seconds);

/* The step loop of simulate (sim.hpp:139-144) for steps
 * [first_step, first_step + num_steps): T x (move, eat), on device.
 * Strategy AUTO: the persistent cluster kernel up to 16,384 fish, the
 * cooperative grid while the school fits in shared memory (about 1.06e6
 * fish), else the graph of step kernels; if the device
 * refuses the co-resident launch the run falls back to the graph (see
 * fsb_engine_last_strategy).  An explicit PERSISTENT / GRID request fails
 * with FSB_ERR_UNSUPPORTED instead.
 * trace[num_steps] receives max_diff per step (EatResult::max_diff);
 * bary[3*num_steps] (may be NULL) the per-step sums {sum x*f, sum y*f, sum f}
 * over all shards.  timing may be NULL. */
int fsb_engine_run(fsb_engine* e, uint64_t first_step, uint64_t num_steps, double* trace,
                   double* bary, fsb_timing* timing);

/* simulate(cfg, exec) (sim.hpp:133-147): init + run(0, cfg.num_steps). */
int fsb_engine_simulate(fsb_engine* e, double* trace, double* bary, fsb_timing* timing);

/* Barycentre query (new; north_star): global f-weighted sums of the current
 * state and B = (sum x*f / sum f, sum y*f / sum f). */
int fsb_engine_barycentre(fsb_engine* e, double sums[3], double xy[2]);

/* Read n fish at arbitrary shard-local indices (Fish layout): sampled-fish
 * verification of schools too large to download whole. */
int fsb_engine_gather(fsb_engine* e, const uint64_t* local_idx, uint64_t n, fsb_fish* out);

/* FNV-1a of this shard's school continuing from h_in (checksum, sim.hpp:158). */
int fsb_engine_checksum(fsb_engine* e, uint64_t h_in, uint64_t* h_out);

/* Block until queued work is done. */
int fsb_engine_synchronize(fsb_engine* e);

/* The engine's CUDA stream (a cudaStream_t), for callers that time or order work on it. */
int fsb_engine_stream(fsb_engine* e, void** stream);

/* Measurement aid: launch the fused step kernel num_steps times eagerly with a
 * CUDA event pair around each launch; kernel_ms[k] = duration of launch k. */
int fsb_engine_time_step_kernels(fsb_engine* e, uint64_t first_step, uint64_t num_steps,
                                 double* kernel_ms);

/* Kernel launch count of the last fsb_engine_run (for bench accounting). */
int fsb_engine_last_launches(const fsb_engine* e, uint64_t* launches);

/* The step-loop strategy the last fsb_engine_run executed (enum fsb_strategy;
 * never AUTO) and, when an AUTO run had to leave its first choice because the
 * device refused to co-schedule the persistent grid or cluster (a profiler
 * replay, MPS, a shared device), the launch error that made it fall back to
 * the graph of step kernels ("" otherwise).  The string lives until the next run. */
int fsb_engine_last_strategy(const fsb_engine* e, int* strategy, const char** fallback_reason);

/* Configuration sweeps (the GPU analogue of the reference's thread-count
 * experiments, bench.hpp:79-148): set the CTA count of the compact-state step
 * and eat kernels (ctas = 0 restores the automatic SMs x occupancy grid).  Each
 * CTA owns one balanced contiguous chunk, so results do not depend on it.
 * fsb_engine_grid reports the grid in use and the threads per CTA. */
int fsb_engine_set_grid(fsb_engine* e, int ctas);
int fsb_engine_grid(const fsb_engine* e, int* ctas, int* threads_per_cta);
/* Work granularity of the claimed-tile step kernel (the dynamic-schedule chunk
 * of the reference's RunConfig, schedule.hpp; the gpu-exp2 sweep): the minimum
 * number of 32-pair groups (64 fish) per tile a warp claims, 0 = the kernel's
 * default (4).  Tiles are also never fewer than the shard needs to fit the
 * kernel's 1024 tile slots per CTA.  Results do not depend on it. */
int fsb_engine_set_tile_groups(fsb_engine* e, int groups);

/* Peer exchange (FSB_FLAG_PEER_EXCHANGE, one process per GPU): each rank
 * exports its 64-byte CUDA IPC handle of its exchange window, the caller
 * all-gathers the handles (rank order) and every rank connects.  The step
 * kernel's last CTA then writes the rank partial into every peer window over
 * NVLink and releases an epoch flag; the next step's kernel acquires the flags.
 * A single rank connects to itself at creation. */
int fsb_engine_peer_handle(fsb_engine* e, void* out, size_t len);
int fsb_engine_peer_connect(fsb_engine* e, const void* handles, size_t len);
/* The same for ranks that live in ONE process (one host thread or process
 * driving several GPUs, SURVEY 8(b) "Threading"; or several shards of one GPU):
 * ranks[q] is rank q's engine (ranks[e's rank] == e), every engine created with
 * FSB_FLAG_PEER_EXCHANGE and the same world_size.  The windows are addressed by
 * their device pointers; peer access is enabled between distinct devices.  Run
 * and simulate launch kernels that wait for the other ranks' partials, so ranks
 * sharing one GPU must use the phase API with every rank's move before any
 * rank's eat (each call returns only when its kernels have finished).  The
 * engines hold each other's window pointers: destroy them together, after the
 * last call on any of them. */
int fsb_engine_peer_connect_local(fsb_engine* e, fsb_engine* const* ranks, int n);

/* Host exchange (FSB_FLAG_HOST_EXCHANGE): the exchange step of eat_phase's
 * max (sim.hpp:110-114 -> executor.hpp:83-103), made explicit for callers
 * that bring their own communicator.  After fsb_engine_move, read this rank's
 * partial {max(prev-cur), sum x*f, sum y*f, sum f, epoch} (out[5]; epoch =
 * the exchange sequence number, equal on every rank at the same step),
 * all-gather the world_size partials in rank order, and hand them back
 * (parts[5*world_size]) before fsb_engine_eat / fsb_engine_barycentre, which
 * combine them in rank order on the device exactly as the NCCL path does.
 * set_partials rejects a set whose entry [rank] is not this rank's partial or
 * whose epochs differ (a rank that moved twice or skipped a move).  Eat
 * without a fresh set_partials fails with FSB_ERR_INVALID_ARGUMENT. */
int fsb_engine_partial(fsb_engine* e, double out[5]);
int fsb_engine_set_partials(fsb_engine* e, const double* parts, size_t count);

/* Device self-test of the guarded fast fp64 paths the step kernel uses
 * (fsb_math.cuh): n generated operands (raw bit patterns incl. NaN, inf,
 * subnormals, and the simulation's value ranges).  out[0..2] = bitwise
 * mismatches vs __ddiv_rn (hoisted divisor), __ddiv_rn (per operand) and
 * __dsqrt_rn; out[3] = guard failures on simulation-range operands. */
int fsb_selftest_fast_math(int device, uint64_t n, uint64_t seed, uint64_t out[4]);

#ifdef __cplusplus
}
#endif

#endif /* FSB_B200_H */
