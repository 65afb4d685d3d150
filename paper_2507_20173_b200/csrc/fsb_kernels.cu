// fsb_kernels.cu -- sm_100a kernels of the B200 FSB engine.
//
//   init_kernel     init_school (sim.hpp:65-79) on device, SoA stores.
//   step_kernel     ONE pass per simulation step: the previous step's eat
//                   (sim.hpp:115-120, deferred: "lazy eat"), this step's swim +
//                   objective (sim.hpp:90-98), and this step's partial
//                   max(prev-cur) (sim.hpp:112-114) plus the f-weighted
//                   barycentre sums, reduced warp -> CTA -> grid (last CTA).
//                   double2 loads/stores, two fish per thread; one static
//                   chunk per 256-thread CTA (FSB_FLAG_STATIC_TILES).
//   step_kernel_dyn the same pass, one 1024-thread CTA per SM whose warps
//                   claim tiles (round-robin stripes) and draw their RNG ahead
//                   of the loaded state (the stream strategy's default: C1-C3).
//   step_kernel_ws  the same pass warp-specialised: a cp.async.bulk producer
//                   warp streams round buffers into shared memory for 31
//                   consumer warps (FSB_FLAG_WS_TILES, opt-in).
//   step_kernel_bulk  the same pass streamed through a shared-memory ring by
//                   cp.async.bulk + mbarriers (FSB_FLAG_FORCE_BULK, A/B).
//   sgrid_kernel    all T steps in one cooperative launch with the school in
//                   shared memory, one CTA per SM (FSB_STRATEGY_GRID; AUTO
//                   16,385 to ~1.06e6 fish: C0).
//   cgrid_kernel    all T steps in one cooperative launch of 8-CTA clusters,
//                   the school in L2, reducing over DSMEM before the grid-wide
//                   exchange (FSB_FLAG_L2_GRID; AUTO's choice above the shared-memory grid until round 2).
//   grid_kernel     the same without clusters (FSB_FLAG_FLAT_GRID).
//   eat_kernel      the trailing / standalone weight update (sim.hpp:115-121).
//   reduce_kernel   max + sums of the current state without moving it (eat()
//                   after an upload).
//   cluster_kernel  small swarms: all T steps in one launch of one thread-block
//                   cluster, state in registers, per-step reduction over DSMEM
//                   (AUTO up to 16,384 fish: C4).
//   soa<->aos       Fish byte layout (sim.hpp:26-32) for upload / download.
//
// In-range runs (fsb_math.cuh) take unguarded instantiations of the hot loops:
// no operand guards, no warp vote and no call to the exact fallback path.
// Determinism: max is exact (any order).  The sums use a fixed tree for a
// fixed (n, grid, step parity), so repeated runs are bit-identical.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>

#include "fsb_kernels.cuh"
#include "fsb_math.cuh"

namespace cg = cooperative_groups;

#ifndef FSB_SPIN_ACQ
#define FSB_SPIN_ACQ 0  // A/B: acquire load on every poll of a counter barrier
#endif

namespace fsb_dev {

namespace {

__device__ __forceinline__ Partial identity() {
    Partial p;
    p.best = -INFINITY;
    p.sx = 0.0;
    p.sy = 0.0;
    p.sf = 0.0;
    return p;
}

// Combine b into a.  max uses the reference's strict '>' (executor.hpp:90).
__device__ __forceinline__ void fold(Partial& a, const Partial& b) {
    a.best = (b.best > a.best) ? b.best : a.best;
    a.sx = __dadd_rn(a.sx, b.sx);
    a.sy = __dadd_rn(a.sy, b.sy);
    a.sf = __dadd_rn(a.sf, b.sf);
}

// Fold one fish's post-move values into a thread partial.
__device__ __forceinline__ void accumulate(Partial& acc, double x, double y, double prev, double cur) {
    const double d = __dsub_rn(prev, cur);
    acc.best = (d > acc.best) ? d : acc.best;
    acc.sx = __dadd_rn(acc.sx, __dmul_rn(x, cur));
    acc.sy = __dadd_rn(acc.sy, __dmul_rn(y, cur));
    acc.sf = __dadd_rn(acc.sf, cur);
}

// Butterfly: every lane ends with the same, order-fixed result.
__device__ __forceinline__ Partial warp_reduce(Partial v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Partial u;
        u.best = __shfl_xor_sync(0xffffffffu, v.best, o);
        u.sx = __shfl_xor_sync(0xffffffffu, v.sx, o);
        u.sy = __shfl_xor_sync(0xffffffffu, v.sy, o);
        u.sf = __shfl_xor_sync(0xffffffffu, v.sf, o);
        fold(v, u);
    }
    return v;
}

// %globaltimer: ns, one clock for every SM (the eat-region clock).
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Persistent kernels: CTA 0 brackets the run with globaltimer and clock64 so
// the host can convert the per-CTA cycle counts of the eat region into ns.
__device__ __forceinline__ void eclk_bracket(EatClock* c, bool end) {
    if (c && blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned long long g = gtimer();
        const unsigned long long k = clock64();
        if (end) {
            c->g1 = g;
            c->c1 = k;
        } else {
            c->g0 = g;
            c->c0 = k;
        }
    }
}

__device__ __forceinline__ void red_max_relaxed_gpu(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block-wide reduction; the result is valid in warp 0 (all lanes).
// If stamp != nullptr, thread 0 stores the globaltimer right after the barrier
// at which every warp of the CTA has finished its fish (the eat-region start).
// `scratch` holds blockDim/32 partials.  Ends with the caller's warp 0 owning
// the value; callers __syncthreads() before reusing scratch.
__device__ __forceinline__ Partial block_reduce(Partial v, Partial* scratch,
                                                unsigned long long* stamp = nullptr, bool cycles = false) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    v = warp_reduce(v);
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (stamp && threadIdx.x == 0) *stamp = cycles ? clock64() : gtimer();
    Partial r = identity();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        if (lane < nw) r = scratch[lane];
        r = warp_reduce(r);
    }
    return r;
}

// Max-only reductions (the persistent kernel when no barycentre is requested).
// Exact fp64 max over a warp with two REDUX (u32) steps instead of five
// shuffle levels: an order-preserving 64-bit key (sign-folded), max of the
// high words, then max of the low words among the lanes that hold that high
// word.  NaN maps to the key of -inf, so -- as in the reference's strict '>'
// fold (executor.hpp:90) -- it never wins.
// The max is carried as a key through a multi-level reduction (the persistent
// cluster kernel): encode once per thread, decode once after the last level.
constexpr unsigned long long kKeyNegInf = ~0xfff0000000000000ull;  // max_key(-inf)
__device__ __forceinline__ unsigned long long max_key(double v) {
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    if (v != v) b = 0xfff0000000000000ull;  // NaN -> -inf
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(unsigned long long m) {
    const unsigned long long bits = (m >> 63) ? (m & 0x7fffffffffffffffull) : ~m;
    return __longlong_as_double(static_cast<long long>(bits));
}
__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long key) {
    const unsigned hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(key >> 32));
    const unsigned lo = __reduce_max_sync(
        0xffffffffu, static_cast<unsigned>(key >> 32) == hi ? static_cast<unsigned>(key) : 0u);
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}
// valid in warp 0 (all lanes)
__device__ __forceinline__ unsigned long long block_max_key(unsigned long long key, unsigned long long* scratch,
                                                            unsigned long long* stamp = nullptr, bool cycles = false) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    key = warp_max_key(key);
    if (lane == 0) scratch[warp] = key;
    __syncthreads();
    if (stamp && threadIdx.x == 0) *stamp = cycles ? clock64() : gtimer();
    unsigned long long r = kKeyNegInf;
    if (warp == 0) {
        if (lane < (int)(blockDim.x >> 5)) r = scratch[lane];
        r = warp_max_key(r);
    }
    return r;
}

__device__ __forceinline__ Partial load_cg(const Partial* p) {
    const double2* q = reinterpret_cast<const double2*>(p);
    const double2 a = __ldcg(q);
    const double2 b = __ldcg(q + 1);
    Partial r;
    r.best = a.x;
    r.sx = a.y;
    r.sy = b.x;
    r.sf = b.y;
    return r;
}

__device__ __forceinline__ void store_partial(Partial* p, const Partial& v) {
    double2* q = reinterpret_cast<double2*>(p);
    q[0] = make_double2(v.best, v.sx);
    q[1] = make_double2(v.sy, v.sf);
}

__device__ __forceinline__ uint64_t epoch_of(const PeerXchg& px, uint64_t add) {
    return add ? (px.seq_ptr ? *px.seq_ptr : 0ull) + add : 0ull;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void red_add_release_gpu(unsigned long long* p, unsigned long long v) {
    asm volatile("red.add.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Spin with relaxed polls (no fence per poll) until *p >= target, then one
// acquire fence: the arrivals' releases synchronise with it.
__device__ __forceinline__ void spin_until_gpu(const unsigned long long* p, unsigned long long target) {
    while (FSB_SPIN_ACQ ? ld_acquire_gpu(p) < target : ld_relaxed_gpu(p) < target) {
    }
    if (!FSB_SPIN_ACQ) asm volatile("fence.acquire.gpu;" ::: "memory");
}

// Peer exchange, producer side (warp 0 of the last CTA): the rank partial into
// every peer's window, then the epoch flag with release semantics.
__device__ __forceinline__ void push_to_peers(const PeerXchg& px, int world, uint64_t epoch, const Partial& tot) {
    FSB_CHECK(world <= kMaxRanks && px.rank >= 0 && px.rank < world);
    const int b = (int)(epoch & 1);
    for (int q = threadIdx.x; q < world; q += 32) {
        PeerWindow* w = px.peers[q];
        store_partial(&w->slots[b][px.rank], tot);
        st_release_sys(&w->flags[b][px.rank], epoch);  // orders the slot stores before the flag
    }
}

// Peer exchange, consumer side (every CTA): thread 0 acquires the epoch's
// flags of all ranks from the local window, then every thread combines the
// slots in rank order.
__device__ __forceinline__ Partial wait_and_combine_peers(const PeerXchg& px, int world, uint64_t epoch) {
    __shared__ Partial combined;
    const int b = (int)(epoch & 1);
    PeerWindow* w = px.local;
    if (threadIdx.x == 0) {
        Partial r = identity();
        const unsigned long long t0 = gtimer();
        bool lost = false;
        for (int q = 0; q < world && !lost; ++q) {
            while (ld_acquire_sys(&w->flags[b][q]) != epoch) {
                __nanosleep(64);
                // failure detection: a rank that never publishes (crashed, or not
                // launched) must not hang this GPU: give up, mark the window for
                // the host (the call fails), and combine nothing -- no max, so
                // this kernel applies no eat and a retry once the rank has
                // published still gives the right state
                if (gtimer() - t0 > px.timeout_ns) {
                    w->fault = epoch;
                    lost = true;
                    break;
                }
            }
            if (lost) break;
            Partial v;
            v.best = ld_relaxed_sys(&w->slots[b][q].best);
            v.sx = ld_relaxed_sys(&w->slots[b][q].sx);
            v.sy = ld_relaxed_sys(&w->slots[b][q].sy);
            v.sf = ld_relaxed_sys(&w->slots[b][q].sf);
            fold(r, v);
        }
        combined = lost ? identity() : r;
    }
    __syncthreads();
    return combined;
}

// CTA partial -> global; the last CTA to arrive combines all CTA partials in
// index order and publishes this rank's partial (and, with a peer exchange,
// pushes it to every rank).
// grid_publish: the CTA total `blk` (valid in thread 0) joins the grid reduction.
// t_done (thread 0): when this CTA's fish were all updated (eat-region clock).
__device__ __forceinline__ void grid_publish(const Partial& blk, const ReduceWs& ws, Partial* part_out,
                                             const PeerXchg& px, int world, EatStamp* ec_out,
                                             unsigned long long t_done, const FastFold* ff = nullptr) {
    __shared__ Partial scratch[32];
    __shared__ bool am_last;
    if (ff && ff->key_out) {  // split fold: nothing to wait for; the kernel boundary publishes both
        if (threadIdx.x == 0) {
            store_partial(&ff->bp_out[blockIdx.x], blk);
            red_max_relaxed_gpu(ff->key_out, max_key(blk.best));
            if (ec_out) red_max_relaxed_gpu(&ec_out->t_done, t_done);
        }
        return;
    }
    if (threadIdx.x == 0) {
        FSB_CHECK(blockIdx.x < ws.cap);
        store_partial(&ws.block_part[blockIdx.x], blk);
        if (ec_out) red_max_relaxed_gpu(&ec_out->t_done, t_done);  // ordered before the release below
        // release: this CTA's partial before its arrival; acquire: the last
        // arriver sees every partial (the counter's release sequence).  The
        // other threads of the last CTA are ordered after it by the barrier
        // and read with ld.cg (L2), so no fence of their own.
        am_last = (atom_add_acq_rel_gpu(ws.counter, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    Partial acc = identity();
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) fold(acc, load_cg(&ws.block_part[i]));
    __syncthreads();  // scratch reuse
    const Partial tot = block_reduce(acc, scratch);
    if (threadIdx.x == 0) {
        store_partial(part_out, tot);
        *ws.counter = 0u;  // ready for the next launch
        if (ec_out) ec_out->t_pub = gtimer();
    }
    const uint64_t epoch = px.peers ? epoch_of(px, px.out_add) : 0ull;
    if (epoch && threadIdx.x < 32) push_to_peers(px, world, epoch, tot);
}

// t_start != 0: the eat region of this CTA starts there (reduce_kernel: the
// whole pass is the max); else when its fish are done (block barrier).
__device__ __forceinline__ void grid_finish(const Partial& local, const ReduceWs& ws, Partial* part_out,
                                            const PeerXchg& px, int world, EatStamp* ec_out,
                                            unsigned long long t_start = 0) {
    __shared__ Partial scratch[32];
    unsigned long long t_done = t_start;
    const Partial blk = block_reduce(local, scratch, (ec_out && !t_start) ? &t_done : nullptr);
    grid_publish(blk, ws, part_out, px, world, ec_out, t_done);
}

// Programmatic Dependent Launch: block until the predecessor grid has completed
// and flushed (no-op when not launched as a dependent), then let the next
// kernel in the stream be scheduled as our CTAs retire.
__device__ __forceinline__ void pdl_wait_and_release() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Combine the ranks' partials of the previous step in rank order: from
// part_in (single rank / NCCL allgather) or from the peer window.
__device__ __forceinline__ Partial combine_prev(const Partial* part_in, int world, const PeerXchg& px) {
    if (px.peers) {
        const uint64_t epoch = epoch_of(px, px.in_add);
        return epoch ? wait_and_combine_peers(px, world, epoch) : identity();
    }
    Partial r = identity();
    if (part_in) {
        for (int k = 0; k < world; ++k) fold(r, part_in[k]);
    }
    return r;
}

// Block 0, thread 0 of the kernel that consumes the previous step's max: the
// trace entries, and the eat-region clock (t_start: this kernel's entry).
__device__ __forceinline__ void publish_prev(const Partial& prev, double* trace_out, double* bary_out,
                                             const EatLink& ec, unsigned long long t_start) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (ec.in && ec.ns) {
            const unsigned long long t_have = gtimer();
            const EatStamp st = *ec.in;
            const unsigned long long region =
                ec.phase ? (st.t_pub - st.t_done) + (t_have - t_start) : t_have - st.t_done;
            // (t_pub is the last CTA's publish stamp: used by the phase API only, absent with the split fold)
            if (st.t_done && (!ec.phase || st.t_done <= st.t_pub) && st.t_done <= t_have) *ec.ns += region;
            ec.in->t_done = 0ull;  // re-armed for the producer two steps on
        }
        if (trace_out) *trace_out = prev.best;
        if (bary_out) {
            bary_out[0] = prev.sx;
            bary_out[1] = prev.sy;
            bary_out[2] = prev.sf;
        }
    }
}

// Split fold, consumer side.  Every CTA: the previous step's max from its key
// slot (after the kernel boundary; identity sums -- only the max feeds the eat).
__device__ __forceinline__ Partial prev_from_key(const FastFold& ff) {
    Partial r = identity();
    r.best = key_value(__ldcg(ff.key_in));
    return r;
}
// One warp of CTA 0: the CTA partials of the previous step folded in index order
// (lane l takes l, l + 32, ...; then the fixed butterfly) into the rank partial
// and the barycentre output; zeroes the next step's key slot.
// (out of line: inlined into the step kernel it cost the hot loop 7 % more instructions -- register moves)
__device__ __noinline__ void fold_prev_outputs(const Partial* bp_in, unsigned bp_in_count, Partial* fold_out,
                                               unsigned long long* key_reset, double* bary_out) {
    const unsigned lane = threadIdx.x & 31;
    Partial f = identity();
    for (unsigned i = lane; i < bp_in_count; i += 32) fold(f, load_cg(&bp_in[i]));
    f = warp_reduce(f);
    if (lane == 0) {
        store_partial(fold_out, f);
        if (bary_out) {
            bary_out[0] = f.sx;
            bary_out[1] = f.sy;
            bary_out[2] = f.sf;
        }
        if (key_reset) *key_reset = 0ull;
    }
}

__device__ __forceinline__ StepParams params_of(const Scalars& k) {
    StepParams P;
    P.pond = k.pond;
    P.half_pond = k.half_pond;
    P.step_base = k.step_base;
    P.w_max = k.w_max;
    P.seed = k.seed;
    P.zero = k.zero;
    return P;
}

// One fish of the fused step.  cur is this fish's current objective before
// the step (recomputed or explicit).  Returns nothing; updates state + acc.
__device__ __forceinline__ void fused_fish(double& x, double& y, double& w, double& p, double cur,
                                           bool eat, const SharedDivisor& M, uint64_t gi,
                                           uint64_t step, const StepParams& P, Partial& acc) {
    if (eat) w = eat_weight(w, p, cur, M, P.w_max);          // sim.hpp:115-120 (step-1)
    const double cn = swim(x, y, w, fold_in(P.seed, gi), step, P);  // sim.hpp:90-97
    p = cur;                                                   // sim.hpp:96
    accumulate(acc, x, y, cur, cn);                            // sim.hpp:112-114
}

// The same fish update on the guarded fast paths: returns the new objective
// and ANDs the operand guards into ok (no accumulation: the caller folds the
// fish into its partial once the result is final).
template <bool kSane>
__device__ __forceinline__ double fused_fish_guarded(double& x, double& y, double& w, double& p,
                                                     double cur, bool eat, const SharedDivisor& M,
                                                     uint64_t gi, uint64_t step, const StepParams& P,
                                                     bool& ok) {
    if (eat) w = eat_weight_guarded<kSane>(w, p, cur, M, P.w_max, ok);
    const double cn = swim_guarded<kSane>(x, y, w, fold_in(P.seed, gi), step, P, ok);
    p = cur;
    return cn;
}

// ... and on the exact intrinsics (the fallback for a failed guard; kept out
// of line so the hot loop carries none of its registers).
struct FishOut {
    double x, y, w, p, cn;
};

__device__ __noinline__ FishOut fused_fish_exact(double x, double y, double w, double p, double cur,
                                                 bool eat, double M, uint64_t gi, uint64_t step,
                                                 StepParams P) {
    if (eat) w = eat_weight(w, p, cur, M, P.w_max);
    const double cn = swim(x, y, w, fold_in(P.seed, gi), step, P);
    return FishOut{x, y, w, cur, cn};
}

// Where a pair's original state can be re-read (global SoA or a smem stage).
struct SoA2 {
    const double2* x;
    const double2* y;
    const double2* w;
    const double2* p;
    const double2* c;
};

// U pairs of fish through the fused step.  X..Q hold each pair's state on
// entry and the new state on exit; pair u is fish gi[u], gi[u]+1 and can be
// re-read from src at index k[u].  All 2U fish run their guarded fast paths
// first (independent chains the scheduler interleaves), then ONE warp vote:
// a pair whose guard failed is recomputed with the exact intrinsics.  Only
// then are the fish folded into the thread partial.  kSane: the state is in
// range (fsb_math.cuh "In-range mode"); the eat divisor -- the global max,
// which other ranks' states feed -- is range-checked here, once per call.
// kPre: H[2u + f] holds fold_in(seed, fish) of pair u's fish f (the
// step-independent RNG prefix, kept by the caller); the draws are made first as
// with kRngFirst, without its scheduling fence.
// Pair u's two draws as the 53-bit integers of swim_units_guarded: fish 2u+f
// of the call draws (U0[u][f], U1[u][f]).
template <int U>
struct PairDraws {
    double U0[U][2], U1[U][2];
};

template <int U>
__device__ __forceinline__ void draw_pairs(PairDraws<U>& d, const uint64_t (&gi)[U], uint64_t seed, uint64_t step) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const uint64_t h_step = fold_in(fold_in(seed, gi[u] + f), step);
            d.U0[u][f] = __ull2double_rn(fold_in(h_step, 0) >> 11);
            d.U1[u][f] = __ull2double_rn(fold_in(h_step, 1) >> 11);
        }
    }
}

// kDrawn: DR holds the pairs' draws, made by the caller ahead of the state
// (step_kernel_ws draws before it waits for the stage to land).
// kFast (with kSane and kRngFirst): the caller has checked the divisor's range
// for the launch, so nothing is guarded -- sqrt_sane, unguarded divisions, no
// vote and no fallback call in the caller's loop.
template <bool kExplicitCur, int U, bool kSane, bool kRngFirst = false, bool kPre = false, bool kDrawn = false,
          bool kFast = false>
__device__ __forceinline__ void fused_pairs(double2 (&X)[U], double2 (&Y)[U], double2 (&W)[U],
                                            double2 (&Q)[U], const double2 (&C)[U], const bool (&valid)[U],
                                            const SoA2& src, const uint64_t (&k)[U], const uint64_t (&gi)[U],
                                            const StepParams& P, bool eat, const SharedDivisor& M,
                                            uint64_t step, Partial& acc, const uint64_t* H = nullptr,
                                            const PairDraws<U>* DR = nullptr) {
    bool ok[U];
    double n0[U], n1[U];
    bool all_ok = true;
    // M.b in [2^-506, 2^502] (positive: as an integer range on its bits)
    const uint64_t mb = static_cast<uint64_t>(__double_as_longlong(M.b));
    const bool ok0 = !kSane || !eat || (mb - 0x2050000000000000ull <= 0x3F00000000000000ull);
    if (kDrawn) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ok[u] = ok0;
            if (valid[u]) {
                const double c0 = kExplicitCur ? C[u].x : objective_guarded<kSane>(X[u].x, Y[u].x, P.half_pond, ok[u]);
                const double c1 = kExplicitCur ? C[u].y : objective_guarded<kSane>(X[u].y, Y[u].y, P.half_pond, ok[u]);
                double w0 = W[u].x, w1 = W[u].y;
                if (eat) w0 = eat_weight_guarded<kSane>(w0, Q[u].x, c0, M, P.w_max, ok[u]);
                if (eat) w1 = eat_weight_guarded<kSane>(w1, Q[u].y, c1, M, P.w_max, ok[u]);
                W[u] = make_double2(w0, w1);
                n0[u] = swim_units_guarded<kSane>(X[u].x, Y[u].x, w0, DR->U0[u][0], DR->U1[u][0], P, ok[u]);
                n1[u] = swim_units_guarded<kSane>(X[u].y, Y[u].y, w1, DR->U0[u][1], DR->U1[u][1], P, ok[u]);
                Q[u] = make_double2(c0, c1);
                all_ok &= ok[u];
            }
        }
    } else if (kRngFirst || kPre) {
        // Every fish's units first: they depend on (seed, fish, step) only, so the
        // chains run while the state loads are in flight.  The loaded values then
        // pass through a fake dependency on the last draws (high word | (bits &
        // zero), zero == 0 at run time), which keeps ptxas from hoisting their
        // arithmetic above the chains.  U0/U1 hold the 53-bit integers of the
        // draws (swim_units_guarded scales them).  Used by the claimed-tile kernel (HBM-latency bound:
        // C2 2.8% faster); the L2-resident cluster grid runs 22% slower with it.
        double U0[U][2], U1[U][2];
        unsigned dep = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                const uint64_t h_step = fold_in(kPre ? H[2 * u + f] : fold_in(P.seed, gi[u] + f), step);
                const uint64_t b0 = fold_in(h_step, 0);
                const uint64_t b1 = fold_in(h_step, 1);
                U0[u][f] = __ull2double_rn(b0 >> 11);
                U1[u][f] = __ull2double_rn(b1 >> 11);
                dep |= static_cast<unsigned>(b1 >> 11);  // a word the conversion computes anyway
            }
        }
        dep = kPre ? 0u : (dep & static_cast<unsigned>(P.zero));
        // the fence goes into high words (one LOP3 each)
        auto fenced = [dep](double v) {
            return __hiloint2double(__double2hiint(v) | static_cast<int>(dep), __double2loint(v));
        };
        const double hp = fenced(P.half_pond);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ok[u] = ok0;
            if (kFast && valid[u]) {
                const double c0 = kExplicitCur ? C[u].x : objective_sane(X[u].x, Y[u].x, hp);
                const double c1 = kExplicitCur ? C[u].y : objective_sane(X[u].y, Y[u].y, hp);
                double w0 = fenced(W[u].x), w1 = fenced(W[u].y), p0 = Q[u].x, p1 = Q[u].y;
                n0[u] = fish_sane_cur(X[u].x, Y[u].x, w0, p0, c0, eat, M, U0[u][0], U1[u][0], P);
                n1[u] = fish_sane_cur(X[u].y, Y[u].y, w1, p1, c1, eat, M, U0[u][1], U1[u][1], P);
                W[u] = make_double2(w0, w1);
                Q[u] = make_double2(p0, p1);
            } else if (valid[u]) {
                const double c0 = kExplicitCur ? C[u].x : objective_guarded<kSane>(X[u].x, Y[u].x, hp, ok[u]);
                const double c1 = kExplicitCur ? C[u].y : objective_guarded<kSane>(X[u].y, Y[u].y, hp, ok[u]);
                double w0 = fenced(W[u].x);
                double w1 = fenced(W[u].y);
                if (eat) w0 = eat_weight_guarded<kSane>(w0, Q[u].x, c0, M, P.w_max, ok[u]);
                if (eat) w1 = eat_weight_guarded<kSane>(w1, Q[u].y, c1, M, P.w_max, ok[u]);
                W[u] = make_double2(w0, w1);
                n0[u] = swim_units_guarded<kSane>(X[u].x, Y[u].x, w0, U0[u][0], U1[u][0], P, ok[u]);
                n1[u] = swim_units_guarded<kSane>(X[u].y, Y[u].y, w1, U0[u][1], U1[u][1], P, ok[u]);
                Q[u] = make_double2(c0, c1);
                all_ok &= ok[u];
            }
        }
    } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ok[u] = ok0;
            if (valid[u]) {
                const double c0 =
                    kExplicitCur ? C[u].x : objective_guarded<kSane>(X[u].x, Y[u].x, P.half_pond, ok[u]);
                const double c1 =
                    kExplicitCur ? C[u].y : objective_guarded<kSane>(X[u].y, Y[u].y, P.half_pond, ok[u]);
                n0[u] = fused_fish_guarded<kSane>(X[u].x, Y[u].x, W[u].x, Q[u].x, c0, eat, M, gi[u], step, P, ok[u]);
                n1[u] = fused_fish_guarded<kSane>(X[u].y, Y[u].y, W[u].y, Q[u].y, c1, eat, M, gi[u] + 1, step, P,
                                                  ok[u]);
                all_ok &= ok[u];
            }
        }
    }
    if (!kFast && __any_sync(__activemask(), !all_ok)) {  // never taken for in-range simulation values
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (valid[u] && !ok[u]) {
                const uint64_t j = k[u];
                const double2 x0 = src.x[j], y0 = src.y[j], w0 = src.w[j], p0 = src.p[j];
                const double e0 = kExplicitCur ? src.c[j].x : objective(x0.x, y0.x, P.half_pond);
                const double e1 = kExplicitCur ? src.c[j].y : objective(x0.y, y0.y, P.half_pond);
                const FishOut f0 = fused_fish_exact(x0.x, y0.x, w0.x, p0.x, e0, eat, M.b, gi[u], step, P);
                const FishOut f1 = fused_fish_exact(x0.y, y0.y, w0.y, p0.y, e1, eat, M.b, gi[u] + 1, step, P);
                X[u] = make_double2(f0.x, f1.x);
                Y[u] = make_double2(f0.y, f1.y);
                W[u] = make_double2(f0.w, f1.w);
                Q[u] = make_double2(f0.p, f1.p);
                n0[u] = f0.cn;
                n1[u] = f1.cn;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (valid[u]) {
            accumulate(acc, X[u].x, Y[u].x, Q[u].x, n0[u]);
            accumulate(acc, X[u].y, Y[u].y, Q[u].y, n1[u]);
        }
    }
}

// In-range state and an in-range divisor (the global max, which other ranks'
// states feed: checked once per step) leave nothing to guard.
template <bool kSane>
__device__ __forceinline__ bool no_guards(bool eat, const SharedDivisor& M) {
    const uint64_t mb = static_cast<uint64_t>(__double_as_longlong(M.b));
    return kSane && (!eat || mb - 0x2050000000000000ull <= 0x3F00000000000000ull);
}

// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kThreads) init_kernel(const InitArgs a) {
    const StepParams P = params_of(a.k);
    const uint64_t init_step = ~0ull;  // kInitStep, rng.hpp:27
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
        const uint64_t h = fold_in(fold_in(P.seed, a.gfirst + i), init_step);
        const double x = uniform(unit_from_bits(fold_in(h, 0)), 0.0, P.pond);
        const double y = uniform(unit_from_bits(fold_in(h, 1)), 0.0, P.pond);
        const double w = uniform(unit_from_bits(fold_in(h, 2)), 1.0, a.w0);
        a.s.x[i] = x;
        a.s.y[i] = y;
        a.s.w[i] = w;
        a.s.p[i] = objective(x, y, P.half_pond);  // prev = cur (sim.hpp:76-77)
    }
}

// This CTA's share of one fused step (LDG path): its balanced chunk of pairs,
// plus the odd tail fish on CTA 0.  Folds every fish into acc.
template <bool kExplicitCur, bool kSane>
__device__ __forceinline__ void step_chunk(const StepArgs& a, const StepParams& P, bool eat,
                                           const SharedDivisor& M, uint64_t step, Partial& acc) {
    const uint64_t n = a.n;
    const uint64_t npairs = n >> 1;
    const bool rev = a.alternate && (step & 1ull);

    // Each CTA owns one balanced contiguous chunk of pairs (boundaries aligned
    // to 64 pairs = 1 KB per array), walked in sub-tiles of kTilePairs.  Odd
    // steps walk it backwards, so the sub-tiles a CTA touched last in step t
    // (still in L2) are the first it reads in step t+1.
    constexpr uint64_t kAlign = 64;
    const uint64_t nblk = (npairs + kAlign - 1) / kAlign;
    const uint64_t lo = (nblk * blockIdx.x / gridDim.x) * kAlign;
    uint64_t hi = (nblk * (blockIdx.x + 1) / gridDim.x) * kAlign;
    if (hi > npairs) hi = npairs;
    const uint64_t nsub = hi > lo ? (hi - lo + kTilePairs - 1) / kTilePairs : 0;
    FSB_CHECK(lo <= npairs || nsub == 0);

    double2* X2 = reinterpret_cast<double2*>(a.s.x);
    double2* Y2 = reinterpret_cast<double2*>(a.s.y);
    double2* W2 = reinterpret_cast<double2*>(a.s.w);
    double2* P2 = reinterpret_cast<double2*>(a.s.p);
    const double2* C2 = reinterpret_cast<const double2*>(a.s.c);

    for (uint64_t j = 0; j < nsub; ++j) {
        const uint64_t sub = rev ? nsub - 1 - j : j;
        const uint64_t base = lo + sub * kTilePairs + threadIdx.x;
        double2 X[kPairsPerThread], Y[kPairsPerThread], W[kPairsPerThread], Q[kPairsPerThread],
            C[kPairsPerThread];
        bool valid[kPairsPerThread];
        uint64_t qs[kPairsPerThread], gi[kPairsPerThread];
#pragma unroll
        for (int u = 0; u < kPairsPerThread; ++u) {
            const uint64_t q = base + (uint64_t)u * kStepThreads;
            qs[u] = q;
            gi[u] = a.gfirst + 2 * q;
            valid[u] = q < hi;
            if (valid[u]) {
                X[u] = X2[q];
                Y[u] = Y2[q];
                W[u] = W2[q];
                Q[u] = P2[q];
                if (kExplicitCur) C[u] = C2[q];
            }
        }
        const SoA2 src{X2, Y2, W2, P2, C2};
        fused_pairs<kExplicitCur, kPairsPerThread, kSane>(X, Y, W, Q, C, valid, src, qs, gi, P, eat, M, step, acc);
#pragma unroll
        for (int u = 0; u < kPairsPerThread; ++u) {
            const uint64_t q = qs[u];
            if (valid[u]) {
                X2[q] = X[u];
                Y2[q] = Y[u];
                W2[q] = W[u];
                P2[q] = Q[u];
            }
        }
    }
    if ((n & 1ull) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd tail fish
        const uint64_t i = n - 1;
        double x = a.s.x[i], y = a.s.y[i], w = a.s.w[i], p = a.s.p[i];
        const double c = kExplicitCur ? a.s.c[i] : objective(x, y, P.half_pond);
        fused_fish(x, y, w, p, c, eat, M, a.gfirst + i, step, P, acc);
        a.s.x[i] = x;
        a.s.y[i] = y;
        a.s.w[i] = w;
        a.s.p[i] = p;
    }
}


template <bool kExplicitCur, bool kSane>
__global__ void __launch_bounds__(kStepThreads, FSB_MIN_BLOCKS) step_kernel(const StepArgs a) {
    const StepParams P = params_of(a.k);
    const unsigned long long t_start = (a.ec.phase && blockIdx.x == 0 && threadIdx.x == 0) ? gtimer() : 0ull;
    pdl_wait_and_release();
    const Partial prev = combine_prev(a.part_in, a.world, a.px);
    publish_prev(prev, a.trace_out, a.bary_out, a.ec, t_start);
    const bool eat = prev.best > 0.0;  // sim.hpp:115
    const SharedDivisor M = make_divisor(eat ? prev.best : 1.0);
    const uint64_t step = (a.step_ptr ? *a.step_ptr : 0ull) + a.step_add;
    Partial acc = identity();
    step_chunk<kExplicitCur, kSane>(a, P, eat, M, step, acc);
    grid_finish(acc, a.ws, a.part_out, a.px, a.world, a.ec.out);
}

// ---------------------------------------------------------------------------
// step_kernel_dyn: the same fused pass, one 1024-thread CTA per SM, with the
// CTA's share cut into at most kDynTiles tiles that its warps CLAIM from a
// shared-memory counter.  With several CTAs per SM the oldest ones win the
// warp scheduler and the last CTA finishes alone at low occupancy (a 90-120 us
// spread across CTAs of one step at 1e7 fish, profiles/r03_grid_ctas.jsonl);
// claiming keeps every warp busy until the share is done.  The share is a set
// of stripes of >= kDynMinGroups 32-pair groups dealt round-robin to the CTAs,
// so all SMs stream one moving front of the arrays (0-3% faster at 1e7 fish
// than one contiguous chunk per CTA; the memory-only probe
// shows 3%, profiles/r04_memory_bound_probe.jsonl).  Each tile's partial is
// accumulated in a fixed order by whichever warp takes it and stored in its own
// slot, and the slots are folded in tile order, so the sums stay
// deterministic.  Odd steps claim tiles from the end, so the front runs
// backwards over the lines the previous step wrote last (L2 reuse).
#ifndef FSB_DYN_FAST
#define FSB_DYN_FAST 1  // A/B: 0 = the guarded loop (ok flags, warp vote, fallback call) in in-range mode too
#endif
#ifndef FSB_DYN_FULL
#define FSB_DYN_FULL 1  // A/B: 0 = the unguarded loop with 64-bit pair indices and the per-pair range predicate
#endif
// The claimed-tile loop of step_kernel_dyn for one warp (see there).  kFast:
// in-range state and divisor, no guards and no fallback call in the loop.
// kFull (with kFast): s_ghi counts full 32-pair groups only and the shard has fewer than 2^32 pairs.
template <bool kExplicitCur, bool kSane, bool kFast, bool kFull = false>
__device__ __forceinline__ void dyn_tiles(const StepArgs& a, const StepParams& P, bool eat, const SharedDivisor& M,
                                          uint64_t step, bool rev, Partial* tile_part, unsigned& next_tile,
                                          const unsigned& s_ghi, const unsigned& s_gpt, const unsigned& s_ntiles) {
    const uint64_t npairs = a.n >> 1;
    double2* X2 = reinterpret_cast<double2*>(a.s.x);
    double2* Y2 = reinterpret_cast<double2*>(a.s.y);
    double2* W2 = reinterpret_cast<double2*>(a.s.w);
    double2* P2 = reinterpret_cast<double2*>(a.s.p);
    const double2* C2 = reinterpret_cast<const double2*>(a.s.c);
    const SoA2 src{X2, Y2, W2, P2, C2};
    const unsigned lane = threadIdx.x & 31;
    // one loop over groups; a warp claims its next tile when the current one
    // is exhausted (warp-uniform branch), flushing the finished tile's partial
    unsigned grp = 0, gend = 0, tile = ~0u;
    Partial acc = identity();
    const bool live = P.zero == 0;  // true (see kFull below)
    for (;;) {
        if (grp == gend) {
            if (tile != ~0u) {
                const Partial tp = warp_reduce(acc);
                if (lane == 0) tile_part[tile] = tp;
                acc = identity();
            }
            unsigned claim = 0;
            if (lane == 0) claim = atomicAdd(&next_tile, 1u);
            claim = __shfl_sync(0xffffffffu, claim, 0);
            const unsigned nt = *(volatile const unsigned*)&s_ntiles;
            if (claim >= nt) break;
            tile = rev ? nt - 1 - claim : claim;
            FSB_CHECK(nt <= (unsigned)kDynTiles && tile < nt);
            const unsigned gpt_ = *(volatile const unsigned*)&s_gpt;
            const unsigned gh = *(volatile const unsigned*)&s_ghi;
            grp = (tile * gridDim.x + blockIdx.x) * gpt_;
            gend = (grp + gpt_ < gh) ? grp + gpt_ : gh;
        }
        if (kFull) {
            // Full groups only (the caller clipped s_ghi to them and takes the
            // ragged last group itself), and fewer than 2^32 pairs: no range
            // predicate, and every address is one IMAD.WIDE.U32 of a 32-bit index.
            const unsigned q = grp * 32u + lane;
            // `live` is always true but opaque to the compiler: the arithmetic stays in
            // its own basic block behind the four loads.  With a compile-time-true
            // predicate ptxas sinks the w and p loads into the RNG chains to save
            // registers, and the step runs 6 % slower (profiles/round2_ab_dyn_full.jsonl).
            double2 X[1], Y[1], W[1], Q[1], C[1];
            const bool valid[1] = {live};
            if (valid[0]) {
                X[0] = X2[q];
                Y[0] = Y2[q];
                W[0] = W2[q];
                Q[0] = P2[q];
                if (kExplicitCur) C[0] = C2[q];
            }
            const uint64_t qs[1] = {q}, gi[1] = {a.gfirst + 2ull * q};
            fused_pairs<kExplicitCur, 1, kSane, true, false, false, kFast>(X, Y, W, Q, C, valid, src, qs, gi, P, eat,
                                                                           M, step, acc);
            if (valid[0]) {
                X2[q] = X[0];
                Y2[q] = Y[0];
                W2[q] = W[0];
                P2[q] = Q[0];
            }
            ++grp;
            continue;
        }
        const uint64_t q = (uint64_t)grp * 32 + lane;
        double2 X[1], Y[1], W[1], Q[1], C[1];
        const bool valid[1] = {q < npairs};
        const uint64_t qs[1] = {q}, gi[1] = {a.gfirst + 2 * q};
        if (valid[0]) {
            X[0] = X2[q];
            Y[0] = Y2[q];
            W[0] = W2[q];
            Q[0] = P2[q];
            if (kExplicitCur) C[0] = C2[q];
        }
        fused_pairs<kExplicitCur, 1, kSane, true, false, false, kFast>(X, Y, W, Q, C, valid, src, qs, gi, P, eat, M,
                                                                       step, acc);
        if (valid[0]) {
            X2[q] = X[0];
            Y2[q] = Y[0];
            W2[q] = W[0];
            P2[q] = Q[0];
        }
        ++grp;
    }
}

template <bool kExplicitCur, bool kSane>
__global__ void __launch_bounds__(kDynThreads, FSB_DYN_MIN_BLOCKS) step_kernel_dyn(const StepArgs a) {
    __shared__ Partial tile_part[kDynTiles];
    // tile bookkeeping lives in shared memory, not in registers: the hot loop
    // is at the 64-register limit of 1024-thread CTAs
    __shared__ unsigned next_tile, s_ghi, s_gpt, s_ntiles;
    const StepParams P = params_of(a.k);
    const unsigned long long t_start = (a.ec.phase && blockIdx.x == 0 && threadIdx.x == 0) ? gtimer() : 0ull;
    // Everything that does not depend on the previous kernel comes BEFORE the
    // programmatic-dependency wait, in the shadow of that kernel's tail: the
    // step index (written by the graph's first node, long complete), the tile
    // geometry with its 64-bit divisions, the shared-memory bookkeeping.
    const uint64_t step = (a.step_ptr ? *a.step_ptr : 0ull) + a.step_add;
    const uint64_t n = a.n;
    const uint64_t npairs = n >> 1;
    const bool rev = a.alternate && (step & 1ull);
    // balanced contiguous chunk of 32-pair groups (32-bit group indices: up
    // to 2^37 fish per shard); tiles of gpt groups
    // In-range launches of fewer than 2^32 pairs run the hot loop over FULL
    // groups only; the ragged last group is warp 1 of CTA 0's (below).
    auto lay_out = [&](bool full_groups) {
        const uint64_t ngroups_all = full_groups ? npairs / 32 : (npairs + 31) / 32;
        // stripes of gpt groups dealt round-robin to the CTAs (tile k of this CTA
        // is stripe k * gridDim + blockIdx.x): every SM works on one moving front
        unsigned gpt =
            (unsigned)((ngroups_all + (uint64_t)gridDim.x * kDynTiles - 1) / ((uint64_t)gridDim.x * kDynTiles));
        const unsigned min_groups = a.tile_groups ? a.tile_groups : kDynMinGroups;
        if (gpt < min_groups) gpt = min_groups;  // claims + tile flushes amortised over >= min_groups groups
        const unsigned nstripes = (unsigned)((ngroups_all + gpt - 1) / gpt);
        if (threadIdx.x == 0) {
            next_tile = 0;
            s_ghi = (unsigned)ngroups_all;
            s_gpt = gpt;
            s_ntiles = nstripes > blockIdx.x ? (nstripes - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
        }
        __syncthreads();
    };
    // the expected mode: in-range state (kSane) with an in-range divisor, checked after the wait
    const bool full_expected = FSB_DYN_FULL && FSB_DYN_FAST && kSane && (npairs >> 32) == 0;
    lay_out(full_expected);

    pdl_wait_and_release();
    const bool split = a.ff.key_in != nullptr;  // split fold: the max from its key slot, the sums folded beside the run
    const Partial prev = split ? prev_from_key(a.ff) : combine_prev(a.part_in, a.world, a.px);
    publish_prev(prev, a.trace_out, split ? nullptr : a.bary_out, a.ec, t_start);
    const bool eat = prev.best > 0.0;  // sim.hpp:115
    const SharedDivisor M = make_divisor(eat ? prev.best : 1.0);
    const bool fast = FSB_DYN_FAST && no_guards<kSane>(eat, M);
    const bool full = FSB_DYN_FULL && fast && (npairs >> 32) == 0;
    if (full != full_expected) lay_out(full);  // an out-of-range divisor (another rank's state): the guarded loop's layout

    const unsigned lane = threadIdx.x & 31;
    __shared__ Partial ragged_part;
    if (full) {
        dyn_tiles<kExplicitCur, kSane, true, true>(a, P, eat, M, step, rev, tile_part, next_tile, s_ghi, s_gpt,
                                                   s_ntiles);
        if (blockIdx.x == 0 && threadIdx.x >= 32 && threadIdx.x < 64 && (npairs & 31)) {  // the ragged last group
            const uint64_t q = (npairs & ~31ull) + lane;
            double2* X2 = reinterpret_cast<double2*>(a.s.x);
            double2* Y2 = reinterpret_cast<double2*>(a.s.y);
            double2* W2 = reinterpret_cast<double2*>(a.s.w);
            double2* P2 = reinterpret_cast<double2*>(a.s.p);
            const double2* C2 = reinterpret_cast<const double2*>(a.s.c);
            const SoA2 src{X2, Y2, W2, P2, C2};
            double2 X[1], Y[1], W[1], Q[1], C[1];
            const bool valid[1] = {q < npairs};
            const uint64_t qs[1] = {q}, gi[1] = {a.gfirst + 2 * q};
            if (valid[0]) {
                X[0] = X2[q];
                Y[0] = Y2[q];
                W[0] = W2[q];
                Q[0] = P2[q];
                if (kExplicitCur) C[0] = C2[q];
            }
            Partial racc = identity();
            fused_pairs<kExplicitCur, 1, kSane, true, false, false, true>(X, Y, W, Q, C, valid, src, qs, gi, P, eat, M,
                                                                          step, racc);
            if (valid[0]) {
                X2[q] = X[0];
                Y2[q] = Y[0];
                W2[q] = W[0];
                P2[q] = Q[0];
            }
            racc = warp_reduce(racc);
            if (lane == 0) ragged_part = racc;
        }
    } else if (fast) {
        dyn_tiles<kExplicitCur, kSane, true>(a, P, eat, M, step, rev, tile_part, next_tile, s_ghi, s_gpt, s_ntiles);
    } else {
        dyn_tiles<kExplicitCur, kSane, false>(a, P, eat, M, step, rev, tile_part, next_tile, s_ghi, s_gpt, s_ntiles);
    }
    __syncthreads();
    const unsigned long long t_done = (a.ec.out && threadIdx.x == 0) ? gtimer() : 0ull;
    // Split fold, consumer side: the last warp of CTA 0 folds the PREVIOUS step's CTA partials into the
    // outputs here, after the run (their buffer is rewritten by the next kernel at the earliest; folding
    // before the tile loop cost the loop 7 % more instructions in register moves).
    if (a.ff.key_in && blockIdx.x == 0 && threadIdx.x >= blockDim.x - 32)
        fold_prev_outputs(a.ff.bp_in, a.ff.bp_in_count, a.ff.fold_out, a.ff.key_reset, a.bary_out);
    Partial cta = identity();
    if (threadIdx.x < 32) {
        for (unsigned i = lane; i < s_ntiles; i += 32) fold(cta, tile_part[i]);
        cta = warp_reduce(cta);
        if (full && blockIdx.x == 0 && (npairs & 31)) fold(cta, ragged_part);
        if ((n & 1ull) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd tail fish
            const uint64_t i = n - 1;
            double x = a.s.x[i], y = a.s.y[i], w = a.s.w[i], p = a.s.p[i];
            const double c = kExplicitCur ? a.s.c[i] : objective(x, y, P.half_pond);
            Partial tail = identity();
            fused_fish(x, y, w, p, c, eat, M, a.gfirst + i, step, P, tail);
            a.s.x[i] = x;
            a.s.y[i] = y;
            a.s.w[i] = w;
            a.s.p[i] = p;
            fold(cta, tail);
        }
    }
    grid_publish(cta, a.ws, a.part_out, a.px, a.world, a.ec.out, t_done, &a.ff);
}

// ---------------------------------------------------------------------------
// grid_kernel: all T steps in ONE cooperative launch for mid-size schools
// (the state stays in L2 between steps; no per-step launch).  Each step is
// step_chunk on every CTA, then a grid barrier that is also the reduction:
// the last CTA to arrive combines the CTA partials in index order, publishes
// the step's partial and trace entry, and opens the next generation; the
// others sleep on the generation word.  Co-residency of all CTAs is
// guaranteed by the cooperative launch.
template <bool kSane>
__global__ void __launch_bounds__(kStepThreads, FSB_MIN_BLOCKS) grid_kernel(const GridArgs g) {
    const StepArgs& a = g.base;
    const StepParams P = params_of(a.k);
    __shared__ Partial scratch[32];
    __shared__ Partial shared_prev;
    Partial prev = identity();  // no pending eat at the start of a run
    __shared__ unsigned long long t_done, ecl;  // eat-region clock (thread 0; kept out of the step loop's registers)
    if (threadIdx.x == 0) ecl = 0;
    eclk_bracket(g.eclk, false);
    for (uint64_t k = 0; k < g.num_steps; ++k) {
        const uint64_t step = g.first_step + k;
        const bool eat = prev.best > 0.0;
        const SharedDivisor M = make_divisor(eat ? prev.best : 1.0);
        Partial acc = identity();
        step_chunk<false, kSane>(a, P, eat, M, step, acc);
        const Partial blk = block_reduce(acc, scratch, &t_done, true);
        // Grid exchange: publish the CTA partial into slot [k&1][b], arrive on
        // the monotonic counter, wait for all G arrivals of this step, then
        // EVERY CTA folds the G partials itself in index order (the same tree
        // as grid_finish, so every CTA -- and the stream path -- gets the same
        // bits).  Two slot sets suffice: a CTA rewrites set k&1 at step k+2
        // only after every CTA has arrived at step k+1, i.e. finished reading.
        Partial* slots = a.ws.block_part + (k & 1) * gridDim.x;
        if (threadIdx.x == 0) {
            FSB_CHECK(2 * gridDim.x <= a.ws.cap);
            store_partial(&slots[blockIdx.x], blk);
            red_add_release_gpu(g.gen, 1ull);
            const unsigned long long target = (k + 1) * (unsigned long long)gridDim.x;
            while (ld_acquire_gpu(g.gen) < target) __nanosleep(20);
        }
        __syncthreads();
        Partial t = identity();
        for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) fold(t, load_cg(&slots[i]));
        const Partial tot = block_reduce(t, scratch);
        if (threadIdx.x == 0) {
            shared_prev = tot;
            ecl += clock64() - t_done;
            if (blockIdx.x == 0) {
                g.trace[k] = tot.best;
                if (g.bary) {
                    g.bary[3 * k + 0] = tot.sx;
                    g.bary[3 * k + 1] = tot.sy;
                    g.bary[3 * k + 2] = tot.sf;
                }
            }
        }
        __syncthreads();
        prev = shared_prev;
        __syncthreads();  // shared_prev / scratch reuse by the next step
    }
    // trailing eat of the last step, on the fish this CTA itself updated
    if (prev.best > 0.0 && g.num_steps) {
        const SharedDivisor M = make_divisor(prev.best);
        const uint64_t npairs = a.n >> 1;
        constexpr uint64_t kAlign = 64;  // the chunk of step_chunk
        const uint64_t nblk = (npairs + kAlign - 1) / kAlign;
        const uint64_t lo = 2 * ((nblk * blockIdx.x / gridDim.x) * kAlign);
        uint64_t hi = 2 * ((nblk * (blockIdx.x + 1) / gridDim.x) * kAlign);
        if (hi > 2 * npairs) hi = 2 * npairs;
        for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
            a.s.w[i] = eat_weight(a.s.w[i], a.s.p[i], objective(a.s.x[i], a.s.y[i], P.half_pond), M, P.w_max);
        if ((a.n & 1ull) && blockIdx.x == 0 && threadIdx.x == 0) {
            const uint64_t i = a.n - 1;
            a.s.w[i] = eat_weight(a.s.w[i], a.s.p[i], objective(a.s.x[i], a.s.y[i], P.half_pond), M, P.w_max);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && g.num_steps) store_partial(a.part_out, prev);
    if (threadIdx.x == 0 && g.eclk) atomicAdd(&g.eclk->ns, ecl);
    eclk_bracket(g.eclk, true);
}

// ---------------------------------------------------------------------------
// step_kernel_bulk: the same fused step with the state streamed HBM -> shared
// memory by the bulk-copy engine (cp.async.bulk, the 1-D TMA path) through a
// kBulkStages-deep ring of sub-tiles, completion tracked by mbarriers.  Thread
// 0 keeps the ring full; every thread computes one pair per sub-tile from
// shared memory and stores the new state straight to HBM.  Loads in flight no
// longer occupy registers, so memory latency is hidden by the ring instead of
// by warps.  Compact state only (the explicit-cur step uses step_kernel).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Wait for the phase with the given parity to complete.  The suspend-time hint
// lets a waiting thread sleep (NANOSLEEP.SYNCS) until the barrier flips instead
// of spinning on issue slots the compute warps need.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "FSB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra FSB_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}

struct BulkStage {
    double2 x[kBulkTilePairs];
    double2 y[kBulkTilePairs];
    double2 w[kBulkTilePairs];
    double2 p[kBulkTilePairs];
};

// Warps 0..7 compute (kBulkPairsPerThread pairs each per sub-tile); warp 8 is
// the producer whose elected lane keeps the ring full.
template <bool kSane>
__global__ void __launch_bounds__(kBulkThreads, FSB_BULK_MIN_BLOCKS) step_kernel_bulk(const StepArgs a) {
    extern __shared__ __align__(128) unsigned char bulk_smem[];
    BulkStage* stage = reinterpret_cast<BulkStage*>(bulk_smem);
    __shared__ __align__(8) uint64_t full[kBulkStages];
    __shared__ __align__(8) uint64_t empty[kBulkStages];

    const StepParams P = params_of(a.k);
    const unsigned long long t_start = (a.ec.phase && blockIdx.x == 0 && threadIdx.x == 0) ? gtimer() : 0ull;
    pdl_wait_and_release();
    const Partial prev = combine_prev(a.part_in, a.world, a.px);
    publish_prev(prev, a.trace_out, a.bary_out, a.ec, t_start);
    const bool eat = prev.best > 0.0;  // sim.hpp:115
    const SharedDivisor M = make_divisor(eat ? prev.best : 1.0);
    const uint64_t step = (a.step_ptr ? *a.step_ptr : 0ull) + a.step_add;
    const uint64_t n = a.n;
    const uint64_t npairs = n >> 1;
    const bool rev = a.alternate && (step & 1ull);

    constexpr uint64_t kAlign = 64;  // balanced chunk per CTA, as in step_kernel
    const uint64_t nblk = (npairs + kAlign - 1) / kAlign;
    const uint64_t lo = (nblk * blockIdx.x / gridDim.x) * kAlign;
    uint64_t hi = (nblk * (blockIdx.x + 1) / gridDim.x) * kAlign;
    if (hi > npairs) hi = npairs;
    const uint64_t nsub = hi > lo ? (hi - lo + kBulkTilePairs - 1) / kBulkTilePairs : 0;

    double2* X2 = reinterpret_cast<double2*>(a.s.x);
    double2* Y2 = reinterpret_cast<double2*>(a.s.y);
    double2* W2 = reinterpret_cast<double2*>(a.s.w);
    double2* P2 = reinterpret_cast<double2*>(a.s.p);

    const unsigned t = threadIdx.x;
    if (t == 0) {
        for (int s = 0; s < kBulkStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kBulkCompute / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto sub_base = [&](uint64_t j) { return lo + (rev ? nsub - 1 - j : j) * (uint64_t)kBulkTilePairs; };
    Partial acc = identity();
    if (t >= kBulkCompute) {
        // Producer warp, elected lane.  Sub-tile j lives in stage j % kBulkStages:
        // bulk-load it; once the compute warps have written its new state back
        // into the stage (empty[s]), bulk-store the stage to HBM and, as soon as
        // the store has read the stage out, reuse it for sub-tile j + kBulkStages.
        if (t == kBulkCompute) {
            auto load = [&](uint64_t j) {
                const int s = (int)(j % kBulkStages);
                const uint64_t base = sub_base(j);
                const uint64_t cnt = (hi - base < (uint64_t)kBulkTilePairs) ? hi - base : (uint64_t)kBulkTilePairs;
                const unsigned bytes = (unsigned)(cnt * sizeof(double2));
                FSB_CHECK(base >= lo && cnt >= 1 && cnt <= (uint64_t)kBulkTilePairs);
                mbar_expect_tx(&full[s], 4 * bytes);
                bulk_load(stage[s].x, X2 + base, bytes, &full[s]);
                bulk_load(stage[s].y, Y2 + base, bytes, &full[s]);
                bulk_load(stage[s].w, W2 + base, bytes, &full[s]);
                bulk_load(stage[s].p, P2 + base, bytes, &full[s]);
            };
            for (uint64_t j = 0; j < nsub && j < (uint64_t)kBulkStages; ++j) load(j);
            for (uint64_t j = 0; j < nsub; ++j) {
                const int s = (int)(j % kBulkStages);
                mbar_wait(&empty[s], (unsigned)((j / kBulkStages) & 1));
                const uint64_t base = sub_base(j);
                const uint64_t cnt = (hi - base < (uint64_t)kBulkTilePairs) ? hi - base : (uint64_t)kBulkTilePairs;
                const unsigned bytes = (unsigned)(cnt * sizeof(double2));
                bulk_store(X2 + base, stage[s].x, bytes);
                bulk_store(Y2 + base, stage[s].y, bytes);
                bulk_store(W2 + base, stage[s].w, bytes);
                bulk_store(P2 + base, stage[s].p, bytes);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                if (j + kBulkStages < nsub) {
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    load(j + kBulkStages);
                }
            }
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete before exit
        }
    } else {
        for (uint64_t j = 0; j < nsub; ++j) {
            const int s = (int)(j % kBulkStages);
            const uint64_t base = sub_base(j);
            mbar_wait(&full[s], (unsigned)((j / kBulkStages) & 1));
            const SoA2 src{stage[s].x, stage[s].y, stage[s].w, stage[s].p, nullptr};
            double2 X[kBulkPairsPerThread], Y[kBulkPairsPerThread], W[kBulkPairsPerThread], Q[kBulkPairsPerThread];
            bool valid[kBulkPairsPerThread];
            uint64_t ks[kBulkPairsPerThread], gi[kBulkPairsPerThread];
#pragma unroll
            for (int u = 0; u < kBulkPairsPerThread; ++u) {
                const unsigned k = t + u * kBulkCompute;
                ks[u] = k;
                gi[u] = a.gfirst + 2 * (base + k);
                valid[u] = base + k < hi;
                if (valid[u]) {
                    X[u] = stage[s].x[k];
                    Y[u] = stage[s].y[k];
                    W[u] = stage[s].w[k];
                    Q[u] = stage[s].p[k];
                }
            }
            fused_pairs<false, kBulkPairsPerThread, kSane>(X, Y, W, Q, X, valid, src, ks, gi, P, eat, M, step, acc);
#pragma unroll
            for (int u = 0; u < kBulkPairsPerThread; ++u) {
                const unsigned k = (unsigned)ks[u];
                if (valid[u]) {
                    // new state back into the stage, bulk-stored by the producer
                    stage[s].x[k] = X[u];
                    stage[s].y[k] = Y[u];
                    stage[s].w[k] = W[u];
                    stage[s].p[k] = Q[u];
                }
            }
            // make the generic-proxy smem writes visible to the bulk-store (async) proxy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if ((t & 31) == 0) mbar_arrive(&empty[s]);
        }
        if ((n & 1ull) && blockIdx.x == 0 && t == 0) {  // odd tail fish
            const uint64_t i = n - 1;
            double x = a.s.x[i], y = a.s.y[i], w = a.s.w[i], p = a.s.p[i];
            fused_fish(x, y, w, p, objective(x, y, P.half_pond), eat, M, a.gfirst + i, step, P, acc);
            a.s.x[i] = x;
            a.s.y[i] = y;
            a.s.w[i] = w;
            a.s.p[i] = p;
        }
    }
    grid_finish(acc, a.ws, a.part_out, a.px, a.world, a.ec.out);
}

// ---------------------------------------------------------------------------
// step_kernel_ws: the fused step, warp-specialised.  One 1024-thread CTA per
// SM: warp 0's elected lane is a producer that streams the CTA's state HBM ->
// shared memory with cp.async.bulk into a ring of kWsRounds round buffers
// (full/empty mbarrier each); warps 1..31 consume.  The shard's 32-pair
// groups form stripes of 31 (one per consumer warp) dealt round-robin to the
// CTAs (one moving front over the arrays, as step_kernel_dyn); in round r a
// CTA takes its r-th stripe (its last first on odd steps: L2 reuse), which is
// contiguous, so one round is four bulk copies of up to 15.5 KB (x, y, w, p)
// and consumer warp c takes group c of it.  A consumer draws its pair's RNG
// (seed, fish, step only) first, then waits for the round, copies its pair
// into registers, releases the buffer at once and computes from registers,
// storing the new state straight to HBM (STG).  The buffers are held only for
// the four LDS, so the ring is almost entirely loads in flight -- up to
// kWsRounds x 62 KB per SM, independent of the registers the step needs
// (which cap the LDG kernels at 1024 resident threads and so their bytes in
// flight).  Every warp's partial, and the fold of the 31 warp partials in
// warp order, are fixed for a fixed (n, grid, step parity).
#ifndef FSB_WS_ROUNDS
#define FSB_WS_ROUNDS 3
#endif
constexpr int kWsThreads = 1024;
constexpr unsigned kWsConsumers = kWsThreads / 32 - 1;  // = groups per stripe
constexpr unsigned kWsRounds = FSB_WS_ROUNDS;
constexpr unsigned kWsPairs = kWsConsumers * 32;        // pairs per stripe
struct WsRound {
    double2 x[kWsPairs], y[kWsPairs], w[kWsPairs], p[kWsPairs];
};
constexpr size_t kWsSmemBytes = kWsRounds * sizeof(WsRound);

// The shared-memory ring of the warp-specialised kernels.
struct WsRing {
    WsRound* buf;
    uint64_t* full;
    uint64_t* empty;
};

// Producer: round buffer b <- the stripe of pairs [q0, q0 + np) of x, y, w, p.
__device__ __forceinline__ void ws_load(const StepArgs& a, const WsRing& R, unsigned b, uint64_t q0, unsigned np) {
    const unsigned bytes = np * (unsigned)sizeof(double2);
    FSB_CHECK(np >= 1 && np <= kWsPairs);
    mbar_expect_tx(&R.full[b], 4 * bytes);
    bulk_load(R.buf[b].x, reinterpret_cast<const double2*>(a.s.x) + q0, bytes, &R.full[b]);
    bulk_load(R.buf[b].y, reinterpret_cast<const double2*>(a.s.y) + q0, bytes, &R.full[b]);
    bulk_load(R.buf[b].w, reinterpret_cast<const double2*>(a.s.w) + q0, bytes, &R.full[b]);
    bulk_load(R.buf[b].p, reinterpret_cast<const double2*>(a.s.p) + q0, bytes, &R.full[b]);
}

// One consumer thread's pair of a round: fetched (draws first, then the stage),
// then computed and stored.
struct WsPair {
    double2 X[1], Y[1], W[1], Q[1];
    PairDraws<1> dr;
    uint64_t q[1], gi[1];
    bool valid[1];
};

// Consumer warp c: pair q = (first group of the stripe + c) x 32 + lane,
// valid below `limit` pairs; round buffer b at parity ph.  Releases b.
__device__ __forceinline__ void ws_fetch(WsPair& f, const StepArgs& a, const StepParams& P, uint64_t step,
                                         const WsRing& R, unsigned b, unsigned ph, unsigned c, unsigned g,
                                         uint64_t limit) {
    const unsigned lane = threadIdx.x & 31;
    f.q[0] = (uint64_t)(g + c) * 32 + lane;
    f.valid[0] = f.q[0] < limit;
    f.gi[0] = a.gfirst + 2 * f.q[0];
    draw_pairs<1>(f.dr, f.gi, P.seed, step);
    mbar_wait(&R.full[b], ph);
    const unsigned k = c * 32 + lane;
    if (f.valid[0]) {
        f.X[0] = R.buf[b].x[k];
        f.Y[0] = R.buf[b].y[k];
        f.W[0] = R.buf[b].w[k];
        f.Q[0] = R.buf[b].p[k];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&R.empty[b]);
}

// kFast: in-range mode with an in-range divisor -- fish_sane, no guard and no
// fallback call in the loop (a call would make ptxas spill the loop's live
// registers around it).
template <bool kSane, bool kFast>
__device__ __forceinline__ void ws_compute(WsPair& f, const StepArgs& a, const StepParams& P, bool eat,
                                           const SharedDivisor& M, uint64_t step, Partial& acc) {
    double2* X2 = reinterpret_cast<double2*>(a.s.x);
    double2* Y2 = reinterpret_cast<double2*>(a.s.y);
    double2* W2 = reinterpret_cast<double2*>(a.s.w);
    double2* P2 = reinterpret_cast<double2*>(a.s.p);
    if (kFast) {
        if (f.valid[0]) {
            const double n0 = fish_sane(f.X[0].x, f.Y[0].x, f.W[0].x, f.Q[0].x, eat, M, f.dr.U0[0][0],
                                        f.dr.U1[0][0], P);
            const double n1 = fish_sane(f.X[0].y, f.Y[0].y, f.W[0].y, f.Q[0].y, eat, M, f.dr.U0[0][1],
                                        f.dr.U1[0][1], P);
            accumulate(acc, f.X[0].x, f.Y[0].x, f.Q[0].x, n0);
            accumulate(acc, f.X[0].y, f.Y[0].y, f.Q[0].y, n1);
        }
    } else {
        const SoA2 src{X2, Y2, W2, P2, nullptr};
        fused_pairs<false, 1, kSane, false, false, true>(f.X, f.Y, f.W, f.Q, f.X, f.valid, src, f.q, f.gi, P, eat, M,
                                                         step, acc, nullptr, &f.dr);
    }
    if (f.valid[0]) {
        const uint64_t q = f.q[0];
        X2[q] = f.X[0];
        Y2[q] = f.Y[0];
        W2[q] = f.W[0];
        P2[q] = f.Q[0];
    }
}


template <bool kSane, bool kFast>
__device__ __forceinline__ void ws_consume(const StepArgs& a, const StepParams& P, bool eat, const SharedDivisor& M,
                                           uint64_t step, const WsRing& R, unsigned c, unsigned g0,
                                           unsigned stride, unsigned rounds, Partial& acc) {
    const uint64_t npairs = a.n >> 1;
    const bool rev = a.alternate && (step & 1ull);
    unsigned b = 0, ph = 0, g = g0;
    for (unsigned r = 0; r < rounds; ++r) {
        WsPair f;
        ws_fetch(f, a, P, step, R, b, ph, c, g, npairs);
        ws_compute<kSane, kFast>(f, a, P, eat, M, step, acc);
        g = rev ? g - stride : g + stride;
        if (++b == kWsRounds) {
            b = 0;
            ph ^= 1u;
        }
    }
}

template <bool kSane>
__global__ void __launch_bounds__(kWsThreads, 1) step_kernel_ws(const StepArgs a) {
    extern __shared__ __align__(128) unsigned char ws_smem[];
    __shared__ __align__(8) uint64_t full[kWsRounds];
    __shared__ __align__(8) uint64_t empty[kWsRounds];
    __shared__ Partial warp_part[32];
    const WsRing R{reinterpret_cast<WsRound*>(ws_smem), full, empty};

    const StepParams P = params_of(a.k);
    const unsigned long long t_start = (a.ec.phase && blockIdx.x == 0 && threadIdx.x == 0) ? gtimer() : 0ull;
    const unsigned t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) {
        for (unsigned s = 0; s < kWsRounds; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWsConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait_and_release();
    const Partial prev = combine_prev(a.part_in, a.world, a.px);
    publish_prev(prev, a.trace_out, a.bary_out, a.ec, t_start);
    const bool eat = prev.best > 0.0;  // sim.hpp:115
    const SharedDivisor M = make_divisor(eat ? prev.best : 1.0);
    const uint64_t step = (a.step_ptr ? *a.step_ptr : 0ull) + a.step_add;
    const uint64_t n = a.n;
    const uint64_t npairs = n >> 1;
    const bool rev = a.alternate && (step & 1ull);

    // 32-bit group indices: up to 2^37 fish per shard
    const unsigned ngroups = (unsigned)((npairs + 31) / 32);
    const unsigned nstripes = (ngroups + kWsConsumers - 1) / kWsConsumers;
    const unsigned rounds = nstripes > blockIdx.x ? (nstripes - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
    // first group of round 0's stripe and the step between rounds' stripes
    const unsigned stride = gridDim.x * kWsConsumers;
    const unsigned g0 = (blockIdx.x + (rev && rounds ? (rounds - 1) * gridDim.x : 0u)) * kWsConsumers;
    __syncthreads();  // barriers initialised

    Partial acc = identity();
    if (warp == 0) {
        if (lane == 0) {
            unsigned b = 0, ph = 0, g = g0;
            for (unsigned r = 0; r < rounds; ++r) {
                if (r >= kWsRounds) mbar_wait(&empty[b], ph ^ 1u);  // round r - kWsRounds consumed
                const uint64_t q0 = (uint64_t)g * 32;                // the stripe is contiguous
                ws_load(a, R, b, q0, (npairs - q0 < kWsPairs) ? (unsigned)(npairs - q0) : kWsPairs);
                g = rev ? g - stride : g + stride;
                if (++b == kWsRounds) {
                    b = 0;
                    ph ^= 1u;
                }
            }
        }
    } else {
        const unsigned c = warp - 1;
        if (no_guards<kSane>(eat, M))
            ws_consume<kSane, true>(a, P, eat, M, step, R, c, g0, stride, rounds, acc);
        else
            ws_consume<kSane, false>(a, P, eat, M, step, R, c, g0, stride, rounds, acc);
        acc = warp_reduce(acc);
        if (lane == 0) warp_part[c] = acc;
    }
    __syncthreads();
    const unsigned long long t_done = (a.ec.out && t == 0) ? gtimer() : 0ull;
    Partial cta = identity();
    if (warp == 0) {
        if (lane < kWsConsumers) cta = warp_part[lane];
        cta = warp_reduce(cta);
        if ((n & 1ull) && blockIdx.x == 0 && t == 0) {  // odd tail fish
            const uint64_t i = n - 1;
            double x = a.s.x[i], y = a.s.y[i], w = a.s.w[i], p = a.s.p[i];
            Partial tail = identity();
            fused_fish(x, y, w, p, objective(x, y, P.half_pond), eat, M, a.gfirst + i, step, P, tail);
            a.s.x[i] = x;
            a.s.y[i] = y;
            a.s.w[i] = w;
            a.s.p[i] = p;
            fold(cta, tail);
        }
    }
    grid_publish(cta, a.ws, a.part_out, a.px, a.world, a.ec.out, t_done);
}

template <bool kExplicitCur>
__global__ void __launch_bounds__(kThreads) eat_kernel(const EatArgs a) {
    const unsigned long long t_start = (a.ec.phase && blockIdx.x == 0 && threadIdx.x == 0) ? gtimer() : 0ull;
    pdl_wait_and_release();
    const bool split = a.ff.key_in != nullptr;
    const Partial prev = split ? prev_from_key(a.ff) : combine_prev(a.part_in, a.world, a.px);
    publish_prev(prev, a.trace_out, split ? nullptr : a.bary_out, a.ec, t_start);
    if (split && blockIdx.x == 0 && threadIdx.x < 32)
        fold_prev_outputs(a.ff.bp_in, a.ff.bp_in_count, a.ff.fold_out, a.ff.key_reset, a.bary_out);
    if (!(prev.best > 0.0)) return;  // sim.hpp:115: no improvement, weights unchanged
    const SharedDivisor M = make_divisor(prev.best);
    const double half = a.k.half_pond;
    const double w_max = a.k.w_max;
    const uint64_t npairs = a.n >> 1;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const double2* X2 = reinterpret_cast<const double2*>(a.s.x);
    const double2* Y2 = reinterpret_cast<const double2*>(a.s.y);
    const double2* P2 = reinterpret_cast<const double2*>(a.s.p);
    const double2* C2 = reinterpret_cast<const double2*>(a.s.c);
    double2* W2 = reinterpret_cast<double2*>(a.s.w);
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < npairs; q += stride) {
        double2 W = W2[q];
        const double2 P = P2[q];
        double c0, c1;
        if (kExplicitCur) {
            const double2 C = C2[q];
            c0 = C.x;
            c1 = C.y;
        } else {
            const double2 X = X2[q], Y = Y2[q];
            c0 = objective(X.x, Y.x, half);
            c1 = objective(X.y, Y.y, half);
        }
        W.x = eat_weight(W.x, P.x, c0, M, w_max);
        W.y = eat_weight(W.y, P.y, c1, M, w_max);
        W2[q] = W;
    }
    if ((a.n & 1ull) && blockIdx.x == 0 && threadIdx.x == 0) {
        const uint64_t i = a.n - 1;
        const double cur = kExplicitCur ? a.s.c[i] : objective(a.s.x[i], a.s.y[i], half);
        a.s.w[i] = eat_weight(a.s.w[i], a.s.p[i], cur, M, w_max);
    }
}

template <bool kExplicitCur>
__global__ void __launch_bounds__(kThreads) reduce_kernel(const ReduceArgs a) {
    const unsigned long long t_start = a.ec.out ? gtimer() : 0ull;  // the whole pass is the max region
    const double half = a.k.half_pond;
    Partial acc = identity();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
        const double x = a.s.x[i], y = a.s.y[i];
        const double cur = kExplicitCur ? a.s.c[i] : objective(x, y, half);
        accumulate(acc, x, y, a.s.p[i], cur);
    }
    grid_finish(acc, a.ws, a.part_out, a.px, a.world, a.ec.out, t_start | 1ull);
}

struct FishAoS {
    double x, y, w, p, c;
};

// Fish [lo, lo+cnt) -- or fish idx[0..cnt) when idx is given -- in Fish layout.
__global__ void soa_to_aos_kernel(const SoA s, double half, uint64_t lo, uint64_t cnt, FishAoS* out,
                                  const uint64_t* idx) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += stride) {
        const uint64_t i = idx ? idx[k] : lo + k;
        FishAoS f;
        f.x = s.x[i];
        f.y = s.y[i];
        f.w = s.w[i];
        f.p = s.p[i];
        f.c = s.c ? s.c[i] : objective(f.x, f.y, half);
        out[k] = f;
    }
}

// {+0} U [2^-454, 2^501]: the objective values an in-range state can hold.
__device__ __forceinline__ bool objective_in_range(double v) {
    return __double_as_longlong(v) == 0 || (v >= 0x1p-454 && v <= 0x1p501);
}

// Upload: AoS -> SoA.  mismatch |= 1 if some current_objective differs from
// objective(x, y) (the state then carries an explicit c[]), |= 2 if some fish
// is outside the in-range mode's preconditions.
__global__ void aos_to_soa_kernel(const FishAoS* in, SoA s, double half, uint64_t lo, uint64_t cnt,
                                  int* mismatch) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    bool bad = false, out = false;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += stride) {
        const uint64_t i = lo + k;
        const FishAoS f = in[k];
        s.x[i] = f.x;
        s.y[i] = f.y;
        s.w[i] = f.w;
        s.p[i] = f.p;
        s.c[i] = f.c;
        // bitwise comparison: is current_objective the objective of (x, y)?
        const double o = objective(f.x, f.y, half);
        bad |= (__double_as_longlong(o) != __double_as_longlong(f.c));
        // in-range mode preconditions (fsb_math.cuh "In-range mode")
        const double pond = 2.0 * half;
        out |= !(f.x >= 0.0 && f.x <= pond && f.y >= 0.0 && f.y <= pond) || f.w > 0x1p501 ||
               !objective_in_range(f.p) || !objective_in_range(f.c);
    }
    const int flags = (__syncthreads_or(bad) ? 1 : 0) | (__syncthreads_or(out) ? 2 : 0);
    if (flags && threadIdx.x == 0) atomicOr(mismatch, flags);
}

// ---------------------------------------------------------------------------
// Small-swarm persistent kernel: one cluster of C CTAs holds the whole school
// in registers for every step.  The per-step exchange has no cluster barrier:
// each CTA pushes its partial into every CTA's slot with st.async, whose bytes
// complete a transaction count on the DESTINATION CTA's mbarrier; each CTA then
// waits on its own mbarrier until all C partials have landed.  Double-buffered
// by step parity; a CTA can reuse a slot only after every CTA has consumed it
// (it needs their next partials first), so no further synchronisation is needed.

constexpr int kMaxCluster = 16;
#ifndef FSB_CLUSTER_F
#define FSB_CLUSTER_F 1
#endif
constexpr int kClusterF = FSB_CLUSTER_F;  // fish per thread of the persistent cluster kernel

__device__ __forceinline__ uint32_t cluster_map(uint32_t local_smem, unsigned rank) {
    uint32_t r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem), "r"(rank));
    return r;
}

__device__ __forceinline__ void st_async_f64x2(uint32_t dst, double a, double b, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
                 "d"(a), "d"(b), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void st_async_f64(uint32_t dst, double a, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(dst), "d"(a),
                 "r"(bar)
                 : "memory");
}

// Wait for a phase of this CTA's mbarrier whose bytes other CTAs of the
// cluster deliver with st.async (complete_tx): the data and the barrier are
// both in this CTA's shared memory, so the default CTA-scope acquire orders
// the reads of the delivered slots.  A cluster-scope acquire would also
// invalidate L1 on every wait (CCTL.IVALL: 20% of the C4 step's stall samples,
// profiles/round2_cluster_kernel_c4_ncu_source_top.txt).
#ifndef FSB_CLUSTER_ACQ
#define FSB_CLUSTER_ACQ 0  // A/B: 1 = acquire at cluster scope
#endif
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
#if FSB_CLUSTER_ACQ
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "FSB_CWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra FSB_CWAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "FSB_CWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra FSB_CWAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}

// kBary: also reduce the barycentre sums each step (only when the caller asked
// for them -- the max alone is a 4x shorter reduction on this latency-bound path).
// kSane: in-range state (init'd or checked at upload): every division and
// square root on its unguarded fast path (fish_sane_cur) -- one rank, so the
// divisor (the school's own max) is in range too.
template <int F, bool kBary, bool kClock, bool kSane>
__global__ void __launch_bounds__(1024) cluster_kernel(const ClusterArgs a) {
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned crank = cluster.block_rank();
    const unsigned ncta = cluster.num_blocks();
    __shared__ __align__(16) Partial slots[2][kMaxCluster];
    __shared__ __align__(8) uint64_t xbar[2];
    __shared__ Partial scratch[32];
    __shared__ unsigned long long scratch_key[32];
    constexpr unsigned kBytes = kBary ? 32 : 8;  // bytes each CTA pushes per destination
    if (threadIdx.x == 0) {
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();  // every CTA's barriers exist before anyone pushes into them

    const StepParams P = params_of(a.k);
    const uint64_t T = blockDim.x;
    const uint64_t stride = (uint64_t)ncta * T;
    const uint64_t g = (uint64_t)crank * T + threadIdx.x;

    double x[F], y[F], w[F], p[F], c[F];
    uint64_t hf[F];
    bool valid[F];
#pragma unroll
    for (int f = 0; f < F; ++f) {
        const uint64_t j = g + (uint64_t)f * stride;
        valid[f] = j < a.n;
        x[f] = y[f] = w[f] = p[f] = c[f] = 0.0;
        hf[f] = 0;
        if (valid[f]) {
            x[f] = a.s.x[j];
            y[f] = a.s.y[j];
            w[f] = a.s.w[j];
            p[f] = a.s.p[j];
            c[f] = a.s.c ? a.s.c[j] : objective(x[f], y[f], P.half_pond);
            hf[f] = fold_in(P.seed, a.gfirst + j);  // step-independent RNG prefix, kept in registers
        }
    }

    double M = -INFINITY;
    Partial tot = identity();
    unsigned long long t_done = 0, ecl = 0;  // eat-region clock (thread 0, SM cycles)
    if (kClock) eclk_bracket(a.eclk, false);
    double u0[F], u1[F];  // this step's RNG draws, made during the previous barrier
#pragma unroll
    for (int f = 0; f < F; ++f) {
        if (kSane) draw_ints(hf[f], a.first_step, u0[f], u1[f]);
        else draw_units(hf[f], a.first_step, u0[f], u1[f]);
    }
    for (uint64_t k = 0; k < a.num_steps; ++k) {
        const uint64_t step = a.first_step + k;
        const unsigned b = (unsigned)(k & 1);
        if (threadIdx.x == 0)
            mbar_expect_tx(&xbar[b], ncta * kBytes);  // may race the pushes: fine
        const bool eat = M > 0.0;
        const SharedDivisor D = make_divisor(eat ? M : 1.0);
        Partial acc = identity();
#pragma unroll
        for (int f = 0; f < F; ++f) {
            if (valid[f]) {
                double cn;
                if (kSane) {
                    cn = fish_sane_cur(x[f], y[f], w[f], p[f], c[f], eat, D, u0[f], u1[f], P);
                } else {
                    if (eat) w[f] = eat_weight(w[f], p[f], c[f], D, P.w_max);
                    cn = swim_with_units(x[f], y[f], w[f], u0[f], u1[f], P);
                    p[f] = c[f];
                }
                c[f] = cn;
                if (kBary) {
                    accumulate(acc, x[f], y[f], p[f], cn);
                } else {
                    const double d = __dsub_rn(p[f], cn);
                    acc.best = (d > acc.best) ? d : acc.best;
                }
            }
        }
        Partial blk = identity();
        if (kBary) {
            blk = block_reduce(acc, scratch, kClock ? &t_done : nullptr, true);
        } else {  // the CTA max travels as its key (bits in .best), decoded after the fold
            blk.best = __longlong_as_double(static_cast<long long>(block_max_key(max_key(acc.best), scratch_key, kClock ? &t_done : nullptr, true)));
        }
        if (threadIdx.x < 32 && threadIdx.x < ncta) {  // lane r pushes this CTA's partial to CTA r
            const uint32_t dst = cluster_map(smem_u32(&slots[b][crank]), threadIdx.x);
            const uint32_t bar = cluster_map(smem_u32(&xbar[b]), threadIdx.x);
            if (kBary) {
                st_async_f64x2(dst, blk.best, blk.sx, bar);
                st_async_f64x2(dst + 16, blk.sy, blk.sf, bar);
            } else {
                st_async_f64(dst, blk.best, bar);
            }
        }
        // draw the next step's random numbers while the partials travel
#pragma unroll
        for (int f = 0; f < F; ++f) {
            if (kSane) draw_ints(hf[f], step + 1, u0[f], u1[f]);
            else draw_units(hf[f], step + 1, u0[f], u1[f]);
        }
        mbar_wait_cluster(&xbar[b], (unsigned)((k >> 1) & 1));
        if (kClock && threadIdx.x == 0) ecl += clock64() - t_done;
        tot = identity();
        if (kBary) {  // every warp folds the <= 16 CTA partials itself (fixed butterfly)
            const unsigned lane = threadIdx.x & 31;
            tot = warp_reduce(lane < ncta ? slots[k & 1][lane] : identity());
        } else {  // every warp folds the <= 16 CTA maxima itself: one LDS + two REDUX
            const unsigned lane = threadIdx.x & 31;
            tot.best = key_value(warp_max_key(
                lane < ncta ? static_cast<unsigned long long>(__double_as_longlong(slots[k & 1][lane].best))
                            : kKeyNegInf));
        }
        M = tot.best;
        if (crank == 0 && threadIdx.x == 0) {
            a.trace[k] = M;
            if (a.bary) {
                a.bary[3 * k + 0] = tot.sx;
                a.bary[3 * k + 1] = tot.sy;
                a.bary[3 * k + 2] = tot.sf;
            }
        }
    }
    // trailing eat of the last step, then write the school back
    const bool eat = M > 0.0;
#pragma unroll
    for (int f = 0; f < F; ++f) {
        if (valid[f]) {
            if (eat) w[f] = eat_weight(w[f], p[f], c[f], M, P.w_max);
            const uint64_t j = g + (uint64_t)f * stride;
            a.s.x[j] = x[f];
            a.s.y[j] = y[f];
            a.s.w[j] = w[f];
            a.s.p[j] = p[f];
        }
    }
    if (a.num_steps > 0 && crank == 0 && threadIdx.x == 0) store_partial(a.part_out, tot);
    if (kClock) {
        if (threadIdx.x == 0) atomicAdd(&a.eclk->ns, ecl);
        eclk_bracket(a.eclk, true);
    }
    cluster.sync();  // no CTA retires while a peer could still address its shared memory
}

// ---------------------------------------------------------------------------
// cgrid_kernel: the grid kernel with a two-level exchange.  Per step each CTA
// block-reduces its chunk, pushes the CTA partial into its cluster leader's
// shared memory with st.async (DSMEM, completing bytes on the leader's mbarrier),
// and each cluster's rank-0 CTA folds the C partials, publishes the cluster
// partial in a self-validating global slot (see cgrid_leader_exchange), polls
// every cluster's slot, folds the cluster partials and pushes the step total
// back into its cluster.  Every tree is fixed by (grid, cluster size), so the
// sums are deterministic.  Shared-memory slots are double-buffered by step
// parity: a CTA reuses a slot only after every cluster has published the next
// step, i.e. after every reader of the old contents has finished.
// Cluster coordinates re-read from special registers where used (volatile):
// the step loop runs at the 64-register limit, and values held across it
// would push the accumulators into local memory.
__device__ __forceinline__ unsigned sreg_cluster_rank() {
    unsigned v;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(v));
    return v;
}
__device__ __forceinline__ unsigned sreg_cluster_size() {
    unsigned v;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(v));
    return v;
}
__device__ __forceinline__ unsigned sreg_cluster_id() {
    unsigned v;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(v));
    return v;
}
__device__ __forceinline__ unsigned sreg_num_clusters() {
    unsigned v;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(v));
    return v;
}

__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ bool is_sentinel(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) == kSlotSentinel;
}

// A value equal to the sentinel pattern (a NaN no arithmetic produces) is
// published as the canonical NaN instead, so a poll can never wait on it.
__device__ __forceinline__ double slot_value(double v) {
    return is_sentinel(v) ? __longlong_as_double(0x7fffffffffffffffll) : v;
}

// The leader warp's half of a step's exchange.
__device__ __forceinline__ void cgrid_leader_exchange(const CGridArgs& g, uint64_t k, Partial (*slots)[kCGridCluster],
                                                   Partial* tslot, uint64_t* xbar, uint64_t* tbar) {
    const unsigned b = (unsigned)(k & 1);
    const unsigned par = (unsigned)((k >> 1) & 1);
    const unsigned lane = threadIdx.x;
    const unsigned C = sreg_cluster_size(), cid = sreg_cluster_id(), NC = sreg_num_clusters();
    mbar_wait_cluster(&xbar[b], par);
    const Partial cpart = warp_reduce(lane < C ? slots[b][lane] : identity());  // fixed butterfly
    // Cluster partials travel in self-validating slots: ring position k % 3,
    // one 128-B line per cluster, every word the SENTINEL until this step's
    // value lands, so a poll that sees four non-sentinel words has the data --
    // one round trip, no separate flag.  The publisher first re-arms its slot
    // of step k-2 (every leader has read it: each published step k-1, which
    // it does only after reading step k-2), then a release fence, then the
    // values; readers end with an acquire fence, which makes the re-arm
    // visible before they poll that slot again at step k+1.
    double* const ring = g.cl_slots;
    if (lane == 0) {
        FSB_CHECK(cid < NC);
        if (k >= 2) {
            volatile double* old = ring + ((k + 1) % kSlotRing * NC + cid) * kSlotWords;
            for (int w = 0; w < 4; ++w) old[w] = __longlong_as_double((long long)kSlotSentinel);
        }
        asm volatile("fence.release.gpu;" ::: "memory");  // MEMBAR only
        double* mine = ring + (k % kSlotRing * NC + cid) * kSlotWords;
        st_relaxed_f64(mine + 0, slot_value(cpart.best));
        st_relaxed_f64(mine + 1, slot_value(cpart.sx));
        st_relaxed_f64(mine + 2, slot_value(cpart.sy));
        st_relaxed_f64(mine + 3, slot_value(cpart.sf));
    }
    Partial t = identity();
    for (unsigned c = lane; c < NC; c += 32) {
        const double* src = ring + (k % kSlotRing * NC + c) * kSlotWords;
        Partial v;
        for (;;) {
            v.best = ld_relaxed_f64(src + 0);
            v.sx = ld_relaxed_f64(src + 1);
            v.sy = ld_relaxed_f64(src + 2);
            v.sf = ld_relaxed_f64(src + 3);
            if (!is_sentinel(v.best) && !is_sentinel(v.sx) && !is_sentinel(v.sy) && !is_sentinel(v.sf)) break;
        }
        fold(t, v);
    }
    __syncwarp();
    asm volatile("fence.acquire.gpu;" ::: "memory");  // L1 invalidate only, no MEMBAR
    t = warp_reduce(t);
    if (lane < C) {
        const uint32_t dst = cluster_map(smem_u32(&tslot[b]), lane);
        const uint32_t bar = cluster_map(smem_u32(&tbar[b]), lane);
        st_async_f64x2(dst, t.best, t.sx, bar);
        st_async_f64x2(dst + 16, t.sy, t.sf, bar);
    }
    if (cid == 0 && lane == 0) {
        g.trace[k] = t.best;
        if (g.bary) {
            g.bary[3 * k + 0] = t.sx;
            g.bary[3 * k + 1] = t.sy;
            g.bary[3 * k + 2] = t.sf;
        }
    }
}

template <bool kSane>
__global__ void __launch_bounds__(kStepThreads, FSB_MIN_BLOCKS) cgrid_kernel(const CGridArgs g) {
    cg::cluster_group cluster = cg::this_cluster();
    const StepArgs& a = g.base;
    const StepParams P = params_of(a.k);
    __shared__ __align__(16) Partial slots[2][kCGridCluster];
    __shared__ __align__(16) Partial tslot[2];
    __shared__ __align__(8) uint64_t xbar[2], tbar[2];
    __shared__ Partial scratch[32];
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xbar[b], 1);
            mbar_init(&tbar[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();  // every CTA's barriers exist before anyone pushes into them

    double prev_best = -INFINITY;  // no pending eat at the start of a run (only the max is kept live)
    __shared__ unsigned long long t_done, ecl;  // eat-region clock (thread 0; kept out of the step loop's registers)
    if (threadIdx.x == 0) ecl = 0;
    eclk_bracket(g.eclk, false);
    for (uint64_t k = 0; k < g.num_steps; ++k) {
        const unsigned b = (unsigned)(k & 1);
        if (threadIdx.x == 0) {  // may race the incoming pushes: fine
            if (sreg_cluster_rank() == 0) mbar_expect_tx(&xbar[b], sreg_cluster_size() * (unsigned)sizeof(Partial));
            mbar_expect_tx(&tbar[b], (unsigned)sizeof(Partial));
        }
        const uint64_t step = g.first_step + k;
        const bool eat = prev_best > 0.0;
        const SharedDivisor M = make_divisor(eat ? prev_best : 1.0);
        Partial acc = identity();
        step_chunk<false, kSane>(a, P, eat, M, step, acc);
        const Partial blk = block_reduce(acc, scratch, &t_done, true);  // every lane of warp 0 holds it
        if (threadIdx.x == 0) {  // this CTA's partial into the leader's slot
            const uint32_t dst = cluster_map(smem_u32(&slots[b][sreg_cluster_rank()]), 0);
            const uint32_t bar = cluster_map(smem_u32(&xbar[b]), 0);
            st_async_f64x2(dst, blk.best, blk.sx, bar);
            st_async_f64x2(dst + 16, blk.sy, blk.sf, bar);
        }
        if (threadIdx.x < 32 && sreg_cluster_rank() == 0) cgrid_leader_exchange(g, k, slots, tslot, xbar, tbar);
        mbar_wait_cluster(&tbar[b], (unsigned)((k >> 1) & 1));
        if (threadIdx.x == 0) ecl += clock64() - t_done;
        prev_best = tslot[b].best;
        __syncthreads();  // also a scheduling fence: keeps the step loop's registers in bounds
    }
    // trailing eat of the last step, on the fish this CTA itself updated
    if (prev_best > 0.0 && g.num_steps) {
        const SharedDivisor M = make_divisor(prev_best);
        const uint64_t npairs = a.n >> 1;
        constexpr uint64_t kAlign = 64;  // the chunk of step_chunk
        const uint64_t nblk = (npairs + kAlign - 1) / kAlign;
        const uint64_t lo = 2 * ((nblk * blockIdx.x / gridDim.x) * kAlign);
        uint64_t hi = 2 * ((nblk * (blockIdx.x + 1) / gridDim.x) * kAlign);
        if (hi > 2 * npairs) hi = 2 * npairs;
        for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
            a.s.w[i] = eat_weight(a.s.w[i], a.s.p[i], objective(a.s.x[i], a.s.y[i], P.half_pond), M, P.w_max);
        if ((a.n & 1ull) && blockIdx.x == 0 && threadIdx.x == 0) {
            const uint64_t i = a.n - 1;
            a.s.w[i] = eat_weight(a.s.w[i], a.s.p[i], objective(a.s.x[i], a.s.y[i], P.half_pond), M, P.w_max);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && g.num_steps) store_partial(a.part_out, tslot[(g.num_steps - 1) & 1]);
    if (threadIdx.x == 0 && g.eclk) atomicAdd(&g.eclk->ns, ecl);
    eclk_bracket(g.eclk, true);
    cluster.sync();  // no CTA retires while a peer could still address its shared memory
}

// ---------------------------------------------------------------------------
// sgrid_kernel: the whole school on chip.  One 1024-thread CTA per SM holds its
// contiguous range of fish pairs in shared memory (x, y, w, p as double2: 64 B
// per pair, 216 KB per SM at C0's 1e6 fish) for all T steps of one cooperative
// launch, so a step touches neither L2 nor HBM; the state is read once at the
// start and written once at the end (sim.hpp:133-147's loop, init aside).
// Per step every thread runs its pairs through the fused step, the CTA
// reduces, and the CTAs meet at a counter barrier (one arrival each, release;
// thread 0 of every CTA spins with acquire):
//  * max only (no barycentre trace asked for): the CTA max travels as its
//    order-preserving 64-bit key (REDUX) through one red.max into a per-step
//    key slot, so after the barrier every CTA reads ONE word;
//  * with the barycentre: the CTA partial goes into its slot of step parity
//    k&1, and after the barrier warp 0 of every CTA folds all G partials in
//    index order (loads issued up front) -- the same fixed tree everywhere, so
//    every CTA holds bit-identical totals.
// No clusters: a plain cooperative launch, which Nsight Compute can replay (it
// terminates the process on cooperative launches of clusters).
constexpr unsigned kSGridMaxGrid = 160;  // warp 0 folds <= 5 partials per lane
#ifndef FSB_SGRID_PAIRS
#define FSB_SGRID_PAIRS 7  // x 512 threads x 148 CTAs x 2 = 1.06e6 fish, the shared-memory capacity anyway
#endif
#ifndef FSB_SGRID_U
#define FSB_SGRID_U 1
#endif
constexpr int kSGridPairs = FSB_SGRID_PAIRS;  // pairs per thread: pair_cap <= kSGridThreads * kSGridPairs
constexpr int kSGridU = FSB_SGRID_U;          // pairs per pass (independent chains per thread)
#ifndef FSB_SGRID_PRE
#define FSB_SGRID_PRE 1
#endif
constexpr bool kSGridPre = FSB_SGRID_PRE;     // keep fold_in(seed, fish) of the thread's pairs in registers
#ifndef FSB_SGRID_PREDRAW
#define FSB_SGRID_PREDRAW 1
#endif
constexpr int kSGridPreDraw = FSB_SGRID_PREDRAW;  // pairs per thread whose next-step RNG is drawn during the barrier
static_assert(kSGridPreDraw <= kSGridPairs && (!kSGridPreDraw || FSB_SGRID_PRE), "predraw needs the kept prefix");

template <bool kSane, bool kBary>
__global__ void __launch_bounds__(kSGridThreads, 1) sgrid_kernel(const SGridArgs g) {
    extern __shared__ __align__(16) double2 sg_smem[];
    const StepArgs& a = g.base;
    const StepParams P = params_of(a.k);
    __shared__ Partial scratch[32];
    __shared__ unsigned long long scratch_key[32];
    __shared__ Partial shared_tot;
    __shared__ double tail[4];  // the odd last fish of the school (CTA 0)
    __shared__ unsigned long long t_done, ecl;  // eat-region clock (thread 0, SM cycles)
    const unsigned t = threadIdx.x;
    const uint64_t npairs = a.n >> 1;
    const uint64_t plo = npairs * blockIdx.x / gridDim.x;
    const unsigned cnt = (unsigned)(npairs * (blockIdx.x + 1) / gridDim.x - plo);
    FSB_CHECK(cnt <= g.pair_cap && g.pair_cap <= (unsigned)(kSGridThreads * kSGridPairs) &&
              gridDim.x <= kSGridMaxGrid);
    double2* sx = sg_smem;
    double2* sy = sx + g.pair_cap;
    double2* sw = sy + g.pair_cap;
    double2* sp = sw + g.pair_cap;
    const double2* X2 = reinterpret_cast<const double2*>(a.s.x) + plo;
    const double2* Y2 = reinterpret_cast<const double2*>(a.s.y) + plo;
    const double2* W2 = reinterpret_cast<const double2*>(a.s.w) + plo;
    const double2* P2 = reinterpret_cast<const double2*>(a.s.p) + plo;
    for (unsigned q = t; q < cnt; q += blockDim.x) {
        sx[q] = X2[q];
        sy[q] = Y2[q];
        sw[q] = W2[q];
        sp[q] = P2[q];
    }
    const bool has_tail = (a.n & 1ull) && blockIdx.x == 0;
    if (has_tail && t == 0) {
        const uint64_t i = a.n - 1;
        tail[0] = a.s.x[i];
        tail[1] = a.s.y[i];
        tail[2] = a.s.w[i];
        tail[3] = a.s.p[i];
    }
    // the step-independent RNG prefix fold_in(seed, fish) (rng.hpp:35) of this
    // thread's pairs, kept in registers for all steps: one fold_in of four per
    // fish-update saved (there is no shared memory left to keep it in)
    uint64_t H[kSGridPre ? kSGridPairs : 1][2];
#pragma unroll
    for (int j = 0; j < (kSGridPre ? kSGridPairs : 0); ++j) {
        const unsigned q = t + j * kSGridThreads;
        const uint64_t gi = a.gfirst + 2 * (plo + q);
        H[j][0] = q < cnt ? fold_in(P.seed, gi) : 0ull;
        H[j][1] = q < cnt ? fold_in(P.seed, gi + 1) : 0ull;
    }
    if (t == 0) ecl = 0;
    eclk_bracket(g.eclk, false);
    __syncthreads();

    const SoA2 src{sx, sy, sw, sp, nullptr};
    double prev_best = -INFINITY;  // no pending eat at the start of a run
    // the next step's draws of the thread's first pair, made while the CTA waits
    // at the step's grid barrier (in-range runs; the draws need no max)
    double pre[kSGridPreDraw ? kSGridPreDraw : 1][2][2];
    auto predraw = [&](uint64_t nstep, bool more) {
#pragma unroll
        for (int j = 0; j < kSGridPreDraw; ++j) {
            if (kSane && kSGridPre && more && t + j * kSGridThreads < cnt) {
                draw_ints(H[j][0], nstep, pre[j][0][0], pre[j][0][1]);
                draw_ints(H[j][1], nstep, pre[j][1][0], pre[j][1][1]);
            }
        }
    };
    for (uint64_t k = 0; k < g.num_steps; ++k) {
        const uint64_t step = g.first_step + k;
        const bool eat = prev_best > 0.0;
        const SharedDivisor M = make_divisor(eat ? prev_best : 1.0);
        Partial acc = identity();
#pragma unroll
        for (int j = 0; j < kSGridPairs; j += kSGridU) {  // kSGridU pairs per pass: independent fish chains
            const unsigned q0 = t + j * kSGridThreads;
            if (q0 < cnt) {
                double2 X[kSGridU], Y[kSGridU], W[kSGridU], Q[kSGridU], C[kSGridU];
                bool valid[kSGridU];
                uint64_t qs[kSGridU], gi[kSGridU];
#pragma unroll
                for (int u = 0; u < kSGridU; ++u) {
                    const unsigned q = q0 + u * kSGridThreads;
                    valid[u] = q < cnt;
                    qs[u] = valid[u] ? q : q0;
                    gi[u] = a.gfirst + 2 * (plo + q);
                    X[u] = sx[qs[u]];
                    Y[u] = sy[qs[u]];
                    W[u] = sw[qs[u]];
                    Q[u] = sp[qs[u]];
                }
                if (kSane && kSGridPre) {
                    // one rank in range: the divisor (the school's own max) is in range too, so
                    // nothing is guarded and there is no fallback call in the step loop
#pragma unroll
                    for (int u = 0; u < kSGridU; ++u) {
                        if (valid[u]) {
                            double m[2][2];
                            if (j + u < kSGridPreDraw && k > 0) {  // drawn during the last barrier
                                m[0][0] = pre[j + u][0][0];
                                m[0][1] = pre[j + u][0][1];
                                m[1][0] = pre[j + u][1][0];
                                m[1][1] = pre[j + u][1][1];
                            } else {
                                draw_ints(H[kSGridPre ? j + u : 0][0], step, m[0][0], m[0][1]);
                                draw_ints(H[kSGridPre ? j + u : 0][1], step, m[1][0], m[1][1]);
                            }
                            const double n0 = fish_sane(X[u].x, Y[u].x, W[u].x, Q[u].x, eat, M, m[0][0], m[0][1], P);
                            const double n1 = fish_sane(X[u].y, Y[u].y, W[u].y, Q[u].y, eat, M, m[1][0], m[1][1], P);
                            accumulate(acc, X[u].x, Y[u].x, Q[u].x, n0);
                            accumulate(acc, X[u].y, Y[u].y, Q[u].y, n1);
                        }
                    }
                } else {
                    fused_pairs<false, kSGridU, kSane, false, kSGridPre>(X, Y, W, Q, C, valid, src, qs, gi, P, eat, M,
                                                                         step, acc, &H[kSGridPre ? j : 0][0]);
                }
#pragma unroll
                for (int u = 0; u < kSGridU; ++u) {
                    if (valid[u]) {
                        sx[qs[u]] = X[u];
                        sy[qs[u]] = Y[u];
                        sw[qs[u]] = W[u];
                        sp[qs[u]] = Q[u];
                    }
                }
            }
        }
        if (has_tail && t == 0) {
            double x = tail[0], y = tail[1], w = tail[2], p = tail[3];
            fused_fish(x, y, w, p, objective(x, y, P.half_pond), eat, M, a.gfirst + a.n - 1, step, P, acc);
            tail[0] = x;
            tail[1] = y;
            tail[2] = w;
            tail[3] = p;
        }
        const unsigned long long target = (k + 1) * (unsigned long long)gridDim.x;
        if (kBary) {
            const Partial blk = block_reduce(acc, scratch, &t_done, true);  // every lane of warp 0 holds it
            Partial* slots = g.parts + (k & 1) * gridDim.x;  // reused at k+2: every CTA read it before arriving at k+1
            if (t == 0) {
                store_partial(&slots[blockIdx.x], blk);
                red_add_release_gpu(g.gen, 1ull);
            }
            predraw(step + 1, k + 1 < g.num_steps);
            if (t == 0) spin_until_gpu(g.gen, target);
            __syncthreads();
            if (t < 32) {
                Partial v[kSGridMaxGrid / 32];
#pragma unroll
                for (unsigned r = 0; r < kSGridMaxGrid / 32; ++r) {
                    const unsigned i = t + 32 * r;
                    v[r] = i < gridDim.x ? load_cg(&slots[i]) : identity();
                }
                Partial f = identity();
#pragma unroll
                for (unsigned r = 0; r < kSGridMaxGrid / 32; ++r) fold(f, v[r]);
                f = warp_reduce(f);
                if (t == 0) {
                    shared_tot = f;
                    ecl += clock64() - t_done;
                    if (blockIdx.x == 0) {
                        g.trace[k] = f.best;
                        g.bary[3 * k + 0] = f.sx;
                        g.bary[3 * k + 1] = f.sy;
                        g.bary[3 * k + 2] = f.sf;
                    }
                }
            }
        } else {
            // max only: the key of the CTA max, one red.max per CTA into this step's key slot
            const unsigned long long key = block_max_key(max_key(acc.best), scratch_key, &t_done, true);
            unsigned long long* slot = g.keys + k % 3;
            if (t == 0) {
                red_max_relaxed_gpu(slot, key);
                red_add_release_gpu(g.gen, 1ull);  // orders the red.max before the arrival
            }
            predraw(step + 1, k + 1 < g.num_steps);
            if (t == 0) {
                spin_until_gpu(g.gen, target);
                const double m = key_value(*reinterpret_cast<volatile unsigned long long*>(slot));
                // slot (k+2)%3 was last read at step k-1 by every CTA (all arrived at k since):
                // clear it for step k+2; this CTA's arrival at k+1 (release) publishes the clear
                if (blockIdx.x == 0) g.keys[(k + 2) % 3] = 0ull;
                shared_tot.best = m;
                ecl += clock64() - t_done;
                if (blockIdx.x == 0) g.trace[k] = m;
            }
        }
        __syncthreads();
        prev_best = shared_tot.best;
    }
    // trailing eat of the last step, then the state goes back to HBM
    const bool eat = prev_best > 0.0 && g.num_steps;
    const SharedDivisor M = make_divisor(eat ? prev_best : 1.0);
    double2* Xo = reinterpret_cast<double2*>(a.s.x) + plo;
    double2* Yo = reinterpret_cast<double2*>(a.s.y) + plo;
    double2* Wo = reinterpret_cast<double2*>(a.s.w) + plo;
    double2* Po = reinterpret_cast<double2*>(a.s.p) + plo;
    for (unsigned q = t; q < cnt; q += blockDim.x) {
        const double2 x = sx[q], y = sy[q], p = sp[q];
        double2 w = sw[q];
        if (eat) {
            w.x = eat_weight(w.x, p.x, objective(x.x, y.x, P.half_pond), M, P.w_max);
            w.y = eat_weight(w.y, p.y, objective(x.y, y.y, P.half_pond), M, P.w_max);
        }
        Xo[q] = x;
        Yo[q] = y;
        Wo[q] = w;
        Po[q] = p;
    }
    if (has_tail && t == 0) {
        const uint64_t i = a.n - 1;
        double w = tail[2];
        if (eat) w = eat_weight(w, tail[3], objective(tail[0], tail[1], P.half_pond), M, P.w_max);
        a.s.x[i] = tail[0];
        a.s.y[i] = tail[1];
        a.s.w[i] = w;
        a.s.p[i] = tail[3];
    }
    if (blockIdx.x == 0 && t == 0 && g.num_steps) {
        Partial last = shared_tot;
        if (!kBary) last.sx = last.sy = last.sf = 0.0;  // max only: sums not kept (engine marks them invalid)
        store_partial(a.part_out, last);
    }
    if (t == 0 && g.eclk) atomicAdd(&g.eclk->ns, ecl);
    eclk_bracket(g.eclk, true);
}

int g_num_sms[64] = {0};

int num_sms(int device) {
    if (device < 0 || device >= 64) return 148;
    if (!g_num_sms[device]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
        g_num_sms[device] = v > 0 ? v : 148;
    }
    return g_num_sms[device];
}

int grid_for(uint64_t work_items, int device, int per_sm) {
    const uint64_t want = (work_items + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)num_sms(device) * per_sm;
    uint64_t g = want < cap ? want : cap;
    return g < 1 ? 1 : (int)g;
}

}  // namespace

int step_dyn_blocks(int device) {
    int per_sm = 0, per_sm_x = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel_dyn<false, false>, kDynThreads, 0) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_x, step_kernel_dyn<true, false>, kDynThreads, 0) !=
            cudaSuccess) {
        cudaGetLastError();
        per_sm = per_sm_x = 1;
    }
    if (per_sm_x < per_sm) per_sm = per_sm_x;
    return num_sms(device) * (per_sm < 1 ? 1 : per_sm);
}

int step_ws_blocks(int device) {
    bool ok = true;
    for (auto k : {step_kernel_ws<false>, step_kernel_ws<true>}) {
        int per_sm = 0;
        ok = ok && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWsSmemBytes) ==
                       cudaSuccess;
        ok = ok && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kWsThreads, kWsSmemBytes) ==
                       cudaSuccess &&
             per_sm >= 1;
    }
    if (!ok) {
        cudaGetLastError();
        return 0;
    }
    return num_sms(device);  // one CTA per SM: the ring is sized for the SM's shared memory
}

int step_grid_blocks(int device, bool explicit_cur, bool bulk) {
    int per_sm = 0;
    cudaError_t e;
    if (bulk && !explicit_cur) {
        cudaFuncSetAttribute(step_kernel_bulk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBulkSmemBytes);
        cudaFuncSetAttribute(step_kernel_bulk<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBulkSmemBytes);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel_bulk<false>, kBulkThreads,
                                                          kBulkSmemBytes);
    } else {
        e = explicit_cur
                ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel<true, false>, kStepThreads, 0)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel<false, false>, kStepThreads, 0);
    }
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    return num_sms(device) * per_sm;
}

cudaError_t launch_init(const InitArgs& a, int grid, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    const int g = grid > 0 ? grid : grid_for(a.n, dev, 8);
    init_kernel<<<g, kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

// Launch with Programmatic Dependent Launch when requested: the kernel may be
// scheduled while its predecessor drains; it waits in griddepcontrol.wait
// (pdl_wait) before touching anything the predecessor wrote.
template <typename Args>
cudaError_t launch_maybe_pdl(void (*kern)(Args), int grid, int block, size_t smem, cudaStream_t st,
                             const Args& a, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

cudaError_t launch_step(const StepArgs& a, int grid, cudaStream_t st) {
    const bool pdl = a.pdl != 0;
    const bool sane = a.sane != 0;
    if (a.wspec && !a.s.c)
        return launch_maybe_pdl(sane ? step_kernel_ws<true> : step_kernel_ws<false>, grid, kWsThreads, kWsSmemBytes,
                                st, a, pdl);
    if (a.dyn && !a.bulk) {
        if (a.s.c)
            return launch_maybe_pdl(sane ? step_kernel_dyn<true, true> : step_kernel_dyn<true, false>, grid,
                                    kDynThreads, 0, st, a, pdl);
        return launch_maybe_pdl(sane ? step_kernel_dyn<false, true> : step_kernel_dyn<false, false>, grid,
                                kDynThreads, 0, st, a, pdl);
    }
    if (a.s.c)
        return launch_maybe_pdl(sane ? step_kernel<true, true> : step_kernel<true, false>, grid, kStepThreads, 0, st,
                                a, pdl);
    if (a.bulk)
        return launch_maybe_pdl(sane ? step_kernel_bulk<true> : step_kernel_bulk<false>, grid, kBulkThreads,
                                kBulkSmemBytes, st, a, pdl);
    return launch_maybe_pdl(sane ? step_kernel<false, true> : step_kernel<false, false>, grid, kStepThreads, 0, st, a,
                            pdl);
}

cudaError_t launch_eat(const EatArgs& a, int grid, cudaStream_t st) {
    const bool pdl = a.pdl != 0;
    if (a.s.c) return launch_maybe_pdl(eat_kernel<true>, grid, kThreads, 0, st, a, pdl);
    return launch_maybe_pdl(eat_kernel<false>, grid, kThreads, 0, st, a, pdl);
}

int grid_kernel_blocks(int device) {
    // co-residency of every CTA: the smaller occupancy of the two instantiations
    int per_sm = 0, per_sm_sane = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, grid_kernel<false>, kStepThreads, 0) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_sane, grid_kernel<true>, kStepThreads, 0) !=
            cudaSuccess) {
        cudaGetLastError();
        per_sm = per_sm_sane = 1;
    }
    if (per_sm_sane < per_sm) per_sm = per_sm_sane;
    return num_sms(device) * (per_sm < 1 ? 1 : per_sm);
}

cudaError_t launch_grid_run(const GridArgs& g, int grid, cudaStream_t st) {
    void* args[] = {const_cast<GridArgs*>(&g)};
    const void* kern = g.base.sane ? reinterpret_cast<const void*>(grid_kernel<true>)
                                   : reinterpret_cast<const void*>(grid_kernel<false>);
    return cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kStepThreads), args,
                                       0, st);
}


#define FSB_SGRID_KERNELS(X) X(false, false) X(false, true) X(true, false) X(true, true)

unsigned sgrid_pair_capacity(int device, int* grid) {
    int optin = 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (num_sms(device) > (int)kSGridMaxGrid) return 0;
    size_t stat = 0;
    bool ok = true;
#define FSB_SG_STAT(S, B)                                                   \
    {                                                                       \
        cudaFuncAttributes fa{};                                            \
        ok = ok && cudaFuncGetAttributes(&fa, sgrid_kernel<S, B>) == cudaSuccess; \
        if (fa.sharedSizeBytes > stat) stat = fa.sharedSizeBytes;           \
    }
    FSB_SGRID_KERNELS(FSB_SG_STAT)
#undef FSB_SG_STAT
    if (!ok || (size_t)optin <= stat + 1024) {
        cudaGetLastError();
        return 0;
    }
    const size_t dyn = ((size_t)optin - stat) / 64 * 64;
#define FSB_SG_SET(S, B)                                                                                 \
    {                                                                                                    \
        int per_sm = 0;                                                                                  \
        ok = ok && cudaFuncSetAttribute(sgrid_kernel<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                        (int)dyn) == cudaSuccess;                                        \
        ok = ok && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sgrid_kernel<S, B>,            \
                                                                 kSGridThreads, dyn) == cudaSuccess &&   \
             per_sm >= 1;                                                                                \
    }
    FSB_SGRID_KERNELS(FSB_SG_SET)
#undef FSB_SG_SET
    if (!ok) {
        cudaGetLastError();
        return 0;
    }
    if (grid) *grid = num_sms(device);
    const size_t cap = dyn / 64;
    return (unsigned)(cap < (size_t)kSGridThreads * kSGridPairs ? cap : (size_t)kSGridThreads * kSGridPairs);
}

cudaError_t launch_sgrid_run(const SGridArgs& g, int grid, cudaStream_t st) {
    void* args[] = {const_cast<SGridArgs*>(&g)};
    const bool sane = g.base.sane != 0, bary = g.bary != nullptr;
    const void* kern = sane ? (bary ? reinterpret_cast<const void*>(sgrid_kernel<true, true>)
                                    : reinterpret_cast<const void*>(sgrid_kernel<true, false>))
                            : (bary ? reinterpret_cast<const void*>(sgrid_kernel<false, true>)
                                    : reinterpret_cast<const void*>(sgrid_kernel<false, false>));
    return cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kSGridThreads), args, (size_t)g.pair_cap * 64, st);
}

namespace {
cudaLaunchConfig_t cgrid_config(int clusters, cudaStream_t st, cudaLaunchAttribute (&at)[2]) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * kCGridCluster);
    cfg.blockDim = dim3(kStepThreads);
    cfg.stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCGridCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cfg;
}
}  // namespace

int cgrid_clusters(int device) {
    (void)device;
    if (kCGridCluster > 8) {  // non-portable cluster sizes (experiment builds)
        cudaFuncSetAttribute(cgrid_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(cgrid_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    cudaLaunchAttribute at[2];
    cudaLaunchConfig_t cfg = cgrid_config(1, nullptr, at);
    int n0 = 0, n1 = 0;
    if (cudaOccupancyMaxActiveClusters(&n0, cgrid_kernel<false>, &cfg) != cudaSuccess ||
        cudaOccupancyMaxActiveClusters(&n1, cgrid_kernel<true>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n0 < n1 ? n0 : n1;
}

cudaError_t launch_cgrid_run(const CGridArgs& g, int clusters, cudaStream_t st) {
    cudaLaunchAttribute at[2];
    const cudaLaunchConfig_t cfg = cgrid_config(clusters, st, at);
    return g.base.sane ? cudaLaunchKernelEx(&cfg, cgrid_kernel<true>, g)
                       : cudaLaunchKernelEx(&cfg, cgrid_kernel<false>, g);
}

cudaError_t launch_reduce(const ReduceArgs& a, int grid, cudaStream_t st) {
    if (a.s.c) reduce_kernel<true><<<grid, kThreads, 0, st>>>(a);
    else reduce_kernel<false><<<grid, kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_soa_to_aos(const SoA& s, double half_pond, uint64_t lo, uint64_t cnt, void* aos,
                              cudaStream_t st) {
    if (cnt == 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    soa_to_aos_kernel<<<grid_for(cnt, dev, 8), kThreads, 0, st>>>(s, half_pond, lo, cnt,
                                                                  static_cast<FishAoS*>(aos), nullptr);
    return cudaGetLastError();
}

cudaError_t launch_gather(const SoA& s, double half_pond, const uint64_t* idx, uint64_t cnt, void* aos,
                          cudaStream_t st) {
    if (cnt == 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    soa_to_aos_kernel<<<grid_for(cnt, dev, 8), kThreads, 0, st>>>(s, half_pond, 0, cnt,
                                                                  static_cast<FishAoS*>(aos), idx);
    return cudaGetLastError();
}

cudaError_t launch_aos_to_soa(const void* aos, SoA s, double half_pond, uint64_t lo, uint64_t cnt,
                              int* mismatch, cudaStream_t st) {
    if (cnt == 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    aos_to_soa_kernel<<<grid_for(cnt, dev, 8), kThreads, 0, st>>>(
        static_cast<const FishAoS*>(aos), s, half_pond, lo, cnt, mismatch);
    return cudaGetLastError();
}


// Largest cluster this device can co-schedule with 1024-thread CTAs.
int cluster_capacity(int device, int* cluster_ctas, int* threads_per_cta) {
    (void)device;
    static int cached = 0;
    if (!cached) {
        for (auto k : {cluster_kernel<kClusterF, true, true, false>, cluster_kernel<kClusterF, false, true, false>,
                       cluster_kernel<kClusterF, true, false, false>, cluster_kernel<kClusterF, false, false, false>,
                       cluster_kernel<kClusterF, true, true, true>, cluster_kernel<kClusterF, false, true, true>,
                       cluster_kernel<kClusterF, true, false, true>, cluster_kernel<kClusterF, false, false, true>})
            cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cached = 8;
        for (int c : {16, 8}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(c);
            cfg.blockDim = dim3(1024);
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = c;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, cluster_kernel<kClusterF, true, true, false>, &cfg) ==
                    cudaSuccess &&
                nclusters >= 1) {
                cached = c;
                break;
            }
            cudaGetLastError();
        }
    }
    if (cluster_ctas) *cluster_ctas = cached;
    if (threads_per_cta) *threads_per_cta = 1024;
    return cached * 1024;  // one fish per thread, at most 1024 threads per CTA
}

cudaError_t launch_cluster_run(const ClusterArgs& a, cudaStream_t st, int* ctas) {
    int dev = 0;
    cudaGetDevice(&dev);
    int cmax = 8;
    const int capacity = cluster_capacity(dev, &cmax, nullptr);
    if (a.n == 0 || a.n > (uint64_t)capacity) return cudaErrorNotSupported;
    // One fish per thread (latency-bound: the chain per fish is the step's
    // critical path), spread over as many CTAs (SMs) of the cluster as give
    // each at least FSB_CLUSTER_MIN_FISH fish.
    uint64_t ncta = (a.n + FSB_CLUSTER_MIN_FISH - 1) / FSB_CLUSTER_MIN_FISH;
    if (ncta > (uint64_t)cmax) ncta = cmax;
    if (ncta < 1) ncta = 1;
    const uint64_t per_cta = (a.n + ncta - 1) / ncta;
    if (per_cta > 1024) return cudaErrorNotSupported;
    const uint64_t threads = ((per_cta + kClusterF * 32 - 1) / (kClusterF * 32)) * 32;  // kClusterF fish per thread

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ncta);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)ncta;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (ctas) *ctas = (int)ncta;
#define FSB_CL_LAUNCH(S)                                                                   \
    if (a.eclk) {                                                                          \
        if (a.bary) return cudaLaunchKernelEx(&cfg, cluster_kernel<kClusterF, true, true, S>, a); \
        return cudaLaunchKernelEx(&cfg, cluster_kernel<kClusterF, false, true, S>, a);     \
    }                                                                                      \
    if (a.bary) return cudaLaunchKernelEx(&cfg, cluster_kernel<kClusterF, true, false, S>, a); \
    return cudaLaunchKernelEx(&cfg, cluster_kernel<kClusterF, false, false, S>, a);
    if (a.sane) {
        FSB_CL_LAUNCH(true)
    }
    FSB_CL_LAUNCH(false)
#undef FSB_CL_LAUNCH
}

}  // namespace fsb_dev

namespace fsb_dev {

namespace {

// Operand generator for the division self-test: raw 64-bit patterns (every
// exponent, NaN, inf, subnormals, zeros) mixed with the simulation's own
// value ranges (objective differences over a max in (0, ~sqrt(2)*pond]).
__device__ __forceinline__ void selftest_operands(uint64_t i, uint64_t seed, double& a, double& b) {
    const uint64_t r0 = mix64(seed ^ (2 * i + 1));
    const uint64_t r1 = mix64(r0 + 0x9E3779B97F4A7C15ull);
    const double u0 = unit_from_bits(r0), u1 = unit_from_bits(r1);
    switch (i & 3) {
        case 0:
            a = __longlong_as_double((long long)r0);
            b = __longlong_as_double((long long)r1);
            break;
        case 1:
            a = (u0 - 0.5) * 0.4;
            b = 1e-3 + u1 * 0.3;
            break;
        case 2:
            a = (u0 - 0.5) * 300.0;
            b = __longlong_as_double((long long)(r1 & 0x7fffffffffffffffull));
            break;
        default:
            a = __longlong_as_double((long long)((r0 & 0x800fffffffffffffull) |
                                                 ((uint64_t)(r1 % 2047) << 52)));
            b = __longlong_as_double((long long)((r1 & 0x000fffffffffffffull) |
                                                 ((uint64_t)((r0 >> 7) % 2047) << 52)));
            break;
    }
}

// Self-test of the guarded fast paths against the intrinsics.  out[0]: shared
// divisor division, out[1]: per-operand division, out[2]: square root --
// bitwise mismatches of (fast path, or intrinsic when the guard fails) vs the
// intrinsic; out[3]: guard failures on simulation-range operands.
__global__ void selftest_fast_math_kernel(uint64_t n, uint64_t seed, unsigned long long* out) {
    unsigned long long bad[4] = {0, 0, 0, 0};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double a, b;
        selftest_operands(i, seed, a, b);
        const bool sim_range = (i & 3) == 1;
        // division, divisor hoisted
        double want = __ddiv_rn(a, b);
        double q = div_shared(a, make_divisor(b));
        if (!((q != q) && (want != want)) && __double_as_longlong(q) != __double_as_longlong(want)) ++bad[0];
        // division, guarded per operand
        bool ok = true;
        q = div_guarded(a, b, ok);
        if (!ok) q = __ddiv_rn(a, b);
        if (sim_range && !ok) ++bad[3];
        if (!((q != q) && (want != want)) && __double_as_longlong(q) != __double_as_longlong(want)) ++bad[1];
        // square root (of |a| scaled into the objective's range for sim cases)
        const double v = sim_range ? fabs(a) * 1e5 : a;
        want = __dsqrt_rn(v);
        ok = true;
        q = sqrt_guarded(v, ok);
        if (!ok) q = __dsqrt_rn(v);
        if (sim_range && !ok && v != 0.0) ++bad[3];
        if (!((q != q) && (want != want)) && __double_as_longlong(q) != __double_as_longlong(want)) ++bad[2];
    }
    for (int k = 0; k < 4; ++k)
        if (bad[k]) atomicAdd(&out[k], bad[k]);
}

}  // namespace

cudaError_t launch_selftest_fast_math(uint64_t n, uint64_t seed, unsigned long long* out, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    selftest_fast_math_kernel<<<grid_for(n, dev, 8), kThreads, 0, st>>>(n, seed, out);
    return cudaGetLastError();
}

}  // namespace fsb_dev
