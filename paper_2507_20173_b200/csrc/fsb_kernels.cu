// fsb_kernels.cu -- sm_100a kernels of the B200 FSB engine.
//
//   init_kernel     init_school (sim.hpp:65-79) on device, SoA stores.
//   step_kernel     ONE pass per simulation step: the previous step's eat
//                   (sim.hpp:115-120, deferred: "lazy eat"), this step's swim +
//                   objective (sim.hpp:90-98), and this step's partial
//                   max(prev-cur) (sim.hpp:112-114) plus the f-weighted
//                   barycentre sums, reduced warp -> CTA -> grid (last CTA).
//   eat_kernel      the trailing / standalone weight update (sim.hpp:115-121).
//   reduce_kernel   max + sums of the current state without moving it (eat()
//                   after an upload).
//   cluster_kernel  small swarms: all T steps in one launch of one thread-block
//                   cluster, state in registers, per-step reduction over DSMEM.
//   soa<->aos       Fish byte layout (sim.hpp:26-32) for upload / download.
//
// Determinism: max is exact (any order).  The sums use a fixed tree for a
// fixed (n, grid, step parity), so repeated runs are bit-identical.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>

#include "fsb_kernels.cuh"
#include "fsb_math.cuh"

namespace cg = cooperative_groups;

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

// Block-wide reduction; the result is valid in warp 0 (all lanes).
// `scratch` holds blockDim/32 partials.  Ends with the caller's warp 0 owning
// the value; callers __syncthreads() before reusing scratch.
__device__ __forceinline__ Partial block_reduce(Partial v, Partial* scratch) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    v = warp_reduce(v);
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    Partial r = identity();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        if (lane < nw) r = scratch[lane];
        r = warp_reduce(r);
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

// CTA partial -> global; the last CTA to arrive combines all CTA partials in
// index order and publishes this rank's partial.
__device__ __forceinline__ void grid_finish(const Partial& local, const ReduceWs& ws, Partial* part_out) {
    __shared__ Partial scratch[kThreads / 32];
    __shared__ bool am_last;
    const Partial blk = block_reduce(local, scratch);
    if (threadIdx.x == 0) {
        store_partial(&ws.block_part[blockIdx.x], blk);
        __threadfence();
        const unsigned prev = atomicAdd(ws.counter, 1u);
        am_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    Partial acc = identity();
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) fold(acc, load_cg(&ws.block_part[i]));
    __syncthreads();  // scratch reuse
    const Partial tot = block_reduce(acc, scratch);
    if (threadIdx.x == 0) {
        store_partial(part_out, tot);
        *ws.counter = 0u;  // ready for the next launch
    }
}

// Combine the ranks' partials of the previous step in rank order.
__device__ __forceinline__ Partial combine_ranks(const Partial* part_in, int world) {
    Partial r = identity();
    if (part_in) {
        for (int k = 0; k < world; ++k) fold(r, part_in[k]);
    }
    return r;
}

__device__ __forceinline__ void publish_prev(const Partial& prev, double* trace_out, double* bary_out) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (trace_out) *trace_out = prev.best;
        if (bary_out) {
            bary_out[0] = prev.sx;
            bary_out[1] = prev.sy;
            bary_out[2] = prev.sf;
        }
    }
}

__device__ __forceinline__ StepParams params_of(const Scalars& k) {
    StepParams P;
    P.pond = k.pond;
    P.half_pond = k.half_pond;
    P.step_base = k.step_base;
    P.w_max = k.w_max;
    P.seed = k.seed;
    return P;
}

// One fish of the fused step.  cur is this fish's current objective before
// the step (recomputed or explicit).  Returns nothing; updates state + acc.
__device__ __forceinline__ void fused_fish(double& x, double& y, double& w, double& p, double cur,
                                           bool eat, double M, uint64_t gi, uint64_t step,
                                           const StepParams& P, Partial& acc) {
    if (eat) w = eat_weight(w, p, cur, M, P.w_max);          // sim.hpp:115-120 (step-1)
    const double cn = swim(x, y, w, fold_in(P.seed, gi), step, P);  // sim.hpp:90-97
    p = cur;                                                   // sim.hpp:96
    accumulate(acc, x, y, cur, cn);                            // sim.hpp:112-114
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

template <bool kExplicitCur>
__global__ void __launch_bounds__(kThreads) step_kernel(const StepArgs a) {
    const StepParams P = params_of(a.k);
    const Partial prev = combine_ranks(a.part_in, a.world);
    publish_prev(prev, a.trace_out, a.bary_out);
    const double M = prev.best;
    const bool eat = M > 0.0;  // sim.hpp:115
    const uint64_t step = (a.step_ptr ? *a.step_ptr : 0ull) + a.step_add;

    const uint64_t n = a.n;
    const uint64_t npairs = n >> 1;
    const uint64_t ntiles = (npairs + kTilePairs - 1) / kTilePairs;
    const bool rev = a.alternate && (step & 1ull);

    double2* X2 = reinterpret_cast<double2*>(a.s.x);
    double2* Y2 = reinterpret_cast<double2*>(a.s.y);
    double2* W2 = reinterpret_cast<double2*>(a.s.w);
    double2* P2 = reinterpret_cast<double2*>(a.s.p);
    const double2* C2 = reinterpret_cast<const double2*>(a.s.c);

    Partial acc = identity();
    for (uint64_t it = blockIdx.x; it < ntiles; it += gridDim.x) {
        const uint64_t tile = rev ? ntiles - 1 - it : it;
        const uint64_t base = tile * kTilePairs + threadIdx.x;
        double2 X[kPairsPerThread], Y[kPairsPerThread], W[kPairsPerThread], Q[kPairsPerThread],
            C[kPairsPerThread];
#pragma unroll
        for (int u = 0; u < kPairsPerThread; ++u) {
            const uint64_t q = base + (uint64_t)u * kThreads;
            if (q < npairs) {
                X[u] = X2[q];
                Y[u] = Y2[q];
                W[u] = W2[q];
                Q[u] = P2[q];
                if (kExplicitCur) C[u] = C2[q];
            }
        }
#pragma unroll
        for (int u = 0; u < kPairsPerThread; ++u) {
            const uint64_t q = base + (uint64_t)u * kThreads;
            if (q < npairs) {
                const uint64_t gi = a.gfirst + 2 * q;
                const double c0 = kExplicitCur ? C[u].x : objective(X[u].x, Y[u].x, P.half_pond);
                const double c1 = kExplicitCur ? C[u].y : objective(X[u].y, Y[u].y, P.half_pond);
                fused_fish(X[u].x, Y[u].x, W[u].x, Q[u].x, c0, eat, M, gi, step, P, acc);
                fused_fish(X[u].y, Y[u].y, W[u].y, Q[u].y, c1, eat, M, gi + 1, step, P, acc);
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
    grid_finish(acc, a.ws, a.part_out);
}

template <bool kExplicitCur>
__global__ void __launch_bounds__(kThreads) eat_kernel(const EatArgs a) {
    const Partial prev = combine_ranks(a.part_in, a.world);
    publish_prev(prev, a.trace_out, a.bary_out);
    const double M = prev.best;
    if (!(M > 0.0)) return;  // sim.hpp:115: no improvement, weights unchanged
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
    const double half = a.k.half_pond;
    Partial acc = identity();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
        const double x = a.s.x[i], y = a.s.y[i];
        const double cur = kExplicitCur ? a.s.c[i] : objective(x, y, half);
        accumulate(acc, x, y, a.s.p[i], cur);
    }
    grid_finish(acc, a.ws, a.part_out);
}

struct FishAoS {
    double x, y, w, p, c;
};

__global__ void soa_to_aos_kernel(const SoA s, double half, uint64_t lo, uint64_t cnt, FishAoS* out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += stride) {
        const uint64_t i = lo + k;
        FishAoS f;
        f.x = s.x[i];
        f.y = s.y[i];
        f.w = s.w[i];
        f.p = s.p[i];
        f.c = s.c ? s.c[i] : objective(f.x, f.y, half);
        out[k] = f;
    }
}

__global__ void aos_to_soa_kernel(const FishAoS* in, SoA s, double half, uint64_t lo, uint64_t cnt,
                                  int* mismatch) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    bool bad = false;
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
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(mismatch, 1);
}

// ---------------------------------------------------------------------------
// Small-swarm persistent kernel: one cluster of C CTAs holds the whole school
// in registers for every step; the per-step global max + sums go through
// distributed shared memory and one cluster barrier per step.

constexpr int kMaxCluster = 16;

template <int F>
__global__ void __launch_bounds__(1024) cluster_kernel(const ClusterArgs a) {
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned crank = cluster.block_rank();
    const unsigned ncta = cluster.num_blocks();
    __shared__ Partial slots[2][kMaxCluster];
    __shared__ Partial scratch[32];

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
    for (uint64_t k = 0; k < a.num_steps; ++k) {
        const uint64_t step = a.first_step + k;
        const bool eat = M > 0.0;
        Partial acc = identity();
#pragma unroll
        for (int f = 0; f < F; ++f) {
            if (valid[f]) {
                if (eat) w[f] = eat_weight(w[f], p[f], c[f], M, P.w_max);
                const double cn = swim(x[f], y[f], w[f], hf[f], step, P);
                p[f] = c[f];
                c[f] = cn;
                accumulate(acc, x[f], y[f], p[f], cn);
            }
        }
        const Partial blk = block_reduce(acc, scratch);
        if (threadIdx.x < 32 && threadIdx.x < ncta) {
            Partial* dst = cluster.map_shared_rank(&slots[k & 1][crank], threadIdx.x);
            *dst = blk;
        }
        cluster.sync();
        tot = identity();
        for (unsigned r = 0; r < ncta; ++r) fold(tot, slots[k & 1][r]);
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

int step_grid_blocks(int device, bool explicit_cur) {
    int per_sm = 0;
    cudaError_t e = explicit_cur
        ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel<true>, kThreads, 0)
        : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel<false>, kThreads, 0);
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

cudaError_t launch_step(const StepArgs& a, int grid, cudaStream_t st) {
    if (a.s.c) step_kernel<true><<<grid, kThreads, 0, st>>>(a);
    else step_kernel<false><<<grid, kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_eat(const EatArgs& a, int grid, cudaStream_t st) {
    if (a.s.c) eat_kernel<true><<<grid, kThreads, 0, st>>>(a);
    else eat_kernel<false><<<grid, kThreads, 0, st>>>(a);
    return cudaGetLastError();
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
                                                                  static_cast<FishAoS*>(aos));
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

cudaError_t launch_copy_cur(SoA, double, uint64_t, cudaStream_t) { return cudaSuccess; }

// Largest cluster this device can co-schedule with 1024-thread CTAs.
int cluster_capacity(int device, int* cluster_ctas, int* threads_per_cta) {
    (void)device;
    static int cached = 0;
    if (!cached) {
        cudaFuncSetAttribute(cluster_kernel<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(cluster_kernel<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
            if (cudaOccupancyMaxActiveClusters(&nclusters, cluster_kernel<2>, &cfg) == cudaSuccess &&
                nclusters >= 1) {
                cached = c;
                break;
            }
            cudaGetLastError();
        }
    }
    if (cluster_ctas) *cluster_ctas = cached;
    if (threads_per_cta) *threads_per_cta = 256;
    return cached * 2048;  // 2048 fish per CTA at most (1024 threads x 2 fish)
}

cudaError_t launch_cluster_run(const ClusterArgs& a, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    int cmax = 8;
    const int capacity = cluster_capacity(dev, &cmax, nullptr);
    if (a.n == 0 || a.n > (uint64_t)capacity) return cudaErrorNotSupported;
    // ~256 fish per CTA, at most cmax CTAs; F fish per thread with F*threads
    // <= 1024 threads; F = 2 still fits the 64-register budget without spills.
    uint64_t ncta = (a.n + 255) / 256;
    if (ncta > (uint64_t)cmax) ncta = cmax;
    if (ncta < 1) ncta = 1;
    const uint64_t per_cta = (a.n + ncta - 1) / ncta;
    const uint64_t fpt = per_cta <= 1024 ? 1 : 2;
    if (per_cta > 2048) return cudaErrorNotSupported;
    const uint64_t threads = (((per_cta + fpt - 1) / fpt + 31) / 32) * 32;

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
    if (fpt == 1) return cudaLaunchKernelEx(&cfg, cluster_kernel<1>, a);
    return cudaLaunchKernelEx(&cfg, cluster_kernel<2>, a);
}

}  // namespace fsb_dev
