// barrier_probe.cu -- cost of one grid-wide exchange of a 64-bit max key among
// all CTAs of a cooperative launch (one CTA per SM), by protocol.  Evidence for
// the shared-memory grid kernel's exchange.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/barrier_probe tools/barrier_probe.cu
//   build/barrier_probe            (prints one JSON line per protocol)
//
// Every protocol leaves every CTA with the exact max of the G keys of the
// round; the probe checks that and reports ns per round (CUDA events over
// `rounds` rounds in one launch).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cg = cooperative_groups;

__device__ __forceinline__ void red_max_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_release(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_max_acqrel(unsigned long long* p, unsigned long long v) {
    unsigned long long o;
    asm volatile("atom.acq_rel.gpu.global.max.u64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(v) : "memory");
    return o;
}

struct Ws {
    unsigned long long* gen;   // [1]
    unsigned long long* keys;  // [3] or [3][G] (protocol dependent), zeroed
    unsigned long long* out;   // [G] last max seen by each CTA (check)
    unsigned long long* bad;   // [1]
};

// key of CTA b in round k: distinct, the max is the key of CTA (k % G)
__device__ __forceinline__ unsigned long long key_of(unsigned b, unsigned long long k, unsigned G) {
    return (k << 16) + ((b + G - (unsigned)(k % G)) % G == 0 ? 0xFFFF : b);
}

template <int P>
__global__ void __launch_bounds__(512, 1) probe(Ws w, unsigned long long rounds) {
    const unsigned G = gridDim.x, b = blockIdx.x, t = threadIdx.x;
    __shared__ unsigned long long got;
    for (unsigned long long k = 0; k < rounds; ++k) {
        const unsigned long long key = key_of(b, k, G);
        const unsigned long long want = (k << 16) + 0xFFFF;
        const unsigned long long target = (k + 1) * G;
        if (P == 0) {  // red.max + red.add.release, relaxed spin, one acquire fence, key reload
            if (t == 0) {
                unsigned long long* slot = w.keys + k % 3;
                red_max_relaxed(slot, key);
                red_add_release(w.gen, 1);
                while (ld_relaxed(w.gen) < target) {
                }
                asm volatile("fence.acquire.gpu;" ::: "memory");
                got = *reinterpret_cast<volatile unsigned long long*>(slot);
                if (b == 0) w.keys[(k + 2) % 3] = 0;
            }
        } else if (P == 1) {  // the same with an acquire load per poll
            if (t == 0) {
                unsigned long long* slot = w.keys + k % 3;
                red_max_relaxed(slot, key);
                red_add_release(w.gen, 1);
                while (ld_acquire(w.gen) < target) {
                }
                got = *reinterpret_cast<volatile unsigned long long*>(slot);
                if (b == 0) w.keys[(k + 2) % 3] = 0;
            }
        } else if (P == 2) {  // counter only (no key): the barrier's own cost
            if (t == 0) {
                red_add_release(w.gen, 1);
                while (ld_relaxed(w.gen) < target) {
                }
                asm volatile("fence.acquire.gpu;" ::: "memory");
                got = want;
            }
        } else if (P == 3) {  // keys in per-CTA slots [2][G] + counter; warp 0 max-reduces G slots after
            unsigned long long* slots = w.keys + (k & 1) * G;
            if (t == 0) {
                st_relaxed(&slots[b], key);
                red_add_release(w.gen, 1);
                while (ld_relaxed(w.gen) < target) {
                }
                asm volatile("fence.acquire.gpu;" ::: "memory");
            }
            __syncthreads();
            if (t < 32) {
                unsigned long long m = 0;
                for (unsigned i = t; i < G; i += 32) {
                    const unsigned long long v = ld_relaxed(&slots[i]);
                    m = v > m ? v : m;
                }
                const unsigned hi = __reduce_max_sync(~0u, (unsigned)(m >> 32));
                const unsigned lo = __reduce_max_sync(~0u, (unsigned)(m >> 32) == hi ? (unsigned)m : 0u);
                if (t == 0) got = ((unsigned long long)hi << 32) | lo;
            }
        } else if (P == 4) {  // round-tagged per-CTA key slots [2][G] (no counter, no fence): a slot is
                              // ready when its tag is this round's; parity double-buffered
            unsigned long long* slots = w.keys + (k & 1) * G;
            const unsigned long long tagged = ((k + 1) << 40) | (key & 0xFFFFFFFFFFull);
            if (t == 0) st_relaxed(&slots[b], tagged);
            if (t < 32) {
                unsigned long long m = 0;
                for (unsigned i = t; i < G; i += 32) {
                    unsigned long long v;
                    while (((v = ld_relaxed(&slots[i])) >> 40) != k + 1) {
                    }
                    v &= 0xFFFFFFFFFFull;
                    m = v > m ? v : m;
                }
                const unsigned hi = __reduce_max_sync(~0u, (unsigned)(m >> 32));
                const unsigned lo = __reduce_max_sync(~0u, (unsigned)(m >> 32) == hi ? (unsigned)m : 0u);
                if (t == 0) got = ((unsigned long long)hi << 32) | lo;
            }
        } else if (P == 5) {  // cooperative groups grid.sync() + key in per-CTA slots
            unsigned long long* slots = w.keys + (k & 1) * G;
            if (t == 0) slots[b] = key;
            cg::this_grid().sync();
            if (t < 32) {
                unsigned long long m = 0;
                for (unsigned i = t; i < G; i += 32) {
                    const unsigned long long v = ld_relaxed(&slots[i]);
                    m = v > m ? v : m;
                }
                const unsigned hi = __reduce_max_sync(~0u, (unsigned)(m >> 32));
                const unsigned lo = __reduce_max_sync(~0u, (unsigned)(m >> 32) == hi ? (unsigned)m : 0u);
                if (t == 0) got = ((unsigned long long)hi << 32) | lo;
            }
        } else if (P == 6 || P == 7) {  // NGRP counters and key slots (one 128-B line each): CTA b arrives
                                        // on group b % NGRP; lanes 0..NGRP-1 of warp 0 poll one group each
            constexpr unsigned NGRP = P == 6 ? 8 : 16;
            constexpr unsigned LINE = 16;  // u64 words per 128-B line
            const unsigned grp = b % NGRP;
            if (t == 0) {
                red_max_relaxed(w.keys + ((k % 3) * NGRP + grp) * LINE, key);
                red_add_release(w.gen + grp * LINE, 1);
            }
            if (t < 32) {
                unsigned long long m = 0;
                if (t < NGRP) {
                    const unsigned long long members = G / NGRP + (t < G % NGRP ? 1 : 0);
                    while (ld_relaxed(w.gen + t * LINE) < (k + 1) * members) {
                    }
                    asm volatile("fence.acquire.gpu;" ::: "memory");
                    m = ld_relaxed(w.keys + ((k % 3) * NGRP + t) * LINE);
                    if (b == 0) *(w.keys + (((k + 2) % 3) * NGRP + t) * LINE) = 0;
                }
                const unsigned hi = __reduce_max_sync(~0u, (unsigned)(m >> 32));
                const unsigned lo = __reduce_max_sync(~0u, (unsigned)(m >> 32) == hi ? (unsigned)m : 0u);
                if (t == 0) got = ((unsigned long long)hi << 32) | lo;
            }
        }
        __syncthreads();
        if (t == 0) {
            const unsigned long long g = got;
            const unsigned long long w4 = (P == 4) ? (want & 0xFFFFFFFFFFull) : want;
            if (g != w4) atomicAdd(w.bad, 1ull);
        }
        __syncthreads();
    }
}

int main(int argc, char** argv) {
    const unsigned long long rounds = argc > 1 ? strtoull(argv[1], nullptr, 10) : 20000;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    Ws w{};
    cudaMalloc(&w.gen, 8 * 16 * 16);
    cudaMalloc(&w.keys, 8 * 3 * 16 * 16 * 4);
    cudaMalloc(&w.out, 8 * 1024);
    cudaMalloc(&w.bad, 8);
    const char* names[] = {"redmax+count, relaxed spin + fence", "redmax+count, acquire spin",
                           "count only (barrier cost)", "per-CTA key slots + count, warp max",
                           "round-tagged key slots, no counter/fence", "cg grid.sync + key slots",
                           "8 group counters + key slots", "16 group counters + key slots"};
    void (*kerns[])(Ws, unsigned long long) = {probe<0>, probe<1>, probe<2>, probe<3>,
                                               probe<4>, probe<5>, probe<6>, probe<7>};
    for (int p = 0; p < 8; ++p) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(w.gen, 0, 8 * 16 * 16);
            cudaMemset(w.keys, 0, 8 * 3 * 16 * 16 * 4);
            cudaMemset(w.bad, 0, 8);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            void* args[] = {&w, (void*)&rounds};
            cudaEventRecord(e0);
            cudaError_t ce = cudaLaunchCooperativeKernel((void*)kerns[p], dim3(sms), dim3(512), args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long bad = 0;
            cudaMemcpy(&bad, w.bad, 8, cudaMemcpyDeviceToHost);
            if (rep == 1)
                printf("{\"protocol\": %d, \"name\": \"%s\", \"ctas\": %d, \"rounds\": %llu, \"ns_per_round\": %.1f, "
                       "\"wrong\": %llu, \"err\": \"%s\"}\n",
                       p, names[p], sms, rounds, ms * 1e6 / rounds, bad, cudaGetErrorString(ce));
        }
    }
    return 0;
}
