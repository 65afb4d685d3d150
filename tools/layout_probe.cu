// Memory-access probe (experiment, not product): the step kernel's memory
// traffic alone -- read and write 32 B per fish -- under different layouts and
// access patterns, to find what bounds the in-place step (C1, 1e7 fish).
//   soa        in place, four SoA double2 arrays (the engine), warps walk 32-pair groups of the CTA chunk
//   aosoa      in place, blocks of 32 pairs (x[32] y[32] w[32] p[32], 2 KB)
//   soa_cs     soa with streaming (.cs) loads and stores
//   soa_u2     soa, two groups per warp iteration (more bytes in flight)
//   soa_pp     ping-pong: read buffer A, write buffer B (copy-like)
//   aosoa_pp   ping-pong AoSoA
//   copy       plain grid-stride copy of the same bytes (calibration)
//   soa_gs     soa, grid-stride over groups (one moving front; 148 x 1024 and, soa_gs4, 592 x 256)
//   soa_many   soa, one short 256-thread CTA per 256 pairs (torch-style grid, 2048 threads per SM)
//   soa_many_occ4 / _occ2 / soa_many512_occ2   the same capped at 4 / 2 CTAs per SM by dynamic shared memory
// Prints device time per pass and GB/s moved (128 B per fish pair: 64 B read + 64 B written).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/layout_probe tools/layout_probe.cu
//   ./build/layout_probe [fish]            (results: profiles/r04_memory_bound_probe.jsonl)
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CHUNK()                                                                  \
    const uint64_t ng = (npairs + 31) / 32;                                      \
    const uint64_t g0 = ng * blockIdx.x / gridDim.x, g1 = ng * (blockIdx.x + 1) / gridDim.x; \
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;

__device__ __forceinline__ void touch(double2& a, double2& b, double2& c, double2& d) {
    a.x += 1.0; b.y += 1.0; c.x += 1.0; d.y += 1.0;
}

__global__ void __launch_bounds__(1024, 1) k_soa(double2* x, double2* y, double2* w, double2* p, uint64_t npairs) {
    CHUNK();
    for (uint64_t g = g0 + wid; g < g1; g += nw) {
        const uint64_t q = g * 32 + lane;
        if (q < npairs) {
            double2 a = x[q], b = y[q], c = w[q], d = p[q];
            touch(a, b, c, d);
            x[q] = a; y[q] = b; w[q] = c; p[q] = d;
        }
    }
}

// grid-stride over 32-pair groups: every warp of the GPU on one moving front
__global__ void __launch_bounds__(1024, 1) k_soa_gs(double2* x, double2* y, double2* w, double2* p, uint64_t npairs) {
    const uint64_t ng = (npairs + 31) / 32;
    const unsigned lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const uint64_t gw = (uint64_t)gridDim.x * nw;
    for (uint64_t g = (uint64_t)blockIdx.x * nw + (threadIdx.x >> 5); g < ng; g += gw) {
        const uint64_t q = g * 32 + lane;
        if (q < npairs) {
            double2 a = x[q], b = y[q], c = w[q], d = p[q];
            touch(a, b, c, d);
            x[q] = a; y[q] = b; w[q] = c; p[q] = d;
        }
    }
}

// many short CTAs (torch-style): one 256-thread CTA per 256 pairs
__global__ void __launch_bounds__(256) k_soa_many2(double2*, double2*, double2*, double2*, uint64_t);
__global__ void __launch_bounds__(256) k_soa_many(double2* x, double2* y, double2* w, double2* p, uint64_t npairs) {
    const uint64_t q = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (q < npairs) {
        double2 a = x[q], b = y[q], c = w[q], d = p[q];
        touch(a, b, c, d);
        x[q] = a; y[q] = b; w[q] = c; p[q] = d;
    }
}

// ... two pairs per thread (loads of both issued first)
__global__ void __launch_bounds__(256) k_soa_many2(double2* x, double2* y, double2* w, double2* p, uint64_t npairs) {
    const uint64_t q = (uint64_t)blockIdx.x * 512 + threadIdx.x, r = q + 256;
    double2 a, b, c, d, e, f, h, i;
    if (q < npairs) { a = x[q]; b = y[q]; c = w[q]; d = p[q]; }
    if (r < npairs) { e = x[r]; f = y[r]; h = w[r]; i = p[r]; }
    if (q < npairs) { touch(a, b, c, d); x[q] = a; y[q] = b; w[q] = c; p[q] = d; }
    if (r < npairs) { touch(e, f, h, i); x[r] = e; y[r] = f; w[r] = h; p[r] = i; }
}

__global__ void __launch_bounds__(1024, 1) k_soa_cs(double2* x, double2* y, double2* w, double2* p, uint64_t npairs) {
    CHUNK();
    for (uint64_t g = g0 + wid; g < g1; g += nw) {
        const uint64_t q = g * 32 + lane;
        if (q < npairs) {
            double2 a = __ldcs(x + q), b = __ldcs(y + q), c = __ldcs(w + q), d = __ldcs(p + q);
            touch(a, b, c, d);
            __stcs(x + q, a); __stcs(y + q, b); __stcs(w + q, c); __stcs(p + q, d);
        }
    }
}

__global__ void __launch_bounds__(1024, 1) k_soa_u2(double2* x, double2* y, double2* w, double2* p, uint64_t npairs) {
    CHUNK();
    for (uint64_t g = g0 + 2 * wid; g < g1; g += 2 * nw) {
        const uint64_t q = g * 32 + lane, r = q + 32;
        const bool vq = q < npairs && g < g1, vr = r < npairs && g + 1 < g1;
        double2 a, b, c, d, e, f, h, i;
        if (vq) { a = x[q]; b = y[q]; c = w[q]; d = p[q]; }
        if (vr) { e = x[r]; f = y[r]; h = w[r]; i = p[r]; }
        if (vq) { touch(a, b, c, d); x[q] = a; y[q] = b; w[q] = c; p[q] = d; }
        if (vr) { touch(e, f, h, i); x[r] = e; y[r] = f; w[r] = h; p[r] = i; }
    }
}

__global__ void __launch_bounds__(1024, 1) k_aosoa(double2* s, uint64_t npairs) {
    CHUNK();
    for (uint64_t g = g0 + wid; g < g1; g += nw) {
        const uint64_t q = g * 32 + lane;
        if (q < npairs) {
            double2* b = s + g * 128 + lane;
            double2 a = b[0], bb = b[32], c = b[64], d = b[96];
            touch(a, bb, c, d);
            b[0] = a; b[32] = bb; b[64] = c; b[96] = d;
        }
    }
}

__global__ void __launch_bounds__(1024, 1) k_soa_pp(const double2* x, const double2* y, const double2* w,
                                                    const double2* p, double2* X, double2* Y, double2* W, double2* P,
                                                    uint64_t npairs) {
    CHUNK();
    for (uint64_t g = g0 + wid; g < g1; g += nw) {
        const uint64_t q = g * 32 + lane;
        if (q < npairs) {
            double2 a = x[q], b = y[q], c = w[q], d = p[q];
            touch(a, b, c, d);
            X[q] = a; Y[q] = b; W[q] = c; P[q] = d;
        }
    }
}

__global__ void __launch_bounds__(1024, 1) k_aosoa_pp(const double2* s, double2* t, uint64_t npairs) {
    CHUNK();
    for (uint64_t g = g0 + wid; g < g1; g += nw) {
        const uint64_t q = g * 32 + lane;
        if (q < npairs) {
            const double2* b = s + g * 128 + lane;
            double2* o = t + g * 128 + lane;
            double2 a = b[0], bb = b[32], c = b[64], d = b[96];
            touch(a, bb, c, d);
            o[0] = a; o[32] = bb; o[64] = c; o[96] = d;
        }
    }
}

__global__ void k_copy(const double2* s, double2* t, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        t[i] = s[i];
}

int main(int argc, char** argv) {
    const uint64_t npairs = argc > 1 ? (uint64_t)atof(argv[1]) / 2 : 5000000;  // default 1e7 fish, 320 MB of state
    const uint64_t nblk = ((npairs + 31) / 32) * 128;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2 *a[8], *s, *t;
    for (auto& v : a) { cudaMalloc(&v, npairs * 16); cudaMemset(v, 0, npairs * 16); }
    cudaMalloc(&s, nblk * 16); cudaMalloc(&t, nblk * 16);
    cudaMemset(s, 0, nblk * 16); cudaMemset(t, 0, nblk * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[] = {"soa", "aosoa", "soa_cs", "soa_u2", "soa_pp", "aosoa_pp", "copy", "soa_gs", "soa_gs4", "soa_many",
                           "soa_many_occ4", "soa_many_occ2", "soa_many512_occ2"};
    cudaFuncSetAttribute(k_soa_many, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaFuncSetAttribute(k_soa_many2, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    for (int rep = 0; rep < 2; ++rep) {
        for (int k = 0; k < 13; ++k) {
            auto launch = [&](int i) {
                switch (k) {
                    case 0: k_soa<<<sms, 1024>>>(a[0], a[1], a[2], a[3], npairs); break;
                    case 1: k_aosoa<<<sms, 1024>>>(s, npairs); break;
                    case 2: k_soa_cs<<<sms, 1024>>>(a[0], a[1], a[2], a[3], npairs); break;
                    case 3: k_soa_u2<<<sms, 1024>>>(a[0], a[1], a[2], a[3], npairs); break;
                    case 4: if (i & 1) k_soa_pp<<<sms, 1024>>>(a[4], a[5], a[6], a[7], a[0], a[1], a[2], a[3], npairs);
                            else k_soa_pp<<<sms, 1024>>>(a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], npairs); break;
                    case 5: if (i & 1) k_aosoa_pp<<<sms, 1024>>>(t, s, npairs); else k_aosoa_pp<<<sms, 1024>>>(s, t, npairs); break;
                    case 6: if (i & 1) k_copy<<<sms * 4, 512>>>(t, s, nblk); else k_copy<<<sms * 4, 512>>>(s, t, nblk); break;
                    case 7: k_soa_gs<<<sms, 1024>>>(a[0], a[1], a[2], a[3], npairs); break;
                    case 8: k_soa_gs<<<sms * 4, 256>>>(a[0], a[1], a[2], a[3], npairs); break;
                    case 9: k_soa_many<<<(unsigned)((npairs + 255) / 256), 256>>>(a[0], a[1], a[2], a[3], npairs); break;
                    // dynamic shared memory only to cap the resident CTAs per SM (4 -> 1024 threads, 2 -> 512)
                    case 10: k_soa_many<<<(unsigned)((npairs + 255) / 256), 256, 50 * 1024>>>(a[0], a[1], a[2], a[3], npairs); break;
                    case 11: k_soa_many<<<(unsigned)((npairs + 255) / 256), 256, 100 * 1024>>>(a[0], a[1], a[2], a[3], npairs); break;
                    case 12: k_soa_many2<<<(unsigned)((npairs + 511) / 512), 256, 100 * 1024>>>(a[0], a[1], a[2], a[3], npairs); break;
                }
            };
            for (int i = 0; i < 6; ++i) launch(i);
            cudaEventRecord(e0);
            const int it = npairs > 20000000 ? 10 : 50;
            for (int i = 0; i < it; ++i) launch(i);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double us = 1e3 * ms / it;
            const double bytes = k == 6 ? nblk * 32.0 : npairs * 128.0;
            printf("{\"pattern\": \"%s\", \"us\": %.2f, \"GBps_moved\": %.1f}\n", names[k], us, bytes / us / 1e3);
        }
    }
    return cudaGetLastError() != cudaSuccess;
}
