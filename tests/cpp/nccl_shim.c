/* nccl_shim.c -- TEST INFRASTRUCTURE: a stand-in for the five libnccl entry
 * points the engine dlopens (fsb_engine.cu nccl_load), so that the in-graph
 * exchange of a world_size > 1 run -- the ncclAllGather node between two step
 * kernels of the captured graph, the rank-order combine in the next kernel,
 * the shard partition and the unique-id bootstrap -- can be exercised by two
 * PROCESSES sharing the one GPU this pool offers.  NCCL itself refuses two
 * ranks on one device.
 *
 * ncclAllGather here is three stream operations, all capturable in a CUDA
 * graph like NCCL's own kernel: a D2H copy of the rank's block into pinned
 * memory, a host node that meets the other ranks in POSIX shared memory (named
 * by the unique id) and gathers every block, and an H2D copy of the gathered
 * blocks.  No kernel ever waits for another rank's kernel -- only host
 * callbacks wait, each on its own process's stream -- so the processes can
 * time-slice one GPU (B200_PROFILING.md: ranks whose kernels wait on one
 * another must not share a GPU).
 *
 * Built by tests/cpp/Makefile into tests/cpp/libnccl_shim.so; loaded only by
 * tests/test_nccl_shim.py through FSB_NCCL_LIB.  Not part of the product.
 */
#define _GNU_SOURCE
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sched.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <time.h>
#include <unistd.h>

typedef enum { ncclSuccess = 0, ncclUnhandledCudaError = 1, ncclSystemError = 2, ncclInternalError = 3,
               ncclInvalidArgument = 4 } ncclResult_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclDataType_t; /* ncclFloat64 = 8 is the only type the engine sends */

#define SHIM_MAX_RANKS 8
#define SHIM_MAX_BYTES 256 /* per rank and call: the engine sends 4 fp64 */

struct shim_shared {
    volatile uint64_t seq[SHIM_MAX_RANKS];                       /* calls completed-or-entered per rank */
    unsigned char slot[2][SHIM_MAX_RANKS][SHIM_MAX_BYTES];       /* by call parity */
};

struct shim_comm {
    int nranks, rank;
    char name[64];
    struct shim_shared* sh;
    uint64_t calls;      /* host-side count of exchanges executed (replays of a graph included) */
    unsigned char* pin;  /* pinned staging: nranks blocks */
    size_t bytes;        /* per-rank bytes of the captured exchange */
};
typedef struct shim_comm* ncclComm_t;

const char* ncclGetErrorString(ncclResult_t r) {
    switch (r) {
        case ncclSuccess: return "no error (nccl shim)";
        case ncclUnhandledCudaError: return "unhandled cuda error (nccl shim)";
        case ncclSystemError: return "unhandled system error (nccl shim)";
        case ncclInvalidArgument: return "invalid argument (nccl shim)";
        default: return "internal error (nccl shim)";
    }
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    if (!id) return ncclInvalidArgument;
    memset(id, 0, sizeof *id);
    struct timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    snprintf(id->internal, sizeof id->internal, "/fsb_nccl_shim_%d_%lld_%ld", (int)getpid(), (long long)ts.tv_sec,
             ts.tv_nsec);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    if (!comm || nranks < 1 || nranks > SHIM_MAX_RANKS || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    struct shim_comm* c = (struct shim_comm*)calloc(1, sizeof *c);
    if (!c) return ncclSystemError;
    c->nranks = nranks;
    c->rank = rank;
    memcpy(c->name, id.internal, sizeof c->name - 1); /* calloc left the terminator */
    int fd = shm_open(c->name, O_CREAT | O_RDWR, 0600);  /* a fresh object is zero-filled */
    if (fd < 0 || ftruncate(fd, sizeof(struct shim_shared)) != 0) {
        free(c);
        return ncclSystemError;
    }
    c->sh = (struct shim_shared*)mmap(NULL, sizeof(struct shim_shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (c->sh == MAP_FAILED) {
        free(c);
        return ncclSystemError;
    }
    if (cudaHostAlloc((void**)&c->pin, (size_t)SHIM_MAX_RANKS * SHIM_MAX_BYTES, cudaHostAllocDefault) != cudaSuccess) {
        munmap((void*)c->sh, sizeof(struct shim_shared));
        free(c);
        return ncclUnhandledCudaError;
    }
    *comm = c;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
    if (!c) return ncclSuccess;
    if (c->pin) cudaFreeHost(c->pin);
    if (c->sh) munmap((void*)c->sh, sizeof(struct shim_shared));
    shm_unlink(c->name); /* the last unlink wins; the others fail harmlessly */
    free(c);
    return ncclSuccess;
}

/* Host node: publish this rank's block under the call's parity, meet the other
 * ranks, gather.  A rank can run at most one call ahead of the slowest one
 * (every call waits for all), so two slot sets are enough. */
static void CUDART_CB shim_exchange(void* arg) {
    struct shim_comm* c = (struct shim_comm*)arg;
    const uint64_t s = c->calls++;
    const int par = (int)(s & 1);
    memcpy(c->sh->slot[par][c->rank], c->pin + (size_t)c->rank * c->bytes, c->bytes);
    __sync_synchronize();
    c->sh->seq[c->rank] = s + 1;
    /* bounded: a rank that died must fail the test (NaN partials), not hang the GPU box */
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    int lost = 0;
    for (int r = 0; r < c->nranks && !lost; ++r) {
        while (c->sh->seq[r] < s + 1) {
            sched_yield();
            clock_gettime(CLOCK_MONOTONIC, &t1);
            if (t1.tv_sec - t0.tv_sec > 120) {
                lost = 1;
                break;
            }
        }
    }
    __sync_synchronize();
    for (int r = 0; r < c->nranks; ++r) {
        if (lost) memset(c->pin + (size_t)r * c->bytes, 0xff, c->bytes); /* NaN */
        else memcpy(c->pin + (size_t)r * c->bytes, c->sh->slot[par][r], c->bytes);
    }
}

ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t type, ncclComm_t c,
                           cudaStream_t stream) {
    if (!c || type != 8 /* ncclFloat64 */) return ncclInvalidArgument;
    const size_t bytes = count * 8;
    if (bytes == 0 || bytes > SHIM_MAX_BYTES) return ncclInvalidArgument;
    if (c->bytes && c->bytes != bytes) return ncclInvalidArgument; /* one message size per communicator */
    c->bytes = bytes;
    if (cudaMemcpyAsync(c->pin + (size_t)c->rank * bytes, sendbuff, bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return ncclUnhandledCudaError;
    if (cudaLaunchHostFunc(stream, shim_exchange, c) != cudaSuccess) return ncclUnhandledCudaError;
    if (cudaMemcpyAsync(recvbuff, c->pin, (size_t)c->nranks * bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return ncclUnhandledCudaError;
    return ncclSuccess;
}
