/*
 * tests/nccl_shim.c — TEST DEVICE: a minimal stand-in for libnccl that lets
 * several processes share ONE GPU (real NCCL refuses two ranks on one device),
 * so the library's NCCL code path (communicator set-up, packed all-reduce on
 * the context stream, sliced all-reduces on the exchange-pipelining stream,
 * the gathers of spdp_counts / spdp_loglik) can be exercised on a 1-GPU box.
 *
 * Implements ncclGetUniqueId, ncclCommInitRank, ncclAllReduce (sum of int32,
 * int64, float64), ncclCommDestroy, ncclGetErrorString.  The ranks meet in a
 * file-backed shared mapping under /tmp: each all-reduce synchronises the
 * caller's stream, copies its buffer to its slot, waits at a barrier, sums all
 * slots in rank order and copies the result back.  Blocking and slow: it
 * checks semantics, not performance.  Selected with SPDP_NCCL_LIB=<this .so>.
 */
#define _GNU_SOURCE
#include <cuda_runtime.h>
#include <fcntl.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#define SLOT (8u << 20)            /* bytes per rank and round */
#define MAXR 8

typedef struct { char b[128]; } ncclUniqueId;
typedef struct {
    volatile int count, generation, joined, pad;
} hdr_t;
typedef struct {
    int nranks, rank;
    hdr_t *h;
    char *slots;
    size_t bytes;
    char path[128];
} comm_t;

static void barrier(comm_t *c) {
    int gen = __atomic_load_n(&c->h->generation, __ATOMIC_ACQUIRE);
    if (__atomic_add_fetch(&c->h->count, 1, __ATOMIC_ACQ_REL) == c->nranks) {
        __atomic_store_n(&c->h->count, 0, __ATOMIC_RELAXED);
        __atomic_add_fetch(&c->h->generation, 1, __ATOMIC_RELEASE);
    } else {
        while (__atomic_load_n(&c->h->generation, __ATOMIC_ACQUIRE) == gen) usleep(50);
    }
}

int ncclGetUniqueId(ncclUniqueId *id) {
    memset(id->b, 0, sizeof id->b);
    struct timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    snprintf(id->b, sizeof id->b, "/tmp/spdp_nccl_shim_%d_%ld_%ld", (int)getpid(), (long)ts.tv_sec, ts.tv_nsec);
    return 0;
}

int ncclCommInitRank(void **comm, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || nranks > MAXR || rank < 0 || rank >= nranks) return 4;
    comm_t *c = (comm_t *)calloc(1, sizeof(comm_t));
    c->nranks = nranks; c->rank = rank;
    snprintf(c->path, sizeof c->path, "%s", id.b);
    c->bytes = 4096 + (size_t)nranks * SLOT;
    int fd = open(c->path, O_RDWR | O_CREAT, 0600);
    if (fd < 0) return 2;
    if (ftruncate(fd, (off_t)c->bytes) != 0) { close(fd); return 2; }
    void *p = mmap(NULL, c->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return 2;
    c->h = (hdr_t *)p;
    c->slots = (char *)p + 4096;
    __atomic_add_fetch(&c->h->joined, 1, __ATOMIC_ACQ_REL);
    while (__atomic_load_n(&c->h->joined, __ATOMIC_ACQUIRE) < nranks) usleep(100);
    *comm = c;
    return 0;
}

int ncclAllReduce(const void *send, void *recv, size_t count, int dtype, int op, void *comm, cudaStream_t st) {
    comm_t *c = (comm_t *)comm;
    size_t es = dtype == 2 ? 4 : (dtype == 4 || dtype == 8) ? 8 : 0;   /* int32, int64, float64 */
    if (!es || op != 0) return 5;
    if (cudaStreamSynchronize(st) != cudaSuccess) return 1;
    const size_t per = SLOT / es;
    char *tmp = (char *)malloc(SLOT);
    for (size_t off = 0; off < count || (count == 0 && off == 0); off += per) {
        size_t n = count - off < per ? count - off : per;
        if (count == 0) n = 0;
        char *mine = c->slots + (size_t)c->rank * SLOT;
        if (n && (cudaMemcpyAsync(mine, (const char *)send + off * es, n * es, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                  cudaStreamSynchronize(st) != cudaSuccess)) return 1;
        barrier(c);
        memset(tmp, 0, n * es);
        for (int r = 0; r < c->nranks; r++) {      /* fixed rank order: deterministic sums */
            const char *src = c->slots + (size_t)r * SLOT;
            for (size_t j = 0; j < n; j++) {
                if (dtype == 2) ((int32_t *)tmp)[j] = (int32_t)((uint32_t)((int32_t *)tmp)[j] + (uint32_t)((const int32_t *)src)[j]);
                else if (dtype == 4) ((int64_t *)tmp)[j] = (int64_t)((uint64_t)((int64_t *)tmp)[j] + (uint64_t)((const int64_t *)src)[j]);
                else ((double *)tmp)[j] += ((const double *)src)[j];
            }
        }
        barrier(c);                                  /* every rank has read every slot */
        /* on the caller's stream, complete before returning (a pageable cudaMemcpy may still be in flight) */
        if (n && (cudaMemcpyAsync((char *)recv + off * es, tmp, n * es, cudaMemcpyHostToDevice, st) != cudaSuccess ||
                  cudaStreamSynchronize(st) != cudaSuccess)) return 1;
        if (count == 0) break;
    }
    free(tmp);
    return 0;
}

int ncclCommDestroy(void *comm) {
    comm_t *c = (comm_t *)comm;
    if (!c) return 0;
    barrier(c);
    munmap((void *)c->h, c->bytes);
    if (c->rank == 0) unlink(c->path);
    free(c);
    return 0;
}

const char *ncclGetErrorString(int r) { return r ? "nccl shim error" : "no error"; }
