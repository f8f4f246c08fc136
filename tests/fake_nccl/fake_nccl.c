/* Test infrastructure, not product code: a stand-in for libnccl.so.2 that lets SEVERAL RANKS SHARE ONE
 * GPU, so the one-process-per-GPU z-slab path of libsmg (smg_create_rank: halo send/recv groups, halo
 * frames, ghost pushes, plane-partial all-reduce, coarse all-gather, solution broadcast) runs with
 * world_size > 1 on the 1-GPU boxes this project is tested on.  Real NCCL refuses two ranks on one
 * device.  Loaded through SMG_NCCL_LIB (host.cpp nccl()); tests/test_gpu_zz_fake_ranks.py drives it.
 *
 * Transport: POSIX shared memory.  Every call first drains its CUDA stream (cudaStreamSynchronize),
 * then moves the data with blocking copies through host memory, so stream order is preserved for
 * eager launches; it cannot be captured into a CUDA graph (the tests set SMG_DIST_GRAPH=0).
 *   send/recv    one byte FIFO per ordered rank pair; inside a group all sends run before the recvs
 *   all-reduce   every rank stages its buffer, barrier, every rank sums the stages in rank order
 *   all-gather / broadcast   staged the same way
 * Only ncclDouble / ncclSum (what libsmg uses).  ncclCommSplit is deliberately absent: libsmg then
 * runs its comm-stream transfers on the rank communicator, the fallback path.
 */
#define _GNU_SOURCE
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <time.h>
#include <unistd.h>

#define MAX_RANKS 16
#define COLL_CAP ((size_t)16 << 20) /* bytes staged per rank in a collective (only touched pages cost /dev/shm) */
#define FIFO_CAP ((size_t)4 << 20)  /* bytes in flight per ordered pair: > the sends of one group; small so that a 64 MB /dev/shm holds every FIFO */
#define WAIT_LIMIT_S 120.0          /* a peer that never shows up fails the call instead of hanging the box */

typedef struct {
    volatile uint64_t head, tail; /* bytes written / consumed */
    char data[];
} Fifo;

typedef struct {
    volatile int count;
    volatile int gen;
    char pad[4096 - 2 * sizeof(int)];
    char stage[];
} Main;

struct ncclComm {
    int rank, nranks;
    char name[64];
    Main* m;
    size_t main_bytes;
    Fifo* out[MAX_RANKS]; /* this rank -> peer */
    Fifo* in[MAX_RANKS];  /* peer -> this rank */
};

typedef struct {
    int kind; /* 0 send, 1 recv, 2 allreduce, 3 allgather, 4 broadcast */
    const void* sbuf;
    void* rbuf;
    size_t count;
    int peer;
    struct ncclComm* comm;
    cudaStream_t stream;
} Op;

static __thread int g_depth = 0;
static __thread Op g_ops[4096];
static __thread int g_nops = 0;

static double now_s(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec + 1e-9 * t.tv_nsec;
}

static void* map_shm(const char* name, size_t bytes) {
    int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
    if (fd < 0) return NULL;
    if (ftruncate(fd, (off_t)bytes) != 0) {
        close(fd);
        return NULL;
    }
    void* p = mmap(NULL, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    return p == MAP_FAILED ? NULL : p;
}

static int barrier(struct ncclComm* c) {
    Main* m = c->m;
    const int gen = __atomic_load_n(&m->gen, __ATOMIC_ACQUIRE);
    if (__atomic_add_fetch(&m->count, 1, __ATOMIC_ACQ_REL) == c->nranks) {
        __atomic_store_n(&m->count, 0, __ATOMIC_RELEASE);
        __atomic_add_fetch(&m->gen, 1, __ATOMIC_ACQ_REL);
        return 0;
    }
    const double t0 = now_s();
    while (__atomic_load_n(&m->gen, __ATOMIC_ACQUIRE) == gen) {
        if (now_s() - t0 > WAIT_LIMIT_S) return -1;
        usleep(20);
    }
    return 0;
}

static Fifo* fifo(struct ncclComm* c, int src, int dst) {
    Fifo** slot = src == c->rank ? &c->out[dst] : &c->in[src];
    if (!*slot) {
        char name[96];
        snprintf(name, sizeof name, "%s_%d_%d", c->name, src, dst);
        *slot = (Fifo*)map_shm(name, sizeof(Fifo) + FIFO_CAP);
    }
    return *slot;
}

static int fifo_put(Fifo* f, const char* src, size_t n) {
    const double t0 = now_s();
    size_t done = 0;
    while (done < n) {
        const uint64_t head = f->head, tail = __atomic_load_n(&f->tail, __ATOMIC_ACQUIRE);
        size_t room = FIFO_CAP - (size_t)(head - tail);
        if (room == 0) {
            if (now_s() - t0 > WAIT_LIMIT_S) return -1;
            usleep(20);
            continue;
        }
        size_t k = n - done < room ? n - done : room;
        const size_t off = (size_t)(head % FIFO_CAP);
        if (k > FIFO_CAP - off) k = FIFO_CAP - off;
        memcpy(f->data + off, src + done, k);
        __atomic_store_n(&f->head, head + k, __ATOMIC_RELEASE);
        done += k;
    }
    return 0;
}

static int fifo_get(Fifo* f, char* dst, size_t n) {
    const double t0 = now_s();
    size_t done = 0;
    while (done < n) {
        const uint64_t tail = f->tail, head = __atomic_load_n(&f->head, __ATOMIC_ACQUIRE);
        size_t avail = (size_t)(head - tail);
        if (avail == 0) {
            if (now_s() - t0 > WAIT_LIMIT_S) return -1;
            usleep(20);
            continue;
        }
        size_t k = n - done < avail ? n - done : avail;
        const size_t off = (size_t)(tail % FIFO_CAP);
        if (k > FIFO_CAP - off) k = FIFO_CAP - off;
        memcpy(dst + done, f->data + off, k);
        __atomic_store_n(&f->tail, tail + k, __ATOMIC_RELEASE);
        done += k;
    }
    return 0;
}

/* copy on the op's own stream and wait: a plain cudaMemcpy from pageable memory may return before the
 * DMA has landed, and the library's non-blocking stream is not ordered after the legacy stream */
static cudaError_t copy_sync(void* dst, const void* src, size_t bytes, enum cudaMemcpyKind kind, cudaStream_t st) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, st);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(st);
}

static ncclResult_t run_op(const Op* o) {
    struct ncclComm* c = o->comm;
    const size_t bytes = o->count * sizeof(double);
    if (o->kind == 0) { /* send: [count][payload] */
        Fifo* f = fifo(c, c->rank, o->peer);
        char* h = (char*)malloc(bytes + 8);
        if (!f || !h) return ncclSystemError;
        const uint64_t n = o->count;
        memcpy(h, &n, 8);
        if (copy_sync(h + 8, o->sbuf, bytes, cudaMemcpyDeviceToHost, o->stream) != cudaSuccess) return ncclUnhandledCudaError;
        const int rc = fifo_put(f, h, bytes + 8);
        free(h);
        return rc ? ncclInternalError : ncclSuccess;
    }
    if (o->kind == 1) { /* recv: sizes must match the sender's */
        Fifo* f = fifo(c, o->peer, c->rank);
        char* h = (char*)malloc(bytes + 8);
        if (!f || !h) return ncclSystemError;
        uint64_t n = 0;
        if (fifo_get(f, (char*)&n, 8)) return ncclInternalError;
        if (n != o->count) {
            fprintf(stderr, "fake_nccl: rank %d recv from %d expects %zu doubles, peer sent %llu\n", c->rank, o->peer,
                    o->count, (unsigned long long)n);
            return ncclInvalidArgument;
        }
        if (fifo_get(f, h, bytes)) return ncclInternalError;
        const cudaError_t e = copy_sync(o->rbuf, h, bytes, cudaMemcpyHostToDevice, o->stream);
        free(h);
        return e == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError;
    }
    /* collectives through the per-rank stages */
    if (bytes > COLL_CAP) return ncclInvalidArgument;
    char* mine = c->m->stage + (size_t)c->rank * COLL_CAP;
    if (o->kind != 4 || c->rank == o->peer)
        if (copy_sync(mine, o->sbuf, bytes, cudaMemcpyDeviceToHost, o->stream) != cudaSuccess) return ncclUnhandledCudaError;
    if (barrier(c)) return ncclInternalError;
    ncclResult_t rc = ncclSuccess;
    if (o->kind == 2) {
        double* acc = (double*)malloc(bytes);
        if (!acc) return ncclSystemError;
        memcpy(acc, c->m->stage, bytes);
        for (int r = 1; r < c->nranks; ++r) {
            const double* s = (const double*)(c->m->stage + (size_t)r * COLL_CAP);
            for (size_t k = 0; k < o->count; ++k) acc[k] = acc[k] + s[k];
        }
        if (copy_sync(o->rbuf, acc, bytes, cudaMemcpyHostToDevice, o->stream) != cudaSuccess) rc = ncclUnhandledCudaError;
        free(acc);
    } else if (o->kind == 3) {
        for (int r = 0; r < c->nranks && rc == ncclSuccess; ++r)
            if (copy_sync((char*)o->rbuf + (size_t)r * bytes, c->m->stage + (size_t)r * COLL_CAP, bytes,
                          cudaMemcpyHostToDevice, o->stream) != cudaSuccess)
                rc = ncclUnhandledCudaError;
    } else {
        if (copy_sync(o->rbuf, c->m->stage + (size_t)o->peer * COLL_CAP, bytes, cudaMemcpyHostToDevice, o->stream) != cudaSuccess)
            rc = ncclUnhandledCudaError;
    }
    if (barrier(c)) return ncclInternalError; /* stages free for the next collective */
    return rc;
}

static ncclResult_t flush(void) {
    ncclResult_t rc = ncclSuccess;
    for (int k = 0; k < g_nops; ++k) /* everything enqueued before the call has run */
        if (cudaStreamSynchronize(g_ops[k].stream) != cudaSuccess) rc = ncclUnhandledCudaError;
    for (int k = 0; k < g_nops && rc == ncclSuccess; ++k)
        if (g_ops[k].kind == 0) rc = run_op(&g_ops[k]);
    for (int k = 0; k < g_nops && rc == ncclSuccess; ++k)
        if (g_ops[k].kind != 0) rc = run_op(&g_ops[k]);
    g_nops = 0;
    return rc;
}

static ncclResult_t enqueue(int kind, const void* s, void* r, size_t count, ncclDataType_t t, int peer, ncclComm_t c,
                            cudaStream_t st) {
    if (t != ncclDouble || !c || g_nops >= 4096) return ncclInvalidArgument;
    Op o = {kind, s, r, count, peer, c, st};
    g_ops[g_nops++] = o;
    return g_depth == 0 ? flush() : ncclSuccess;
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    memset(id, 0, sizeof *id);
    FILE* f = fopen("/dev/urandom", "rb");
    uint64_t r = (uint64_t)getpid() * 2654435761u ^ (uint64_t)time(NULL);
    if (f) {
        if (fread(&r, 8, 1, f) != 1) r ^= 0x9e3779b97f4a7c15ull;
        fclose(f);
    }
    snprintf(id->internal, sizeof id->internal, "/fnccl_%016llx", (unsigned long long)r);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || nranks > MAX_RANKS || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    struct ncclComm* c = (struct ncclComm*)calloc(1, sizeof *c);
    if (!c) return ncclSystemError;
    c->rank = rank;
    c->nranks = nranks;
    memcpy(c->name, id.internal, sizeof c->name - 1);
    c->main_bytes = sizeof(Main) + (size_t)nranks * COLL_CAP;
    c->m = (Main*)map_shm(c->name, c->main_bytes);
    if (!c->m) {
        free(c);
        return ncclSystemError;
    }
    if (barrier(c)) return ncclInternalError;
    *out = c;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
    if (!c) return ncclSuccess;
    barrier(c);
    char name[96];
    for (int r = 0; r < c->nranks; ++r) {
        if (c->out[r]) {
            munmap(c->out[r], sizeof(Fifo) + FIFO_CAP);
            snprintf(name, sizeof name, "%s_%d_%d", c->name, c->rank, r);
            shm_unlink(name);
        }
        if (c->in[r]) munmap(c->in[r], sizeof(Fifo) + FIFO_CAP);
    }
    munmap(c->m, c->main_bytes);
    if (c->rank == 0) shm_unlink(c->name);
    free(c);
    return ncclSuccess;
}

ncclResult_t ncclGroupStart(void) {
    ++g_depth;
    return ncclSuccess;
}
ncclResult_t ncclGroupEnd(void) {
    if (g_depth <= 0) return ncclInvalidUsage;
    return --g_depth == 0 ? flush() : ncclSuccess;
}
ncclResult_t ncclSend(const void* s, size_t n, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st) {
    return enqueue(0, s, NULL, n, t, peer, c, st);
}
ncclResult_t ncclRecv(void* r, size_t n, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st) {
    return enqueue(1, NULL, r, n, t, peer, c, st);
}
ncclResult_t ncclAllReduce(const void* s, void* r, size_t n, ncclDataType_t t, ncclRedOp_t op, ncclComm_t c,
                           cudaStream_t st) {
    if (op != ncclSum) return ncclInvalidArgument;
    return enqueue(2, s, r, n, t, -1, c, st);
}
ncclResult_t ncclAllGather(const void* s, void* r, size_t n, ncclDataType_t t, ncclComm_t c, cudaStream_t st) {
    return enqueue(3, s, r, n, t, -1, c, st);
}
ncclResult_t ncclBroadcast(const void* s, void* r, size_t n, ncclDataType_t t, int root, ncclComm_t c,
                           cudaStream_t st) {
    return enqueue(4, s, r, n, t, root, c, st);
}
const char* ncclGetErrorString(ncclResult_t r) {
    return r == ncclSuccess ? "no error" : "fake_nccl: transport error (see stderr; peer missing, size mismatch or CUDA)";
}
