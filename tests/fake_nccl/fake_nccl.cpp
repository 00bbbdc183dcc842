// fake_nccl.cpp -- TEST INFRASTRUCTURE: a minimal host-staged stand-in for the NCCL calls libmf
// makes, so the multi-rank partitioned path (one process per rank) can run as several processes on
// ONE GPU, which real NCCL refuses ("duplicate GPU").  LD_PRELOAD it into every rank process.
//
// Semantics kept: stream ordering (every op synchronises its stream before touching the buffers and
// completes before returning), point-to-point pairing by (src, dst, per-pair sequence number),
// grouped send/recv (sends are posted before receives, so a ring exchange cannot deadlock),
// all-gather and sum all-reduce (float64 sum).  Transport: a shared mmap of a file in /tmp named
// after the unique id.  Slow and simple; it checks the protocol, not performance.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

namespace {

constexpr int kMaxRanks = 4;
constexpr size_t kSlotBytes = 4u << 20;  // per (src, dst) mailbox
constexpr size_t kCollBytes = 4u << 20;  // per rank, collectives

struct Mailbox {
    std::atomic<uint64_t> seq;   // number of messages posted so far on this (src, dst) pair
    std::atomic<uint64_t> taken; // number of messages consumed
    uint64_t bytes;
};

struct Shared {
    std::atomic<int> joined;
    std::atomic<uint64_t> coll_arrive[kMaxRanks];  // per-rank collective counter (barrier)
    Mailbox box[kMaxRanks][kMaxRanks];
};

struct Comm {
    int rank, nranks;
    char *base;
    Shared *sh;
    uint64_t sent[kMaxRanks] = {}, recvd[kMaxRanks] = {};
    uint64_t coll = 0;
    struct Op {
        bool send;
        const void *sbuf;
        void *rbuf;
        size_t bytes;
        int peer;
        cudaStream_t st;
    };
    std::vector<Op> pending;
    char *slot(int src, int dst) {
        return base + sizeof(Shared) + ((size_t)src * kMaxRanks + dst) * kSlotBytes;
    }
    char *coll_buf(int r) { return base + sizeof(Shared) + (size_t)kMaxRanks * kMaxRanks * kSlotBytes + r * kCollBytes; }
};

int g_group = 0;
std::vector<Comm *> g_comms;

size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: case ncclBfloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        default: return 8;
    }
}

void spin_until(const std::atomic<uint64_t> &a, uint64_t v) {
    while (a.load(std::memory_order_acquire) < v) std::this_thread::sleep_for(std::chrono::microseconds(20));
}

void do_send(Comm *c, const Comm::Op &op) {
    Mailbox &mb = c->sh->box[c->rank][op.peer];
    // one message in flight per pair: wait until the previous one was taken
    spin_until(mb.taken, c->sent[op.peer]);
    if (op.bytes > kSlotBytes) { fprintf(stderr, "fake nccl: message too large\n"); abort(); }
    cudaMemcpyAsync(c->slot(c->rank, op.peer), op.sbuf, op.bytes, cudaMemcpyDeviceToHost, op.st);
    cudaStreamSynchronize(op.st);
    mb.bytes = op.bytes;
    c->sent[op.peer]++;
    mb.seq.store(c->sent[op.peer], std::memory_order_release);
}

void do_recv(Comm *c, const Comm::Op &op) {
    Mailbox &mb = c->sh->box[op.peer][c->rank];
    spin_until(mb.seq, c->recvd[op.peer] + 1);
    // copies run on the op's stream and complete before the call returns (a legacy-stream cudaMemcpy
    // from pageable memory may still be in flight when the caller's non-blocking stream reads rbuf)
    cudaMemcpyAsync(op.rbuf, c->slot(op.peer, c->rank), op.bytes, cudaMemcpyHostToDevice, op.st);
    cudaStreamSynchronize(op.st);
    c->recvd[op.peer]++;
    mb.taken.store(c->recvd[op.peer], std::memory_order_release);
}

void flush(Comm *c) {
    for (auto &op : c->pending)
        if (op.send) do_send(c, op);
    for (auto &op : c->pending)
        if (!op.send) do_recv(c, op);
    c->pending.clear();
}

void barrier(Comm *c) {
    c->coll++;
    c->sh->coll_arrive[c->rank].store(c->coll, std::memory_order_release);
    for (int r = 0; r < c->nranks; r++) spin_until(c->sh->coll_arrive[r], c->coll);
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId *id) {
    std::random_device rd;
    std::memset(id, 0, sizeof *id);
    snprintf(id->internal, sizeof id->internal, "/tmp/fakenccl_%08x%08x", rd(), rd());
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t *comm, int nranks, ncclUniqueId id, int rank) {
    if (nranks > kMaxRanks) return ncclInvalidArgument;
    const size_t total = sizeof(Shared) + (size_t)kMaxRanks * kMaxRanks * kSlotBytes + kMaxRanks * kCollBytes;
    int fd = open(id.internal, O_CREAT | O_RDWR, 0600);  // a file in /tmp (no /dev/shm size limit)
    if (fd < 0) return ncclSystemError;
    if (ftruncate(fd, (off_t)total) != 0) return ncclSystemError;
    void *p = mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return ncclSystemError;
    Comm *c = new Comm();
    c->rank = rank;
    c->nranks = nranks;
    c->base = (char *)p;
    c->sh = (Shared *)p;
    c->sh->joined.fetch_add(1);
    while (c->sh->joined.load() < nranks) std::this_thread::sleep_for(std::chrono::microseconds(50));
    *comm = (ncclComm_t)c;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    delete (Comm *)comm;  // the mapping stays until exit; the shm file is removed by the test
    return ncclSuccess;
}

const char *ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "success (fake nccl)" : "error (fake nccl)"; }

ncclResult_t ncclGroupStart() {
    g_group++;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
    if (--g_group == 0) {
        for (Comm *c : g_comms) flush(c);
        g_comms.clear();
    }
    return ncclSuccess;
}

static ncclResult_t post(Comm *c, const Comm::Op &op) {
    c->pending.push_back(op);
    if (g_group == 0) flush(c);
    else if (std::find(g_comms.begin(), g_comms.end(), c) == g_comms.end()) g_comms.push_back(c);
    return ncclSuccess;
}

ncclResult_t ncclSend(const void *buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm, cudaStream_t st) {
    return post((Comm *)comm, {true, buf, nullptr, count * type_size(dt), peer, st});
}

ncclResult_t ncclRecv(void *buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm, cudaStream_t st) {
    return post((Comm *)comm, {false, nullptr, buf, count * type_size(dt), peer, st});
}

ncclResult_t ncclAllGather(const void *sbuf, void *rbuf, size_t count, ncclDataType_t dt, ncclComm_t comm,
                           cudaStream_t st) {
    Comm *c = (Comm *)comm;
    const size_t bytes = count * type_size(dt);
    if (bytes > kCollBytes) return ncclInvalidArgument;
    cudaMemcpyAsync(c->coll_buf(c->rank), sbuf, bytes, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    barrier(c);
    for (int r = 0; r < c->nranks; r++)
        cudaMemcpyAsync((char *)rbuf + r * bytes, c->coll_buf(r), bytes, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    barrier(c);
    return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void *sbuf, void *rbuf, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t st) {
    Comm *c = (Comm *)comm;
    if (dt != ncclFloat64 || op != ncclSum || count * 8 > kCollBytes) return ncclInvalidArgument;
    cudaMemcpyAsync(c->coll_buf(c->rank), sbuf, count * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    barrier(c);
    std::vector<double> acc(count, 0.0);
    for (int r = 0; r < c->nranks; r++) {
        const double *x = (const double *)c->coll_buf(r);
        for (size_t i = 0; i < count; i++) acc[i] += x[i];
    }
    barrier(c);
    cudaMemcpyAsync(rbuf, acc.data(), count * 8, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    if (getenv("FAKE_NCCL_DEBUG")) {
        const double *mine = (const double *)c->coll_buf(c->rank);
        fprintf(stderr, "fake nccl rank %d allreduce count %zu: mine[0]=%.17g sum[0]=%.17g sum[1]=%.17g\n", c->rank,
                count, mine[0], acc[0], count > 1 ? acc[1] : 0.0);
    }
    return ncclSuccess;
}

}  // extern "C"
