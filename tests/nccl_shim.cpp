// nccl_shim.cpp -- TEST INFRASTRUCTURE: a stand-in for libnccl.so.2 that lets several
// PROCESSES on ONE GPU run libfgf.so's multi-rank band path (fgf_filter_band /
// fgf_filter_band_ex: the library's own ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd
// call sequence, halo geometry and stream orchestration) when only one GPU is available.
// Loaded by libfgf.so instead of NCCL when FGF_DEV=1 and FGF_NCCL_LIB=<this .so> are set
// (tests/test_band_multirank_gpu.py).  Not part of the product and never used by bench.py.
//
// Point-to-point semantics as NCCL's, restricted to what the band path uses (ncclFloat32
// send / recv inside groups, matched in posting order per (sender, receiver) pair):
//   ncclSend    copies the buffer, stream-ordered on the caller's stream, into a staging
//               buffer of its own and records an interprocess event after the copy (so the
//               caller may reuse its buffer as soon as its stream passes the send, as with
//               NCCL), then publishes the staging buffer's IPC handle and the event's IPC
//               handle in a message file  <dir>/m_<src>_<dst>_<seq>  (written, then renamed);
//   ncclRecv    queues the receive;
//   ncclGroupEnd (or a receive outside a group) waits on the HOST until each queued receive's
//               message file exists -- every process posts all the sends of a group before it
//               waits, and a send never waits, so there is no cycle -- then makes the
//               receiver's stream wait for the sender's event (recorded before the file was
//               written: the GPU never waits on work that is not yet enqueued) and copies the
//               staging buffer into the receive buffer on that stream;
//   ncclCommDestroy  writes <dir>/d_<rank> and waits for every rank's file before it frees
//               its staging buffers (each receiver synchronised its copies before returning).
// ncclUniqueId carries the rendezvous directory.  No kernel of one process ever spins on
// another process's work.
#include <cuda_runtime.h>
#include <dirent.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <string>
#include <vector>

extern "C" {

typedef struct ncclComm* ncclComm_t;
typedef enum { ncclSuccess = 0, ncclUnhandledCudaError = 1, ncclSystemError = 2,
               ncclInternalError = 3, ncclInvalidArgument = 4, ncclInvalidUsage = 5 } ncclResult_t;
typedef enum { ncclInt8 = 0, ncclUint8 = 1, ncclInt32 = 2, ncclUint32 = 3, ncclInt64 = 4,
               ncclUint64 = 5, ncclFloat16 = 6, ncclFloat32 = 7, ncclFloat64 = 8 } ncclDataType_t;
#define NCCL_UNIQUE_ID_BYTES 128
typedef struct { char internal[NCCL_UNIQUE_ID_BYTES]; } ncclUniqueId;

}

namespace {

struct Msg {                       // one published send
    cudaIpcMemHandle_t mem;
    cudaIpcEventHandle_t ev;
    size_t bytes;
};

struct PendingRecv {
    void* buf;
    size_t bytes;
    int peer;
    long seq;
    cudaStream_t st;
};

struct Staged {
    void* buf;
    cudaEvent_t ev;
};

thread_local int g_group = 0;
thread_local std::vector<std::pair<ncclComm_t, PendingRecv>> g_pending;

size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        default: return 8;
    }
}

bool wait_file(const std::string& path, double timeout_s) {
    struct timespec t0, t;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    struct stat sb;
    while (stat(path.c_str(), &sb) != 0) {
        clock_gettime(CLOCK_MONOTONIC, &t);
        if ((t.tv_sec - t0.tv_sec) + 1e-9 * (t.tv_nsec - t0.tv_nsec) > timeout_s) return false;
        usleep(200);
    }
    return true;
}

}  // namespace

struct ncclComm {
    std::string dir;
    int rank, nranks;
    std::vector<long> send_seq, recv_seq;
    std::vector<Staged> staged;
};

namespace {

ncclResult_t do_recv(ncclComm_t c, const PendingRecv& r) {
    char name[512];
    snprintf(name, sizeof name, "%s/m_%d_%d_%ld", c->dir.c_str(), r.peer, c->rank, r.seq);
    if (!wait_file(name, 120.0)) return ncclSystemError;
    Msg m;
    FILE* f = fopen(name, "rb");
    if (!f) return ncclSystemError;
    const bool ok = fread(&m, sizeof m, 1, f) == 1;
    fclose(f);
    if (!ok || m.bytes != r.bytes) return ncclInvalidUsage;   // mismatched send / recv sizes
    if (r.bytes == 0) return ncclSuccess;
    void* src = nullptr;
    cudaEvent_t ev = nullptr;
    if (cudaIpcOpenMemHandle(&src, m.mem, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return ncclUnhandledCudaError;
    if (cudaIpcOpenEventHandle(&ev, m.ev) != cudaSuccess ||
        cudaStreamWaitEvent(r.st, ev, 0) != cudaSuccess ||
        cudaMemcpyAsync(r.buf, src, r.bytes, cudaMemcpyDeviceToDevice, r.st) != cudaSuccess ||
        cudaStreamSynchronize(r.st) != cudaSuccess)
        return ncclUnhandledCudaError;
    cudaEventDestroy(ev);
    cudaIpcCloseMemHandle(src);
    return ncclSuccess;
}

ncclResult_t flush() {
    ncclResult_t e = ncclSuccess;
    for (auto& p : g_pending)
        if (e == ncclSuccess) e = do_recv(p.first, p.second);
    g_pending.clear();
    return e;
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    if (!id) return ncclInvalidArgument;
    memset(id, 0, sizeof *id);
    char tmpl[] = "/tmp/fgf_nccl_shim_XXXXXX";
    if (!mkdtemp(tmpl)) return ncclSystemError;
    snprintf(id->internal, NCCL_UNIQUE_ID_BYTES, "%s", tmpl);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    ncclComm* c = new ncclComm;
    c->dir.assign(id.internal, strnlen(id.internal, NCCL_UNIQUE_ID_BYTES));
    mkdir(c->dir.c_str(), 0700);
    c->rank = rank;
    c->nranks = nranks;
    c->send_seq.assign(nranks, 0);
    c->recv_seq.assign(nranks, 0);
    *comm = c;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
    if (!c) return ncclInvalidArgument;
    char name[512];
    snprintf(name, sizeof name, "%s/d_%d", c->dir.c_str(), c->rank);
    if (FILE* f = fopen(name, "wb")) fclose(f);
    bool all = true;
    for (int k = 0; k < c->nranks; ++k) {
        snprintf(name, sizeof name, "%s/d_%d", c->dir.c_str(), k);
        all = wait_file(name, 120.0) && all;
    }
    for (auto& s : c->staged) {
        cudaEventDestroy(s.ev);
        cudaFree(s.buf);
    }
    delete c;
    return all ? ncclSuccess : ncclSystemError;
}

ncclResult_t ncclCommGetAsyncError(ncclComm_t c, ncclResult_t* err) {
    if (!c || !err) return ncclInvalidArgument;
    *err = ncclSuccess;
    return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
    ++g_group;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
    if (g_group < 1) return ncclInvalidUsage;
    return --g_group == 0 ? flush() : ncclSuccess;
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t c,
                      cudaStream_t st) {
    if (!c || peer < 0 || peer >= c->nranks || peer == c->rank) return ncclInvalidArgument;
    Msg m;
    memset(&m, 0, sizeof m);
    m.bytes = count * type_size(dt);
    if (m.bytes) {
        Staged s;
        if (cudaMalloc(&s.buf, m.bytes) != cudaSuccess) return ncclUnhandledCudaError;
        if (cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming | cudaEventInterprocess) != cudaSuccess)
            return ncclUnhandledCudaError;
        c->staged.push_back(s);
        if (cudaMemcpyAsync(s.buf, buf, m.bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
            cudaEventRecord(s.ev, st) != cudaSuccess ||
            cudaIpcGetMemHandle(&m.mem, s.buf) != cudaSuccess ||
            cudaIpcGetEventHandle(&m.ev, s.ev) != cudaSuccess)
            return ncclUnhandledCudaError;
    }
    char name[512], tmp[520];
    snprintf(name, sizeof name, "%s/m_%d_%d_%ld", c->dir.c_str(), c->rank, peer, c->send_seq[peer]++);
    snprintf(tmp, sizeof tmp, "%s.tmp", name);
    FILE* f = fopen(tmp, "wb");
    if (!f) return ncclSystemError;
    const bool ok = fwrite(&m, sizeof m, 1, f) == 1;
    fclose(f);
    if (!ok || rename(tmp, name) != 0) return ncclSystemError;
    return ncclSuccess;
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t c,
                      cudaStream_t st) {
    if (!c || peer < 0 || peer >= c->nranks || peer == c->rank) return ncclInvalidArgument;
    PendingRecv r{buf, count * type_size(dt), peer, c->recv_seq[peer]++, st};
    if (g_group > 0) {
        g_pending.emplace_back(c, r);
        return ncclSuccess;
    }
    return do_recv(c, r);
}

}  // extern "C"
