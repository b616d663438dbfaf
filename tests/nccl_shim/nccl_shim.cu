// Test NCCL: G ranks as G host threads of ONE process on ONE GPU (test infrastructure).
//
// libiabn.so loads NCCL with dlopen (IABN_NCCL_LIB overrides the path, iabn.cu); this
// library implements the subset it calls -- ncclGetUniqueId, ncclCommInitRank,
// ncclAllReduce (sum of float64 / float32), ncclAllGather, ncclCommDestroy,
// ncclGetErrorString -- with the semantics of the real collectives, so that the
// reduce / all-reduce / apply path of iabn_forward_sync / iabn_backward_sync
// runs with nranks >= 2 on a one-GPU lease.
//
// Every collective is a host rendezvous of the G threads plus stream-ordered device
// work: each rank records an event after its pending work and publishes its buffer;
// after a barrier every rank's stream waits for all the others' events, a kernel sums
// the G inputs in rank order into a private scratch buffer (bit-identical on every
// rank), a second barrier + event wait guarantees that no rank overwrites its buffer
// while another still reads it, and the scratch is copied to recvbuff.  No kernel ever
// waits on another rank's kernel (only stream-event waits), so nothing depends on two
// kernels being co-resident (B200_PROFILING.md: ranks that spin on each other must not
// share a GPU as separate launches).
//
// Shares nothing with the library under test beyond the public nccl.h types.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#define SHIM_API extern "C" __attribute__((visibility("default")))

namespace {

struct Group {
    int nranks = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    int members = 0;
    // per-rank published state of the current collective
    std::vector<const void*> src;
    std::vector<cudaEvent_t> ev_in, ev_mid;

    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

std::mutex g_reg_mu;
std::map<std::string, Group*> g_reg;
std::atomic<uint64_t> g_allreduce_calls{0}, g_allgather_calls{0};

}  // namespace

struct ncclComm {
    Group* grp;
    int rank;
    int device;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
};

namespace {

template <typename T>
__global__ void sum_ranks(const T* const* src, int nranks, size_t count, T* out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x) {
        T s = src[0][i];
        for (int r = 1; r < nranks; ++r) s += src[r][i];  // rank order: same bits on every rank
        out[i] = s;
    }
}

size_t type_bytes(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: case ncclBfloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
        default: return 0;
    }
}

bool ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fprintf(stderr, "nccl_shim: %s: %s\n", what, cudaGetErrorString(e));
    return e == cudaSuccess;
}

ncclResult_t ensure_scratch(ncclComm* c, size_t bytes) {
    if (c->scratch_bytes >= bytes) return ncclSuccess;
    if (c->scratch) cudaFree(c->scratch);
    c->scratch = nullptr;
    // pointer table (nranks entries) + payload
    const size_t want = bytes + 256;
    if (!ok(cudaMalloc(&c->scratch, want), "cudaMalloc")) return ncclUnhandledCudaError;
    c->scratch_bytes = want - 256;
    return ncclSuccess;
}

// phase 1: publish this rank's input and its readiness event, wait for all ranks
ncclResult_t enter(ncclComm* c, const void* src, cudaStream_t st) {
    Group* g = c->grp;
    g->src[c->rank] = src;
    if (!ok(cudaEventRecord(g->ev_in[c->rank], st), "cudaEventRecord")) return ncclUnhandledCudaError;
    g->barrier();
    for (int r = 0; r < g->nranks; ++r)
        if (r != c->rank && !ok(cudaStreamWaitEvent(st, g->ev_in[r], 0), "cudaStreamWaitEvent"))
            return ncclUnhandledCudaError;
    return ncclSuccess;
}

// phase 2: every rank finished reading the others' inputs before anyone writes its output
ncclResult_t leave(ncclComm* c, cudaStream_t st) {
    Group* g = c->grp;
    if (!ok(cudaEventRecord(g->ev_mid[c->rank], st), "cudaEventRecord")) return ncclUnhandledCudaError;
    g->barrier();
    for (int r = 0; r < g->nranks; ++r)
        if (r != c->rank && !ok(cudaStreamWaitEvent(st, g->ev_mid[r], 0), "cudaStreamWaitEvent"))
            return ncclUnhandledCudaError;
    g->barrier();  // nobody re-records ev_in / ev_mid before every rank has enqueued its waits
    return ncclSuccess;
}

}  // namespace

SHIM_API const char* ncclGetErrorString(ncclResult_t r) {
    switch (r) {
        case ncclSuccess: return "no error (shim)";
        case ncclUnhandledCudaError: return "unhandled cuda error (shim)";
        case ncclInvalidArgument: return "invalid argument (shim)";
        case ncclInvalidUsage: return "invalid usage (shim)";
        default: return "error (shim)";
    }
}

SHIM_API ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    if (!id) return ncclInvalidArgument;
    static std::mutex mu;
    static std::mt19937_64 rng{std::random_device{}()};
    std::lock_guard<std::mutex> lk(mu);
    memset(id->internal, 0, sizeof(id->internal));
    memcpy(id->internal, "iabn-nccl-shim", 14);
    for (int i = 16; i + 8 <= (int)sizeof(id->internal); i += 8) {
        const uint64_t v = rng();
        memcpy(id->internal + i, &v, 8);
    }
    return ncclSuccess;
}

SHIM_API ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
    if (!out || nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    const std::string key(id.internal, sizeof(id.internal));
    Group* g;
    {
        std::lock_guard<std::mutex> lk(g_reg_mu);
        auto it = g_reg.find(key);
        if (it == g_reg.end()) {
            g = new Group;
            g->nranks = nranks;
            g->src.assign(nranks, nullptr);
            g->ev_in.assign(nranks, nullptr);
            g->ev_mid.assign(nranks, nullptr);
            g_reg[key] = g;
        } else {
            g = it->second;
            if (g->nranks != nranks) return ncclInvalidUsage;
        }
        if (g->ev_in[rank]) return ncclInvalidUsage;  // rank initialised twice
        if (!ok(cudaEventCreateWithFlags(&g->ev_in[rank], cudaEventDisableTiming), "event") ||
            !ok(cudaEventCreateWithFlags(&g->ev_mid[rank], cudaEventDisableTiming), "event"))
            return ncclUnhandledCudaError;
        ++g->members;
    }
    auto* c = new ncclComm{g, rank, 0};
    cudaGetDevice(&c->device);
    g->barrier();  // like ncclCommInitRank: returns once every rank has joined
    *out = c;
    return ncclSuccess;
}

SHIM_API ncclResult_t ncclCommDestroy(ncclComm_t c) {
    if (!c) return ncclSuccess;
    cudaDeviceSynchronize();
    if (c->scratch) cudaFree(c->scratch);
    Group* g = c->grp;
    {
        std::lock_guard<std::mutex> lk(g_reg_mu);
        cudaEventDestroy(g->ev_in[c->rank]);
        cudaEventDestroy(g->ev_mid[c->rank]);
        g->ev_in[c->rank] = g->ev_mid[c->rank] = nullptr;
        if (--g->members == 0) {
            for (auto it = g_reg.begin(); it != g_reg.end(); ++it)
                if (it->second == g) {
                    g_reg.erase(it);
                    break;
                }
            delete g;
        }
    }
    delete c;
    return ncclSuccess;
}

SHIM_API ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count,
                                    ncclDataType_t dt, ncclRedOp_t op, ncclComm_t c,
                                    cudaStream_t st) {
    if (!c || op != ncclSum || (dt != ncclFloat64 && dt != ncclFloat32)) return ncclInvalidArgument;
    const size_t bytes = count * type_bytes(dt);
    Group* g = c->grp;
    ncclResult_t r = ensure_scratch(c, bytes);
    if (r != ncclSuccess) return r;
    if ((r = enter(c, send, st)) != ncclSuccess) return r;
    // the rank-ordered pointer table, then the sum into this rank's scratch
    const void** table = (const void**)c->scratch;
    void* out = (char*)c->scratch + 256;
    if (!ok(cudaMemcpyAsync(table, g->src.data(), sizeof(void*) * g->nranks, cudaMemcpyHostToDevice, st),
            "table copy"))
        return ncclUnhandledCudaError;
    // the pageable H2D copy above is staged before it returns, so g->src may change after it
    if (count) {
        const unsigned blocks = (unsigned)std::min<size_t>((count + 255) / 256, 1184);
        if (dt == ncclFloat64)
            sum_ranks<double><<<blocks, 256, 0, st>>>((const double* const*)table, g->nranks, count,
                                                     (double*)out);
        else
            sum_ranks<float><<<blocks, 256, 0, st>>>((const float* const*)table, g->nranks, count,
                                                    (float*)out);
        if (!ok(cudaGetLastError(), "sum kernel")) return ncclUnhandledCudaError;
    }
    if ((r = leave(c, st)) != ncclSuccess) return r;
    if (count && !ok(cudaMemcpyAsync(recv, out, bytes, cudaMemcpyDeviceToDevice, st), "result copy"))
        return ncclUnhandledCudaError;
    g_allreduce_calls.fetch_add(1);
    return ncclSuccess;
}

SHIM_API ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t dt,
                                    ncclComm_t c, cudaStream_t st) {
    if (!c || !type_bytes(dt)) return ncclInvalidArgument;
    const size_t bytes = count * type_bytes(dt);
    Group* g = c->grp;
    ncclResult_t r = ensure_scratch(c, bytes * g->nranks);
    if (r != ncclSuccess) return r;
    if ((r = enter(c, send, st)) != ncclSuccess) return r;
    char* out = (char*)c->scratch + 256;
    for (int k = 0; k < g->nranks; ++k)
        if (bytes && !ok(cudaMemcpyAsync(out + k * bytes, g->src[k], bytes, cudaMemcpyDeviceToDevice, st),
                         "gather copy"))
            return ncclUnhandledCudaError;
    if ((r = leave(c, st)) != ncclSuccess) return r;
    if (bytes && !ok(cudaMemcpyAsync(recv, out, bytes * g->nranks, cudaMemcpyDeviceToDevice, st),
                     "result copy"))
        return ncclUnhandledCudaError;
    g_allgather_calls.fetch_add(1);
    return ncclSuccess;
}

// test hooks: how many collectives completed (proves the exchange step really ran)
SHIM_API uint64_t shim_allreduce_calls(void) { return g_allreduce_calls.load(); }
SHIM_API uint64_t shim_allgather_calls(void) { return g_allgather_calls.load(); }
