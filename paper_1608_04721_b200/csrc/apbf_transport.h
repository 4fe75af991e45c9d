// apbf_transport.h -- rank-to-rank transport of the z-slab decomposition.
//
// Two implementations of one small interface:
//  * LoopbackTransport: G ranks as host threads of one process (each with its
//    own device and stream; all on one GPU for tests, one GPU per thread for
//    single-process multi-GPU).  Collectives rendezvous on a host barrier;
//    bulk exchanges are device-to-device (peer) copies.  No kernel ever waits
//    on another kernel: the waiting is on the host.
//  * NcclTransport: one process per GPU; NCCL all-reduce and grouped
//    send/recv over NVLink.  libnccl is dlopen'ed (RTLD_NOLOAD first), so the
//    library shares the communicator runtime torch already loaded.
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace apbf_gpu {

enum class RType { I32, I64, U32, F64 };
enum class ROp { Sum, Min, Max };

inline size_t rtype_size(RType t) { return (t == RType::I64 || t == RType::F64) ? 8 : 4; }

struct Transport {
    virtual ~Transport() = default;
    virtual int rank() const = 0;
    virtual int size() const = 0;
    // In-place all-reduce of a device buffer, ordered on `st`: work enqueued on
    // `st` afterwards sees the result; the host must synchronise `st` before
    // reading it.
    virtual void allreduce(void* dev, size_t count, RType t, ROp op, cudaStream_t st) = 0;
    // Device all-to-all, ordered on `st` like allreduce: send[q] (sendBytes[q])
    // to rank q, recv[q] (recvBytes[q]) from rank q.  Entries for q == rank()
    // are ignored (the caller copies locally).
    virtual void alltoallv(const void* const* send, const size_t* sendBytes, void* const* recv,
                           const size_t* recvBytes, cudaStream_t st) = 0;
    // Host all-to-all of one int64 per destination, ordered on `st` (returns
    // once recv is filled: the solver stream is synchronised).
    virtual void alltoall_counts(const long long* send, long long* recv, cudaStream_t st) = 0;
    // True when allreduce/alltoallv only enqueue work on `st` (no host
    // synchronisation), so they can be recorded into a CUDA graph by stream
    // capture.
    virtual bool capturable() const { return false; }
};

template <class T>
inline void reduce_into(T* acc, const T* v, size_t n, ROp op) {
    for (size_t k = 0; k < n; ++k) {
        if (op == ROp::Sum) acc[k] += v[k];
        else if (op == ROp::Min) acc[k] = v[k] < acc[k] ? v[k] : acc[k];
        else acc[k] = v[k] > acc[k] ? v[k] : acc[k];
    }
}

// ------------------------------------------------------------- loopback

struct LoopbackHub {
    explicit LoopbackHub(int g, std::vector<int> devs) : G(g), devices(std::move(devs)), host(g),
        sendPtrs(g), sendBytes(g), counts(g, std::vector<long long>(g)) {}
    int G;
    std::vector<int> devices;
    std::vector<std::vector<unsigned char>> host;
    std::vector<std::vector<const void*>> sendPtrs;
    std::vector<std::vector<size_t>> sendBytes;
    std::vector<std::vector<long long>> counts;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long long generation = 0;
    bool poisoned = false;

    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        if (poisoned) throw std::runtime_error("slab peer rank failed");
        const long long gen = generation;
        if (++arrived == G) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen || poisoned; });
            if (poisoned) throw std::runtime_error("slab peer rank failed");
        }
    }
    void poison() {
        std::lock_guard<std::mutex> lk(m);
        poisoned = true;
        cv.notify_all();
    }
    void reset() {
        std::lock_guard<std::mutex> lk(m);
        poisoned = false;
        arrived = 0;
    }
};

struct LoopbackTransport final : Transport {
    LoopbackTransport(LoopbackHub* h, int r) : hub(h), r_(r) {}
    LoopbackHub* hub;
    int r_;
    int rank() const override { return r_; }
    int size() const override { return hub->G; }

    void allreduce(void* dev, size_t count, RType t, ROp op, cudaStream_t st) override {
        const size_t bytes = count * rtype_size(t);
        auto& mine = hub->host[r_];
        mine.resize(bytes);
        if (cudaMemcpyAsync(mine.data(), dev, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            throw std::runtime_error("loopback allreduce: device read failed");
        hub->barrier();
        // every rank reduces all contributions in rank order (deterministic)
        std::vector<unsigned char> acc(hub->host[0]);
        for (int q = 1; q < hub->G; ++q) {
            const void* v = hub->host[q].data();
            switch (t) {
                case RType::I32: reduce_into((int*)acc.data(), (const int*)v, count, op); break;
                case RType::U32: reduce_into((unsigned*)acc.data(), (const unsigned*)v, count, op); break;
                case RType::I64: reduce_into((long long*)acc.data(), (const long long*)v, count, op); break;
                case RType::F64: reduce_into((double*)acc.data(), (const double*)v, count, op); break;
            }
        }
        hub->barrier();  // nobody overwrites its staging before all have read
        if (cudaMemcpyAsync(dev, acc.data(), bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            throw std::runtime_error("loopback allreduce: device write failed");
    }

    void alltoallv(const void* const* send, const size_t* sendBytes, void* const* recv,
                   const size_t* recvBytes, cudaStream_t st) override {
        if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("loopback alltoallv: sync");
        hub->sendPtrs[r_].assign(send, send + hub->G);
        hub->sendBytes[r_].assign(sendBytes, sendBytes + hub->G);
        hub->barrier();
        for (int q = 0; q < hub->G; ++q) {
            if (q == r_ || recvBytes[q] == 0) continue;
            if (hub->sendBytes[q][r_] != recvBytes[q])
                throw std::runtime_error("loopback alltoallv: size mismatch");
            const cudaError_t e =
                hub->devices[q] == hub->devices[r_]
                    ? cudaMemcpyAsync(recv[q], hub->sendPtrs[q][r_], recvBytes[q], cudaMemcpyDeviceToDevice, st)
                    : cudaMemcpyPeerAsync(recv[q], hub->devices[r_], hub->sendPtrs[q][r_], hub->devices[q],
                                          recvBytes[q], st);
            if (e != cudaSuccess) throw std::runtime_error("loopback alltoallv: copy failed");
        }
        if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("loopback alltoallv: sync");
        hub->barrier();  // senders may reuse their buffers now
    }

    void alltoall_counts(const long long* send, long long* recv, cudaStream_t) override {
        hub->counts[r_].assign(send, send + hub->G);
        hub->barrier();
        for (int q = 0; q < hub->G; ++q) recv[q] = hub->counts[q][r_];
        hub->barrier();
    }
};

// ----------------------------------------------------------------- NCCL

struct NcclApi {
    typedef int (*GetUniqueId)(void*);
    typedef int (*CommInitRank)(void**, int, const void* /*by value in C; see call*/, int);
    void* lib = nullptr;
    int (*getUniqueId)(void*) = nullptr;
    void* commInitRankSym = nullptr;
    int (*commDestroy)(void*) = nullptr;
    int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*groupStart)() = nullptr;
    int (*groupEnd)() = nullptr;
    const char* (*getErrorString)(int) = nullptr;

    static NcclApi& get() {
        static NcclApi api;
        if (!api.lib) {
            const char* names[] = {"libnccl.so.2", "libnccl.so"};
            for (const char* nm : names) {
                api.lib = dlopen(nm, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
                if (api.lib) break;
            }
            for (const char* nm : names) {
                if (api.lib) break;
                api.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            }
            if (!api.lib) throw std::runtime_error("NCCL not found (libnccl.so.2)");
            api.getUniqueId = (int (*)(void*))dlsym(api.lib, "ncclGetUniqueId");
            api.commInitRankSym = dlsym(api.lib, "ncclCommInitRank");
            api.commDestroy = (int (*)(void*))dlsym(api.lib, "ncclCommDestroy");
            using AllReduceFn = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
            using SendFn = int (*)(const void*, size_t, int, int, void*, cudaStream_t);
            using RecvFn = int (*)(void*, size_t, int, int, void*, cudaStream_t);
            api.allReduce = (AllReduceFn)dlsym(api.lib, "ncclAllReduce");
            api.send = (SendFn)dlsym(api.lib, "ncclSend");
            api.recv = (RecvFn)dlsym(api.lib, "ncclRecv");
            api.groupStart = (int (*)())dlsym(api.lib, "ncclGroupStart");
            api.groupEnd = (int (*)())dlsym(api.lib, "ncclGroupEnd");
            api.getErrorString = (const char* (*)(int))dlsym(api.lib, "ncclGetErrorString");
            if (!api.getUniqueId || !api.commInitRankSym || !api.allReduce || !api.send || !api.recv)
                throw std::runtime_error("NCCL symbols missing");
        }
        return api;
    }
};

struct NcclUniqueIdT {
    char internal[128];
};

struct NcclTransport final : Transport {
    NcclTransport(int rank, int nranks, const unsigned char id[128]) : r_(rank), g_(nranks) {
        // The slab frame re-records its segments (with NCCL calls inside)
        // every substep with new sizes: no user-buffer registration per
        // recording (unless the user asks for it).
        setenv("NCCL_GRAPH_REGISTER", "0", 0);
        NcclApi& api = NcclApi::get();
        NcclUniqueIdT uid;
        std::memcpy(uid.internal, id, 128);
        auto init = (int (*)(void**, int, NcclUniqueIdT, int))api.commInitRankSym;
        const int rc = init(&comm, nranks, uid, rank);
        if (rc != 0) throw std::runtime_error(std::string("ncclCommInitRank: ") + api.getErrorString(rc));
        if (cudaMalloc(&scratch, 64 * 8) != cudaSuccess) throw std::runtime_error("nccl scratch");
    }
    ~NcclTransport() override {
        if (comm) NcclApi::get().commDestroy(comm);
        if (scratch) cudaFree(scratch);
    }
    int r_, g_;
    void* comm = nullptr;
    void* scratch = nullptr;
    int rank() const override { return r_; }
    int size() const override { return g_; }
    bool capturable() const override { return true; }  // NCCL supports stream capture

    static int nccl_type(RType t) {  // ncclInt32 2, ncclUint32 3, ncclInt64 4, ncclFloat64 8
        return t == RType::I32 ? 2 : t == RType::U32 ? 3 : t == RType::I64 ? 4 : 8;
    }
    static int nccl_op(ROp o) { return o == ROp::Sum ? 0 : o == ROp::Max ? 2 : 3; }
    void check(int rc, const char* what) {
        if (rc != 0) throw std::runtime_error(std::string(what) + ": " + NcclApi::get().getErrorString(rc));
    }
    // Both stream-ordered: no host synchronisation (NCCL runs on `st`).
    void allreduce(void* dev, size_t count, RType t, ROp op, cudaStream_t st) override {
        check(NcclApi::get().allReduce(dev, dev, count, nccl_type(t), nccl_op(op), comm, st), "ncclAllReduce");
    }
    void alltoallv(const void* const* send, const size_t* sendBytes, void* const* recv,
                   const size_t* recvBytes, cudaStream_t st) override {
        bool any = false;
        for (int q = 0; q < g_; ++q) any = any || (q != r_ && (sendBytes[q] || recvBytes[q]));
        if (!any) return;  // nothing to exchange (e.g. one rank): no NCCL group
        NcclApi& api = NcclApi::get();
        check(api.groupStart(), "ncclGroupStart");
        for (int q = 0; q < g_; ++q) {
            if (q == r_) continue;
            if (sendBytes[q]) check(api.send(send[q], sendBytes[q], 0, q, comm, st), "ncclSend");
            if (recvBytes[q]) check(api.recv(recv[q], recvBytes[q], 0, q, comm, st), "ncclRecv");
        }
        check(api.groupEnd(), "ncclGroupEnd");
    }
    void alltoall_counts(const long long* send, long long* recv, cudaStream_t st) override {
        // scratch layout: [0, g) send, [g, 2g) recv; all on the solver stream
        long long* d = (long long*)scratch;
        cuda_check(cudaMemcpyAsync(d, send, sizeof(long long) * g_, cudaMemcpyHostToDevice, st), "counts upload");
        NcclApi& api = NcclApi::get();
        check(api.groupStart(), "ncclGroupStart");
        for (int q = 0; q < g_; ++q) {
            if (q == r_) continue;
            check(api.send(d + q, 8, 0, q, comm, st), "ncclSend");
            check(api.recv(d + g_ + q, 8, 0, q, comm, st), "ncclRecv");
        }
        check(api.groupEnd(), "ncclGroupEnd");
        cuda_check(cudaMemcpyAsync(recv, d + g_, sizeof(long long) * g_, cudaMemcpyDeviceToHost, st),
                   "counts download");
        cuda_check(cudaStreamSynchronize(st), "counts exchange");
        recv[r_] = send[r_];
    }
    static void cuda_check(cudaError_t e, const char* what) {
        if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
    }
};

// Equal-count partition of the global per-layer histogram into G slabs of
// whole layers: zlo[g] .. zhi[g] (exclusive), every slab at least minLayers
// thick.  Returns false when the grid has too few layers.  Pure host logic,
// identical on every rank (same histogram in, same slabs out).
// (__host__ __device__: the slab frame runs it on the device, k_slab_partition,
// and the host entry point apbf_slab_partition is the same code.)
template <class H>
__host__ __device__ inline bool slab_partition(const H* hist, int dz, int G, int minLayers, int* zlo, int* zhi) {
    if (dz < G * minLayers) return false;
    long long total = 0;
    for (int z = 0; z < dz; ++z) total += hist[z];
    int z = 0;
    long long acc = 0;
    for (int g = 0; g < G; ++g) {
        zlo[g] = z;
        if (g == G - 1) {
            zhi[g] = dz;
            break;
        }
        // cut where the prefix first reaches (g+1)/G of the particles,
        // keeping >= minLayers for this and every later slab
        const long long target = (total * (g + 1) + G - 1) / G;
        int end = z + minLayers;
        acc = 0;
        for (int k = 0; k < end; ++k) acc += hist[k];
        while (end < dz - (G - 1 - g) * minLayers && acc < target) acc += hist[end++];
        zhi[g] = end;
        z = end;
    }
    return true;
}

}  // namespace apbf_gpu
