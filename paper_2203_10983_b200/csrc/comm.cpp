// comm.cpp -- transports for the exchange steps of Algorithm 1:
//   a5  forward halo exchange  (l.9 "Send H_{S_{i,j}} ... Receive H_{U_i}")
//   a11 backward exchange       (boundary-node gradients back to their owners)
//   a13 AllReduce of the weight gradients (l.13)
//
// NCCL: one process per GPU; the all-to-allv is a grouped ncclSend/ncclRecv straight into the halo rows of the
// stacked feature buffer (no staging on the receive side); the weight-gradient sum is one ncclAllReduce.
// LOCAL: several contexts in one process (one host thread each); every rank PULLS the rows addressed to it with
// device-to-device copies after a host barrier, ordered by CUDA events.  The sum is taken in rank order.
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>

#include <nccl.h>

#include "common.h"
#include "kernels.h"
#include "transport.h"

struct bns_group {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<const void*> src;
    std::vector<std::vector<int64_t>> src_off;
    std::vector<cudaEvent_t> ev_ready, ev_done;
    std::vector<int64_t> ival;
    std::vector<float*> fbuf;
    std::vector<double*> dbuf;
    std::vector<int> attached;
};

namespace bns {

namespace {

void group_barrier(bns_group* g) {
    std::unique_lock<std::mutex> lk(g->mu);
    const uint64_t my = g->gen;
    if (++g->arrived == g->world) {
        g->arrived = 0;
        g->gen++;
        g->cv.notify_all();
        return;
    }
    if (!g->cv.wait_for(lk, std::chrono::seconds(300), [&] { return g->gen != my; }))
        throw Error(BNS_ERR_RUNTIME, "local transport: barrier timeout (a rank did not reach the collective)");
}

#define BNS_NCCL(x)                                                                                         \
    do {                                                                                                    \
        ncclResult_t r__ = (x);                                                                             \
        if (r__ != ncclSuccess)                                                                             \
            throw ::bns::Error(BNS_ERR_RUNTIME, std::string(#x) + ": " + ncclGetErrorString(r__));          \
    } while (0)

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    int64_t* d_i64 = nullptr;
    NcclTransport(Ctx& c, const uint8_t* id) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        BNS_NCCL(ncclCommInitRank(&comm, c.cfg.world, uid, c.cfg.rank));
        BNS_CUDA(cudaMalloc(&d_i64, 64));
    }
    ~NcclTransport() override {
        if (d_i64) cudaFree(d_i64);
        if (comm) ncclCommDestroy(comm);
    }
    void exchange(Ctx& c, const void* src, const int64_t* src_off, void* dst, const int64_t* dst_off,
                  size_t rowbytes) override {
        const int m = c.cfg.world, me = c.cfg.rank;
        BNS_NCCL(ncclGroupStart());
        for (int j = 0; j < m; ++j) {
            if (j == me) continue;
            const int64_t ns = src_off[j + 1] - src_off[j], nr = dst_off[j + 1] - dst_off[j];
            if (ns > 0)
                BNS_NCCL(ncclSend(static_cast<const char*>(src) + src_off[j] * rowbytes, ns * rowbytes, ncclUint8, j,
                                  comm, c.stream));
            if (nr > 0)
                BNS_NCCL(ncclRecv(static_cast<char*>(dst) + dst_off[j] * rowbytes, nr * rowbytes, ncclUint8, j, comm,
                                  c.stream));
        }
        BNS_NCCL(ncclGroupEnd());
    }
    void allreduce(Ctx& c, float* buf, int64_t n, double* scal, int64_t ns) override {
        BNS_NCCL(ncclGroupStart());
        BNS_NCCL(ncclAllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, comm, c.stream));
        BNS_NCCL(ncclAllReduce(scal, scal, (size_t)ns, ncclFloat64, ncclSum, comm, c.stream));
        BNS_NCCL(ncclGroupEnd());
    }
    int64_t allreduce_host_i64(Ctx& c, int64_t v) override {
        BNS_CUDA(cudaMemcpyAsync(d_i64, &v, sizeof(v), cudaMemcpyHostToDevice, c.stream));
        BNS_NCCL(ncclAllReduce(d_i64, d_i64, 1, ncclInt64, ncclSum, comm, c.stream));
        BNS_CUDA(cudaMemcpyAsync(&v, d_i64, sizeof(v), cudaMemcpyDeviceToHost, c.stream));
        BNS_CUDA(cudaStreamSynchronize(c.stream));
        return v;
    }
    void poll(Ctx&) override {
        ncclResult_t st;
        if (ncclCommGetAsyncError(comm, &st) == ncclSuccess && st != ncclSuccess && st != ncclInProgress)
            throw Error(BNS_ERR_RUNTIME, std::string("NCCL async error: ") + ncclGetErrorString(st));
    }
};

struct LocalTransport : Transport {
    bns_group* g;
    int me;
    float* d_fout = nullptr;
    double* d_dout = nullptr;
    const float** d_fptrs = nullptr;
    const double** d_dptrs = nullptr;
    int64_t fcap = 0, dcap = 0;
    LocalTransport(Ctx& c, bns_group* grp) : g(grp), me(c.cfg.rank) {
        if (g->world != c.cfg.world) throw Error(BNS_ERR_INVALID, "local group size != cfg.world");
        {
            std::lock_guard<std::mutex> lk(g->mu);
            if (g->attached[me]) throw Error(BNS_ERR_INVALID, "local group: rank attached twice");
            g->attached[me] = 1;
        }
        BNS_CUDA(cudaEventCreateWithFlags(&g->ev_ready[me], cudaEventDisableTiming));
        BNS_CUDA(cudaEventCreateWithFlags(&g->ev_done[me], cudaEventDisableTiming));
    }
    ~LocalTransport() override {
        if (d_fout) cudaFree(d_fout);
        if (d_dout) cudaFree(d_dout);
        if (d_fptrs) cudaFree(d_fptrs);
        if (d_dptrs) cudaFree(d_dptrs);
        std::lock_guard<std::mutex> lk(g->mu);
        if (g->ev_ready[me]) cudaEventDestroy(g->ev_ready[me]);
        if (g->ev_done[me]) cudaEventDestroy(g->ev_done[me]);
        g->ev_ready[me] = g->ev_done[me] = nullptr;
        g->attached[me] = 0;
    }
    void wait_all(Ctx& c, std::vector<cudaEvent_t>& ev) {
        for (int j = 0; j < g->world; ++j)
            if (j != me) BNS_CUDA(cudaStreamWaitEvent(c.stream, ev[j], 0));
    }
    void exchange(Ctx& c, const void* src, const int64_t* src_off, void* dst, const int64_t* dst_off,
                  size_t rowbytes) override {
        const int m = g->world;
        g->src[me] = src;
        g->src_off[me].assign(src_off, src_off + m + 1);
        BNS_CUDA(cudaEventRecord(g->ev_ready[me], c.stream));
        group_barrier(g);
        for (int j = 0; j < m; ++j) {
            if (j == me) continue;
            const int64_t n = g->src_off[j][me + 1] - g->src_off[j][me];
            if (n != dst_off[j + 1] - dst_off[j])
                throw Error(BNS_ERR_RUNTIME, "local transport: row count mismatch between ranks " +
                                                 std::to_string(j) + " -> " + std::to_string(me));
            if (n == 0) continue;
            BNS_CUDA(cudaStreamWaitEvent(c.stream, g->ev_ready[j], 0));
            BNS_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + dst_off[j] * rowbytes,
                                     static_cast<const char*>(g->src[j]) + g->src_off[j][me] * rowbytes, n * rowbytes,
                                     cudaMemcpyDeviceToDevice, c.stream));
        }
        BNS_CUDA(cudaEventRecord(g->ev_done[me], c.stream));
        group_barrier(g);
        wait_all(c, g->ev_done);   // peers have finished reading my rows
    }
    void allreduce(Ctx& c, float* buf, int64_t n, double* scal, int64_t ns) override {
        const int m = g->world;
        if (n > fcap) {
            if (d_fout) cudaFree(d_fout);
            BNS_CUDA(cudaMalloc(&d_fout, n * sizeof(float)));
            fcap = n;
        }
        if (ns > dcap) {
            if (d_dout) cudaFree(d_dout);
            BNS_CUDA(cudaMalloc(&d_dout, ns * sizeof(double)));
            dcap = ns;
        }
        if (!d_fptrs) {
            BNS_CUDA(cudaMalloc(&d_fptrs, m * sizeof(float*)));
            BNS_CUDA(cudaMalloc(&d_dptrs, m * sizeof(double*)));
        }
        g->fbuf[me] = buf;
        g->dbuf[me] = scal;
        BNS_CUDA(cudaEventRecord(g->ev_ready[me], c.stream));
        group_barrier(g);
        std::vector<const float*> fp(g->fbuf.begin(), g->fbuf.end());
        std::vector<const double*> dp(g->dbuf.begin(), g->dbuf.end());
        BNS_CUDA(cudaMemcpy(d_fptrs, fp.data(), m * sizeof(float*), cudaMemcpyHostToDevice));
        BNS_CUDA(cudaMemcpy(d_dptrs, dp.data(), m * sizeof(double*), cudaMemcpyHostToDevice));
        wait_all(c, g->ev_ready);
        launch_sum_ptrs(c, d_fptrs, m, d_fout, n);
        launch_sum_ptrs_d(c, d_dptrs, m, d_dout, ns);
        BNS_CUDA(cudaEventRecord(g->ev_done[me], c.stream));
        group_barrier(g);
        wait_all(c, g->ev_done);
        BNS_CUDA(cudaMemcpyAsync(buf, d_fout, n * sizeof(float), cudaMemcpyDeviceToDevice, c.stream));
        BNS_CUDA(cudaMemcpyAsync(scal, d_dout, ns * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    }
    int64_t allreduce_host_i64(Ctx&, int64_t v) override {
        g->ival[me] = v;
        group_barrier(g);
        int64_t s = 0;
        for (int j = 0; j < g->world; ++j) s += g->ival[j];
        group_barrier(g);
        return s;
    }
    void poll(Ctx&) override {}
};

// Timing emulation of one rank of an m-rank job on a single GPU: every call is a no-op (no rows move, no sum is
// taken), so the rank runs exactly its own kernels with its own sampled sizes.  Results are NOT the method's.
struct NullTransport : Transport {
    void exchange(Ctx&, const void*, const int64_t*, void*, const int64_t*, size_t) override {}
    void allreduce(Ctx&, float*, int64_t, double*, int64_t) override {}
    int64_t allreduce_host_i64(Ctx&, int64_t v) override { return v; }
    void poll(Ctx&) override {}
};

}  // namespace

Transport* make_transport(Ctx& c) {
    switch (c.cfg.transport) {
        case BNS_TRANSPORT_NULL_EMULATE:
            return new NullTransport();
        case BNS_TRANSPORT_NCCL:
            if (!c.cfg.nccl_id) throw Error(BNS_ERR_INVALID, "transport NCCL needs cfg.nccl_id");
            return new NcclTransport(c, c.cfg.nccl_id);
        case BNS_TRANSPORT_LOCAL:
            if (!c.cfg.group) throw Error(BNS_ERR_INVALID, "transport LOCAL needs cfg.group");
            return new LocalTransport(c, c.cfg.group);
        default:
            return nullptr;
    }
}

}  // namespace bns

extern "C" {

bns_status bns_get_unique_id(uint8_t* out) {
    if (!out) return BNS_ERR_INVALID;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return BNS_ERR_RUNTIME;
    std::memcpy(out, &id, sizeof(id));
    return BNS_OK;
}

bns_status bns_group_create(int32_t world, bns_group** out) {
    if (!out || world < 1) return BNS_ERR_INVALID;
    bns_group* g = new bns_group();
    g->world = world;
    g->src.assign(world, nullptr);
    g->src_off.assign(world, {});
    g->ev_ready.assign(world, nullptr);
    g->ev_done.assign(world, nullptr);
    g->ival.assign(world, 0);
    g->fbuf.assign(world, nullptr);
    g->dbuf.assign(world, nullptr);
    g->attached.assign(world, 0);
    *out = g;
    return BNS_OK;
}

void bns_group_destroy(bns_group* g) { delete g; }

}  // extern "C"
