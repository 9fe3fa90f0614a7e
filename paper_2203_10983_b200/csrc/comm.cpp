// comm.cpp -- transports for the exchange steps of Algorithm 1:
//   a5  forward halo exchange  (l.9 "Send H_{S_{i,j}} ... Receive H_{U_i}")
//   a11 backward exchange       (boundary-node gradients back to their owners)
//   a13 AllReduce of the weight gradients (l.13)
//
// NCCL: one process per GPU; the all-to-allv is a grouped ncclSend/ncclRecv straight into the halo rows of the
// stacked feature buffer (no staging on the receive side); the weight-gradient sum is one ncclAllReduce.
// LOCAL: several contexts in one process (one host thread each); every rank PULLS the rows addressed to it with
// device-to-device copies after a host barrier, ordered by CUDA events.  The sum is taken in rank order.
// PEER (LOCAL + BNS_PEER_MEMORY, or IPC): the exchanges are fused into gather kernels that read the
// other ranks' buffers directly (peer.cu), ordered by device flag barriers; buffer pointers are shared at setup
// (in-process: raw pointers through the group; IPC: cudaIpcMemHandle_t through the caller's host all-gather).
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>

#include <cuda.h>
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
    std::vector<const void*> blob;   // host all-gather staging (peer-memory transport in-process)
    std::vector<void*> deferred;     // peer arenas of detached in-process members, freed by the last one out
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

// In-process transports hand the other contexts' raw device pointers to kernels (k_sum_ptrs, k_halo_pull,
// k_scatter_peer, k_peer_barrier): contexts on different devices need peer access, which is enabled here for every
// device of the group; a group whose devices cannot reach each other is refused.
void enable_peer_access(const Ctx& c, const std::vector<int64_t>& devs) {
    for (int64_t d64 : devs) {
        const int d = (int)d64;
        if (d == c.cfg.device) continue;
        int ok = 0;
        BNS_CUDA(cudaDeviceCanAccessPeer(&ok, c.cfg.device, d));
        if (!ok)
            throw Error(BNS_ERR_INVALID, "local group: device " + std::to_string(c.cfg.device) +
                                             " has no peer access to device " + std::to_string(d));
        const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) throw Error(BNS_ERR_RUNTIME, std::string("cudaDeviceEnablePeerAccess: ") +
                                                                  cudaGetErrorString(e));
    }
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
        pdl_hold();
    }
    void allreduce(Ctx& c, float* buf, int64_t n, double* scal, int64_t ns) override {
        BNS_NCCL(ncclGroupStart());
        BNS_NCCL(ncclAllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, comm, c.stream));
        BNS_NCCL(ncclAllReduce(scal, scal, (size_t)ns, ncclFloat64, ncclSum, comm, c.stream));
        BNS_NCCL(ncclGroupEnd());
        pdl_hold();
    }
    int64_t allreduce_host_i64(Ctx& c, int64_t v) override {
        BNS_CUDA_HOLD(cudaMemcpyAsync(d_i64, &v, sizeof(v), cudaMemcpyHostToDevice, c.stream));
        BNS_NCCL(ncclAllReduce(d_i64, d_i64, 1, ncclInt64, ncclSum, comm, c.stream));
        pdl_hold();
        BNS_CUDA_HOLD(cudaMemcpyAsync(&v, d_i64, sizeof(v), cudaMemcpyDeviceToHost, c.stream));
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
        g->ival[me] = c.cfg.device;
        group_barrier(g);
        std::vector<int64_t> devs(g->ival.begin(), g->ival.end());
        group_barrier(g);
        enable_peer_access(c, devs);
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
            if (j != me) BNS_CUDA_HOLD(cudaStreamWaitEvent(c.stream, ev[j], 0));
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
            BNS_CUDA_HOLD(cudaStreamWaitEvent(c.stream, g->ev_ready[j], 0));
            BNS_CUDA_HOLD(cudaMemcpyAsync(static_cast<char*>(dst) + dst_off[j] * rowbytes,
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
        pdl_hold();   // both sums read the peers' buffers
        launch_sum_ptrs_d(c, d_dptrs, m, d_dout, ns);
        BNS_CUDA(cudaEventRecord(g->ev_done[me], c.stream));
        group_barrier(g);
        wait_all(c, g->ev_done);
        BNS_CUDA_HOLD(cudaMemcpyAsync(buf, d_fout, n * sizeof(float), cudaMemcpyDeviceToDevice, c.stream));
        BNS_CUDA_HOLD(cudaMemcpyAsync(scal, d_dout, ns * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
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

void* driver_entry(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    BNS_CUDA(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw Error(BNS_ERR_RUNTIME, std::string(name) + " unavailable");
    return p;
}

// ---------------------------------------------------------------------------------------------
// Peer-memory transport (f1).  Shared buffers per rank, in table order (kind k, rank j) -> d_tab[k m + j]:
//   H^(0..L-1), dX (two alternating buffers), partial weight gradients (two, by all-reduce parity), loss scalars
//   (two), compaction segment offsets, barrier flags, send buffer (setup-time / debug generic exchange only)
// ---------------------------------------------------------------------------------------------
struct PeerTransport : Transport {
    bns_group* g = nullptr;                      // in-process group (LOCAL), else null
    bns_allgather_fn ag = nullptr;               // IPC host all-gather
    void* ag_user = nullptr;
    int m, me, L;
    enum { K_DX = 0, K_G = 2, K_S = 4, K_SEG = 6, K_FLAGS = 7, K_SEND = 8, K_H = 9 };
    int nk;
    std::vector<void*> own;                      // my buffers in kind order
    std::vector<void*> opened;                   // IPC mappings to close
    void** d_tab = nullptr;                      // nk x m device table
    int64_t* d_pnin = nullptr;                   // n_in of every rank
    int64_t* d_delta = nullptr;                  // row offset of my rows in each peer's halo gradient
    int32_t* d_owner_of_b = nullptr;             // owner rank of every boundary node
    int32_t* d_row_of_b = nullptr;               // ... and its row in the owner's H
    uint64_t* d_flags = nullptr;
    void *dx2 = nullptr, *g2 = nullptr, *s2 = nullptr;
    int* h_err = nullptr;                        // mapped pinned: barrier timeout flag
    int* d_err = nullptr;
    uint64_t bar = 0, ar_count = 0;
    bool first = true;

    PeerTransport(Ctx& c, bns_group* grp, bns_allgather_fn fn, void* user)
        : g(grp), ag(fn), ag_user(user), m(c.cfg.world), me(c.cfg.rank), L(c.L) {
        if (m > 32) throw Error(BNS_ERR_INVALID, "peer-memory transport: world <= 32");
        if (g) {
            if (g->world != m) throw Error(BNS_ERR_INVALID, "local group size != cfg.world");
            std::lock_guard<std::mutex> lk(g->mu);
            if (g->attached[me]) throw Error(BNS_ERR_INVALID, "local group: rank attached twice");
            g->attached[me] = 1;
        }
        preload_module_functions();
        const Plan& P = c.plan;
        if (!c.arena) throw Error(BNS_ERR_RUNTIME, "peer-memory transport without a peer arena");
        dx2 = c.d_dx2;
        g2 = c.d_gflat2;
        s2 = c.d_scal2;
        d_flags = c.d_pflags;
        BNS_CUDA(cudaMalloc(&d_delta, 32 * sizeof(int64_t)));
        BNS_CUDA(cudaMemset(d_delta, 0, 32 * sizeof(int64_t)));
        BNS_CUDA(cudaHostAlloc(&h_err, sizeof(int), cudaHostAllocMapped));
        *h_err = 0;
        BNS_CUDA(cudaHostGetDevicePointer((void**)&d_err, h_err, 0));
        c.d_abort = d_err;
        if (g) {
            std::vector<int64_t> devs(m);
            const int64_t dev = c.cfg.device;
            allgather(c, &dev, devs.data(), sizeof(int64_t));
            enable_peer_access(c, devs);
        }
        std::vector<int32_t> owner(P.n_bd + 1, 0);
        for (int j = 0; j < m; ++j)
            for (int64_t b = P.B_off[j]; b < P.B_off[j + 1]; ++b) owner[b] = j;
        std::vector<int32_t> row(P.B_row);
        row.push_back(0);
        BNS_CUDA(cudaMalloc(&d_owner_of_b, owner.size() * 4));
        BNS_CUDA(cudaMalloc(&d_row_of_b, row.size() * 4));
        BNS_CUDA(cudaMemcpy(d_owner_of_b, owner.data(), owner.size() * 4, cudaMemcpyHostToDevice));
        BNS_CUDA(cudaMemcpy(d_row_of_b, row.data(), row.size() * 4, cudaMemcpyHostToDevice));

        nk = K_H + L;
        own.assign(nk, nullptr);
        own[K_DX] = c.d_dx;      own[K_DX + 1] = dx2;
        own[K_G] = c.d_gflat;    own[K_G + 1] = g2;
        own[K_S] = c.d_scal;     own[K_S + 1] = s2;
        own[K_SEG] = c.d_seg_pos;
        own[K_FLAGS] = d_flags;
        own[K_SEND] = c.d_sendbuf;
        for (int l = 0; l < L; ++l) own[K_H + l] = c.H[l];
        std::vector<void*> tab((size_t)nk * m, nullptr);
        if (g) {   // same process: raw pointers
            std::vector<void*> all((size_t)nk * m);
            allgather(c, own.data(), all.data(), nk * sizeof(void*));
            for (int j = 0; j < m; ++j)
                for (int k = 0; k < nk; ++k) tab[(size_t)k * m + j] = all[(size_t)j * nk + k];
        } else {   // IPC: each underlying allocation exported ONCE (one handle), buffers as (allocation, offset)
            constexpr int kMaxAlloc = 32;
            struct Exp {
                int32_t n;
                int32_t idx[kMaxAlloc];
                int64_t off[kMaxAlloc];
                cudaIpcMemHandle_t h[kMaxAlloc];
            };
            if (nk > kMaxAlloc) throw Error(BNS_ERR_RUNTIME, "peer-memory transport: too many shared buffers");
            auto range = reinterpret_cast<CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr)>(
                driver_entry("cuMemGetAddressRange"));
            Exp mine;
            std::memset(&mine, 0, sizeof(mine));
            std::vector<CUdeviceptr> bases;
            for (int k = 0; k < nk; ++k) {
                CUdeviceptr base = 0;
                size_t sz = 0;
                if (range(&base, &sz, (CUdeviceptr)own[k]) != CUDA_SUCCESS)
                    throw Error(BNS_ERR_RUNTIME, "cuMemGetAddressRange failed");
                int a = -1;
                for (size_t q = 0; q < bases.size(); ++q)
                    if (bases[q] == base) a = (int)q;
                if (a < 0) {
                    a = (int)bases.size();
                    bases.push_back(base);
                    BNS_CUDA(cudaIpcGetMemHandle(&mine.h[a], (void*)base));
                }
                mine.idx[k] = a;
                mine.off[k] = (int64_t)((CUdeviceptr)own[k] - base);
            }
            mine.n = (int32_t)bases.size();
            std::vector<Exp> all(m);
            allgather(c, &mine, all.data(), sizeof(Exp));
            for (int j = 0; j < m; ++j) {
                std::vector<char*> mapped(all[j].n, nullptr);
                if (j != me)
                    for (int a = 0; a < all[j].n; ++a) {
                        void* q = nullptr;
                        const cudaError_t e = cudaIpcOpenMemHandle(&q, all[j].h[a], cudaIpcMemLazyEnablePeerAccess);
                        if (e != cudaSuccess)
                            throw Error(BNS_ERR_RUNTIME, std::string("cudaIpcOpenMemHandle(rank ") + std::to_string(j) +
                                                             ", allocation " + std::to_string(a) + "): " +
                                                             cudaGetErrorString(e));
                        opened.push_back(q);
                        mapped[a] = static_cast<char*>(q);
                    }
                for (int k = 0; k < nk; ++k)
                    tab[(size_t)k * m + j] = j == me ? own[k] : (void*)(mapped[all[j].idx[k]] + all[j].off[k]);
            }
        }
        BNS_CUDA(cudaMalloc(&d_tab, tab.size() * sizeof(void*)));
        BNS_CUDA(cudaMemcpy(d_tab, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice));
        std::vector<int64_t> nin(m);
        const int64_t my_nin = P.n_in;
        allgather(c, &my_nin, nin.data(), sizeof(int64_t));
        BNS_CUDA(cudaMalloc(&d_pnin, m * sizeof(int64_t)));
        BNS_CUDA(cudaMemcpy(d_pnin, nin.data(), m * sizeof(int64_t), cudaMemcpyHostToDevice));
        // the caller's allocations are complete on every rank before anyone's first barrier
        int ok = 1;
        std::vector<int> oks(m);
        allgather(c, &ok, oks.data(), sizeof(int));
    }
    ~PeerTransport() override {
        for (void* p : opened) cudaIpcCloseMemHandle(p);
        for (void* p : {(void*)d_tab, (void*)d_pnin, (void*)d_delta, (void*)d_owner_of_b, (void*)d_row_of_b})
            if (p) cudaFree(p);
        if (h_err) cudaFreeHost(h_err);
        if (g) {
            std::lock_guard<std::mutex> lk(g->mu);
            g->attached[me] = 0;
            bool any = false;
            for (int a : g->attached) any = any || a;
            if (!any) {   // every member has drained its stream: nobody reads a peer arena any more
                for (void* p : g->deferred) cudaFree(p);
                g->deferred.clear();
            }
        }
    }
    // IPC (one process per GPU, destroyed concurrently): one more device barrier, then drain -- after it every peer
    // has finished its last read of this rank's buffers.  In-process members are usually closed one after another
    // from one thread, where a barrier would deadlock: the arena is handed to the group instead and freed when the
    // last member detaches (each member syncs its own stream in bns_destroy first).
    void shutdown(Ctx& c) override {
        c.d_abort = nullptr;
        if (g) {
            std::lock_guard<std::mutex> lk(g->mu);
            for (auto it = c.allocs.begin(); it != c.allocs.end(); ++it)
                if (*it == (void*)c.arena) {
                    c.allocs.erase(it);
                    g->deferred.push_back(c.arena);
                    break;
                }
            return;
        }
        if (!*(volatile int*)h_err) barrier(c, false);
        cudaStreamSynchronize(c.stream);
    }
    void allgather(Ctx&, const void* mine, void* all, size_t bytes) {
        if (g) {
            g->blob[me] = mine;
            group_barrier(g);
            for (int j = 0; j < m; ++j) std::memcpy(static_cast<char*>(all) + j * bytes, g->blob[j], bytes);
            group_barrier(g);
        } else {
            if (ag(mine, all, (int64_t)bytes, ag_user) != 0)
                throw Error(BNS_ERR_RUNTIME, "peer-memory transport: host all-gather callback failed");
        }
    }
    void* const* row(int k) const { return d_tab + (size_t)k * m; }
    void barrier(Ctx& c, bool fetch) {
        launch_peer_barrier(c, reinterpret_cast<uint64_t* const*>(row(K_FLAGS)), ++bar, d_err,
                            fetch ? reinterpret_cast<const int64_t* const*>(row(K_SEG)) : nullptr, d_pnin,
                            fetch ? d_delta : nullptr);
    }
    bool peer() const override { return true; }
    void begin_epoch(Ctx& c) override {
        const int q = (int)(ar_count & 1);
        c.d_gflat = static_cast<float*>(own[K_G + q]);
        c.d_scal = static_cast<double*>(own[K_S + q]);
        c.d_dx = own[K_DX];
        first = true;
    }
    void halo_pull(Ctx& c, int l, void* dst_halo, int64_t din) override {
        barrier(c, true);   // the owners' H^(l-1) is complete; also fetch the peers' segment offsets
        first = false;
        launch_halo_pull(c, dst_halo, din, row(K_H + l - 1), d_owner_of_b, d_row_of_b, (int32_t)din);
    }
    void* dx_buffer(Ctx&, int l) override { return own[K_DX + (l & 1)]; }
    void grad_scatter(Ctx& c, int l, int64_t din) override {
        barrier(c, first);   // the peers' halo gradients of layer l are complete
        first = false;
        launch_scatter_peer(c, c.d_dx, din, row(K_DX + (l & 1)), d_delta, (int32_t)din);
    }
    bool grad_barrier(Ctx& c, int l, const void* const** peer, const int64_t** delta) override {
        barrier(c, first);
        first = false;
        *peer = row(K_DX + (l & 1));
        *delta = d_delta;
        return true;
    }
    void exchange(Ctx& c, const void* src, const int64_t* src_off, void* dst, const int64_t* dst_off,
                  size_t rowbytes) override {
        if (src != c.d_sendbuf) throw Error(BNS_ERR_RUNTIME, "peer-memory transport: generic exchange needs the send buffer");
        std::vector<int64_t> offs((size_t)(m + 1) * m);
        allgather(c, src_off, offs.data(), (m + 1) * sizeof(int64_t));
        std::vector<void*> send(m);
        BNS_CUDA(cudaMemcpy(send.data(), row(K_SEND), m * sizeof(void*), cudaMemcpyDeviceToHost));
        barrier(c, false);
        for (int j = 0; j < m; ++j) {
            if (j == me) continue;
            const int64_t* oj = offs.data() + (size_t)j * (m + 1);
            const int64_t n = oj[me + 1] - oj[me];
            if (n != dst_off[j + 1] - dst_off[j])
                throw Error(BNS_ERR_RUNTIME, "peer-memory transport: row count mismatch between ranks " +
                                                 std::to_string(j) + " -> " + std::to_string(me));
            if (n > 0)
                BNS_CUDA_HOLD(cudaMemcpyAsync(static_cast<char*>(dst) + dst_off[j] * rowbytes,
                                         static_cast<const char*>(send[j]) + oj[me] * rowbytes, n * rowbytes,
                                         cudaMemcpyDeviceToDevice, c.stream));
        }
        barrier(c, false);   // peers have finished reading my send buffer
    }
    void allreduce(Ctx& c, float* buf, int64_t n, double* scal, int64_t ns) override {
        const int q = (int)(ar_count & 1);
        if (buf != own[K_G + q] || scal != own[K_S + q])
            throw Error(BNS_ERR_RUNTIME, "peer-memory transport: all-reduce of an unregistered buffer");
        barrier(c, false);   // every rank's partial gradients are complete
        float* gout = static_cast<float*>(own[K_G + (q ^ 1)]);
        double* sout = static_cast<double*>(own[K_S + (q ^ 1)]);
        launch_sum_ptrs(c, reinterpret_cast<const float* const*>(row(K_G + q)), m, gout, n);
        pdl_hold();   // both sums read the peers' buffers
        launch_sum_ptrs_d(c, reinterpret_cast<const double* const*>(row(K_S + q)), m, sout, ns);
        // no second barrier: a peer reads my buffer q again only after the next epoch's barriers (ping-pong)
        c.d_gflat = gout;
        c.d_scal = sout;
        ++ar_count;
    }
    int64_t allreduce_host_i64(Ctx& c, int64_t v) override {
        std::vector<int64_t> all(m);
        allgather(c, &v, all.data(), sizeof(int64_t));
        int64_t s = 0;
        for (int64_t x : all) s += x;
        return s;
    }
    void poll(Ctx&) override {
        if (*(volatile int*)h_err)
            throw Error(BNS_ERR_RUNTIME, "peer-memory transport: device barrier timed out (a rank did not reach the "
                                         "collective within 20 s)");
    }
};

}  // namespace

Transport* make_transport(Ctx& c) {
    if (c.cfg.transport == BNS_TRANSPORT_IPC) {
        if (!c.cfg.allgather) throw Error(BNS_ERR_INVALID, "transport IPC needs cfg.allgather");
        return new PeerTransport(c, nullptr, c.cfg.allgather, c.cfg.allgather_user);
    }
    if (c.cfg.transport == BNS_TRANSPORT_LOCAL && (c.cfg.flags & BNS_PEER_MEMORY) && c.cfg.world > 1) {
        if (!c.cfg.group) throw Error(BNS_ERR_INVALID, "transport LOCAL needs cfg.group");
        return new PeerTransport(c, c.cfg.group, nullptr, nullptr);
    }
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
    g->blob.assign(world, nullptr);
    *out = g;
    return BNS_OK;
}

void bns_group_destroy(bns_group* g) { delete g; }

}  // extern "C"
