// peer.cu -- SURVEY §8(f) f1: the exchange steps of Algorithm 1 fused with their producer / consumer over peer
// memory (NVLink 5 / NVSwitch loads of the other GPUs' HBM through CUDA IPC mappings; in-process contexts share
// pointers directly).  No staging buffer, no NCCL kernel, no per-peer message:
//   a4 + a5   k_halo_pull     the halo rows of [H ; H_U] are read straight from the owners' H^(l-1) inner rows
//                             (Alg.1 l.9 "Send H_{S_{i,j}} / Receive H_{U_i}"): pack and exchange
//                             become one gather kernel on the receiving GPU.
//   a11 + a12 k_scatter_peer  every owner row adds the halo-row gradients the peers computed for it, read straight
//                             from the peers' dX halo rows, local value first then peers ascending (PAPER.md:179,
//                             :336; R25) -- the reverse exchange and the scatter-add become one kernel.
//   a13       k_sum_ptrs      (misc.cu) the weight-gradient sum reads every rank's partial gradient in rank order
//                             (Alg.1 l.13), so every rank holds bitwise the same sum.
// Ordering between GPUs is a device-side flag barrier (k_peer_barrier): each rank stores an increasing barrier
// number into every peer's flag slot with a system-scope release and spins with system-scope acquires until all
// peers' numbers arrived.  It is bounded by a 20 s %globaltimer timeout that raises an error flag instead of hanging.
#include <mutex>

#include <cuda.h>

#include "common.h"
#include "dev.cuh"
#include "kernels.h"

namespace bns {

namespace {

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr uint64_t kBarrierTimeoutNs = 20ull * 1000 * 1000 * 1000;

// one warp; lane j < m (j != me) signals peer j and then waits for peer j's signal.  With fetch, lane j also derives
// the row offset of this rank's rows inside peer j's halo gradient (delta[j], used by k_scatter_peer):
//   peer row = n_in_j + (seg_j[me] - seg_j[0]) + (k - (seg_me[m + j] - seg_me[m])),  k = index in S_{me, j}
__global__ void k_peer_barrier(uint64_t* const* __restrict__ flags, int me, int m, uint64_t val, int* err,
                               const int64_t* const* __restrict__ pseg, const int64_t* __restrict__ pnin,
                               int64_t* __restrict__ delta) {
    pdl_grid_sync();
    const int j = threadIdx.x;
    if (j >= m || j == me) return;
    if (*(volatile int*)err) return;   // an earlier barrier timed out: the epoch is already failed, do not wait again
    __threadfence_system();   // every earlier write of this stream is performed before the signal
    uint64_t* dst = flags[j] + me;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(val) : "memory");
    const uint64_t* src = flags[me] + j;
    const uint64_t t0 = globaltimer_ns();
    for (;;) {
        uint64_t v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(src) : "memory");
        if (v >= val) break;
        if (globaltimer_ns() - t0 > kBarrierTimeoutNs) {
            atomicExch_system(err, 1);
            return;
        }
        __nanosleep(200);
    }
    if (delta) {
        const int64_t* ps = pseg[me];   // my own segment offsets
        const int64_t* qs = pseg[j];    // peer j's (read over NVLink after the barrier)
        const int64_t seg_in_peer = __ldcg(qs + me) - __ldcg(qs + 0);
        const int64_t my_send = ps[m + j] - ps[m];
        delta[j] = pnin[j] + seg_in_peer - my_send;
    }
}

// a4 + a5: halo slot s of this rank (U_i[s] = boundary index b) <- row row_of_b[b] of owner owner_of_b[b]'s H
template <typename T>
__global__ void __launch_bounds__(256) k_halo_pull(T* __restrict__ dst, int64_t ld, const int32_t* __restrict__ U_b,
                                                   int64_t n, const int32_t* __restrict__ owner_of_b,
                                                   const int32_t* __restrict__ row_of_b, T* const* __restrict__ peerH,
                                                   int32_t d) {
    pdl_grid_sync();
    using R = typename Vec<T>::raw;
    const int nvec = d / Vec<T>::N;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = warp; s < n; s += nwarps) {
        const int32_t b = U_b[s];
        const R* src = reinterpret_cast<const R*>(peerH[owner_of_b[b]] + (int64_t)row_of_b[b] * ld);
        R* o = reinterpret_cast<R*>(dst + s * ld);
        for (int v = lane; v < nvec; v += 32) o[v] = __ldcg(src + v);
    }
}

// a11 + a12: owner row r += peers' halo-gradient rows, peers ascending, rounded to the storage type after every add
// (the per-peer sequence of R25 / R19, identical to k_scatter_rows on the received buffer)
template <typename T>
__global__ void __launch_bounds__(256) k_scatter_peer(T* __restrict__ dst, int64_t ld, int32_t d,
                                                      const uint32_t* __restrict__ mask, const int32_t* __restrict__ pos,
                                                      int m, int64_t n_rows, T* const* __restrict__ peerdx,
                                                      const int64_t* __restrict__ delta) {
    pdl_grid_sync();
    using V = Vec<T>;
    using R = typename V::raw;
    constexpr int VN = V::N;
    const int nvec = d / VN;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nwarps) {
        const uint32_t mk = mask[r];
        if (!mk) continue;
        R* o = reinterpret_cast<R*>(dst + r * ld);
        for (int v = lane; v < nvec; v += 32) {
            float a[VN], b[VN];
            V::to_float(o[v], a);
            uint32_t mm = mk;
            while (mm) {
                const int j = __ffs(mm) - 1;
                mm &= mm - 1;
                const int64_t row = pos[r * m + j] + delta[j];
                V::to_float(__ldcg(reinterpret_cast<const R*>(peerdx[j] + row * ld) + v), b);
#pragma unroll
                for (int q = 0; q < VN; ++q) a[q] += b[q];
                V::to_float(V::from_float(a), a);
            }
            o[v] = V::from_float(a);
        }
    }
}

}  // namespace

// CUDA 12 loads kernels lazily, and loading one waits for the device to go idle: a rank whose first launch of some
// kernel happens while a peer's barrier kernel spins on the same GPU would wait for that spinner, which waits for the
// rank -- so peer-memory contexts load every function of the library's (device-linked, single) module up front.
void preload_module_functions() {
    static std::once_flag once;
    std::call_once(once, [] {
    auto entry = [](const char* name) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        BNS_CUDA(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw Error(BNS_ERR_RUNTIME, std::string(name) + " unavailable");
        return p;
    };
    auto getmod = reinterpret_cast<CUresult (*)(CUmodule*, CUfunction)>(entry("cuFuncGetModule"));
    auto count = reinterpret_cast<CUresult (*)(unsigned*, CUmodule)>(entry("cuModuleGetFunctionCount"));
    auto enumf = reinterpret_cast<CUresult (*)(CUfunction*, unsigned, CUmodule)>(entry("cuModuleEnumerateFunctions"));
    auto load = reinterpret_cast<CUresult (*)(CUfunction)>(entry("cuFuncLoad"));
    cudaFunction_t f0;
    BNS_CUDA(cudaGetFuncBySymbol(&f0, (const void*)k_peer_barrier));
    CUmodule mod;
    unsigned n = 0;
    if (getmod(&mod, (CUfunction)f0) != CUDA_SUCCESS || count(&n, mod) != CUDA_SUCCESS)
        throw Error(BNS_ERR_RUNTIME, "cannot enumerate the library's kernels");
    std::vector<CUfunction> fs(n);
    if (n && enumf(fs.data(), n, mod) != CUDA_SUCCESS) throw Error(BNS_ERR_RUNTIME, "cuModuleEnumerateFunctions failed");
    for (CUfunction f : fs)
        if (load(f) != CUDA_SUCCESS) throw Error(BNS_ERR_RUNTIME, "cuFuncLoad failed");
    });
}

void launch_peer_barrier(Ctx& c, uint64_t* const* d_flags, uint64_t val, int* err, const int64_t* const* d_pseg,
                         const int64_t* d_pnin, int64_t* d_delta) {
    // strict stream order on both sides of the barrier: it starts after everything before it (the peers may read
    // this rank's buffers once it signals), and the kernel after it -- a gather from the peers' memory -- starts
    // only when it has completed
    pdl_hold();
    pdl_launch(c.stream, k_peer_barrier, 1, 32, 0, d_flags, c.cfg.rank, c.cfg.world, val, err, d_pseg, d_pnin, d_delta);
    pdl_hold();
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

void launch_halo_pull(Ctx& c, void* dst, int64_t ld, void* const* d_peerH, const int32_t* d_owner_of_b,
                      const int32_t* d_row_of_b, int32_t d) {
    const int64_t n = c.n_halo;
    if (n <= 0) return;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 7) / 8, 148 * 16);
    if (c.prec == BNS_BF16)
        pdl_launch(c.stream, k_halo_pull<__nv_bfloat16>, grid, 256, 0, (__nv_bfloat16*)dst, ld, c.d_cand_out, n, d_owner_of_b,
                                                               d_row_of_b, (__nv_bfloat16* const*)d_peerH, d);
    else
        pdl_launch(c.stream, k_halo_pull<float>, grid, 256, 0, (float*)dst, ld, c.d_cand_out, n, d_owner_of_b, d_row_of_b,
                                                       (float* const*)d_peerH, d);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

void launch_scatter_peer(Ctx& c, void* dst, int64_t ld, void* const* d_peerdx, const int64_t* d_delta, int32_t d) {
    const int64_t n = c.plan.n_in;
    if (n <= 0 || c.n_sent <= 0) return;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 7) / 8, 148 * 16);
    if (c.prec == BNS_BF16)
        pdl_launch(c.stream, k_scatter_peer<__nv_bfloat16>, grid, 256, 0, (__nv_bfloat16*)dst, ld, d, c.d_scat_mask,
                                                                  c.d_scat_pos, c.cfg.world, n,
                                                                  (__nv_bfloat16* const*)d_peerdx, d_delta);
    else
        pdl_launch(c.stream, k_scatter_peer<float>, grid, 256, 0, (float*)dst, ld, d, c.d_scat_mask, c.d_scat_pos,
                                                          c.cfg.world, n, (float* const*)d_peerdx, d_delta);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

}  // namespace bns
