// misc.cu -- bandwidth-bound helpers on the hot path:
//   a4  pack        sendbuf_j[r] = H[S_{i,j}[r]]                   (Alg.1 l.9 "Send H_{S_{i,j}}")
//   a8  loss        softmax-CE over train-masked inner rows / N_train(global) (Alg.1 l.11; R8, R22)
//   a9  relu mask   dPre = dH ⊙ 1[H > 0] (R12: ReLU'(0) = 0)
//   a12 scatter-add dH[S_{i,j}[r]] += recv_j[r] for peers j ascending (R25)
//   a14 update      W <- W - lr g (Alg.1 l.14), g copied to the caller
//   weight pack, local all-reduce sum (rank order), GCN column scales.
#include <cmath>
#include <cstdlib>

#include "common.h"
#include "dev.cuh"
#include "kernels.h"

namespace bns {

namespace {
thread_local bool t_pdl_hold = false;
}
void pdl_hold() { t_pdl_hold = true; }
bool pdl_take_hold() {
    const bool h = t_pdl_hold;
    t_pdl_hold = false;
    return h;
}

bool pdl_enabled() {
    static const bool v = [] { const char* e = std::getenv("BNS_PDL"); return !(e && e[0] == '0'); }();
    return v;
}

// one warp per row, 16-byte vectors
template <typename T>
__global__ void k_pack(const T* __restrict__ src, int64_t ld_src, const int32_t* __restrict__ idx, int64_t n,
                       T* __restrict__ dst, int32_t d) {
    pdl_grid_sync();
    using R = typename Vec<T>::raw;
    const int nvec = d / Vec<T>::N;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = warp; k < n; k += nwarps) {
        const R* s = reinterpret_cast<const R*>(src + (int64_t)idx[k] * ld_src);
        R* o = reinterpret_cast<R*>(dst + k * (int64_t)d);
        for (int v = lane; v < nvec; v += 32) o[v] = s[v];
    }
}

void launch_pack_rows(Ctx& c, const void* src, int64_t ld_src, const int32_t* idx, int64_t n, void* dst, int32_t d) {
    if (n <= 0) return;
    unsigned grid = (unsigned)std::min<int64_t>((n + 7) / 8, 148 * 16);
    if (c.prec == BNS_BF16)
        pdl_launch(c.stream, k_pack<__nv_bfloat16>, grid, 256, 0, (const __nv_bfloat16*)src, ld_src, idx, n, (__nv_bfloat16*)dst, d);
    else
        pdl_launch(c.stream, k_pack<float>, grid, 256, 0, (const float*)src, ld_src, idx, n, (float*)dst, d);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

template <typename T>
__global__ void k_scatter_add(T* __restrict__ dst, int64_t ld_dst, const int32_t* __restrict__ idx,
                              const T* __restrict__ src, int64_t n, int32_t d) {
    pdl_grid_sync();
    using V = Vec<T>;
    using R = typename V::raw;
    constexpr int VN = V::N;
    const int nvec = d / VN;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = warp; k < n; k += nwarps) {
        R* o = reinterpret_cast<R*>(dst + (int64_t)idx[k] * ld_dst);
        const R* s = reinterpret_cast<const R*>(src + k * (int64_t)d);
        for (int v = lane; v < nvec; v += 32) {
            float a[VN], b[VN];
            V::to_float(o[v], a);
            V::to_float(s[v], b);
#pragma unroll
            for (int q = 0; q < VN; ++q) a[q] += b[q];
            o[v] = V::from_float(a);
        }
    }
}

void launch_scatter_add(Ctx& c, void* dst, int64_t ld_dst, const int32_t* idx, const void* src, int64_t n, int32_t d) {
    if (n <= 0) return;
    unsigned grid = (unsigned)std::min<int64_t>((n + 7) / 8, 148 * 16);
    if (c.prec == BNS_BF16)
        pdl_launch(c.stream, k_scatter_add<__nv_bfloat16>, grid, 256, 0, (__nv_bfloat16*)dst, ld_dst, idx,
                                                                 (const __nv_bfloat16*)src, n, d);
    else
        pdl_launch(c.stream, k_scatter_add<float>, grid, 256, 0, (float*)dst, ld_dst, idx, (const float*)src, n, d);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// a12 with every peer in one launch.  k_scatter_prep (once per draw) marks, for each owner row r, the peers j holding
// it (bit j of mask[r]) and the row's position in the returned buffer (pos[r m + j]); k_scatter_rows then adds the
// peers' rows in ascending j, rounding to the storage type after every add -- the same values as one launch per
// peer in ascending order (R25, R19).
__global__ void k_scatter_prep(const int32_t* __restrict__ S_local, int64_t n_sent, const int64_t* __restrict__ seg_pos,
                               int m, uint32_t* __restrict__ mask, int32_t* __restrict__ pos) {
    pdl_grid_sync();
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_sent) return;
    const int64_t base = seg_pos[m];
    int j = 0;
    while (j < m - 1 && seg_pos[m + j + 1] - base <= k) ++j;
    const int32_t r = S_local[k];
    atomicOr(&mask[r], 1u << j);
    pos[(int64_t)r * m + j] = (int32_t)k;
}

template <typename T>
__global__ void __launch_bounds__(256) k_scatter_rows(T* __restrict__ dst, int64_t ld, const T* __restrict__ src,
                                                      int32_t d, const uint32_t* __restrict__ mask,
                                                      const int32_t* __restrict__ pos, int m, int64_t n_rows) {
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
                const int64_t k = pos[r * m + j];
                V::to_float(reinterpret_cast<const R*>(src + k * (int64_t)d)[v], b);
#pragma unroll
                for (int q = 0; q < VN; ++q) a[q] += b[q];
                V::to_float(V::from_float(a), a);   // stored after every peer, as the per-peer sequence
            }
            o[v] = V::from_float(a);
        }
    }
}

void launch_scatter_prep(Ctx& c, int64_t n_sent) {
    const int m = c.cfg.world;
    BNS_CUDA_HOLD(cudaMemsetAsync(c.d_scat_mask, 0, (c.plan.n_in + 1) * sizeof(uint32_t), c.stream));
    if (n_sent <= 0) return;
    pdl_launch(c.stream, k_scatter_prep, (unsigned)((n_sent + 255) / 256), 256, 0, c.d_cand_out + c.n_halo, n_sent,
                                                                           c.d_seg_pos, m, c.d_scat_mask,
                                                                           c.d_scat_pos);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

void launch_scatter_rows(Ctx& c, void* dst, int64_t ld, const void* src, int32_t d) {
    const int64_t n = c.plan.n_in;
    if (n <= 0 || c.n_sent <= 0) return;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 7) / 8, 148 * 16);
    if (c.prec == BNS_BF16)
        pdl_launch(c.stream, k_scatter_rows<__nv_bfloat16>, grid, 256, 0, (__nv_bfloat16*)dst, ld, (const __nv_bfloat16*)src,
                                                                  d, c.d_scat_mask, c.d_scat_pos, c.cfg.world, n);
    else
        pdl_launch(c.stream, k_scatter_rows<float>, grid, 256, 0, (float*)dst, ld, (const float*)src, d, c.d_scat_mask,
                                                          c.d_scat_pos, c.cfg.world, n);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------------------------
// a8 loss: one warp per row; fixed row -> warp -> block assignment and in-order reductions (deterministic).
// ---------------------------------------------------------------------------------------------
constexpr int kXentBlocks = 1184;   // 148 SMs x 8: enough warps to hide the per-row latency

// NPL = logits per lane held in registers (C <= 32 NPL); the row is read once
// the last block to finish sums the per-block partials (nv interleaved values) in a fixed order -- one warp,
// lane-strided then a fixed butterfly: deterministic, and the same values as a separate final kernel would give
__device__ __forceinline__ void last_block_final(const double* part, int nv, double* scal, unsigned* ctr) {
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32)
        for (int q = 0; q < nv; ++q) {
            double a = 0.0;
            for (int k = lane; k < (int)gridDim.x; k += 32) a += __ldcg(part + nv * k + q);
#pragma unroll
            for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (lane == 0) scal[q] = a;
        }
    if (threadIdx.x == 0) *ctr = 0u;
}

// rows [r0, r0 + nrows) of a dPre buffer (pitch ldp, ld columns) set to zero: the halo rows of the transform-first
// [dY | dPre] operand (R42: halo rows have no dPre)
template <typename T>
__device__ __forceinline__ void zero_rows(T* dpre, int64_t ldp, int64_t r0, int64_t nrows, int64_t ld) {
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows * ld; i += nt)
        dpre[(r0 + i / ld) * ldp + i % ld] = from_f<T>(0.f);
}

template <typename T, int NPL>
__global__ void __launch_bounds__(256) k_xent(const float* __restrict__ logits, int64_t ld, int64_t n, int32_t C,
                                              const int32_t* __restrict__ labels, double inv_ntr,
                                              float* __restrict__ dlog, T* __restrict__ dpre, int64_t ldp, int64_t nzero,
                                              double* __restrict__ part, const float* __restrict__ rs,
                                              T* __restrict__ dps, double* __restrict__ scal, unsigned* ctr) {
    pdl_grid_sync();
    __shared__ double s_loss[8];
    __shared__ double s_cor[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t warp = (int64_t)blockIdx.x * 8 + w;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    double loss = 0.0, cor = 0.0;
    for (int64_t r = warp; r < n; r += nwarps) {
        const float* x = logits + r * ld;
        const int y = labels[r];
        float* g = dlog ? dlog + r * ld : nullptr;   // fp32 dLogits only for BNS_Q_DH (BNS_RETAIN_GRADS)
        T* gp = dpre + r * ldp;
        if (y < 0) {
            for (int c = lane; c < ld; c += 32) {
                if (g) g[c] = 0.f;
                gp[c] = from_f<T>(0.f);
                if (dps) dps[r * ld + c] = from_f<T>(0.f);
            }
            continue;
        }
        float xv[NPL];
#pragma unroll
        for (int k = 0; k < NPL; ++k) {
            const int c = lane + 32 * k;
            xv[k] = c < C ? x[c] : -INFINITY;
        }
        float mx = -INFINITY;
        int arg = 0x7fffffff;
#pragma unroll
        for (int k = 0; k < NPL; ++k)
            if (xv[k] > mx) { mx = xv[k]; arg = lane + 32 * k; }   // ascending c per lane: first max kept (R22)
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            float om = __shfl_xor_sync(0xffffffffu, mx, o);
            int oa = __shfl_xor_sync(0xffffffffu, arg, o);
            if (om > mx || (om == mx && oa < arg)) { mx = om; arg = oa; }
        }
        float se = 0.f;
#pragma unroll
        for (int k = 0; k < NPL; ++k)
            if (lane + 32 * k < C) se += expf(xv[k] - mx);
#pragma unroll
        for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        const float lse = mx + logf(se);
        const float rsr = dps ? rs[r] : 0.f;
#pragma unroll
        for (int k = 0; k < NPL; ++k) {
            const int c = lane + 32 * k;
            if (c >= ld) break;
            float v = 0.f;
            if (c < C) v = (float)(((double)expf(xv[k] - lse) - (c == y ? 1.0 : 0.0)) * inv_ntr);
            if (g) g[c] = v;
            const T q = from_f<T>(v);
            gp[c] = q;
            if (dps) dps[r * ld + c] = from_f<T>(to_f(q) * rsr);   // R42: dPre / deg_G(v), from the stored dPre
        }
        if (lane == 0) {
            loss += (double)lse - (double)x[y];
            cor += (arg == y) ? 1.0 : 0.0;
        }
    }
    zero_rows(dpre, ldp, n, nzero, ld);
    if (lane == 0) { s_loss[w] = loss; s_cor[w] = cor; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < 8; ++k) { a += s_loss[k]; b += s_cor[k]; }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
    }
    last_block_final(part, 2, scal, ctr);
}

// f4 / R44 multi-label: per train row and class, softplus(x) - y x (= BCE(σ(x), y)); dLogits = (σ(x) - y) / (N_train C);
// TP / FP / FN of x > 0 for F1-micro.  Block partials [loss, tp, fp, fn], fixed order as k_xent.
template <typename T, int NPL>
__global__ void __launch_bounds__(256) k_bce(const float* __restrict__ logits, int64_t ld, int64_t n, int32_t C,
                                             const int32_t* __restrict__ labels, const uint8_t* __restrict__ tgt,
                                             double inv, float* __restrict__ dlog, T* __restrict__ dpre, int64_t ldp, int64_t nzero,
                                             double* __restrict__ part, const float* __restrict__ rs,
                                             T* __restrict__ dps, double* __restrict__ scal, unsigned* ctr) {
    pdl_grid_sync();
    __shared__ double s_v[4][8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t warp = (int64_t)blockIdx.x * 8 + w;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    double loss = 0.0, tp = 0.0, fp = 0.0, fn = 0.0;
    for (int64_t r = warp; r < n; r += nwarps) {
        const bool train = labels[r] >= 0;
        const float rsr = dps ? rs[r] : 0.f;
        float lsum = 0.f;
        int ntp = 0, nfp = 0, nfn = 0;
#pragma unroll
        for (int k = 0; k < NPL; ++k) {
            const int c = lane + 32 * k;
            if (c >= ld) break;
            float v = 0.f;
            if (train && c < C) {
                const float x = logits[r * ld + c];
                const float y = tgt[r * C + c] ? 1.f : 0.f;
                lsum += fmaxf(x, 0.f) - x * y + log1pf(expf(-fabsf(x)));
                v = (float)((1.0 / (1.0 + exp(-(double)x)) - (double)y) * inv);
                const bool pred = x > 0.f;
                ntp += (pred && y > 0.f);
                nfp += (pred && y == 0.f);
                nfn += (!pred && y > 0.f);
            }
            if (dlog) dlog[r * ld + c] = v;
            const T q = from_f<T>(v);
            dpre[r * ldp + c] = q;
            if (dps) dps[r * ld + c] = from_f<T>(to_f(q) * rsr);
        }
        if (!train) continue;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
            ntp += __shfl_xor_sync(0xffffffffu, ntp, o);
            nfp += __shfl_xor_sync(0xffffffffu, nfp, o);
            nfn += __shfl_xor_sync(0xffffffffu, nfn, o);
        }
        loss += (double)lsum;
        tp += ntp;
        fp += nfp;
        fn += nfn;
    }
    zero_rows(dpre, ldp, n, nzero, ld);
    if (lane == 0) { s_v[0][w] = loss; s_v[1][w] = tp; s_v[2][w] = fp; s_v[3][w] = fn; }
    __syncthreads();
    if (threadIdx.x < 4) {
        double a = 0.0;
        for (int k = 0; k < 8; ++k) a += s_v[threadIdx.x][k];
        part[4 * blockIdx.x + threadIdx.x] = a;
    }
    last_block_final(part, 4, scal, ctr);
}

void launch_bce(Ctx& c, const float* logits, int64_t ld, int32_t C, float* dlogits, void* dpre_t, const float* rs,
                void* dps, int64_t ldp, int64_t nzero) {
    if (ldp < 0) ldp = ld;
    const double inv = c.n_train_global > 0 ? 1.0 / ((double)c.n_train_global * C) : 0.0;
    const int64_t n = c.plan.n_in;
    const int npl = ld <= 32 ? 1 : ld <= 64 ? 2 : ld <= 128 ? 4 : 8;
#define BNS_BCE(T, NPL)                                                                                              \
    pdl_launch(c.stream, k_bce<T, NPL>, kXentBlocks, 256, 0, logits, ld, n, C, c.d_labels, c.d_targets, inv, dlogits,        \
                                                     (T*)dpre_t, ldp, nzero, c.d_lpart, rs, (T*)dps, c.d_scal, c.d_lb_ctr + 8)
    if (c.prec == BNS_BF16) {
        if (npl == 1) BNS_BCE(__nv_bfloat16, 1); else if (npl == 2) BNS_BCE(__nv_bfloat16, 2);
        else if (npl == 4) BNS_BCE(__nv_bfloat16, 4); else BNS_BCE(__nv_bfloat16, 8);
    } else {
        if (npl == 1) BNS_BCE(float, 1); else if (npl == 2) BNS_BCE(float, 2);
        else if (npl == 4) BNS_BCE(float, 4); else BNS_BCE(float, 8);
    }
#undef BNS_BCE
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

void launch_xent(Ctx& c, const float* logits, int64_t ld, int32_t C, float* dlogits, void* dpre_t, const float* rs,
                 void* dps, int64_t ldp, int64_t nzero) {
    if (ldp < 0) ldp = ld;
    const double inv = c.n_train_global > 0 ? 1.0 / (double)c.n_train_global : 0.0;
    const int64_t n = c.plan.n_in;
    const int npl = ld <= 32 ? 1 : ld <= 64 ? 2 : ld <= 128 ? 4 : ld <= 256 ? 8 : 0;
    if (npl == 0) throw Error(BNS_ERR_INVALID, "more than 256 classes are not supported by k_xent");
#define BNS_XENT(T, NPL)                                                                                          \
    pdl_launch(c.stream, k_xent<T, NPL>, kXentBlocks, 256, 0, logits, ld, n, C, c.d_labels, inv, dlogits, (T*)dpre_t, ldp, nzero,   \
                                                      c.d_lpart, rs, (T*)dps, c.d_scal, c.d_lb_ctr + 8)
    if (c.prec == BNS_BF16) {
        if (npl == 1) BNS_XENT(__nv_bfloat16, 1); else if (npl == 2) BNS_XENT(__nv_bfloat16, 2);
        else if (npl == 4) BNS_XENT(__nv_bfloat16, 4); else BNS_XENT(__nv_bfloat16, 8);
    } else {
        if (npl == 1) BNS_XENT(float, 1); else if (npl == 2) BNS_XENT(float, 2);
        else if (npl == 4) BNS_XENT(float, 4); else BNS_XENT(float, 8);
    }
#undef BNS_XENT
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// 16-byte vectors: dpre = dh where h > 0 else 0 (bit select on the storage words; R12 ReLU'(0) = 0)
template <typename T>
__global__ void k_relu_mask(const T* __restrict__ dh, const T* __restrict__ h, int64_t ld, int64_t n,
                            T* __restrict__ dpre, const float* __restrict__ rs, T* __restrict__ dps,
                            const ScatterIn sc) {
    pdl_grid_sync();
    using R = typename Vec<T>::raw;
    constexpr int VN = Vec<T>::N;
    const int64_t nv = n / VN;
    const int64_t vpr = ld / VN;   // vectors per row
    const R* dv = reinterpret_cast<const R*>(dh);
    const R* hv = reinterpret_cast<const R*>(h);
    R* ov = reinterpret_cast<R*>(dpre);
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (; t < nv; t += stride) {
        float a[VN], b[VN];
        Vec<T>::to_float(dv[t], a);
        if (sc.mask) {   // a12 fused: the peers' returned rows of this owner row, peers ascending, rounded to the
                         // storage type after every add (R25, R19) -- the values k_scatter_rows / k_scatter_peer store
            const int64_t r = t / vpr, v = t - r * vpr;
            uint32_t mm = sc.mask[r];
            while (mm) {
                const int j = __ffs(mm) - 1;
                mm &= mm - 1;
                const int64_t k = sc.pos[r * sc.m + j];
                const R* src = sc.peer ? reinterpret_cast<const R*>(static_cast<const T*>(sc.peer[j]) + (k + sc.delta[j]) * ld)
                                       : reinterpret_cast<const R*>(static_cast<const T*>(sc.src) + k * ld);
                Vec<T>::to_float(sc.peer ? __ldcg(src + v) : src[v], b);
#pragma unroll
                for (int q = 0; q < VN; ++q) a[q] += b[q];
                Vec<T>::to_float(Vec<T>::from_float(a), a);
            }
        }
        Vec<T>::to_float(hv[t], b);
#pragma unroll
        for (int k = 0; k < VN; ++k) a[k] = (b[k] > 0.f) ? a[k] : 0.f;
        ov[t] = Vec<T>::from_float(a);
        if (dps) {   // R42: dPre / deg_G(v) for the transform-first SpMM^T (a is exact in T: masked copies of dh)
            const float f = rs[t * VN / ld];
#pragma unroll
            for (int k = 0; k < VN; ++k) a[k] *= f;
            reinterpret_cast<R*>(dps)[t] = Vec<T>::from_float(a);
        }
    }
}

void launch_relu_mask(Ctx& c, const void* dh, const void* h, int64_t ld, int64_t rows, int32_t d, void* dpre,
                      const float* rs, void* dps, const ScatterIn* sc) {
    const int64_t n = rows * ld;   // ld is a multiple of 8: whole 16-byte vectors
    if (n <= 0) return;
    const ScatterIn s = sc ? *sc : ScatterIn{};
    unsigned grid = (unsigned)std::min<int64_t>((n / 4 + 255) / 256, 148 * 16);
    if (c.prec == BNS_BF16)
        pdl_launch(c.stream, k_relu_mask<__nv_bfloat16>, grid, 256, 0, (const __nv_bfloat16*)dh, (const __nv_bfloat16*)h, ld,
                                                               n, (__nv_bfloat16*)dpre, rs, (__nv_bfloat16*)dps, s);
    else
        pdl_launch(c.stream, k_relu_mask<float>, grid, 256, 0, (const float*)dh, (const float*)h, ld, n, (float*)dpre, rs,
                                                       (float*)dps, s);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------------------------
// weights: caller layout (logical, SAGE halves [z-rows ; h-rows]) <-> padded internal layout
// ---------------------------------------------------------------------------------------------
// kind: 0 SAGE (rows [z-half ; h-half], 2 din), 1 GCN (din), 2 GAT ([W ; a_l ; a_r], din + 2)
__device__ __forceinline__ int64_t logical_row(int64_t pr, int kind, int64_t din, int64_t dpin) {
    if (kind == 1) return pr < din ? pr : -1;
    if (pr < dpin) return pr < din ? pr : -1;
    int64_t q = pr - dpin;
    return q < (kind == 0 ? din : 2) ? din + q : -1;
}
__host__ __device__ __forceinline__ int64_t logical_rows(int kind, int64_t din) {
    return kind == 0 ? 2 * din : kind == 2 ? din + 2 : din;
}
__device__ __forceinline__ int64_t padded_row(int64_t lr, int kind, int64_t din, int64_t dpin) {
    return (kind != 1 && lr >= din) ? dpin + (lr - din) : lr;
}

// all layers in one launch: blockIdx.y = layer (blockIdx.y >= L: the W^T copy of layer y - L)
constexpr int kMaxLayers = 16;
struct WDesc {
    const float* W[kMaxLayers];
    float* G[kMaxLayers];
    float* Wp[kMaxLayers];
    void* Wt[kMaxLayers];
    void* WT[kMaxLayers];
    const float* gpad[kMaxLayers];
    int64_t rows_p[kMaxLayers], cols_p[kMaxLayers], din[kMaxLayers], dpin[kMaxLayers], dout[kMaxLayers];
    int64_t K64[kMaxLayers], Kw[kMaxLayers];
    void* Wcat[kMaxLayers];   // R42 transform-first layers: [W_top | W_bot] (storage type) and its transpose
    void* WTtf[kMaxLayers];
    uint32_t tf_mask;
    int L, kind, tc;
};

template <typename T>
__global__ void k_wpack_all(const WDesc d) {
    pdl_grid_sync();
    const int y = blockIdx.y;
    const int l = y % d.L;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t cp = d.cols_p[l];
    // padded weight element (pr, pc) straight from the caller's logical weights
    auto wval = [&](int64_t pr, int64_t pc) -> float {
        const int64_t lr = logical_row(pr, d.kind, d.din[l], d.dpin[l]);
        return (lr >= 0 && pc < d.dout[l]) ? d.W[l][lr * d.dout[l] + pc] : 0.f;
    };
    if (y < d.L) {
        if (t >= d.rows_p[l] * cp) return;
        const int64_t pr = t / cp, pc = t % cp;
        const float v = wval(pr, pc);
        d.Wp[l][t] = v;
        if (d.Wt[l] != (void*)d.Wp[l]) static_cast<T*>(d.Wt[l])[t] = from_f<T>(v);
    } else if (y >= 2 * d.L) {
        // R42: [W_top | W_bot] (dpin x 2 dpout) and its transpose (2 dpout x K64), same launch (no extra pass)
        if (!((d.tf_mask >> l) & 1u)) return;
        const int64_t dpin = d.dpin[l], dpout = cp, n2 = 2 * dpout, K64 = d.K64[l];
        if (t < dpin * n2) {
            const int64_t k = t / n2, c = t % n2;
            static_cast<T*>(d.Wcat[l])[t] = from_f<T>(c < dpout ? wval(k, c) : wval(dpin + k, c - dpout));
        }
        if (d.WTtf[l] && t < n2 * K64) {
            const int64_t n = t / K64, k = t % K64;
            float v = 0.f;
            if (k < dpin) v = n < dpout ? wval(k, n) : wval(dpin + k, n - dpout);
            static_cast<T*>(d.WTtf[l])[t] = from_f<T>(v);
        }
    } else {
        // W^T for the tcgen05 forward: WT[n][kw], kw = half * K64 + j <-> padded row half * dpin + j
        if (!d.tc || t >= cp * d.Kw[l]) return;
        const int64_t n = t / d.Kw[l], kw = t % d.Kw[l];
        const int64_t half = kw / d.K64[l], j = kw % d.K64[l];
        float v = 0.f;
        if (j < d.dpin[l]) {
            const int64_t lr = logical_row(half * d.dpin[l] + j, d.kind, d.din[l], d.dpin[l]);
            if (lr >= 0 && n < d.dout[l]) v = d.W[l][lr * d.dout[l] + n];
        }
        static_cast<T*>(d.WT[l])[t] = from_f<T>(v);   // bf16 (kind::f16) or fp32 (split-TF32 (4 MMAs)) tensor-core operand
    }
}

static WDesc make_desc(Ctx& c, float* const* W, float* const* G) {
    if (c.L > kMaxLayers) throw Error(BNS_ERR_INVALID, "too many layers");
    WDesc d{};
    d.L = c.L;
    d.kind = c.layer == BNS_LAYER_SAGE_MEAN ? 0 : c.layer == BNS_LAYER_GCN ? 1 : 2;
    d.tc = c.use_tc ? 1 : 0;
    for (int l = 0; l < c.L; ++l) {
        d.W[l] = W[l];
        d.G[l] = G ? G[l] : nullptr;
        d.Wp[l] = c.Wpad[l];
        d.Wt[l] = c.Wt[l];
        d.WT[l] = c.use_tc ? c.WT[l] : nullptr;
        d.gpad[l] = c.d_gflat + c.goff[l];
        d.rows_p[l] = c.wrows[l];
        d.cols_p[l] = c.wcols[l];
        d.din[l] = c.dims[l];
        d.dpin[l] = c.dp[l];
        d.dout[l] = c.dims[l + 1];
        d.K64[l] = (c.dp[l] + 63) / 64 * 64;
        d.Kw[l] = c.wkw[l];
        d.Wcat[l] = ((c.tf_mask >> l) & 1u) ? c.Wcat[l] : nullptr;
        d.WTtf[l] = ((c.tf_mask >> l) & 1u) && c.use_tc ? c.WTtf[l] : nullptr;
    }
    d.tf_mask = c.tf_mask;
    return d;
}

void launch_wpack_all(Ctx& c, float* const* W) {
    const WDesc d = make_desc(c, W, nullptr);
    int64_t mx = 0;
    for (int l = 0; l < c.L; ++l) {
        mx = std::max<int64_t>(std::max<int64_t>(mx, d.rows_p[l] * d.cols_p[l]), d.tc ? d.cols_p[l] * d.Kw[l] : 0);
        if ((c.tf_mask >> l) & 1u)
            mx = std::max<int64_t>(mx, std::max(d.dpin[l] * 2 * d.cols_p[l], 2 * d.cols_p[l] * d.K64[l]));
    }
    // y: [0, L) padded W (+ storage copy), [L, 2L) W^T for the tensor cores, [2L, 3L) transform-first packs (R42)
    const dim3 grid((unsigned)((mx + 255) / 256), (unsigned)(c.L * (c.tf_mask ? 3 : d.tc ? 2 : 1)));
    if (c.prec == BNS_BF16) pdl_launch(c.stream, k_wpack_all<__nv_bfloat16>, grid, 256, 0, d);
    else pdl_launch(c.stream, k_wpack_all<float>, grid, 256, 0, d);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// a14 W <- W - lr g for every layer (g copied to the caller); skipped when the all-reduced loss is not finite
__global__ void k_sgd_all(const WDesc d, float lr, const double* __restrict__ scal, int32_t* __restrict__ nonfinite,
                          const volatile int* abort) {
    pdl_grid_sync();
    const int l = blockIdx.y;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t rows_l = logical_rows(d.kind, d.din[l]), dout = d.dout[l];
    if (t >= rows_l * dout) return;
    const bool bad = !isfinite(scal[0]);
    if (t == 0 && l == 0) *nonfinite = bad ? 1 : 0;
    if (abort && *abort) return;   // a peer barrier timed out: the gradient is incomplete, leave W untouched
    const int64_t lr_ = t / dout, lc = t % dout;
    const int64_t pr = padded_row(lr_, d.kind, d.din[l], d.dpin[l]);
    const float g = d.gpad[l][pr * d.cols_p[l] + lc];
    if (d.G[l]) d.G[l][t] = g;
    if (!bad) const_cast<float*>(d.W[l])[t] -= lr * g;
}

void launch_sgd(Ctx& c, float* const* W, float* const* G, float lr) {
    const WDesc d = make_desc(c, W, G);
    int64_t mx = 0;
    for (int l = 0; l < c.L; ++l) mx = std::max(mx, logical_rows(d.kind, d.din[l]) * d.dout[l]);
    pdl_launch(c.stream, k_sgd_all, dim3((unsigned)((mx + 255) / 256), (unsigned)c.L), 256, 0, d, lr, c.d_scal, c.d_nonfinite,
                                                                                     c.d_abort);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

__global__ void k_sum_ptrs(const float* const* __restrict__ p, int np, float* __restrict__ out, int64_t n) {
    pdl_grid_sync();
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    float s = 0.f;
    for (int k = 0; k < np; ++k) s += p[k][t];
    out[t] = s;
}
__global__ void k_sum_ptrs_d(const double* const* __restrict__ p, int np, double* __restrict__ out, int64_t n) {
    pdl_grid_sync();
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double s = 0.0;
    for (int k = 0; k < np; ++k) s += p[k][t];
    out[t] = s;
}
void launch_sum_ptrs(Ctx& c, const float* const* d_ptrs, int nptr, float* out, int64_t n) {
    if (n <= 0) return;
    pdl_launch(c.stream, k_sum_ptrs, (unsigned)((n + 255) / 256), 256, 0, d_ptrs, nptr, out, n);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}
void launch_sum_ptrs_d(Ctx& c, const double* const* d_ptrs, int nptr, double* out, int64_t n) {
    if (n <= 0) return;
    pdl_launch(c.stream, k_sum_ptrs_d, (unsigned)((n + 255) / 256), 256, 0, d_ptrs, nptr, out, n);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// GCN: per-column scale of the sampled propagation [rs_in ; (1/p) rs_bd[U_b]] (App. A S diagonal)
__global__ void k_gcn_cscale(const float* __restrict__ rs_in, int64_t n_in, const float* __restrict__ rs_bd,
                             const int32_t* __restrict__ U_b, const int64_t* __restrict__ seg_pos, int m, float inv_p,
                             int64_t cap, float* __restrict__ cs) {
    pdl_grid_sync();
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_in) { cs[t] = rs_in[t]; return; }
    int64_t s = t - n_in;
    if (s >= cap) return;
    if (s < seg_pos[m] - seg_pos[0]) cs[t] = inv_p * rs_bd[U_b[s]];
}

void launch_gcn_cscale(Ctx& c) {
    const int64_t n = c.plan.n_in + c.halo_cap;
    if (n <= 0) return;
    pdl_launch(c.stream, k_gcn_cscale, (unsigned)((n + 255) / 256), 256, 0, c.d_rs_in, c.plan.n_in, c.d_rs_bd, c.d_cand_out,
                                                                    c.d_seg_pos, c.cfg.world, c.inv_p, c.halo_cap,
                                                                    c.d_cscale);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

template <typename T>
__global__ void k_to_storage(const float* __restrict__ src, int64_t rows, int32_t dlog, int64_t ld_src,
                             T* __restrict__ dst, int64_t ld_dst) {
    pdl_grid_sync();
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * ld_dst) return;
    int64_t r = t / ld_dst, k = t % ld_dst;
    dst[t] = from_f<T>(k < dlog ? src[r * ld_src + k] : 0.f);
}

void launch_to_storage(Ctx& c, const float* src, int64_t rows, int32_t dlog, int64_t ld_src, void* dst, int64_t ld_dst) {
    const int64_t n = rows * ld_dst;
    if (n <= 0) return;
    if (c.prec == BNS_BF16)
        pdl_launch(c.stream, k_to_storage<__nv_bfloat16>, (unsigned)((n + 255) / 256), 256, 0, src, rows, dlog, ld_src,
                                                                                      (__nv_bfloat16*)dst, ld_dst);
    else
        pdl_launch(c.stream, k_to_storage<float>, (unsigned)((n + 255) / 256), 256, 0, src, rows, dlog, ld_src, (float*)dst,
                                                                              ld_dst);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

}  // namespace bns

namespace bns {

// ---------------------------------------------------------------------------------------------
// f2 dropout (R38): dst[r][c] = src[r][c] * (keep ? 1/(1-r) : 0), one Philox call per 4 columns, keyed by the
// row's global id, the column quad, the layer and the epoch.  Used on the layer input (forward) and, in place, on
// the gradient w.r.t. it (backward).
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void k_dropout(const T* __restrict__ src, T* __restrict__ dst, int64_t rows, int64_t ld,
                          const int32_t* __restrict__ gid, uint32_t layer, uint32_t e_lo, uint32_t k0, uint32_t k1,
                          uint64_t thr, float scale) {
    pdl_grid_sync();
    const int64_t nq = (ld + 3) / 4;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * nq) return;
    const int64_t r = t / nq, q = t % nq;
    const uint4 w = philox4((uint32_t)gid[r], (uint32_t)q, layer, e_lo, k0, k1);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t c = q * 4 + k;
        if (c >= ld) break;
        const float f = ((uint64_t)ws[k] >= thr) ? scale : 0.f;
        dst[r * ld + c] = from_f<T>(to_f<T>(src[r * ld + c]) * f);
    }
}

void launch_dropout(Ctx& c, const void* src, void* dst, int64_t rows, int64_t ld, int layer) {
    if (rows <= 0 || c.drop <= 0.0) return;
    const uint64_t thr = (uint64_t)std::floor(c.drop * 4294967296.0);
    const float scale = (float)(1.0 / (1.0 - c.drop));
    const uint32_t k0 = (uint32_t)(c.drop_seed & 0xffffffffu) ^ 0xD809u, k1 = (uint32_t)(c.drop_seed >> 32);
    const int64_t n = rows * ((ld + 3) / 4);
    const unsigned grid = (unsigned)((n + 255) / 256);
    if (c.prec == BNS_BF16)
        pdl_launch(c.stream, k_dropout<__nv_bfloat16>, grid, 256, 0, (const __nv_bfloat16*)src, (__nv_bfloat16*)dst, rows, ld,
                                                             c.d_rowgid, (uint32_t)layer, (uint32_t)c.epoch_id, k0, k1,
                                                             thr, scale);
    else
        pdl_launch(c.stream, k_dropout<float>, grid, 256, 0, (const float*)src, (float*)dst, rows, ld, c.d_rowgid,
                                                     (uint32_t)layer, (uint32_t)c.epoch_id, k0, k1, thr, scale);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// global ids of the halo rows of this epoch: rowgid[n_in + s] = gid of boundary node U_b[s]
__global__ void k_halo_gid(const int32_t* __restrict__ cand_gid, const int32_t* __restrict__ U_b, int64_t n_halo,
                           int64_t n_in, int32_t* __restrict__ rowgid) {
    pdl_grid_sync();
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n_halo) rowgid[n_in + s] = cand_gid[U_b[s]];
}

void launch_halo_gid(Ctx& c) {
    if (c.n_halo <= 0) return;
    pdl_launch(c.stream, k_halo_gid, (unsigned)((c.n_halo + 255) / 256), 256, 0, c.d_cand_gid, c.d_cand_out, c.n_halo,
                                                                         c.plan.n_in, c.d_rowgid);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// f2 Adam (bias-corrected; Kingma & Ba) over every layer in one launch, moments in fp32 at the logical layout;
// skipped (moments untouched) when the all-reduced loss is not finite
struct AdamArgs {
    float* m;
    float* v;
    int64_t moff[kMaxLayers];
    float lr, b1, b2, eps, c1, c2;
};

__global__ void k_adam_all(const WDesc d, const AdamArgs a, const double* __restrict__ scal,
                           int32_t* __restrict__ nonfinite, const volatile int* abort) {
    pdl_grid_sync();
    const int l = blockIdx.y;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t rows_l = logical_rows(d.kind, d.din[l]), dout = d.dout[l];
    if (t >= rows_l * dout) return;
    const bool bad = !isfinite(scal[0]);
    if (t == 0 && l == 0) *nonfinite = bad ? 1 : 0;
    if (abort && *abort) return;   // a peer barrier timed out: no update, moments untouched
    const int64_t lr_ = t / dout, lc = t % dout;
    const int64_t pr = padded_row(lr_, d.kind, d.din[l], d.dpin[l]);
    const float g = d.gpad[l][pr * d.cols_p[l] + lc];
    if (d.G[l]) d.G[l][t] = g;
    if (bad) return;
    float* mm = a.m + a.moff[l] + t;
    float* vv = a.v + a.moff[l] + t;
    const float m1 = a.b1 * *mm + (1.f - a.b1) * g;
    const float v1 = a.b2 * *vv + (1.f - a.b2) * g * g;
    *mm = m1;
    *vv = v1;
    const_cast<float*>(d.W[l])[t] -= a.lr * (m1 / a.c1) / (sqrtf(v1 / a.c2) + a.eps);
}

void launch_adam(Ctx& c, float* const* W, float* const* G, float lr) {
    const WDesc d = make_desc(c, W, G);
    AdamArgs a{};
    a.m = c.d_adam_m;
    a.v = c.d_adam_v;
    int64_t off = 0, mx = 0;
    for (int l = 0; l < c.L; ++l) {
        a.moff[l] = off;
        const int64_t n = logical_rows(d.kind, d.din[l]) * d.dout[l];
        off += n;
        mx = std::max(mx, n);
    }
    a.lr = lr;
    a.b1 = (float)c.beta1;
    a.b2 = (float)c.beta2;
    a.eps = (float)c.eps;
    a.c1 = (float)(1.0 - std::pow(c.beta1, (double)c.adam_t));
    a.c2 = (float)(1.0 - std::pow(c.beta2, (double)c.adam_t));
    pdl_launch(c.stream, k_adam_all, dim3((unsigned)((mx + 255) / 256), (unsigned)c.L), 256, 0, d, a, c.d_scal, c.d_nonfinite,
                                                                                      c.d_abort);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

}  // namespace bns
