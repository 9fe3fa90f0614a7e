// gat.cu -- f4 / R45: the pieces of a one-head GAT layer (Velickovic et al., Table tab:gat) that
// are not the shared GEMM / segment-SpMM kernels.  With Y = H W (stacked rows), el = Y a_l, er = Y a_r,
// s_vu = el_v + er_u, e = LeakyReLU_0.2(s), alpha_vu = softmax over N'(v) = {sampled neighbours} ∪ {v}:
//   k_gat_scores     el, er per stacked row
//   k_gat_stats      max and 1/Σexp of e over N'(v), per segment then in segment order (deterministic)
//   (k_spmm SC = 3)  pre_v = Σ alpha_vu Y_u  (+ alpha_vv Y_v, ReLU in the epilogue)
// backward, g = dPre:
//   k_gat_rowdots    c_v = g_v . pre_v, selfds_v = alpha_vv (g_v . Y_v - c_v) LeakyReLU'(s_vv)
//   del_v = Σ_u ds_vu, der_u = Σ_v ds_vu with ds_vu = alpha_vu (g_v . Y_u - c_v) LeakyReLU'(s_vu), rewritten without
//   per-edge dot products: w = alpha LeakyReLU'(s); Q_v = Σ_u w_vu Y_u and P_u = Σ_v w_vu g_v by the segment SpMM
//   (SC 5 / 6, GAT_RAW), q_v = Σ_u w_vu and r_u = Σ_v w_vu c_v by k_gat_wsum, then k_gat_final:
//   del_v = g_v . Q_v - c_v q_v + selfds_v, der_u = Y_u . P_u - r_u + [inner] selfds_u
//   (k_spmm SC = 4)  dY_u = Σ_v alpha_vu g_v + [inner] (alpha_uu g_u + del_u a_l) + der_u a_r
//   k_gat_da         da_l = Σ_v del_v Y_v, da_r = Σ_u der_u Y_u (two-stage, fixed order)
#include "common.h"
#include "dev.cuh"
#include "kernels.h"

namespace bns {

__device__ __forceinline__ float lrelu(float x) { return x > 0.f ? x : 0.2f * x; }

template <typename T>
__device__ __forceinline__ float row_dot(const T* __restrict__ x, const float* __restrict__ y, int d, int lane) {
    using V = Vec<T>;
    constexpr int VN = V::N;
    float s = 0.f;
    for (int v = lane; v < d / VN; v += 32) {
        float f[VN];
        V::to_float(reinterpret_cast<const typename V::raw*>(x)[v], f);
#pragma unroll
        for (int k = 0; k < VN; ++k) s = fmaf(f[k], y[v * VN + k], s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

template <typename T>
__global__ void __launch_bounds__(256) k_gat_scores(const T* __restrict__ Y, int64_t ld, int64_t rows, int32_t d,
                                                    const float* __restrict__ al, const float* __restrict__ ar,
                                                    float* __restrict__ el, float* __restrict__ er) {
    pdl_grid_sync();
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
        const float a = row_dot(Y + r * ld, al, d, lane);
        const float b = row_dot(Y + r * ld, ar, d, lane);
        if (lane == 0) { el[r] = a; er[r] = b; }
    }
}

// online softmax merge of (m, s) pairs: s = Σ exp(e - m)
__device__ __forceinline__ void sm_merge(float& m, float& s, float m2, float s2) {
    const float mx = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * expf(m - mx)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - mx));
    m = mx;
}

__global__ void __launch_bounds__(256) k_gat_stats(const Seg* __restrict__ segs, int64_t n_segs,
                                                   const int32_t* __restrict__ col, const float* __restrict__ el,
                                                   const float* __restrict__ er, float* __restrict__ part,
                                                   float* __restrict__ m_out, float* __restrict__ inv_out) {
    pdl_grid_sync();
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sid < n_segs; sid += nw) {
        const Seg sg = segs[sid];
        const float ev = el[sg.row];
        float m = -INFINITY, s = 0.f;
        for (int64_t e = sg.e0 + lane; e < sg.e1; e += 32) sm_merge(m, s, lrelu(ev + er[col[e]]), 1.f);
#pragma unroll
        for (int o = 16; o; o >>= 1) sm_merge(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
        if (lane) continue;
        if (sg.nseg > 1) {
            part[2 * sid] = m;
            part[2 * sid + 1] = s;
        } else {
            sm_merge(m, s, lrelu(ev + er[sg.row]), 1.f);   // self loop
            m_out[sg.row] = m;
            inv_out[sg.row] = 1.f / s;
        }
    }
}

__global__ void k_gat_stats_fix(const Seg* __restrict__ segs, const int64_t* __restrict__ split, int64_t n_split,
                                const float* __restrict__ el, const float* __restrict__ er,
                                const float* __restrict__ part, float* __restrict__ m_out,
                                float* __restrict__ inv_out) {
    pdl_grid_sync();
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_split) return;
    const int64_t sid = split[q];
    const Seg sg = segs[sid];
    float m = -INFINITY, s = 0.f;
    for (int k = 0; k < sg.nseg; ++k) sm_merge(m, s, part[2 * (sid + k)], part[2 * (sid + k) + 1]);
    sm_merge(m, s, lrelu(el[sg.row] + er[sg.row]), 1.f);
    m_out[sg.row] = m;
    inv_out[sg.row] = 1.f / s;
}

template <typename T, bool OUT_F32>
__global__ void __launch_bounds__(256) k_gat_rowdots(const T* __restrict__ g, const void* __restrict__ out,
                                                     const T* __restrict__ Y, int64_t ld, int64_t n, int32_t d,
                                                     const float* __restrict__ el, const float* __restrict__ er,
                                                     const float* __restrict__ m, const float* __restrict__ inv,
                                                     float* __restrict__ cdot, float* __restrict__ selfds) {
    pdl_grid_sync();
    using V = Vec<T>;
    constexpr int VN = V::N;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
        float c = 0.f, gy = 0.f;
        for (int v = lane; v < d / VN; v += 32) {
            float fg[VN], fo[VN], fy[VN];
            V::to_float(reinterpret_cast<const typename V::raw*>(g + r * ld)[v], fg);
            V::to_float(reinterpret_cast<const typename V::raw*>(Y + r * ld)[v], fy);
            if (OUT_F32) {
#pragma unroll
                for (int k = 0; k < VN; ++k) fo[k] = static_cast<const float*>(out)[r * ld + v * VN + k];
            } else {
                V::to_float(reinterpret_cast<const typename V::raw*>(static_cast<const T*>(out) + r * ld)[v], fo);
            }
#pragma unroll
            for (int k = 0; k < VN; ++k) {
                c = fmaf(fg[k], fo[k], c);
                gy = fmaf(fg[k], fy[k], gy);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            c += __shfl_xor_sync(0xffffffffu, c, o);
            gy += __shfl_xor_sync(0xffffffffu, gy, o);
        }
        if (lane == 0) {
            const float t = el[r] + er[r];
            const float a = expf(lrelu(t) - m[r]) * inv[r];
            cdot[r] = c;
            selfds[r] = a * (gy - c) * (t > 0.f ? 1.f : 0.2f);
        }
    }
}

// scalar edge sums over segments (self edges excluded): DIR 0 q_v = Σ_u w_vu, DIR 1 r_u = Σ_v w_vu c_v,
// w_vu = alpha_vu LeakyReLU'(s_vu); whole rows store, split rows leave per-segment partials for k_gat_wsum_fix
template <int DIR>
__global__ void __launch_bounds__(256) k_gat_wsum(const Seg* __restrict__ segs, int64_t n_segs,
                                                  const int32_t* __restrict__ col, const float* __restrict__ el,
                                                  const float* __restrict__ er, const float* __restrict__ m,
                                                  const float* __restrict__ inv, const float* __restrict__ cdot,
                                                  float* __restrict__ part, float* __restrict__ out) {
    pdl_grid_sync();
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sid < n_segs; sid += nw) {
        const Seg sg = segs[sid];
        float acc = 0.f;
        for (int64_t e = sg.e0 + lane; e < sg.e1; e += 32) {
            const int32_t x = col[e];
            const int64_t vv = DIR == 0 ? sg.row : x;
            const int64_t uu = DIR == 0 ? x : sg.row;
            const float t = el[vv] + er[uu];
            float w = expf(lrelu(t) - m[vv]) * inv[vv] * (t > 0.f ? 1.f : 0.2f);
            if (DIR == 1) w *= cdot[vv];
            acc += w;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane) continue;
        if (sg.nseg > 1) part[sid] = acc;
        else out[sg.row] = acc;
    }
}

__global__ void k_gat_wsum_fix(const Seg* __restrict__ segs, const int64_t* __restrict__ split, int64_t n_split,
                               const float* __restrict__ part, float* __restrict__ out) {
    pdl_grid_sync();
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_split) return;
    const int64_t sid = split[q];
    const Seg sg = segs[sid];
    float acc = 0.f;
    for (int k = 0; k < sg.nseg; ++k) acc += part[sid + k];
    out[sg.row] = acc;
}

// DIR 0: del_v = g_v . Q_v - c_v q_v + selfds_v (inner rows);  DIR 1: der_u = Y_u . P_u - r_u + [inner] selfds_u
template <typename T, int DIR>
__global__ void __launch_bounds__(256) k_gat_final(const T* __restrict__ own, const float* __restrict__ qp,
                                                   int64_t ld, int32_t d, int64_t rows, int64_t n_in,
                                                   const float* __restrict__ cdot, const float* __restrict__ qr,
                                                   const float* __restrict__ selfds, float* __restrict__ out) {
    pdl_grid_sync();
    using V = Vec<T>;
    constexpr int VN = V::N;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
        const float s = row_dot(own + r * ld, qp + r * ld, d, lane);
        if (lane == 0)
            out[r] = s - (DIR == 0 ? cdot[r] * qr[r] : qr[r]) + (r < n_in ? selfds[r] : 0.f);
    }
}

// out[c] = Σ_r w_r Y_r[c]: block b sums its row range in order per column, then one pass over the blocks in order
constexpr int kDaBlocks = 296;
template <typename T>
__global__ void __launch_bounds__(256) k_gat_da1(const T* __restrict__ Y, int64_t ld, int32_t d,
                                                 const float* __restrict__ w, int64_t rows, float* __restrict__ part) {
    pdl_grid_sync();
    const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(rows, r0 + per);
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        float s = 0.f;
        for (int64_t r = r0; r < r1; ++r) s = fmaf(w[r], to_f(Y[r * ld + c]), s);
        part[(int64_t)blockIdx.x * d + c] = s;
    }
}

__global__ void k_gat_da2(const float* __restrict__ part, int nb, int32_t d, float* __restrict__ out) {
    pdl_grid_sync();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d) return;
    float s = 0.f;
    for (int b = 0; b < nb; ++b) s += part[(int64_t)b * d + c];
    out[c] = s;
}

// ------------------------------------------------------------------------------------------------
void launch_gat_scores(Ctx& c, const void* Y, int64_t ld, int64_t rows, int32_t d, const float* al, const float* ar,
                       float* el, float* er) {
    if (rows <= 0) return;
    const unsigned grid = (unsigned)std::min<int64_t>((rows + 7) / 8, 148 * 16);
    if (c.prec == BNS_BF16)
        pdl_launch(c.stream, k_gat_scores<__nv_bfloat16>, grid, 256, 0, (const __nv_bfloat16*)Y, ld, rows, d, al, ar, el, er);
    else
        pdl_launch(c.stream, k_gat_scores<float>, grid, 256, 0, (const float*)Y, ld, rows, d, al, ar, el, er);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

void launch_gat_stats(Ctx& c, const Seg* segs, int64_t n_segs, const int32_t* col, const int64_t* split,
                      int64_t n_split, const float* el, const float* er, float* m, float* inv) {
    if (n_segs <= 0) return;
    const unsigned grid = (unsigned)std::min<int64_t>((n_segs + 7) / 8, 148 * 16);
    pdl_launch(c.stream, k_gat_stats, grid, 256, 0, segs, n_segs, col, el, er, c.d_partial, m, inv);
    c.kernels += 1;
    if (n_split > 0) {
        pdl_launch(c.stream, k_gat_stats_fix, (unsigned)((n_split + 127) / 128), 128, 0, segs, split, n_split, el, er,
                                                                                 c.d_partial, m, inv);
        c.kernels += 1;
    }
    BNS_CHECK_LAUNCH();
}

void launch_gat_rowdots(Ctx& c, const void* g, const void* out, bool out_f32, const void* Y, int64_t ld, int32_t d,
                        const float* el, const float* er, const float* m, const float* inv, float* cdot, float* selfds) {
    const int64_t n = c.plan.n_in;
    if (n <= 0) return;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 7) / 8, 148 * 16);
#define BNS_RD(T, F) pdl_launch(c.stream, k_gat_rowdots<T, F>, grid, 256, 0, (const T*)g, out, (const T*)Y, ld, n, d, el, er, m, inv, cdot, selfds)
    if (c.prec == BNS_BF16) { if (out_f32) BNS_RD(__nv_bfloat16, true); else BNS_RD(__nv_bfloat16, false); }
    else { if (out_f32) BNS_RD(float, true); else BNS_RD(float, false); }
#undef BNS_RD
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

void launch_gat_wsum(Ctx& c, int dir, const Seg* segs, int64_t n_segs, const int32_t* col, const int64_t* split,
                     int64_t n_split, const float* el, const float* er, const float* m, const float* inv,
                     const float* cdot, float* out) {
    if (n_segs <= 0) return;
    const unsigned grid = (unsigned)std::min<int64_t>((n_segs + 7) / 8, 148 * 16);
    if (dir == 0) pdl_launch(c.stream, k_gat_wsum<0>, grid, 256, 0, segs, n_segs, col, el, er, m, inv, cdot, c.d_partial, out);
    else pdl_launch(c.stream, k_gat_wsum<1>, grid, 256, 0, segs, n_segs, col, el, er, m, inv, cdot, c.d_partial, out);
    c.kernels += 1;
    if (n_split > 0) {
        pdl_launch(c.stream, k_gat_wsum_fix, (unsigned)((n_split + 127) / 128), 128, 0, segs, split, n_split, c.d_partial, out);
        c.kernels += 1;
    }
    BNS_CHECK_LAUNCH();
}

void launch_gat_final(Ctx& c, int dir, const void* own, const float* qp, int64_t ld, int32_t d, int64_t rows,
                      const float* cdot, const float* qr, const float* selfds, float* out) {
    if (rows <= 0) return;
    const unsigned grid = (unsigned)std::min<int64_t>((rows + 7) / 8, 148 * 16);
    const int64_t n_in = c.plan.n_in;
#define BNS_FIN(T, DIR) pdl_launch(c.stream, k_gat_final<T, DIR>, grid, 256, 0, (const T*)own, qp, ld, d, rows, n_in, cdot, qr, selfds, out)
    if (c.prec == BNS_BF16) { if (dir == 0) BNS_FIN(__nv_bfloat16, 0); else BNS_FIN(__nv_bfloat16, 1); }
    else { if (dir == 0) BNS_FIN(float, 0); else BNS_FIN(float, 1); }
#undef BNS_FIN
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

void launch_gat_da(Ctx& c, const void* Y, int64_t ld, int32_t d, const float* w, int64_t rows, float* out) {
    float* part = c.d_splitk;   // kDaBlocks x d floats (<= the split-K scratch)
    if (c.prec == BNS_BF16)
        pdl_launch(c.stream, k_gat_da1<__nv_bfloat16>, kDaBlocks, 256, 0, (const __nv_bfloat16*)Y, ld, d, w, rows, part);
    else
        pdl_launch(c.stream, k_gat_da1<float>, kDaBlocks, 256, 0, (const float*)Y, ld, d, w, rows, part);
    pdl_launch(c.stream, k_gat_da2, (unsigned)((d + 255) / 256), 256, 0, part, kDaBlocks, d, out);
    c.kernels += 2;
    BNS_CHECK_LAUNCH();
}

}  // namespace bns
