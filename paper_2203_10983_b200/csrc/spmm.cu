// spmm.cu -- a6 forward aggregation and a10 transposed aggregation (segment SpMM, HBM/L2-gather bound).
//
// Forward (Alg.1 l.10):
//   SAGE (R1-R3):  z_v = (1/deg_G(v)) Σ_{u ∈ N(v) ∩ (V_i ∪ U_i)} c_u h_u, c_u = 1 inner, 1/p halo
//   GCN  (App. A):   z_v = rs_v (Σ_u c_u rs_u h_u + rs_v h_v),   rs = 1/sqrt(deg_G + 1)
// Backward (transpose of the same sampled operator):
//   SAGE:  dX_u = c_u Σ_{v ∈ N(u) ∩ V_i} dZ'_v + [u inner] dXself_u     (dZ'_v = dZ_v / deg_G(v), GEMM epilogue)
//   GCN:   dX_u = c_u rs_u (Σ_{v ∈ N(u) ∩ V_i} dZ'_v + [u inner] dZ'_u)   (dZ'_v = rs_v dZ_v)
//
// Work unit = one warp per segment (<= kSeg edges of one output row, edges in CSR order).  Each lane owns VPL
// 16-byte vectors of the row (LPR lanes per row; with narrow rows the warp's 32/LPR lane groups take alternate
// edges and are reduced at the end).  Column indices are loaded 32 at a time and broadcast with shuffles; U edges
// are in flight per lane.  fp32 accumulation for both storage types.  Hub rows (deg > kSeg) are split into several
// segments whose fp32 partials are summed in segment order by k_spmm_fixup -- deterministic, and the split
// depends only on the row length.
#include "common.h"
#include "dev.cuh"
#include "kernels.h"

namespace bns {

template <typename T>
__device__ __forceinline__ void epilogue_store(const SpmmArgs& a, int64_t row, int vi, float* acc) {
    using V = Vec<T>;
    constexpr int VN = V::N;
    float rs;
    switch (a.mode) {
        case SAGE_FWD:
            rs = a.rowscale[row];
#pragma unroll
            for (int k = 0; k < VN; ++k) acc[k] *= rs;
            break;
        case GCN_FWD: {
            float f[VN];
            V::to_float(*reinterpret_cast<const typename V::raw*>(static_cast<const T*>(a.src) + row * a.ld_src + vi * VN), f);
            float cs = a.cscale[row];
            rs = a.rowscale[row];
#pragma unroll
            for (int k = 0; k < VN; ++k) acc[k] = (acc[k] + cs * f[k]) * rs;
            break;
        }
        case SAGE_BWD: {
            if (row < a.n_in) {
                float f[VN];
                V::to_float(*reinterpret_cast<const typename V::raw*>(static_cast<const T*>(a.self) + row * a.ld_self + vi * VN), f);
#pragma unroll
                for (int k = 0; k < VN; ++k) acc[k] += f[k];
            } else {
#pragma unroll
                for (int k = 0; k < VN; ++k) acc[k] *= a.inv_p;
            }
            break;
        }
        default: {  // GCN_BWD
            rs = a.cscale[row];
            if (row < a.n_in) {
                float f[VN];
                V::to_float(*reinterpret_cast<const typename V::raw*>(static_cast<const T*>(a.src) + row * a.ld_src + vi * VN), f);
#pragma unroll
                for (int k = 0; k < VN; ++k) acc[k] = (acc[k] + f[k]) * rs;
            } else {
#pragma unroll
                for (int k = 0; k < VN; ++k) acc[k] *= rs;
            }
            break;
        }
    }
    *reinterpret_cast<typename V::raw*>(static_cast<T*>(a.out) + row * a.ld_out + vi * VN) = V::from_float(acc);
}

template <typename T, int LPR, int VPL>
__global__ void __launch_bounds__(256) k_spmm(const SpmmArgs a) {
    using V = Vec<T>;
    using R = typename V::raw;
    constexpr int VN = V::N;
    constexpr int G = 32 / LPR;                              // edge groups per warp
    constexpr int U0 = (VPL <= 1) ? 4 : (VPL <= 2) ? 2 : 1;
    constexpr int U = (G * U0 > 32) ? (32 / G) : U0;         // edges in flight per group
    static_assert(32 % (G * U) == 0, "bad unroll");
    const int lane = threadIdx.x & 31, g = lane / LPR, l = lane % LPR;
    const int nvec = a.d / VN;
    const T* __restrict__ src = static_cast<const T*>(a.src);
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sid = warp; sid < a.n_segs; sid += nwarps) {
        const Seg s = a.segs[sid];
        float acc[VPL][VN];
#pragma unroll
        for (int v = 0; v < VPL; ++v)
#pragma unroll
            for (int k = 0; k < VN; ++k) acc[v][k] = 0.f;
        for (int64_t eb = s.e0; eb < s.e1; eb += 32) {
            const int cnt = (s.e1 - eb < 32) ? (int)(s.e1 - eb) : 32;
            int32_t ci = 0;
            float sc = 1.f;
            if (lane < cnt) {
                ci = a.col[eb + lane];
                if (a.mode == SAGE_FWD) sc = (ci >= a.n_in) ? a.inv_p : 1.f;
                else if (a.mode == GCN_FWD) sc = a.cscale[ci];
            }
            for (int j0 = 0; j0 < cnt; j0 += G * U) {
                R r[U][VPL];
                float sj[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = j0 + u * G + g;
                    const int32_t cj = __shfl_sync(0xffffffffu, ci, j);
                    sj[u] = __shfl_sync(0xffffffffu, sc, j);
                    const bool ok = j < cnt;
                    const R* rowp = reinterpret_cast<const R*>(src + (int64_t)cj * a.ld_src);
#pragma unroll
                    for (int v = 0; v < VPL; ++v) {
                        const int vi = l + v * LPR;
                        if (ok && vi < nvec) r[u][v] = ldg_nc(rowp + vi);
                        else r[u][v] = R{};
                    }
                    if (!ok) sj[u] = 0.f;
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int v = 0; v < VPL; ++v) V::add_scaled(acc[v], r[u][v], sj[u]);
            }
        }
        if (G > 1) {
#pragma unroll
            for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
                for (int v = 0; v < VPL; ++v)
#pragma unroll
                    for (int k = 0; k < VN; ++k) acc[v][k] += __shfl_xor_sync(0xffffffffu, acc[v][k], o);
        }
        if (g != 0) continue;
        if (s.nseg > 1) {
            float* pp = a.partial + sid * (int64_t)a.d;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int vi = l + v * LPR;
                if (vi < nvec)
#pragma unroll
                    for (int k = 0; k < VN; k += 4)
                        *reinterpret_cast<float4*>(pp + vi * VN + k) = make_float4(acc[v][k], acc[v][k + 1], acc[v][k + 2], acc[v][k + 3]);
            }
        } else {
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int vi = l + v * LPR;
                if (vi < nvec) epilogue_store<T>(a, s.row, vi, acc[v]);
            }
        }
    }
}

// Sum the partials of every split row in segment order, then the same epilogue.
template <typename T>
__global__ void __launch_bounds__(256) k_spmm_fixup(const SpmmArgs a) {
    using V = Vec<T>;
    constexpr int VN = V::N;
    const int lane = threadIdx.x & 31;
    const int nvec = a.d / VN;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sid = warp; sid < a.n_segs; sid += nwarps) {
        const Seg s = a.segs[sid];
        if (s.nseg <= 1 || sid != s.first) continue;
        for (int vi = lane; vi < nvec; vi += 32) {
            float acc[VN];
#pragma unroll
            for (int k = 0; k < VN; ++k) acc[k] = 0.f;
            for (int q = 0; q < s.nseg; ++q) {
                const float* pp = a.partial + (sid + q) * (int64_t)a.d + vi * VN;
#pragma unroll
                for (int k = 0; k < VN; ++k) acc[k] += pp[k];
            }
            epilogue_store<T>(a, s.row, vi, acc);
        }
    }
}

template <typename T, int LPR, int VPL>
static void go(Ctx& c, const SpmmArgs& a, unsigned grid) {
    k_spmm<T, LPR, VPL><<<grid, 256, 0, c.stream>>>(a);
}

template <typename T>
static void dispatch(Ctx& c, const SpmmArgs& a, unsigned grid) {
    const int nvec = a.d / Vec<T>::N;
    if (nvec >= 32) {
        const int vpl = (nvec + 31) / 32;
        switch (vpl) {
            case 1: go<T, 32, 1>(c, a, grid); return;
            case 2: go<T, 32, 2>(c, a, grid); return;
            case 3: go<T, 32, 3>(c, a, grid); return;
            case 4: go<T, 32, 4>(c, a, grid); return;
            case 5: go<T, 32, 5>(c, a, grid); return;
            case 6: go<T, 32, 6>(c, a, grid); return;
            case 7: case 8: go<T, 32, 8>(c, a, grid); return;
            case 9: case 10: case 11: case 12: go<T, 32, 12>(c, a, grid); return;
            case 13: case 14: case 15: case 16: go<T, 32, 16>(c, a, grid); return;
            default: throw Error(BNS_ERR_INVALID, "feature dim too large for the SpMM kernel");
        }
    }
    int lpr = 1;
    while (lpr * 2 <= nvec) lpr *= 2;
    const int vpl = (nvec + lpr - 1) / lpr;
#define BNS_SPMM_CASE(L)                                        \
    if (lpr == L) {                                             \
        if (vpl == 1) go<T, L, 1>(c, a, grid); else go<T, L, 2>(c, a, grid); \
        return;                                                 \
    }
    BNS_SPMM_CASE(16) BNS_SPMM_CASE(8) BNS_SPMM_CASE(4) BNS_SPMM_CASE(2) BNS_SPMM_CASE(1)
#undef BNS_SPMM_CASE
}

void launch_spmm(Ctx& c, const SpmmArgs& a) {
    if (a.n_segs <= 0) return;
    unsigned grid = (unsigned)std::min<int64_t>((a.n_segs + 7) / 8, 148 * 32);
    if (c.prec == BNS_BF16) dispatch<__nv_bfloat16>(c, a, grid);
    else dispatch<float>(c, a, grid);
    BNS_CHECK_LAUNCH();
    if (c.prec == BNS_BF16) k_spmm_fixup<__nv_bfloat16><<<grid, 256, 0, c.stream>>>(a);
    else k_spmm_fixup<float><<<grid, 256, 0, c.stream>>>(a);
    c.kernels += 2;
    BNS_CHECK_LAUNCH();
}

}  // namespace bns
