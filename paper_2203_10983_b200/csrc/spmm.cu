// spmm.cu -- a6 forward aggregation and a10 transposed aggregation (segment SpMM, HBM/L2-gather bound).
//
// Forward (Alg.1 l.10):
//   SAGE (R1-R3):  z_v = (1/deg_G(v)) Σ_{u ∈ N(v) ∩ (V_i ∪ U_i)} c_u h_u, c_u = 1 inner, 1/p halo
//   GCN  (App. A):   z_v = rs_v (Σ_u c_u rs_u h_u + rs_v h_v),   rs = 1/sqrt(deg_G + 1)
// Backward (transpose of the same sampled operator):
//   SAGE:  dX_u = c_u Σ_{v ∈ N(u) ∩ V_i} dZ'_v + [u inner] dXself_u     (dZ'_v = dZ_v / deg_G(v), GEMM epilogue)
//   GCN:   dX_u = c_u rs_u (Σ_{v ∈ N(u) ∩ V_i} dZ'_v + [u inner] dZ'_u)   (dZ'_v = rs_v dZ_v)
// Edge samplers (f3, R41): the CSR holds only the sampled arcs; BES carries 1/q as c_u of halo columns (like 1/p),
// DropEdge 1/q on every arc as nscale, applied to the neighbour sum before the self terms.
//
// Work unit = one warp per segment (<= kSeg edges of one output row, edges in CSR order).  Each lane owns VPL
// 16-byte vectors of the row (LPR lanes per row; with narrow rows the warp's 32/LPR lane groups take alternate
// edges and are reduced at the end).  Column indices are loaded 32 at a time and broadcast with shuffles; U edges
// are in flight per lane.  fp32 accumulation for both storage types.  Hub rows (deg > kSeg) are split into several
// segments whose fp32 partials are summed in segment order by k_spmm_fixup -- deterministic, and the split
// depends only on the row length.
#include <cstdlib>
#include <cstring>

#include <cuda.h>

#include "common.h"
#include "dev.cuh"
#include "kernels.h"

namespace bns {

// segments per dynamic claim: ~64 claims per warp over the launch, at least 1, at most 64 segments
static int claim_chunk(int64_t n_segs, int64_t warps) {
    static const int fixed = [] { const char* e = std::getenv("BNS_SPMM_CHUNK"); return e ? std::atoi(e) : 0; }();
    if (fixed > 0) return fixed;
    return (int)std::max<int64_t>(1, std::min<int64_t>(64, n_segs / std::max<int64_t>(1, warps * 64)));
}

template <typename T>
__device__ __forceinline__ void epilogue_store(const SpmmArgs& a, int64_t row, int vi, float* acc) {
    using V = Vec<T>;
    constexpr int VN = V::N;
    float rs;
    if (a.nscale != 1.f) {   // f3 DropEdge: 1/q on every sampled arc (R41), before the self terms
#pragma unroll
        for (int k = 0; k < VN; ++k) acc[k] *= a.nscale;
    }
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
        case SAGE_FWD_TF: {   // R42: pre_v = (1/deg_G(v)) Σ_u c_u Y_u + S_v, ReLU on hidden layers
            float f[VN];
            V::to_float(*reinterpret_cast<const typename V::raw*>(static_cast<const T*>(a.self) + row * a.ld_self + vi * VN), f);
            rs = a.rowscale[row];
#pragma unroll
            for (int k = 0; k < VN; ++k) {
                acc[k] = acc[k] * rs + f[k];
                if (a.relu) acc[k] = fmaxf(acc[k], 0.f);
            }
            if (a.out_f32) {
                float* o = static_cast<float*>(a.out) + row * a.ld_out + vi * VN;
#pragma unroll
                for (int k = 0; k < VN; k += 4) *reinterpret_cast<float4*>(o + k) = make_float4(acc[k], acc[k + 1], acc[k + 2], acc[k + 3]);
                return;
            }
            break;
        }
        case GAT_FWD: {   // R45: pre_v = Σ_u alpha_vu Y_u + alpha_vv Y_v, ReLU on hidden layers
            float f[VN];
            V::to_float(*reinterpret_cast<const typename V::raw*>(static_cast<const T*>(a.self) + row * a.ld_self + vi * VN), f);
            const float t = a.gat_el[row] + a.gat_er[row];
            const float av = expf((t > 0.f ? t : 0.2f * t) - a.gat_m[row]) * a.gat_inv[row];
#pragma unroll
            for (int k = 0; k < VN; ++k) {
                acc[k] = fmaf(av, f[k], acc[k]);
                if (a.relu) acc[k] = fmaxf(acc[k], 0.f);
            }
            if (a.out_f32) {
                float* o = static_cast<float*>(a.out) + row * a.ld_out + vi * VN;
#pragma unroll
                for (int k = 0; k < VN; k += 4) *reinterpret_cast<float4*>(o + k) = make_float4(acc[k], acc[k + 1], acc[k + 2], acc[k + 3]);
                return;
            }
            break;
        }
        case GAT_RAW: {
            float* o = static_cast<float*>(a.out) + row * a.ld_out + vi * VN;
#pragma unroll
            for (int k = 0; k < VN; k += 4) *reinterpret_cast<float4*>(o + k) = make_float4(acc[k], acc[k + 1], acc[k + 2], acc[k + 3]);
            return;
        }
        case GAT_BWD: {   // R45: dY_u = Σ_v alpha_vu g_v + [u inner] (alpha_uu g_u + del_u a_l) + der_u a_r
            const float dr = a.gat_der[row];
            if (row < a.n_in) {
                float f[VN];
                V::to_float(*reinterpret_cast<const typename V::raw*>(static_cast<const T*>(a.src) + row * a.ld_src + vi * VN), f);
                const float t = a.gat_el[row] + a.gat_er[row];
                const float au = expf((t > 0.f ? t : 0.2f * t) - a.gat_m[row]) * a.gat_inv[row];
                const float dl = a.gat_del[row];
#pragma unroll
                for (int k = 0; k < VN; ++k) acc[k] = fmaf(au, f[k], acc[k]) + dl * a.gat_al[vi * VN + k];
            }
#pragma unroll
            for (int k = 0; k < VN; ++k) acc[k] += dr * a.gat_ar[vi * VN + k];
            break;
        }
        case SAGE_BWD: {
            if (row < a.n_in) {
                if (!a.self) break;   // R42 backward: dY has no self term
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

// Sum the fp32 partials of a split row in segment order (the row's segments first .. first + nseg - 1), then the
// epilogue; all 32 lanes, one 16-byte vector each per step.  L2 loads (__ldcg): the partials were written by other
// SMs during this grid (fused path) or the previous one.  Shared by the fused path and k_spmm_fixup, so both give
// the same bits.
template <typename T>
__device__ __forceinline__ void split_sum_store(const SpmmArgs& a, int64_t first, int32_t row, int32_t nseg, int lane) {
    constexpr int VN = Vec<T>::N;
    const int nvec = a.d / VN;
    for (int vi = lane; vi < nvec; vi += 32) {
        float acc[VN];
#pragma unroll
        for (int k = 0; k < VN; ++k) acc[k] = 0.f;
        const float* pp = a.partial + first * (int64_t)a.d + vi * VN;
        int q = 0;
        // 4 segments' partials in flight (16-byte loads), still added in segment order
        for (; q + 4 <= nseg; q += 4) {
            float4 t[4][VN / 4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int k = 0; k < VN / 4; ++k)
                    t[j][k] = __ldcg(reinterpret_cast<const float4*>(pp + (int64_t)(q + j) * a.d + 4 * k));
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int k = 0; k < VN / 4; ++k) {
                    acc[4 * k] += t[j][k].x;
                    acc[4 * k + 1] += t[j][k].y;
                    acc[4 * k + 2] += t[j][k].z;
                    acc[4 * k + 3] += t[j][k].w;
                }
        }
        for (; q < nseg; ++q)
#pragma unroll
            for (int k = 0; k < VN / 4; ++k) {
                const float4 t = __ldcg(reinterpret_cast<const float4*>(pp + (int64_t)q * a.d + 4 * k));
                acc[4 * k] += t.x;
                acc[4 * k + 1] += t.y;
                acc[4 * k + 2] += t.z;
                acc[4 * k + 3] += t.w;
            }
        epilogue_store<T>(a, row, vi, acc);
    }
}

// Fused split-row fixup: after writing its partial, the warp counts itself in; the warp that finishes a row's
// last segment (in any order) sums all the row's partials in segment order and stores the row.  The counter is
// reset by that warp, so the next launch finds it zero.
template <typename T>
__device__ __forceinline__ void split_arrive(const SpmmArgs& a, const Seg& s, int lane) {
    __threadfence();   // this lane's partial is visible device-wide before the count
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomicAdd(a.arrive + s.first, 1) == s.nseg - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();   // every other segment's partial is visible to this warp
    if (lane == 0) a.arrive[s.first] = 0;
    split_sum_store<T>(a, s.first, s.row, s.nseg, lane);
}

// Dynamic scheduling epilogue: every warp counts itself out after its last (failed) claim; the last one resets the
// claim counter and the done counter for the next launch.
__device__ __forceinline__ void work_done(unsigned long long* work, int lane) {
    if (!work || lane != 0) return;
    const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    if (atomicAdd(work + 1, 1ull) == nw - 1) {
        atomicExch(work, 0ull);
        atomicExch(work + 1, 0ull);
    }
}

// SC 7 (bf16 rows, 1/p exact in bf16, e.g. p = 0.1, 0.01, 0.5): acc += s * x with x and s read as bf16 by the
// mixed-precision FMA (fma.rn.f32.bf16 -> FHFMA.BF16 on each packed half) -- the exact product rounded once, so
// bitwise the SC 1 result (FFMA2 of the widened value by the same fp32 scale), without the unpack
template <typename R>
__device__ __forceinline__ void acc_vec_bf16s(uint64_t* a, const R& v, uint32_t sbits) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float lo, hi;
        upk2(a[k], lo, hi);
        asm("{\n\t.reg .b16 l, h, sl, sh;\n\tmov.b32 {l, h}, %2;\n\tmov.b32 {sl, sh}, %3;\n\t"
            "fma.rn.f32.bf16 %0, l, sl, %0;\n\tfma.rn.f32.bf16 %1, h, sl, %1;\n\t}"
            : "+f"(lo), "+f"(hi) : "r"(w[k]), "r"(sbits));
        a[k] = pk2(lo, hi);
    }
}

// SC: per-edge column scale -- 0 none (backward modes, and the forward when every column has c_u = 1),
//     1 c_u = 1/p for halo columns (col >= n_in, SAGE forward), 2 c_u from cscale[] (GCN forward).
#ifndef BNS_SPMM_U1
#define BNS_SPMM_U1 8       // edges in flight per lane group for 1-vector rows
#endif
#ifndef BNS_SPMM_PREFETCH
#define BNS_SPMM_PREFETCH 1
#endif
#ifndef BNS_SPMM_MINB1
#define BNS_SPMM_MINB1 4    // resident 256-thread blocks per SM for 1-vector rows
#endif
#ifndef BNS_SPMM_MINB7
#define BNS_SPMM_MINB7 3    // ... with the bf16 1/p scale (SC 7)
#endif
template <typename T, int LPR, int VPL, int SC>
__global__ void __launch_bounds__(256, (VPL <= 1 && SC == 0) ? BNS_SPMM_MINB1 : (VPL <= 1 && SC == 7) ? BNS_SPMM_MINB7
                                         : (VPL <= 2) ? 3 : (VPL <= 6) ? 2 : 1)
k_spmm(const SpmmArgs a) {
    pdl_grid_sync();
    using V = Vec<T>;
    using R = typename V::raw;
    constexpr int VN = V::N;
    constexpr int G = 32 / LPR;                              // edge groups per warp
    constexpr int U0 = (VPL <= 1) ? BNS_SPMM_U1 : (VPL <= 2) ? 4 : (VPL <= 4) ? 2 : 1;
    constexpr int U = (G * U0 > 32) ? (32 / G) : U0;         // edges in flight per group
    static_assert(32 % (G * U) == 0, "bad unroll");
    const int lane = threadIdx.x & 31, g = lane / LPR, l = lane % LPR;
    const int nvec = a.d / VN;
    const char* __restrict__ base = reinterpret_cast<const char*>(static_cast<const R*>(a.src) + l);
    const uint32_t rvb = (uint32_t)(a.ld_src * sizeof(T));   // row pitch in bytes (32-bit multiply per edge)
    // lanes past the row end re-load the last vector (same address as a live lane: no extra sectors) and
    // accumulate into registers that are never stored -- no branches in the edge loop
    int voff[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) voff[v] = min(l + v * LPR, nvec - 1) - l;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // static: grid-stride over the segments; dynamic (a.work): each warp claims the next segment when it is done, so
    // a block never idles behind its longest segment (short partitions: ~1 segment per warp).  Claiming the next
    // segment ahead (atomic issued at segment start) was measured slower at m = 8 (2.05 vs 1.99 ms): rejected.
    // claims take a.chunk consecutive segments at once: with millions of 1-2 edge segments (C5) one atomic per
    // segment on one address serialised the whole kernel
    const int64_t chunk = a.work ? a.chunk : 1;
    auto claim = [&]() -> int64_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(a.work, (unsigned long long)chunk);
        return (int64_t)__shfl_sync(0xffffffffu, v, 0);
    };
    for (int64_t c0 = a.work ? claim() : warp; c0 < a.n_segs; c0 = a.work ? claim() : c0 + nwarps)
    for (int64_t vid = c0; vid < c0 + chunk && vid < a.n_segs; ++vid) {
        // claim order: the hub rows' segments first (placed at the end of the list, longest work first), then the
        // single-segment rows
        const int64_t sid = vid < a.hub_n ? a.hub_base + vid : vid - a.hub_n;
        const Seg s = a.segs[sid];
        uint64_t acc2[VPL][VN / 2];
#pragma unroll
        for (int v = 0; v < VPL; ++v)
#pragma unroll
            for (int k = 0; k < VN / 2; ++k) acc2[v][k] = 0ull;
#if BNS_SPMM_PREFETCH
        // the next chunk's 32 column indices are loaded while this chunk's rows are gathered (one dependent round
        // trip less per 32 edges: short rows / small partitions are latency-bound)
        int32_t ci_next = (lane < s.e1 - s.e0) ? a.col[s.e0 + lane] : 0;
#endif
        for (int64_t eb = s.e0; eb < s.e1; eb += 32) {
            const int cnt = (s.e1 - eb < 32) ? (int)(s.e1 - eb) : 32;
            int32_t ci = 0;
            float sc = 1.f;
#if BNS_SPMM_PREFETCH
            const int32_t ci_cur = ci_next;
            if (eb + 32 + lane < s.e1) ci_next = a.col[eb + 32 + lane];
#endif
            if (lane < cnt) {
#if BNS_SPMM_PREFETCH
                ci = ci_cur;
#else
                ci = a.col[eb + lane];
#endif
                if (SC == 1 || SC == 7) sc = (ci >= a.n_in) ? a.inv_p : 1.f;
                if (SC == 2) sc = a.cscale[ci];
                if (SC == 3) {   // GAT forward: alpha_vu, v = this row (R45)
                    const float t = a.gat_el[s.row] + a.gat_er[ci];
                    sc = expf((t > 0.f ? t : 0.2f * t) - a.gat_m[s.row]) * a.gat_inv[s.row];
                }
                if (SC == 4 || SC == 6) {   // GAT transposed: alpha_vu with v = the gathered row, u = this row
                    const float t = a.gat_el[ci] + a.gat_er[s.row];
                    sc = expf((t > 0.f ? t : 0.2f * t) - a.gat_m[ci]) * a.gat_inv[ci];
                    if (SC == 6) sc *= (t > 0.f ? 1.f : 0.2f);   // w_vu = alpha_vu LeakyReLU'(s_vu)
                }
                if (SC == 5) {   // GAT forward w_vu = alpha_vu LeakyReLU'(s_vu), v = this row
                    const float t = a.gat_el[s.row] + a.gat_er[ci];
                    sc = expf((t > 0.f ? t : 0.2f * t) - a.gat_m[s.row]) * a.gat_inv[s.row] * (t > 0.f ? 1.f : 0.2f);
                }
            }
            if (cnt == 32) {
                // full chunk: no bounds checks on the edges
#pragma unroll 1
                for (int j0 = 0; j0 < 32; j0 += G * U) {
                    R r[U][VPL];
                    uint64_t sj[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int j = j0 + u * G + g;
                        const uint32_t cj = (uint32_t)__shfl_sync(0xffffffffu, ci, j);
                        if (SC == 7) {   // the scale's bf16 bits (exact by construction of SC 7)
                            sj[u] = __shfl_sync(0xffffffffu, __float_as_uint(sc) >> 16, j);
                        } else if (SC) {
                            const float t = __shfl_sync(0xffffffffu, sc, j);
                            sj[u] = pk2(t, t);
                        }
                        const R* rowp = reinterpret_cast<const R*>(base + (uint64_t)cj * rvb);
#pragma unroll
                        for (int v = 0; v < VPL; ++v)
                            r[u][v] = ldg_nc(rowp + voff[v]);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int v = 0; v < VPL; ++v)
                            if (SC == 7) acc_vec_bf16s(acc2[v], r[u][v], (uint32_t)sj[u]);
                            else acc_vec2<T, SC != 0>(acc2[v], r[u][v], SC ? sj[u] : 0ull);
                }
            } else {
                // tail chunk (< 32 edges): one edge per lane group per step
                for (int j0 = 0; j0 < cnt; j0 += G) {
                    const int j = j0 + g;
                    const uint32_t cj = (uint32_t)__shfl_sync(0xffffffffu, ci, j & 31);
                    const float t = SC ? __shfl_sync(0xffffffffu, sc, j & 31) : 1.f;
                    if (j < cnt) {
                        const R* rowp = reinterpret_cast<const R*>(base + (uint64_t)cj * rvb);
#pragma unroll
                        for (int v = 0; v < VPL; ++v)
                            if (SC == 7) acc_vec_bf16s(acc2[v], ldg_nc(rowp + voff[v]), __float_as_uint(t) >> 16);
                            else acc_vec2<T, SC != 0>(acc2[v], ldg_nc(rowp + voff[v]), pk2(t, t));
                    }
                }
            }
        }
        float acc[VPL][VN];
#pragma unroll
        for (int v = 0; v < VPL; ++v)
#pragma unroll
            for (int k = 0; k < VN / 2; ++k) upk2(acc2[v][k], acc[v][2 * k], acc[v][2 * k + 1]);
        if (G > 1) {
#pragma unroll
            for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
                for (int v = 0; v < VPL; ++v)
#pragma unroll
                    for (int k = 0; k < VN; ++k) acc[v][k] += __shfl_xor_sync(0xffffffffu, acc[v][k], o);
        }
        if (s.nseg > 1) {
            if (g == 0) {
                float* pp = a.partial + sid * (int64_t)a.d;
#pragma unroll
                for (int v = 0; v < VPL; ++v) {
                    const int vi = l + v * LPR;
                    if (vi < nvec)
#pragma unroll
                        for (int k = 0; k < VN; k += 4)
                            *reinterpret_cast<float4*>(pp + vi * VN + k) = make_float4(acc[v][k], acc[v][k + 1], acc[v][k + 2], acc[v][k + 3]);
                }
            }
            if (a.arrive) split_arrive<T>(a, s, lane);
        } else if (g == 0) {
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int vi = l + v * LPR;
                if (vi < nvec) epilogue_store<T>(a, s.row, vi, acc[v]);
            }
        }
    }
    work_done(a.work, lane);
}

// ------------------------------------------------------------------------------------------------------------------
// A/B variant (BNS_SPMM_TMA=1; bf16 rows of 256 elements = 512 B, the hidden-layer gathers of the Reddit shape):
// the gathered rows are staged through shared memory by TMA (cp.async.bulk.tensor.2d.tile::gather4 -- four rows per
// instruction, named by their row indices) into a per-warp ring of G4_STAGES x 4 rows tracked by mbarriers; lane 0
// issues, all 32 lanes then read their 16-byte vector of each landed row from shared memory.  Same segments, same
// claiming, same per-lane edge order and arithmetic as k_spmm<bf16, 32, 1, SC>, so the results are bitwise equal.
// ------------------------------------------------------------------------------------------------------------------
constexpr int G4_STAGES = 4;
constexpr int G4_ROW_BYTES = 512;
constexpr int G4_WARP_BYTES = G4_STAGES * 4 * G4_ROW_BYTES;   // 8 KB per warp

__device__ __forceinline__ uint32_t g4_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int SC>
__global__ void __launch_bounds__(256, 3) k_spmm_g4(const __grid_constant__ CUtensorMap map, const SpmmArgs a) {
    pdl_grid_sync();
    extern __shared__ __align__(128) uint8_t g4_smem_raw[];
    __shared__ __align__(8) uint64_t bars[8][G4_STAGES];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint8_t* ring = g4_smem_raw + w * G4_WARP_BYTES;
    uint64_t* bar = bars[w];
    if (lane == 0) {
        for (int st = 0; st < G4_STAGES; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(g4_smem(&bar[st])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
    }
    __syncwarp();
    uint32_t cons = 0;   // groups consumed by this warp so far (stage = cons % G4_STAGES, parity = cons / G4_STAGES)
    auto issue = [&](int64_t e, int64_t e1, uint32_t idx) {   // lane 0: rows of edges e .. e + 3 into stage idx
        const int st = (int)(idx % G4_STAGES);
        int32_t r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) r[j] = a.col[(e + j < e1) ? e + j : e];   // pad with a row the group reads
        const uint32_t b = g4_smem(&bar[st]), dst = g4_smem(ring + st * 4 * G4_ROW_BYTES);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4 * G4_ROW_BYTES) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(dst), "l"(&map), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(b) : "memory");
    };
    auto claim = [&]() -> int64_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(a.work, (unsigned long long)a.chunk);
        return (int64_t)__shfl_sync(0xffffffffu, v, 0);
    };
    for (int64_t c0 = claim(); c0 < a.n_segs; c0 = claim())
    for (int64_t vid = c0; vid < c0 + a.chunk && vid < a.n_segs; ++vid) {
        const int64_t sid = vid < a.hub_n ? a.hub_base + vid : vid - a.hub_n;
        const Seg s = a.segs[sid];
        const int64_t ng = (s.e1 - s.e0 + 3) / 4;
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
        if (lane == 0)
            for (int64_t g = 0; g < ng && g < G4_STAGES; ++g) issue(s.e0 + 4 * g, s.e1, cons + (uint32_t)g);
        for (int64_t g = 0; g < ng; ++g, ++cons) {
            const int st = (int)(cons % G4_STAGES);
            const uint32_t par = (cons / G4_STAGES) & 1u;
            const int64_t e = s.e0 + 4 * g;
            const int cnt = (s.e1 - e < 4) ? (int)(s.e1 - e) : 4;
            float sc[4] = {1.f, 1.f, 1.f, 1.f};
            if (SC == 1)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j < cnt) sc[j] = (a.col[e + j] >= a.n_in) ? a.inv_p : 1.f;
            uint32_t done = 0;
            const uint32_t b = g4_smem(&bar[st]);
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(b), "r"(par) : "memory");
            const uint4* rows = reinterpret_cast<const uint4*>(ring + st * 4 * G4_ROW_BYTES);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < cnt) acc_vec2<__nv_bfloat16, SC != 0>(acc2, rows[j * 32 + lane], SC ? pk2(sc[j], sc[j]) : 0ull);
            __syncwarp();
            if (lane == 0 && g + G4_STAGES < ng) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // our reads before the TMA rewrite
                issue(s.e0 + 4 * (g + G4_STAGES), s.e1, cons + G4_STAGES);
            }
        }
        float acc[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) upk2(acc2[k], acc[2 * k], acc[2 * k + 1]);
        if (s.nseg > 1) {
            float* pp = a.partial + sid * (int64_t)a.d + lane * 8;
            *reinterpret_cast<float4*>(pp) = make_float4(acc[0], acc[1], acc[2], acc[3]);
            *reinterpret_cast<float4*>(pp + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
            if (a.arrive) split_arrive<__nv_bfloat16>(a, s, lane);
        } else {
            epilogue_store<__nv_bfloat16>(a, s.row, lane, acc);
        }
    }
    work_done(a.work, lane);
}

static bool spmm_tma() {
    static const bool v = [] { const char* e = std::getenv("BNS_SPMM_TMA"); return e && e[0] == '1'; }();
    return v;
}

typedef CUresult (*G4EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// the TMA path takes bf16 rows of exactly 256 elements, per-edge scale none or 1/p on halo columns
static bool launch_spmm_g4(Ctx& c, SpmmArgs a, int sc) {
    if (!spmm_tma() || c.prec != BNS_BF16 || a.d != 256 || (sc != 0 && sc != 1) || a.mode == GAT_FWD ||
        a.mode == GAT_BWD || a.mode == GAT_RAW)
        return false;
    static G4EncodeFn enc = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) p = nullptr;
        return reinterpret_cast<G4EncodeFn>(p);
    }();
    if (!enc) throw Error(BNS_ERR_RUNTIME, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap map;
    const int64_t rows = c.plan.n_in + c.halo_cap;
    cuuint64_t dims[2] = {(cuuint64_t)a.d, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(a.ld_src * 2)};
    cuuint32_t box[2] = {(cuuint32_t)a.d, 1u};
    cuuint32_t es[2] = {1u, 1u};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.src), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        throw Error(BNS_ERR_RUNTIME, "gather4 tensor map encode failed");
    const int smem = 8 * G4_WARP_BYTES;
    auto kern = sc ? k_spmm_g4<1> : k_spmm_g4<0>;
    static bool cfg0 = false, cfg1 = false;
    bool& cfg = sc ? cfg1 : cfg0;
    if (!cfg) {
        BNS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cfg = true;
    }
    int per_sm = 0;
    BNS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((a.n_segs + 7) / 8, (int64_t)std::max(1, per_sm) * sms));
    a.work = c.d_spmm_work;
    a.chunk = claim_chunk(a.n_segs, (int64_t)grid * 8);
    pdl_launch(c.stream, kern, grid, 256, smem, map, a);
    return true;
}

// Sum the partials of every split row in segment order, then the same epilogue.  (A block-per-row variant -- eight
// warps each summing an eighth of the segments -- measured slower: Reddit m = 1 22.7 -> 24.2 ms per epoch, m = 8
// rank 1.56 -> 1.66 ms; most split rows have few segments and the block's barrier and idle warps cost more than the
// hub rows' serial tail.)
template <typename T>
__global__ void __launch_bounds__(256) k_spmm_fixup(const SpmmArgs a) {
    pdl_grid_sync();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q0 = warp; q0 < a.n_split; q0 += nwarps) {
        const int64_t sid = a.split[q0];
        const Seg s = a.segs[sid];
        split_sum_store<T>(a, sid, s.row, s.nseg, lane);
    }
}

// BNS_SPMM_SCHED: 0 = grid-stride over min(n_segs / 8, 148 x 32) blocks; 1 = the same over one resident wave;
// 2 (default) = one resident wave, segments claimed dynamically (a.work)
static int spmm_sched() {
    static const int v = [] { const char* e = std::getenv("BNS_SPMM_SCHED"); return e ? std::atoi(e) : 2; }();
    return v;
}

static int resident_per_gpu(const void* kern) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, 0) != cudaSuccess || b < 1) b = 1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return b * sms;
}

template <typename T, int LPR, int VPL, int SC>
static void go_sc(Ctx& c, SpmmArgs a, unsigned grid) {
    auto kern = k_spmm<T, LPR, VPL, SC>;
    static const int wave = resident_per_gpu((const void*)kern);   // per kernel instance (thread-safe init)
    if (spmm_sched() != 0) grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((a.n_segs + 7) / 8, wave));
    if (spmm_sched() == 2) {
        a.work = c.d_spmm_work;
        a.chunk = claim_chunk(a.n_segs, (int64_t)grid * 8);
    } else {
        a.work = nullptr;
    }
    pdl_launch(c.stream, kern, grid, 256, 0, a);
}

template <typename T, int LPR, int VPL>
static void go(Ctx& c, const SpmmArgs& a, unsigned grid) {
    // per-edge column scale needed?  SAGE forward only when halo columns carry 1/p != 1
    int sc = 0;
    if (a.sc >= 0) sc = a.sc;
    else if (a.mode == GCN_FWD) sc = 2;
    else if ((a.mode == SAGE_FWD || a.mode == SAGE_FWD_TF) && a.inv_p != 1.f) sc = 1;
    if (LPR == 32 && VPL == 1 && launch_spmm_g4(c, a, sc)) return;
    uint32_t ib;
    std::memcpy(&ib, &a.inv_p, 4);
    if constexpr (sizeof(T) == 2) {
        if (sc == 1 && (ib & 0xffffu) == 0u) {   // 1/p exact in bf16: SC 7 (the same bits as SC 1)
            go_sc<T, LPR, VPL, 7>(c, a, grid);
            return;
        }
    }
    if (sc == 0) go_sc<T, LPR, VPL, 0>(c, a, grid);
    else if (sc == 1) go_sc<T, LPR, VPL, 1>(c, a, grid);
    else if (sc == 2) go_sc<T, LPR, VPL, 2>(c, a, grid);
    else if (sc == 3) go_sc<T, LPR, VPL, 3>(c, a, grid);
    else if (sc == 4) go_sc<T, LPR, VPL, 4>(c, a, grid);
    else if (sc == 5) go_sc<T, LPR, VPL, 5>(c, a, grid);
    else go_sc<T, LPR, VPL, 6>(c, a, grid);
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
    // rows narrower than a warp: one vector per lane and the next power of two of lanes per edge (idle lanes re-load
    // the last vector: no extra sectors).  Measured on the Reddit shape (48 bf16 = 6 vectors): 8 x 1 beats 4 x 2
    // (-0.3 ms per pass: fewer registers, more edges in flight) and 2 x 3 (+0.3 ms).  BNS_SPMM_LANES=0: 4 x 2 style.
    static const int pow2up = [] { const char* e = std::getenv("BNS_SPMM_LANES"); return e ? std::atoi(e) : 1; }();
    if (pow2up) {
        int l2 = 1;
        while (l2 < nvec) l2 *= 2;
        switch (l2) {
            case 1: go<T, 1, 1>(c, a, grid); return;
            case 2: go<T, 2, 1>(c, a, grid); return;
            case 4: go<T, 4, 1>(c, a, grid); return;
            case 8: go<T, 8, 1>(c, a, grid); return;
            case 16: go<T, 16, 1>(c, a, grid); return;
            default: break;
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

// Feature-dimension tiling: when the gathered rows (n_in + |U| rows x d) exceed an L2 budget, the aggregation is
// run as several passes over column tiles of 512 bytes per row, each with an L2-resident working set (the column
// indices are re-read per pass: 4 B per edge against 512 B of row data).
constexpr int64_t kL2Budget = 96ll << 20;

void launch_spmm(Ctx& c, const SpmmArgs& a0) {
    if (a0.n_segs <= 0) return;
    const int64_t ts = c.prec == BNS_BF16 ? 2 : 4;
    const int64_t rows = c.plan.n_in + c.n_halo;
    int64_t tile = a0.d;
    if (rows * a0.d * ts > kL2Budget) {
        static const int mode = [] { const char* e = std::getenv("BNS_SPMM_TILE"); return e ? std::atoi(e) : 0; }();
        if (mode == 0) {
            tile = std::min<int64_t>(a0.d, 512 / ts);                      // 512-byte tiles
        } else if (mode == 2 || mode == 3) {                               // balanced tiles of <= / >= 512 bytes
            const int64_t nt = mode == 2 ? (a0.d * ts + 511) / 512 : std::max<int64_t>(1, a0.d * ts / 512);
            tile = ((a0.d + nt - 1) / nt + 7) / 8 * 8;
        } else {
            const int64_t nt = (rows * a0.d * ts + kL2Budget - 1) / kL2Budget;   // balanced tiles
            tile = ((a0.d + nt - 1) / nt + 7) / 8 * 8;
        }
    }
    unsigned grid = (unsigned)std::min<int64_t>((a0.n_segs + 7) / 8, 148 * 32);
    // split rows summed inside the SpMM by the warp finishing their last segment (no fixup launch) on jobs without
    // long segments (R37: their hub rows have few 256-edge partials); large jobs keep the separate fixup pass, where
    // one warp summing a hub row's hundreds of partials would be a serial tail.  BNS_SPMM_FUSE=0/1 forces it.
    static const int fuse_env = [] { const char* e = std::getenv("BNS_SPMM_FUSE"); return e ? std::atoi(e) : -1; }();
    const bool fuse = a0.n_split > 0 && (fuse_env >= 0 ? fuse_env == 1 : c.seg_long == 0);
    for (int64_t c0 = 0; c0 < a0.d; c0 += tile) {
        SpmmArgs a = a0;
        a.arrive = fuse ? c.d_spmm_arrive : nullptr;
        a.d = (int32_t)std::min<int64_t>(tile, a0.d - c0);
        a.src = static_cast<const char*>(a0.src) + c0 * ts;
        a.out = static_cast<char*>(a0.out) + c0 * ((a0.out_f32 || a0.mode == GAT_RAW) ? 4 : ts);
        if (a0.self) a.self = static_cast<const char*>(a0.self) + c0 * ts;
        if (a0.gat_al) a.gat_al = a0.gat_al + c0;
        if (a0.gat_ar) a.gat_ar = a0.gat_ar + c0;
        if (c.prec == BNS_BF16) dispatch<__nv_bfloat16>(c, a, grid);
        else dispatch<float>(c, a, grid);
        c.kernels += 1;
        BNS_CHECK_LAUNCH();
        if (a.n_split > 0 && !fuse) {   // only the split (hub) rows, listed by their first segment
            const unsigned fg = (unsigned)std::min<int64_t>((a.n_split + 7) / 8, 148 * 8);
            if (c.prec == BNS_BF16) pdl_launch(c.stream, k_spmm_fixup<__nv_bfloat16>, fg, 256, 0, a);
            else pdl_launch(c.stream, k_spmm_fixup<float>, fg, 256, 0, a);
            c.kernels += 1;
            BNS_CHECK_LAUNCH();
        }
    }
}

}  // namespace bns
