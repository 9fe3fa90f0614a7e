// gemm_simt.cu -- a7 / a9 dense update GEMMs, CUDA-core (SIMT) fp32-accumulate path.
//
// This is the fp32-accurate path of BNS_FP32 (R19: plain single-pass TF32 cannot meet 1e-5) and the generic
// fallback for shapes the tcgen05 kernel does not take.  The BNS_BF16 forward/backward GEMMs run on the tcgen05
// tensor cores (gemm_tc.cu).
//   fwd  Pre = [Z | H_in] W          (SAGE, CONCAT(z_v, h_v) PAPER.md:100) or Z W (GCN)
//   dW   = [Z | H_in]^T dPre          (split-K over the node dimension, partials reduced in fixed order)
//   dX   = dPre W^T, columns [0, d_in) scaled by the row's 1/deg_G (SAGE) or rs (GCN)
#include "common.h"
#include "dev.cuh"
#include "kernels.h"

namespace bns {

constexpr int BM = 64, BN = 64, BK = 16;

template <typename T> __device__ __forceinline__ float ld_f(const T* p) { return to_f<T>(*p); }

// MODE 0: fwd (A row-major with concat, B row-major K x N)
// MODE 1: wgrad (A^T: A is M x K row-major; B = D, M x N row-major)  -- tile over (K, N), reduction over M range
// MODE 2: dx (A = D, M x K row-major; B^T: B is Nc x K row-major)
template <typename T, typename TC, int MODE>
__global__ void __launch_bounds__(256) k_gemm(int64_t M, int64_t N, int64_t K, const T* __restrict__ A0,
                                              int64_t K0, int64_t lda0, const T* __restrict__ A1, int64_t lda1,
                                              const T* __restrict__ B, int64_t ldb, TC* __restrict__ C, int64_t ldc,
                                              bool relu, const float* __restrict__ rowscale, int64_t scale_cols,
                                              int64_t kchunk) {
    pdl_grid_sync();
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t i0 = (int64_t)blockIdx.y * BM, j0 = (int64_t)blockIdx.x * BN;
    int64_t k_begin = 0, k_end = K;
    if (MODE == 1) {
        k_begin = (int64_t)blockIdx.z * kchunk;
        k_end = (K < k_begin + kchunk) ? K : (k_begin + kchunk);
        C += (int64_t)blockIdx.z * M * ldc;   // partial slice
    }
    float acc[4][4] = {};
    for (int64_t kb = k_begin; kb < k_end; kb += BK) {
        // A tile -> As[k][i]
        for (int t = threadIdx.x; t < BK * BM; t += 256) {
            int kk, ii;
            float v = 0.f;
            if (MODE == 1) { ii = t % BM; kk = t / BM; }
            else { kk = t % BK; ii = t / BK; }
            const int64_t gi = i0 + ii, gk = kb + kk;
            if (gi < M && gk < k_end) {
                if (MODE == 0) v = (gk < K0) ? ld_f(A0 + gi * lda0 + gk) : ld_f(A1 + gi * lda1 + (gk - K0));
                else if (MODE == 1) v = ld_f(A0 + gk * lda0 + gi);
                else v = ld_f(A0 + gi * lda0 + gk);
            }
            As[kk][ii] = v;
        }
        // B tile -> Bs[k][j]
        for (int t = threadIdx.x; t < BK * BN; t += 256) {
            int kk, jj;
            float v = 0.f;
            if (MODE == 2) { kk = t % BK; jj = t / BK; }
            else { jj = t % BN; kk = t / BN; }
            const int64_t gj = j0 + jj, gk = kb + kk;
            if (gj < N && gk < k_end) {
                if (MODE == 2) v = ld_f(B + gj * ldb + gk);
                else v = ld_f(B + gk * ldb + gj);
            }
            Bs[kk][jj] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) { a[q] = As[kk][ty * 4 + q]; b[q] = Bs[kk][tx * 4 + q]; }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[q][r] = fmaf(a[q], b[r], acc[q][r]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t gi = i0 + ty * 4 + q;
        if (gi >= M) continue;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t gj = j0 + tx * 4 + r;
            if (gj >= N) continue;
            float v = acc[q][r];
            if (MODE == 0 && relu) v = v > 0.f ? v : 0.f;
            if (MODE == 2 && gj < scale_cols) v *= rowscale[gi];
            C[gi * ldc + gj] = from_f<TC>(v);
        }
    }
}

// fixed-order sum of the split-K partial slices (deterministic, depends only on S): a block covers 32 float4 output
// chunks (one per lane); warp g sums the g-th contiguous eighth of the slices in slice order -- all its loads in
// flight at once -- and warp 0 adds the eight group sums in group order.  (One thread summing all S slices was
// latency-bound: ~9 us per launch at m = 8 for a few MB.)
constexpr int kRedGroups = 8;
__global__ void __launch_bounds__(kRedGroups * 32) k_splitk_reduce(const float* __restrict__ part, int S, int64_t M,
                                                                  int64_t N, int64_t ldp, int64_t zs,
                                                                  int64_t gap_row, int64_t gap,
                                                                  float* __restrict__ out, int64_t ldo) {
    pdl_grid_sync();
    __shared__ float4 s_g[kRedGroups][32];
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int64_t n4 = N / 4;
    const int64_t t = (int64_t)blockIdx.x * 32 + lane;
    const bool live = t < M * n4;
    const int64_t i = live ? t / n4 : 0, j = live ? (t % n4) * 4 : 0;
    const float* p0 = part + (i < gap_row ? i : i + gap) * ldp + j;   // partial rows [gap_row, +gap) are padding
    const int per = (S + kRedGroups - 1) / kRedGroups;
    const int z0 = min(S, g * per), z1 = min(S, z0 + per);
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) {
        int z = z0;
        for (; z + 8 <= z1; z += 8) {
            float4 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldg(reinterpret_cast<const float4*>(p0 + (int64_t)(z + q) * zs));
#pragma unroll
            for (int q = 0; q < 8; ++q) { s.x += v[q].x; s.y += v[q].y; s.z += v[q].z; s.w += v[q].w; }
        }
        for (; z < z1; ++z) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(p0 + (int64_t)z * zs));
            s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
        }
    }
    s_g[g][lane] = s;
    __syncthreads();
    if (g != 0 || !live) return;
    float4 r = s_g[0][lane];
    for (int q = 1; q < kRedGroups; ++q) {
        const float4 v = s_g[q][lane];
        r.x += v.x; r.y += v.y; r.z += v.z; r.w += v.w;
    }
    *reinterpret_cast<float4*>(out + i * ldo + j) = r;
}

// several reductions in one launch: job q owns blocks [jb[q], jb[q + 1])
constexpr int kRedJobs = 8;
struct RedTable {
    int njobs;
    int64_t jb[kRedJobs + 1];
    const float* part[kRedJobs];
    int S[kRedJobs];
    int64_t M[kRedJobs], N[kRedJobs], zs[kRedJobs], gap_row[kRedJobs], gap[kRedJobs], ldo[kRedJobs];
    float* out[kRedJobs];
};
__global__ void __launch_bounds__(kRedGroups * 32) k_splitk_reduce_multi(const RedTable tb) {
    pdl_grid_sync();
    __shared__ float4 s_g[kRedGroups][32];
    int q = 0;
    while (q + 1 < tb.njobs && (int64_t)blockIdx.x >= tb.jb[q + 1]) ++q;
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int64_t N = tb.N[q], n4 = N / 4;
    const int S = tb.S[q];
    const int64_t t = ((int64_t)blockIdx.x - tb.jb[q]) * 32 + lane;
    const bool live = t < tb.M[q] * n4;
    const int64_t i = live ? t / n4 : 0, j = live ? (t % n4) * 4 : 0;
    const float* p0 = tb.part[q] + (i < tb.gap_row[q] ? i : i + tb.gap[q]) * N + j;
    const int64_t zs = tb.zs[q];
    const int per = (S + kRedGroups - 1) / kRedGroups;
    const int z0 = min(S, g * per), z1 = min(S, z0 + per);
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) {
        int z = z0;
        for (; z + 8 <= z1; z += 8) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(p0 + (int64_t)(z + u) * zs));
#pragma unroll
            for (int u = 0; u < 8; ++u) { s.x += v[u].x; s.y += v[u].y; s.z += v[u].z; s.w += v[u].w; }
        }
        for (; z < z1; ++z) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(p0 + (int64_t)z * zs));
            s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
        }
    }
    s_g[g][lane] = s;
    __syncthreads();
    if (g != 0 || !live) return;
    float4 r = s_g[0][lane];
    for (int u = 1; u < kRedGroups; ++u) {
        const float4 v = s_g[u][lane];
        r.x += v.x; r.y += v.y; r.z += v.z; r.w += v.w;
    }
    *reinterpret_cast<float4*>(tb.out[q] + i * tb.ldo[q] + j) = r;
}

void splitk_flush(Ctx& c) {
    if (c.red_jobs.empty()) {
        c.splitk_used = 0;
        return;
    }
    for (size_t q0 = 0; q0 < c.red_jobs.size(); q0 += kRedJobs) {
        RedTable tb{};
        tb.njobs = (int)std::min<size_t>(kRedJobs, c.red_jobs.size() - q0);
        int64_t nb = 0;
        for (int q = 0; q < tb.njobs; ++q) {
            const Ctx::RedJob& jb = c.red_jobs[q0 + q];
            tb.jb[q] = nb;
            tb.part[q] = jb.part; tb.S[q] = jb.S; tb.M[q] = jb.M; tb.N[q] = jb.N; tb.zs[q] = jb.zs;
            tb.gap_row[q] = jb.gap_row; tb.gap[q] = jb.gap; tb.out[q] = jb.out; tb.ldo[q] = jb.ldo;
            nb += (jb.M * jb.N / 4 + 31) / 32;
        }
        tb.jb[tb.njobs] = nb;
        pdl_launch(c.stream, k_splitk_reduce_multi, (unsigned)nb, kRedGroups * 32, 0, tb);
        c.kernels += 1;
        BNS_CHECK_LAUNCH();
    }
    c.red_jobs.clear();
    c.splitk_used = 0;
}

float* splitk_reserve(Ctx& c, int64_t floats) {
    if (!c.defer_red) return c.d_splitk;
    if (c.splitk_used + floats > c.splitk_cap) splitk_flush(c);
    return c.d_splitk + c.splitk_used;
}

void splitk_reduce(Ctx& c, int S, int64_t K, int64_t N, float* Wg, int64_t ldw, int64_t gap_row, int64_t gap) {
    if (c.defer_red) {   // the slices were written at d_splitk + splitk_used (splitk_reserve)
        Ctx::RedJob jb{c.d_splitk + c.splitk_used, S, K, N, (K + gap) * N, gap_row, gap, Wg, ldw};
        c.red_jobs.push_back(jb);
        c.splitk_used += (int64_t)S * (K + gap) * N;
        return;
    }
    const int64_t n4 = K * N / 4;
    pdl_launch(c.stream, k_splitk_reduce, (unsigned)((n4 + 31) / 32), kRedGroups * 32, 0, c.d_splitk, S, K, N, N, (K + gap) * N,
                                                                                   gap_row, gap, Wg, ldw);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

template <typename T>
static void fwd_t(Ctx& c, int64_t M, int64_t N, const void* A0, int64_t K0, int64_t lda0, const void* A1, int64_t K1,
                  int64_t lda1, const void* B, int64_t ldb, void* C, int64_t ldc, bool relu, bool out_f32) {
    dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
    const int64_t K = K0 + K1;
    if (out_f32)
        pdl_launch(c.stream, k_gemm<T, float, 0>, grid, 256, 0, M, N, K, (const T*)A0, K0, lda0, (const T*)A1, lda1,
                                                        (const T*)B, ldb, (float*)C, ldc, relu, nullptr, 0, 0);
    else
        pdl_launch(c.stream, k_gemm<T, T, 0>, grid, 256, 0, M, N, K, (const T*)A0, K0, lda0, (const T*)A1, lda1,
                                                    (const T*)B, ldb, (T*)C, ldc, relu, nullptr, 0, 0);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

void gemm_fwd(Ctx& c, int64_t M, int64_t N, const void* A0, int64_t K0, int64_t lda0, const void* A1, int64_t K1,
              int64_t lda1, const void* B, int64_t ldb, void* C, int64_t ldc, bool relu, bool out_f32) {
    if (M <= 0 || N <= 0) return;
    if (c.prec == BNS_BF16) fwd_t<__nv_bfloat16>(c, M, N, A0, K0, lda0, A1, K1, lda1, B, ldb, C, ldc, relu, out_f32);
    else fwd_t<float>(c, M, N, A0, K0, lda0, A1, K1, lda1, B, ldb, C, ldc, relu, out_f32);
}

template <typename T>
static void wgrad_t(Ctx& c, int64_t M, int64_t K, int64_t N, const void* A, int64_t lda, const void* D, int64_t ldd,
                    float* Wg, int64_t ldw) {
    // output (K x N); reduction over M in S fixed chunks
    const int64_t tiles = ((K + BM - 1) / BM) * ((N + BN - 1) / BN);
    int64_t S = std::max<int64_t>(1, std::min<int64_t>((296 + tiles - 1) / tiles, (M + 255) / 256));
    while (S > 1 && S * K * N > c.splitk_cap) --S;
    int64_t chunk = ((M + S - 1) / S + BK - 1) / BK * BK;
    S = (M + chunk - 1) / chunk;
    if (S < 1) S = 1;
    dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((K + BM - 1) / BM), (unsigned)S);
    pdl_launch(c.stream, k_gemm<T, float, 1>, grid, 256, 0, K, N, M, (const T*)A, 0, lda, nullptr, 0, (const T*)D, ldd,
                                                    c.d_splitk, N, false, nullptr, 0, chunk);
    int64_t tot = K * N;
    pdl_launch(c.stream, k_splitk_reduce, (unsigned)((tot / 4 + 31) / 32), kRedGroups * 32, 0, c.d_splitk, (int)S, K, N, N, tot,
                                                                                   INT64_MAX, 0, Wg, ldw);
    c.kernels += 2;
    BNS_CHECK_LAUNCH();
}

void gemm_wgrad(Ctx& c, int64_t M, int64_t K, int64_t N, const void* A, int64_t lda, const void* D, int64_t ldd,
                float* Wg, int64_t ldw) {
    if (K <= 0 || N <= 0) return;
    if (M <= 0) {
        for (int64_t i = 0; i < K; ++i) BNS_CUDA_HOLD(cudaMemsetAsync(Wg + i * ldw, 0, N * sizeof(float), c.stream));
        return;
    }
    if (c.prec == BNS_BF16) wgrad_t<__nv_bfloat16>(c, M, K, N, A, lda, D, ldd, Wg, ldw);
    else wgrad_t<float>(c, M, K, N, A, lda, D, ldd, Wg, ldw);
}

template <typename T>
static void dx_t(Ctx& c, int64_t M, int64_t Nc, int64_t K, const void* D, int64_t ldd, const void* B, int64_t ldb,
                 void* C, int64_t ldc, const float* rowscale, int64_t scale_cols) {
    dim3 grid((unsigned)((Nc + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
    pdl_launch(c.stream, k_gemm<T, T, 2>, grid, 256, 0, M, Nc, K, (const T*)D, K, ldd, nullptr, 0, (const T*)B, ldb, (T*)C, ldc,
                                                false, rowscale, scale_cols, 0);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

void gemm_dx(Ctx& c, int64_t M, int64_t Nc, int64_t K, const void* D, int64_t ldd, const void* B, int64_t ldb, void* C,
             int64_t ldc, const float* rowscale, int64_t scale_cols) {
    if (M <= 0 || Nc <= 0) return;
    if (c.prec == BNS_BF16) dx_t<__nv_bfloat16>(c, M, Nc, K, D, ldd, B, ldb, C, ldc, rowscale, scale_cols);
    else dx_t<float>(c, M, Nc, K, D, ldd, B, ldb, C, ldc, rowscale, scale_cols);
}

}  // namespace bns
