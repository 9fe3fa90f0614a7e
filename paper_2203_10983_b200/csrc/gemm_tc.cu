// gemm_tc.cu -- a7 / a9 dense update on the 5th-generation tensor cores (tcgen05).
//
// The update φ(z_v, h_v) = σ(W · CONCAT(z_v, h_v)) is the only true contraction on the path:
//   fwd  Pre[n_in x d_out] = [Z | H] · W              A K-major (two tensor maps, concat along K), B = W^T K-major
//   dW   dW[d_in x d_out]  = Z^T · dPre (and H^T ·)   A and B MN-major (the node dimension is the reduction),
//                                                     split-K over nodes, fp32 partials reduced in fixed order
//   dX   [dZ'|dXself]      = dPre · W^T               A K-major, B = W K-major; epilogue x 1/deg_G (or rs) on dZ'
//
// Two precisions, one kernel template:
//   BNS_BF16  kind::f16 with bf16 operands (R19), 64-element (128 B) k-blocks, 4-stage ring.
//   BNS_FP32  split TF32 (kind::tf32): every fp32 operand tile is split in shared memory into hi = x rounded to
//             tf32 (exactly representable) and lo = (x - hi) rounded to tf32, and the tile product is accumulated as
//             hi·hi + hi·lo + lo·hi + lo·lo in fp32 TMEM -- what is dropped is lo's rounding residual, <= 2^-22 |x|
//             per operand, so each product is within ~2^-21 relative and the GEMM meets the fp32 mode's 1e-5 (plain
//             1xTF32 would not; the 3-term form without lo·lo and with the tensor core's own
//             tf32 conversion of lo measured 1.2e-5 on a cancellation-heavy last-layer dW).  32-element (128 B)
//             k-blocks, 2-stage ring of [hi | lo] tiles; four more warps do the split between the TMA landing and the
//             MMA issue.
// Both element types use the same byte layout (128 B SWIZZLE_128B rows, 32 B per K-major MMA k-step).  The fp32
// weight gradient (whose operands are MN-major: the node dimension is the reduction) runs K-major on transposed
// copies made by k_transpose32 (one extra read + write of the two operands); MN-major tf32 operands need the
// SWIZZLE_128B variant with 32-byte atoms (TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) -- not used here.
//
// One CTA = one 128 x BN output tile (BN <= 256): warp 0 lane 0 issues TMA into an mbarrier ring, warp 1 lane 0
// issues tcgen05.mma.cta_group::1 (M=128, N=BN, fp32 accumulator in TMEM) and releases stages with tcgen05.commit;
// warps 2-5 drain TMEM with tcgen05.ld.32x32b and apply the epilogue (ReLU / cast / row scale); fp32: warps 6-9 split
// the operands.  K tails and partial M / N tiles are handled by TMA's zero fill and masked stores.
#include <cuda.h>
#include <cstdint>

#include "common.h"
#include "dev.cuh"
#include "kernels.h"

namespace bns {

constexpr int TC_BM = 128;
constexpr int TC_ROW_BYTES = 128;                          // one SWIZZLE_128B row: 64 bf16 or 32 fp32 k-elements
constexpr int TC_A_BYTES = TC_BM * TC_ROW_BYTES;           // 16 KB
constexpr int TC_B_BYTES = 256 * TC_ROW_BYTES;             // 32 KB (max BN)
constexpr int TC_HALF_BYTES = TC_A_BYTES + TC_B_BYTES;     // one [A | B] operand pair
template <bool F32> struct TcCfg {
    static constexpr int STAGES = F32 ? 2 : 4;
    static constexpr int STAGE_BYTES = (F32 ? 2 : 1) * TC_HALF_BYTES;   // fp32: [A hi | B hi | A lo | B lo]
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
    static constexpr int THREADS = F32 ? 320 : 192;
    static constexpr int KE = F32 ? 32 : 64;               // k-elements per block (one 128 B row)
    static constexpr int MNE = F32 ? 32 : 64;              // MN-elements per 128 B row (MN-major operands)
};

enum TcEpi { EPI_BF16 = 0, EPI_F32 = 1, EPI_BF16_ROWSCALE = 2, EPI_F32_ROWSCALE = 3 };

struct TcArgs {
    int64_t M, N;
    int BN;                 // MMA N (multiple of 16; multiple of 64 when B is MN-major)
    int nk0, nk;            // k-blocks from map A0, total k-blocks
    int kb_per_split;       // k-blocks per blockIdx.z (split-K), 0 = all
    int epi;
    int relu;
    void* out;
    int64_t ldc;
    int64_t split_stride;   // elements between split-K partial slices
    const float* rowscale;
    int64_t scale_cols;
    int64_t msplit = INT64_MAX;   // MN-major A: output rows >= msplit come from map A1 (row m - msplit)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t a = smem_u32(b);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// the same box written into the smem of every CTA in ctamask (same offset), complete_tx on each CTA's mbarrier at the
// same offset
__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                               uint16_t ctamask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(ctamask)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);   // version 1, SWIZZLE_128B
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// arrive on the mbarrier at this offset in every CTA of ctamask once the issued MMAs have completed
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t ctamask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(bar)), "h"(ctamask) : "memory");
}

// Persistent, warp-specialized: grid = min(#tiles, #SMs); tile t = (m-tile, n-tile, split) visited in
// blockIdx-strided order.  warp 0 lane 0: TMA producer over the smem ring; warp 1 lane 0: MMA issuer into one of two
// TMEM accumulators (2 x 256 columns), so the epilogue of tile i overlaps the MMAs of tile i+1; warps 2-5: epilogue
// (warp w drains TMEM lanes 32*(w%4) .. +31); fp32 (split-TF32 (4 MMAs)): warps 6-9 split each landed stage into hi / lo.
// MC = 2 (bf16): clusters of two CTAs own consecutive 128-row tiles of the same output columns and split-K range;
// each CTA loads its own A tile and HALF of the shared B tile, written into both CTAs' shared memory by TMA multicast
// (B traffic from L2 halved); a stage is refilled only when both CTAs' MMAs have released it (the MMA commit arrives
// on the empty barrier of both CTAs).
template <bool A_MN, bool B_MN, bool F32, int MC = 1>
__global__ void __launch_bounds__(TcCfg<F32>::THREADS, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapA1,
          const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapB1, const TcArgs args) {
    using Cfg = TcCfg<F32>;
    constexpr int STAGES = Cfg::STAGES, STAGE_BYTES = Cfg::STAGE_BYTES, KE = Cfg::KE, MNE = Cfg::MNE;
    constexpr int BOX_BYTES = KE * TC_ROW_BYTES;          // one MN-major box {MNE, KE}: 8 KB bf16, 4 KB fp32
    constexpr int KSTEP_MN = (F32 ? 8 : 16) * TC_ROW_BYTES;   // MN-major: k-rows per MMA k-step x 128 B
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* conv = full + STAGES;           // fp32: stage split into hi / lo (MMA waits on this instead of full)
    uint64_t* empty = conv + STAGES;
    uint64_t* tfull = empty + STAGES;         // [2] accumulator ready
    uint64_t* tempty = tfull + 2;             // [2] accumulator drained (4 epilogue warps arrive)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = MC == 2 ? cluster_ctarank() : 0u;
    const int64_t tiles_m = (args.M + TC_BM - 1) / TC_BM;
    const int64_t tiles_mu = (tiles_m + MC - 1) / MC;   // m units: tiles (MC 1) or tile pairs (MC 2)
    const int64_t tiles_n = (args.N + args.BN - 1) / args.BN;
    const int splits = args.kb_per_split > 0 ? (args.nk + args.kb_per_split - 1) / args.kb_per_split : 1;
    const int64_t tiles = tiles_mu * tiles_n * splits;
    const int64_t t_first = MC == 2 ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
    const int64_t t_step = MC == 2 ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;
    auto decode = [&](int64_t t, int64_t& m0, int64_t& n0, int& z, int& kb0, int& nk) {
        z = (int)(t / (tiles_mu * tiles_n));
        const int64_t r = t % (tiles_mu * tiles_n);
        m0 = ((r % tiles_mu) * MC + crank) * TC_BM;   // MC 2: the pair's second tile may lie past M (zero-filled)
        n0 = (r / tiles_mu) * args.BN;
        kb0 = args.kb_per_split > 0 ? z * args.kb_per_split : 0;
        const int kb1 = args.kb_per_split > 0 ? min(args.nk, kb0 + args.kb_per_split) : args.nk;
        nk = kb1 - kb0;    // >= 1 by construction of the split count
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&conv[s], 1); mbar_init(&empty[s], MC); }
        for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA0) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA1) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB1) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (MC == 2) cluster_sync_all();   // the peer's barriers are initialised before any multicast reaches them
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // PDL: barrier init, descriptor prefetch and the TMEM allocation above overlap the previous kernel's tail; no
    // global memory is touched before this point
    pdl_grid_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t b_bytes = (uint32_t)args.BN * TC_ROW_BYTES;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            int s = 0;
            uint32_t ph = 0;
            for (int64_t t = t_first; t < tiles; t += t_step) {
                int64_t m0, n0;
                int z, kb0, nk;
                decode(t, m0, n0, z, kb0, nk);
                for (int i = 0; i < nk; ++i) {
                    mbar_wait(&empty[s], ph ^ 1u);
                    uint8_t* sa = smem + s * STAGE_BYTES;
                    uint8_t* sb = sa + TC_A_BYTES;
                    mbar_expect_tx(&full[s], TC_A_BYTES + b_bytes);
                    const int kb = kb0 + i;
                    if (!A_MN) {
                        // A K-major: box {KE (k), 128 (m)}; concat along K: blocks [0, nk0) from A0, the rest from A1
                        if (kb < args.nk0) tma_load_2d(&mapA0, &full[s], sa, kb * KE, (int)m0);
                        else tma_load_2d(&mapA1, &full[s], sa, (kb - args.nk0) * KE, (int)m0);
                    } else {
                        // A MN-major (A^T stored row-major as [k][m]): 128 / MNE boxes {MNE (m), KE (k)}; output rows
                        // past msplit read the second operand (two dW GEMMs sharing D in one launch)
                        const bool second = m0 >= args.msplit;
                        const CUtensorMap* ma = second ? &mapA1 : &mapA0;
                        const int mm = (int)(second ? m0 - args.msplit : m0);
#pragma unroll
                        for (int j = 0; j < TC_BM / MNE; ++j)
                            tma_load_2d(ma, &full[s], sa + j * BOX_BYTES, mm + MNE * j, kb * KE);
                    }
                    // output rows past msplit also take their B operand from mapB1 (a pair of dW GEMMs with
                    // different A and D in one launch)
                    const CUtensorMap* mb = m0 >= args.msplit ? &mapB1 : &mapB;
                    if (MC == 2) {   // this CTA's half of B, multicast into both CTAs of the pair
                        if (!B_MN) {   // box {KE (k), BN / 2 (n)}
                            const int hb = args.BN >> 1;
                            tma_load_2d_mc(mb, &full[s], sb + crank * hb * TC_ROW_BYTES, kb * KE, (int)n0 + (int)crank * hb,
                                           (uint16_t)3);
                        } else {
                            for (int j = (int)crank; j < args.BN / MNE; j += 2)
                                tma_load_2d_mc(mb, &full[s], sb + j * BOX_BYTES, (int)n0 + MNE * j, kb * KE, (uint16_t)3);
                        }
                    } else if (!B_MN) {
                        tma_load_2d(mb, &full[s], sb, kb * KE, (int)n0);              // box {KE (k), BN (n)}
                    } else {
                        for (int j = 0; j < args.BN / MNE; ++j)                        // boxes {MNE (n), KE (k)}
                            tma_load_2d(mb, &full[s], sb + j * BOX_BYTES, (int)n0 + MNE * j, kb * KE);
                    }
                    if (++s == STAGES) { s = 0; ph ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer ----------------
            // instruction descriptor: D fp32, A/B bf16 (1) or tf32 (2), A/B major, N >> 3, M >> 4
            constexpr uint32_t fmt = F32 ? 2u : 1u;
            const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((A_MN ? 1u : 0u) << 15) |
                                   ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(args.BN >> 3) << 17) |
                                   ((uint32_t)(TC_BM >> 4) << 24);
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (int64_t t = t_first; t < tiles; t += t_step, ++it) {
                int64_t m0, n0;
                int z, kb0, nk;
                decode(t, m0, n0, z, kb0, nk);
                const int b = it & 1;
                mbar_wait(&tempty[b], (((uint32_t)it >> 1) & 1u) ^ 1u);   // accumulator b drained by the epilogue
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + (uint32_t)(b * 256);
                for (int i = 0; i < nk; ++i) {
                    mbar_wait(F32 ? &conv[s] : &full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
                    const uint32_t sb = sa + TC_A_BYTES;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        // K-major SW128: +32 B per k step (16 bf16 / 8 tf32) inside the 128 B row; SBO = 8 rows (1 KB)
                        // MN-major SW128: +KSTEP_MN per k step; LBO = MN-atom (box) stride, SBO = 8 k-rows
                        const uint64_t ad = A_MN ? umma_desc(sa + k * KSTEP_MN, BOX_BYTES, 1024)
                                                 : umma_desc(sa + k * 32, 16, 1024);
                        const uint64_t bd = B_MN ? umma_desc(sb + k * KSTEP_MN, BOX_BYTES, 1024)
                                                 : umma_desc(sb + k * 32, 16, 1024);
                        if (!F32) {
                            umma_bf16(d, ad, bd, idesc, (i > 0 || k > 0) ? 1u : 0u);
                        } else {
                            // hi·hi into the hi accumulator (columns [0, 128) of the buffer), hi·lo + lo·hi + lo·lo
                            // into the lo accumulator ([128, 256)); lo tiles sit one [A | B] pair further
                            constexpr uint64_t lo = (uint64_t)(TC_HALF_BYTES >> 4);   // descriptor start-address units
                            const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
                            umma_tf32(d, ad, bd, idesc, acc);
                            umma_tf32(d + 128, ad, bd + lo, idesc, acc);
                            umma_tf32(d + 128, ad + lo, bd, idesc, 1u);
                            umma_tf32(d + 128, ad + lo, bd + lo, idesc, 1u);
                        }
                    }
                    if (MC == 2) umma_commit_mc(&empty[s], (uint16_t)3);   // both CTAs' stage s: B came from both
                    else umma_commit(&empty[s]);     // stage free once these MMAs have read it
                    if (++s == STAGES) { s = 0; ph ^= 1u; }
                }
                umma_commit(&tfull[b]);         // accumulator b complete
            }
        }
    } else if (F32 && warp >= 6) {
        // ---------------- split-TF32 operands (warps 6..9): hi = x rounded to tf32 (11 significant bits, ties away
        // from zero; exactly representable), lo = x - hi (exact in fp32, |lo| <= 2^-11 |x|) rounded to tf32 -------
        // elementwise on the raw stage bytes, so the swizzled layout carries over to the lo tiles unchanged
        const int ct = threadIdx.x - 192;
        int s = 0;
        uint32_t ph = 0;
        for (int64_t t = t_first; t < tiles; t += t_step) {
            int64_t m0, n0;
            int z, kb0, nk;
            decode(t, m0, n0, z, kb0, nk);
            for (int i = 0; i < nk; ++i) {
                mbar_wait(&full[s], ph);
                uint8_t* st = smem + s * STAGE_BYTES;
                const int nvec = (TC_A_BYTES + (int)b_bytes) / 16;
                for (int v = ct; v < nvec; v += 128) {
                    uint4* p = reinterpret_cast<uint4*>(st) + v;
                    uint4 x = *p, h, l;
                    h.x = (x.x + 0x1000u) & 0xFFFFE000u; h.y = (x.y + 0x1000u) & 0xFFFFE000u;
                    h.z = (x.z + 0x1000u) & 0xFFFFE000u; h.w = (x.w + 0x1000u) & 0xFFFFE000u;
                    // lo rounded to tf32 as well, so the tensor core's own tf32 conversion changes nothing
                    l.x = (__float_as_uint(__uint_as_float(x.x) - __uint_as_float(h.x)) + 0x1000u) & 0xFFFFE000u;
                    l.y = (__float_as_uint(__uint_as_float(x.y) - __uint_as_float(h.y)) + 0x1000u) & 0xFFFFE000u;
                    l.z = (__float_as_uint(__uint_as_float(x.z) - __uint_as_float(h.z)) + 0x1000u) & 0xFFFFE000u;
                    l.w = (__float_as_uint(__uint_as_float(x.w) - __uint_as_float(h.w)) + 0x1000u) & 0xFFFFE000u;
                    *p = h;
                    *reinterpret_cast<uint4*>(st + TC_HALF_BYTES + 16 * v) = l;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor-core reads
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (ct == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&conv[s])) : "memory");
                if (++s == STAGES) { s = 0; ph ^= 1u; }
            }
        }
    } else {
        // ---------------- epilogue: TMEM -> registers -> global (warps 2..5) ----------------
        const int q = warp & 3;                 // TMEM lane quarter this warp may access
        int it = 0;
        for (int64_t t = t_first; t < tiles; t += t_step, ++it) {
            int64_t m0, n0;
            int z, kb0, nk;
            decode(t, m0, n0, z, kb0, nk);
            const int b = it & 1;
            mbar_wait(&tfull[b], ((uint32_t)it >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int64_t row = m0 + q * 32 + lane;
            const int ncols = (args.N - n0 < args.BN) ? (int)(args.N - n0) : args.BN;
            const bool rsc = args.epi == EPI_BF16_ROWSCALE || args.epi == EPI_F32_ROWSCALE;
            const float rs = (rsc && row < args.M) ? args.rowscale[row] : 1.f;
            for (int c0 = 0; c0 < ncols; c0 += 16) {
                uint32_t r[16];
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * 256 + c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                float v[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r[k]);
                if (F32) {   // + the lo accumulator, 128 columns further (fp32 round-to-nearest add)
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                        : "r"(taddr + 128u));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int k = 0; k < 16; ++k) v[k] += __uint_as_float(r[k]);
                }
                if (row >= args.M) continue;
                const int64_t col = n0 + c0;
                if (rsc)
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        if (col + k < args.scale_cols) v[k] *= rs;
                if (args.relu)
#pragma unroll
                    for (int k = 0; k < 16; ++k) v[k] = fmaxf(v[k], 0.f);
                if (args.epi == EPI_F32 || args.epi == EPI_F32_ROWSCALE) {
                    float* o = static_cast<float*>(args.out) + (int64_t)z * args.split_stride + row * args.ldc + col;
#pragma unroll
                    for (int h = 0; h < 4; ++h)
                        if (c0 + 4 * h < ncols)
                            *reinterpret_cast<float4*>(o + 4 * h) = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2],
                                                                                v[4 * h + 3]);
                } else {
                    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(args.out) + row * args.ldc + col;
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if (c0 + 8 * h < ncols) *reinterpret_cast<uint4*>(o + 8 * h) = Vec<__nv_bfloat16>::from_float(v + 8 * h);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[b])) : "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (MC == 2) cluster_sync_all();   // no multicast write or commit arrival is still headed for either CTA
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        BNS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw Error(BNS_ERR_RUNTIME, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D row-major tensor [outer][inner] (bf16 or fp32) with row pitch ld (elements); box {one 128 B row of inner
// elements, box_outer}, SWIZZLE_128B
static CUtensorMap make_map(const void* base, int64_t inner, int64_t outer, int64_t ld, int box_outer, bool f32) {
    CUtensorMap m;
    const int es_bytes = f32 ? 4 : 2;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * es_bytes)};
    cuuint32_t box[2] = {(cuuint32_t)(TC_ROW_BYTES / es_bytes), (cuuint32_t)box_outer};
    cuuint32_t es[2] = {1u, 1u};
    CUresult r = encode_fn()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                             const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(BNS_ERR_RUNTIME, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

template <bool A_MN, bool B_MN, bool F32, int MC>
static void launch_tc_t(Ctx& c, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b,
                        const CUtensorMap& b1, const TcArgs& args, dim3 grid) {
    using Cfg = TcCfg<F32>;
    auto kern = k_gemm_tc<A_MN, B_MN, F32, MC>;
    static bool configured = false;
    if (!configured) {
        BNS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
        configured = true;
    }
    if (MC == 1) {
        pdl_launch(c.stream, kern, grid, Cfg::THREADS, Cfg::SMEM, a0, a1, b, b1, args);
    } else {   // CTA pairs: cluster dimension 2 (+ PDL as every other launch)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(Cfg::THREADS);
        cfg.dynamicSmemBytes = Cfg::SMEM;
        cfg.stream = c.stream;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = (!pdl_take_hold() && pdl_enabled()) ? 2 : 1;
        BNS_CUDA(cudaLaunchKernelEx(&cfg, kern, a0, a1, b, b1, args));
    }
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

template <bool A_MN, bool B_MN>
static void launch_tc(Ctx& c, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b, const TcArgs& args,
                      dim3 grid, const CUtensorMap* b1 = nullptr, int mc = 1) {
    if (c.prec == BNS_FP32) launch_tc_t<A_MN, B_MN, true, 1>(c, a0, a1, b, b1 ? *b1 : b, args, grid);
    else if (mc == 2) launch_tc_t<A_MN, B_MN, false, 2>(c, a0, a1, b, b1 ? *b1 : b, args, grid);
    else launch_tc_t<A_MN, B_MN, false, 1>(c, a0, a1, b, b1 ? *b1 : b, args, grid);
}

// bf16 GEMMs run as CTA pairs sharing the B operand when the node dimension is large (`rows`: the output rows of the
// forward / dX GEMMs, the reduction length of dW) and the shared operand is wide (`width`: the reduction length K of
// the forward / dX GEMMs, the output rows of dW).  Measured (A/B in one run): Yelp m = 1 (717 K rows, K = 1024)
// GEMMs 8.69 -> 8.40 ms; Reddit m = 1 (233 K) unchanged; products m = 1 (2.4 M rows, K <= 256) 3.28 -> 4.06 ms;
// the m = 8 rank (32-50 K rows) 0.270 -> 0.278 ms backward.  BNS_GEMM_MC = 0: never, 2: always (M > 128).
static int gemm_mc(const Ctx& c, int64_t M, int64_t rows, int64_t width) {
    const char* e = std::getenv("BNS_GEMM_MC");   // read per call: tests switch it
    const int env = e ? std::atoi(e) : 1;
    if (env == 0 || c.prec == BNS_FP32 || M <= 128) return 1;
    return (env == 2 || (rows >= (1ll << 18) && width >= 512)) ? 2 : 1;
}
// persistent grid of CTA pairs over tile pairs
static dim3 pair_grid(const Ctx& c, int64_t pairs) {
    return dim3((unsigned)(2 * std::max<int64_t>(1, std::min<int64_t>(pairs, c.num_sms / 2))));
}

static inline bool is_f32(const Ctx& c) { return c.prec == BNS_FP32; }
static inline int k_elems(const Ctx& c) { return is_f32(c) ? 32 : 64; }   // k-elements per block (128 B row)

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

static dim3 persistent_grid(int64_t tiles) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        BNS_CUDA(cudaGetDevice(&dev));
        BNS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, sms)));
}

// fwd: C[M x N] = [A0 | A1] · W, B = W^T stored [N][Kw] (Kw = 64-padded per concat half)
void gemm_fwd_tc(Ctx& c, int64_t M, int64_t N, const void* A0, int64_t K0, int64_t lda0, const void* A1, int64_t K1,
                 int64_t lda1, const void* WT, int64_t Kw, void* C, int64_t ldc, bool relu, bool out_f32) {
    if (M <= 0 || N <= 0) return;
    const bool f32 = is_f32(c);
    const int KE = k_elems(c);
    TcArgs a{};
    a.M = M;
    a.N = N;
    a.BN = (int)std::min<int64_t>(f32 ? 128 : 256, cdiv(N, 16) * 16);   // fp32: [hi | lo] accumulators of 128 columns
    // A1's k-blocks start where W^T's second concat half starts: each half is padded to a multiple of 64
    a.nk0 = A1 ? (int)(cdiv(K0, 64) * 64 / KE) : (int)cdiv(K0, KE);
    a.nk = a.nk0 + (int)cdiv(K1, KE);
    a.epi = (out_f32 || f32) ? EPI_F32 : EPI_BF16;
    a.relu = relu ? 1 : 0;
    a.out = C;
    a.ldc = ldc;
    const int mc = gemm_mc(c, M, M, K0 + K1);
    CUtensorMap m0 = make_map(A0, K0, M, lda0, TC_BM, f32);
    CUtensorMap m1 = A1 ? make_map(A1, K1, M, lda1, TC_BM, f32) : m0;
    CUtensorMap mb = make_map(WT, Kw, N, Kw, a.BN / mc, f32);   // MC 2: each CTA of a pair loads half of B
    launch_tc<false, false>(c, m0, m1, mb, a,
                            mc == 2 ? pair_grid(c, cdiv(cdiv(M, TC_BM), 2) * cdiv(N, a.BN))
                                    : persistent_grid(cdiv(M, TC_BM) * cdiv(N, a.BN)),
                            nullptr, mc);
}

// fp32 weight gradient: out^T operands.  dst[c][r] = src[r][c] for r < rows (the node dimension), c < cols;
// dst row pitch ldd >= rows (padded to 4 floats for TMA); 32 x 32 tiles through shared memory
__global__ void k_transpose32(const float* __restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                              float* __restrict__ dst, int64_t ldd) {
    pdl_grid_sync();
    __shared__ float t[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        t[i][threadIdx.x] = (r < rows && c < cols) ? src[r * lds + c] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (c < cols && r < ldd) dst[c * ldd + r] = t[threadIdx.x][i];
    }
}

static void transpose32(Ctx& c, const void* src, int64_t rows, int64_t cols, int64_t lds, float* dst, int64_t ldd) {
    const dim3 grid((unsigned)cdiv(ldd, 32), (unsigned)cdiv(cols, 32));
    pdl_launch(c.stream, k_transpose32, grid, dim3(32, 8), 0, static_cast<const float*>(src), rows, cols, lds, dst, ldd);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// fp32 (split-TF32 (4 MMAs)) dW: [A0 | A1]^T D as a K-major GEMM of the transposed operands, split-K over nodes, fixed-order reduce
static void wgrad_f32(Ctx& c, int64_t Mn, int64_t K, int64_t N, const void* A0, const void* A1, int64_t lda,
                      const void* D, int64_t ldd, float* Wg, int64_t ldw) {
    const int64_t halves = A1 ? 2 : 1, K2 = halves * K, ldt = (Mn + 3) / 4 * 4;
    if ((K2 + N) * ldt > c.tr_cap)
        throw Error(BNS_ERR_RUNTIME, "fp32 weight-gradient transpose scratch too small");
    float* At = c.d_tr;                        // [K2][ldt]
    float* Dt = c.d_tr + K2 * ldt;             // [N][ldt]
    transpose32(c, A0, Mn, K, lda, At, ldt);
    if (A1) transpose32(c, A1, Mn, K, lda, At + K * ldt, ldt);
    transpose32(c, D, Mn, N, ldd, Dt, ldt);
    TcArgs a{};
    a.M = K2;
    a.N = N;
    a.BN = (int)std::min<int64_t>(128, cdiv(N, 16) * 16);
    a.nk = (int)cdiv(Mn, 32);
    a.nk0 = a.nk;
    const int64_t tiles = cdiv(K2, TC_BM) * cdiv(N, a.BN);
    // the tensor core's fp32 accumulation loses accuracy with the length of the accumulation chain (measured: the
    // error grows linearly with the k-blocks per split, 2e-5 .. 6e-5 at 100 .. 250 blocks): at most kF32Chain
    // 32-node k-blocks per split, the fixed-order split-K reduce then adds the partials in IEEE fp32
    constexpr int kF32Chain = 16;
    int64_t S = std::max<int64_t>(cdiv(a.nk, kF32Chain), std::min<int64_t>(cdiv(148, tiles), std::max(1, a.nk / 32)));
    if (S * K2 * N > c.splitk_cap) throw Error(BNS_ERR_RUNTIME, "fp32 split-K partial buffer too small");
    a.kb_per_split = (int)cdiv(a.nk, S);
    S = cdiv(a.nk, a.kb_per_split);
    c.last_splitk = (int)S;
    a.epi = EPI_F32;
    a.out = c.d_splitk;
    a.ldc = N;
    a.split_stride = K2 * N;
    CUtensorMap ma = make_map(At, ldt, K2, ldt, TC_BM, true);
    CUtensorMap mb = make_map(Dt, ldt, N, ldt, a.BN, true);
    launch_tc<false, false>(c, ma, ma, mb, a, persistent_grid(tiles * S));
    splitk_reduce(c, (int)S, K2, N, Wg, ldw);
}

// dW partials: out[z][K x N] = A^T · D over k-block range z; A is [M_nodes][K] row-major, D is [M_nodes][N]
void gemm_wgrad_tc(Ctx& c, int64_t Mn, int64_t K, int64_t N, const void* A, int64_t lda, const void* D, int64_t ldd,
                   float* Wg, int64_t ldw) {
    if (K <= 0 || N <= 0) return;
    const bool f32 = is_f32(c);
    if (f32) return wgrad_f32(c, Mn, K, N, A, nullptr, lda, D, ldd, Wg, ldw);
    const int KE = k_elems(c);
    TcArgs a{};
    a.M = K;
    a.N = N;
    a.BN = (int)std::min<int64_t>(256, cdiv(N, 64) * 64);
    a.nk = (int)cdiv(Mn, KE);
    a.nk0 = a.nk;
    const int64_t tiles = cdiv(K, TC_BM) * cdiv(N, a.BN);
    // ~one CTA per SM, but at least 1024 nodes (kmin k-blocks of 64 bf16 / 32 fp32 nodes) per split so the partial
    // slices stay small.  16 x 64 (was 32 x 64; A/B at m = 8: gemm_bwd 0.355 -> 0.344 ms): small partitions get ~2x
    // the CTAs
    static const int kmin0 = [] { const char* e = std::getenv("BNS_WGRAD_KMIN"); return e ? std::max(1, std::atoi(e)) : 16; }();
    const int kmin = kmin0 * 64 / KE;
    int64_t S = std::max<int64_t>(1, std::min<int64_t>(cdiv(148, tiles), std::max(1, a.nk / kmin)));
    while (S > 1 && S * K * N > c.splitk_cap) --S;
    a.kb_per_split = (int)cdiv(a.nk, S);
    S = cdiv(a.nk, a.kb_per_split);
    c.last_splitk = (int)S;
    a.epi = EPI_F32;
    a.out = splitk_reserve(c, S * K * N);
    a.ldc = N;
    a.split_stride = K * N;
    CUtensorMap ma = make_map(A, K, Mn, lda, KE, f32);
    CUtensorMap mb = make_map(D, N, Mn, ldd, KE, f32);
    const int mc = gemm_mc(c, K, Mn, K);
    launch_tc<true, true>(c, ma, ma, mb, a,
                          mc == 2 ? pair_grid(c, cdiv(cdiv(K, TC_BM), 2) * cdiv(N, a.BN) * S)
                                  : persistent_grid(cdiv(K, TC_BM) * cdiv(N, a.BN) * S),
                          nullptr, mc);
    splitk_reduce(c, (int)S, K, N, Wg, ldw);
}

// [dW_0 ; dW_1] = [A0^T D0 ; A1^T D1] in one launch + one split-K reduce: output rows [0, K) from (A0, D0) over Mn0
// nodes, rows [K, 2K) from (A1, D1) over Mn1 nodes (Wg rows contiguous).  The second product starts at the 128-row
// tile boundary Kp >= K; the node range is max(Mn0, Mn1) and the TMA zero-fills the rows past each operand's own
// count.  Uses: the GraphSAGE dW_z / dW_h pair (D1 = D0, Mn1 = Mn0) and the transform-first dW_top / dW_bot pair
// (R42: D0 = dY over every stacked row, D1 = dPre over the inner rows).
void gemm_wgrad2_tc(Ctx& c, int64_t Mn0, int64_t Mn1, int64_t K, int64_t N, const void* A0, const void* A1,
                    int64_t lda, const void* D0, int64_t ldd0, const void* D1, int64_t ldd1, float* Wg, int64_t ldw) {
    if (N <= 0 || K <= 0) return;
    const bool f32 = is_f32(c);
    if (f32 && D1 == D0 && Mn1 == Mn0) return wgrad_f32(c, Mn0, K, N, A0, A1, lda, D0, ldd0, Wg, ldw);
    if (f32) {
        gemm_wgrad_tc(c, Mn0, K, N, A0, lda, D0, ldd0, Wg, ldw);
        gemm_wgrad_tc(c, Mn1, K, N, A1, lda, D1, ldd1, Wg + K * ldw, ldw);
        return;
    }
    const int KE = k_elems(c);
    // the second product starts on a tile boundary -- a tile-PAIR boundary for CTA pairs, whose two tiles must read
    // the same B operand
    // (no pairs where the pair boundary would add a padding tile)
    const int mc = ((K + TC_BM - 1) / TC_BM) % 2 == 0 ? gemm_mc(c, 2 * K, std::max(Mn0, Mn1), 2 * K) : 1;
    const int64_t Kp = cdiv(K, TC_BM * mc) * TC_BM * mc, M2 = Kp + K;
    const int64_t Mn = std::max(Mn0, Mn1);
    if (Mn <= 0) {
        BNS_CUDA_HOLD(cudaMemset2DAsync(Wg, ldw * sizeof(float), 0, N * sizeof(float), 2 * K, c.stream));
        return;
    }
    TcArgs a{};
    a.M = M2;
    a.N = N;
    a.BN = (int)std::min<int64_t>(256, cdiv(N, 64) * 64);
    a.nk = (int)cdiv(Mn, KE);
    a.nk0 = a.nk;
    a.msplit = Kp;
    const int64_t tiles = cdiv(M2, TC_BM) * cdiv(N, a.BN);
    static const int kmin0 = [] { const char* e = std::getenv("BNS_WGRAD_KMIN"); return e ? std::max(1, std::atoi(e)) : 16; }();
    const int kmin = kmin0 * 64 / KE;
    int64_t S = std::max<int64_t>(1, std::min<int64_t>(cdiv(148, tiles), std::max(1, a.nk / kmin)));
    while (S > 1 && S * M2 * N > c.splitk_cap) --S;
    if (M2 * N > c.splitk_cap) {   // cannot happen with the setup sizing; keep the two-launch form as the guard
        gemm_wgrad_tc(c, Mn0, K, N, A0, lda, D0, ldd0, Wg, ldw);
        gemm_wgrad_tc(c, Mn1, K, N, A1, lda, D1, ldd1, Wg + K * ldw, ldw);
        return;
    }
    a.kb_per_split = (int)cdiv(a.nk, S);
    S = cdiv(a.nk, a.kb_per_split);
    c.last_splitk = (int)S;
    a.epi = EPI_F32;
    a.out = splitk_reserve(c, S * M2 * N);
    a.ldc = N;
    a.split_stride = M2 * N;
    CUtensorMap m0 = make_map(A0, K, std::max<int64_t>(Mn0, 1), lda, KE, f32);
    CUtensorMap m1 = make_map(A1, K, std::max<int64_t>(Mn1, 1), lda, KE, f32);
    CUtensorMap mb0 = make_map(D0, N, std::max<int64_t>(Mn0, 1), ldd0, KE, f32);
    CUtensorMap mb1 = make_map(D1, N, std::max<int64_t>(Mn1, 1), ldd1, KE, f32);
    launch_tc<true, true>(c, m0, m1, mb0, a,
                          mc == 2 ? pair_grid(c, cdiv(cdiv(M2, TC_BM), 2) * cdiv(N, a.BN) * S) : persistent_grid(tiles * S),
                          &mb1, mc);
    splitk_reduce(c, (int)S, 2 * K, N, Wg, ldw, K, Kp - K);
}

// dX: C[M x Nc] = D[M x K] · B^T with B = W [Nc][K] row-major; columns < scale_cols scaled by rowscale[row]
void gemm_dx_tc(Ctx& c, int64_t M, int64_t Nc, int64_t K, const void* D, int64_t ldd, const void* B, int64_t ldb,
                void* C, int64_t ldc, const float* rowscale, int64_t scale_cols) {
    if (M <= 0 || Nc <= 0) return;
    const bool f32 = is_f32(c);
    TcArgs a{};
    a.M = M;
    a.N = Nc;
    a.BN = (int)std::min<int64_t>(f32 ? 128 : 256, cdiv(Nc, 16) * 16);
    a.nk = (int)cdiv(K, k_elems(c));
    a.nk0 = a.nk;
    a.epi = f32 ? (rowscale ? EPI_F32_ROWSCALE : EPI_F32) : (rowscale ? EPI_BF16_ROWSCALE : EPI_BF16);
    a.out = C;
    a.ldc = ldc;
    a.rowscale = rowscale;
    a.scale_cols = scale_cols;
    const int mc = gemm_mc(c, M, M, K);
    CUtensorMap ma = make_map(D, K, M, ldd, TC_BM, f32);
    CUtensorMap mb = make_map(B, K, Nc, ldb, a.BN / mc, f32);
    launch_tc<false, false>(c, ma, ma, mb, a,
                            mc == 2 ? pair_grid(c, cdiv(cdiv(M, TC_BM), 2) * cdiv(Nc, a.BN))
                                    : persistent_grid(cdiv(M, TC_BM) * cdiv(Nc, a.BN)),
                            nullptr, mc);
}

}  // namespace bns
