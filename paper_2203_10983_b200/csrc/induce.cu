// induce.cu -- a1 + a2 + a3 of the BNS draw in three single-pass kernels (decoupled look-back scans):
//
//   k_sample_fused   Alg.1 l.4 (R5-R7, R23): the Philox Bernoulli draw of every candidate, the
//                    order-preserving compaction into [U_i ; S_{i,*}] (Alg.1 l.6-7, R24, R27), the boundary keep
//                    bitmask the induce pass tests against, slot_of_b and the 2m+1 segment offsets (per-peer counts).
//   k_induce_count / k_induce_scatter   Alg.1 l.5: the node-induced subgraph on V_i ∪ U_i -- keep
//                    bit of every static arc (inner columns always, boundary columns by the bitmask), then the kept
//                    columns scattered in global neighbour order and remapped to halo rows n_in + slot, and the
//                    induced row pointers (two independent passes: per-tile counts, then prefix + scatter).
//   k_segs_fused     SpMM work lists: forward segments of the induced rows and backward (transposed) segments of the
//                    sampled halo rows, both chains in one launch, split (hub) rows appended for the fixup.
//
// The draw and the segment lists are one pass over their tiles (a few hundred): a tile publishes its aggregate, looks back over its predecessors' published
// aggregates / inclusive prefixes (a warp reads 32 predecessors at a time), and then writes its outputs at their final
// positions.  Tiles are handed out in launch order by an atomic counter (a tile only waits on tiles that already
// started, so the look-back cannot deadlock); the tile states carry a launch generation, so nothing is cleared between
// launches.  Results are bitwise those of the multi-pass version (count -> scan -> scatter): positions are exact
// prefix sums.
#include "common.h"
#include "dev.cuh"
#include "kernels.h"

namespace bns {

namespace {

constexpr int kTile = 1024;          // candidates / rows / halo slots per tile (one per thread)
constexpr int kEdgeThreads = kInduceTileArcs / 32;   // induce: one 32-arc word per thread
constexpr uint64_t kValMask = (1ull << 38) - 1;
enum { LB_NONE = 0, LB_AGG = 1, LB_PREFIX = 2 };

__device__ __forceinline__ uint64_t lb_pack(uint32_t gen, int flag, int64_t v) {
    return ((uint64_t)(gen & 0xFFFFFFu) << 40) | ((uint64_t)flag << 38) | ((uint64_t)v & kValMask);
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// tile id in launch order; the block that draws the last id resets the counter for the next launch
__device__ __forceinline__ int64_t next_tile(unsigned* ctr, int64_t ntiles, int64_t* s_tile) {
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(ctr, 1u);
        if ((int64_t)t == ntiles - 1) atomicExch(ctr, 0u);
        *s_tile = t;
    }
    __syncthreads();
    return *s_tile;
}

// exclusive prefix of tile t with aggregate agg (every thread passes the same agg); all threads get the result
__device__ int64_t lookback(uint64_t* state, uint32_t gen, int64_t t, int64_t agg, int64_t* s_excl) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const uint32_t g = gen & 0xFFFFFFu;
        int64_t excl = 0;
        if (t > 0) {
            if (lane == 0) st_release(state + t, lb_pack(gen, LB_AGG, agg));
            int64_t p = t - 1;
            for (;;) {
                const int64_t q = p - lane;
                const uint64_t s = q >= 0 ? ld_acquire(state + q) : lb_pack(gen, LB_PREFIX, 0);
                const int flag = (int)((s >> 38) & 3u);
                const bool ready = (uint32_t)(s >> 40) == g && flag != LB_NONE;
                if (!__all_sync(0xffffffffu, ready)) {   // back off: hundreds of warps poll the same few lines
                    __nanosleep(64);
                    continue;
                }
                const unsigned pm = __ballot_sync(0xffffffffu, flag == LB_PREFIX);
                const int upto = pm ? __ffs(pm) - 1 : 31;
                int64_t x = lane <= upto ? (int64_t)(s & kValMask) : 0;
#pragma unroll
                for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                excl += x;
                if (pm) break;
                p -= 32;
            }
        }
        if (lane == 0) {
            st_release(state + t, lb_pack(gen, LB_PREFIX, excl + agg));
            *s_excl = excl;
        }
    }
    __syncthreads();
    return *s_excl;
}

// block-wide exclusive scan of one int per thread (blockDim.x <= 1024); returns the thread's exclusive prefix, the
// block total in *s_total
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int* s_total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < nw ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        s_warp[lane] = s;
        if (lane == 31) *s_total = s;
    }
    __syncthreads();
    return (w ? s_warp[w - 1] : 0) + x - v;
}

struct SampleArgs {
    const int32_t* gid; const int32_t* key; const int32_t* payload; int64_t n, n_bd;
    uint64_t T; uint32_t e_lo, e_hi, s_lo, s_hi;
    const int64_t* cand_seg; int nseg;
    uint8_t* flags; uint32_t* bkeep; int32_t* out; int32_t* slot_of_b; int64_t* seg_pos;
    int64_t* zero; int nzero;                     // counters the later passes add to (split-list lengths)
    uint64_t* state; unsigned* ctr; uint32_t gen; int64_t ntiles;
};

__global__ void __launch_bounds__(kTile) k_sample_fused(const SampleArgs a) {
    pdl_grid_sync();
    __shared__ int64_t s_tile, s_excl;
    __shared__ int s_warp[32], s_total;
    const int64_t t = next_tile(a.ctr, a.ntiles, &s_tile);
    const int64_t i = t * kTile + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int keep = 0;
    if (i < a.n) {
        const uint32_t r = philox4((uint32_t)a.gid[i], (uint32_t)a.key[i], a.e_lo, a.e_hi, a.s_lo, a.s_hi).x;
        keep = ((uint64_t)r < a.T) ? 1 : 0;
        a.flags[i] = (uint8_t)keep;
    }
    // boundary keep bitmask (bit b of word b / 32 = keep(B_i[b], i)) for the induce pass
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int64_t i0 = i - lane;
    if (lane == 0 && i0 < a.n_bd) {
        const int64_t valid = a.n_bd - i0;
        a.bkeep[i0 >> 5] = valid >= 32 ? bal : (bal & ((1u << valid) - 1u));
    }
    if (t == 0 && threadIdx.x < a.nzero) a.zero[threadIdx.x] = 0;
    const int ex = block_excl_scan(keep, s_warp, &s_total);
    const int64_t excl = lookback(a.state, a.gen, t, s_total, &s_excl);
    const int64_t pos = excl + ex;
    if (i < a.n) {
        if (keep) a.out[pos] = a.payload[i];
        if (i < a.n_bd) a.slot_of_b[a.payload[i]] = keep ? (int32_t)pos : -1;
        for (int k = 0; k < a.nseg; ++k)
            if (a.cand_seg[k] == i) a.seg_pos[k] = pos;
    }
    if (t == a.ntiles - 1 && threadIdx.x == 0)   // segments that start at the end (empty trailing segments)
        for (int k = 0; k < a.nseg; ++k)
            if (a.cand_seg[k] >= a.n) a.seg_pos[k] = excl + s_total;
}

__device__ __forceinline__ bool arc_kept(int32_t x, const uint32_t* __restrict__ bkeep) {
    if (x >= 0) return true;
    const uint32_t b = (uint32_t)(-x - 1);
    return (__ldg(bkeep + (b >> 5)) >> (b & 31)) & 1u;
}

struct InduceArgs {
    const int32_t* col_enc; int64_t nnz; const uint32_t* bkeep; const int32_t* slot_of_b; int64_t n_in;
    const int64_t* row_ptr; const int64_t* tile_row; int32_t* out_col; int64_t* out_ptr; int64_t* total;
    uint32_t* words; int32_t* wex; int32_t* tile_cnt; int64_t* tile_pre; unsigned* ctr; int64_t ntiles; int64_t nbw;
};

// pass 1 (one block per tile of kInduceTileArcs arcs): the keep word of every 32-arc block -- warp w owns arcs
// [e0 + 1024 w, +1024): 32 coalesced 128 B loads, lane l holding arc 32 j + l in v[j]; the ballot of load j is the
// keep word of arcs 32 j .. 32 j + 31 -- its exclusive prefix inside the tile, and the tile's count.  The last block
// to finish scans the tile counts into tile prefixes.  No look-back chain (over ~2,000 tiles one measured 95-127 us:
// the inclusive prefix travels ~32 tiles per round trip).
// SMEM: the boundary keep bitmask (|B_i| / 8 bytes) is staged in shared memory -- a warp's 32 lookups hit 32 random
// words, which L1 serves one sector per lane (the pass measured 48 us L1-bound at m = 8).
template <bool SMEM>
__global__ void __launch_bounds__(kEdgeThreads) k_induce_count(const InduceArgs a) {
    pdl_grid_sync();
    __shared__ int s_warp[32], s_total;
    __shared__ bool s_last;
    extern __shared__ uint32_t s_bk[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ewarp = (int64_t)blockIdx.x * kInduceTileArcs + (int64_t)wid * 1024;
    int32_t v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const int64_t e = ewarp + 32 * j + lane;
        v[j] = e < a.nnz ? __ldg(a.col_enc + e) : 0;
    }
    if (SMEM) {
        for (int64_t k = threadIdx.x; k < a.nbw; k += blockDim.x) s_bk[k] = __ldg(a.bkeep + k);
        __syncthreads();
    }
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const int64_t e = ewarp + 32 * j + lane;
        bool kept;
        if (SMEM) {
            const uint32_t b = (uint32_t)(-v[j] - 1);
            kept = v[j] >= 0 || ((s_bk[b >> 5] >> (b & 31)) & 1u);
        } else {
            kept = arc_kept(v[j], a.bkeep);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, e < a.nnz && kept);
        if (lane == j) word = bal;
    }
    const int64_t wi = (int64_t)blockIdx.x * kEdgeThreads + threadIdx.x;
    a.words[wi] = word;
    a.wex[wi] = block_excl_scan(__popc(word), s_warp, &s_total);
    if (threadIdx.x == 0) a.tile_cnt[blockIdx.x] = s_total;
    // last block: exclusive scan of the tile counts (fixed order) -> tile prefixes and the kept total
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.ctr, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    int64_t carry = 0;
    for (int64_t base = 0; base < a.ntiles; base += blockDim.x) {
        const int64_t k = base + threadIdx.x;
        const int c = k < a.ntiles ? __ldcg(a.tile_cnt + k) : 0;
        const int ex = block_excl_scan(c, s_warp, &s_total);
        if (k < a.ntiles) a.tile_pre[k] = carry + ex;
        carry += s_total;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *a.total = carry;
        *a.ctr = 0u;
    }
}

// pass 2 (one warp per 1024-arc chunk, no block barriers): lane j loads word j and its in-tile prefix, every lane
// issues the column loads of its kept arcs of all 32 words, then the slot lookups of the kept halo columns, then the
// order-preserving stores (remapped: halo column -> n_in + slot); then the induced row pointers of the rows whose first
// static arc lies in this chunk (kept arcs before that arc, from the setup tile table and pass 1's words / prefixes)
__global__ void __launch_bounds__(256) k_induce_scatter(const InduceArgs a) {
    pdl_grid_sync();
    const int lane = threadIdx.x & 31;
    const int64_t chunk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nchunks = (a.nnz + 1023) >> 10;
    if (chunk >= nchunks) return;
    constexpr int kChunksPerTile = (int)(kInduceTileArcs / 1024);
    const int64_t t = chunk / kChunksPerTile;
    const int64_t ec = chunk * 1024;
    const int64_t wbase = chunk * 32;   // word index of word 0 of this chunk
    const uint32_t myword = a.words[wbase + lane];
    const int64_t base = __ldg(a.tile_pre + t) + a.wex[wbase + lane];   // lane j: output position of word j
    const int32_t* __restrict__ col = a.col_enc;
    const int32_t* __restrict__ slot = a.slot_of_b;
    int32_t* __restrict__ out = a.out_col;
#pragma unroll 1
    for (int h = 0; h < 32; h += 16) {
        int32_t x[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t wk = __shfl_sync(0xffffffffu, myword, h + k);
            x[k] = ((wk >> lane) & 1u) ? __ldg(col + ec + 32 * (h + k) + lane) : 0;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (x[k] < 0) x[k] = (int32_t)a.n_in + __ldg(slot - x[k] - 1);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t wk = __shfl_sync(0xffffffffu, myword, h + k);
            const int64_t bk = __shfl_sync(0xffffffffu, base, h + k);
            if ((wk >> lane) & 1u) out[bk + __popc(wk & ((1u << lane) - 1u))] = x[k];
        }
    }
    // rows starting in this chunk (setup table; the last chunk also takes the rows starting at nnz)
    const int64_t rlo = a.tile_row[chunk], rhi = a.tile_row[chunk + 1];
    for (int64_t r = rlo + lane; r < rhi; r += 32) {
        const int64_t e = a.row_ptr[r];
        if (e >= a.nnz) {   // trailing empty rows and r = n_in
            a.out_ptr[r] = *a.total;
            continue;
        }
        const int64_t w = e >> 5;
        const int b = (int)(e & 31);
        a.out_ptr[r] = __ldg(a.tile_pre + t) + a.wex[w] + __popc(a.words[w] & ((1u << b) - 1u));
    }
}

struct SegArgs {
    // forward chain: rows of the induced CSR
    const int64_t* ind_ptr; int64_t n_in; Seg* fsegs; int64_t* fsplit; int64_t ntiles_f;
    // backward chain: halo slots -> their boundary rows (transposed arcs after the static A_II part)
    const int64_t* seg_pos; int m; const int32_t* U_b; const int64_t* br_ptr; int64_t cap; int64_t seg_base;
    int64_t e_base; Seg* bsegs; int64_t* bsplit; int64_t ntiles_b;
    int64_t* tot;                       // [1] fwd segments, [2] bwd halo segments, [3] bwd splits, [4] fwd splits,
                                        // [5] fwd hub segments (lpt)
    int64_t fcap; int lpt;              // lpt: forward hub rows' segments from the end of the list (fcap) down
    int32_t seg_long;
    uint64_t* state_f; uint64_t* state_b; unsigned* ctr_f; unsigned* ctr_b; uint32_t gen;
};

__global__ void __launch_bounds__(kTile) k_segs_fused(const SegArgs a) {
    pdl_grid_sync();
    __shared__ int64_t s_tile, s_excl;
    __shared__ int s_warp[32], s_total;
    const bool fwd = blockIdx.x < a.ntiles_f;
    const int64_t t = next_tile(fwd ? a.ctr_f : a.ctr_b, fwd ? a.ntiles_f : a.ntiles_b, &s_tile);
    const int64_t r = t * kTile + threadIdx.x;
    int ns = 0;
    int64_t b0 = 0, b1 = 0;
    int32_t row = 0;
    if (fwd) {
        if (r < a.n_in) {
            b0 = a.ind_ptr[r];
            b1 = a.ind_ptr[r + 1];
            ns = seg_count(b1 - b0, a.seg_long);
            row = (int32_t)r;
        }
    } else {
        const int64_t n_halo = a.seg_pos[a.m] - a.seg_pos[0];
        if (r < n_halo) {
            const int32_t b = a.U_b[r];
            b0 = a.e_base + a.br_ptr[b];
            b1 = a.e_base + a.br_ptr[b + 1];
            ns = seg_count(b1 - b0, a.seg_long);
            row = (int32_t)(a.n_in + r);
        }
    }
    // lpt (forward): a row of several segments (a hub) takes its block from the end of the list by an atomic, the
    // single-segment rows are scanned into the front -- the SpMM claims the hub segments first (longest first)
    const bool hub = a.lpt && fwd && ns > 1;
    const int ex = block_excl_scan(hub ? 0 : ns, s_warp, &s_total);
    const int64_t excl = lookback(fwd ? a.state_f : a.state_b, a.gen, t, s_total, &s_excl);
    if (ns > 0) {
        const int64_t s0 = hub ? a.fcap - (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(a.tot + 5),
                                                             (unsigned long long)ns) - ns
                               : (fwd ? 0 : a.seg_base) + excl + ex;
        Seg* out = fwd ? a.fsegs : a.bsegs;
        if (ns > 1) {
            int64_t* cnt = fwd ? a.tot + 4 : a.tot + 3;
            (fwd ? a.fsplit : a.bsplit)[atomicAdd(reinterpret_cast<unsigned long long*>(cnt), 1ull)] = s0;
        }
        const int64_t L = seg_len(b1 - b0, a.seg_long);
        for (int k = 0; k < ns; ++k) {
            Seg sg;
            sg.row = row;
            sg.nseg = ns;
            sg.e0 = b0 + k * L;
            sg.e1 = min(b1, sg.e0 + L);
            sg.first = s0;
            out[s0 + k] = sg;
        }
    }
    if (threadIdx.x == 0 && t == (fwd ? a.ntiles_f : a.ntiles_b) - 1) a.tot[fwd ? 1 : 2] = excl + s_total;
}

}  // namespace

void launch_sample_fused(Ctx& c, uint64_t T, uint64_t seed, uint64_t epoch) {
    const int m = c.cfg.world;
    int64_t* tot = c.d_seg_pos + 2 * m + 1;
    const int64_t n = c.n_cand;
    const int64_t nt = (n + kTile - 1) / kTile;
    if (nt == 0) {   // nothing to draw: every offset 0, split counters cleared
        BNS_CUDA_HOLD(cudaMemsetAsync(c.d_seg_pos, 0, (2 * m + 1 + 8) * sizeof(int64_t), c.stream));
        return;
    }
    SampleArgs a{};
    a.gid = c.d_cand_gid; a.key = c.d_cand_key; a.payload = c.d_cand_payload; a.n = n; a.n_bd = c.plan.n_bd;
    a.T = T; a.e_lo = (uint32_t)epoch; a.e_hi = (uint32_t)(epoch >> 32); a.s_lo = (uint32_t)seed;
    a.s_hi = (uint32_t)(seed >> 32);
    a.cand_seg = c.d_cand_seg; a.nseg = 2 * m + 1;
    a.flags = c.d_flags; a.bkeep = c.d_bkeep; a.out = c.d_cand_out; a.slot_of_b = c.d_slot_of_b;
    a.seg_pos = c.d_seg_pos;
    a.zero = tot + 3; a.nzero = 3;   // split counters [3], [4] and the forward hub count [5]
    a.state = c.d_lb_state; a.ctr = c.d_lb_ctr; a.gen = ++c.lb_gen; a.ntiles = nt;
    pdl_launch(c.stream, k_sample_fused, (unsigned)nt, kTile, 0, a);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

void launch_induce_fused(Ctx& c) {
    const int m = c.cfg.world;
    int64_t* tot = c.d_seg_pos + 2 * m + 1;
    const int64_t nnz = c.nnz_i;
    const int64_t nt = (nnz + kInduceTileArcs - 1) / kInduceTileArcs;
    if (nt == 0) {
        BNS_CUDA_HOLD(cudaMemsetAsync(c.d_ind_ptr, 0, (c.plan.n_in + 1) * sizeof(int64_t), c.stream));
        BNS_CUDA_HOLD(cudaMemsetAsync(tot, 0, sizeof(int64_t), c.stream));
        return;
    }
    InduceArgs a{};
    a.col_enc = c.d_col_enc; a.nnz = nnz; a.bkeep = c.d_bkeep; a.slot_of_b = c.d_slot_of_b; a.n_in = c.plan.n_in;
    a.row_ptr = c.d_row_ptr; a.tile_row = c.d_tile_row; a.out_col = c.d_ind_col; a.out_ptr = c.d_ind_ptr; a.total = tot;
    a.words = c.d_ebits; a.wex = c.d_ewex; a.tile_cnt = c.d_eblk; a.tile_pre = c.d_eboff; a.ctr = c.d_lb_ctr + 9;
    a.ntiles = nt;
    a.nbw = (c.plan.n_bd + 31) / 32;
    constexpr int64_t kSmemMax = 96 << 10;   // bitmask up to 768 K boundary nodes in shared memory
    if (a.nbw * 4 <= kSmemMax) {
        static bool cfg = false;
        if (!cfg) {
            BNS_CUDA(cudaFuncSetAttribute(k_induce_count<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kSmemMax));
            cfg = true;
        }
        pdl_launch(c.stream, k_induce_count<true>, (unsigned)nt, kEdgeThreads, (size_t)(a.nbw * 4), a);
    } else {
        pdl_launch(c.stream, k_induce_count<false>, (unsigned)nt, kEdgeThreads, 0, a);
    }
    const int64_t nchunks = (nnz + 1023) / 1024;
    pdl_launch(c.stream, k_induce_scatter, (unsigned)((nchunks + 7) / 8), 256, 0, a);
    c.kernels += 2;
    BNS_CHECK_LAUNCH();
}

void launch_segments_fused(Ctx& c, bool fwd) {
    const int m = c.cfg.world;
    int64_t* tot = c.d_seg_pos + 2 * m + 1;
    SegArgs a{};
    a.ind_ptr = c.d_ind_ptr; a.n_in = c.plan.n_in; a.fsegs = c.d_seg_fwd; a.fsplit = c.d_split_fwd;
    a.ntiles_f = fwd ? (c.plan.n_in + kTile - 1) / kTile : 0;
    a.seg_pos = c.d_seg_pos; a.m = m; a.U_b = c.d_cand_out; a.br_ptr = c.d_br_ptr; a.cap = c.plan.n_bd;
    a.seg_base = c.n_seg_bwd_inner; a.e_base = c.ii_nnz; a.bsegs = c.d_seg_bwd;
    a.bsplit = c.d_split_bwd + c.n_split_bwd_inner;
    a.ntiles_b = (c.plan.n_bd + kTile - 1) / kTile;
    a.tot = tot; a.seg_long = c.seg_long;
    a.fcap = c.seg_fwd_cap; a.lpt = fwd_lpt(c) ? 1 : 0;
    a.state_f = c.d_lb_state + c.lb_off_segf; a.state_b = c.d_lb_state + c.lb_off_segb;
    a.ctr_f = c.d_lb_ctr + 2; a.ctr_b = c.d_lb_ctr + 3; a.gen = ++c.lb_gen;
    if (a.ntiles_b == 0) BNS_CUDA_HOLD(cudaMemsetAsync(tot + 2, 0, sizeof(int64_t), c.stream));
    if (fwd && a.ntiles_f == 0) BNS_CUDA_HOLD(cudaMemsetAsync(tot + 1, 0, sizeof(int64_t), c.stream));
    const int64_t grid = a.ntiles_f + a.ntiles_b;
    if (grid == 0) return;
    pdl_launch(c.stream, k_segs_fused, (unsigned)grid, kTile, 0, a);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

}  // namespace bns
