// sample.cu -- a1 sample, a2 compact, a3 induce (+ SpMM work segments).
//
// The BNS draw itself (a1-a3 for BNS) runs as three single-pass kernels in induce.cu; this file keeps the scan
// helpers, the shared compaction scatter and the f3 edge-sampler passes.
// a1  Alg.1 l.4: every candidate is one independent Bernoulli(p) draw (R5, R6).  The
//     candidates of rank i are (recv side) every u in B_i keyed by i, and (send side) every u in D_{i->j} keyed by
//     j -- i recomputes j's draw instead of receiving the broadcast U_j (Alg.1 l.6-7, R27).
//     keep = Philox4x32-10(ctr = {u, key, e_lo, e_hi}, key = {s_lo, s_hi}).x < floor(p 2^32)  (R7)
// a2  order-preserving compaction (block count -> scan -> warp-ballot scatter) into U_i (owner-major, R24) and
//     S_{i,j}; the 2m+1 segment offsets give the per-peer counts.
// a3  Alg.1 l.5: node-induced subgraph on V_i ∪ U_i -- the static inner rows with dropped
//     boundary columns removed (global neighbour order kept), boundary columns remapped to halo rows n_in + slot.
#include "common.h"
#include "dev.cuh"
#include "kernels.h"

namespace bns {

constexpr int kSampleBlock = 1024;

// Single-block exclusive scan of n int32 (n arbitrary) -> int64 out[0..n], out[n] = total; optional extra total.
__global__ void __launch_bounds__(1024) k_scan_top(const int32_t* __restrict__ in, int64_t* __restrict__ out,
                                                   int64_t n, int64_t* __restrict__ total) {
    pdl_grid_sync();
    __shared__ int64_t warp_sums[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t base = 0; base < n; base += 1024) {
        int64_t i = base + threadIdx.x;
        int64_t v = (i < n) ? in[i] : 0;
        int64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[w] = x;
        __syncthreads();
        if (w == 0) {
            int64_t s = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int64_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        int64_t excl = carry + (w ? warp_sums[w - 1] : 0) + x - v;
        if (i < n) out[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[n] = carry;
        if (total) *total = carry;
    }
}

// Block-level exclusive scan (1024 elements per block), block sums to bsum.
__global__ void __launch_bounds__(1024) k_scan_block(const int32_t* __restrict__ in, int64_t* __restrict__ out,
                                                     int64_t n, int32_t* __restrict__ bsum) {
    pdl_grid_sync();
    __shared__ int32_t warp_sums[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
    int32_t v = (i < n) ? in[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
        int32_t s = warp_sums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;
    }
    __syncthreads();
    if (i < n) out[i] = (int64_t)((w ? warp_sums[w - 1] : 0) + x - v);
    if (threadIdx.x == 0) bsum[blockIdx.x] = warp_sums[31];
}

__global__ void k_scan_add(int64_t* __restrict__ out, int64_t n, const int64_t* __restrict__ boff) {
    pdl_grid_sync();
    int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
    if (i < n) out[i] += boff[blockIdx.x];
}

void scan_i32(Ctx& c, const int32_t* in, int64_t* out, int64_t n, int64_t* d_total) {
    if (n <= 4096) {
        pdl_launch(c.stream, k_scan_top, 1, 1024, 0, in, out, n, d_total);
        c.kernels += 1;
        BNS_CHECK_LAUNCH();
        return;
    }
    int64_t nb = (n + 1023) / 1024;
    int32_t* bsum = reinterpret_cast<int32_t*>(c.d_scan_tmp);        // nb int32
    int64_t* boff = c.d_scan_tmp + (nb + 1) / 2 + 1;                  // nb+1 int64
    pdl_launch(c.stream, k_scan_block, (unsigned)nb, 1024, 0, in, out, n, bsum);
    pdl_launch(c.stream, k_scan_top, 1, 1024, 0, bsum, boff, nb, nullptr);
    pdl_launch(c.stream, k_scan_add, (unsigned)nb, 1024, 0, out, n, boff);
    c.kernels += 3;
    BNS_CHECK_LAUNCH();
    BNS_CUDA_HOLD(cudaMemcpyAsync(out + n, boff + nb, sizeof(int64_t), cudaMemcpyDeviceToDevice, c.stream));
    if (d_total) BNS_CUDA_HOLD(cudaMemcpyAsync(d_total, boff + nb, sizeof(int64_t), cudaMemcpyDeviceToDevice, c.stream));
}

// a2: scatter kept candidates to their compacted position; recv candidates also publish slot_of_b.
__global__ void __launch_bounds__(kSampleBlock) k_sample_scatter(const uint8_t* __restrict__ flags, int64_t n,
                                                                 int64_t n_bd, const int64_t* __restrict__ boff,
                                                                 const int32_t* __restrict__ payload,
                                                                 const int64_t* __restrict__ cand_seg, int nseg,
                                                                 int32_t* __restrict__ out,
                                                                 int32_t* __restrict__ slot_of_b,
                                                                 int64_t* __restrict__ seg_pos) {
    pdl_grid_sync();
    __shared__ int32_t warp_cnt[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t i = (int64_t)blockIdx.x * kSampleBlock + threadIdx.x;
    int keep = (i < n) ? flags[i] : 0;
    unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_cnt[w] = __popc(bal);
    __syncthreads();
    if (w == 0) {
        int s = warp_cnt[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_cnt[lane] = s;
    }
    __syncthreads();
    int64_t pos = boff[blockIdx.x] + (w ? warp_cnt[w - 1] : 0) + __popc(bal & ((1u << lane) - 1u));
    if (i < n) {
        if (keep) out[pos] = payload[i];
        if (i < n_bd) slot_of_b[payload[i]] = keep ? (int32_t)pos : -1;
        for (int k = 0; k < nseg; ++k)
            if (cand_seg[k] == i) seg_pos[k] = pos;
    }
    if (i == 0 && n == 0)
        for (int k = 0; k < nseg; ++k) seg_pos[k] = 0;
}

__global__ void k_seg_tail(const int64_t* __restrict__ cand_seg, int nseg, int64_t n, const int64_t* __restrict__ boff,
                           int64_t nb, int64_t* __restrict__ seg_pos) {
    pdl_grid_sync();
    int k = threadIdx.x;
    if (k < nseg && cand_seg[k] >= n) seg_pos[k] = boff[nb];
}

// ---------------------------------------------------------------------------------------------
// a3 induce, edge-parallel (balanced over nnz, so hub rows cost no more than their edges):
//   K1 keep bit of every static edge (one 32-edge word per thread) + per-1024-edge counts, K2 scan of the counts,
//   K3 order-preserving scatter of the kept (remapped) columns, K4 row pointers from the bit prefix + segment
//   counts per row, scan, K5 segment list.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_induce_scatter_w(const int32_t* __restrict__ col, int64_t nnz,
                                                          const int32_t* __restrict__ slot_of_b,
                                                          const uint32_t* __restrict__ bits,
                                                          const int64_t* __restrict__ boff, int64_t n_in,
                                                          int32_t* __restrict__ out_col) {
    pdl_grid_sync();
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nw = (nnz + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t word = w < nw ? bits[w] : 0u;
    const int c = __popc(word);
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    // warp-cooperative over the warp's 1024-edge block: word k is processed by all lanes (lane j = edge 32k + j),
    // so the column reads are 128-byte lines and the kept columns are written contiguously
    const int64_t base = (w >> 5) < ((nnz + 1023) >> 10) ? boff[w >> 5] : 0;
    const int64_t e_blk = (w - lane) << 5;
    const int excl = x - c;
    // loads of a batch of words first, then the stores (stores interleaved with the loads serialise them)
#pragma unroll 1
    for (int h = 0; h < 32; h += 16) {
        int32_t v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t wk = __shfl_sync(0xffffffffu, word, h + k);
            v[k] = ((wk >> lane) & 1u) ? __ldg(col + e_blk + 32 * (h + k) + lane) : 0;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (v[k] < 0) v[k] = (int32_t)n_in + __ldg(slot_of_b - v[k] - 1);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t wk = __shfl_sync(0xffffffffu, word, h + k);
            const int ek = __shfl_sync(0xffffffffu, excl, h + k);
            if ((wk >> lane) & 1u) out_col[base + ek + __popc(wk & ((1u << lane) - 1u))] = v[k];
        }
    }
}

void launch_induce_flags_edge(Ctx& c, int64_t nb, uint64_t T, uint64_t seed, uint64_t epoch);

// number of kept edges before static edge position e
__device__ __forceinline__ int64_t kept_before(int64_t e, const uint32_t* __restrict__ bits,
                                               const int64_t* __restrict__ boff) {
    const int64_t b = e >> 10;
    int64_t s = boff[b];
    for (int64_t w = b << 5; w < (e >> 5); ++w) s += __popc(bits[w]);
    if (e & 31) s += __popc(bits[e >> 5] & ((1u << (e & 31)) - 1u));
    return s;
}

__global__ void k_induce_rows(const int64_t* __restrict__ ptr, int64_t n_in, const uint32_t* __restrict__ bits,
                              const int64_t* __restrict__ boff, int64_t* __restrict__ out_ptr,
                              int32_t* __restrict__ nseg, int32_t seg_long) {
    pdl_grid_sync();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > n_in) return;
    const int64_t a = kept_before(ptr[r], bits, boff);
    out_ptr[r] = a;
    if (r == n_in) return;
    const int64_t cnt = kept_before(ptr[r + 1], bits, boff) - a;
    nseg[r] = seg_count(cnt, seg_long);
}

// rows split into several segments are appended (first segment index) to a split list for the SpMM fixup;
// list order is irrelevant (each row's partials are summed in segment order)
__device__ __forceinline__ void push_split(int64_t* list, int64_t* count, int64_t s0) {
    list[atomicAdd(reinterpret_cast<unsigned long long*>(count), 1ull)] = s0;
}

__global__ void k_induce_segs(const int64_t* __restrict__ out_ptr, int64_t n_in, const int64_t* __restrict__ seg_off,
                              Seg* __restrict__ segs, int64_t* __restrict__ split, int64_t* __restrict__ n_split, int32_t seg_long) {
    pdl_grid_sync();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_in) return;
    const int64_t b0 = out_ptr[r], b1 = out_ptr[r + 1];
    const int64_t s0 = seg_off[r], ns = seg_off[r + 1] - s0;
    if (ns > 1) push_split(split, n_split, s0);
    for (int64_t k = 0; k < ns; ++k) {
        Seg sg;
        sg.row = (int32_t)r;
        sg.nseg = (int32_t)ns;
        sg.e0 = b0 + k * seg_len(b1 - b0, seg_long);
        sg.e1 = min(b1, sg.e0 + seg_len(b1 - b0, seg_long));
        sg.first = s0;
        segs[s0 + k] = sg;
    }
}

// a3 for the edge samplers (f3): arc keep bits from the arc draws, scan, order-preserving scatter, row pointers,
// segment counts, scan, segment list (the BNS draw runs the single-pass kernels of induce.cu instead)
void launch_induce_edges(Ctx& c, uint64_t T, uint64_t seed, uint64_t epoch) {
    const int64_t n_in = c.plan.n_in;
    const int64_t nnz = c.nnz_i;
    const int m = c.cfg.world;
    int64_t* tot = c.d_seg_pos + 2 * m + 1;   // [nnz_kept, n_seg_fwd, n_seg_bwd_halo]
    const int64_t nb = (nnz + 1023) / 1024;
    if (nb > 0) {
        const unsigned wb = (unsigned)((((nnz + 31) >> 5) + 255) / 256);
        launch_induce_flags_edge(c, nb, T, seed, epoch);
        pdl_launch(c.stream, k_scan_top, 1, 1024, 0, c.d_eblk, c.d_eboff, nb, tot + 0);
        pdl_launch(c.stream, k_induce_scatter_w, wb, 256, 0, c.d_col_enc, nnz, c.d_slot_of_b, c.d_ebits, c.d_eboff, n_in,
                                                     c.d_ind_col);
        c.kernels += 3;
    } else {
        BNS_CUDA_HOLD(cudaMemsetAsync(c.d_eboff, 0, sizeof(int64_t), c.stream));
        BNS_CUDA_HOLD(cudaMemsetAsync(tot, 0, sizeof(int64_t), c.stream));
    }
    pdl_launch(c.stream, k_induce_rows, (unsigned)((n_in + 1 + 255) / 256), 256, 0, c.d_row_ptr, n_in, c.d_ebits, c.d_eboff,
                                                                          c.d_ind_ptr, c.d_row_nseg, c.seg_long);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
    scan_i32(c, c.d_row_nseg, c.d_row_soff, n_in, tot + 1);
    BNS_CUDA_HOLD(cudaMemsetAsync(tot + 4, 0, sizeof(int64_t), c.stream));
    pdl_launch(c.stream, k_induce_segs, (unsigned)((n_in + 255) / 256), 256, 0, c.d_ind_ptr, n_in, c.d_row_soff, c.d_seg_fwd,
                                                                       c.d_split_fwd, tot + 4, c.seg_long);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------------------------
// f3 edge samplers: BES keeps each cross-partition arc with probability q, DropEdge every arc.
// R40 arc draw: keep(v <- u) = Philox4x32-10(ctr = {v, u, e_lo, e_hi}, key = {s_lo ^ 0xED6E, s_hi}).x < T(q).
// ---------------------------------------------------------------------------------------------
struct ArcKey {
    uint64_t T;
    uint32_t e_lo, e_hi, k0, k1;
    __device__ __forceinline__ bool keep(int32_t v, int32_t u) const {
        return (uint64_t)philox4((uint32_t)v, (uint32_t)u, e_lo, e_hi, k0, k1).x < T;
    }
};

inline ArcKey arc_key(uint64_t T, uint64_t seed, uint64_t epoch) {
    return ArcKey{T, (uint32_t)epoch, (uint32_t)(epoch >> 32), (uint32_t)seed ^ 0xED6Eu, (uint32_t)(seed >> 32)};
}

// a1 for the edge samplers: receive candidate b in B_i is communicated iff one of its arcs into V_i survives;
// send candidate (u, peer j) iff one of u's arcs into V_j survives (j's draw recomputed, R27).  Same flags/block
// count contract the compaction scatter (k_sample_scatter) expects.
__global__ void __launch_bounds__(kSampleBlock) k_edge_cand(int64_t n_bd, int64_t n, const int32_t* __restrict__ gid,
                                                            const int32_t* __restrict__ key,
                                                            const int32_t* __restrict__ payload,
                                                            const int32_t* __restrict__ vgid,
                                                            const int64_t* __restrict__ br_ptr,
                                                            const int32_t* __restrict__ br_col,
                                                            const int64_t* __restrict__ row_ptr,
                                                            const int32_t* __restrict__ col_enc,
                                                            const int64_t* __restrict__ b_off, ArcKey ak,
                                                            uint8_t* __restrict__ flags, int32_t* __restrict__ blk) {
    pdl_grid_sync();
    const int64_t i = (int64_t)blockIdx.x * kSampleBlock + threadIdx.x;
    int keep = 0;
    if (i < n) {
        if (i < n_bd) {
            const int32_t ug = gid[i];
            for (int64_t e = br_ptr[i]; e < br_ptr[i + 1] && !keep; ++e) keep = ak.keep(vgid[br_col[e]], ug);
        } else {
            const int32_t u = payload[i], j = key[i], ug = gid[i];
            const int64_t lo = b_off[j], hi = b_off[j + 1];
            for (int64_t e = row_ptr[u]; e < row_ptr[u + 1] && !keep; ++e) {
                const int32_t x = col_enc[e];
                if (x < 0 && -x - 1 >= lo && -x - 1 < hi) keep = ak.keep(gid[-x - 1], ug);
            }
        }
        flags[i] = (uint8_t)keep;
    }
    const int cnt = __syncthreads_count(keep);
    if (threadIdx.x == 0) blk[blockIdx.x] = cnt;
}

void launch_sample_edges(Ctx& c, uint64_t T, uint64_t seed, uint64_t epoch) {
    const int m = c.cfg.world;
    const int64_t n = c.n_cand;
    const int64_t nb = (n + kSampleBlock - 1) / kSampleBlock;
    int64_t* boff = c.d_scan_tmp;
    if (nb > 0) {
        pdl_launch(c.stream, k_edge_cand, (unsigned)nb, kSampleBlock, 0, 
            c.plan.n_bd, n, c.d_cand_gid, c.d_cand_key, c.d_cand_payload, c.d_vgid, c.d_br_ptr, c.d_tcol + c.ii_nnz,
            c.d_row_ptr, c.d_col_enc, c.d_cand_seg, arc_key(T, seed, epoch), c.d_flags, c.d_blk);
        pdl_launch(c.stream, k_scan_top, 1, 1024, 0, c.d_blk, boff, nb, nullptr);
        pdl_launch(c.stream, k_sample_scatter, (unsigned)nb, kSampleBlock, 0, c.d_flags, n, c.plan.n_bd, boff,
                                                                      c.d_cand_payload, c.d_cand_seg, 2 * m + 1,
                                                                      c.d_cand_out, c.d_slot_of_b, c.d_seg_pos);
        c.kernels += 3;
    } else {
        BNS_CUDA_HOLD(cudaMemsetAsync(boff, 0, sizeof(int64_t), c.stream));
    }
    pdl_launch(c.stream, k_seg_tail, 1, 128, 0, c.d_cand_seg, 2 * m + 1, n, boff, nb, c.d_seg_pos);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
}

// a3 for the edge samplers, forward: arc (v <- x) of the static CSR kept by its draw (DropEdge: every arc; BES:
// boundary columns only).  A kept boundary arc implies its column's node is in U_i, so the remap is defined.
__global__ void __launch_bounds__(1024) k_induce_flags_edge(const int32_t* __restrict__ col_enc,
                                                            const int32_t* __restrict__ erow, int64_t nnz,
                                                            const int32_t* __restrict__ vgid,
                                                            const int32_t* __restrict__ bgid, int dropedge, ArcKey ak,
                                                            uint32_t* __restrict__ bits, int32_t* __restrict__ blk) {
    pdl_grid_sync();
    const int64_t e = (int64_t)blockIdx.x * 1024 + threadIdx.x;
    int keep = 0;
    if (e < nnz) {
        const int32_t x = col_enc[e];
        if (x >= 0) keep = dropedge ? ak.keep(vgid[erow[e]], vgid[x]) : 1;
        else keep = ak.keep(vgid[erow[e]], bgid[-x - 1]);
    }
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    if ((threadIdx.x & 31) == 0) bits[e >> 5] = b;
    const int cnt = __syncthreads_count(keep);
    if (threadIdx.x == 0) blk[blockIdx.x] = cnt;
}

void launch_induce_flags_edge(Ctx& c, int64_t nb, uint64_t T, uint64_t seed, uint64_t epoch) {
    pdl_launch(c.stream, k_induce_flags_edge, (unsigned)nb, 1024, 0, c.d_col_enc, c.d_erow, c.nnz_i, c.d_vgid, c.d_cand_gid,
                                                             c.sampler == BNS_SAMPLER_DROPEDGE,
                                                             arc_key(T, seed, epoch), c.d_ebits, c.d_eblk);
}

// backward: the transposed arcs (row u <- column v means v aggregates u) -- inner rows u (A_II^T), then boundary
// rows b (the arcs v <- b of every inner v); the same draw keep(v <- u) decides both directions of use
__global__ void __launch_bounds__(1024) k_tinduce_flags(const int32_t* __restrict__ tcol,
                                                        const int32_t* __restrict__ terow, int64_t nnz, int64_t n_in,
                                                        const int32_t* __restrict__ vgid,
                                                        const int32_t* __restrict__ bgid, int dropedge, ArcKey ak,
                                                        uint32_t* __restrict__ bits, int32_t* __restrict__ blk) {
    pdl_grid_sync();
    const int64_t e = (int64_t)blockIdx.x * 1024 + threadIdx.x;
    int keep = 0;
    if (e < nnz) {
        const int32_t r = terow[e], v = tcol[e];
        if (r < n_in) keep = dropedge ? ak.keep(vgid[v], vgid[r]) : 1;
        else keep = ak.keep(vgid[v], bgid[r - n_in]);
    }
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    if ((threadIdx.x & 31) == 0) bits[e >> 5] = b;
    const int cnt = __syncthreads_count(keep);
    if (threadIdx.x == 0) blk[blockIdx.x] = cnt;
}

// output row of transposed row r: inner r -> r; boundary b -> halo row n_in + slot (or none if b is not in U_i)
__device__ __forceinline__ int64_t trow_out(int64_t r, int64_t n_in, const int32_t* __restrict__ slot_of_b) {
    if (r < n_in) return r;
    const int32_t s = slot_of_b[r - n_in];
    return s < 0 ? -1 : n_in + s;
}

__global__ void k_tinduce_rows(const int64_t* __restrict__ ptr, int64_t n_rows, int64_t n_in,
                               const int32_t* __restrict__ slot_of_b, const uint32_t* __restrict__ bits,
                               const int64_t* __restrict__ boff, int64_t* __restrict__ out_ptr,
                               int32_t* __restrict__ nseg, int32_t seg_long) {
    pdl_grid_sync();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > n_rows) return;
    const int64_t a = kept_before(ptr[r], bits, boff);
    out_ptr[r] = a;
    if (r == n_rows) return;
    const int64_t cnt = kept_before(ptr[r + 1], bits, boff) - a;
    nseg[r] = trow_out(r, n_in, slot_of_b) < 0 ? 0 : seg_count(cnt, seg_long);
}

__global__ void k_tinduce_segs(const int64_t* __restrict__ out_ptr, int64_t n_rows, int64_t n_in,
                               const int32_t* __restrict__ slot_of_b, const int64_t* __restrict__ seg_off,
                               Seg* __restrict__ segs, int64_t* __restrict__ split, int64_t* __restrict__ n_split, int32_t seg_long) {
    pdl_grid_sync();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rows) return;
    const int64_t s0 = seg_off[r], ns = seg_off[r + 1] - s0;
    if (ns == 0) return;
    const int64_t b0 = out_ptr[r], b1 = out_ptr[r + 1];
    if (ns > 1) push_split(split, n_split, s0);
    const int32_t row = (int32_t)trow_out(r, n_in, slot_of_b);
    for (int64_t k = 0; k < ns; ++k) {
        Seg sg;
        sg.row = row;
        sg.nseg = (int32_t)ns;
        sg.e0 = b0 + k * seg_len(b1 - b0, seg_long);
        sg.e1 = min(b1, sg.e0 + seg_len(b1 - b0, seg_long));
        sg.first = s0;
        segs[s0 + k] = sg;
    }
}

void launch_induce_bwd_edges(Ctx& c, uint64_t T, uint64_t seed, uint64_t epoch) {
    const int64_t n_in = c.plan.n_in, n_rows = n_in + c.plan.n_bd;
    const int m = c.cfg.world;
    int64_t* tot = c.d_seg_pos + 2 * m + 1;   // [5] kept transposed arcs, [6] segments, [7] split rows
    const int64_t nnz = c.tnnz;
    const int64_t nb = (nnz + 1023) / 1024;
    if (nb > 0) {
        pdl_launch(c.stream, k_tinduce_flags, (unsigned)nb, 1024, 0, c.d_tcol, c.d_terow, nnz, n_in, c.d_vgid, c.d_cand_gid,
                                                             c.sampler == BNS_SAMPLER_DROPEDGE,
                                                             arc_key(T, seed, epoch), c.d_ebits, c.d_eblk);
        pdl_launch(c.stream, k_scan_top, 1, 1024, 0, c.d_eblk, c.d_eboff, nb, tot + 5);
        // every transposed column is an inner id (>= 0): the scatter's remap is the identity
        pdl_launch(c.stream, k_induce_scatter_w, (unsigned)((((nnz + 31) >> 5) + 255) / 256), 256, 0, 
            c.d_tcol, nnz, c.d_slot_of_b, c.d_ebits, c.d_eboff, n_in, c.d_ind_tcol);
        c.kernels += 3;
    } else {
        BNS_CUDA_HOLD(cudaMemsetAsync(c.d_eboff, 0, sizeof(int64_t), c.stream));
        BNS_CUDA_HOLD(cudaMemsetAsync(tot + 5, 0, sizeof(int64_t), c.stream));
    }
    pdl_launch(c.stream, k_tinduce_rows, (unsigned)((n_rows + 1 + 255) / 256), 256, 0, 
        c.d_tptr, n_rows, n_in, c.d_slot_of_b, c.d_ebits, c.d_eboff, c.d_ind_tptr, c.d_trow_nseg, c.seg_long);
    c.kernels += 1;
    BNS_CHECK_LAUNCH();
    scan_i32(c, c.d_trow_nseg, c.d_trow_soff, n_rows, tot + 6);
    BNS_CUDA_HOLD(cudaMemsetAsync(tot + 7, 0, sizeof(int64_t), c.stream));
    if (n_rows > 0) {
        pdl_launch(c.stream, k_tinduce_segs, (unsigned)((n_rows + 255) / 256), 256, 0, 
            c.d_ind_tptr, n_rows, n_in, c.d_slot_of_b, c.d_trow_soff, c.d_eseg_bwd, c.d_esplit_bwd, tot + 7, c.seg_long);
        c.kernels += 1;
        BNS_CHECK_LAUNCH();
    }
}

}  // namespace bns
