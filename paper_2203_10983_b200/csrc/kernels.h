// kernels.h -- host launchers of the sm_100a kernels (implemented in *.cu).  All launches go on ctx.stream and
// bump ctx.kernels.
#pragma once
#include "common.h"

namespace bns {

// a1 + a2: Philox Bernoulli draw, order-preserving compaction, boundary keep bitmask (induce.cu, one pass)
void launch_sample_fused(Ctx& c, uint64_t T, uint64_t seed, uint64_t epoch);
// a3: induced subgraph over V_i ∪ U_i (induce.cu, one pass); SpMM segments of the induced rows (fwd) and of the
// sampled halo rows (transposed), one launch
void launch_induce_fused(Ctx& c);
void launch_segments_fused(Ctx& c, bool fwd);
// f3 edge samplers (sample.cu): candidate flags from the arc draws, the induced forward CSR + its segments, and the
// sampled transposed CSR + backward segments
void launch_induce_edges(Ctx& c, uint64_t T, uint64_t seed, uint64_t epoch);
void launch_sample_edges(Ctx& c, uint64_t T, uint64_t seed, uint64_t epoch);
void launch_induce_bwd_edges(Ctx& c, uint64_t T, uint64_t seed, uint64_t epoch);
// static segments for a static CSR (setup)
int64_t build_static_segments(Ctx& c, const int64_t* d_ptr, int64_t rows, int64_t ptr_base, Seg* d_out);
// exclusive scan of int32 -> int64 (n elements), total written to *d_total if non-null
void scan_i32(Ctx& c, const int32_t* in, int64_t* out, int64_t n, int64_t* d_total);

// a6 / a10: segment SpMM (spmm.cu)
enum SpmmMode { SAGE_FWD = 0, GCN_FWD = 1, SAGE_BWD = 2, GCN_BWD = 3, SAGE_FWD_TF = 4, GAT_FWD = 5, GAT_BWD = 6,
                GAT_RAW = 7 /* the weighted sum stored as fp32, no epilogue terms */ };
struct SpmmArgs {
    int mode;
    const Seg* segs; int64_t n_segs;
    const int32_t* col;
    const void* src; int64_t ld_src;      // gather source rows (elements)
    void* out; int64_t ld_out;
    const void* self; int64_t ld_self;    // SAGE_BWD: dXself rows (inner; null = none); SAGE_FWD_TF: S rows (inner)
    int32_t d;                            // padded feature width
    int64_t n_in;
    float inv_p;
    float nscale = 1.f;                   // neighbour-sum scale before the epilogue terms (DropEdge 1/q; else 1)
    const float* rowscale;                // per output row
    const float* cscale;                  // GCN_FWD per column
    const int32_t* halo_b;                // GCN_BWD: boundary index of halo slot
    const float* rs_bd;                   // GCN_BWD
    float* partial;
    const int64_t* split; int64_t n_split;  // first-segment index of every split (hub) row -> in-order fixup
    int sc = -1;                          // per-edge column scale override (-1: by mode; 2: cscale[col])
    int relu = 0;                         // SAGE_FWD_TF: ReLU in the epilogue
    int out_f32 = 0;                      // SAGE_FWD_TF / GAT_FWD: fp32 output (logits) instead of the storage type
    unsigned long long* work = nullptr;   // dynamic segment scheduling: [next unclaimed segment, warps done]; the
                                          // last warp to finish resets both (no memset between launches)
    int32_t* arrive = nullptr;            // non-null: split rows are summed by the warp finishing their last segment
    int64_t hub_n = 0, hub_base = 0;      // the first hub_n claims are segments hub_base.. (the hub rows' segments,
                                          // stored at the end of the list), then segments 0..
    int chunk = 1;                        // segments per claim
    // f4 / R45 GAT: per-node attention scores and softmax statistics (fp32), attention vectors a_l / a_r (dout),
    // del / der (backward)
    const float *gat_el = nullptr, *gat_er = nullptr, *gat_m = nullptr, *gat_inv = nullptr;
    const float *gat_al = nullptr, *gat_ar = nullptr, *gat_del = nullptr, *gat_der = nullptr;
};
void launch_spmm(Ctx& c, const SpmmArgs& a);

// f4 / R45 GAT pieces (gat.cu)
void launch_gat_scores(Ctx& c, const void* Y, int64_t ld, int64_t rows, int32_t d, const float* al, const float* ar,
                       float* el, float* er);
void launch_gat_stats(Ctx& c, const Seg* segs, int64_t n_segs, const int32_t* col, const int64_t* split,
                      int64_t n_split, const float* el, const float* er, float* m, float* inv);
void launch_gat_rowdots(Ctx& c, const void* g, const void* out, bool out_f32, const void* Y, int64_t ld, int32_t d,
                        const float* el, const float* er, const float* m, const float* inv, float* cdot, float* selfds);
// del / der without per-edge dot products: with w_vu = alpha_vu LeakyReLU'(s_vu),
//   del_v = g_v . Q_v - c_v q_v,  Q_v = Σ_u w_vu Y_u (segment SpMM, SC 5),   q_v = Σ_u w_vu        (k_gat_wsum 0)
//   der_u = Y_u . P_u - r_u,      P_u = Σ_v w_vu g_v (transposed, SC 6),     r_u = Σ_v w_vu c_v    (k_gat_wsum 1)
// plus the self edge (selfds) -- k_gat_final
void launch_gat_wsum(Ctx& c, int dir, const Seg* segs, int64_t n_segs, const int32_t* col, const int64_t* split,
                     int64_t n_split, const float* el, const float* er, const float* m, const float* inv,
                     const float* cdot, float* out);
void launch_gat_final(Ctx& c, int dir, const void* own, const float* qp, int64_t ld, int32_t d, int64_t rows,
                      const float* cdot, const float* qr, const float* selfds, float* out);
void launch_gat_da(Ctx& c, const void* Y, int64_t ld, int32_t d, const float* w, int64_t rows, float* out);

// a7 / a9: GEMMs (gemm_simt.cu; tcgen05 in gemm_tc.cu)
// C[M x N] = [A0 | A1] (M x (K0+K1), row-major, lda0/lda1) * B (K x N row-major, ldb); epilogue ReLU or none;
// output fp32 (out_f32) or storage type.
void gemm_fwd(Ctx& c, int64_t M, int64_t N, const void* A0, int64_t K0, int64_t lda0, const void* A1, int64_t K1,
              int64_t lda1, const void* B, int64_t ldb, void* C, int64_t ldc, bool relu, bool out_f32);
// dW (K x N) = A^T (M x K, lda) * D (M x N, ldd); result fp32 written to Wg (ldw) (deterministic split-K)
void gemm_wgrad(Ctx& c, int64_t M, int64_t K, int64_t N, const void* A, int64_t lda, const void* D, int64_t ldd,
                float* Wg, int64_t ldw);
// C (M x Nc) = D (M x K, ldd) * B^T where B is (Nc x K, ldb) row-major; columns [0, scale_cols) multiplied by
// rowscale[row]; output storage type
void gemm_dx(Ctx& c, int64_t M, int64_t Nc, int64_t K, const void* D, int64_t ldd, const void* B, int64_t ldb,
             void* C, int64_t ldc, const float* rowscale, int64_t scale_cols);

// out[K x N] = sum over S partial slices (fixed order); partial rows [gap_row, gap_row + gap) are skipped padding
void splitk_reduce(Ctx& c, int S, int64_t K, int64_t N, float* Wg, int64_t ldw, int64_t gap_row = INT64_MAX,
                   int64_t gap = 0);
// deferred reductions (c.defer_red): the slices of a new job start at c.d_splitk + c.splitk_used; splitk_reserve
// makes room for `floats` more (flushing the pending jobs first when they would not fit); splitk_flush reduces every
// pending job in one launch, each in the fixed slice order of k_splitk_reduce (the same bits)
float* splitk_reserve(Ctx& c, int64_t floats);
void splitk_flush(Ctx& c);

// tcgen05 bf16 versions (gemm_tc.cu); fwd takes B = W^T stored [N][Kw] with each concat half padded to 64
void gemm_fwd_tc(Ctx& c, int64_t M, int64_t N, const void* A0, int64_t K0, int64_t lda0, const void* A1, int64_t K1,
                 int64_t lda1, const void* WT, int64_t Kw, void* C, int64_t ldc, bool relu, bool out_f32);
void gemm_wgrad_tc(Ctx& c, int64_t Mn, int64_t K, int64_t N, const void* A, int64_t lda, const void* D, int64_t ldd,
                   float* Wg, int64_t ldw);
void gemm_wgrad2_tc(Ctx& c, int64_t Mn0, int64_t Mn1, int64_t K, int64_t N, const void* A0, const void* A1,
                    int64_t lda, const void* D0, int64_t ldd0, const void* D1, int64_t ldd1, float* Wg, int64_t ldw);
void gemm_dx_tc(Ctx& c, int64_t M, int64_t Nc, int64_t K, const void* D, int64_t ldd, const void* B, int64_t ldb,
                void* C, int64_t ldc, const float* rowscale, int64_t scale_cols);

// misc (misc.cu)
void launch_pack_rows(Ctx& c, const void* src, int64_t ld_src, const int32_t* idx, int64_t n, void* dst, int32_t d);
void launch_scatter_add(Ctx& c, void* dst, int64_t ld_dst, const int32_t* idx, const void* src, int64_t n, int32_t d);
// a12 merged over peers (world <= 32): prep once per draw, then one launch per layer
void launch_scatter_prep(Ctx& c, int64_t n_sent);
void launch_scatter_rows(Ctx& c, void* dst, int64_t ld, const void* src, int32_t d);
// rs / dps (optional, R42): also write dps = dPre * rs[row] (the transform-first SpMM^T source)
// ldp: row pitch of dpre_t (-1: ld); nzero: rows after the inner rows of dpre_t set to zero (R42 halo rows)
void launch_xent(Ctx& c, const float* logits, int64_t ld, int32_t C, float* dlogits, void* dpre_t,
                 const float* rs = nullptr, void* dps = nullptr, int64_t ldp = -1, int64_t nzero = 0);
void launch_bce(Ctx& c, const float* logits, int64_t ld, int32_t C, float* dlogits, void* dpre_t, const float* rs,
                void* dps, int64_t ldp = -1, int64_t nzero = 0);
// a12 folded into the ReLU mask of the layer below (one launch less per layer): mask / pos from k_scatter_prep; the
// returned rows are in the staged buffer src (row k of the returned rows) or, over peer memory, row pos + delta[j]
// of peer j's dX (peer[j])
struct ScatterIn {
    const uint32_t* mask = nullptr;
    const int32_t* pos = nullptr;
    int m = 0;
    const void* src = nullptr;
    const void* const* peer = nullptr;
    const int64_t* delta = nullptr;
};
void launch_relu_mask(Ctx& c, const void* dh, const void* h, int64_t ld, int64_t rows, int32_t d, void* dpre,
                      const float* rs = nullptr, void* dps = nullptr, const ScatterIn* sc = nullptr);
void launch_wpack_all(Ctx& c, float* const* W);
void launch_sgd(Ctx& c, float* const* W, float* const* G, float lr);
void launch_adam(Ctx& c, float* const* W, float* const* G, float lr);
void launch_dropout(Ctx& c, const void* src, void* dst, int64_t rows, int64_t ld, int layer);
void launch_halo_gid(Ctx& c);
void launch_sum_ptrs(Ctx& c, const float* const* d_ptrs, int nptr, float* out, int64_t n);
void launch_sum_ptrs_d(Ctx& c, const double* const* d_ptrs, int nptr, double* out, int64_t n);
void launch_fill_rowscale_bwd(Ctx& c, float* rs);
void launch_gcn_cscale(Ctx& c);
// f1 peer-memory exchange (peer.cu): device flag barrier over the ranks' flag slots (+ the per-peer row offsets of
// this rank's rows in the peers' halo gradients), fused pack + forward exchange (gather from the owners' H), fused
// reverse exchange + scatter-add (gather from the peers' dX halo rows)
void preload_module_functions();   // load every kernel now (lazy loading would wait on a spinning barrier)
void launch_peer_barrier(Ctx& c, uint64_t* const* d_flags, uint64_t val, int* err, const int64_t* const* d_pseg,
                         const int64_t* d_pnin, int64_t* d_delta);
void launch_halo_pull(Ctx& c, void* dst, int64_t ld, void* const* d_peerH, const int32_t* d_owner_of_b,
                      const int32_t* d_row_of_b, int32_t d);
void launch_scatter_peer(Ctx& c, void* dst, int64_t ld, void* const* d_peerdx, const int64_t* d_delta, int32_t d);
void launch_to_storage(Ctx& c, const float* src, int64_t rows, int32_t dlog, int64_t ld_src, void* dst, int64_t ld_dst);

}  // namespace bns
