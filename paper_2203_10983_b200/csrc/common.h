// common.h -- internal declarations shared by the libbns translation units (host side).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>
#include <stdexcept>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "bns.h"

namespace bns {

struct Error : std::runtime_error {
    bns_status code;
    Error(bns_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define BNS_CUDA(x)                                                                                  \
    do {                                                                                             \
        cudaError_t e__ = (x);                                                                       \
        if (e__ != cudaSuccess)                                                                      \
            throw ::bns::Error(BNS_ERR_RUNTIME, std::string(#x) + ": " + cudaGetErrorString(e__) +   \
                                                    " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

#define BNS_CHECK_LAUNCH() BNS_CUDA(cudaGetLastError())

// PDL (dev.cuh): the next kernel this host thread launches is launched with plain stream serialisation -- called
// after every non-kernel stream operation (copies, memsets, cross-stream event waits, NCCL calls) and around the
// peer-memory barrier, so a kernel never starts early behind work whose completion griddepcontrol.wait does not
// cover (another stream's, another context's, the copy engines')
void pdl_hold();
bool pdl_take_hold();
#define BNS_CUDA_HOLD(x)  \
    do {                  \
        BNS_CUDA(x);      \
        ::bns::pdl_hold(); \
    } while (0)

#ifndef BNS_KSEG
#define BNS_KSEG 256   // A/B on one B200 (make kseg128 / kseg256): 512 -> 256 = m=8 rank epoch 2.23 -> 2.12 ms, m=1 24.3 -> 24.0
#endif
constexpr int kSeg = BNS_KSEG;     // SpMM segment length in edges (hub rows are split into segments of this size)
// rows longer than kLongRow are split into seg_long-edge segments instead when the job is large enough (seg_long =
// kSegLong when the graph has >= kLongJobNnz arcs per partition, else 0 = never): fewer fp32 partials for the
// fixup to move on big partitions, no long single-warp tails on small ones.  The split depends only on the row
// length and that job-wide constant (R37).  Measured (one B200): Reddit m = 1 23.1 -> 22.5 ms with long segments;
// at m = 8 they cost +13 %.
#ifndef BNS_KSEG_LONG
#define BNS_KSEG_LONG 1024
#endif
constexpr int kSegLong = BNS_KSEG_LONG;
constexpr int64_t kLongRow = 2048;
constexpr int64_t kLongJobNnz = 38ll * 1000 * 1000;   // ~32 x 256 edges per resident SpMM warp on 148 SMs
__host__ __device__ inline int64_t seg_len(int64_t cnt, int32_t seg_long) {
    return (seg_long > 0 && cnt > kLongRow) ? (int64_t)seg_long : (int64_t)kSeg;
}
__host__ __device__ inline int32_t seg_count(int64_t cnt, int32_t seg_long) {
    const int64_t L = seg_len(cnt, seg_long);
    return cnt > L ? (int32_t)((cnt + L - 1) / L) : 1;
}
constexpr int64_t kInduceTileArcs = 32768;  // induce.cu: arcs per tile (1024 threads x one 32-arc word)
constexpr int kPad = 8;            // feature dims padded to multiples of 8 (16-byte rows for fp32x4 / bf16x8)

inline int64_t pad8(int64_t d) { return (d + kPad - 1) / kPad * kPad; }

// ----------------------------------------------------------------------------------------------
// Host plan (a0): PAPER.md:173-176 -- inner set V_i, boundary set B_i, send candidates D_{i->j}.
// ----------------------------------------------------------------------------------------------
struct Plan {
    int rank = 0, world = 1;
    int64_t N = 0;
    int64_t n_in = 0, n_bd = 0, n_send = 0;   // |V_i|, |B_i|, Σ_j |D_{i->j}|
    std::vector<int32_t> V;                   // inner gids, ascending
    std::vector<int32_t> B;                   // boundary gids, (owner, gid)
    std::vector<int64_t> B_off;               // [m+1]
    std::vector<int32_t> D_local;             // send candidates as local inner rows, per peer j ascending gid
    std::vector<int64_t> D_off;               // [m+1]
    std::vector<int64_t> row_ptr;             // static CSR over inner rows (full rows, global order)
    std::vector<int32_t> col_enc;             // >= 0: inner local id;  < 0: -(b+1) boundary index
    std::vector<int64_t> ii_ptr;              // inner-only part (A_II), local ids
    std::vector<int32_t> ii_col;
    std::vector<int64_t> br_ptr;              // boundary rows: inner neighbours of each b (local ids ascending)
    std::vector<int32_t> br_col;
    std::vector<float> deg_in, deg_bd;        // full-graph degrees deg_G
    std::vector<int32_t> B_row;               // row of B[b] in its owner's V (f1 peer-memory pull)
};

void build_plan(Plan& P, int rank, int world, int64_t N, const int64_t* indptr, const int32_t* indices,
                const int32_t* part_of);

// ----------------------------------------------------------------------------------------------
// Segments: a warp-sized unit of SpMM work -- out_row, edge range [e0, e1), and for hub rows split into
// several segments, the index of the first segment of the row and the number of segments (nseg > 1 ->
// partial sums go through a deterministic in-order fixup).
// ----------------------------------------------------------------------------------------------
struct Seg {
    int32_t row;
    int32_t nseg;       // segments of this row
    int64_t e0, e1;
    int64_t first;      // index of the row's first segment
};

struct Transport;

struct Ctx {
    bns_config cfg{};
    std::vector<int32_t> dims, dp;            // logical, padded (L+1)
    int L = 1;
    int layer = 0, prec = 0;
    bool plan_only = false, timing = false, debug_idx = false, retain = false;
    int fwd_mode = 0;                         // 0 static full CSR (p=1 / no boundary), 1 A_II only (p=0), 2 induced
    size_t ev_used = 0;
    std::vector<int> ev_phase;
    int64_t hostw_n = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    bool failed = false;
    bool sampled = false;
    // BNS_PREFETCH_DRAW (R48): bns_step enqueues the draw of (pf_p, pf_seed, pf_ep) before its closing sync
    bool pf_want = false, pf_pending = false;
    double pf_p = 0.0;
    uint64_t pf_seed = 0, pf_ep = 0;
    Plan plan;
    Transport* tr = nullptr;
    int64_t halo_cap = 0;
    int64_t nnz_i = 0;
    int64_t glob_nnz = 0;          // arcs of the whole graph
    int32_t seg_long = 0;          // R37 long-row segment length of this job (0: every segment kSeg edges)
    int64_t kernels = 0;
    int64_t dev_bytes = 0;
    std::vector<void*> allocs;
    // f1 peer memory: every buffer another rank reads or writes lives in ONE allocation (the only one exported
    // through CUDA IPC -- small cudaMallocs may be sub-allocated and cannot be exported one by one)
    char* arena = nullptr;
    int64_t arena_off = 0, arena_size = 0;
    void* d_dx2 = nullptr;         // second dX buffer (alternating layers)
    float* d_gflat2 = nullptr;     // second weight-gradient buffer (all-reduce parity)
    double* d_scal2 = nullptr;
    uint64_t* d_pflags = nullptr;  // device barrier flag slots [32]
    std::vector<double> times;
    std::vector<cudaEvent_t> ev;              // timing events, 2 per phase slot
    // --- per-epoch host copies of counts
    double p = 1.0, inv_p = 1.0;
    int64_t n_halo = 0, n_sent = 0, nnz_kept = 0;
    int64_t n_seg_fwd = 0, n_seg_bwd = 0;
    std::vector<int64_t> recv_off, send_off;  // [m+1] rows
    // --- device plan
    int64_t* d_row_ptr = nullptr;  int32_t* d_col_enc = nullptr;
    int32_t* d_cand_gid = nullptr; int32_t* d_cand_key = nullptr; int32_t* d_cand_payload = nullptr;
    int64_t n_cand = 0;
    int64_t* d_cand_seg = nullptr; // [2m+1] candidate segment offsets
    int32_t* d_br_len = nullptr;   // boundary-row lengths
    int64_t* d_br_ptr = nullptr;
    int32_t* d_tcol = nullptr;     // [ii_col ; br_col] columns of the transposed aggregation
    int64_t ii_nnz = 0;
    float* d_deg_in = nullptr;     // deg_G(v), inner
    float* d_rs_in = nullptr;      // 1/sqrt(deg+1), inner
    float* d_rs_bd = nullptr;      // 1/sqrt(deg+1), boundary
    int32_t* d_labels = nullptr;
    // --- per-epoch device
    uint8_t* d_flags = nullptr;    // keep flag per candidate
    int32_t* d_blk = nullptr;      // per-block counts / offsets for compaction
    int32_t* d_cand_out = nullptr; // compacted payloads: [U_b (|U|) ; S_local (ΣS)]
    int32_t* d_slot_of_b = nullptr;
    uint32_t* d_bkeep = nullptr;   // keep bit per boundary node (induce)
    int64_t* d_tile_row = nullptr;  // induce: first inner row whose first static arc lies in each 1024-arc chunk
    uint64_t* d_lb_state = nullptr; // decoupled look-back tile states (induce.cu): draw | induce | segs fwd | segs bwd
    unsigned* d_lb_ctr = nullptr;   // tile-order counters of those four chains (each reset by its last tile)
    int64_t lb_off_induce = 0, lb_off_segf = 0, lb_off_segb = 0;
    uint32_t lb_gen = 0;            // launch generation stamped into the tile states (nothing cleared per launch)
    int64_t* d_seg_pos = nullptr;  // [2m+1] compacted segment offsets
    int64_t* h_seg_pos = nullptr;  // pinned host copy
    uint32_t* d_ebits = nullptr;   // induce: keep bit per static edge
    int32_t* d_ewex = nullptr;     // induce: exclusive kept-arc prefix of every 32-arc word inside its tile
    int32_t* d_eblk = nullptr;     // induce: kept edges per 1024-edge block
    int64_t* d_eboff = nullptr;    // induce: scanned block offsets
    int64_t* d_ind_ptr = nullptr;  // induced CSR (n_in+1)
    int32_t* d_ind_col = nullptr;
    int32_t* d_row_cnt = nullptr;  // scratch per row counts
    int32_t* d_row_nseg = nullptr;
    int64_t* d_row_off = nullptr;  // scratch scans
    int64_t* d_row_soff = nullptr;
    int64_t* d_scan_tmp = nullptr;
    Seg* d_seg_fwd = nullptr;  int64_t seg_fwd_cap = 0;
    Seg* d_seg_bwd = nullptr;  int64_t seg_bwd_cap = 0;
    Seg* d_seg_static_fwd = nullptr; int64_t n_seg_static_fwd = 0;  // p = 1 / no boundary: static induced CSR
    int32_t* d_static_col = nullptr; int64_t* d_static_ptr = nullptr;
    int64_t n_seg_bwd_inner = 0;
    float* d_partial = nullptr;    // hub-row partial sums
    unsigned long long* d_spmm_work = nullptr;   // SpMM dynamic scheduling: [next segment, warps done] (self-resetting)
    int32_t* d_spmm_arrive = nullptr;  // fused split-row fixup: segments of each split row finished (by first segment)
    int64_t* d_split_sf = nullptr;  int64_t n_split_sf = 0;      // split rows of the static forward segments
    int64_t* d_split_bwd = nullptr; int64_t n_split_bwd_inner = 0; // [static inner part ; per-epoch halo part]
    int64_t* d_split_fwd = nullptr;                                  // per-epoch induced forward segments
    int64_t n_split_fwd = 0, n_split_bwd = 0;                        // this epoch's list lengths
    int64_t fwd_hub_n = 0;          // per-epoch forward list: hub-row segments at [seg_fwd_cap - fwd_hub_n, seg_fwd_cap)
    float* d_cscale = nullptr;     // per-column scale (GCN forward)
    float* d_gat = nullptr;          // f4 / R45 GAT scalars: per layer el, er (stacked rows) and softmax max / 1/Σ
                                     // (inner rows), then c, selfds, del (inner), der (stacked)
    void* d_gat_dy = nullptr;        // GAT dY, (n_in + halo_cap) x maxd storage
    float* d_gat_qp = nullptr;       // GAT Q / P (fp32 weighted sums), (n_in + halo_cap) x maxd
    bool multilabel = false;         // f4 / R44: sigmoid BCE + F1-micro (bns_set_multilabel)
    uint8_t* d_targets = nullptr;    // n_in x C multi-hot targets
    void* d_x0cache = nullptr;       // f1 / R43: X^(0) rows of every boundary node, B_i order (BNS_CACHE_INPUT_HALO)
    uint32_t* d_scat_mask = nullptr; // a12 merged scatter: peers holding each owner row (bit j), world <= 32
    int32_t* d_scat_pos = nullptr;   // ... and the row's position in the returned buffer, n_in x world
    // --- activations (storage type T: float or bf16)
    std::vector<void*> H;          // H[l], l = 0..L-1: (n_in + halo_cap) x dp[l]
    std::vector<void*> Z;          // Z[l], l = 1..L: n_in x dp[l-1]
    float* d_logits = nullptr;     // n_in x dp[L]
    float* d_dlogits = nullptr;
    void* d_dpre = nullptr;        // n_in x maxd (T)
    void* d_dxcat = nullptr;       // n_in x 2 maxd (T) : [dZ' | dXself]
    void* d_dx = nullptr;          // (n_in + halo_cap) x maxd (T)
    void* d_dh = nullptr;          // n_in x maxd (T): gradient w.r.t. H^(l) inner rows (after accumulation)
    std::vector<void*> dH_keep;    // debug copies of dH^l (fp32) per layer (only if retained)
    void* d_sendbuf = nullptr;     // n_send x maxd (T)
    void* d_gradbuf = nullptr;     // n_send x maxd (T)
    int32_t maxd = 0;
    // --- weights
    std::vector<float*> Wpad;      // fp32 padded weights per layer
    std::vector<void*> Wt;         // storage-type copy (bf16 in BNS_BF16; == Wpad in FP32)
    std::vector<int64_t> wrows, wcols;   // padded shape per layer
    std::vector<void*> WT;         // bf16 W^T [wcols][wkw] for the tcgen05 forward (K-major B operand)
    // --- R42 transform-first SAGE layers (bit l-1 of tf_mask <=> layer l)
    uint32_t tf_mask = 0;
    void* d_tfy = nullptr;         // (n_in + halo_cap) x 2 dout: forward [Y | S], backward [dY | dPre]
    std::vector<void*> Wcat;       // storage type [W_top | W_bot]: dpin x 2 dpout (SIMT forward B, dX B operand)
    std::vector<void*> WTtf;       // bf16 [W_top | W_bot]^T: 2 dpout x K64 (tcgen05 forward B operand)
    std::vector<int64_t> wkw;      // K of W^T: each concat half padded to a multiple of 64
    bool use_tc = false;           // tcgen05 GEMMs (BNS_BF16)
    // --- f2: Adam + dropout
    int optimizer = 0;
    double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
    int64_t adam_t = 0;
    float* d_adam_m = nullptr;     // logical-size moments, all layers flat (hostw_n)
    float* d_adam_v = nullptr;
    double drop = 0.0;
    uint64_t drop_seed = 0, epoch_id = 0;
    std::vector<void*> Xd;         // dropped-out layer inputs [inner ; halo] (storage type), per layer
    int32_t* d_rowgid = nullptr;   // global id of every stacked row [V_i ; U_i]
    float* d_gflat = nullptr;      // all-reduce buffer: Σ_l padded dW (fp32)
    int64_t gflat_n = 0;
    std::vector<int64_t> goff;     // per-layer offset in gflat
    float* d_splitk = nullptr;     // split-K partials
    int64_t splitk_cap = 0;
    float* d_tr = nullptr;         // fp32 tensor-core dW: transposed operands [A^T ; D^T] (node dimension contiguous)
    int64_t tr_cap = 0;
    double* d_scal = nullptr;      // [loss_sum, correct] (all-reduced)
    double* d_lpart = nullptr;     // per-block loss partials
    int32_t* d_nonfinite = nullptr;
    const int* d_abort = nullptr;  // peer transports: mapped barrier-timeout flag (update kernels skip when set)
    int last_splitk = 1;           // split-K factor of the last tcgen05 weight-gradient GEMM (bns_gemm reports it)
    // bf16 epochs: the split-K reductions of all layers' weight gradients run as ONE launch after the backward
    // (splitk_flush); partial slices of the pending layers sit side by side in d_splitk
    struct RedJob {
        const float* part; int S; int64_t M, N, zs, gap_row, gap; float* out; int64_t ldo;
    };
    int num_sms = 148;             // multiprocessors of cfg.device (persistent grids)
    bool defer_red = false;
    std::vector<RedJob> red_jobs;
    int64_t splitk_used = 0;
    // --- f3: edge samplers (BES / DropEdge); allocated by the first bns_sample_edges
    int sampler = 0;               // BNS_SAMPLER_* of the last draw
    float nscale = 1.f;            // neighbour-sum scale (DropEdge: 1/q on every arc; else 1)
    bool edge_ready = false;
    int32_t* d_vgid = nullptr;     // inner gids
    int32_t* d_erow = nullptr;     // row of every static forward arc
    int64_t* d_tptr = nullptr;     // transposed rows [A_II rows ; boundary rows], n_in + n_bd + 1
    int32_t* d_terow = nullptr;    // row of every transposed arc
    int64_t tnnz = 0;
    int32_t* d_ind_tcol = nullptr; int64_t* d_ind_tptr = nullptr;
    int32_t* d_trow_nseg = nullptr; int64_t* d_trow_soff = nullptr;
    Seg* d_eseg_bwd = nullptr; int64_t* d_esplit_bwd = nullptr;
    float* d_hostw = nullptr;      // staging for host-pointer weights (flat)
    int64_t n_train_global = 0;
    int64_t n_train_local = 0;
};

// the per-epoch forward segment list puts the hub rows' segments first in claim order (not for GAT, whose weight
// kernels walk the list front to back); BNS_SPMM_LPT=0 keeps plain row order (A/B)
inline bool fwd_lpt(const Ctx& c) {
    const char* e = std::getenv("BNS_SPMM_LPT");
    return c.layer != BNS_LAYER_GAT && !(e && e[0] == '0');
}

// kernel launchers (kernels.cu / gemm.cu)
struct Launch;

}  // namespace bns
