/* bns.h -- C ABI of libbns.so: the per-epoch hot path of BNS-GCN (Wan et al., MLSys'22, arXiv 2203.10983)
 * on B200 (sm_100a).
 *
 * The three main calls follow the paper's statement of the problem, Algorithm 1:
 *   bns_setup            Alg.1 inputs "partition number m, partition id i, graph partition G_i, boundary node set
 *                        B_i, node feature X_i, label Y_i" and l.1-2 (V_i, H^(0) = X_i).
 *   bns_sample_boundary  Alg.1 l.4-7: Bernoulli(p) selection of U_i ⊆ B_i, node-induced
 *                        subgraph on V_i ∪ U_i, and the send lists S_{i,j} = U_j ∩ V_i.
 *   bns_epoch            Alg.1 l.8-14: L x (send/recv H_{S_{i,j}} -> GCN layer), loss,
 *                        backward with boundary-gradient exchange, AllReduce, SGD update.
 *
 * Process model: one context per process and GPU, rank r == partition id i, world == m.  The three main calls are
 * COLLECTIVE: every rank calls them in the same order with identical p / seed / epoch / lr.
 * Transports: NONE (world == 1), NCCL (one process per GPU; grouped ncclSend/ncclRecv + ncclAllReduce), LOCAL
 * (several contexts of one process, each driven by its own host thread; halo rows are pulled with device copies
 * -- used to run multi-partition parity on a single GPU), or IPC (one process per GPU, peer memory: SURVEY §8(f) f1,
 * see BNS_PEER_MEMORY).
 *
 * Readings of the paper where it is silent are numbered R1..R35.  The ones that
 * shape this ABI: R1 mean denominator = full-graph degree; R3 1/p applied on the receiving side as a column scale
 * (exchanged rows are bit-exact copies); R7 Philox4x32-10 keep(u,i) = out.x < floor(p*2^32) with
 * ctr = {u, i, epoch_lo, epoch_hi}, key = {seed_lo, seed_hi}; R8 loss = global mean CE over train nodes (labels >= 0),
 * sum-all-reduced; R14 weight layout; R18 acc = train accuracy of this epoch's sampled forward; R24 U_i ordered by
 * (owner, gid); R27 "broadcast U_i" replaced by recomputation under the shared counter-based RNG.
 *
 * Errors: no C++ exception crosses the ABI.  BNS_ERR_INVALID leaves the context unchanged.  BNS_ERR_RUNTIME (any
 * CUDA / NCCL failure) makes the context sticky-failed: every later call returns BNS_ERR_STATE.  The message of
 * the last error is bns_last_error(ctx) (or bns_last_error(NULL) for errors raised before a context exists).
 */
#ifndef BNS_H_
#define BNS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BNS_OK = 0,
    BNS_ERR_INVALID = 1,    /* bad argument; context unchanged */
    BNS_ERR_RUNTIME = 2,    /* CUDA / NCCL / transport failure; context becomes sticky-failed */
    BNS_ERR_STATE = 3,      /* call out of order (bns_epoch before any bns_sample_boundary) or failed context */
    BNS_ERR_OOM = 4,        /* device allocation failed, or a draw exceeded the halo capacity sized by max_p */
    BNS_ERR_NONFINITE = 5   /* global loss not finite; no weight update applied */
} bns_status;

typedef enum {
    BNS_LAYER_SAGE_MEAN = 0,  /* GraphSAGE-mean: h_v = σ(W · CONCAT(z_v, h_v)), z_v = mean aggregate */
    BNS_LAYER_GCN = 1,        /* GCN: Z = P H W, P = D~^-1/2 (A+I) D~^-1/2 (App. A) */
    BNS_LAYER_GAT = 2         /* f4 / R45: one-head GAT (Table tab:gat): Y = H W, e_vu =
                                 LeakyReLU_0.2(Y_v a_l + Y_u a_r), alpha = softmax over the sampled neighbours and v
                                 itself, h'_v = σ(Σ_u alpha_vu Y_u); weights (d_in + 2) x d_out rows [W ; a_l ; a_r] */
} bns_layer;

typedef enum {
    BNS_FP32 = 0,   /* fp32 storage of H / Z / halo rows / gradients, fp32 accumulation, fp32 GEMM */
    BNS_BF16 = 1    /* bf16 storage of H / Z / halo / GEMM operands, fp32 accumulation, fp32 master weights,
                       tcgen05 bf16 tensor-core GEMM (R19) */
} bns_precision;

typedef enum {
    BNS_TRANSPORT_NONE = 0,   /* world must be 1 */
    BNS_TRANSPORT_NCCL = 1,   /* cfg.nccl_id: 128-byte ncclUniqueId, identical on all ranks (bns_get_unique_id) */
    BNS_TRANSPORT_LOCAL = 2,  /* cfg.group: in-process group from bns_group_create(world) */
    BNS_TRANSPORT_NULL_EMULATE = 3, /* BENCHMARKING ONLY: run one rank of an m-rank job alone on one GPU; the
                                       exchanges and the all-reduce are no-ops, so outputs are not the method's */
    BNS_TRANSPORT_IPC = 4     /* SURVEY §8(f) f1, one process per GPU (several processes may share a GPU): the exchanges
                                 and the all-reduce run over peer memory (BNS_PEER_MEMORY semantics, implied).  Buffer
                                 handles (cudaIpcMemHandle_t) and setup-time integers move through cfg.allgather; no
                                 NCCL communicator is created.  cfg.allgather == NULL -> BNS_ERR_INVALID. */
} bns_transport;

/* cfg.flags */
#define BNS_PLAN_ONLY               0x1u  /* host plan only: no device memory, no kernels (CPU-testable) */
#define BNS_DEBUG_EXCHANGE_INDICES  0x2u  /* also exchange the sampled gid lists and check them against the
                                             recomputed S_{i,j} (R27); mismatch -> BNS_ERR_RUNTIME */
#define BNS_TIMING                  0x4u  /* record CUDA events per phase; read with BNS_Q_TIMES */
#define BNS_RETAIN_GRADS            0x8u  /* keep a copy of dL/dH^(l) per layer for BNS_Q_DH (parity tests) */
/* GraphSAGE layers whose (8-padded) output is narrower than their input are evaluated transform-first by default
 * (R42): [Y | S] = H [W_top | W_bot] on every stacked row, then z'_v = (1/deg_G(v)) Σ_u c_u Y_u + S_v -- the same
 * layer by linearity, with the neighbour gather at the narrow width (Reddit: 608 -> 256, 256 -> 41).  Z^(l) is then
 * not materialised (BNS_Q_Z fails with BNS_ERR_STATE on those layers).  This flag keeps aggregate-first everywhere. */
#define BNS_NO_TRANSFORM_FIRST      0x10u
/* the input features never change, so with this flag bns_setup exchanges every boundary node's
 * X^(0) row once (collective, the p = 1 lists) into a per-rank cache of |B_i| rows, and each epoch's layer-1 halo is
 * gathered locally from it (U_i ⊆ B_i) instead of being packed and exchanged: identical values, no layer-1 message
 * (R43).  Costs |B_i| x dims[0] stored elements of HBM. */
#define BNS_CACHE_INPUT_HALO        0x20u
/* SURVEY §8(f) f1, with transport LOCAL (IPC implies it): the exchange steps are fused with their producer / consumer
 * over peer memory instead of staged copies --
 *   a4 + a5: the receiving rank gathers its halo rows H_{U_i} straight from the owners' H^(l-1)
 *            (one kernel; no pack, no send buffer, no message);
 *   a11 + a12: each owner adds the peers' halo-row gradients of its rows read straight from the
 *            peers' dX, local value first then peers ascending (R25; one kernel);
 *   a13: every rank sums all ranks' weight gradients in rank order (bitwise equal on every rank).
 * Ordering between ranks: device-side flag barriers (system-scope release / acquire, 20 s timeout -> the epoch
 * fails with BNS_ERR_RUNTIME instead of hanging).  Results are bitwise those of the LOCAL transport. */
#define BNS_PEER_MEMORY             0x40u
/* R48: bns_step(p, seed, e) also enqueues the draw of (p, seed, e + 1) after the epoch's update kernels, before the
 * closing stream sync, so the per-peer counts of the next draw reach the host with that sync.  The next
 * bns_step(p, seed, e + 1) then starts its epoch at once: one host wait per step instead of two (the draw kernels
 * and their results are unchanged).  A step with other arguments discards the prefetch and draws as usual.  After
 * such a bns_step the context's current draw IS the prefetched one: bns_epoch / bns_query see draw e + 1. */
#define BNS_PREFETCH_DRAW           0x80u

/* Host all-gather used by BNS_TRANSPORT_IPC at setup (buffer handles, counts) and by debug exchanges: copy `bytes`
 * bytes from `send` of every rank into recv[rank * bytes]; every rank calls it with the same `bytes`.  Return 0 on
 * success.  Called only from inside bns_setup / bns_sample_boundary on the calling thread. */
typedef int32_t (*bns_allgather_fn)(const void* send, void* recv, int64_t bytes, void* user);

typedef struct bns_ctx bns_ctx;
typedef struct bns_group bns_group;

typedef struct {
    int32_t rank;             /* partition id i, 0 <= rank < world */
    int32_t world;            /* number of partitions m */
    int32_t device;           /* CUDA device ordinal */
    int32_t transport;        /* bns_transport */
    const uint8_t* nccl_id;   /* 128 bytes when transport == NCCL, else NULL */
    bns_group* group;         /* when transport == LOCAL, else NULL */
    void* stream;             /* cudaStream_t to enqueue on, or NULL: the library creates a non-blocking stream */
    int32_t num_layers;       /* L >= 1 */
    const int32_t* dims;      /* L+1 logical dims: dims[0] = feature dim, dims[L] = number of classes C (<= 256) */
    int32_t layer;            /* bns_layer */
    int32_t precision;        /* bns_precision */
    double max_p;             /* halo capacity: <= 0 or >= 1 -> sized for p = 1 (|B_i| rows); else
                                 ceil(max_p*|B_i| + 8 sqrt(max_p*|B_i|) + 64) rows (R34) */
    uint32_t flags;           /* BNS_PLAN_ONLY | BNS_DEBUG_EXCHANGE_INDICES | BNS_TIMING | BNS_RETAIN_GRADS |
                                 BNS_NO_TRANSFORM_FIRST | BNS_CACHE_INPUT_HALO | BNS_PEER_MEMORY |
                                 BNS_PREFETCH_DRAW */
    bns_allgather_fn allgather;   /* transport IPC: host all-gather over the ranks (e.g. a torch gloo group); else NULL */
    void* allgather_user;         /* passed through to allgather */
} bns_config;

/* ncclGetUniqueId into out[128] (rank 0 calls it and broadcasts the bytes, e.g. over a torch process group). */
bns_status bns_get_unique_id(uint8_t* out);

/* In-process group for BNS_TRANSPORT_LOCAL: `world` contexts, each driven by its own host thread. */
bns_status bns_group_create(int32_t world, bns_group** out);
void bns_group_destroy(bns_group* g);

/* Build this rank's plan (V_i, B_i ordered by (owner, gid), D_{i->j} = B_j ∩ V_i, static CSR split, degrees),
 * allocate every device buffer at its capacity (no allocation happens later), copy to HBM, attach the transport.
 *   num_nodes, indptr[num_nodes+1] (int64), indices[indptr[N]] (int32): HOST, full graph, symmetric, ascending
 *       columns, no self loops, no duplicates.  Borrowed for the call only.
 *   part_of[num_nodes]: HOST, values in [0, world); every partition non-empty.
 *   features: HOST, row-major |V_i| x dims[0] fp32 -- this rank's inner nodes in ascending global id (X_i).
 *   labels:   HOST, [|V_i|] int32: -1 = not a training node, else [0, dims[L]) (Y_i).
 * Collective (transport attach).  Invalid input -> BNS_ERR_INVALID with a message in bns_last_error(NULL). */
bns_status bns_setup(const bns_config* cfg, int64_t num_nodes, const int64_t* indptr, const int32_t* indices,
                     const int32_t* part_of, const float* features, const int32_t* labels, bns_ctx** out);

/* Alg.1 l.4-7: draw U_i (keep(u, i) for u in B_i) and recompute S_{i,j} (keep(u, j) for u in D_{i->j}),
 * build the induced subgraph over V_i ∪ U_i.  p in [0, 1] (p = 0 allowed: isolated partitions).  Returns after
 * one stream sync (the per-peer counts come to the host for the exchange sizes).  Collective in effect (no
 * messages are sent).  p > max_p, or a draw larger than the halo capacity -> BNS_ERR_OOM. */
bns_status bns_sample_boundary(bns_ctx* ctx, double p, uint64_t seed, uint64_t epoch);

/* the edge-sampling baselines of PAPER.md:676-688 (Table tab:bes), on the same exchange
 * machinery; a replacement for bns_sample_boundary before bns_epoch.
 *   sampler BNS_SAMPLER_BES: every cross-partition arc (v <- u), v in V_i, u in B_i, kept with probability q;
 *       intra-partition arcs always kept.  BNS_SAMPLER_DROPEDGE: every arc of the graph kept with probability q.
 *   Arc draw (R40): keep(v <- u) = Philox4x32-10(ctr = {v, u, e_lo, e_hi}, key = {seed_lo ^ 0xED6E, seed_hi}).x
 *       < floor(q 2^32), global ids; each direction of an edge is its own arc.
 *   U_i = the u in B_i with at least one kept arc into V_i (B order); the owner recomputes the same draws for S_{i,j}
 *   (R27).  Kept arcs carry the column scale 1/q (R41: unbiased; BES intra arcs 1; GCN self loops 1, never
 *   dropped); the SAGE denominator stays deg_G(v).
 *   q in [0, 1].  The first call allocates the per-arc buffers (two int32 per static arc).  A halo larger than
 *   the capacity (cfg.max_p) -> BNS_ERR_OOM.  Same sync / collective behaviour as bns_sample_boundary. */
typedef enum { BNS_SAMPLER_BNS = 0, BNS_SAMPLER_BES = 1, BNS_SAMPLER_DROPEDGE = 2 } bns_sampler;
bns_status bns_sample_edges(bns_ctx* ctx, int32_t sampler, double q, uint64_t seed, uint64_t epoch);

/* Alg.1 l.8-14 with the draw of the last bns_sample_boundary (or bns_sample_edges).
 *   weights[l], l < L: fp32 row-major, SAGE (2*dims[l]) x dims[l+1] (rows [0,dims[l]) multiply z_v, R14),
 *       GCN dims[l] x dims[l+1], GAT (dims[l] + 2) x dims[l+1] ([W ; a_l ; a_r]).  Device pointers on cfg.device
 *       (updated in place: W <- W - lr*g) or host
 *       pointers (copied in and out inside the call).
 *   grads[l]: same shapes, out: the all-reduced gradient g (identical on every rank); may be NULL.
 *   loss: out, global mean cross-entropy over train nodes (R8); acc: out, global train accuracy (R18, R22).
 * Returns after a stream sync.  Collective. */
bns_status bns_epoch(bns_ctx* ctx, float* const* weights, float lr, float* const* grads, double* loss, double* acc);

/* One training step = bns_sample_boundary(p, seed, epoch) followed by bns_epoch(weights, lr, grads, loss, acc) in
 * one call (Alg.1 l.4-14): the same work and results, without a return to the caller between the draw and the epoch
 * (the host only waits for the per-peer counts, then enqueues the epoch; with BNS_PREFETCH_DRAW not even that when
 * the previous step prefetched this draw, R48).  Errors as the two calls. */
bns_status bns_step(bns_ctx* ctx, double p, uint64_t seed, uint64_t epoch, float* const* weights, float lr,
                    float* const* grads, double* loss, double* acc);

/* the paper's training recipe ("a GraphSAGE model with an Adam optimizer",
 * per-dataset dropout).  Defaults after bns_setup: SGD (Alg.1 l.14), no dropout.
 *   optimizer: BNS_OPT_SGD or BNS_OPT_ADAM (bias-corrected Adam; beta1, beta2, eps as usual).  The Adam moments live
 *       on the device (fp32, allocated here -- not in the hot path) and advance on every bns_epoch call (R39);
 *       calling this function resets them.
 *   dropout: rate r in [0, 1) applied to the input of every layer, inner and halo rows alike (R38):
 *       keep(u, c, l, e) = Philox4x32-10(ctr = {u, c >> 2, l, epoch_lo}, key = {seed_lo ^ 0xD809, seed_hi})
 *       .word[c & 3] >= floor(r 2^32), kept values scaled by 1/(1-r); u = global node id, l = layer (1-based),
 *       epoch = the epoch of the last bns_sample_boundary.  Keyed by the global id, so every copy of a row agrees.
 * Not collective; every rank must pass the same values.  Invalid values -> BNS_ERR_INVALID. */
typedef enum { BNS_OPT_SGD = 0, BNS_OPT_ADAM = 1 } bns_optimizer;
bns_status bns_set_training(bns_ctx* ctx, int32_t optimizer, double beta1, double beta2, double eps, double dropout,
                            uint64_t dropout_seed);

/* the multi-label task of the Yelp experiments: targets = HOST uint8
 * |V_i| x dims[L] in {0, 1} (this rank's inner rows, ascending global id; copied), the train rows are those with
 * labels >= 0 as given to bns_setup.  Then bns_epoch's loss is the mean over train rows x classes of
 * BCE(σ(x), y) = softplus(x) - y x, dLogits = (σ(x) - y) / (N_train C), and acc is F1-micro of x > 0 over the train
 * rows (R44; all-reduced TP / FP / FN).  NULL restores the single-label cross entropy.  Not collective; every rank
 * must choose the same mode.  A value other than 0 / 1 -> BNS_ERR_INVALID. */
bns_status bns_set_multilabel(bns_ctx* ctx, const uint8_t* targets);

/* Debug / parity queries: copy a host-side view into host_dst (capacity in bytes); *written = bytes written.
 * Row tensors are returned as fp32 row-major with LOGICAL dims (padding stripped), inner rows in ascending gid. */
typedef enum {
    BNS_Q_COUNTS = 0,        /* int64[6 + 2m]: n_in, n_bd, |U_i|, ΣS, nnz_i(static), nnz_kept(epoch),
                                recv_cnt[m] (rows received from each owner), send_cnt[m] (rows sent to each peer) */
    BNS_Q_INNER = 1,         /* int32[n_in]  V_i global ids */
    BNS_Q_BOUNDARY = 2,      /* int32[n_bd]  B_i global ids, (owner, gid) order */
    BNS_Q_BOUNDARY_OFF = 3,  /* int64[m+1]   owner offsets into B_i */
    BNS_Q_SENDCAND = 4,      /* int32[ΣD]    D_{i->j} global ids, concatenated over j ascending */
    BNS_Q_SENDCAND_OFF = 5,  /* int64[m+1] */
    BNS_Q_MASK = 6,          /* uint8[n_bd]  keep flag of every B_i entry (this epoch) */
    BNS_Q_HALO = 7,          /* int32[|U_i|] U_i global ids (owner-major, gid ascending) */
    BNS_Q_HALO_OFF = 8,      /* int64[m+1] */
    BNS_Q_SEND = 9,          /* int32[ΣS]    S_{i,j} global ids, concatenated over j ascending */
    BNS_Q_SEND_OFF = 10,     /* int64[m+1] */
    BNS_Q_H = 11,            /* layer l in [0,L]: H^(l) inner rows, n_in x dims[l] (l = L: logits) */
    BNS_Q_Z = 12,            /* layer l in [1,L]: aggregation output Z^(l), n_in x dims[l-1] */
    BNS_Q_DH = 13,           /* layer l in [1,L]: dL/dH^(l) after owner accumulation (l = L: dLogits);
                                needs BNS_RETAIN_GRADS (the fp32 dLogits are only written then) */
    BNS_Q_HALO_ROWS = 14,    /* layer l in [1,L]: received halo rows of the layer-l input, |U_i| x dims[l-1] */
    BNS_Q_INDUCED = 15,      /* int64[n_in+1] row pointers then int32[nnz_kept] local columns of the induced
                                subgraph (inner j -> j, halo slot s -> n_in + s) */
    BNS_Q_TIMES = 16,        /* double[BNS_NUM_PHASES]: ms accumulated per phase since setup (BNS_TIMING) */
    BNS_Q_STATIC_CSR = 17,   /* int64[n_in+1] then int32[nnz_i]: static rows, columns encoded inner j -> j,
                                boundary index b -> -(b+1) (plan, available in BNS_PLAN_ONLY) */
    BNS_Q_MEMORY = 18,       /* int64[2]: device bytes allocated by the context, peak device bytes */
    BNS_Q_KERNEL_COUNT = 19, /* int64[1]: kernels launched by this context since setup */
    BNS_Q_INDUCED_T = 20,    /* edge samplers: int64[n_in+n_bd+1] row pointers then int32[nnz] local inner columns
                                of the sampled TRANSPOSED aggregation (rows: inner u, then boundary index b) */
    BNS_Q_TF_LAYERS = 21,    /* int32[1]: bit l-1 set <=> layer l runs transform-first (R42) */
    BNS_Q_BOUNDARY_ROW = 22  /* int32[n_bd]: row of B_i[b] in its owner's V_j, i.e. where the peer-memory pull reads
                                it (f1; plan, available in BNS_PLAN_ONLY) */
} bns_query_what;

enum { BNS_PH_SAMPLE = 0, BNS_PH_INDUCE, BNS_PH_PACK, BNS_PH_EXCHANGE, BNS_PH_SPMM_FWD, BNS_PH_GEMM_FWD,
       BNS_PH_LOSS, BNS_PH_GEMM_BWD, BNS_PH_SPMM_BWD, BNS_PH_EXCHANGE_BWD, BNS_PH_SCATTER, BNS_PH_ALLREDUCE,
       BNS_PH_UPDATE, BNS_PH_EPOCH_TOTAL, BNS_PH_SAMPLE_TOTAL, BNS_NUM_PHASES };

bns_status bns_query(bns_ctx* ctx, int32_t what, int32_t layer, void* host_dst, int64_t capacity_bytes,
                     int64_t* written);

/* Per-phase CUDA events on (1) or off (0) for the following calls; the context must have been created with
 * BNS_TIMING (else BNS_ERR_STATE).  Each phase event pair costs a few microseconds of pipeline drain: ~0.3 ms per
 * epoch at m = 8 on the Reddit shape, so throughput runs at small partitions switch them off. */
bns_status bns_set_timing(bns_ctx* ctx, int32_t on);

/* One dense GEMM of the epoch (§8(a) a7 / a9: Alg.1 l.10 "update" φ = W·CONCAT(z, h), and
 * its gradients, l.12 PAPER.md:290), run in isolation by the SAME kernels bns_epoch launches -- so the tensor-core
 * GEMMs can be checked element by element at full size against a float64 product of the same operands.  No context
 * needed; all pointers are caller-owned DEVICE memory, row-major, leading dimensions in elements.
 *   precision  BNS_BF16: tcgen05 kind::f16 (bf16 operands, fp32 accumulation in TMEM); BNS_FP32: split-TF32 (4 MMAs)
 *              (tcgen05 kind::tf32 on hi / lo splits of fp32 operands, fp32 accumulation) -- every operand and
 *              output below is then fp32.
 *   kind 0  FWD     C[M x N] = [A0 | A1] · W, A0 / A1 M x K (lda; A1 may be NULL), B = Wᵀ stored [N][Kw] with each
 *                   concat half zero-padded to a multiple of 64 columns (Kw = 64⌈K/64⌉ or 2·64⌈K/64⌉), ldb = Kw;
 *                   flags bit 0 = ReLU epilogue, bit 1 = fp32 output (else the storage type).
 *   kind 1  WGRAD   C[K x N] (fp32, ldc) = A0ᵀ · B, A0 M x K (lda), B M x N (ldb) -- M (the node count) is the
 *                   reduction, split over CTAs (split-K) and reduced in a fixed order.
 *   kind 2  WGRAD2  C[2K x N] (fp32) = [A0 | A1]ᵀ · B in one launch (the GraphSAGE dW_z / dW_h pair; K % 128 == 0).
 *   kind 3  DX      C[M x N] (storage type) = A0 · Bᵀ, A0 M x K (lda), B [N][K] (ldb); columns < scale_cols x
 *                   rowscale[row] (rowscale may be NULL).
 * stream: cudaStream_t (NULL = legacy default).  *splits (may be NULL) receives the split-K factor used (kinds 1-2;
 * 1 otherwise).  Returns after a stream sync; errors: BNS_ERR_INVALID (shapes / kind / precision), BNS_ERR_RUNTIME. */
bns_status bns_gemm(int32_t precision, int32_t kind, int64_t M, int64_t N, int64_t K, const void* A0, const void* A1,
                    int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, const float* rowscale,
                    int64_t scale_cols, int32_t flags, void* stream, int32_t* splits);

/* The cudaStream_t the context enqueues on (as void*). */
void* bns_stream(const bns_ctx* ctx);

const char* bns_last_error(const bns_ctx* ctx);
void bns_destroy(bns_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* BNS_H_ */
