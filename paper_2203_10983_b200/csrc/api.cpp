// api.cpp -- the C ABI (include/bns.h): context lifecycle, setup (a0), per-epoch orchestration of Algorithm 1
// (PAPER.md:269-297), debug queries.  Every arithmetic step runs in the sm_100a kernels; this file only sequences
// launches, exchanges and the two host syncs per epoch (counts after sampling; loss/acc at the end).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>

#include <thread>

#include "common.h"
#include "kernels.h"
#include "layers.h"
#include "transport.h"

struct bns_ctx {
    bns::Ctx c;
};

namespace bns {
namespace {

thread_local std::string g_err;

bns_status fail(bns_ctx* h, const Error& e) {
    if (h) {
        h->c.err = e.what();
        if (e.code == BNS_ERR_RUNTIME) h->c.failed = true;
    } else {
        g_err = e.what();
    }
    return e.code;
}

template <typename F>
bns_status guard(bns_ctx* h, F&& f) {
    try {
        f();
        return BNS_OK;
    } catch (const Error& e) {
        return fail(h, e);
    } catch (const std::bad_alloc&) {
        return fail(h, Error(BNS_ERR_OOM, "host allocation failed"));
    } catch (const std::exception& e) {
        return fail(h, Error(BNS_ERR_RUNTIME, e.what()));
    }
}

void* dalloc(Ctx& c, size_t bytes) {
    if (bytes == 0) bytes = 16;
    bytes = (bytes + 255) & ~size_t(255);
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(BNS_ERR_OOM, "cudaMalloc(" + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e));
    }
    c.allocs.push_back(p);
    c.dev_bytes += (int64_t)bytes;
    return p;
}

// a buffer peers access (f1): carved from the arena when the context runs a peer-memory transport
void* salloc(Ctx& c, size_t bytes) {
    if (!c.arena) return dalloc(c, bytes);
    bytes = (std::max<size_t>(bytes, 16) + 255) & ~size_t(255);
    if (c.arena_off + (int64_t)bytes > c.arena_size) throw Error(BNS_ERR_RUNTIME, "peer arena too small");
    void* p = c.arena + c.arena_off;
    c.arena_off += (int64_t)bytes;
    return p;
}

bool peer_mode(const bns_config& cfg) {
    return cfg.world > 1 && (cfg.transport == BNS_TRANSPORT_IPC ||
                             (cfg.transport == BNS_TRANSPORT_LOCAL && (cfg.flags & BNS_PEER_MEMORY)));
}

template <typename T>
T* upload(Ctx& c, const std::vector<T>& v) {
    T* d = static_cast<T*>(dalloc(c, v.size() * sizeof(T)));
    if (!v.empty()) BNS_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

size_t tsize(const Ctx& c) { return c.prec == BNS_BF16 ? 2 : 4; }

// logical rows of layer l's weight at the ABI: SAGE 2 d_in, GCN d_in, GAT d_in + 2 ([W ; a_l ; a_r])
int64_t wlogical_rows(const Ctx& c, int l) {
    return c.layer == BNS_LAYER_SAGE_MEAN ? 2 * (int64_t)c.dims[l]
           : c.layer == BNS_LAYER_GAT ? (int64_t)c.dims[l] + 2 : (int64_t)c.dims[l];
}

void validate(const bns_config* cfg, int64_t N, const int64_t* indptr, const int32_t* indices, const int32_t* part_of) {
    if (!cfg) throw Error(BNS_ERR_INVALID, "cfg is NULL");
    if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) throw Error(BNS_ERR_INVALID, "bad rank/world");
    if (cfg->num_layers < 1 || !cfg->dims) throw Error(BNS_ERR_INVALID, "num_layers < 1 or dims NULL");
    for (int l = 0; l <= cfg->num_layers; ++l)
        if (cfg->dims[l] <= 0) throw Error(BNS_ERR_INVALID, "dims must be positive");
    if (cfg->dims[cfg->num_layers] > 256) throw Error(BNS_ERR_INVALID, "at most 256 classes (dims[L])");
    if (cfg->layer != BNS_LAYER_SAGE_MEAN && cfg->layer != BNS_LAYER_GCN && cfg->layer != BNS_LAYER_GAT)
        throw Error(BNS_ERR_INVALID, "bad layer");
    if (cfg->precision != BNS_FP32 && cfg->precision != BNS_BF16) throw Error(BNS_ERR_INVALID, "bad precision");
    if (cfg->world > 1 && cfg->transport != BNS_TRANSPORT_NCCL && cfg->transport != BNS_TRANSPORT_LOCAL &&
        cfg->transport != BNS_TRANSPORT_NULL_EMULATE && cfg->transport != BNS_TRANSPORT_IPC &&
        !(cfg->flags & BNS_PLAN_ONLY))
        throw Error(BNS_ERR_INVALID, "world > 1 needs transport NCCL, LOCAL or IPC");
    if (cfg->transport == BNS_TRANSPORT_IPC && !cfg->allgather && !(cfg->flags & BNS_PLAN_ONLY))
        throw Error(BNS_ERR_INVALID, "transport IPC needs cfg.allgather");
    if (N < 1 || !indptr || !indices || !part_of) throw Error(BNS_ERR_INVALID, "empty graph or NULL arrays");
    if (N >= INT32_MAX) throw Error(BNS_ERR_INVALID, "num_nodes must fit int32");
    if (indptr[0] != 0) throw Error(BNS_ERR_INVALID, "indptr[0] != 0");
    for (int64_t v = 0; v < N; ++v) {
        if (indptr[v + 1] < indptr[v]) throw Error(BNS_ERR_INVALID, "indptr not monotone at row " + std::to_string(v));
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
            int32_t u = indices[e];
            if (u < 0 || u >= N) throw Error(BNS_ERR_INVALID, "column id out of range at row " + std::to_string(v));
            if (u == v) throw Error(BNS_ERR_INVALID, "self loop at node " + std::to_string(v));
            if (e > indptr[v] && indices[e - 1] >= u)
                throw Error(BNS_ERR_INVALID, "columns not strictly ascending at row " + std::to_string(v));
        }
    }
    // symmetric (bns.h): every arc v -> u has its reverse u -> v (D_{i->j} = B_j ∩ V_i relies on it); rows are
    // sorted by now, so each reverse is a binary search -- split over host threads (1.6 B arcs at C5)
    {
        const int nt = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<int64_t> bad(nt, -1);
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                for (int64_t v = N * t / nt; v < N * (t + 1) / nt; ++v)
                    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
                        const int32_t u = indices[e];
                        if (!std::binary_search(indices + indptr[u], indices + indptr[u + 1], (int32_t)v)) {
                            bad[t] = v;
                            return;
                        }
                    }
            });
        for (auto& x : th) x.join();
        for (int64_t v : bad)
            if (v >= 0) throw Error(BNS_ERR_INVALID, "graph not symmetric: an arc of row " + std::to_string(v) +
                                                         " has no reverse arc");
    }
    std::vector<int64_t> cnt(cfg->world, 0);
    for (int64_t v = 0; v < N; ++v) {
        if (part_of[v] < 0 || part_of[v] >= cfg->world)
            throw Error(BNS_ERR_INVALID, "part_of out of range at node " + std::to_string(v));
        cnt[part_of[v]]++;
    }
    for (int j = 0; j < cfg->world; ++j)
        if (cnt[j] == 0) throw Error(BNS_ERR_INVALID, "partition " + std::to_string(j) + " is empty");
}

// host-built segments over a static CSR whose row r spans [ptr[r], ptr[r+1]) (+ptr_base in the column array)
std::vector<Seg> host_segments(const std::vector<int64_t>& ptr, int64_t rows, int64_t ptr_base, int64_t row_base,
                              int32_t seg_long) {
    std::vector<Seg> s;
    for (int64_t r = 0; r < rows; ++r) {
        int64_t len = ptr[r + 1] - ptr[r];
        int32_t ns = seg_count(len, seg_long);
        int64_t first = (int64_t)s.size();
        for (int32_t k = 0; k < ns; ++k) {
            Seg g;
            g.row = (int32_t)(row_base + r);
            g.nseg = ns;
            g.e0 = ptr_base + ptr[r] + (int64_t)k * seg_len(len, seg_long);
            g.e1 = std::min(ptr_base + ptr[r + 1], g.e0 + seg_len(len, seg_long));
            g.first = first;
            s.push_back(g);
        }
    }
    return s;
}

void collect_times(Ctx& c) {
    if (!c.timing) return;
    for (size_t s = 0; s + 1 < c.ev_used; s += 2) {
        float ms = 0.f;
        BNS_CUDA(cudaEventElapsedTime(&ms, c.ev[s], c.ev[s + 1]));
        c.times[c.ev_phase[s / 2]] += ms;
    }
    c.ev_used = 0;
}

void setup_device(Ctx& c, const float* features, const int32_t* labels) {
    BNS_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, c.cfg.device));
    Plan& P = c.plan;
    const int m = c.cfg.world;
    BNS_CUDA(cudaSetDevice(c.cfg.device));
    if (c.cfg.stream) {
        c.stream = static_cast<cudaStream_t>(c.cfg.stream);
    } else {
        BNS_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        c.own_stream = true;
    }
    const int L = c.L;
    c.maxd = 0;
    for (int l = 0; l <= L; ++l) c.maxd = std::max<int32_t>(c.maxd, c.dp[l]);
    if (c.cfg.max_p > 0.0 && c.cfg.max_p < 1.0) {
        double mu = c.cfg.max_p * (double)P.n_bd;
        c.halo_cap = std::min<int64_t>(P.n_bd, (int64_t)std::ceil(mu + 8.0 * std::sqrt(mu) + 64.0));
    } else {
        c.halo_cap = P.n_bd;
    }
    c.nnz_i = P.row_ptr[P.n_in];
    // R37: long-row segments only for jobs with >= kLongJobNnz arcs per partition (a job-wide constant: every rank
    // of the job makes the same choice)
    c.seg_long = c.glob_nnz / std::max(1, c.cfg.world) >= kLongJobNnz ? kSegLong : 0;
    if (const char* e = std::getenv("BNS_SEG_LONG")) c.seg_long = std::max(0, std::atoi(e));   // tests / A/B
    const size_t ts = tsize(c);
    if (peer_mode(c.cfg)) {   // f1: one exported allocation for everything the peers touch
        const size_t rows = (size_t)(P.n_in + c.halo_cap);
        int64_t gn = 0;
        for (int l = 0; l < L; ++l)
            gn += (c.layer == BNS_LAYER_SAGE_MEAN ? 2 * (int64_t)c.dp[l]
                   : c.layer == BNS_LAYER_GAT ? (int64_t)c.dp[l] + 8 : (int64_t)c.dp[l]) * c.dp[l + 1];
        size_t total = 2 * rows * c.maxd * ts + (size_t)P.n_send * c.maxd * ts + 2 * (size_t)gn * 4 + 4096 + 64 * 256;
        for (int l = 0; l < L; ++l) total += rows * c.dp[l] * ts;
        c.arena_size = (int64_t)((total + (2u << 20) - 1) & ~size_t((2u << 20) - 1));
        c.arena = static_cast<char*>(dalloc(c, (size_t)c.arena_size));
        c.arena_off = 0;
        c.d_pflags = static_cast<uint64_t*>(salloc(c, 32 * sizeof(uint64_t)));
        BNS_CUDA(cudaMemset(c.d_pflags, 0, 32 * sizeof(uint64_t)));
        c.d_dx2 = salloc(c, rows * c.maxd * ts);
        c.d_gflat2 = static_cast<float*>(salloc(c, (size_t)gn * sizeof(float)));
        BNS_CUDA(cudaMemset(c.d_gflat2, 0, (size_t)gn * sizeof(float)));
        c.d_scal2 = static_cast<double*>(salloc(c, 4 * sizeof(double)));
        BNS_CUDA(cudaMemset(c.d_scal2, 0, 4 * sizeof(double)));
    }

    // ---- static plan on device
    c.d_row_ptr = upload(c, P.row_ptr);
    c.d_col_enc = upload(c, P.col_enc);
    {   // induce (induce.cu): first inner row whose first static arc lies in each 1024-arc chunk
        const int64_t nt = (c.nnz_i + 1023) / 1024;
        std::vector<int64_t> tr(nt + 1);
        int64_t r = 0;
        for (int64_t t = 0; t <= nt; ++t) {
            const int64_t e0 = std::min<int64_t>(t * 1024, c.nnz_i + 1);
            while (r <= P.n_in && P.row_ptr[r] < e0) ++r;
            tr[t] = r;
        }
        tr[nt] = P.n_in + 1;
        c.d_tile_row = upload(c, tr);
    }
    c.n_cand = P.n_bd + P.n_send;
    std::vector<int32_t> gid(c.n_cand), key(c.n_cand), pay(c.n_cand);
    for (int64_t b = 0; b < P.n_bd; ++b) { gid[b] = P.B[b]; key[b] = c.cfg.rank; pay[b] = (int32_t)b; }
    for (int j = 0; j < m; ++j)
        for (int64_t e = P.D_off[j]; e < P.D_off[j + 1]; ++e) {
            gid[P.n_bd + e] = P.V[P.D_local[e]];
            key[P.n_bd + e] = j;
            pay[P.n_bd + e] = P.D_local[e];
        }
    c.d_cand_gid = upload(c, gid);
    c.d_cand_key = upload(c, key);
    c.d_cand_payload = upload(c, pay);
    std::vector<int64_t> cseg(2 * m + 1);
    for (int k = 0; k <= m; ++k) cseg[k] = P.B_off[k];
    for (int k = 1; k <= m; ++k) cseg[m + k] = P.n_bd + P.D_off[k];
    c.d_cand_seg = upload(c, cseg);
    c.d_br_ptr = upload(c, P.br_ptr);
    std::vector<int32_t> tcol(P.ii_col);
    c.ii_nnz = (int64_t)P.ii_col.size();
    tcol.insert(tcol.end(), P.br_col.begin(), P.br_col.end());
    c.d_tcol = upload(c, tcol);
    std::vector<float> inv_deg(P.n_in), rs_in(P.n_in), rs_bd(P.n_bd);
    for (int64_t r = 0; r < P.n_in; ++r) {
        inv_deg[r] = P.deg_in[r] > 0 ? (float)(1.0 / (double)P.deg_in[r]) : 0.f;
        rs_in[r] = (float)(1.0 / std::sqrt((double)P.deg_in[r] + 1.0));
    }
    for (int64_t b = 0; b < P.n_bd; ++b) rs_bd[b] = (float)(1.0 / std::sqrt((double)P.deg_bd[b] + 1.0));
    c.d_deg_in = upload(c, inv_deg);   // holds 1/deg_G (0 for isolated nodes)
    c.d_rs_in = upload(c, rs_in);
    c.d_rs_bd = upload(c, rs_bd);

    // static segments: backward inner part (A_II, columns in d_tcol[0, ii_nnz)) ...
    std::vector<Seg> sb = host_segments(P.ii_ptr, P.n_in, 0, 0, c.seg_long);
    c.n_seg_bwd_inner = (int64_t)sb.size();
    int64_t halo_seg_cap = P.n_bd + (int64_t)P.br_col.size() / kSeg + 1;
    c.seg_bwd_cap = c.n_seg_bwd_inner + halo_seg_cap;
    c.d_seg_bwd = static_cast<Seg*>(dalloc(c, c.seg_bwd_cap * sizeof(Seg)));
    BNS_CUDA(cudaMemcpy(c.d_seg_bwd, sb.data(), sb.size() * sizeof(Seg), cudaMemcpyHostToDevice));
    // ... and the full static induced CSR used when every boundary node is kept (p = 1)
    std::vector<int32_t> scol(P.col_enc.size());
    for (size_t k = 0; k < scol.size(); ++k)
        scol[k] = P.col_enc[k] >= 0 ? P.col_enc[k] : (int32_t)(P.n_in + (-P.col_enc[k] - 1));
    c.d_static_col = upload(c, scol);
    std::vector<Seg> sf = host_segments(P.row_ptr, P.n_in, 0, 0, c.seg_long);
    c.n_seg_static_fwd = (int64_t)sf.size();
    c.d_seg_static_fwd = upload(c, sf);
    c.seg_fwd_cap = P.n_in + c.nnz_i / kSeg + 1;
    c.d_seg_fwd = static_cast<Seg*>(dalloc(c, c.seg_fwd_cap * sizeof(Seg)));
    int64_t seg_max = std::max({c.seg_fwd_cap, c.seg_bwd_cap, c.n_seg_static_fwd});
    c.d_partial = static_cast<float*>(dalloc(c, (size_t)seg_max * c.maxd * sizeof(float)));
    c.d_spmm_work = static_cast<unsigned long long*>(dalloc(c, 64));
    c.d_spmm_arrive = static_cast<int32_t*>(dalloc(c, (size_t)seg_max * sizeof(int32_t)));
    BNS_CUDA_HOLD(cudaMemsetAsync(c.d_spmm_work, 0, 64, c.stream));
    BNS_CUDA_HOLD(cudaMemsetAsync(c.d_spmm_arrive, 0, (size_t)seg_max * sizeof(int32_t), c.stream));
    // split (hub) row lists: first segment of every row with more than one segment
    auto split_list = [](const std::vector<Seg>& s) {
        std::vector<int64_t> l;
        for (size_t k = 0; k < s.size(); ++k)
            if (s[k].nseg > 1 && (int64_t)k == s[k].first) l.push_back((int64_t)k);
        return l;
    };
    {
        std::vector<int64_t> lf = split_list(sf), lb = split_list(sb);
        c.n_split_sf = (int64_t)lf.size();
        c.d_split_sf = upload(c, lf);
        c.n_split_bwd_inner = (int64_t)lb.size();
        c.d_split_bwd = static_cast<int64_t*>(dalloc(c, (lb.size() + P.n_bd + 1) * sizeof(int64_t)));
        if (!lb.empty())
            BNS_CUDA(cudaMemcpy(c.d_split_bwd, lb.data(), lb.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
        c.d_split_fwd = static_cast<int64_t*>(dalloc(c, (P.n_in + 1) * sizeof(int64_t)));
    }

    // ---- per-epoch scratch
    c.d_flags = static_cast<uint8_t*>(dalloc(c, c.n_cand));
    c.d_blk = static_cast<int32_t*>(dalloc(c, (c.n_cand / 1024 + 2) * sizeof(int32_t)));
    c.d_cand_out = static_cast<int32_t*>(dalloc(c, (c.n_cand + 1) * sizeof(int32_t)));
    c.d_slot_of_b = static_cast<int32_t*>(dalloc(c, (P.n_bd + 1) * sizeof(int32_t)));
    c.d_bkeep = static_cast<uint32_t*>(dalloc(c, ((P.n_bd + 31) / 32 + 1) * sizeof(uint32_t)));
    {   // single-pass scans (induce.cu): tile states of the draw, the induce pass and the two segment chains
        c.lb_off_induce = c.n_cand / 1024 + 1;
        c.lb_off_segf = c.lb_off_induce + c.nnz_i / 8192 + 1;
        c.lb_off_segb = c.lb_off_segf + P.n_in / 1024 + 1;
        const int64_t n = c.lb_off_segb + P.n_bd / 1024 + 1;
        c.d_lb_state = static_cast<uint64_t*>(dalloc(c, n * sizeof(uint64_t)));
        BNS_CUDA(cudaMemset(c.d_lb_state, 0, n * sizeof(uint64_t)));
        c.d_lb_ctr = static_cast<unsigned*>(dalloc(c, 16 * sizeof(unsigned)));
        BNS_CUDA(cudaMemset(c.d_lb_ctr, 0, 16 * sizeof(unsigned)));
    }
    c.d_seg_pos = static_cast<int64_t*>(salloc(c, (2 * m + 1 + 8) * sizeof(int64_t)));
    BNS_CUDA(cudaMemset(c.d_seg_pos, 0, (2 * m + 1 + 8) * sizeof(int64_t)));   // slots a draw does not write stay 0
    BNS_CUDA(cudaMallocHost(&c.h_seg_pos, (2 * m + 1 + 8) * sizeof(int64_t)));
    c.d_ind_ptr = static_cast<int64_t*>(dalloc(c, (P.n_in + 1) * sizeof(int64_t)));
    c.d_ind_col = static_cast<int32_t*>(dalloc(c, (c.nnz_i + 1) * sizeof(int32_t)));
    {
        const int64_t nb = (c.nnz_i + 1023) / 1024;
        c.d_ebits = static_cast<uint32_t*>(dalloc(c, (nb * 32 + kInduceTileArcs / 32 + 32) * sizeof(uint32_t)));
        c.d_ewex = static_cast<int32_t*>(dalloc(c, (nb * 32 + kInduceTileArcs / 32 + 32) * sizeof(int32_t)));
        c.d_eblk = static_cast<int32_t*>(dalloc(c, (nb + 1) * sizeof(int32_t)));
        c.d_eboff = static_cast<int64_t*>(dalloc(c, (nb + 2) * sizeof(int64_t)));
    }
    const int64_t rmax = std::max<int64_t>(P.n_in, P.n_bd) + 1;
    c.d_row_cnt = static_cast<int32_t*>(dalloc(c, rmax * sizeof(int32_t)));
    c.d_row_nseg = static_cast<int32_t*>(dalloc(c, rmax * sizeof(int32_t)));
    c.d_row_soff = static_cast<int64_t*>(dalloc(c, (rmax + 1) * sizeof(int64_t)));
    c.d_scan_tmp = static_cast<int64_t*>(dalloc(c, (std::max(rmax, c.n_cand) / 1024 + 16) * 3 * sizeof(int64_t)));
    c.d_cscale = static_cast<float*>(dalloc(c, (P.n_in + c.halo_cap + 1) * sizeof(float)));
    if (m > 1 && m <= 32) {
        c.d_scat_mask = static_cast<uint32_t*>(dalloc(c, (P.n_in + 1) * sizeof(uint32_t)));
        c.d_scat_pos = static_cast<int32_t*>(dalloc(c, (size_t)(P.n_in + 1) * m * sizeof(int32_t)));
    }

    // ---- activations
    c.H.assign(L, nullptr);
    c.Z.assign(L + 1, nullptr);
    for (int l = 0; l < L; ++l) c.H[l] = salloc(c, (size_t)(P.n_in + c.halo_cap) * c.dp[l] * ts);
    for (int l = 1; l <= L; ++l) c.Z[l] = dalloc(c, (size_t)P.n_in * c.dp[l - 1] * ts);
    c.d_logits = static_cast<float*>(dalloc(c, (size_t)P.n_in * c.dp[L] * sizeof(float)));
    c.d_dlogits = static_cast<float*>(dalloc(c, (size_t)P.n_in * c.dp[L] * sizeof(float)));
    c.d_dpre = dalloc(c, (size_t)P.n_in * c.maxd * ts);
    c.d_dxcat = dalloc(c, (size_t)P.n_in * 2 * c.maxd * ts);
    c.d_dx = salloc(c, (size_t)(P.n_in + c.halo_cap) * c.maxd * ts);
    c.d_sendbuf = salloc(c, (size_t)P.n_send * c.maxd * ts);
    c.d_gradbuf = dalloc(c, (size_t)P.n_send * c.maxd * ts);
    if (c.retain) {
        c.dH_keep.assign(L + 1, nullptr);
        for (int l = 1; l < L; ++l) c.dH_keep[l] = dalloc(c, (size_t)P.n_in * c.dp[l] * ts);
    }
    BNS_CUDA(cudaMemset(c.H[0], 0, (size_t)(P.n_in + c.halo_cap) * c.dp[0] * ts));
    if (P.n_in > 0) {
        float* stage = nullptr;
        BNS_CUDA(cudaMalloc(&stage, (size_t)P.n_in * c.dims[0] * sizeof(float)));
        BNS_CUDA(cudaMemcpy(stage, features, (size_t)P.n_in * c.dims[0] * sizeof(float), cudaMemcpyHostToDevice));
        launch_to_storage(c, stage, P.n_in, c.dims[0], c.dims[0], c.H[0], c.dp[0]);
        BNS_CUDA(cudaStreamSynchronize(c.stream));
        BNS_CUDA(cudaFree(stage));
    }
    std::vector<int32_t> lab(labels, labels + P.n_in);
    c.d_labels = upload(c, lab);

    // ---- weights and gradients
    c.Wpad.assign(L, nullptr);
    c.Wt.assign(L, nullptr);
    c.wrows.assign(L, 0);
    c.wcols.assign(L, 0);
    c.goff.assign(L + 1, 0);
    c.WT.assign(L, nullptr);
    c.wkw.assign(L, 0);
    {
        // tensor-core GEMMs in both modes (bf16: kind::f16; fp32: split-TF32 (4 MMAs)); BNS_NO_TC=1 selects the SIMT kernels
        const char* no_tc = std::getenv("BNS_NO_TC");
        c.use_tc = !(no_tc && no_tc[0] == '1');
    }
    int64_t wmax = 0, wlog = 0;
    for (int l = 0; l < L; ++l) {
        // padded rows: SAGE [z-half ; h-half] 2 dp; GCN dp; GAT [W (dp) ; a_l ; a_r ; 6 zero rows]
        c.wrows[l] = c.layer == BNS_LAYER_SAGE_MEAN ? 2 * (int64_t)c.dp[l]
                     : c.layer == BNS_LAYER_GAT ? (int64_t)c.dp[l] + 8 : (int64_t)c.dp[l];
        c.wcols[l] = c.dp[l + 1];
        c.goff[l + 1] = c.goff[l] + c.wrows[l] * c.wcols[l];
        wmax = std::max(wmax, c.wrows[l] * c.wcols[l]);
        wlog += wlogical_rows(c, l) * c.dims[l + 1];
        c.Wpad[l] = static_cast<float*>(dalloc(c, c.wrows[l] * c.wcols[l] * sizeof(float)));
        c.Wt[l] = (c.prec == BNS_BF16) ? dalloc(c, c.wrows[l] * c.wcols[l] * 2) : (void*)c.Wpad[l];
        c.wkw[l] = (c.layer == BNS_LAYER_SAGE_MEAN ? 2 : 1) * ((int64_t)(c.dp[l] + 63) / 64 * 64);
        if (c.use_tc) c.WT[l] = dalloc(c, c.wcols[l] * c.wkw[l] * tsize(c));
    }
    // R42: transform-first SAGE layers (narrower padded output than input), unless BNS_NO_TRANSFORM_FIRST
    c.tf_mask = 0;
    c.Wcat.assign(L, nullptr);
    c.WTtf.assign(L, nullptr);
    int64_t tfw = 0;
    if (c.layer == BNS_LAYER_SAGE_MEAN && !(c.cfg.flags & BNS_NO_TRANSFORM_FIRST))
        for (int l = 0; l < L; ++l)
            if (c.dp[l + 1] < c.dp[l]) {
                c.tf_mask |= 1u << l;
                tfw = std::max<int64_t>(tfw, 2 * (int64_t)c.dp[l + 1]);
                c.Wcat[l] = dalloc(c, (size_t)c.dp[l] * 2 * c.dp[l + 1] * ts);
                if (c.use_tc) c.WTtf[l] = dalloc(c, (size_t)2 * c.dp[l + 1] * ((c.dp[l] + 63) / 64 * 64) * tsize(c));
            }
    if (c.layer == BNS_LAYER_GAT) {   // f4 / R45: Y buffer, per-layer attention scalars, dY
        for (int l = 0; l < L; ++l) tfw = std::max<int64_t>(tfw, c.dp[l + 1]);
        const int64_t R = P.n_in + c.halo_cap;
        c.d_gat = static_cast<float*>(dalloc(c, (size_t)(2 * L * R + 2 * L * P.n_in + 3 * P.n_in + 2 * R + 16) * sizeof(float)));
        c.d_gat_dy = dalloc(c, (size_t)R * c.maxd * ts);
        c.d_gat_qp = static_cast<float*>(dalloc(c, (size_t)R * c.maxd * sizeof(float)));
    }
    if (c.tf_mask || c.layer == BNS_LAYER_GAT) c.d_tfy = dalloc(c, (size_t)(P.n_in + c.halo_cap) * tfw * ts);
    c.gflat_n = c.goff[L];
    c.d_gflat = static_cast<float*>(salloc(c, c.gflat_n * sizeof(float)));
    c.splitk_cap = 32 * wmax;
    if (c.use_tc && c.prec == BNS_BF16 && c.layer != BNS_LAYER_GAT) {
        // every layer's partial slices at once (deferred reduction, splitk_flush): at most ceil(148 / tiles) slices
        // of an (M2 = 128-padded d_in + d_in) x d_out product per layer (gemm_tc.cu's split rule)
        int64_t tot = 0;
        for (int l = 0; l < L; ++l) {
            const int64_t K = c.dp[l], N = c.dp[l + 1], M2 = (K + 255) / 256 * 256 + K;   // CTA-pair padding
            const int64_t tiles = ((M2 + 127) / 128) * ((N + 255) / 256);
            tot += std::max<int64_t>(1, (148 + tiles - 1) / tiles) * M2 * N;
        }
        c.splitk_cap = std::max(c.splitk_cap, tot);
    }
    if (c.use_tc && c.prec == BNS_FP32) {   // fp32 dW runs K-major on transposed operands (gemm_tc.cu)
        int64_t kn = 0, w2 = 0;
        for (int l = 0; l < L; ++l) {
            kn = std::max<int64_t>(kn, 2 * (int64_t)c.dp[l] + 2 * (int64_t)c.dp[l + 1]);
            w2 = std::max<int64_t>(w2, 2 * (int64_t)c.dp[l] * c.dp[l + 1]);
        }
        const int64_t rows = P.n_in + c.halo_cap;
        c.tr_cap = kn * ((rows + 3) / 4 * 4);
        c.d_tr = static_cast<float*>(dalloc(c, c.tr_cap * sizeof(float)));
        // one partial slice per 512 nodes (16 k-blocks of 32: the split-TF32 accumulation-chain cap)
        c.splitk_cap = std::max<int64_t>(c.splitk_cap, ((rows + 511) / 512 + 1) * w2);
    }
    c.d_splitk = static_cast<float*>(dalloc(c, c.splitk_cap * sizeof(float)));
    c.d_scal = static_cast<double*>(salloc(c, 4 * sizeof(double)));
    c.d_lpart = static_cast<double*>(dalloc(c, 4 * 2048 * sizeof(double)));   // k_xent / k_bce block partials
    c.d_nonfinite = static_cast<int32_t*>(dalloc(c, 16));
    c.d_hostw = static_cast<float*>(dalloc(c, 2 * wlog * sizeof(float)));
    c.hostw_n = wlog;

    if (c.timing) {
        c.ev.resize(256);
        c.ev_phase.assign(128, 0);
        for (auto& e : c.ev) BNS_CUDA(cudaEventCreate(&e));
    }
    c.times.assign(BNS_NUM_PHASES, 0.0);
    c.recv_off.assign(m + 1, 0);
    c.send_off.assign(m + 1, 0);
    BNS_CUDA(cudaStreamSynchronize(c.stream));
}

// f3: the edge samplers' static per-arc arrays, built by the first bns_sample_edges (not on the BNS path)
void edge_init(Ctx& c) {
    if (c.edge_ready) return;
    const Plan& P = c.plan;
    const int64_t n_rows = P.n_in + P.n_bd;
    c.d_vgid = upload(c, P.V);
    std::vector<int32_t> erow(c.nnz_i);
    for (int64_t r = 0; r < P.n_in; ++r)
        for (int64_t e = P.row_ptr[r]; e < P.row_ptr[r + 1]; ++e) erow[e] = (int32_t)r;
    c.d_erow = upload(c, erow);
    c.tnnz = c.ii_nnz + (int64_t)P.br_col.size();
    if (c.tnnz != c.nnz_i) throw Error(BNS_ERR_RUNTIME, "transposed arc count != static arc count");
    std::vector<int64_t> tptr(n_rows + 1);
    for (int64_t r = 0; r <= P.n_in; ++r) tptr[r] = P.ii_ptr[r];
    for (int64_t b = 1; b <= P.n_bd; ++b) tptr[P.n_in + b] = c.ii_nnz + P.br_ptr[b];
    std::vector<int32_t> terow(c.tnnz);
    for (int64_t r = 0; r < n_rows; ++r)
        for (int64_t e = tptr[r]; e < tptr[r + 1]; ++e) terow[e] = (int32_t)r;
    c.d_tptr = upload(c, tptr);
    c.d_terow = upload(c, terow);
    c.d_ind_tcol = static_cast<int32_t*>(dalloc(c, (c.tnnz + 1) * sizeof(int32_t)));
    c.d_ind_tptr = static_cast<int64_t*>(dalloc(c, (n_rows + 1) * sizeof(int64_t)));
    c.d_trow_nseg = static_cast<int32_t*>(dalloc(c, (n_rows + 1) * sizeof(int32_t)));
    c.d_trow_soff = static_cast<int64_t*>(dalloc(c, (n_rows + 2) * sizeof(int64_t)));
    c.d_eseg_bwd = static_cast<Seg*>(dalloc(c, c.seg_bwd_cap * sizeof(Seg)));
    c.d_esplit_bwd = static_cast<int64_t*>(dalloc(c, (c.n_split_bwd_inner + P.n_bd + 1) * sizeof(int64_t)));
    c.edge_ready = true;
}

// f1 / R43: one p = 1 exchange of the input rows (every send candidate D_{i->j} to j, received in B_i order) into
// the per-rank boundary-feature cache; layer 1 then gathers its halo rows from it every epoch
void fill_x0_cache(Ctx& c) {
    const Plan& P = c.plan;
    const size_t ts = tsize(c);
    const int64_t d0 = c.dp[0];
    c.d_x0cache = dalloc(c, (size_t)(P.n_bd + 1) * d0 * ts);
    launch_pack_rows(c, c.H[0], d0, c.d_cand_payload + P.n_bd, P.n_send, c.d_sendbuf, (int32_t)d0);
    c.tr->exchange(c, c.d_sendbuf, P.D_off.data(), c.d_x0cache, P.B_off.data(), d0 * ts);
    BNS_CUDA(cudaStreamSynchronize(c.stream));
}

// ---------------------------------------------------------------------------------------------
// bns_sample_boundary / bns_sample_edges: a1-a3
// ---------------------------------------------------------------------------------------------
// a1-a3 enqueued: the draw, the induced lists / segments, and the async copy of the per-peer counts to the host
void draw_enqueue(Ctx& c, int sampler, double p, uint64_t seed, uint64_t epoch) {
    const int m = c.cfg.world;
    const uint64_t T = (uint64_t)std::floor(p * 4294967296.0);
    const bool edges = sampler != BNS_SAMPLER_BNS;
    c.sampler = sampler;
    c.p = p;
    if (sampler == BNS_SAMPLER_DROPEDGE) {   // R41: 1/q on every arc -> neighbour-sum scale, no column scale
        c.inv_p = 1.0;
        c.nscale = p > 0.0 ? (float)(1.0 / p) : 0.f;
    } else {                                 // BNS 1/p, BES 1/q: column scale of the halo columns (R3, R41)
        c.inv_p = p > 0.0 ? 1.0 / p : 0.0;
        c.nscale = 1.f;
    }
    c.sampled = false;
    std::unique_ptr<PhaseTimer> total(new PhaseTimer(c, BNS_PH_SAMPLE_TOTAL));
    {
        PhaseTimer t(c, BNS_PH_SAMPLE);
        if (edges) launch_sample_edges(c, T, seed, epoch);
        else launch_sample_fused(c, T, seed, epoch);
    }
    const bool has_bd = c.plan.n_bd > 0;
    c.fwd_mode = edges ? 2 : (!has_bd || T >= (1ull << 32)) ? 0 : (T == 0 ? 1 : 2);
    {
        PhaseTimer t(c, BNS_PH_INDUCE);
        if (edges) {
            launch_induce_edges(c, T, seed, epoch);
            launch_induce_bwd_edges(c, T, seed, epoch);
        } else {
            if (c.fwd_mode == 2) launch_induce_fused(c);
            launch_segments_fused(c, c.fwd_mode == 2);
        }
        if (c.layer == BNS_LAYER_GCN) launch_gcn_cscale(c);
    }
    total.reset();
    const int64_t nslot = 2 * m + 1 + 8;
    BNS_CUDA_HOLD(cudaMemcpyAsync(c.h_seg_pos, c.d_seg_pos, nslot * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
}

// the host side of a draw: wait for the counts (unless an earlier sync already covered the copy), size the epoch
void draw_finish(Ctx& c, uint64_t epoch, bool sync) {
    const int m = c.cfg.world;
    const bool edges = c.sampler != BNS_SAMPLER_BNS;
    const bool has_bd = c.plan.n_bd > 0;
    if (sync) BNS_CUDA(cudaStreamSynchronize(c.stream));
    const int64_t* sp = c.h_seg_pos;
    for (int j = 0; j <= m; ++j) c.recv_off[j] = sp[j] - sp[0];
    for (int j = 0; j <= m; ++j) c.send_off[j] = sp[m + j] - sp[m];
    c.n_halo = c.recv_off[m];
    c.n_sent = c.send_off[m];
    const int64_t* tot = sp + 2 * m + 1;
    if (c.fwd_mode == 0) { c.nnz_kept = c.nnz_i; c.n_seg_fwd = c.n_seg_static_fwd; c.n_split_fwd = c.n_split_sf; }
    else if (c.fwd_mode == 1) { c.nnz_kept = c.ii_nnz; c.n_seg_fwd = c.n_seg_bwd_inner; c.n_split_fwd = c.n_split_bwd_inner; }
    else { c.nnz_kept = tot[0]; c.n_seg_fwd = tot[1] + (edges ? 0 : tot[5]); c.n_split_fwd = tot[4]; }
    c.fwd_hub_n = (c.fwd_mode == 2 && !edges) ? tot[5] : 0;   // hub segments of the per-epoch forward list (LPT)
    if (edges) {
        c.n_seg_bwd = tot[6];
        c.n_split_bwd = tot[7];
    } else {
        c.n_seg_bwd = c.n_seg_bwd_inner + (has_bd ? tot[2] : 0);
        c.n_split_bwd = c.n_split_bwd_inner + (has_bd ? tot[3] : 0);
    }
    if (c.n_halo > c.halo_cap)
        throw Error(BNS_ERR_OOM, "sampled halo (" + std::to_string(c.n_halo) + " rows) exceeds capacity " +
                                     std::to_string(c.halo_cap) + " (raise cfg.max_p)");
    if (c.d_scat_mask) launch_scatter_prep(c, c.n_sent);
    if (c.debug_idx && m > 1) {
        // R27 check: exchange the gids of S_{i,j} and compare with U_i's owner segments
        std::vector<int32_t> sl(c.n_sent), ub(c.n_halo);
        if (c.n_sent)
            BNS_CUDA(cudaMemcpy(sl.data(), c.d_cand_out + c.n_halo, c.n_sent * 4, cudaMemcpyDeviceToHost));
        if (c.n_halo) BNS_CUDA(cudaMemcpy(ub.data(), c.d_cand_out, c.n_halo * 4, cudaMemcpyDeviceToHost));
        std::vector<int32_t> sg(c.n_sent);
        for (int64_t k = 0; k < c.n_sent; ++k) sg[k] = c.plan.V[sl[k]];
        int32_t* d_s = static_cast<int32_t*>(c.d_sendbuf);
        int32_t* d_r = static_cast<int32_t*>(c.d_gradbuf);
        if (c.n_sent) BNS_CUDA(cudaMemcpy(d_s, sg.data(), c.n_sent * 4, cudaMemcpyHostToDevice));
        int32_t* d_rr = static_cast<int32_t*>(c.d_dx);
        c.tr->exchange(c, d_s, c.send_off.data(), d_rr, c.recv_off.data(), 4);
        std::vector<int32_t> got(c.n_halo);
        BNS_CUDA(cudaStreamSynchronize(c.stream));
        if (c.n_halo) BNS_CUDA(cudaMemcpy(got.data(), d_rr, c.n_halo * 4, cudaMemcpyDeviceToHost));
        for (int64_t s = 0; s < c.n_halo; ++s)
            if (got[s] != c.plan.B[ub[s]])
                throw Error(BNS_ERR_RUNTIME, "BNS_DEBUG_EXCHANGE_INDICES: received gid != recomputed U_i at slot " +
                                                 std::to_string(s));
        (void)d_r;
    }
    collect_times(c);
    c.epoch_id = epoch;
    c.sampled = true;
}

void sample_boundary(Ctx& c, int sampler, double p, uint64_t seed, uint64_t epoch) {
    c.pf_pending = false;   // a prefetched draw (R48) is simply overwritten
    draw_enqueue(c, sampler, p, seed, epoch);
    draw_finish(c, epoch, true);
}

// R48: any call that reads the current draw first adopts a prefetched one (device buffers already hold it)
void settle(Ctx& c) {
    if (!c.pf_pending) return;
    c.pf_pending = false;
    draw_finish(c, c.pf_ep, true);
}

// ---------------------------------------------------------------------------------------------
// bns_epoch: a4-a14
// ---------------------------------------------------------------------------------------------
void epoch(Ctx& c, float* const* W_in, float lr, float* const* G_in, double* loss, double* acc) {
    Plan& P = c.plan;
    const int L = c.L, m = c.cfg.world;
    const size_t ts = tsize(c);
    const int64_t n_in = P.n_in;
    // c_u = 1/p only exists on halo columns; with no halo every column scale is 1 (the kernels then skip it)
    const float inv_p = (c.n_halo > 0) ? (float)c.inv_p : 1.f;

    std::unique_ptr<PhaseTimer> total(new PhaseTimer(c, BNS_PH_EPOCH_TOTAL));
    const bool peer = m > 1 && c.tr && c.tr->peer();   // f1: exchanges fused over peer memory
    if (peer) c.tr->begin_epoch(c);
    // weights may be host or device pointers
    cudaPointerAttributes attr{};
    bool host_w = false;
    if (cudaPointerGetAttributes(&attr, W_in[0]) != cudaSuccess) { cudaGetLastError(); host_w = true; }
    else host_w = (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged);
    std::vector<float*> W(L), G(L);
    std::vector<int64_t> wl(L);
    int64_t off = 0;
    for (int l = 0; l < L; ++l) {
        wl[l] = wlogical_rows(c, l) * c.dims[l + 1];
        if (host_w) {
            W[l] = c.d_hostw + off;
            G[l] = c.d_hostw + c.hostw_n + off;
            BNS_CUDA_HOLD(cudaMemcpyAsync(W[l], W_in[l], wl[l] * sizeof(float), cudaMemcpyHostToDevice, c.stream));
        } else {
            W[l] = W_in[l];
            G[l] = G_in ? G_in[l] : nullptr;
        }
        off += wl[l];
    }
    {
        PhaseTimer t(c, BNS_PH_UPDATE);
        launch_wpack_all(c, W.data());   // padded W, storage copy, W^T, and the R42 packs in one launch
    }
    const bool ebw = c.sampler != BNS_SAMPLER_BNS;   // f3: the sampled transposed CSR of this epoch
    EpochView ev;
    ev.fsegs = c.fwd_mode == 0 ? c.d_seg_static_fwd : (c.fwd_mode == 1 ? c.d_seg_bwd : c.d_seg_fwd);
    ev.fcol = c.fwd_mode == 0 ? c.d_static_col : (c.fwd_mode == 1 ? c.d_tcol : c.d_ind_col);
    ev.fsplit = c.fwd_mode == 0 ? c.d_split_sf : (c.fwd_mode == 1 ? c.d_split_bwd : c.d_split_fwd);
    ev.bsegs = ebw ? c.d_eseg_bwd : c.d_seg_bwd;
    ev.bcol = ebw ? c.d_ind_tcol : c.d_tcol;
    ev.bsplit = ebw ? c.d_esplit_bwd : c.d_split_bwd;
    ev.inv_p = inv_p;
    if (c.fwd_mode == 2 && c.fwd_hub_n > 0) {   // the per-epoch forward list: hub segments at its end, claimed first
        ev.fhub_n = c.fwd_hub_n;
        ev.fhub_base = c.seg_fwd_cap - c.fwd_hub_n;
    }
    const int32_t* S_local = c.d_cand_out + c.n_halo;
    const bool dropout = c.drop > 0.0;
    if (dropout) launch_halo_gid(c);

    // ------------------------------ forward (Alg.1 l.8-10) ------------------------------
    for (int l = 1; l <= L; ++l) {
        const int64_t din = c.dp[l - 1];
        void* Hin = c.H[l - 1];
        if (m > 1 && l == 1 && c.d_x0cache) {   // R43: layer-1 halo rows from the boundary-feature cache
            PhaseTimer t(c, BNS_PH_PACK);
            launch_pack_rows(c, c.d_x0cache, din, c.d_cand_out, c.n_halo, static_cast<char*>(Hin) + n_in * din * ts,
                             (int32_t)din);
        } else if (peer) {   // f1: pack + exchange = one gather from the owners' H^(l-1)
            PhaseTimer t(c, BNS_PH_EXCHANGE);
            c.tr->halo_pull(c, l, static_cast<char*>(Hin) + n_in * din * ts, din);
        } else if (m > 1) {
            {
                PhaseTimer t(c, BNS_PH_PACK);
                launch_pack_rows(c, Hin, din, S_local, c.n_sent, c.d_sendbuf, (int32_t)din);
            }
            PhaseTimer t(c, BNS_PH_EXCHANGE);
            c.tr->exchange(c, c.d_sendbuf, c.send_off.data(), static_cast<char*>(Hin) + n_in * din * ts,
                           c.recv_off.data(), din * ts);
        }
        if (dropout) {   // f2 / R38: the layer input as seen by the aggregation and the CONCAT self term
            PhaseTimer t(c, BNS_PH_UPDATE);
            launch_dropout(c, Hin, c.Xd[l - 1], n_in + c.n_halo, din, l);
            Hin = c.Xd[l - 1];
        }
        if (c.layer == BNS_LAYER_GAT) forward_layer_gat(c, ev, l, Hin);
        else if ((c.tf_mask >> (l - 1)) & 1u) forward_layer_tf(c, ev, l, Hin);
        else forward_layer_std(c, ev, l, Hin);
    }
    // ------------------------------ loss (l.11) ------------------------------
    {
        PhaseTimer t(c, BNS_PH_LOSS);
        const bool tfL = (c.tf_mask >> (L - 1)) & 1u;
        // R42 with a dX (L > 1): dPre goes straight into the dPre half of the [dY | dPre] operand, halo rows zeroed
        void* dpre = c.d_dpre;
        int64_t ldp = c.dp[L], nzero = 0;
        if (tf_dpre_in_tfy(c, L)) {
            dpre = static_cast<char*>(c.d_tfy) + c.dp[L] * ts;
            ldp = 2 * c.dp[L];
            nzero = c.n_halo;
        }
        if (c.multilabel)
            launch_bce(c, c.d_logits, c.dp[L], c.dims[L], c.retain ? c.d_dlogits : nullptr, dpre, tfL ? c.d_deg_in : nullptr,
                       tfL ? c.d_dxcat : nullptr, ldp, nzero);
        else
            launch_xent(c, c.d_logits, c.dp[L], c.dims[L], c.retain ? c.d_dlogits : nullptr, dpre, tfL ? c.d_deg_in : nullptr,
                        tfL ? c.d_dxcat : nullptr, ldp, nzero);
    }
    // ------------------------------ backward (l.12) ------------------------------
    // a12 (owner scatter-add of the returned halo gradients) is folded into the ReLU mask of the layer below when
    // one launch serves every peer (d_scat_mask) and no per-layer dH copy is kept: pend holds its sources
    ScatterIn pend{};
    const bool fold_scatter = m > 1 && c.d_scat_mask && !c.retain;
    c.defer_red = c.use_tc && c.prec == BNS_BF16 && c.layer != BNS_LAYER_GAT;   // one split-K reduce launch
    for (int l = L; l >= 1; --l) {
        const int64_t din = c.dp[l - 1], dout = c.dp[l];
        void* Hin = dropout ? c.Xd[l - 1] : c.H[l - 1];
        if (l < L) {
            PhaseTimer t(c, BNS_PH_GEMM_BWD);
            if (c.retain)
                BNS_CUDA_HOLD(cudaMemcpyAsync(c.dH_keep[l], c.d_dx, n_in * dout * ts, cudaMemcpyDeviceToDevice, c.stream));
            const bool tfl = (c.tf_mask >> (l - 1)) & 1u;   // R42: + dPre / deg_G into d_dxcat (unused there)
            launch_relu_mask(c, c.d_dx, c.H[l], dout, n_in, (int32_t)dout, c.d_dpre, tfl ? c.d_deg_in : nullptr,
                             tfl ? c.d_dxcat : nullptr, pend.mask ? &pend : nullptr);
            pend = ScatterIn{};
        }
        if (peer) c.d_dx = c.tr->dx_buffer(c, l);   // f1: layer l's dX; a peer may still read layer l+1's
        if (c.layer == BNS_LAYER_GAT) backward_layer_gat(c, ev, l, Hin);
        else if ((c.tf_mask >> (l - 1)) & 1u) backward_layer_tf(c, ev, l, Hin);
        else backward_layer_std(c, ev, l, Hin);
        if (l == 1) break;   // R29: no gradient w.r.t. the input features
        if (dropout) {   // R38: gradient w.r.t. the dropped-out input -> w.r.t. the layer input (all stacked rows)
            PhaseTimer t(c, BNS_PH_UPDATE);
            launch_dropout(c, c.d_dx, c.d_dx, n_in + c.n_halo, din, l);
        }
        if (peer) {   // f1: reverse exchange + scatter-add = one gather from the peers' dX halo rows
            PhaseTimer t(c, BNS_PH_SCATTER);
            if (fold_scatter && c.n_sent > 0 && c.tr->grad_barrier(c, l, &pend.peer, &pend.delta)) {
                pend.mask = c.d_scat_mask;
                pend.pos = c.d_scat_pos;
                pend.m = m;
            } else {
                c.tr->grad_scatter(c, l, din);
            }
        } else if (m > 1) {
            {
                PhaseTimer t(c, BNS_PH_EXCHANGE_BWD);
                c.tr->exchange(c, static_cast<char*>(c.d_dx) + n_in * din * ts, c.recv_off.data(), c.d_gradbuf,
                               c.send_off.data(), din * ts);
            }
            PhaseTimer t(c, BNS_PH_SCATTER);
            if (fold_scatter) {             // R25 in the ReLU mask of layer l - 1 (the next launch)
                if (c.n_sent > 0) {
                    pend.mask = c.d_scat_mask;
                    pend.pos = c.d_scat_pos;
                    pend.m = m;
                    pend.src = c.d_gradbuf;
                }
            } else if (c.d_scat_mask) {     // R25: local contribution first, then peers ascending, one launch
                launch_scatter_rows(c, c.d_dx, din, c.d_gradbuf, (int32_t)din);
            } else {
                for (int j = 0; j < m; ++j) {
                    if (j == c.cfg.rank) continue;
                    const int64_t n = c.send_off[j + 1] - c.send_off[j];
                    launch_scatter_add(c, c.d_dx, din, S_local + c.send_off[j],
                                       static_cast<char*>(c.d_gradbuf) + c.send_off[j] * din * ts, n, (int32_t)din);
                }
            }
        }
    }
    {
        PhaseTimer t(c, BNS_PH_GEMM_BWD);
        splitk_flush(c);   // every layer's dW from its split-K slices, one launch
        c.defer_red = false;
    }
    // ------------------------------ AllReduce (l.13) + update (l.14) ------------------------------
    if (m > 1) {
        PhaseTimer t(c, BNS_PH_ALLREDUCE);
        c.tr->allreduce(c, c.d_gflat, c.gflat_n, c.d_scal, c.multilabel ? 4 : 2);
    }
    {
        PhaseTimer t(c, BNS_PH_UPDATE);
        float* const* Gp = host_w ? G.data() : (G_in ? G.data() : nullptr);
        if (c.optimizer == BNS_OPT_ADAM) {
            ++c.adam_t;   // R39: one Adam step per bns_epoch call (taken back below if the step is skipped)
            launch_adam(c, W.data(), Gp, lr);
        } else {
            launch_sgd(c, W.data(), Gp, lr);
        }
    }
    total.reset();
    if (c.pf_want) {   // R48: the next draw rides on this epoch's closing sync (stream order keeps it after a4-a14)
        c.pf_want = false;
        draw_enqueue(c, BNS_SAMPLER_BNS, c.pf_p, c.pf_seed, c.pf_ep);
        c.pf_pending = true;
    }
    double scal[4] = {0.0, 0.0, 0.0, 0.0};
    int32_t nonfinite = 0;
    BNS_CUDA_HOLD(cudaMemcpyAsync(scal, c.d_scal, sizeof(scal), cudaMemcpyDeviceToHost, c.stream));
    BNS_CUDA_HOLD(cudaMemcpyAsync(&nonfinite, c.d_nonfinite, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
    if (host_w) {
        for (int l = 0; l < L; ++l) {
            BNS_CUDA_HOLD(cudaMemcpyAsync(W_in[l], W[l], wl[l] * sizeof(float), cudaMemcpyDeviceToHost, c.stream));
            if (G_in && G_in[l])
                BNS_CUDA_HOLD(cudaMemcpyAsync(G_in[l], G[l], wl[l] * sizeof(float), cudaMemcpyDeviceToHost, c.stream));
        }
    }
    BNS_CUDA(cudaStreamSynchronize(c.stream));
    if (nonfinite && c.optimizer == BNS_OPT_ADAM) --c.adam_t;   // no update, no step: bias corrections stay in step
    if (c.tr) c.tr->poll(c);
    collect_times(c);
    const double ntr = (double)c.n_train_global;
    if (c.multilabel) {   // R44: mean BCE over train rows x classes; F1-micro = 2TP / (2TP + FP + FN)
        if (loss) *loss = ntr > 0 ? scal[0] / (ntr * c.dims[L]) : 0.0;
        const double den = 2.0 * scal[1] + scal[2] + scal[3];
        if (acc) *acc = den > 0 ? 2.0 * scal[1] / den : 0.0;
    } else {
        if (loss) *loss = ntr > 0 ? scal[0] / ntr : 0.0;
        if (acc) *acc = ntr > 0 ? scal[1] / ntr : 0.0;
    }
    if (nonfinite) throw Error(BNS_ERR_NONFINITE, "loss is not finite; weights left unchanged");
}

// device tensor (storage type, padded ld) -> host fp32 logical
void fetch_rows(Ctx& c, const void* dptr, int64_t rows, int64_t ld, int64_t dlog, bool is_f32, float* out) {
    const size_t es = is_f32 ? 4 : tsize(c);
    std::vector<uint8_t> buf((size_t)rows * ld * es);
    if (!buf.empty()) BNS_CUDA(cudaMemcpy(buf.data(), dptr, buf.size(), cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t k = 0; k < dlog; ++k) {
            const size_t i = (size_t)(r * ld + k);
            if (es == 4) {
                std::memcpy(&out[r * dlog + k], &buf[i * 4], 4);
            } else {
                uint16_t h;
                std::memcpy(&h, &buf[i * 2], 2);
                uint32_t u = (uint32_t)h << 16;
                std::memcpy(&out[r * dlog + k], &u, 4);
            }
        }
}

}  // namespace
}  // namespace bns

using namespace bns;

extern "C" {

bns_status bns_setup(const bns_config* cfg, int64_t num_nodes, const int64_t* indptr, const int32_t* indices,
                     const int32_t* part_of, const float* features, const int32_t* labels, bns_ctx** out) {
    if (!out) return BNS_ERR_INVALID;
    *out = nullptr;
    std::unique_ptr<bns_ctx> h(new bns_ctx());
    bns_status st = guard(nullptr, [&] {
        validate(cfg, num_nodes, indptr, indices, part_of);
        Ctx& c = h->c;
        c.cfg = *cfg;
        c.cfg.dims = nullptr;
        c.L = cfg->num_layers;
        c.dims.assign(cfg->dims, cfg->dims + c.L + 1);
        c.dp.resize(c.L + 1);
        for (int l = 0; l <= c.L; ++l) c.dp[l] = (int32_t)pad8(c.dims[l]);
        c.layer = cfg->layer;
        c.prec = cfg->precision;
        c.plan_only = (cfg->flags & BNS_PLAN_ONLY) != 0;
        c.timing = (cfg->flags & BNS_TIMING) != 0;
        c.debug_idx = (cfg->flags & BNS_DEBUG_EXCHANGE_INDICES) != 0;
        c.retain = (cfg->flags & BNS_RETAIN_GRADS) != 0;
        build_plan(c.plan, cfg->rank, cfg->world, num_nodes, indptr, indices, part_of);
        c.glob_nnz = indptr[num_nodes];
        const int64_t n_in = c.plan.n_in;
        if (n_in > 0 && (!features || !labels)) throw Error(BNS_ERR_INVALID, "features/labels NULL");
        int64_t ntr = 0;
        for (int64_t r = 0; r < n_in; ++r) {
            if (labels[r] < -1 || labels[r] >= c.dims[c.L])
                throw Error(BNS_ERR_INVALID, "label out of range at inner row " + std::to_string(r));
            ntr += labels[r] >= 0;
        }
        c.n_train_local = ntr;
        if (c.plan_only) return;
        setup_device(c, features, labels);
        c.tr = make_transport(c);
        c.n_train_global = c.tr ? c.tr->allreduce_host_i64(c, ntr) : ntr;
        if ((cfg->flags & BNS_CACHE_INPUT_HALO) && c.tr && c.cfg.world > 1) fill_x0_cache(c);
    });
    if (st != BNS_OK) {
        if (h->c.tr) { delete h->c.tr; h->c.tr = nullptr; }
        for (void* p : h->c.allocs) cudaFree(p);
        h->c.allocs.clear();
        return st;
    }
    *out = h.release();
    return BNS_OK;
}

bns_status bns_sample_boundary(bns_ctx* h, double p, uint64_t seed, uint64_t epoch) {
    if (!h) return BNS_ERR_INVALID;
    Ctx& c = h->c;
    if (c.failed || c.plan_only) return BNS_ERR_STATE;
    if (!(p >= 0.0 && p <= 1.0)) { c.err = "p must be in [0, 1]"; return BNS_ERR_INVALID; }
    if (c.cfg.max_p > 0.0 && c.cfg.max_p < 1.0 && p > c.cfg.max_p) {
        c.err = "p > cfg.max_p (halo buffers are sized for max_p)";
        return BNS_ERR_OOM;
    }
    return guard(h, [&] {
        BNS_CUDA(cudaSetDevice(c.cfg.device));
        sample_boundary(c, BNS_SAMPLER_BNS, p, seed, epoch);
    });
}

bns_status bns_sample_edges(bns_ctx* h, int32_t sampler, double q, uint64_t seed, uint64_t epoch) {
    if (!h) return BNS_ERR_INVALID;
    Ctx& c = h->c;
    if (c.failed || c.plan_only) return BNS_ERR_STATE;
    if (sampler != BNS_SAMPLER_BES && sampler != BNS_SAMPLER_DROPEDGE) { c.err = "bad sampler"; return BNS_ERR_INVALID; }
    if (!(q >= 0.0 && q <= 1.0)) { c.err = "q must be in [0, 1]"; return BNS_ERR_INVALID; }
    return guard(h, [&] {
        BNS_CUDA(cudaSetDevice(c.cfg.device));
        edge_init(c);
        sample_boundary(c, sampler, q, seed, epoch);
    });
}

bns_status bns_epoch(bns_ctx* h, float* const* weights, float lr, float* const* grads, double* loss, double* acc) {
    if (!h) return BNS_ERR_INVALID;
    Ctx& c = h->c;
    if (c.failed || c.plan_only) return BNS_ERR_STATE;
    if (!c.sampled && !c.pf_pending) { c.err = "bns_epoch before bns_sample_boundary"; return BNS_ERR_STATE; }
    if (!weights) { c.err = "weights is NULL"; return BNS_ERR_INVALID; }
    for (int l = 0; l < c.L; ++l)
        if (!weights[l]) { c.err = "weights[l] is NULL"; return BNS_ERR_INVALID; }
    return guard(h, [&] {
        BNS_CUDA(cudaSetDevice(c.cfg.device));
        settle(c);
        epoch(c, weights, lr, grads, loss, acc);
    });
}

bns_status bns_step(bns_ctx* h, double p, uint64_t seed, uint64_t ep, float* const* weights, float lr,
                    float* const* grads, double* loss, double* acc) {
    if (!h) return BNS_ERR_INVALID;
    Ctx& c = h->c;
    const bool prefetch = (c.cfg.flags & BNS_PREFETCH_DRAW) != 0;
    if (prefetch && c.pf_pending && c.sampler == BNS_SAMPLER_BNS && c.p == p && c.pf_seed == seed && c.pf_ep == ep &&
        !c.failed) {
        // the draw of this step was enqueued by the previous bns_step and its counts arrived with that step's
        // closing sync: no wait, no re-draw
        const bns_status st = guard(h, [&] {
            c.pf_pending = false;
            draw_finish(c, ep, false);
        });
        if (st != BNS_OK) return st;
    } else {
        const bns_status st = bns_sample_boundary(h, p, seed, ep);
        if (st != BNS_OK) return st;
    }
    if (prefetch && ep != UINT64_MAX) {
        c.pf_want = true;
        c.pf_p = p;
        c.pf_seed = seed;
        c.pf_ep = ep + 1;
    }
    const bns_status st = bns_epoch(h, weights, lr, grads, loss, acc);
    c.pf_want = false;
    return st;
}

bns_status bns_set_training(bns_ctx* h, int32_t optimizer, double beta1, double beta2, double eps, double dropout,
                            uint64_t dropout_seed) {
    if (!h) return BNS_ERR_INVALID;
    Ctx& c = h->c;
    if (c.failed || c.plan_only) return BNS_ERR_STATE;
    if ((optimizer != BNS_OPT_SGD && optimizer != BNS_OPT_ADAM) || !(dropout >= 0.0 && dropout < 1.0) ||
        !(beta1 >= 0.0 && beta1 < 1.0) || !(beta2 >= 0.0 && beta2 < 1.0) || !(eps > 0.0)) {
        c.err = "bns_set_training: invalid optimizer / betas / eps / dropout";
        return BNS_ERR_INVALID;
    }
    return guard(h, [&] {
        BNS_CUDA(cudaSetDevice(c.cfg.device));
        BNS_CUDA(cudaStreamSynchronize(c.stream));
        c.optimizer = optimizer;
        c.beta1 = beta1;
        c.beta2 = beta2;
        c.eps = eps;
        c.adam_t = 0;
        if (optimizer == BNS_OPT_ADAM) {
            if (!c.d_adam_m) {
                c.d_adam_m = static_cast<float*>(dalloc(c, c.hostw_n * sizeof(float)));
                c.d_adam_v = static_cast<float*>(dalloc(c, c.hostw_n * sizeof(float)));
            }
            BNS_CUDA(cudaMemset(c.d_adam_m, 0, c.hostw_n * sizeof(float)));
            BNS_CUDA(cudaMemset(c.d_adam_v, 0, c.hostw_n * sizeof(float)));
        }
        c.drop = dropout;
        c.drop_seed = dropout_seed;
        if (dropout > 0.0 && c.Xd.empty()) {
            const size_t ts = tsize(c);
            c.Xd.assign(c.L, nullptr);
            for (int l = 0; l < c.L; ++l)
                c.Xd[l] = dalloc(c, (size_t)(c.plan.n_in + c.halo_cap) * c.dp[l] * ts);
            c.d_rowgid = static_cast<int32_t*>(dalloc(c, (c.plan.n_in + c.halo_cap + 1) * sizeof(int32_t)));
            BNS_CUDA(cudaMemcpy(c.d_rowgid, c.plan.V.data(), c.plan.n_in * sizeof(int32_t), cudaMemcpyHostToDevice));
        }
    });
}

bns_status bns_set_multilabel(bns_ctx* h, const uint8_t* targets) {
    if (!h) return BNS_ERR_INVALID;
    Ctx& c = h->c;
    if (c.failed || c.plan_only) return BNS_ERR_STATE;
    return guard(h, [&] {
        BNS_CUDA(cudaSetDevice(c.cfg.device));
        BNS_CUDA(cudaStreamSynchronize(c.stream));
        if (!targets) { c.multilabel = false; return; }
        const int64_t n = c.plan.n_in * (int64_t)c.dims[c.L];
        for (int64_t k = 0; k < n; ++k)
            if (targets[k] > 1) throw Error(BNS_ERR_INVALID, "targets must be 0 or 1");
        if (!c.d_targets) c.d_targets = static_cast<uint8_t*>(dalloc(c, (size_t)n + 16));
        if (n) BNS_CUDA(cudaMemcpy(c.d_targets, targets, (size_t)n, cudaMemcpyHostToDevice));
        c.multilabel = true;
    });
}

bns_status bns_query(bns_ctx* h, int32_t what, int32_t layer, void* dst, int64_t cap, int64_t* written) {
    if (!h) return BNS_ERR_INVALID;
    Ctx& c = h->c;
    return guard(h, [&] {
        if (!c.plan_only && !c.failed) settle(c);
        const Plan& P = c.plan;
        const int m = c.cfg.world, L = c.L;
        std::vector<uint8_t> out;
        auto put = [&](const void* p, size_t n) {
            size_t o = out.size();
            out.resize(o + n);
            if (n) std::memcpy(out.data() + o, p, n);
        };
        auto need_dev = [&] {
            if (c.plan_only) throw Error(BNS_ERR_STATE, "query needs device state (context is BNS_PLAN_ONLY)");
        };
        auto need_sample = [&] {
            need_dev();
            if (!c.sampled) throw Error(BNS_ERR_STATE, "query needs a bns_sample_boundary first");
        };
        auto rows_f32 = [&](const void* d, int64_t rows, int64_t ld, int64_t dl, bool f32) {
            std::vector<float> t((size_t)rows * dl);
            fetch_rows(c, d, rows, ld, dl, f32, t.data());
            put(t.data(), t.size() * 4);
        };
        auto vec32 = [&](const int32_t* d, int64_t n) {
            std::vector<int32_t> t(n);
            if (n) BNS_CUDA(cudaMemcpy(t.data(), d, n * 4, cudaMemcpyDeviceToHost));
            return t;
        };
        switch (what) {
            case BNS_Q_COUNTS: {
                std::vector<int64_t> v = {P.n_in, P.n_bd, c.n_halo, c.n_sent, (int64_t)P.col_enc.size(), c.nnz_kept};
                for (int j = 0; j < m; ++j) v.push_back(c.recv_off[j + 1] - c.recv_off[j]);
                for (int j = 0; j < m; ++j) v.push_back(c.send_off[j + 1] - c.send_off[j]);
                put(v.data(), v.size() * 8);
                break;
            }
            case BNS_Q_INNER: put(P.V.data(), P.V.size() * 4); break;
            case BNS_Q_BOUNDARY: put(P.B.data(), P.B.size() * 4); break;
            case BNS_Q_BOUNDARY_OFF: put(P.B_off.data(), P.B_off.size() * 8); break;
            case BNS_Q_BOUNDARY_ROW: put(P.B_row.data(), P.B_row.size() * 4); break;
            case BNS_Q_SENDCAND: {
                std::vector<int32_t> g(P.D_local.size());
                for (size_t k = 0; k < g.size(); ++k) g[k] = P.V[P.D_local[k]];
                put(g.data(), g.size() * 4);
                break;
            }
            case BNS_Q_SENDCAND_OFF: put(P.D_off.data(), P.D_off.size() * 8); break;
            case BNS_Q_STATIC_CSR:
                put(P.row_ptr.data(), P.row_ptr.size() * 8);
                put(P.col_enc.data(), P.col_enc.size() * 4);
                break;
            case BNS_Q_MASK: {
                need_sample();
                std::vector<uint8_t> f(P.n_bd);
                if (P.n_bd) BNS_CUDA(cudaMemcpy(f.data(), c.d_flags, P.n_bd, cudaMemcpyDeviceToHost));
                put(f.data(), f.size());
                break;
            }
            case BNS_Q_HALO: {
                need_sample();
                std::vector<int32_t> ub = vec32(c.d_cand_out, c.n_halo);
                for (auto& x : ub) x = P.B[x];
                put(ub.data(), ub.size() * 4);
                break;
            }
            case BNS_Q_HALO_OFF: need_sample(); put(c.recv_off.data(), (m + 1) * 8); break;
            case BNS_Q_SEND: {
                need_sample();
                std::vector<int32_t> s = vec32(c.d_cand_out + c.n_halo, c.n_sent);
                for (auto& x : s) x = P.V[x];
                put(s.data(), s.size() * 4);
                break;
            }
            case BNS_Q_SEND_OFF: need_sample(); put(c.send_off.data(), (m + 1) * 8); break;
            case BNS_Q_H: {
                need_sample();
                if (layer < 0 || layer > L) throw Error(BNS_ERR_INVALID, "layer out of range");
                if (layer == L) rows_f32(c.d_logits, P.n_in, c.dp[L], c.dims[L], true);
                else rows_f32(c.H[layer], P.n_in, c.dp[layer], c.dims[layer], false);
                break;
            }
            case BNS_Q_Z: {
                need_sample();
                if (layer < 1 || layer > L) throw Error(BNS_ERR_INVALID, "layer out of range");
                if (((c.tf_mask >> (layer - 1)) & 1u) || c.layer == BNS_LAYER_GAT)
                    throw Error(BNS_ERR_STATE, "layer runs transform-first (R42) or is GAT: Z is not materialised");
                rows_f32(c.Z[layer], P.n_in, c.dp[layer - 1], c.dims[layer - 1], false);
                break;
            }
            case BNS_Q_DH: {
                need_sample();
                if (layer < 1 || layer > L) throw Error(BNS_ERR_INVALID, "layer out of range");
                if (!c.retain) throw Error(BNS_ERR_STATE, "BNS_Q_DH needs BNS_RETAIN_GRADS");
                if (layer == L) rows_f32(c.d_dlogits, P.n_in, c.dp[L], c.dims[L], true);
                else rows_f32(c.dH_keep[layer], P.n_in, c.dp[layer], c.dims[layer], false);
                break;
            }
            case BNS_Q_HALO_ROWS: {
                need_sample();
                if (layer < 1 || layer > L) throw Error(BNS_ERR_INVALID, "layer out of range");
                const size_t ts = tsize(c);
                rows_f32(static_cast<const char*>(c.H[layer - 1]) + P.n_in * c.dp[layer - 1] * ts, c.n_halo,
                         c.dp[layer - 1], c.dims[layer - 1], false);
                break;
            }
            case BNS_Q_INDUCED: {
                need_sample();
                std::vector<int64_t> ptr(P.n_in + 1);
                std::vector<int32_t> col;
                if (c.fwd_mode == 2) {
                    BNS_CUDA(cudaMemcpy(ptr.data(), c.d_ind_ptr, (P.n_in + 1) * 8, cudaMemcpyDeviceToHost));
                    col = vec32(c.d_ind_col, ptr[P.n_in]);
                } else if (c.fwd_mode == 0) {
                    ptr = P.row_ptr;
                    col = vec32(c.d_static_col, (int64_t)P.col_enc.size());
                } else {
                    ptr = P.ii_ptr;
                    col = P.ii_col;
                }
                put(ptr.data(), ptr.size() * 8);
                put(col.data(), col.size() * 4);
                break;
            }
            case BNS_Q_TIMES: put(c.times.data(), c.times.size() * 8); break;
            case BNS_Q_MEMORY: {
                size_t fr = 0, tot = 0;
                if (!c.plan_only) cudaMemGetInfo(&fr, &tot);
                int64_t v[2] = {c.dev_bytes, (int64_t)(tot - fr)};
                put(v, 16);
                break;
            }
            case BNS_Q_KERNEL_COUNT: put(&c.kernels, 8); break;
            case BNS_Q_TF_LAYERS: {
                const int32_t v = (int32_t)c.tf_mask;
                put(&v, 4);
                break;
            }
            case BNS_Q_INDUCED_T: {
                need_sample();
                if (c.sampler == BNS_SAMPLER_BNS) throw Error(BNS_ERR_STATE, "BNS_Q_INDUCED_T needs bns_sample_edges");
                const int64_t n_rows = P.n_in + P.n_bd;
                std::vector<int64_t> ptr(n_rows + 1);
                BNS_CUDA(cudaMemcpy(ptr.data(), c.d_ind_tptr, (n_rows + 1) * 8, cudaMemcpyDeviceToHost));
                std::vector<int32_t> col = vec32(c.d_ind_tcol, ptr[n_rows]);
                put(ptr.data(), ptr.size() * 8);
                put(col.data(), col.size() * 4);
                break;
            }
            default: throw Error(BNS_ERR_INVALID, "unknown query");
        }
        if (written) *written = (int64_t)out.size();
        if (dst && cap > 0) std::memcpy(dst, out.data(), std::min<size_t>(out.size(), (size_t)cap));
    });
}

bns_status bns_set_timing(bns_ctx* h, int32_t on) {
    if (!h) return BNS_ERR_INVALID;
    Ctx& c = h->c;
    if (c.failed || c.plan_only || c.ev.empty()) {
        c.err = "bns_set_timing needs a context created with BNS_TIMING";
        return BNS_ERR_STATE;
    }
    return guard(h, [&] {
        BNS_CUDA(cudaStreamSynchronize(c.stream));
        collect_times(c);
        c.timing = on != 0;
    });
}

bns_status bns_gemm(int32_t precision, int32_t kind, int64_t M, int64_t N, int64_t K, const void* A0, const void* A1,
                    int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, const float* rowscale,
                    int64_t scale_cols, int32_t flags, void* stream, int32_t* splits) {
    using namespace bns;
    return guard(nullptr, [&] {
        if (precision != BNS_BF16 && precision != BNS_FP32) throw Error(BNS_ERR_INVALID, "bns_gemm: bad precision");
        if (M < 0 || N <= 0 || K <= 0 || !A0 || !B || !C || kind < 0 || kind > 3)
            throw Error(BNS_ERR_INVALID, "bns_gemm: bad kind / shape / NULL operand");
        if (kind == 2 && (K % 128 != 0 || !A1)) throw Error(BNS_ERR_INVALID, "bns_gemm: WGRAD2 needs A1 and K % 128 == 0");
        Ctx c;
        c.prec = precision;
        c.use_tc = true;
        c.stream = static_cast<cudaStream_t>(stream);
        c.splitk_cap = 0;
        std::vector<void*> mine;
        if (kind == 1 || kind == 2) {   // room for one fp32 K x N (x2) slice per split, up to 148 splits
            c.splitk_cap = 148 * (kind == 2 ? 2 * K + 128 : K) * N;
            if (precision == BNS_FP32) {
                c.tr_cap = ((kind == 2 ? 2 : 1) * K + N) * ((M + 3) / 4 * 4);
                c.d_tr = static_cast<float*>(dalloc(c, c.tr_cap * sizeof(float)));
                c.splitk_cap = std::max<int64_t>(c.splitk_cap, ((M + 511) / 512 + 1) * (kind == 2 ? 2 * K + 128 : K) * N);
            }
            c.d_splitk = static_cast<float*>(dalloc(c, c.splitk_cap * sizeof(float)));
        }
        const int64_t Kw = (K + 63) / 64 * 64;   // W^T concat halves are padded to 64 in both precisions
        try {
            switch (kind) {
                case 0: gemm_fwd_tc(c, M, N, A0, K, lda, A1, A1 ? K : 0, lda, B, ldb ? ldb : (A1 ? 2 * Kw : Kw), C,
                                    ldc, flags & 1, (flags >> 1) & 1); break;
                case 1: gemm_wgrad_tc(c, M, K, N, A0, lda, B, ldb, static_cast<float*>(C), ldc); break;
                case 2: gemm_wgrad2_tc(c, M, M, K, N, A0, A1, lda, B, ldb, B, ldb, static_cast<float*>(C), ldc); break;
                default: gemm_dx_tc(c, M, N, K, A0, lda, B, ldb, C, ldc, rowscale, scale_cols); break;
            }
            BNS_CUDA(cudaStreamSynchronize(c.stream));
        } catch (...) {
            for (void* p : c.allocs) cudaFree(p);
            throw;
        }
        for (void* p : c.allocs) cudaFree(p);
        if (splits) *splits = (kind == 1 || kind == 2) ? c.last_splitk : 1;
    });
}

void* bns_stream(const bns_ctx* h) { return h ? (void*)h->c.stream : nullptr; }

const char* bns_last_error(const bns_ctx* h) { return h ? h->c.err.c_str() : g_err.c_str(); }

void bns_destroy(bns_ctx* h) {
    if (!h) return;
    Ctx& c = h->c;
    if (!c.plan_only) {
        cudaSetDevice(c.cfg.device);
        if (c.stream) cudaStreamSynchronize(c.stream);
        if (c.tr && c.stream) {
            try {
                c.tr->shutdown(c);
            } catch (...) {   // no exception crosses the ABI; teardown goes on
            }
        }
    }
    delete c.tr;
    for (void* p : c.allocs) cudaFree(p);
    if (c.h_seg_pos) cudaFreeHost(c.h_seg_pos);
    for (auto& e : c.ev) cudaEventDestroy(e);
    if (c.own_stream && c.stream) cudaStreamDestroy(c.stream);
    delete h;
}

}  // extern "C"
