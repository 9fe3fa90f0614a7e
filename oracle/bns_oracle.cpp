// bns_oracle.cpp -- the CPU ORACLE for BNS-GCN (arXiv 2203.10983).
//
// TEST INFRASTRUCTURE ONLY.  Nothing on the product path may include, link, load or call this file:
// only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs use it.
// It shares no code with paper_2203_10983_b200/csrc (own Philox, own plan, own CSR handling).
//
// What it is: a plain, slow, single-threaded, double-precision implementation of Algorithm 1
// ("Boundary node sampling for partition-parallel training (per-partition view)")
// that simulates all m partitions in one process, visiting ranks in order 0..m-1.
// Every step follows the cited passage in the paper's order and notation; where the paper is silent the
// reading used is the numbered item of SURVEY.md §8(c) ("R<n>" below), listed again in DESIGN.md §3.
//
//   plan     V_i, B_i, D_{i->j}           PAPER.md:173-176 (§3.1, Fig. fig:framework), :273 (Alg.1 l.1)
//   sample   U_i <- Bernoulli_p(B_i)        PAPER.md:276 (Alg.1 l.4), :332; R5, R6, R7, R23
//   record   S_{i,j} = U_j ∩ V_i            PAPER.md:280-282 (Alg.1 l.6-7); R24, R27
//   layer    exchange + GCN^(l)             PAPER.md:285-287 (Alg.1 l.9-10), :100 (GraphSAGE-mean),
//                                           :335 (H -> H/p), :736-778 (App.A, P and S); R1-R3, R11-R16
//   loss     f_i = sum_{v in V_i} loss      PAPER.md:289 (Alg.1 l.11); R8, R22
//   backward g_i = df_i/dw                  PAPER.md:290 (Alg.1 l.12), :179, :336; R12, R25, R29
//   reduce   g = AllReduce(g_i)             PAPER.md:291 (Alg.1 l.13); R21
//   update   w <- w - eta g                 PAPER.md:292 (Alg.1 l.14); R9
//
// Arithmetic: double throughout, in the definition's order (aggregate first, then the update).  The
// oracle has no bf16 mode and no knowledge of the kernel's evaluation order: the GPU's bf16-storage mode (R19) and
// its transform-first order (R42) are compared against this float64 definition directly (tests/gpu_harness.py).
//
// Pins (tests/test_oracle_*.py, all `-m "not gpu"`): Random123 Philox KATs; dense-adjacency float64
// brute force with torch autograd (independent backward); central finite differences of the oracle's own
// loss; SPEC hand examples (P4, K1,5); the survey's tiny goldens E1-E6 (tests/golden/); p=1 == unpartitioned;
// p=0 == dense on A∘[same part]; Binomial(|B_i|, p) counts; Eq. 3 identity.
// Every function here is pinned; none is "parity unpinned".
#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <vector>

namespace {

// ---------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11).  R7: the paper names no RNG; this is the counter-based
// generator SURVEY.md §8(c) item 7 fixes, written out from its definition.
// ---------------------------------------------------------------------------------------------
const uint32_t PHILOX_M0 = 0xD2511F53u, PHILOX_M1 = 0xCD9E8D57u;
const uint32_t PHILOX_W0 = 0x9E3779B9u, PHILOX_W1 = 0xBB67AE85u;

void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
        uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// keep(u, i): Alg.1 l.4 "randomly pick elements in B_i with probability p", one
// independent Bernoulli per (receiving partition i, node u) (R5, R23), threshold T(p) = floor(p*2^32) (R7).
uint64_t threshold_of(double p) { return (uint64_t)std::floor(p * 4294967296.0); }

uint32_t draw(uint32_t u, uint32_t i, uint64_t epoch, uint64_t seed) {
    uint32_t ctr[4] = {u, i, (uint32_t)(epoch & 0xffffffffu), (uint32_t)(epoch >> 32)};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t out[4];
    philox4x32_10(ctr, key, out);
    return out[0];
}

bool keep(uint32_t u, uint32_t i, uint64_t epoch, uint64_t seed, uint64_t T) {
    return (uint64_t)draw(u, i, epoch, seed) < T;
}

enum { KIND_SAGE = 0, KIND_GCN = 1, KIND_GAT = 2 };

struct Partition {
    // plan (static)
    std::vector<int32_t> V;                 // inner nodes, ascending gid (Alg.1 l.1)
    std::vector<int32_t> B;                 // boundary nodes, ordered by (owner, gid) (R24)
    std::vector<int64_t> B_off;             // [m+1] owner offsets into B
    std::vector<std::vector<int32_t>> D;    // D[j] = B_j ∩ V_i, ascending gid
    // per epoch
    std::vector<uint8_t> keep_B;            // keep flag for each B entry
    std::vector<int32_t> U;                 // sampled boundary nodes, B order (Alg.1 l.4)
    std::vector<int64_t> U_off;             // [m+1]
    std::vector<std::vector<int32_t>> S;    // S[j] = U_j ∩ V_i, ascending gid (Alg.1 l.7)
};

struct Oracle {
    int64_t N = 0;
    std::vector<int64_t> indptr;
    std::vector<int32_t> indices;
    std::vector<int32_t> part_of;
    int m = 1;
    int L = 1;
    std::vector<int32_t> dims;              // L+1
    int kind = KIND_SAGE;
    std::vector<double> X;                  // N x dims[0]
    std::vector<int32_t> labels;            // N, -1 = not a training node
    std::vector<Partition> parts;
    double p = 1.0;
    bool sampled = false;
    // recorded tensors, indexed by global id (each node is inner to exactly one partition)
    std::vector<std::vector<double>> H;     // H[l], l=0..L : N x dims[l]  (H[L] = logits)
    std::vector<std::vector<double>> Z;     // Z[l], l=1..L : N x dims[l-1] (aggregation output)
    std::vector<std::vector<double>> dH;    // dH[l], l=0..L : N x dims[l]  (dH[0] is not computed)
    std::vector<std::vector<double>> G;     // all-reduced weight gradients, per layer
    std::vector<int64_t> rows_sent_fwd;     // per layer, total rows exchanged (Eq. 3 accounting)
    // f2: the paper's training recipe, Adam + dropout
    int optimizer = 0;                      // 0 SGD (Alg.1 l.14), 1 Adam
    double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
    int64_t adam_t = 0;
    std::vector<std::vector<double>> adam_m, adam_v;
    double drop = 0.0;                      // dropout rate r on every layer's input (R38)
    uint64_t drop_seed = 0;
    uint64_t epoch_id = 0;                  // epoch of the last draw (keys the dropout masks)
    // f3: edge samplers BES / DropEdge (Table tab:bes)
    int sampler = 0;                        // 0 BNS (node), 1 BES, 2 DropEdge
    // f4: multi-label targets (Yelp): sigmoid BCE over the train rows' C logits, F1-micro (R44)
    bool multilabel = false;
    std::vector<uint8_t> targets;           // N x C in {0, 1}
    double q = 1.0;                         // arc keep probability of the edge samplers
    uint64_t sample_seed = 0;
};

enum { SAMPLER_BNS = 0, SAMPLER_BES = 1, SAMPLER_DROPEDGE = 2 };

// R40 arc draw of the edge samplers: the arc (v <- u) -- target v aggregates source u -- is kept iff
// Philox4x32-10(ctr = {v, u, e_lo, e_hi}, key = {s_lo ^ 0xED6E, s_hi}).x < floor(q 2^32).  Each direction of an
// undirected edge is its own arc (it feeds a different node's aggregation); keyed by global ids only, so the
// draw does not depend on the partitioning.
bool arc_keep(const Oracle& o, int32_t v, int32_t u) {
    uint32_t ctr[4] = {(uint32_t)v, (uint32_t)u, (uint32_t)(o.epoch_id & 0xffffffffu), (uint32_t)(o.epoch_id >> 32)};
    uint32_t key[2] = {(uint32_t)(o.sample_seed & 0xffffffffu) ^ 0xED6Eu, (uint32_t)(o.sample_seed >> 32)};
    uint32_t out[4];
    philox4x32_10(ctr, key, out);
    return (uint64_t)out[0] < threshold_of(o.q);
}

// Arc (v <- u) of partition i's sampled aggregation, v in V_i: is it in the sampled graph, and with which
// column scale c (R3, R41)?
//   BNS      (Alg.1 l.4-5):      u inner -> 1;  u in U_i -> 1/p;  other boundary u -> dropped
//   BES:     u inner -> 1;  u boundary -> own Bernoulli(q) arc draw, kept -> 1/q
//   DropEdge:     every arc -> own Bernoulli(q) draw, kept -> 1/q
// u_row = stacked row of u in partition i (-1 if absent), n_in = |V_i|.
bool arc_in(const Oracle& o, int32_t v, int32_t u, int64_t u_row, int64_t n_in, double* c) {
    const bool inner = u_row >= 0 && u_row < n_in;
    if (o.sampler == SAMPLER_BNS) {
        if (u_row < 0) return false;
        *c = inner ? 1.0 : (o.p > 0.0 ? 1.0 / o.p : 0.0);
        return true;
    }
    const double inv_q = o.q > 0.0 ? 1.0 / o.q : 0.0;
    if (o.sampler == SAMPLER_BES && inner) { *c = 1.0; return true; }
    if (!arc_keep(o, v, u)) return false;
    *c = inv_q;
    return true;
}

// R38 dropout mask: keep(u, c, l, e) = Philox4x32-10(ctr = {u, c >> 2, l, e_lo}, key = {s_lo ^ 0xD809, s_hi})
// .word[c & 3] >= floor(r 2^32); a kept value is scaled by 1/(1-r).  Keyed by the global node id, so every copy
// of a row (owner and halo) gets the same mask.
double drop_factor(const Oracle& o, int32_t u, int c, int l) {
    if (o.drop <= 0.0) return 1.0;
    uint32_t ctr[4] = {(uint32_t)u, (uint32_t)(c >> 2), (uint32_t)l, (uint32_t)(o.epoch_id & 0xffffffffu)};
    uint32_t key[2] = {(uint32_t)(o.drop_seed & 0xffffffffu) ^ 0xD809u, (uint32_t)(o.drop_seed >> 32)};
    uint32_t out[4];
    philox4x32_10(ctr, key, out);
    return ((uint64_t)out[c & 3] >= threshold_of(o.drop)) ? 1.0 / (1.0 - o.drop) : 0.0;
}

int64_t deg(const Oracle& o, int32_t v) { return o.indptr[v + 1] - o.indptr[v]; }

// ---------------------------------------------------------------------------------------------
// Plan: PAPER.md:173-176 -- inner set V_i = nodes assigned to i; boundary set B_i = nodes of other
// partitions with at least one neighbour in V_i; D_{i->j} = B_j ∩ V_i (what i must send to j).
// ---------------------------------------------------------------------------------------------
void build_plan(Oracle& o) {
    o.parts.assign(o.m, Partition());
    for (int32_t v = 0; v < o.N; ++v) o.parts[o.part_of[v]].V.push_back(v);
    for (int i = 0; i < o.m; ++i) {
        Partition& P = o.parts[i];
        std::vector<uint8_t> is_bd(o.N, 0);
        for (int32_t v : P.V)
            for (int64_t e = o.indptr[v]; e < o.indptr[v + 1]; ++e) {
                int32_t u = o.indices[e];
                if (o.part_of[u] != i) is_bd[u] = 1;
            }
        // order by (owner, gid): iterate owners, then ascending gid
        P.B_off.assign(o.m + 1, 0);
        for (int j = 0; j < o.m; ++j) {
            P.B_off[j] = (int64_t)P.B.size();
            for (int32_t u = 0; u < o.N; ++u)
                if (is_bd[u] && o.part_of[u] == j) P.B.push_back(u);
        }
        P.B_off[o.m] = (int64_t)P.B.size();
    }
    for (int i = 0; i < o.m; ++i) {
        Partition& P = o.parts[i];
        P.D.assign(o.m, std::vector<int32_t>());
        for (int j = 0; j < o.m; ++j) {
            if (j == i) continue;
            const Partition& Q = o.parts[j];
            for (int64_t k = Q.B_off[i]; k < Q.B_off[i + 1]; ++k) P.D[j].push_back(Q.B[k]);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Sample + record: Alg.1 l.4-7.  U_i keeps B order (owner-major, gid ascending, R24).
// "Broadcast U_i" is realised literally here: S_{i,j} is computed as U_j ∩ V_i from partition j's U_j.
// ---------------------------------------------------------------------------------------------
void sample(Oracle& o, double p, uint64_t seed, uint64_t epoch) {
    uint64_t T = threshold_of(p);
    o.p = p;
    o.sampler = SAMPLER_BNS;
    for (int i = 0; i < o.m; ++i) {
        Partition& P = o.parts[i];
        P.keep_B.assign(P.B.size(), 0);
        for (size_t k = 0; k < P.B.size(); ++k)
            P.keep_B[k] = keep((uint32_t)P.B[k], (uint32_t)i, epoch, seed, T) ? 1 : 0;
    }
}

// f3 edge samplers: a boundary node u in B_i is communicated to i iff at least
// one of its arcs into V_i survives (u's owner recomputes the same arc draws, R27) -- so U_i is B_i filtered by
// "some kept arc", in B order, and S_{i,j} = U_j ∩ V_i exactly as for BNS.
void sample_edges(Oracle& o, int sampler, double q, uint64_t seed, uint64_t epoch) {
    o.sampler = sampler;
    o.q = q;
    o.p = q;
    o.sample_seed = seed;
    o.epoch_id = epoch;
    for (int i = 0; i < o.m; ++i) {
        Partition& P = o.parts[i];
        std::vector<uint8_t> hit(o.N, 0);
        for (int32_t v : P.V)
            for (int64_t e = o.indptr[v]; e < o.indptr[v + 1]; ++e) {
                const int32_t u = o.indices[e];
                if (o.part_of[u] != i && arc_keep(o, v, u)) hit[u] = 1;
            }
        P.keep_B.assign(P.B.size(), 0);
        for (size_t k = 0; k < P.B.size(); ++k) P.keep_B[k] = hit[P.B[k]];
    }
}

void finish_sample(Oracle& o) {
    for (int i = 0; i < o.m; ++i) {
        Partition& P = o.parts[i];
        P.U.clear();
        P.U_off.assign(o.m + 1, 0);
        for (int j = 0; j < o.m; ++j) {
            P.U_off[j] = (int64_t)P.U.size();
            for (int64_t k = P.B_off[j]; k < P.B_off[j + 1]; ++k)
                if (P.keep_B[k]) P.U.push_back(P.B[k]);
        }
        P.U_off[o.m] = (int64_t)P.U.size();
    }
    for (int i = 0; i < o.m; ++i) {             // Alg.1 l.7: S_{i,j} <- U_j ∩ V_i
        Partition& P = o.parts[i];
        P.S.assign(o.m, std::vector<int32_t>());
        for (int j = 0; j < o.m; ++j) {
            if (j == i) continue;
            for (int32_t u : o.parts[j].U)
                if (o.part_of[u] == i) P.S[j].push_back(u);
            std::sort(P.S[j].begin(), P.S[j].end());
        }
    }
    o.sampled = true;
}

// Column scale c_u of the sampled aggregation: 1 for inner u, 1/p for sampled boundary u
// ("replace ... H with H/p"; App. A diagonal S; R3).
struct LocalIndex {
    std::vector<int64_t> row;   // gid -> stacked row (inner 0..n_in-1, halo n_in..), -1 if absent
};

// ---------------------------------------------------------------------------------------------
// f4 / R45: GAT layer (Velickovic et al.; the paper's Table tab:gat ablation), one head, on the
// sampled graph of partition i: Y = X W on every stacked row, el = Y a_l, er = Y a_r,
//   e_vu = LeakyReLU_0.2(el_v + er_u) over u in N'(v) = {kept neighbours} ∪ {v},
//   alpha_vu = softmax_u(e_vu),  pre_v = Σ_u alpha_vu Y_u.
// Dropped boundary neighbours simply leave N'(v) (the softmax renormalises; no 1/p).  Weights: (din + 2) x dout
// rows [W ; a_l ; a_r].
// ---------------------------------------------------------------------------------------------
struct GatEdges {
    std::vector<int64_t> ptr;   // per inner row r: [ptr[r], ptr[r+1]) into col / s
    std::vector<int64_t> col;   // stacked row of u (self last)
    std::vector<double> s;      // el_v + er_u
};

void gat_setup(const Oracle& o, int i, const std::vector<int64_t>& row, const std::vector<double>& X, int din,
               int dout, const std::vector<double>& W, std::vector<double>& Y, std::vector<double>& el,
               std::vector<double>& er, GatEdges& E) {
    const Partition& P = o.parts[i];
    const size_t n_in = P.V.size(), n_h = P.U.size(), n = n_in + n_h;
    Y.assign(n * dout, 0.0);
    el.assign(n, 0.0);
    er.assign(n, 0.0);
    for (size_t r = 0; r < n; ++r) {
        for (int c = 0; c < dout; ++c) {
            double y = 0.0;
            for (int k = 0; k < din; ++k) y += X[r * din + k] * W[(size_t)k * dout + c];
            Y[r * dout + c] = y;
        }
        for (int c = 0; c < dout; ++c) {
            el[r] += Y[r * dout + c] * W[(size_t)din * dout + c];
            er[r] += Y[r * dout + c] * W[(size_t)(din + 1) * dout + c];
        }
    }
    E.ptr.assign(1, 0);
    E.col.clear();
    E.s.clear();
    for (size_t r = 0; r < n_in; ++r) {
        const int32_t v = P.V[r];
        for (int64_t e = o.indptr[v]; e < o.indptr[v + 1]; ++e) {
            const int32_t u = o.indices[e];
            double c;
            if (!arc_in(o, v, u, row[u], (int64_t)n_in, &c)) continue;
            E.col.push_back(row[u]);
            E.s.push_back(el[r] + er[row[u]]);
        }
        E.col.push_back((int64_t)r);   // self loop
        E.s.push_back(el[r] + er[r]);
        E.ptr.push_back((int64_t)E.col.size());
    }
}

double leaky(double x) { return x > 0.0 ? x : 0.2 * x; }

void gat_alpha(const GatEdges& E, size_t r, std::vector<double>& a) {
    double mx = -INFINITY;
    for (int64_t e = E.ptr[r]; e < E.ptr[r + 1]; ++e) mx = std::max(mx, leaky(E.s[e]));
    double den = 0.0;
    for (int64_t e = E.ptr[r]; e < E.ptr[r + 1]; ++e) den += std::exp(leaky(E.s[e]) - mx);
    a.clear();
    for (int64_t e = E.ptr[r]; e < E.ptr[r + 1]; ++e) a.push_back(std::exp(leaky(E.s[e]) - mx) / den);
}

void gat_forward(const Oracle& o, int i, const std::vector<int64_t>& row, const std::vector<double>& X, int din,
                 int dout, const std::vector<double>& W, std::vector<double>& pre) {
    std::vector<double> Y, el, er, a;
    GatEdges E;
    gat_setup(o, i, row, X, din, dout, W, Y, el, er, E);
    const size_t n_in = o.parts[i].V.size();
    pre.assign(n_in * dout, 0.0);
    for (size_t r = 0; r < n_in; ++r) {
        gat_alpha(E, r, a);
        for (int64_t e = E.ptr[r]; e < E.ptr[r + 1]; ++e)
            for (int c = 0; c < dout; ++c) pre[r * dout + c] += a[e - E.ptr[r]] * Y[(size_t)E.col[e] * dout + c];
    }
}

// backward: c_v = g_v . pre_v; per edge dalpha = g_v . Y_u, ds = alpha (dalpha - c_v) LeakyReLU'(s);
// dY_u += alpha g_v; del_v += ds; der_u += ds; then dY_v += del_v a_l, dY_u += der_u a_r;
// dW = X^T dY, da_l = Σ_v del_v Y_v, da_r = Σ_u der_u Y_u; dX = dY W^T (then the layer's dropout)
void gat_backward(const Oracle& o, int i, const std::vector<int64_t>& row, const std::vector<double>& X, int din,
                  int dout, const std::vector<double>& W, const std::vector<double>& dpre, std::vector<double>& g,
                  std::vector<double>* dX, int l) {
    std::vector<double> Y, el, er, a;
    GatEdges E;
    gat_setup(o, i, row, X, din, dout, W, Y, el, er, E);
    const Partition& P = o.parts[i];
    const size_t n_in = P.V.size(), n = n_in + P.U.size();
    std::vector<double> dY(n * dout, 0.0), del(n, 0.0), der(n, 0.0);
    for (size_t r = 0; r < n_in; ++r) {
        gat_alpha(E, r, a);
        const double* gv = &dpre[r * dout];
        std::vector<double> outv(dout, 0.0);
        for (int64_t e = E.ptr[r]; e < E.ptr[r + 1]; ++e)
            for (int c = 0; c < dout; ++c) outv[c] += a[e - E.ptr[r]] * Y[(size_t)E.col[e] * dout + c];
        double cv = 0.0;
        for (int c = 0; c < dout; ++c) cv += gv[c] * outv[c];
        for (int64_t e = E.ptr[r]; e < E.ptr[r + 1]; ++e) {
            const size_t u = (size_t)E.col[e];
            const double al = a[e - E.ptr[r]];
            double da = 0.0;
            for (int c = 0; c < dout; ++c) da += gv[c] * Y[u * dout + c];
            const double ds = al * (da - cv) * (E.s[e] > 0.0 ? 1.0 : 0.2);
            del[r] += ds;
            der[u] += ds;
            for (int c = 0; c < dout; ++c) dY[u * dout + c] += al * gv[c];
        }
    }
    for (size_t r = 0; r < n; ++r)
        for (int c = 0; c < dout; ++c) {
            double x = dY[r * dout + c] + der[r] * W[(size_t)(din + 1) * dout + c];
            if (r < n_in) x += del[r] * W[(size_t)din * dout + c];
            dY[r * dout + c] = x;
        }
    // g[k][c] accumulates over r in ascending order (loop order k-inner or c-inner gives the same sums)
    for (size_t r = 0; r < n; ++r) {
        for (int k = 0; k < din; ++k) {
            const double xk = X[r * din + k];
            for (int c = 0; c < dout; ++c) g[(size_t)k * dout + c] += xk * dY[r * dout + c];
        }
        for (int c = 0; c < dout; ++c) {
            if (r < n_in) g[(size_t)din * dout + c] += del[r] * Y[r * dout + c];
            g[(size_t)(din + 1) * dout + c] += der[r] * Y[r * dout + c];
        }
    }
    if (!dX) return;
    dX->assign(n * din, 0.0);
    for (size_t r = 0; r < n; ++r)
        for (int k = 0; k < din; ++k) {
            double x = 0.0;
            for (int c = 0; c < dout; ++c) x += dY[r * dout + c] * W[(size_t)k * dout + c];
            if (o.drop > 0.0) {
                const int32_t u = (r < n_in) ? P.V[r] : P.U[r - n_in];
                x = x * drop_factor(o, u, k, l);
            }
            (*dX)[r * din + k] = x;
        }
}

// ---------------------------------------------------------------------------------------------
// One epoch of Algorithm 1 for all partitions (l.8-14).
// W[l] (l=0..L-1) is row-major: SAGE (2*d_in) x d_out with rows [0,d_in) multiplying z (R14);
// GCN d_in x d_out.
// ---------------------------------------------------------------------------------------------
int epoch(Oracle& o, std::vector<std::vector<double>>& W, double lr, double* loss_out, double* acc_out) {
    if (!o.sampled) return 3;
    const int m = o.m, L = o.L;

    o.H.assign(L + 1, std::vector<double>());
    o.Z.assign(L + 1, std::vector<double>());
    o.dH.assign(L + 1, std::vector<double>());
    o.H[0] = o.X;
    o.rows_sent_fwd.assign(L + 1, 0);

    // stacked-row index per partition: inner rows then halo rows in U_i order
    std::vector<LocalIndex> idx(m);
    for (int i = 0; i < m; ++i) {
        const Partition& P = o.parts[i];
        idx[i].row.assign(o.N, -1);
        for (size_t r = 0; r < P.V.size(); ++r) idx[i].row[P.V[r]] = (int64_t)r;
        for (size_t s = 0; s < P.U.size(); ++s) idx[i].row[P.U[s]] = (int64_t)(P.V.size() + s);
    }

    // saved per partition per layer: stacked input X (inner + halo rows), aggregation Z, pre-activation
    std::vector<std::vector<std::vector<double>>> Xs(L + 1, std::vector<std::vector<double>>(m));
    std::vector<std::vector<std::vector<double>>> Zs(L + 1, std::vector<std::vector<double>>(m));
    std::vector<std::vector<std::vector<double>>> PREs(L + 1, std::vector<std::vector<double>>(m));

    // ---------------- forward (Alg.1 l.8-10) ----------------
    for (int l = 1; l <= L; ++l) {
        const int din = o.dims[l - 1], dout = o.dims[l];
        const std::vector<double>& Hprev = o.H[l - 1];
        // l.9: partition i sends H_{S_{i,j}} to j; j receives H_{U_j}, owner-major (R24).
        std::vector<std::vector<std::vector<double>>> sendbuf(m, std::vector<std::vector<double>>(m));
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
                if (j == i) continue;
                for (int32_t u : o.parts[i].S[j])
                    for (int k = 0; k < din; ++k) sendbuf[i][j].push_back(Hprev[(size_t)u * din + k]);
            }
        for (int i = 0; i < m; ++i) {
            const Partition& P = o.parts[i];
            const size_t n_in = P.V.size(), n_h = P.U.size();
            std::vector<double>& X = Xs[l][i];
            X.assign((n_in + n_h) * din, 0.0);
            for (size_t r = 0; r < n_in; ++r)
                for (int k = 0; k < din; ++k) X[r * din + k] = Hprev[(size_t)P.V[r] * din + k];
            for (int j = 0; j < m; ++j) {           // receive: halo segment of owner j
                if (j == i) continue;
                const std::vector<double>& buf = sendbuf[j][i];
                size_t rows = buf.size() / (din ? din : 1);
                if (din && rows != (size_t)(P.U_off[j + 1] - P.U_off[j])) return 2;  // R27 invariant
                for (size_t k = 0; k < buf.size(); ++k) X[(size_t)(n_in + P.U_off[j]) * din + k] = buf[k];
                o.rows_sent_fwd[l] += (int64_t)rows;
            }
            // R38 dropout on the layer input (inner and halo rows alike, mask keyed by global id)
            if (o.drop > 0.0)
                for (size_t r = 0; r < n_in + n_h; ++r) {
                    const int32_t u = (r < n_in) ? P.V[r] : P.U[r - n_in];
                    for (int k = 0; k < din; ++k) X[r * din + k] = X[r * din + k] * drop_factor(o, u, k, l);
                }
            if (o.kind == KIND_GAT) {   // f4 / R45: the attention layer on the same sampled graph
                gat_forward(o, i, idx[i].row, X, din, dout, W[l - 1], PREs[l][i]);
                Zs[l][i].assign(n_in * din, 0.0);   // GAT has no separate aggregation tensor Z
                continue;
            }
            // l.10: GCN^(l)(H_i, [H; H_U], w)
            std::vector<double>& Zl = Zs[l][i];
            Zl.assign(n_in * din, 0.0);
            for (size_t r = 0; r < n_in; ++r) {
                int32_t v = P.V[r];
                int64_t dv = deg(o, v);
                double* z = &Zl[r * din];
                if (o.kind == KIND_SAGE) {
                    // z_v = (1/deg_G(v)) sum_{u in N(v) ∩ (V_i ∪ U_i)} c_u x_u   (R1, R2, R15)
                    if (dv == 0) continue;
                    for (int64_t e = o.indptr[v]; e < o.indptr[v + 1]; ++e) {
                        int32_t u = o.indices[e];
                        int64_t ru = idx[i].row[u];
                        double c;
                        if (!arc_in(o, v, u, ru, (int64_t)n_in, &c)) continue;   // dropped: contributes 0
                        for (int k = 0; k < din; ++k) z[k] += c * X[(size_t)ru * din + k];
                    }
                    for (int k = 0; k < din; ++k) z[k] = z[k] / (double)dv;
                } else {
                    // z_v = x_v / d~_v + sum_u c_u x_u / sqrt(d~_v d~_u)   (App.A P = D~^-1/2 (A+I) D~^-1/2,
                    // PAPER.md:736; S diagonal PAPER.md:771-778; R2, R16)
                    double dtv = (double)(dv + 1);
                    for (int k = 0; k < din; ++k) z[k] = X[r * din + k] / dtv;
                    for (int64_t e = o.indptr[v]; e < o.indptr[v + 1]; ++e) {
                        int32_t u = o.indices[e];
                        int64_t ru = idx[i].row[u];
                        double c;
                        if (!arc_in(o, v, u, ru, (int64_t)n_in, &c)) continue;
                        double dtu = (double)(deg(o, u) + 1);
                        double a = c / std::sqrt(dtv * dtu);
                        for (int k = 0; k < din; ++k) z[k] += a * X[(size_t)ru * din + k];
                    }
                }
            }
            // update phi: SAGE pre = W^T [z ; x]  (CONCAT(z_v, h_v); R13 no bias, R14 layout)
            //             GCN  pre = W^T z          (App.A Z = P H W)
            std::vector<double>& pre = PREs[l][i];
            pre.assign(n_in * dout, 0.0);
            const std::vector<double>& Wl = W[l - 1];
            for (size_t r = 0; r < n_in; ++r) {
                double* out = &pre[r * dout];
                for (int k = 0; k < din; ++k) {
                    double zk = Zl[r * din + k];
                    for (int c = 0; c < dout; ++c) out[c] += zk * Wl[(size_t)k * dout + c];
                }
                if (o.kind == KIND_SAGE)
                    for (int k = 0; k < din; ++k) {
                        double xk = X[r * din + k];
                        for (int c = 0; c < dout; ++c) out[c] += xk * Wl[(size_t)(din + k) * dout + c];
                    }
            }
        }
        // record H^l (ReLU on hidden layers, identity on the last: R11) and Z^l by gid
        o.H[l].assign((size_t)o.N * dout, 0.0);
        o.Z[l].assign((size_t)o.N * din, 0.0);
        for (int i = 0; i < m; ++i) {
            const Partition& P = o.parts[i];
            for (size_t r = 0; r < P.V.size(); ++r) {
                size_t g = (size_t)P.V[r];
                for (int c = 0; c < dout; ++c) {
                    double x = PREs[l][i][r * dout + c];
                    o.H[l][g * dout + c] = (l < L) ? (x > 0.0 ? x : 0.0) : x;
                }
                for (int k = 0; k < din; ++k) o.Z[l][g * din + k] = Zs[l][i][r * din + k];
            }
        }
    }

    // ---------------- loss (Alg.1 l.11; R8 global-train-count normalisation; R22 ties) ----------------
    const int C = o.dims[L];
    int64_t n_train = 0;
    for (int64_t v = 0; v < o.N; ++v) if (o.labels[v] >= 0) ++n_train;
    double loss = 0.0, correct = 0.0;
    o.dH[L].assign((size_t)o.N * C, 0.0);
    if (o.multilabel) {
        // R44: loss = (1/(N_train C)) Σ_{v train} Σ_c [softplus(x_vc) - y_vc x_vc] (= BCE(σ(x), y), mean over the
        // train rows x classes); dLogits = (σ(x) - y)/(N_train C); "accuracy" = F1-micro of x > 0 over the train rows
        double tp = 0.0, fp = 0.0, fn = 0.0;
        const double inv = n_train > 0 ? 1.0 / ((double)n_train * C) : 0.0;
        for (int i = 0; i < m; ++i) {
            double f_i = 0.0;
            for (int32_t v : o.parts[i].V) {
                if (o.labels[v] < 0) continue;
                const double* x = &o.H[L][(size_t)v * C];
                double* g = &o.dH[L][(size_t)v * C];
                for (int c = 0; c < C; ++c) {
                    const double y = o.targets[(size_t)v * C + c] ? 1.0 : 0.0;
                    f_i += std::max(x[c], 0.0) - x[c] * y + std::log1p(std::exp(-std::fabs(x[c])));
                    g[c] = (1.0 / (1.0 + std::exp(-x[c])) - y) * inv;
                    const bool pred = x[c] > 0.0;
                    if (pred && y > 0.0) tp += 1.0;
                    if (pred && y == 0.0) fp += 1.0;
                    if (!pred && y > 0.0) fn += 1.0;
                }
            }
            loss += f_i;
        }
        *loss_out = loss * inv;
        *acc_out = (2.0 * tp + fp + fn) > 0.0 ? 2.0 * tp / (2.0 * tp + fp + fn) : 0.0;
    }
    for (int i = 0; i < m && !o.multilabel; ++i) {   // f_i summed per partition, then across (rank order)
        double f_i = 0.0, c_i = 0.0;
        for (int32_t v : o.parts[i].V) {
            int32_t y = o.labels[v];
            if (y < 0) continue;
            const double* x = &o.H[L][(size_t)v * C];
            double mx = x[0];
            int arg = 0;
            for (int c = 1; c < C; ++c) if (x[c] > mx) { mx = x[c]; arg = c; }
            double se = 0.0;
            for (int c = 0; c < C; ++c) se += std::exp(x[c] - mx);
            double lse = mx + std::log(se);
            f_i += lse - x[y];
            if (arg == y) c_i += 1.0;
            double* g = &o.dH[L][(size_t)v * C];
            for (int c = 0; c < C; ++c) g[c] = std::exp(x[c] - lse) / (double)n_train;
            g[y] -= 1.0 / (double)n_train;
        }
        loss += f_i;
        correct += c_i;
    }
    if (!o.multilabel) {
        if (n_train > 0) { loss /= (double)n_train; correct /= (double)n_train; }
        *loss_out = loss;
        *acc_out = correct;
    }

    // ---------------- backward (Alg.1 l.12) ----------------
    std::vector<std::vector<std::vector<double>>> gW(m, std::vector<std::vector<double>>(L));
    for (int l = L; l >= 1; --l) {
        const int din = o.dims[l - 1], dout = o.dims[l];
        const std::vector<double>& Wl = W[l - 1];
        std::vector<std::vector<double>> dXs(m);     // gradient w.r.t. stacked input rows (inner + halo)
        for (int i = 0; i < m; ++i) {
            const Partition& P = o.parts[i];
            const size_t n_in = P.V.size(), n_h = P.U.size();
            // dPre = dH^l ⊙ 1[pre > 0] on hidden layers (R12), dPre = dLogits on the last
            std::vector<double> dpre(n_in * dout, 0.0);
            for (size_t r = 0; r < n_in; ++r)
                for (int c = 0; c < dout; ++c) {
                    double g = o.dH[l][(size_t)P.V[r] * dout + c];
                    dpre[r * dout + c] = (l < L) ? (PREs[l][i][r * dout + c] > 0.0 ? g : 0.0) : g;
                }
            // weight gradient of this partition
            const int wrows = (o.kind == KIND_SAGE) ? 2 * din : (o.kind == KIND_GAT) ? din + 2 : din;
            std::vector<double>& g = gW[i][l - 1];
            g.assign((size_t)wrows * dout, 0.0);
            if (o.kind == KIND_GAT) {
                std::vector<double>& dX = dXs[i];
                gat_backward(o, i, idx[i].row, Xs[l][i], din, dout, W[l - 1], dpre, g, l > 1 ? &dX : nullptr, l);
                continue;
            }
            // dW = [Z | X]^T dPre: g[k][c] accumulates over r in ascending order (the loop nest order only changes
            // which element is visited next, not the order of any element's sum)
            for (size_t r = 0; r < n_in; ++r) {
                const double* d = &dpre[r * dout];
                for (int k = 0; k < din; ++k) {
                    const double zk = Zs[l][i][r * din + k];
                    double* gk = &g[(size_t)k * dout];
                    for (int c = 0; c < dout; ++c) gk[c] += zk * d[c];
                }
                if (o.kind == KIND_SAGE)
                    for (int k = 0; k < din; ++k) {
                        const double xk = Xs[l][i][r * din + k];
                        double* gk = &g[(size_t)(din + k) * dout];
                        for (int c = 0; c < dout; ++c) gk[c] += xk * d[c];
                    }
            }
            if (l == 1) continue;                   // R29: input features are not trainable
            // dZ' = (dPre W_top^T) s_v with s_v = 1/deg_G(v) (SAGE, 0 if deg 0) or 1/sqrt(d~_v) (GCN) -- the
            // row factor of the aggregation coefficient; dXself = dPre W_bot^T (SAGE self half of CONCAT)
            std::vector<double> dZp(n_in * din, 0.0), dXself(n_in * din, 0.0);
            for (size_t r = 0; r < n_in; ++r) {
                int64_t dv = deg(o, P.V[r]);
                double sv = (o.kind == KIND_SAGE) ? (dv ? 1.0 / (double)dv : 0.0) : 1.0 / std::sqrt((double)(dv + 1));
                for (int k = 0; k < din; ++k) {
                    double a = 0.0, b = 0.0;
                    for (int c = 0; c < dout; ++c) {
                        a += dpre[r * dout + c] * Wl[(size_t)k * dout + c];
                        if (o.kind == KIND_SAGE) b += dpre[r * dout + c] * Wl[(size_t)(din + k) * dout + c];
                    }
                    dZp[r * din + k] = a * sv;
                    dXself[r * din + k] = b;
                }
            }
            // transpose of the aggregation over the kept edges of every inner v:
            //   SAGE dX_u = [u inner] dXself_u + c_u sum_{v: u in N(v)} dZ'_v
            //   GCN  dX_u = c_u rs_u (sum_{v: u in N(v)} dZ'_v + [u inner] dZ'_u)
            std::vector<double>& dX = dXs[i];
            dX.assign((n_in + n_h) * din, 0.0);
            for (size_t r = 0; r < n_in; ++r) {
                int32_t v = P.V[r];
                if (o.kind == KIND_GCN) {
                    double rs = 1.0 / std::sqrt((double)(deg(o, v) + 1));
                    for (int k = 0; k < din; ++k) dX[r * din + k] += rs * dZp[r * din + k];
                }
                for (int64_t e = o.indptr[v]; e < o.indptr[v + 1]; ++e) {
                    int32_t u = o.indices[e];
                    int64_t ru = idx[i].row[u];
                    double c;
                    if (!arc_in(o, v, u, ru, (int64_t)n_in, &c)) continue;
                    if (o.kind == KIND_GCN) c /= std::sqrt((double)(deg(o, u) + 1));
                    for (int k = 0; k < din; ++k) dX[(size_t)ru * din + k] += c * dZp[r * din + k];
                }
            }
            for (size_t r = 0; r < n_in + n_h; ++r)
                for (int k = 0; k < din; ++k) {
                    double x = dX[r * din + k];
                    if (o.kind == KIND_SAGE && r < n_in) x += dXself[r * din + k];
                    if (o.drop > 0.0) {   // R38: through the dropout of this layer's input
                        const int32_t u = (r < n_in) ? P.V[r] : P.U[r - n_in];
                        x = x * drop_factor(o, u, k, l);
                    }
                    dX[r * din + k] = x;
                }
        }
        if (l == 1) continue;
        // reverse exchange: halo-row gradients go back to their owners and are added into the owners'
        // rows, local contribution first, then peers in ascending id (R25).
        o.dH[l - 1].assign((size_t)o.N * din, 0.0);
        for (int j = 0; j < m; ++j) {
            const Partition& Q = o.parts[j];
            for (size_t r = 0; r < Q.V.size(); ++r)
                for (int k = 0; k < din; ++k) o.dH[l - 1][(size_t)Q.V[r] * din + k] = dXs[j][r * din + k];
        }
        for (int j = 0; j < m; ++j) {               // owner j
            for (int i = 0; i < m; ++i) {           // sender i (holds j's rows as halo), ascending
                if (i == j) continue;
                const Partition& P = o.parts[i];
                const size_t n_in = P.V.size();
                for (int64_t s = P.U_off[j]; s < P.U_off[j + 1]; ++s) {
                    int32_t u = P.U[s];
                    for (int k = 0; k < din; ++k) {
                        double& t = o.dH[l - 1][(size_t)u * din + k];
                        t = t + dXs[i][(n_in + (size_t)s) * din + k];
                    }
                }
            }
        }
    }

    // ---------------- AllReduce (l.13, sum in rank order, R21) and SGD update (l.14) ----------------
    o.G.assign(L, std::vector<double>());
    if (o.optimizer == 1) {
        ++o.adam_t;
        if ((int)o.adam_m.size() != L) { o.adam_m.assign(L, {}); o.adam_v.assign(L, {}); }
    }
    for (int l = 0; l < L; ++l) {
        o.G[l].assign(W[l].size(), 0.0);
        for (int i = 0; i < m; ++i)
            for (size_t k = 0; k < W[l].size(); ++k) o.G[l][k] += gW[i][l][k];
        if (o.optimizer == 0) {
            for (size_t k = 0; k < W[l].size(); ++k) W[l][k] -= lr * o.G[l][k];
        } else {
            // Adam (Kingma & Ba; bias-corrected), the paper's optimizer, f2
            std::vector<double>& mm = o.adam_m[l];
            std::vector<double>& vv = o.adam_v[l];
            if (mm.size() != W[l].size()) { mm.assign(W[l].size(), 0.0); vv.assign(W[l].size(), 0.0); }
            const double c1 = 1.0 - std::pow(o.beta1, (double)o.adam_t), c2 = 1.0 - std::pow(o.beta2, (double)o.adam_t);
            for (size_t k = 0; k < W[l].size(); ++k) {
                const double g = o.G[l][k];
                mm[k] = o.beta1 * mm[k] + (1.0 - o.beta1) * g;
                vv[k] = o.beta2 * vv[k] + (1.0 - o.beta2) * g * g;
                W[l][k] -= lr * (mm[k] / c1) / (std::sqrt(vv[k] / c2) + o.eps);
            }
        }
    }
    return 0;
}

}  // namespace

// =============================================================================================
// C ABI (ctypes) -- used only by tests/ and bench.py's oracle legs.
// =============================================================================================
extern "C" {

void orc_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) { philox4x32_10(ctr, key, out); }
uint32_t orc_draw(uint32_t u, uint32_t i, uint64_t epoch, uint64_t seed) { return draw(u, i, epoch, seed); }
uint64_t orc_threshold(double p) { return threshold_of(p); }

void* orc_create(int64_t N, const int64_t* indptr, const int32_t* indices, const int32_t* part_of, int32_t m,
                 int32_t L, const int32_t* dims, int32_t kind, const float* features, const int32_t* labels) {
    Oracle* o = new Oracle();
    o->N = N;
    o->indptr.assign(indptr, indptr + N + 1);
    o->indices.assign(indices, indices + indptr[N]);
    o->part_of.assign(part_of, part_of + N);
    o->m = m;
    o->L = L;
    o->dims.assign(dims, dims + L + 1);
    o->kind = kind;
    o->X.assign((size_t)N * dims[0], 0.0);
    if (features) for (size_t k = 0; k < o->X.size(); ++k) o->X[k] = (double)features[k];
    o->labels.assign(labels, labels + N);
    build_plan(*o);
    return o;
}

void orc_destroy(void* h) { delete (Oracle*)h; }

// what: 0=V_i 1=B_i 2=B_off 3=D_{i->peer} 4=U_i 5=U_off 6=S_{i,peer} 7=keep mask of B_i (as int32)
int64_t orc_list(void* h, int32_t what, int32_t rank, int32_t peer, int64_t* out, int64_t cap) {
    Oracle& o = *(Oracle*)h;
    const Partition& P = o.parts[rank];
    std::vector<int64_t> v;
    switch (what) {
        case 0: v.assign(P.V.begin(), P.V.end()); break;
        case 1: v.assign(P.B.begin(), P.B.end()); break;
        case 2: v.assign(P.B_off.begin(), P.B_off.end()); break;
        case 3: v.assign(P.D[peer].begin(), P.D[peer].end()); break;
        case 4: v.assign(P.U.begin(), P.U.end()); break;
        case 5: v.assign(P.U_off.begin(), P.U_off.end()); break;
        case 6: v.assign(P.S[peer].begin(), P.S[peer].end()); break;
        case 7: v.assign(P.keep_B.begin(), P.keep_B.end()); break;
        case 8:     // induced (sampled) forward CSR of partition rank: row pointers over V_i
        case 9: {   // ... and the gids of the kept arcs, rows in V_i order, neighbours in global order
            if (!o.sampled) return -1;
            std::vector<int64_t> row(o.N, -1);
            for (size_t r = 0; r < P.V.size(); ++r) row[P.V[r]] = (int64_t)r;
            for (size_t s = 0; s < P.U.size(); ++s) row[P.U[s]] = (int64_t)(P.V.size() + s);
            std::vector<int64_t> ptr(1, 0), col;
            for (int32_t x : P.V) {
                for (int64_t e = o.indptr[x]; e < o.indptr[x + 1]; ++e) {
                    double c;
                    if (arc_in(o, x, o.indices[e], row[o.indices[e]], (int64_t)P.V.size(), &c)) col.push_back(o.indices[e]);
                }
                ptr.push_back((int64_t)col.size());
            }
            if (what == 8) v = ptr; else v = col;
            break;
        }
        default: return -1;
    }
    int64_t n = (int64_t)v.size();
    if (out) for (int64_t k = 0; k < std::min(n, cap); ++k) out[k] = v[k];
    return n;
}

int32_t orc_sample(void* h, double p, uint64_t seed, uint64_t epoch) {
    Oracle& o = *(Oracle*)h;
    if (!(p >= 0.0 && p <= 1.0)) return 1;
    sample(o, p, seed, epoch);
    finish_sample(o);
    o.epoch_id = epoch;
    return 0;
}

// f2: optimizer (0 SGD, 1 Adam) and dropout rate / seed.  Resets the Adam state.
int32_t orc_set_training(void* h, int32_t optimizer, double beta1, double beta2, double eps, double drop,
                         uint64_t drop_seed) {
    Oracle& o = *(Oracle*)h;
    if (optimizer < 0 || optimizer > 1 || !(drop >= 0.0 && drop < 1.0)) return 1;
    o.optimizer = optimizer;
    o.beta1 = beta1;
    o.beta2 = beta2;
    o.eps = eps;
    o.drop = drop;
    o.drop_seed = drop_seed;
    o.adam_t = 0;
    o.adam_m.clear();
    o.adam_v.clear();
    return 0;
}

double orc_drop_factor(void* h, int32_t u, int32_t c, int32_t l) { return drop_factor(*(Oracle*)h, u, c, l); }

// f3: edge samplers (1 BES, 2 DropEdge) with arc keep probability q; then S_{i,j} as for BNS.
int32_t orc_sample_edges(void* h, int32_t sampler, double q, uint64_t seed, uint64_t epoch) {
    Oracle& o = *(Oracle*)h;
    if (!(q >= 0.0 && q <= 1.0) || (sampler != SAMPLER_BES && sampler != SAMPLER_DROPEDGE)) return 1;
    sample_edges(o, sampler, q, seed, epoch);
    finish_sample(o);
    return 0;
}

// R40 arc draw (v <- u) under the last orc_sample_edges' q / seed / epoch
int32_t orc_arc_keep(void* h, int32_t v, int32_t u) { return arc_keep(*(Oracle*)h, v, u) ? 1 : 0; }

// f4 / R44: multi-label targets, N x C (global ids) in {0, 1}; switches the loss to sigmoid BCE and acc to F1-micro
void orc_set_multilabel(void* h, const uint8_t* targets) {
    Oracle& o = *(Oracle*)h;
    const int C = o.dims[o.L];
    o.multilabel = targets != nullptr;
    o.targets.assign(targets ? targets : (const uint8_t*)nullptr, targets ? targets + (size_t)o.N * C : nullptr);
}

// Explicit draw (for the hand-computed goldens): keep flags for B_rank in B order.
int32_t orc_set_keep(void* h, double p, int32_t rank, const int32_t* flags) {
    Oracle& o = *(Oracle*)h;
    o.p = p;
    o.sampler = SAMPLER_BNS;
    Partition& P = o.parts[rank];
    P.keep_B.assign(P.B.size(), 0);
    for (size_t k = 0; k < P.B.size(); ++k) P.keep_B[k] = flags[k] ? 1 : 0;
    bool all = true;
    for (const Partition& Q : o.parts) if (Q.keep_B.size() != Q.B.size()) all = false;
    if (all) finish_sample(o);
    return 0;
}

// W: L pointers to row-major weights (updated in place), G: L pointers receiving the all-reduced gradient.
int32_t orc_epoch(void* h, double* const* W, double lr, double* const* G, double* loss, double* acc) {
    Oracle& o = *(Oracle*)h;
    std::vector<std::vector<double>> Wv(o.L);
    for (int l = 0; l < o.L; ++l) {
        int din = o.dims[l], dout = o.dims[l + 1];
        size_t rows = (o.kind == KIND_SAGE) ? 2 * (size_t)din : (o.kind == KIND_GAT) ? (size_t)din + 2 : (size_t)din;
        Wv[l].assign(W[l], W[l] + rows * dout);
    }
    int rc = epoch(o, Wv, lr, loss, acc);
    if (rc) return rc;
    for (int l = 0; l < o.L; ++l) {
        std::copy(Wv[l].begin(), Wv[l].end(), W[l]);
        if (G && G[l]) std::copy(o.G[l].begin(), o.G[l].end(), G[l]);
    }
    return 0;
}

// what: 0 = H^l (N x dims[l]; l=L gives logits), 1 = Z^l (N x dims[l-1]), 2 = dH^l (N x dims[l], l<L;
// l=L gives dLogits).  Returns elements written, -1 if unavailable.
int64_t orc_tensor(void* h, int32_t what, int32_t layer, double* out, int64_t cap) {
    Oracle& o = *(Oracle*)h;
    const std::vector<std::vector<double>>* T = (what == 0) ? &o.H : (what == 1) ? &o.Z : (what == 2) ? &o.dH : nullptr;
    if (!T || layer < 0 || layer >= (int)T->size()) return -1;
    const std::vector<double>& t = (*T)[layer];
    int64_t n = (int64_t)t.size();
    if (out) std::copy(t.begin(), t.begin() + std::min(n, cap), out);
    return n;
}

int64_t orc_rows_sent(void* h, int32_t layer) {
    Oracle& o = *(Oracle*)h;
    return (layer >= 0 && layer < (int)o.rows_sent_fwd.size()) ? o.rows_sent_fwd[layer] : -1;
}

}  // extern "C"
