// gen.cpp -- seeded synthetic INPUT generators (SETUP, never timed).  Serves both the oracle-side tests and
// the CUDA path; holds none of the method's arithmetic (no sampling, aggregation, update or loss).
//
//   gen_rmat_*        R-MAT graph (Graph500 a,b,c,d = .57,.19,.19,.05), symmetrised, deduplicated, no self loops,
//                     ascending columns, relabelled by a seeded permutation.  Workload recipe: SURVEY.md §8(d)
//                     "Workload generation"; shapes from PAPER.md:375-387 (Table tab:setups).
//   gen_features      x = k/64, k = (Philox(seed, gid, col).x >> 25) - 64 -- exact in fp32 and bf16.
//   gen_labels        uniform class in [0,C); train mask Bernoulli(train_frac) (tab:setups split), else -1.
//   gen_weights       Glorot-uniform from Philox.
//   part_ldg2         deterministic two-constraint (nodes, nnz) linear-deterministic-greedy partitioner
//                     (METIS stand-in; PAPER.md:239-247 Goal-1/Goal-2; SURVEY.md §8(d) partitioner choice).
//   part_random       balanced random partition.
//
// Philox here is a third, private copy (generator stream only); the sampler's Philox lives separately in
// oracle/ and in csrc/.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>
#include <parallel/algorithm>
#include <omp.h>

namespace {

inline void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, uint32_t out[4]) {
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

struct RmatGraph {
    int64_t N = 0;
    std::vector<int64_t> indptr;
    std::vector<int32_t> indices;
};

}  // namespace

extern "C" {

// ------------------------------------------------------------------------------------------------
// R-MAT.  Draw batches of undirected edges until the symmetric arc count reaches target_nnz.
// ------------------------------------------------------------------------------------------------
void* gen_rmat_build(int64_t N, int64_t target_nnz, double a, double b, double c, uint64_t seed) {
    int scale = 0;
    while ((int64_t(1) << scale) < N) ++scale;
    const uint32_t ta = (uint32_t)std::min(4294967295.0, std::floor(a * 4294967296.0));
    const uint32_t tab = (uint32_t)std::min(4294967295.0, std::floor((a + b) * 4294967296.0));
    const uint32_t tabc = (uint32_t)std::min(4294967295.0, std::floor((a + b + c) * 4294967296.0));
    std::vector<uint64_t> arcs;   // (u << 32) | v, sorted unique
    uint32_t batch = 0;
    uint64_t drawn = 0;
    while ((int64_t)arcs.size() < target_nnz && N > 1) {
        int64_t need = (target_nnz - (int64_t)arcs.size()) / 2 + 1;
        int64_t nb = need + 32;
        std::vector<uint64_t> fresh(2 * nb, ~0ull);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < nb; ++k) {
            uint64_t id = drawn + (uint64_t)k;
            uint32_t u = 0, v = 0;
            uint32_t r[4];
            for (int lvl = 0; lvl < scale; ++lvl) {
                if ((lvl & 3) == 0) philox((uint32_t)id, (uint32_t)(id >> 32), (uint32_t)(lvl >> 2), batch,
                                           (uint32_t)seed, (uint32_t)(seed >> 32) ^ 0x52u, r);
                uint32_t x = r[lvl & 3];
                uint32_t bu = 0, bv = 0;
                if (x < ta) { bu = 0; bv = 0; }
                else if (x < tab) { bu = 0; bv = 1; }
                else if (x < tabc) { bu = 1; bv = 0; }
                else { bu = 1; bv = 1; }
                u = (u << 1) | bu;
                v = (v << 1) | bv;
            }
            if ((int64_t)u >= N || (int64_t)v >= N || u == v) continue;
            fresh[2 * k] = ((uint64_t)u << 32) | v;
            fresh[2 * k + 1] = ((uint64_t)v << 32) | u;
        }
        drawn += (uint64_t)nb;
        ++batch;
        __gnu_parallel::sort(fresh.begin(), fresh.end());
        fresh.erase(std::unique(fresh.begin(), fresh.end()), fresh.end());
        if (!fresh.empty() && fresh.back() == ~0ull) fresh.pop_back();
        std::vector<uint64_t> merged;
        merged.reserve(arcs.size() + fresh.size());
        std::merge(arcs.begin(), arcs.end(), fresh.begin(), fresh.end(), std::back_inserter(merged));
        merged.erase(std::unique(merged.begin(), merged.end()), merged.end());
        arcs.swap(merged);
        if (batch > 200) break;
    }
    // relabel with a seeded random permutation: new id = rank of Philox key
    std::vector<uint64_t> key((size_t)N);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; ++v) {
        uint32_t r[4];
        philox((uint32_t)v, 0x5045524du, 0, 0, (uint32_t)seed, (uint32_t)(seed >> 32) ^ 0x9u, r);
        key[v] = ((uint64_t)r[0] << 32) | (uint64_t)r[1];
    }
    std::vector<int32_t> order((size_t)N);
    std::iota(order.begin(), order.end(), 0);
    __gnu_parallel::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
        return key[x] < key[y] || (key[x] == key[y] && x < y);
    });
    std::vector<int32_t> newid((size_t)N);
    for (int64_t r = 0; r < N; ++r) newid[order[r]] = (int32_t)r;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)arcs.size(); ++k) {
        uint32_t u = (uint32_t)(arcs[k] >> 32), v = (uint32_t)arcs[k];
        arcs[k] = ((uint64_t)(uint32_t)newid[u] << 32) | (uint32_t)newid[v];
    }
    __gnu_parallel::sort(arcs.begin(), arcs.end());
    RmatGraph* g = new RmatGraph();
    g->N = N;
    g->indptr.assign((size_t)N + 1, 0);
    g->indices.resize(arcs.size());
    for (size_t k = 0; k < arcs.size(); ++k) {
        g->indptr[(arcs[k] >> 32) + 1]++;
        g->indices[k] = (int32_t)(uint32_t)arcs[k];
    }
    for (int64_t v = 0; v < N; ++v) g->indptr[v + 1] += g->indptr[v];
    return g;
}

int64_t gen_rmat_nnz(void* h) { return (int64_t)((RmatGraph*)h)->indices.size(); }

void gen_rmat_fetch(void* h, int64_t* indptr, int32_t* indices) {
    RmatGraph* g = (RmatGraph*)h;
    std::memcpy(indptr, g->indptr.data(), g->indptr.size() * sizeof(int64_t));
    std::memcpy(indices, g->indices.data(), g->indices.size() * sizeof(int32_t));
}

void gen_rmat_free(void* h) { delete (RmatGraph*)h; }

// features for the listed rows (global ids), row-major n_rows x d
void gen_features(int64_t n_rows, const int32_t* gids, int32_t d, uint64_t seed, float* out) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n_rows; ++r) {
        uint32_t rr[4];
        for (int32_t c = 0; c < d; ++c) {
            philox((uint32_t)gids[r], (uint32_t)c, 0x46454154u, 0, (uint32_t)seed, (uint32_t)(seed >> 32), rr);
            int32_t k = (int32_t)(rr[0] >> 25) - 64;
            out[r * (int64_t)d + c] = (float)k / 64.0f;
        }
    }
}

void gen_labels(int64_t N, int32_t C, double train_frac, uint64_t seed, int32_t* out) {
    const uint64_t T = (uint64_t)std::floor(train_frac * 4294967296.0);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; ++v) {
        uint32_t r[4];
        philox((uint32_t)v, 0x4C41424Cu, 0, 0, (uint32_t)seed, (uint32_t)(seed >> 32), r);
        int32_t y = (int32_t)(((uint64_t)r[0] * (uint64_t)C) >> 32);
        out[v] = ((uint64_t)r[1] < T) ? y : -1;
    }
}

// Glorot-uniform rows x cols, limit sqrt(6/(rows+cols)); `layer` separates the streams of different layers.
void gen_weights(int64_t rows, int64_t cols, int32_t layer, uint64_t seed, float* out) {
    const double lim = std::sqrt(6.0 / (double)(rows + cols));
    for (int64_t k = 0; k < rows * cols; ++k) {
        uint32_t r[4];
        philox((uint32_t)k, (uint32_t)(k >> 32), (uint32_t)layer, 0x57u, (uint32_t)seed, (uint32_t)(seed >> 32), r);
        double u = (double)r[0] / 4294967296.0;
        out[k] = (float)((2.0 * u - 1.0) * lim);
    }
}

// ------------------------------------------------------------------------------------------------
// Balanced random partition: nodes sorted by a Philox key, dealt round-robin (sizes differ by <= 1).
// ------------------------------------------------------------------------------------------------
void part_random(int64_t N, int32_t m, uint64_t seed, int32_t* part_of) {
    std::vector<uint64_t> key((size_t)N);
    for (int64_t v = 0; v < N; ++v) {
        uint32_t r[4];
        philox((uint32_t)v, 0x52414E44u, 0, 0, (uint32_t)seed, (uint32_t)(seed >> 32), r);
        key[v] = ((uint64_t)r[0] << 32) | r[1];
    }
    std::vector<int32_t> order((size_t)N);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
        return key[x] < key[y] || (key[x] == key[y] && x < y);
    });
    for (int64_t r = 0; r < N; ++r) part_of[order[r]] = (int32_t)(r % m);
}

// ------------------------------------------------------------------------------------------------
// Two-constraint LDG.  Stream order: BFS from a seeded root (restarting at the lowest unvisited id).
// Node x goes to argmax_k |N(x) ∩ P_k| * (1 - max(n_k/cap_n, e_k/cap_e)) over parts that stay within
// both caps (cap = (1+slack) * total/m); ties -> smaller max fill, then lowest id.  If no part has room
// the least-filled part is used.
// ------------------------------------------------------------------------------------------------
void part_ldg2(int64_t N, const int64_t* indptr, const int32_t* indices, int32_t m, double slack, uint64_t seed,
               int32_t* part_of) {
    const int64_t nnz = indptr[N];
    const double cap_n = (1.0 + slack) * (double)N / m;
    const double cap_e = (1.0 + slack) * (double)std::max<int64_t>(nnz, 1) / m;
    std::vector<double> fill_n(m, 0.0), fill_e(m, 0.0);
    std::vector<int64_t> cnt(m, 0);
    std::fill(part_of, part_of + N, -1);
    std::vector<uint8_t> seen((size_t)N, 0);
    std::vector<int32_t> queue;
    queue.reserve((size_t)N);
    uint32_t r[4];
    philox(0x524F4F54u, 0, 0, 0, (uint32_t)seed, (uint32_t)(seed >> 32), r);
    int64_t root = N ? (int64_t)(((uint64_t)r[0] * (uint64_t)N) >> 32) : 0;
    int64_t next_unvisited = 0;
    size_t head = 0;
    auto assign = [&](int32_t x) {
        for (int k = 0; k < m; ++k) cnt[k] = 0;
        for (int64_t e = indptr[x]; e < indptr[x + 1]; ++e) {
            int32_t p = part_of[indices[e]];
            if (p >= 0) cnt[p]++;
        }
        const double dx = (double)(indptr[x + 1] - indptr[x]);
        int best = -1;
        double best_score = -1.0, best_fill = 2.0;
        for (int k = 0; k < m; ++k) {
            double fn = (fill_n[k] + 1.0) / cap_n, fe = (fill_e[k] + dx) / cap_e;
            if (fn > 1.0 || fe > 1.0) continue;
            double f = std::max(fill_n[k] / cap_n, fill_e[k] / cap_e);
            double score = (double)cnt[k] * (1.0 - f);
            if (score > best_score || (score == best_score && f < best_fill)) {
                best = k; best_score = score; best_fill = f;
            }
        }
        if (best < 0) {
            double bf = 1e300;
            for (int k = 0; k < m; ++k) {
                double f = std::max(fill_n[k] / cap_n, fill_e[k] / cap_e);
                if (f < bf) { bf = f; best = k; }
            }
        }
        part_of[x] = best;
        fill_n[best] += 1.0;
        fill_e[best] += dx;
    };
    for (int64_t done = 0; done < N;) {
        if (head == queue.size()) {
            int64_t s = root;
            if (seen[s]) {
                while (next_unvisited < N && seen[next_unvisited]) ++next_unvisited;
                s = next_unvisited;
            }
            seen[s] = 1;
            queue.push_back((int32_t)s);
        }
        int32_t x = queue[head++];
        assign(x);
        ++done;
        for (int64_t e = indptr[x]; e < indptr[x + 1]; ++e) {
            int32_t u = indices[e];
            if (!seen[u]) { seen[u] = 1; queue.push_back(u); }
        }
    }
}

}  // extern "C"
