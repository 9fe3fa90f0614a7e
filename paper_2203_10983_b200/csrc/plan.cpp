// plan.cpp -- a0: the static per-rank plan (SETUP, host, never timed).
//
// PAPER.md:173-176 (§3.1, Fig. fig:framework): every partition holds an inner node set V_i and a boundary node set
// B_i of nodes owned by other partitions that neighbour V_i.  Alg.1 l.1.  Ordering readings:
// V_i ascending gid (local row r <-> V_i[r]); B_i by (owner, gid) (R24); D_{i->j} = B_j ∩ V_i ascending gid --
// the candidates from which S_{i,j} = U_j ∩ V_i is recomputed every epoch (R27).
#include "common.h"

#include <algorithm>

namespace bns {

void build_plan(Plan& P, int rank, int world, int64_t N, const int64_t* indptr, const int32_t* indices,
                const int32_t* part_of) {
    P = Plan();
    P.rank = rank;
    P.world = world;
    P.N = N;
    std::vector<int32_t> local(N, -1), bidx(N, -1);
    for (int64_t v = 0; v < N; ++v)
        if (part_of[v] == rank) {
            local[v] = (int32_t)P.V.size();
            P.V.push_back((int32_t)v);
        }
    P.n_in = (int64_t)P.V.size();

    // B_i: neighbours of inner nodes owned elsewhere, grouped by owner, ascending gid within an owner
    std::vector<uint8_t> mark(N, 0);
    for (int32_t v : P.V)
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
            int32_t u = indices[e];
            if (part_of[u] != rank) mark[u] = 1;
        }
    std::vector<std::vector<int32_t>> by_owner(world);
    for (int64_t u = 0; u < N; ++u)
        if (mark[u]) by_owner[part_of[u]].push_back((int32_t)u);
    P.B_off.assign(world + 1, 0);
    for (int j = 0; j < world; ++j) {
        P.B_off[j] = (int64_t)P.B.size();
        P.B.insert(P.B.end(), by_owner[j].begin(), by_owner[j].end());
    }
    P.B_off[world] = (int64_t)P.B.size();
    P.n_bd = (int64_t)P.B.size();
    for (int64_t b = 0; b < P.n_bd; ++b) bidx[P.B[b]] = (int32_t)b;
    {   // owner-local row of every boundary node: its rank among the owner's nodes in ascending gid
        std::vector<int32_t> seen(world, 0);
        P.B_row.assign(P.n_bd, 0);
        for (int64_t u = 0; u < N; ++u) {
            const int32_t r = seen[part_of[u]]++;
            if (bidx[u] >= 0) P.B_row[bidx[u]] = r;
        }
    }

    // D_{i->j}: inner v with >= 1 neighbour in partition j != i, ascending gid
    std::vector<std::vector<int32_t>> D(world);
    std::vector<int64_t> stamp(world, -1);
    for (int64_t r = 0; r < P.n_in; ++r) {
        int32_t v = P.V[r];
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
            int32_t j = part_of[indices[e]];
            if (j != rank && stamp[j] != r) {
                stamp[j] = r;
                D[j].push_back((int32_t)r);
            }
        }
    }
    P.D_off.assign(world + 1, 0);
    for (int j = 0; j < world; ++j) {
        P.D_off[j] = (int64_t)P.D_local.size();
        P.D_local.insert(P.D_local.end(), D[j].begin(), D[j].end());
    }
    P.D_off[world] = (int64_t)P.D_local.size();
    P.n_send = (int64_t)P.D_local.size();

    // static CSR over inner rows (full rows in global neighbour order) + its inner-only part A_II
    P.row_ptr.assign(P.n_in + 1, 0);
    P.ii_ptr.assign(P.n_in + 1, 0);
    for (int64_t r = 0; r < P.n_in; ++r) {
        int32_t v = P.V[r];
        P.row_ptr[r + 1] = P.row_ptr[r] + (indptr[v + 1] - indptr[v]);
        int64_t c = 0;
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) c += (local[indices[e]] >= 0);
        P.ii_ptr[r + 1] = P.ii_ptr[r] + c;
    }
    P.col_enc.resize(P.row_ptr[P.n_in]);
    P.ii_col.resize(P.ii_ptr[P.n_in]);
    std::vector<int64_t> br_cnt(P.n_bd + 1, 0);
    for (int64_t r = 0; r < P.n_in; ++r) {
        int32_t v = P.V[r];
        int64_t k = P.row_ptr[r], q = P.ii_ptr[r];
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
            int32_t u = indices[e];
            if (local[u] >= 0) {
                P.col_enc[k++] = local[u];
                P.ii_col[q++] = local[u];
            } else {
                P.col_enc[k++] = -(bidx[u] + 1);
                br_cnt[bidx[u] + 1]++;
            }
        }
    }
    // boundary rows: inner neighbours of each boundary node, ascending local id (= ascending gid)
    P.br_ptr.assign(P.n_bd + 1, 0);
    for (int64_t b = 0; b < P.n_bd; ++b) P.br_ptr[b + 1] = P.br_ptr[b] + br_cnt[b + 1];
    P.br_col.resize(P.br_ptr[P.n_bd]);
    std::vector<int64_t> fill(P.br_ptr.begin(), P.br_ptr.end() - 1);
    for (int64_t r = 0; r < P.n_in; ++r)
        for (int64_t k = P.row_ptr[r]; k < P.row_ptr[r + 1]; ++k)
            if (P.col_enc[k] < 0) P.br_col[fill[-P.col_enc[k] - 1]++] = (int32_t)r;

    P.deg_in.resize(P.n_in);
    for (int64_t r = 0; r < P.n_in; ++r) P.deg_in[r] = (float)(indptr[P.V[r] + 1] - indptr[P.V[r]]);
    P.deg_bd.resize(P.n_bd);
    for (int64_t b = 0; b < P.n_bd; ++b) P.deg_bd[b] = (float)(indptr[P.B[b] + 1] - indptr[P.B[b]]);
}

}  // namespace bns
