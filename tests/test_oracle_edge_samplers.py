"""f3 oracle pins: the edge samplers BES and DropEdge (Table tab:bes P:629-651)
under readings R40 (one Philox arc draw per directed arc v <- u) and R41 (kept arcs carry 1/q; BES keeps every
intra-partition arc; a boundary node is communicated iff one of its arcs into the receiving partition survives).

Pins, none of which reuses the oracle's own sampling or aggregation code:
* the communicated sets U_i re-derived from the arc definition with the KAT-pinned Philox;
* q = 1 reduces both samplers to BNS p = 1, q = 0 reduces BES to BNS p = 0 (bitwise equal epochs);
* dense float64 brute force with torch autograd on the arc-sampled adjacency (forward AND backward);
* closed forms: K1,5 P(center communicated) = 1 - (1-q)^5; E|U| = sum_b 1 - (1-q)^{deg_i(b)};
* unbiasedness of the 1/q-scaled aggregate (Monte Carlo);
* the paper's Table 8 ordering at matched dropped-edge counts: BNS <= BES <= DropEdge rows sent.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2203_10983_b200 import inputs as I

from dense_ref import forward_backward

M32 = 0xFFFFFFFF


def arc_draw(v, u, epoch, seed, q):
    """R40 restated: Philox4x32-10(ctr={v,u,e_lo,e_hi}, key={s_lo^0xED6E, s_hi}).x < floor(q 2^32)."""
    out = O.philox4x32_10([v, u, epoch & M32, epoch >> 32], [(seed & M32) ^ 0xED6E, seed >> 32])
    return out[0] < O.threshold(q)


def case(seed, N=24, m=3, layer=0, dims=(3, 5, 4, 3), nnz_per=4):
    rng = np.random.default_rng(seed)
    ip, ix = I.rmat(N, nnz_per * N, seed=2000 + seed)
    part = rng.integers(0, m, N).astype(np.int32)
    part[:m] = np.arange(m)
    X = rng.uniform(-1, 1, (N, dims[0])).astype(np.float32)
    y = rng.integers(0, dims[-1], N).astype(np.int32)
    y[rng.uniform(size=N) > 0.8] = -1
    Ws = [rng.uniform(-1, 1, ((2 if layer == 0 else 1) * dims[l], dims[l + 1])) for l in range(len(dims) - 1)]
    return ip, ix, part, X, y, Ws


def arcs_of(ip, ix, part, sampler, q, seed, epoch):
    """(v, u) -> column scale of every arc in the sampled graph (R41)."""
    arcs = {}
    for v in range(len(ip) - 1):
        for u in ix[ip[v]:ip[v + 1]]:
            u = int(u)
            if sampler == O.SAMPLER_BES and part[u] == part[v]:
                arcs[(v, u)] = 1.0
            elif arc_draw(v, u, epoch, seed, q):
                arcs[(v, u)] = 1.0 / q
    return arcs


@pytest.mark.parametrize("sampler", [O.SAMPLER_BES, O.SAMPLER_DROPEDGE])
def test_communicated_sets_from_arc_definition(sampler):
    ip, ix, part, X, y, _ = case(3, N=40, m=4)
    o = O.Oracle(ip, ix, part, 4, [3, 5, 4, 3], 0, X, y)
    q, seed, ep = 0.4, 0xABCDEF0123, 7
    o.sample_edges(sampler, q, seed, ep)
    for i in range(4):
        B = [int(b) for b in o.list(O.B_LIST, i)]
        want = [b for b in B if any(part[v] == i and arc_draw(v, b, ep, seed, q) for v in ix[ip[b]:ip[b + 1]])]
        assert [int(u) for u in o.list(O.U_LIST, i)] == want            # B order (owner-major), R24
        assert list(o.list(O.KEEP, i)) == [1 if b in set(want) else 0 for b in B]
        for j in range(4):                                              # S_{i,j} = U_j ∩ V_i, ascending
            if j != i:
                Uj = [int(u) for u in o.list(O.U_LIST, j)]
                assert [int(s) for s in o.list(O.S_LIST, i, j)] == sorted(u for u in Uj if part[u] == i)
    # the exported predicate is the same draw
    for v in range(10):
        for u in ix[ip[v]:ip[v + 1]]:
            assert o.arc_keep(v, int(u)) == arc_draw(v, int(u), ep, seed, q)


@pytest.mark.parametrize("layer", [0, 1])
@pytest.mark.parametrize("sampler", [O.SAMPLER_BES, O.SAMPLER_DROPEDGE])
def test_q1_is_bns_p1_and_bes_q0_is_bns_p0(layer, sampler):
    ip, ix, part, X, y, Ws = case(4, layer=layer)
    dims = [3, 5, 4, 3]
    ref, got = O.Oracle(ip, ix, part, 3, dims, layer, X, y), O.Oracle(ip, ix, part, 3, dims, layer, X, y)
    for q in ([1.0, 0.0] if sampler == O.SAMPLER_BES else [1.0]):
        ref.sample(q, 5, 5)
        got.sample_edges(sampler, q, 5, 5)
        for r in range(3):
            assert list(ref.list(O.U_LIST, r)) == list(got.list(O.U_LIST, r))
        a = ref.epoch([w.copy() for w in Ws], 0.1)
        b = got.epoch([w.copy() for w in Ws], 0.1)
        assert a[0] == b[0] and a[1] == b[1]
        for g1, g2 in zip(a[2], b[2]):
            assert np.array_equal(g1, g2)
        for l in range(1, 4):
            assert np.array_equal(ref.tensor(O.T_H, l), got.tensor(O.T_H, l))


@pytest.mark.parametrize("layer", [0, 1])
@pytest.mark.parametrize("sampler,q,seed,m", [(O.SAMPLER_BES, 0.5, 1, 3), (O.SAMPLER_BES, 0.2, 2, 4),
                                              (O.SAMPLER_DROPEDGE, 0.5, 3, 3), (O.SAMPLER_DROPEDGE, 0.7, 4, 2),
                                              (O.SAMPLER_DROPEDGE, 0.3, 5, 1), (O.SAMPLER_DROPEDGE, 0.0, 6, 3)])
def test_dense_bruteforce_edge_samplers(layer, sampler, q, seed, m):
    ip, ix, part, X, y, Ws = case(seed, m=m, layer=layer)
    dims = [3, 5, 4, 3]
    o = O.Oracle(ip, ix, part, m, dims, layer, X, y)
    o.sample_edges(sampler, q, 31, seed)
    ref = forward_backward(ip, ix, part, None, None, layer, X, y, Ws, arcs=arcs_of(ip, ix, part, sampler, q, 31, seed))
    loss, acc, G = o.epoch([w.copy() for w in Ws], 0.0)
    assert abs(loss - ref["loss"]) <= 1e-12 * max(1.0, abs(ref["loss"]))
    assert acc == ref["acc"]
    for l in range(1, 4):
        np.testing.assert_allclose(o.tensor(O.T_H, l), ref["H"][l], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(o.tensor(O.T_Z, l), ref["Z"][l - 1], rtol=1e-12, atol=1e-12)
    for l in range(1, 3):
        np.testing.assert_allclose(o.tensor(O.T_DH, l), ref["dH"][l], rtol=1e-10, atol=1e-13)
    for g, r in zip(G, ref["dW"]):
        np.testing.assert_allclose(g, r, rtol=1e-10, atol=1e-13)


def star_k15():
    """K1,5: center 0 in partition 0, leaves 1..5 in partition 1."""
    ip = np.array([0, 5, 6, 7, 8, 9, 10], np.int64)
    ix = np.array([1, 2, 3, 4, 5, 0, 0, 0, 0, 0], np.int32)
    part = np.array([0, 1, 1, 1, 1, 1], np.int32)
    return ip, ix, part


def test_k15_closed_form():
    ip, ix, part = star_k15()
    o = O.Oracle(ip, ix, part, 2, [1, 1], 0, np.zeros((6, 1), np.float32), np.full(6, -1, np.int32))
    T, q = 4000, 0.5
    center = leaves = 0
    for e in range(T):
        o.sample_edges(O.SAMPLER_BES, q, 11, e)
        center += len(o.list(O.U_LIST, 1))     # U_1 ⊆ {0}: the center, needed by the leaves
        leaves += len(o.list(O.U_LIST, 0))     # U_0 ⊆ leaves: one arc each
    pc = 1 - (1 - q) ** 5                      # = 0.96875: "multiple boundary edges connect to the same node"
    assert abs(center / T - pc) <= 4 * np.sqrt(pc * (1 - pc) / T)
    assert abs(leaves / (5 * T) - q) <= 4 * np.sqrt(q * (1 - q) / (5 * T))


@pytest.mark.parametrize("sampler", [O.SAMPLER_BES, O.SAMPLER_DROPEDGE])
@pytest.mark.parametrize("layer", [0, 1])
def test_unbiased_edge_aggregate(sampler, layer):
    # E[z~] = z (1/q on every sampled arc, R41): Monte Carlo mean within 4.5 standard errors
    ip, ix, part, X, y, Ws = case(50, N=30, m=3, layer=layer, dims=(2, 2))
    o = O.Oracle(ip, ix, part, 3, [2, 2], layer, X, y)
    o.sample(1.0, 0, 0)
    o.epoch([Ws[0].copy()], 0.0)
    z_exact = o.tensor(O.T_Z, 1)
    T, q = 3000, 0.4
    acc = []
    for e in range(T):
        o.sample_edges(sampler, q, 99, e)
        o.epoch([Ws[0].copy()], 0.0)
        acc.append(o.tensor(O.T_Z, 1))
    a = np.array(acc)
    se = a.std(0) / np.sqrt(T) + 1e-12
    assert np.all(np.abs(a.mean(0) - z_exact) <= 4.5 * se + 1e-12)


def test_table8_ordering_at_matched_dropped_edges():
    """P:681 "all methods drop the same number of edges with BNS-GCN (p=0.1) over the full graph" -> BES q = p
    (every cross arc survives with probability p in both), DropEdge q' = 1 - (1-p) * cross / nnz."""
    N, m, p = 400, 4, 0.1
    rng = np.random.default_rng(8)
    ip, ix = I.rmat(N, 8 * N, seed=77)
    part = rng.integers(0, m, N).astype(np.int32)
    X = np.zeros((N, 1), np.float32)
    o = O.Oracle(ip, ix, part, m, [1, 1], 0, X, np.full(N, -1, np.int32))
    src = np.repeat(np.arange(N), np.diff(ip))
    cross = int((part[src] != part[ix]).sum())
    q_de = 1 - (1 - p) * cross / len(ix)
    # closed forms: E|U| under BNS = p sum|B_i|; under BES = sum_i sum_{b in B_i} 1 - (1-p)^{deg_i(b)}
    e_bns = e_bes = 0.0
    for i in range(m):
        for b in o.list(O.B_LIST, i):
            di = int((part[ix[ip[b]:ip[b + 1]]] == i).sum())
            e_bns += p
            e_bes += 1 - (1 - p) ** di
    T = 60
    rows = {"bns": [], "bes": [], "de": []}
    for e in range(T):
        o.sample(p, 3, e)
        rows["bns"].append(sum(len(o.list(O.U_LIST, i)) for i in range(m)))
        o.sample_edges(O.SAMPLER_BES, p, 3, e)
        rows["bes"].append(sum(len(o.list(O.U_LIST, i)) for i in range(m)))
        o.sample_edges(O.SAMPLER_DROPEDGE, q_de, 3, e)
        rows["de"].append(sum(len(o.list(O.U_LIST, i)) for i in range(m)))
    mb, me, md = (np.mean(rows[k]) for k in ("bns", "bes", "de"))
    assert abs(mb - e_bns) <= 4 * np.sqrt(e_bns / T) + 1
    assert abs(me - e_bes) <= 4 * np.sqrt(e_bes / T) + 1
    assert mb < me < md    # strict: R-MAT boundary nodes have several cross arcs
