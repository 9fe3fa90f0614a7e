"""Oracle pins: Philox core (Random123 KATs), the sampling layout and threshold (R7), Binomial counts,
independence, inclusion.  Alg.1 l.4: "randomly pick elements in B_i with probability p"."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "philox_kat.json")))


def h(x):
    return int(x, 16) if isinstance(x, str) else int(x)


@pytest.mark.parametrize("kat", G["kat"])
def test_philox_random123_kat(kat):
    out = O.philox4x32_10([h(c) for c in kat["ctr"]], [h(k) for k in kat["key"]])
    assert out == [h(o) for o in kat["out"]]


@pytest.mark.parametrize("v", G["layout"])
def test_layout_vectors(v):
    assert O.draw(v["u"], v["i"], v["epoch"], h(G["seed"])) == h(v["r"])


def test_layout_is_philox_of_counter():
    # the layout definition restated: ctr={u,i,e_lo,e_hi}, key={seed_lo,seed_hi}, r = out.x
    seed, e = h(G["seed"]), (1 << 32) + 5
    out = O.philox4x32_10([77, 3, e & 0xFFFFFFFF, e >> 32], [seed & 0xFFFFFFFF, seed >> 32])
    assert O.draw(77, 3, e, seed) == out[0]


def test_thresholds():
    for p, t in G["thresholds"].items():
        assert O.threshold(float(p)) == t
    # T(p)/2^32 within 2.4e-10 of p
    for p in np.linspace(0, 1, 101):
        assert abs(O.threshold(p) / 2**32 - p) < 2.4e-10


def _tiny(N=60, m=3, seed=11):
    from paper_2203_10983_b200 import inputs as I
    indptr, indices = I.rmat(N, 6 * N, seed=seed)
    part = I.partition(indptr, indices, m, "random")
    dims = [2, 2]
    X = I.features(np.arange(N, dtype=np.int32), 2)
    y = I.labels(N, 2, 1.0)
    return O.Oracle(indptr, indices, part, m, dims, 0, X, y), indptr, indices, part


def test_count_check_and_extremes():
    c = G["count_check"]
    seed = h(G["seed"])
    T = O.threshold(c["p"])
    # count over u in [0, 200000) -- a survey regression pin (its own Python re-implementation)
    kept = sum(1 for u in range(c["u_range"]) if O.draw(u, c["i"], c["epoch"], seed) < T)
    assert kept == c["kept"]
    orc, *_ = _tiny()
    for p, expect_all in ((1.0, True), (0.0, False)):
        orc.sample(p, seed, 3)
        for r in range(orc.m):
            B = orc.list(O.B_LIST, r)
            U = orc.list(O.U_LIST, r)
            assert (list(U) == list(B)) if expect_all else (len(U) == 0)


def test_binomial_counts_and_independence():
    orc, *_ = _tiny(N=200, m=4)
    seed, p, E = 12345, 0.3, 1000
    nB = [len(orc.list(O.B_LIST, r)) for r in range(4)]
    counts = np.zeros((E, 4))
    first = []
    for e in range(E):
        orc.sample(p, seed, e)
        for r in range(4):
            counts[e, r] = len(orc.list(O.U_LIST, r))
        first.append(orc.list(O.KEEP, 0).copy())
    pp = O.threshold(p) / 2**32
    for r in range(4):
        mu, sd = nB[r] * pp, np.sqrt(nB[r] * pp * (1 - pp) / E)
        assert abs(counts[:, r].mean() - mu) < 4 * sd + 1e-12
    f = np.array(first, float)
    a, b = f[:-1].ravel(), f[1:].ravel()
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.05       # epoch-to-epoch independence


def test_inclusion_under_coupled_uniforms():
    orc, *_ = _tiny()
    for e in range(5):
        orc.sample(0.2, 9, e)
        small = [set(orc.list(O.U_LIST, r)) for r in range(orc.m)]
        orc.sample(0.6, 9, e)
        big = [set(orc.list(O.U_LIST, r)) for r in range(orc.m)]
        assert all(s <= b for s, b in zip(small, big))


def test_send_lists_are_receivers_segments():
    # R27: S_{i,j} = U_j ∩ V_i equals the segment of U_j owned by i (S:228 union invariant)
    orc, *_ = _tiny()
    orc.sample(0.5, 1, 2)
    for j in range(orc.m):
        U = orc.list(O.U_LIST, j)
        Uo = orc.list(O.U_OFF, j)
        union = []
        for i in range(orc.m):
            if i == j:
                continue
            S = orc.list(O.S_LIST, i, j)
            assert list(S) == list(U[Uo[i]:Uo[i + 1]])
            union += list(S)
        assert sorted(union) == sorted(U)
