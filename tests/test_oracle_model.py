"""Oracle pins for the layer, loss and backward (Alg.1 l.9-14; GraphSAGE PAPER.md:100;
H/p PAPER.md:335; App. A):

* tiny goldens E1-E6 whose logits are checked by hand below;
* dense-adjacency float64 brute force with torch autograd (tests/dense_ref.py) on random graphs, partitions and
  draws -- independent forward AND backward (incl. reverse exchange + owner accumulation);
* central finite differences of the oracle's own loss;
* invariants: p=1 == unpartitioned (bitwise first-epoch forward), m=1 == full graph, zero upstream -> zero grads,
  uniform logits -> ln C, Eq. 3 accounting of exchanged rows, unbiasedness of the sampled aggregate.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2203_10983_b200 import inputs as I

from dense_ref import forward_backward

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "p4_goldens.json")))


def p4_oracle(layer, dims):
    g = GOLD["graph"]
    ip, ix = I.csr_from_edges(g["N"], g["edges"])
    return O.Oracle(ip, ix, np.array(g["part_of"], np.int32), 2, dims, layer,
                    np.array(g["X"], np.float32), np.array(g["labels"], np.int32))


@pytest.mark.parametrize("name", list(GOLD["cases"]))
def test_goldens(name):
    c = GOLD["cases"][name]
    layer = 0 if c["layer"] == "sage" else 1
    Ws = [np.array(w, np.float64) for w in GOLD[c["W"]]]
    dims = [1] + [w.shape[1] for w in Ws]
    o = p4_oracle(layer, dims)
    if "draw" in c:
        d = GOLD[c["draw"]]
        o.set_keep(c["p"], [d["keep_rank0"], d["keep_rank1"]])
    else:
        o.sample(c["p"], 1, 0)          # p in {0, 1}: draw-independent
    loss, acc, G = o.epoch([w.copy() for w in Ws], 0.0)
    assert abs(loss - c["loss"]) < 1e-8
    assert acc == c["acc"]
    if "logits" in c:
        np.testing.assert_allclose(o.tensor(O.T_H, len(Ws)), c["logits"], atol=1e-12)
        # closed form of the mean CE of the printed logits (labels y)
        y = GOLD["graph"]["labels"]
        ce = [math.log(sum(math.exp(t) for t in row)) - row[y[v]] for v, row in enumerate(c["logits"])]
        assert abs(sum(ce) / 4 - c["loss"]) < 1e-8
    if "H1" in c:
        np.testing.assert_allclose(o.tensor(O.T_H, 1), c["H1"], atol=1e-12)
    if "z" in c:
        np.testing.assert_allclose(o.tensor(O.T_Z, 1), c["z"], atol=1e-12)
    for l, g in enumerate(c.get("dW", [])):
        np.testing.assert_allclose(G[l], g, atol=1e-8)


def test_hand_examples_sage_z():
    # P4, partition {0,1}, halo {2}: z_1 = (1+3)/2 = 2.0 at p=1; (1 + 3/0.5)/2 = 3.5 if kept at
    # p=0.5, (1+0)/2 = 0.5 if dropped; the two equiprobable outcomes average to 2.0 (unbiasedness)
    o = p4_oracle(0, [1, 1])
    W = [np.array([[1.0], [0.0]])]
    vals = []
    for p, keep0 in ((1.0, [1]), (0.5, [1]), (0.5, [0])):
        o.set_keep(p, [keep0, [1]])
        o.epoch([W[0].copy()], 0.0)
        vals.append(o.tensor(O.T_Z, 1)[1, 0])
    assert vals == [2.0, 3.5, 0.5]
    assert (vals[1] + vals[2]) / 2 == vals[0]


def test_gcn_p01():
    # P4 with self loops, d~ = [2,3,3,2], P_{0,1} = 1/sqrt(6); one-hot H picks the column
    o = p4_oracle(1, [4, 4])
    g = GOLD["graph"]
    ip, ix = I.csr_from_edges(4, g["edges"])
    X = np.eye(4, dtype=np.float32)
    o = O.Oracle(ip, ix, np.array(g["part_of"], np.int32), 2, [4, 4], 1, X, np.zeros(4, np.int32))
    o.sample(1.0, 0, 0)
    o.epoch([np.eye(4)], 0.0)
    Z = o.tensor(O.T_Z, 1)
    assert abs(Z[0, 1] - 1 / math.sqrt(6)) < 1e-15
    assert abs(Z[0, 0] - 0.5) < 1e-15 and abs(Z[1, 1] - 1 / 3) < 1e-15


def random_case(seed, N=24, m=3, layer=0, dims=(3, 4, 2), p=0.5, nnz_per=4, train=0.8):
    rng = np.random.default_rng(seed)
    ip, ix = I.rmat(N, nnz_per * N, seed=1000 + seed)
    part = rng.integers(0, m, N).astype(np.int32)
    part[:m] = np.arange(m)               # no empty partition
    X = rng.uniform(-1, 1, (N, dims[0])).astype(np.float32)
    y = rng.integers(0, dims[-1], N).astype(np.int32)
    y[rng.uniform(size=N) > train] = -1
    Ws = [rng.uniform(-1, 1, ((2 if layer == 0 else 1) * dims[l], dims[l + 1])) for l in range(len(dims) - 1)]
    return ip, ix, part, X, y, Ws


@pytest.mark.parametrize("layer", [0, 1])
@pytest.mark.parametrize("seed,m,p", [(1, 2, 0.5), (2, 3, 0.3), (3, 4, 1.0), (4, 3, 0.0), (5, 1, 0.7), (6, 5, 0.9)])
def test_dense_bruteforce(layer, seed, m, p):
    ip, ix, part, X, y, Ws = random_case(seed, m=m, layer=layer, p=p, dims=(3, 5, 4, 3))
    o = O.Oracle(ip, ix, part, m, [3, 5, 4, 3], layer, X, y)
    o.sample(p, 77, seed)
    kept = [set(int(u) for u in o.list(O.U_LIST, r)) for r in range(m)]
    ref = forward_backward(ip, ix, part, kept, p, layer, X, y, Ws)
    loss, acc, G = o.epoch([w.copy() for w in Ws], 0.0)
    assert abs(loss - ref["loss"]) <= 1e-12 * max(1.0, abs(ref["loss"]))
    assert acc == ref["acc"]
    for l in range(1, 4):
        np.testing.assert_allclose(o.tensor(O.T_H, l), ref["H"][l], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(o.tensor(O.T_Z, l), ref["Z"][l - 1], rtol=1e-12, atol=1e-12)
    for l in range(1, 3):   # dH^l: total derivative incl. halo copies returned to owners
        np.testing.assert_allclose(o.tensor(O.T_DH, l), ref["dH"][l], rtol=1e-10, atol=1e-13)
    for g, r in zip(G, ref["dW"]):
        np.testing.assert_allclose(g, r, rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("layer", [0, 1])
def test_finite_differences(layer):
    ip, ix, part, X, y, Ws = random_case(9, N=20, m=2, layer=layer, dims=(3, 2, 2))
    o = O.Oracle(ip, ix, part, 2, [3, 2, 2], layer, X, y)
    o.set_keep(0.5, [np.arange(len(o.list(O.B_LIST, r))) % 2 for r in range(2)])
    _, _, G = o.epoch([w.copy() for w in Ws], 0.0)
    h = 1e-6
    for l in range(2):
        for idx in np.ndindex(Ws[l].shape):
            Wp = [w.copy() for w in Ws]
            Wm = [w.copy() for w in Ws]
            Wp[l][idx] += h
            Wm[l][idx] -= h
            fp = o.epoch(Wp, 0.0)[0]
            fm = o.epoch(Wm, 0.0)[0]
            fd = (fp - fm) / (2 * h)
            assert abs(fd - G[l][idx]) <= 1e-4 * max(1e-3, abs(fd)), (l, idx, fd, G[l][idx])


def test_p1_equals_unpartitioned():
    ip, ix, part, X, y, Ws = random_case(21, N=40, m=4, dims=(3, 4, 3))
    ref = O.Oracle(ip, ix, np.zeros(40, np.int32), 1, [3, 4, 3], 0, X, y)
    ref.sample(1.0, 0, 0)
    o = O.Oracle(ip, ix, part, 4, [3, 4, 3], 0, X, y)
    o.sample(1.0, 5, 0)
    Wa = [w.copy() for w in Ws]
    Wb = [w.copy() for w in Ws]
    for e in range(10):
        la = ref.epoch(Wa, 0.05)[0]
        lb = o.epoch(Wb, 0.05)[0]
        if e == 0:   # first epoch forward is bitwise: same global CSR summation order, c_u = 1.0 exactly
            assert np.array_equal(ref.tensor(O.T_H, 2), o.tensor(O.T_H, 2))
        assert abs(la - lb) <= 1e-9 * abs(la)


def test_zero_upstream_and_uniform_logits():
    ip, ix, part, X, y, Ws = random_case(30, m=2, dims=(3, 4))
    Ws = [np.zeros_like(Ws[0])]
    o = O.Oracle(ip, ix, part, 2, [3, 4], 0, X, y)
    o.sample(0.5, 1, 1)
    loss, acc, G = o.epoch([Ws[0].copy()], 0.0)
    assert abs(loss - math.log(4)) < 1e-15          # S:341 uniform logits -> ln C
    ntr = (y >= 0).sum()
    assert acc == ((y == 0).sum() / ntr)            # argmax of ties is class 0 (R22)
    y0 = np.full_like(y, -1)                         # empty train set: loss 0, grads 0, acc 0
    o2 = O.Oracle(ip, ix, part, 2, [3, 4], 0, X, y0)
    o2.sample(0.5, 1, 1)
    loss, acc, G = o2.epoch([np.ones((6, 4))], 0.0)
    assert loss == 0.0 and acc == 0.0 and not np.any(G[0])


def test_rows_exchanged_eq3():
    # Eq. 3 at p=1: rows exchanged per layer == Σ_i |B_i|
    ip, ix, part, X, y, Ws = random_case(40, N=50, m=4, dims=(3, 3, 2))
    o = O.Oracle(ip, ix, part, 4, [3, 3, 2], 0, X, y)
    o.sample(1.0, 0, 0)
    o.epoch([w.copy() for w in Ws], 0.0)
    total_B = sum(len(o.list(O.B_LIST, i)) for i in range(4))
    assert o.rows_sent(1) == total_B and o.rows_sent(2) == total_B
    o.sample(0.4, 3, 3)
    o.epoch([w.copy() for w in Ws], 0.0)
    assert o.rows_sent(1) == sum(len(o.list(O.U_LIST, i)) for i in range(4))


def test_unbiased_aggregate():
    # E over draws of z~ equals exact z: Monte Carlo mean within 4 standard errors
    ip, ix, part, X, y, Ws = random_case(50, N=30, m=3, dims=(2, 2))
    o1 = O.Oracle(ip, ix, part, 3, [2, 2], 0, X, y)
    o1.sample(1.0, 0, 0)
    o1.epoch([Ws[0].copy()], 0.0)
    z_exact = o1.tensor(O.T_Z, 1)
    T, p = 3000, 0.3
    acc = []
    for e in range(T):
        o1.sample(p, 99, e)
        o1.epoch([Ws[0].copy()], 0.0)
        acc.append(o1.tensor(O.T_Z, 1))
    a = np.array(acc)
    se = a.std(0) / np.sqrt(T) + 1e-12
    assert np.all(np.abs(a.mean(0) - z_exact) <= 4.5 * se + 1e-12)


# ---------------- f2: Adam and dropout (readings R38, R39) ----------------
def test_adam_matches_torch_optim():
    import torch
    ip, ix, part, X, y, Ws = random_case(71, N=30, m=3, dims=(3, 5, 4))
    o = O.Oracle(ip, ix, part, 3, [3, 5, 4], 0, X, y)
    o.set_training(optimizer=1, beta1=0.8, beta2=0.95, eps=1e-6)
    g_orc = O.Oracle(ip, ix, part, 3, [3, 5, 4], 0, X, y)       # SGD at lr=0: plain gradient at given weights
    o.sample(0.5, 3, 1)
    g_orc.sample(0.5, 3, 1)
    Wo = [w.copy() for w in Ws]
    Wt = [torch.tensor(w.copy(), requires_grad=False) for w in Ws]
    opt = torch.optim.Adam(Wt, lr=0.05, betas=(0.8, 0.95), eps=1e-6)
    for _ in range(4):
        o.epoch(Wo, 0.05)
        _, _, G = g_orc.epoch([w.numpy().copy() for w in Wt], 0.0)
        for w, g in zip(Wt, G):
            w.grad = torch.tensor(g)
        opt.step()
        for a, b in zip(Wo, Wt):
            np.testing.assert_allclose(a, b.numpy(), rtol=0, atol=1e-12)


def test_dropout_mask_definition_and_rate():
    ip, ix, part, X, y, Ws = random_case(72, N=40, m=2, dims=(8, 4))
    o = O.Oracle(ip, ix, part, 2, [8, 4], 0, X, y)
    r, seed = 0.3, 0xABCDEF0123
    o.set_training(dropout=r, dropout_seed=seed)
    o.sample(1.0, 1, 5)
    T = O.threshold(r)
    kept = 0
    for u in range(40):
        for c in range(8):
            for l in (1, 2):
                out = O.philox4x32_10([u, c >> 2, l, 5], [(seed & 0xFFFFFFFF) ^ 0xD809, seed >> 32])
                f = o.drop_factor(u, c, l)
                assert f == ((1.0 / (1.0 - r)) if out[c & 3] >= T else 0.0)
                kept += f > 0
    n = 40 * 8 * 2
    assert abs(kept / n - (1 - r)) < 4 * np.sqrt(r * (1 - r) / n)


@pytest.mark.parametrize("layer", [0, 1])
def test_dropout_dense_bruteforce(layer):
    ip, ix, part, X, y, Ws = random_case(73, N=24, m=3, layer=layer, dims=(3, 5, 4, 3))
    dims = [3, 5, 4, 3]
    o = O.Oracle(ip, ix, part, 3, dims, layer, X, y)
    o.set_training(dropout=0.4, dropout_seed=77)
    o.sample(0.5, 9, 4)
    kept = [set(int(u) for u in o.list(O.U_LIST, r)) for r in range(3)]
    masks = [np.array([[o.drop_factor(u, c, l + 1) for c in range(dims[l])] for u in range(24)]) for l in range(3)]
    ref = forward_backward(ip, ix, part, kept, 0.5, layer, X, y, Ws, masks=masks)
    loss, acc, G = o.epoch([w.copy() for w in Ws], 0.0)
    assert abs(loss - ref["loss"]) <= 1e-12 * max(1.0, abs(ref["loss"]))
    for l in range(1, 3):
        np.testing.assert_allclose(o.tensor(O.T_DH, l), ref["dH"][l], rtol=1e-10, atol=1e-13)
    for g, r in zip(G, ref["dW"]):
        np.testing.assert_allclose(g, r, rtol=1e-10, atol=1e-13)


def test_dropout_zero_is_identity_and_unbiased():
    ip, ix, part, X, y, Ws = random_case(74, N=30, m=2, dims=(3, 4))
    base = O.Oracle(ip, ix, part, 2, [3, 4], 0, X, y)
    base.sample(0.5, 1, 1)
    l0, _, g0 = base.epoch([w.copy() for w in Ws], 0.0)
    o = O.Oracle(ip, ix, part, 2, [3, 4], 0, X, y)
    o.set_training(dropout=0.0, dropout_seed=5)
    o.sample(0.5, 1, 1)
    l1, _, g1 = o.epoch([w.copy() for w in Ws], 0.0)
    assert l0 == l1 and all(np.array_equal(a, b) for a, b in zip(g0, g1))
    # E over epochs of the dropped-out aggregate equals the aggregate without dropout (p = 1 sampling)
    o.set_training(dropout=0.5, dropout_seed=6)
    base.sample(1.0, 0, 0)
    base.epoch([w.copy() for w in Ws], 0.0)
    z = base.tensor(O.T_Z, 1)
    acc = []
    for e in range(1500):
        o.sample(1.0, 0, e)
        o.epoch([w.copy() for w in Ws], 0.0)
        acc.append(o.tensor(O.T_Z, 1))
    a = np.array(acc)
    assert np.all(np.abs(a.mean(0) - z) <= 4.5 * a.std(0) / np.sqrt(len(acc)) + 1e-12)


# ---------------- f4: multi-label sigmoid BCE + F1-micro (Yelp; reading R44) ----------------
@pytest.mark.parametrize("layer", [0, 1])
@pytest.mark.parametrize("seed,m,p", [(81, 3, 0.5), (82, 1, 1.0), (83, 4, 0.2)])
def test_multilabel_bce_dense_bruteforce(layer, seed, m, p):
    dims = [3, 5, 6]
    ip, ix, part, X, y, Ws = random_case(seed, m=m, layer=layer, dims=tuple(dims))
    T = I.multilabels(len(ip) - 1, dims[-1], 0.3, seed=seed)
    o = O.Oracle(ip, ix, part, m, dims, layer, X, y)
    o.set_multilabel(T)
    o.sample(p, 77, seed)
    kept = [set(int(u) for u in o.list(O.U_LIST, r)) for r in range(m)]
    ref = forward_backward(ip, ix, part, kept, p, layer, X, y, Ws, targets=T)
    loss, acc, G = o.epoch([w.copy() for w in Ws], 0.0)
    assert abs(loss - ref["loss"]) <= 1e-12 * max(1.0, abs(ref["loss"]))
    assert abs(acc - ref["acc"]) <= 1e-12
    np.testing.assert_allclose(o.tensor(O.T_DH, 2), ref["dH"][2], rtol=1e-10, atol=1e-15)
    for g, r in zip(G, ref["dW"]):
        np.testing.assert_allclose(g, r, rtol=1e-10, atol=1e-15)


def test_multilabel_closed_forms():
    """zero logits: loss = ln 2 exactly, no positive prediction -> F1 = 0; CE mode restored by set_multilabel(None)"""
    dims = [3, 4, 5]
    ip, ix, part, X, y, Ws = random_case(84, m=2, dims=tuple(dims))
    T = I.multilabels(len(ip) - 1, dims[-1], 0.5, seed=3)
    o = O.Oracle(ip, ix, part, 2, dims, 0, X, y)
    o.set_multilabel(T)
    o.sample(0.5, 1, 1)
    Wz = [w.copy() for w in Ws]
    Wz[-1][...] = 0.0
    loss, acc, G = o.epoch(Wz, 0.0)
    assert abs(loss - math.log(2.0)) < 1e-15 and acc == 0.0
    o.set_multilabel(None)
    loss, acc, G = o.epoch([w.copy() for w in Wz], 0.0)
    assert abs(loss - math.log(dims[-1])) < 1e-12


# ---------------- f4: GAT layer (Table tab:gat; reading R45) ----------------
@pytest.mark.parametrize("seed,m,p", [(91, 3, 0.5), (92, 1, 1.0), (93, 4, 0.0), (94, 2, 0.3)])
def test_gat_dense_bruteforce(seed, m, p):
    from dense_ref import gat_forward_backward
    dims = [3, 5, 4, 3]
    ip, ix, part, X, y, _ = random_case(seed, m=m, layer=1, dims=tuple(dims))
    rng = np.random.default_rng(seed)
    Ws = [rng.uniform(-1, 1, (dims[l] + 2, dims[l + 1])) for l in range(3)]
    o = O.Oracle(ip, ix, part, m, dims, 2, X, y)
    o.sample(p, 77, seed)
    kept = [set(int(u) for u in o.list(O.U_LIST, r)) for r in range(m)]
    ref = gat_forward_backward(ip, ix, part, kept, X, y, Ws)
    loss, acc, G = o.epoch([w.copy() for w in Ws], 0.0)
    assert abs(loss - ref["loss"]) <= 1e-12 * max(1.0, abs(ref["loss"]))
    for l in range(1, 4):
        np.testing.assert_allclose(o.tensor(O.T_H, l), ref["H"][l], rtol=1e-11, atol=1e-12)
    for l in range(1, 3):
        np.testing.assert_allclose(o.tensor(O.T_DH, l), ref["dH"][l], rtol=1e-9, atol=1e-13)
    for g, r in zip(G, ref["dW"]):
        np.testing.assert_allclose(g, r, rtol=1e-9, atol=1e-13)


def test_gat_single_neighbour_closed_form():
    """a node whose only sampled neighbour is itself gets alpha_vv = 1: pre_v = x_v W (p = 0, isolated partitions)"""
    dims = [3, 2]
    ip, ix, part, X, y, _ = random_case(95, m=3, layer=1, dims=tuple(dims))
    W = [np.random.default_rng(1).uniform(-1, 1, (5, 2))]
    o = O.Oracle(ip, ix, part, 3, dims, 2, X, y)
    o.sample(0.0, 1, 1)
    o.epoch([W[0].copy()], 0.0)
    H1 = o.tensor(O.T_H, 1)
    alone = [v for v in range(len(ip) - 1) if np.all(part[ix[ip[v]:ip[v + 1]]] != part[v])]
    assert len(alone) >= 3
    for v in alone:
        np.testing.assert_allclose(H1[v], X[v].astype(np.float64) @ W[0][:3], rtol=1e-12, atol=1e-14)
