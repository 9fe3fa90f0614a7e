"""GPU parity: libbns.so (sm_100a kernels, through the C ABI) against the oracle, element by element.

Bar (BASELINE.json north_star): sampling masks, compacted index lists, send/recv maps and the induced subgraph
bit-exact; per-layer activations and gradients within 1e-5 (fp32) / 2e-2 (bf16) normwise relative error
(SURVEY.md §8(c) item 20); loss within 1e-3 relative.  Multi-partition runs use the LOCAL transport (m contexts
on one GPU, one host thread each) -- the same pack / exchange / scatter-add / all-reduce code path as NCCL except
the copy engine that moves the rows.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2203_10983_b200 import bns
from paper_2203_10983_b200 import inputs as I

from gpu_harness import GpuRun, LOSS_TOL, TOL, compare_epoch, parallel, relerr, relu_flips

pytestmark = pytest.mark.gpu
SEED = I.BNS_SEED


def wl(N, nnz, m, d0, C, seed, method="random", train=0.7):
    indptr, indices = I.rmat(N, nnz, seed=seed)
    part = I.partition(indptr, indices, m, method)
    X = I.features(np.arange(N, dtype=np.int32), d0)
    y = I.labels(N, C, train, seed=seed + 7)
    return indptr, indices, part, X, y


@pytest.mark.parametrize("N,nnz,m,method", [(2000, 40000, 2, "random"), (3000, 60000, 5, "ldg2"),
                                            (1000, 8000, 3, "random"), (500, 3000, 8, "ldg2")])
def test_sampling_lists_bitexact(N, nnz, m, method):
    indptr, indices, part, X, y = wl(N, nnz, m, 4, 3, 11, method)
    run = GpuRun(indptr, indices, part, m, [4, 3], 0, bns.BNS_FP32, X, y, flags=bns.BNS_DEBUG_EXCHANGE_INDICES)
    orc = O.Oracle(indptr, indices, part, m, [1, 1], 0, np.zeros((N, 1), np.float32), np.zeros(N, np.int32))
    try:
        for p in (0.0, 0.1, 0.5, 1.0):
            for e in (0, 1, (1 << 32) + 3):
                run.sample(p, SEED, e)
                orc.sample(p, SEED, e)
                for r in range(m):
                    c = run.ctx[r]
                    assert np.array_equal(c.mask(), orc.list(O.KEEP, r).astype(np.uint8))
                    U = c.i32(bns.BNS_Q_HALO)
                    assert np.array_equal(U, orc.list(O.U_LIST, r))
                    assert np.array_equal(c.i64(bns.BNS_Q_HALO_OFF), orc.list(O.U_OFF, r))
                    S = c.i32(bns.BNS_Q_SEND)
                    So = c.i64(bns.BNS_Q_SEND_OFF)
                    for j in range(m):
                        assert np.array_equal(S[So[j]:So[j + 1]], orc.list(O.S_LIST, r, j)), (p, e, r, j)
                    # induced subgraph (Alg.1 l.5): kept columns in global neighbour order, halo -> n_in + slot
                    V = c.i32(bns.BNS_Q_INNER)
                    local = {int(v): k for k, v in enumerate(V)}
                    slot = {int(u): s for s, u in enumerate(U)}
                    ptr, col = c.induced(len(V))
                    for k in range(0, len(V), max(1, len(V) // 200)):
                        v = V[k]
                        exp = [local[u] if u in local else len(V) + slot[u]
                               for u in map(int, indices[indptr[v]:indptr[v + 1]]) if u in local or u in slot]
                        assert list(col[ptr[k]:ptr[k + 1]]) == exp
    finally:
        run.close()


CASES = [  # (m, p, method)
    (1, 1.0, "random"), (2, 0.5, "random"), (4, 0.1, "ldg2"), (3, 0.0, "random"), (3, 1.0, "ldg2"), (5, 0.3, "random"),
]


@pytest.mark.parametrize("prec", [bns.BNS_FP32, bns.BNS_BF16])
@pytest.mark.parametrize("layer,tf", [(bns.BNS_LAYER_SAGE_MEAN, True), (bns.BNS_LAYER_SAGE_MEAN, False),
                                      (bns.BNS_LAYER_GCN, False)])
@pytest.mark.parametrize("m,p,method", CASES)
def test_epoch_parity(prec, layer, tf, m, p, method):
    # SAGE: [37, 24, 16, 5] runs every layer transform-first (R42); BNS_NO_TRANSFORM_FIRST keeps aggregate-first
    dims = [37, 24, 16, 5] if layer == bns.BNS_LAYER_SAGE_MEAN else [37, 16, 5]
    N, nnz = 3000, 90000                       # R-MAT: hub rows > kSeg exercise the split-row fixup
    indptr, indices, part, X, y = wl(N, nnz, m, dims[0], dims[-1], 21 + m, method)
    L = len(dims) - 1
    Ws = I.weights(dims, layer)
    Wd = [w.astype(np.float64) for w in Ws]
    flags = bns.BNS_RETAIN_GRADS | (0 if tf else bns.BNS_NO_TRANSFORM_FIRST)
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y, flags=flags)
    orc = O.Oracle(indptr, indices, part, m, dims, layer, X, y)
    try:
        for e in range(2):
            run.sample(p, SEED, e)
            orc.sample(p, SEED, e)
            Ws = compare_epoch(run, orc, L, Ws, Wd, 0.5, prec, tag=f"epoch{e}")
    finally:
        run.close()


@pytest.mark.parametrize("dims,prec", [([37, 64, 41], bns.BNS_BF16), ([37, 64, 24], bns.BNS_FP32),
                                       ([37, 64, 41], bns.BNS_FP32)])
@pytest.mark.parametrize("m,p", [(1, 1.0), (3, 0.3)])
def test_six_vector_rows_parity(dims, prec, m, p):
    """Transform-first last layer gathered at a width of 6 16-byte vectors (48 bf16 = Reddit's 41 classes padded;
    24 fp32): the SpMM's 2-lanes x 3-vectors layout, forward and transposed, against the oracle."""
    layer = bns.BNS_LAYER_SAGE_MEAN
    L = len(dims) - 1
    indptr, indices, part, X, y = wl(3000, 90000, m, dims[0], dims[-1], 91 + m)
    Ws = I.weights(dims, layer)
    Wd = [w.astype(np.float64) for w in Ws]
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y)
    orc = O.Oracle(indptr, indices, part, m, dims, layer, X, y)
    try:
        for e in range(2):
            run.sample(p, SEED, e)
            orc.sample(p, SEED, e)
            Ws = compare_epoch(run, orc, L, Ws, Wd, 0.5, prec, tag=f"six-vector epoch{e}")
    finally:
        run.close()


@pytest.mark.parametrize("prec", [bns.BNS_FP32, bns.BNS_BF16])
@pytest.mark.parametrize("m,p", [(1, 1.0), (3, 0.5)])
def test_long_row_segments_parity(prec, m, p, monkeypatch):
    """R37 long-row segments (rows above 2048 kept edges split into 1024-edge segments; the default only for jobs with
    >= 38 M arcs per partition) forced on a small dense graph: forward / transposed segment builders, the split-row
    fixup and the static p = 1 segments against the oracle."""
    monkeypatch.setenv("BNS_SEG_LONG", "1024")
    dims, layer = [37, 24, 16, 5], bns.BNS_LAYER_SAGE_MEAN
    L = len(dims) - 1
    indptr, indices, part, X, y = wl(20000, 1500000, m, dims[0], dims[-1], 101 + m)
    assert (np.diff(indptr) > 4096).sum() >= 2   # long rows of several 1024-edge segments
    Ws = I.weights(dims, layer)
    Wd = [w.astype(np.float64) for w in Ws]
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y)
    orc = O.Oracle(indptr, indices, part, m, dims, layer, X, y)
    try:
        for e in range(2):
            run.sample(p, SEED, e)
            orc.sample(p, SEED, e)
            Ws = compare_epoch(run, orc, L, Ws, Wd, 0.5, prec, tag=f"long-seg epoch{e}")
    finally:
        run.close()


@pytest.mark.parametrize("tf", [False, True])
@pytest.mark.parametrize("m,p", [(1, 1.0), (3, 0.4)])
def test_merged_wgrad_parity(tf, m, p):
    """Aggregate-first GraphSAGE layers with d_in % 128 == 0 compute dW_z and dW_h in ONE tcgen05 launch (two A
    operands split by output row) + one split-K reduce: gradients against the oracle (bf16, 2e-2)."""
    dims, layer, prec = [37, 128, 128, 5], bns.BNS_LAYER_SAGE_MEAN, bns.BNS_BF16
    L = len(dims) - 1
    indptr, indices, part, X, y = wl(3000, 90000, m, dims[0], dims[-1], 111 + m)
    Ws = I.weights(dims, layer)
    Wd = [w.astype(np.float64) for w in Ws]
    flags = bns.BNS_RETAIN_GRADS | (0 if tf else bns.BNS_NO_TRANSFORM_FIRST)
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y, flags=flags)
    orc = O.Oracle(indptr, indices, part, m, dims, layer, X, y)
    try:
        for e in range(2):
            run.sample(p, SEED, e)
            orc.sample(p, SEED, e)
            Ws = compare_epoch(run, orc, L, Ws, Wd, 0.5, prec, tag=f"merged-wgrad epoch{e}")
    finally:
        run.close()


def test_cora_config0():
    """BASELINE.json configs[0]: Cora-shaped, 2-layer GCN hidden 16, 2 partitions, p=0.5, fixed Philox seed."""
    sh = I.SHAPES["cora"]
    indptr, indices = I.rmat(sh.N, sh.nnz)
    part = I.partition(indptr, indices, 2)
    X = I.features(np.arange(sh.N, dtype=np.int32), sh.d0)
    y = I.labels(sh.N, sh.C, sh.train_frac)
    Ws = I.weights(sh.dims, sh.layer)
    Wd = [w.astype(np.float64) for w in Ws]
    for prec in (bns.BNS_FP32, bns.BNS_BF16):
        run = GpuRun(indptr, indices, part, 2, sh.dims, sh.layer, prec, X, y)
        orc = O.Oracle(indptr, indices, part, 2, sh.dims, sh.layer, X, y)
        Wp, Wdp = [w.copy() for w in Ws], [w.copy() for w in Wd]
        try:
            for e in range(3):
                run.sample(0.5, SEED, e)
                orc.sample(0.5, SEED, e)
                Wp = compare_epoch(run, orc, sh.L, Wp, Wdp, 0.1, prec, tag=f"cora prec{prec} e{e}")
        finally:
            run.close()


def find_epoch_for_draw():
    """first epoch whose Philox draw at p=0.5 gives U_0 = {2}, U_1 = {} on the P4 golden graph"""
    T = O.threshold(0.5)
    for e in range(1000):
        if O.draw(2, 0, e, SEED) < T and O.draw(1, 1, e, SEED) >= T:
            return e
    raise AssertionError


@pytest.mark.parametrize("name", ["E1", "E2", "E3", "E4", "E5", "E6"])
def test_goldens_on_gpu(name):
    G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "p4_goldens.json")))
    c = G["cases"][name]
    g = G["graph"]
    layer = 0 if c["layer"] == "sage" else 1
    Ws = [np.array(w, np.float32) for w in G[c["W"]]]
    dims = [1] + [w.shape[1] for w in Ws]
    indptr, indices = I.csr_from_edges(4, g["edges"])
    X = np.array(g["X"], np.float32)
    y = np.array(g["labels"], np.int32)
    run = GpuRun(indptr, indices, np.array(g["part_of"], np.int32), 2, dims, layer, bns.BNS_FP32, X, y)
    try:
        e = find_epoch_for_draw() if "draw" in c else 0
        run.sample(c["p"], SEED, e)
        assert list(run.ctx[0].i32(bns.BNS_Q_HALO)) == ([2] if c["p"] > 0 else [])
        loss, acc, Gr, _ = run.epoch(Ws, 0.0)
        assert abs(loss - c["loss"]) < 1e-6
        assert acc == c["acc"]
        for l, gd in enumerate(c.get("dW", [])):
            np.testing.assert_allclose(Gr[l], gd, atol=1e-6)
        if "logits" in c:
            np.testing.assert_allclose(run.gather(bns.BNS_Q_H, len(Ws), 2), c["logits"], atol=1e-6)
    finally:
        run.close()


def test_host_pointer_weights_equal_device_path():
    indptr, indices, part, X, y = wl(1500, 30000, 2, 16, 4, 5)
    dims = [16, 8, 4]
    Ws = I.weights(dims, 0)
    run = GpuRun(indptr, indices, part, 2, dims, 0, bns.BNS_FP32, X, y)
    try:
        run.sample(0.4, SEED, 7)
        a = run.epoch(Ws, 0.3, host=False)
        b = run.epoch(Ws, 0.3, host=True)
        assert a[0] == b[0] and a[1] == b[1]
        for x, z in zip(a[2] + a[3], b[2] + b[3]):
            assert np.array_equal(x, z)
    finally:
        run.close()


def test_determinism_two_runs():
    indptr, indices, part, X, y = wl(2500, 70000, 3, 20, 6, 8)
    dims = [20, 16, 6]
    outs = []
    for _ in range(2):
        run = GpuRun(indptr, indices, part, 3, dims, 0, bns.BNS_BF16, X, y)
        Ws = I.weights(dims, 0)
        try:
            rec = []
            for e in range(3):
                run.sample(0.3, SEED, e)
                loss, acc, G, Ws = run.epoch(Ws, 0.2)
                rec.append((loss, acc, [g.tobytes() for g in G], run.ctx[1].mask().tobytes()))
            outs.append((rec, [w.tobytes() for w in Ws]))
        finally:
            run.close()
    assert outs[0] == outs[1]


@pytest.mark.parametrize("m", [1, 3])
def test_step_equals_sample_then_epoch(m):
    """bns_step(p, seed, epoch, W, lr, G) is bns_sample_boundary + bns_epoch in one call: bitwise the same."""
    import torch
    indptr, indices, part, X, y = wl(2500, 70000, m, 20, 6, 18)
    dims = [20, 16, 6]
    outs = []
    for fused in (False, True):
        run = GpuRun(indptr, indices, part, m, dims, 0, bns.BNS_BF16, X, y)
        Ws = I.weights(dims, 0)
        W = [[torch.tensor(w, device="cuda") for w in Ws] for _ in range(m)]
        G = [[torch.zeros_like(w) for w in W[0]] for _ in range(m)]
        try:
            rec = []
            for e in range(3):
                if fused:
                    out = parallel(m, lambda r: run.ctx[r].step(0.3, SEED, e, W[r], 0.2, G[r]))
                else:
                    run.sample(0.3, SEED, e)
                    out = parallel(m, lambda r: run.ctx[r].epoch(W[r], 0.2, G[r]))
                torch.cuda.synchronize()
                rec.append((out[0], [g.cpu().numpy().tobytes() for g in G[0]], run.ctx[0].mask().tobytes()))
            outs.append((rec, [w.cpu().numpy().tobytes() for w in W[0]]))
        finally:
            run.close()
    assert outs[0] == outs[1]


def test_set_timing_toggles_phase_events():
    indptr, indices, part, X, y = wl(1500, 30000, 1, 20, 6, 28)
    dims = [20, 16, 6]
    run = GpuRun(indptr, indices, part, 1, dims, 0, bns.BNS_FP32, X, y, flags=bns.BNS_TIMING)
    Ws = I.weights(dims, 0)
    try:
        c = run.ctx[0]
        run.sample(0.5, SEED, 0)
        run.epoch(Ws, 0.1)
        t0 = c.times()
        assert t0["epoch_total"] > 0
        c.set_timing(False)
        run.sample(0.5, SEED, 1)
        run.epoch(Ws, 0.1)
        assert c.times() == t0
        c.set_timing(True)
        run.sample(0.5, SEED, 2)
        run.epoch(Ws, 0.1)
        assert c.times()["epoch_total"] > t0["epoch_total"]
    finally:
        run.close()
    run = GpuRun(indptr, indices, part, 1, dims, 0, bns.BNS_FP32, X, y, flags=0)
    try:
        with pytest.raises(bns.BnsError) as e:
            run.ctx[0].set_timing(True)
        assert e.value.code == bns.BNS_ERR_STATE
    finally:
        run.close()


def test_binomial_counts_gpu():
    indptr, indices, part, X, y = wl(3000, 60000, 4, 4, 3, 3)
    run = GpuRun(indptr, indices, part, 4, [4, 3], 0, bns.BNS_FP32, X, y, flags=0)
    try:
        p, E = 0.1, 400
        nB = [run.ctx[r].counts()["n_bd"] for r in range(4)]
        cnt = np.zeros((E, 4))
        for e in range(E):
            run.sample(p, 99, e)
            for r in range(4):
                cnt[e, r] = run.ctx[r].counts()["n_halo"]
        pp = O.threshold(p) / 2**32
        for r in range(4):
            mu, sd = nB[r] * pp, np.sqrt(nB[r] * pp * (1 - pp))
            assert abs(cnt[:, r].mean() - mu) < 4 * sd / np.sqrt(E)
            assert abs(cnt[:, r].std() - sd) < 0.15 * sd
    finally:
        run.close()


def test_nonfinite_loss_leaves_weights():
    indptr, indices, part, X, y = wl(800, 8000, 2, 8, 3, 4)
    dims = [8, 3]
    Ws = I.weights(dims, 0)
    Ws[0][0, 0] = np.inf
    run = GpuRun(indptr, indices, part, 2, dims, 0, bns.BNS_FP32, X, y)
    try:
        run.sample(1.0, SEED, 0)
        with pytest.raises(bns.BnsError) as e:
            run.epoch(Ws, 0.1)
        assert e.value.code == bns.BNS_ERR_NONFINITE
    finally:
        run.close()


def test_skipped_adam_step_is_not_counted():
    """A non-finite loss skips the Adam update (moments untouched); the step count must not advance either, so the
    next finite epoch applies the bias corrections of step 1 -- bitwise the same as a run without the failed epoch."""
    import torch
    indptr, indices, part, X, y = wl(800, 8000, 1, 8, 3, 4)
    dims = [8, 6, 3]
    outs = []
    for fail_first in (False, True):
        run = GpuRun(indptr, indices, part, 1, dims, 0, bns.BNS_FP32, X, y)
        run.ctx[0].set_training(bns.BNS_OPT_ADAM, 0.9, 0.999, 1e-8, 0.0, 1)
        try:
            run.sample(1.0, SEED, 0)
            if fail_first:
                Wbad = [torch.tensor(w, device="cuda") for w in I.weights(dims, 0)]
                Wbad[0][0, 0] = float("inf")
                with pytest.raises(bns.BnsError) as e:
                    run.ctx[0].epoch(Wbad, 0.01)
                assert e.value.code == bns.BNS_ERR_NONFINITE
            W = [torch.tensor(w, device="cuda") for w in I.weights(dims, 0)]
            run.ctx[0].epoch(W, 0.01)
            torch.cuda.synchronize()
            outs.append([w.cpu().numpy().tobytes() for w in W])
        finally:
            run.close()
    assert outs[0] == outs[1]


def test_epoch_before_sample_is_state_error():
    indptr, indices, part, X, y = wl(300, 2000, 1, 8, 3, 4)
    run = GpuRun(indptr, indices, part, 1, [8, 3], 0, bns.BNS_FP32, X, y)
    try:
        with pytest.raises(bns.BnsError) as e:
            run.epoch(I.weights([8, 3], 0), 0.1)
        assert e.value.code == bns.BNS_ERR_STATE
        with pytest.raises(bns.BnsError) as e:
            run.ctx[0].sample_boundary(1.5, 1, 0)
        assert e.value.code == bns.BNS_ERR_INVALID
    finally:
        run.close()


def test_nccl_transport_world1_matches_none():
    """The NCCL transport (communicator init, grouped send/recv skipping self, ncclAllReduce of the gradient and
    loss scalars) at world = 1 gives the same bits as no transport (a 1-GPU box cannot host 2 NCCL ranks)."""
    indptr, indices, part, X, y = wl(2000, 40000, 1, 24, 5, 12)
    dims = [24, 16, 5]
    outs = []
    for transport in (bns.BNS_TRANSPORT_NONE, bns.BNS_TRANSPORT_NCCL):
        nid = bns.bns_get_unique_id() if transport == bns.BNS_TRANSPORT_NCCL else None
        c = bns.Context(rank=0, world=1, dims=dims, layer=0, precision=bns.BNS_BF16, indptr=indptr, indices=indices,
                        part_of=part, features=X, labels=y, transport=transport, nccl_id=nid)
        Ws = [w.copy() for w in I.weights(dims, 0)]
        G = [np.zeros_like(w) for w in Ws]
        c.sample_boundary(0.3, SEED, 1)
        loss, acc = c.epoch(Ws, 0.1, G)
        outs.append((loss, acc, [w.tobytes() for w in Ws], [g.tobytes() for g in G]))
        c.close()
    assert outs[0] == outs[1]


# ---------------- f2: Adam + dropout, the paper's recipe ----------------
@pytest.mark.parametrize("prec", [bns.BNS_FP32, bns.BNS_BF16])
@pytest.mark.parametrize("layer", [bns.BNS_LAYER_SAGE_MEAN, bns.BNS_LAYER_GCN])
@pytest.mark.parametrize("m,p,drop", [(1, 1.0, 0.5), (3, 0.5, 0.3)])
def test_adam_dropout_parity(prec, layer, m, p, drop):
    dims = [37, 24, 16, 5] if layer == bns.BNS_LAYER_SAGE_MEAN else [37, 16, 5]
    indptr, indices, part, X, y = wl(3000, 90000, m, dims[0], dims[-1], 31 + m)
    L = len(dims) - 1
    Ws = I.weights(dims, layer)
    Wd = [w.astype(np.float64) for w in Ws]
    lr, seed = 0.01, 0xD0D0
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y)
    for c in run.ctx:
        c.set_training(bns.BNS_OPT_ADAM, 0.9, 0.999, 1e-8, drop, seed)
    orc = O.Oracle(indptr, indices, part, m, dims, layer, X, y)
    orc.set_training(optimizer=1, beta1=0.9, beta2=0.999, eps=1e-8, dropout=drop, dropout_seed=seed)
    tol = TOL[prec]
    # Adam normalises each step to ~lr, so a gradient entry within its rounding error of zero can take a step of
    # either sign: weights are compared on the scale of the steps (all within 2 lr per step, and almost all
    # entries within 0.1 lr).  In bf16 those weight differences then move the next forward beyond the bf16
    # tolerance, so bf16 is compared over one epoch and fp32 over three.
    try:
        for e in range(3 if prec == bns.BNS_FP32 else 1):
            run.sample(p, SEED, e)
            orc.sample(p, SEED, e)
            loss, acc, G, Wn = run.epoch(Ws, lr)
            lo, ao, Go = orc.epoch(Wd, lr)
            assert abs(loss - lo) <= LOSS_TOL * abs(lo), (e, loss, lo)
            F = relu_flips(run, orc, L, prec, f"adam{e}")[0]
            for l in range(1, L + 1):
                if not (run.tf >> (l - 1)) & 1:
                    assert relerr(run.gather(bns.BNS_Q_Z, l, dims[l - 1]), orc.tensor(O.T_Z, l)) <= tol, ("Z", e, l)
                if l >= F:
                    assert relerr(run.gather(bns.BNS_Q_DH, l, dims[l]), orc.tensor(O.T_DH, l)) <= tol, ("dH", e, l)
            for l in range(L):
                if l + 1 <= F:
                    continue
                assert relerr(G[l], Go[l]) <= tol, ("dW", e, l)
                dw = np.abs(Wn[l] - Wd[l])
                assert dw.max() <= 2.01 * lr * (e + 1), ("W", e, l, dw.max())
                assert np.mean(dw > 0.1 * lr) < 0.01, ("W", e, l, np.mean(dw > 0.1 * lr))
            Ws = [w.astype(np.float32) for w in Wn]
    finally:
        run.close()


def test_dropout_masks_change_per_epoch_and_zero_rate_is_identity():
    indptr, indices, part, X, y = wl(1500, 30000, 2, 16, 4, 13)
    dims = [16, 8, 4]
    outs = []
    for drop in (0.0, 0.0, 0.4):
        run = GpuRun(indptr, indices, part, 2, dims, 0, bns.BNS_FP32, X, y)
        if drop or len(outs) == 1:
            for c in run.ctx:
                c.set_training(bns.BNS_OPT_SGD, 0.9, 0.999, 1e-8, drop, 3)
        try:
            run.sample(0.5, SEED, 1)
            outs.append(run.epoch(I.weights(dims, 0), 0.1)[:3])
        finally:
            run.close()
    assert outs[0][0] == outs[1][0] and all(np.array_equal(a, b) for a, b in zip(outs[0][2], outs[1][2]))
    assert outs[2][0] != outs[0][0]


# ---------------- f1 / R43: boundary-feature (X^(0)) cache ----------------
@pytest.mark.parametrize("prec", [bns.BNS_FP32, bns.BNS_BF16])
@pytest.mark.parametrize("layer", [bns.BNS_LAYER_SAGE_MEAN, bns.BNS_LAYER_GCN])
def test_input_halo_cache_is_bit_identical(prec, layer):
    """BNS_CACHE_INPUT_HALO replaces the layer-1 pack + exchange by a local gather from rows exchanged once at setup:
    every output must be bitwise the same as the literal per-epoch exchange (R28), across BNS and edge draws."""
    m = 3
    dims = [37, 24, 16, 5] if layer == bns.BNS_LAYER_SAGE_MEAN else [37, 16, 5]
    indptr, indices, part, X, y = wl(2500, 60000, m, dims[0], dims[-1], 17)
    Ws = I.weights(dims, layer)
    outs = []
    for flags in (bns.BNS_RETAIN_GRADS, bns.BNS_RETAIN_GRADS | bns.BNS_CACHE_INPUT_HALO):
        run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y, flags=flags)
        W = [w.copy() for w in Ws]
        rec = []
        try:
            for e in range(3):
                if e == 2:
                    parallel(m, lambda r: run.ctx[r].sample_edges(bns.BNS_SAMPLER_BES, 0.3, SEED, 2))
                else:
                    run.sample(0.3 if e == 0 else 1.0, SEED, e)
                loss, acc, G, W = run.epoch(W, 0.3)
                W = [w.astype(np.float32) for w in W]
                rec.append((loss, acc, [g.copy() for g in G],
                            [run.gather(bns.BNS_Q_H, l, dims[l]) for l in range(1, len(dims))],
                            [run.gather(bns.BNS_Q_DH, l, dims[l]) for l in range(1, len(dims))]))
        finally:
            run.close()
        outs.append(rec)
    for a, b in zip(outs[0], outs[1]):
        assert a[0] == b[0] and a[1] == b[1]
        for x, z in zip(a[2] + a[3] + a[4], b[2] + b[3] + b[4]):
            assert np.array_equal(x, z)


# ---------------- f4: multi-label sigmoid BCE + F1-micro (Yelp; R44) ----------------
@pytest.mark.parametrize("prec", [bns.BNS_FP32, bns.BNS_BF16])
@pytest.mark.parametrize("layer", [bns.BNS_LAYER_SAGE_MEAN, bns.BNS_LAYER_GCN])
@pytest.mark.parametrize("m,p", [(1, 1.0), (3, 0.3)])
def test_multilabel_parity(prec, layer, m, p):
    dims = [37, 24, 16, 12] if layer == bns.BNS_LAYER_SAGE_MEAN else [37, 16, 12]
    indptr, indices, part, X, y = wl(3000, 90000, m, dims[0], dims[-1], 51 + m)
    N, L = len(indptr) - 1, len(dims) - 1
    T = I.multilabels(N, dims[-1], 0.2, seed=7)
    Ws = I.weights(dims, layer)
    Wd = [w.astype(np.float64) for w in Ws]
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y)
    for r, c in enumerate(run.ctx):
        c.set_multilabel(T[run.inner[r]])
    orc = O.Oracle(indptr, indices, part, m, dims, layer, X, y)
    orc.set_multilabel(T)
    tol = TOL[prec]
    try:
        for e in range(2 if prec == bns.BNS_FP32 else 1):
            run.sample(p, SEED, e)
            orc.sample(p, SEED, e)
            loss, f1, G, Wn = run.epoch(Ws, 0.5)
            lo, fo, Go = orc.epoch(Wd, 0.5)
            assert abs(loss - lo) <= LOSS_TOL * abs(lo), (e, loss, lo)
            assert abs(f1 - fo) <= (1e-3 if prec == bns.BNS_FP32 else 2e-2), (e, f1, fo)
            F = relu_flips(run, orc, L, prec, f"bce{e}")[0]
            assert relerr(run.gather(bns.BNS_Q_DH, L, dims[L]), orc.tensor(O.T_DH, L)) <= tol
            for l in range(L):
                if l + 1 > F:
                    assert relerr(G[l], Go[l]) <= tol, ("dW", e, l)
            Ws = [w.astype(np.float32) for w in Wn]
    finally:
        run.close()


def test_multilabel_rejects_non_binary_targets():
    indptr, indices, part, X, y = wl(300, 2000, 1, 4, 3, 3)
    run = GpuRun(indptr, indices, part, 1, [4, 3], 0, bns.BNS_FP32, X, y)
    try:
        with pytest.raises(bns.BnsError) as ei:
            run.ctx[0].set_multilabel(np.full((len(indptr) - 1, 3), 2, np.uint8))
        assert ei.value.code == bns.BNS_ERR_INVALID
    finally:
        run.close()


# ---------------- f4: GAT (Table tab:gat; R45) ----------------
@pytest.mark.parametrize("prec", [bns.BNS_FP32, bns.BNS_BF16])
@pytest.mark.parametrize("m,p,sampler", [(1, 1.0, 0), (3, 0.3, 0), (4, 0.1, 0), (3, 0.0, 0), (3, 0.4, 1), (2, 0.5, 2)])
def test_gat_parity(prec, m, p, sampler):
    layer = bns.BNS_LAYER_GAT
    dims = [37, 24, 16, 5]
    L = len(dims) - 1
    indptr, indices, part, X, y = wl(3000, 90000, m, dims[0], dims[-1], 61 + m)   # hub rows: split segments
    Ws = I.weights(dims, layer)
    assert Ws[0].shape == (dims[0] + 2, dims[1])
    Wd = [w.astype(np.float64) for w in Ws]
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y)
    orc = O.Oracle(indptr, indices, part, m, dims, layer, X, y)
    try:
        for e in range(2 if prec == bns.BNS_FP32 else 1):
            if sampler:
                run.sample_edges(sampler, p, SEED, e)
                orc.sample_edges(sampler, p, SEED, e)
            else:
                run.sample(p, SEED, e)
                orc.sample(p, SEED, e)
            Ws = compare_epoch(run, orc, L, Ws, Wd, 0.5, prec, tag=f"gat epoch{e}")
    finally:
        run.close()
