"""the exchange steps fused with their producer / consumer over peer memory (BNS_PEER_MEMORY with the
in-process LOCAL group; BNS_TRANSPORT_IPC across processes).

Pins:
  * bitwise equality with the staged LOCAL transport (pack + device copies + scatter-add + rank-order sum), which the
    oracle parity tests already hold to the north-star tolerances -- the fused path moves the same rows and adds
    them in the same order (R25), so nothing may change by one bit;
  * oracle parity of the fused path itself (fp32 1e-5, bf16 2e-2, loss 1e-3);
  * two processes sharing cuda:0 through CUDA IPC mappings (the multi-process code path on a one-GPU box);
  * a rank that never arrives makes the device barrier time out into BNS_ERR_RUNTIME instead of hanging the GPU.
"""
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np
import pytest

from oracle import oracle as O
from paper_2203_10983_b200 import bns
from paper_2203_10983_b200 import inputs as I

from gpu_harness import GpuRun, parallel
from gpu_harness import compare_epoch
from test_gpu_parity import wl

pytestmark = pytest.mark.gpu
SEED = I.BNS_SEED
HERE = os.path.dirname(os.path.abspath(__file__))


def record(run, dims, Ws, draws, lr=0.3, train=None):
    """Run the draws [(kind, p), ...] epoch after epoch; return loss / acc / grads / H / dH per epoch."""
    m = run.m
    W = [w.copy() for w in Ws]
    rec = []
    if train:
        parallel(m, lambda r: run.ctx[r].set_training(**train))
    for e, (kind, p) in enumerate(draws):
        if kind == "bns":
            run.sample(p, SEED, e)
        else:
            parallel(m, lambda r: run.ctx[r].sample_edges(kind, p, SEED, e))
        loss, acc, G, W = run.epoch(W, lr)
        W = [w.astype(np.float32) for w in W]
        rec.append((loss, acc, [g.copy() for g in G], [w.copy() for w in W],
                    [run.gather(bns.BNS_Q_H, l, dims[l]) for l in range(1, len(dims))],
                    [run.gather(bns.BNS_Q_DH, l, dims[l]) for l in range(1, len(dims))]))
    return rec


def assert_same(a_rec, b_rec):
    for e, (a, b) in enumerate(zip(a_rec, b_rec)):
        assert a[0] == b[0] and a[1] == b[1], (e, a[0], b[0])
        for x, z in zip(a[2] + a[3] + a[4] + a[5], b[2] + b[3] + b[4] + b[5]):
            assert np.array_equal(x, z), e


DRAWS = [("bns", 0.3), ("bns", 1.0), (bns.BNS_SAMPLER_BES, 0.4), ("bns", 0.0), ("bns", 0.1)]


@pytest.mark.parametrize("prec", [bns.BNS_FP32, bns.BNS_BF16])
@pytest.mark.parametrize("layer", [bns.BNS_LAYER_SAGE_MEAN, bns.BNS_LAYER_GCN, bns.BNS_LAYER_GAT])
@pytest.mark.parametrize("m,extra", [(2, 0), (4, bns.BNS_CACHE_INPUT_HALO), (5, 0)])
def test_peer_memory_bit_identical_to_staged(prec, layer, m, extra):
    dims = [37, 24, 16, 5] if layer != bns.BNS_LAYER_GCN else [37, 16, 5]
    indptr, indices, part, X, y = wl(2500, 70000, m, dims[0], dims[-1], 31 + m)
    Ws = I.weights(dims, layer)
    recs = []
    for peer in (0, bns.BNS_PEER_MEMORY):
        run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y,
                     flags=bns.BNS_RETAIN_GRADS | extra | peer)
        try:
            recs.append(record(run, dims, Ws, DRAWS))
        finally:
            run.close()
    assert_same(recs[0], recs[1])


def test_peer_memory_adam_dropout_bit_identical():
    m, dims, layer, prec = 3, [37, 24, 16, 5], bns.BNS_LAYER_SAGE_MEAN, bns.BNS_BF16
    indptr, indices, part, X, y = wl(2500, 70000, m, dims[0], dims[-1], 41)
    Ws = I.weights(dims, layer)
    train = dict(optimizer=bns.BNS_OPT_ADAM, dropout=0.4, dropout_seed=9)
    recs = []
    for peer in (0, bns.BNS_PEER_MEMORY):
        run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y, flags=bns.BNS_RETAIN_GRADS | peer)
        try:
            recs.append(record(run, dims, Ws, DRAWS[:3], lr=0.01, train=train))
        finally:
            run.close()
    assert_same(recs[0], recs[1])


@pytest.mark.parametrize("prec", [bns.BNS_FP32, bns.BNS_BF16])
@pytest.mark.parametrize("m,p", [(3, 0.5), (4, 0.1)])
def test_peer_memory_oracle_parity(prec, m, p):
    dims, layer = [37, 24, 16, 5], bns.BNS_LAYER_SAGE_MEAN
    L = len(dims) - 1
    indptr, indices, part, X, y = wl(3000, 90000, m, dims[0], dims[-1], 51 + m)
    Ws = I.weights(dims, layer)
    Wd = [w.astype(np.float64) for w in Ws]
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y,
                 flags=bns.BNS_RETAIN_GRADS | bns.BNS_PEER_MEMORY)
    orc = O.Oracle(indptr, indices, part, m, dims, layer, X, y)
    try:
        for e in range(2):
            run.sample(p, SEED, e)
            orc.sample(p, SEED, e)
            Ws = compare_epoch(run, orc, L, Ws, Wd, 0.5, prec, tag=f"peer epoch{e}")
    finally:
        run.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("layer", [bns.BNS_LAYER_SAGE_MEAN, bns.BNS_LAYER_GAT])
def test_ipc_two_processes_share_one_gpu(tmp_path, layer):
    """BNS_TRANSPORT_IPC: two processes (torchrun, gloo group for the host all-gather of the cudaIpcMemHandle_t's)
    on cuda:0 -- the multi-process peer-memory path -- bitwise equal to the in-process staged LOCAL run."""
    m, prec = 2, bns.BNS_BF16
    dims = [37, 24, 16, 5]
    wlargs = dict(N=2500, nnz=70000, m=m, d0=dims[0], C=dims[-1], seed=71)
    indptr, indices, part, X, y = wl(**wlargs)
    Ws = I.weights(dims, layer)
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y, flags=bns.BNS_RETAIN_GRADS)
    try:
        ref = record(run, dims, Ws, DRAWS)
    finally:
        run.close()
    out = tmp_path / "ipc"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={m}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(HERE, "ipc_worker.py"),
           json.dumps(dict(wl=wlargs, dims=dims, layer=layer, prec=prec, draws=[list(d) for d in DRAWS],
                           out=str(out)))]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=os.path.dirname(HERE))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = [np.load(f"{out}_{k}.npz") for k in range(m)]
    inner = [np.nonzero(part == k)[0] for k in range(m)]
    for e, a in enumerate(ref):
        for k in range(m):
            g = got[k]
            assert float(g[f"loss{e}"]) == a[0] and float(g[f"acc{e}"]) == a[1], (e, k)
            for l in range(len(dims) - 1):
                assert np.array_equal(g[f"g{e}_{l}"], a[2][l]), (e, k, l)
                assert np.array_equal(g[f"w{e}_{l}"], a[3][l]), (e, k, l)
            for l in range(1, len(dims)):
                assert np.array_equal(g[f"h{e}_{l}"], a[4][l - 1][inner[k]].astype(np.float32)), (e, k, l)
                assert np.array_equal(g[f"dh{e}_{l}"], a[5][l - 1][inner[k]].astype(np.float32)), (e, k, l)


def test_barrier_timeout_is_an_error_not_a_hang():
    """Rank 1 never calls bns_epoch: rank 0's first device barrier must give up (20 s) and the epoch must return
    BNS_ERR_RUNTIME; the context is then sticky-failed."""
    m, dims, layer = 2, [37, 16, 5], bns.BNS_LAYER_GCN
    indptr, indices, part, X, y = wl(1500, 30000, m, dims[0], dims[-1], 81)
    Ws = I.weights(dims, layer)
    run = GpuRun(indptr, indices, part, m, dims, layer, bns.BNS_FP32, X, y,
                 flags=bns.BNS_PEER_MEMORY)
    try:
        run.sample(0.5, SEED, 0)
        import torch
        W = [torch.tensor(w, device="cuda") for w in Ws]
        t0 = time.time()
        with pytest.raises(bns.BnsError) as ei:
            run.ctx[0].epoch(W, 0.1)
        assert ei.value.code == bns.BNS_ERR_RUNTIME and "timed out" in str(ei.value)
        # one 20 s wait, not one per barrier: later barriers of the failed epoch return at once
        assert time.time() - t0 < 40
        # the update saw an incomplete gradient sum and must not have touched the caller's weights
        for w, w0 in zip(W, Ws):
            assert np.array_equal(w.cpu().numpy(), w0)
        with pytest.raises(bns.BnsError) as ei:
            run.ctx[0].sample_boundary(0.5, SEED, 1)
        assert ei.value.code == bns.BNS_ERR_STATE
    finally:
        run.close()
