"""Full-size parity (BASELINE.json configs[1], Reddit-shaped: 232,965 nodes, 114.6 M arcs, 602 features, SAGE 4x256):

* the north-star Target (BASELINE.json north_star, Alg. 1 PAPER.md:269-297 with the 4 x 256 model of PAPER.md:416):
  m = 8 partitions (LOCAL transport on one GPU; two-constraint LDG and random partitions), p = 0.1, two epochs, fp32
  and bf16, against the float64 oracle on EVERY row of every layer: loss within 1e-3, H^l / Z^l / dH^l / dW^l within
  1e-5 (fp32) and 2e-2 (bf16, with the ReLU-flip rule and the layer-local check of tests/gpu_harness.py); plus the
  bench configuration (m = 1, bf16) for one epoch, gradients included;

* m = 1 in bench.py's launch configuration (bf16, tcgen05 GEMMs): sampled rows of Z^1 and H^1 recomputed one by one
  in float64 from raw neighbours (PAPER.md:100 / R1), and a finite loss;
* m = 8, p = 0.1 on one GPU (LOCAL transport): keep masks, U_i and S_{i,j} bit-exact against the oracle's plan +
  sample at full size, and sampled rows of Z^1 recomputed from the oracle's U_i (1/p on kept halo columns, R3).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2203_10983_b200 import bns
from paper_2203_10983_b200 import inputs as I

import threading

from gpu_harness import GpuRun, OracleView, check_epoch, layer_local, parallel, sampled_operator, snapshot

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
SEED = I.BNS_SEED


@pytest.fixture(scope="module")
def reddit():
    sh = I.SHAPES["reddit"]
    indptr, indices = I.rmat(sh.N, sh.nnz)
    y = I.labels(sh.N, sh.C, sh.train_frac)
    return sh, indptr, indices, y


def z_rows(indptr, indices, X_of, rows, kept_of=None, inv_p=1.0, part=None):
    """z_v = (1/deg_G v) Σ_{u ∈ N(v), kept} c_u x_u in float64 for the listed gids"""
    out = []
    for v in rows:
        nb = indices[indptr[v]:indptr[v + 1]]
        if len(nb) == 0:
            out.append(np.zeros(X_of(np.array([v])).shape[1]))
            continue
        if kept_of is None:
            use, c = nb, np.ones(len(nb))
        else:
            inner = part[nb] == part[v]
            keep = inner | np.isin(nb, kept_of)
            use = nb[keep]
            c = np.where(inner[keep], 1.0, inv_p)
        out.append((X_of(use).astype(np.float64) * c[:, None]).sum(0) / len(nb))
    return np.array(out)


def test_reddit_m1_bench_config(reddit):
    sh, indptr, indices, y = reddit
    part = np.zeros(sh.N, np.int32)
    X = I.features(np.arange(sh.N, dtype=np.int32), sh.d0)
    run = GpuRun(indptr, indices, part, 1, sh.dims, sh.layer, bns.BNS_BF16, X, y, flags=0)
    try:
        Ws = I.weights(sh.dims, sh.layer)
        run.sample(0.1, SEED, 0)
        loss, acc, G, _ = run.epoch(Ws, 0.0)
        assert np.isfinite(loss) and 0.5 * np.log(sh.C) < loss < 3 * np.log(sh.C)
        rng = np.random.default_rng(0)
        rows = np.sort(rng.choice(sh.N, 400, replace=False))
        deg = np.diff(indptr)
        rows = np.union1d(rows, np.argsort(-deg)[:8])          # include the biggest hubs (split rows)
        assert run.tf == 0b1001                 # R42: 608 -> 256 and 256 -> 41 run transform-first
        zr = z_rows(indptr, indices, lambda g: X[g], rows)
        H1 = run.ctx[0].rows(bns.BNS_Q_H, 1, sh.hidden)
        W0 = Ws[0].astype(np.float64)
        pre = np.concatenate([zr, X[rows].astype(np.float64)], 1) @ W0
        h = np.maximum(pre, 0)
        err = np.abs(H1[rows] - h).max() / np.abs(h).max()
        assert err < 2e-2, err
    finally:
        run.close()


def test_reddit_m8_sampling_bitexact_and_rows(reddit):
    sh, indptr, indices, y = reddit
    m, p = 8, 0.1
    part = I.partition(indptr, indices, m, "ldg2")
    dims = [sh.d0, 16, 8]
    y = I.labels(sh.N, dims[-1], sh.train_frac)
    X = I.features(np.arange(sh.N, dtype=np.int32), sh.d0)
    run = GpuRun(indptr, indices, part, m, dims, sh.layer, bns.BNS_BF16, X, y, flags=0, max_p=0.2)
    orc = O.Oracle(indptr, indices, part, m, [1, 1], 0, np.zeros((sh.N, 1), np.float32), np.zeros(sh.N, np.int32))
    try:
        for e in (0, 1):
            run.sample(p, SEED, e)
            orc.sample(p, SEED, e)
            for r in range(m):
                c = run.ctx[r]
                assert np.array_equal(c.mask(), orc.list(O.KEEP, r).astype(np.uint8))
                assert np.array_equal(c.i32(bns.BNS_Q_HALO), orc.list(O.U_LIST, r))
                S, So = c.i32(bns.BNS_Q_SEND), c.i64(bns.BNS_Q_SEND_OFF)
                for j in range(m):
                    assert np.array_equal(S[So[j]:So[j + 1]], orc.list(O.S_LIST, r, j))
        Ws = I.weights(dims, sh.layer)
        run.epoch(Ws, 0.0)
        rng = np.random.default_rng(1)
        for r in (0, 5):
            V = run.inner[r]
            H1 = run.ctx[r].rows(bns.BNS_Q_H, 1, dims[1])   # layer 1 runs transform-first (608 -> 16, R42)
            k = np.sort(rng.choice(len(V), 200, replace=False))
            U = orc.list(O.U_LIST, r)
            zr = z_rows(indptr, indices, lambda g: X[g], V[k], kept_of=U, inv_p=1.0 / p, part=part)
            h = np.maximum(np.concatenate([zr, X[V[k]].astype(np.float64)], 1) @ Ws[0].astype(np.float64), 0)
            err = np.abs(H1[k] - h).max() / np.abs(h).max()
            assert err < 2e-2, (r, err)
    finally:
        run.close()


@pytest.mark.parametrize("name", ["products", "yelp"])
def test_other_shapes_m1_two_layers(name):
    """BASELINE.json configs[2] / [3] at full size, m = 1, bf16 (bench.py's launch configuration): sampled rows of H^1
    recomputed in float64 from X (layer 1), and of H^2 from the kernel's own H^1 rows (layer 2 -- on the Yelp shape
    its 512-wide gather runs as two 256-column L2 tiles), against R1 / PAPER.md:100."""
    sh = I.SHAPES[name]
    indptr, indices = I.rmat(sh.N, sh.nnz)
    y = I.labels(sh.N, sh.C, sh.train_frac)
    part = np.zeros(sh.N, np.int32)
    X = I.features(np.arange(sh.N, dtype=np.int32), sh.d0)
    run = GpuRun(indptr, indices, part, 1, sh.dims, sh.layer, bns.BNS_BF16, X, y, flags=0)
    try:
        Ws = I.weights(sh.dims, sh.layer)
        run.sample(0.1, SEED, 0)
        loss, acc, G, _ = run.epoch(Ws, 0.0)
        assert np.isfinite(loss)
        rng = np.random.default_rng(1)
        deg = np.diff(indptr)
        rows = np.union1d(np.sort(rng.choice(sh.N, 300, replace=False)), np.argsort(-deg)[:6])
        H1 = run.ctx[0].rows(bns.BNS_Q_H, 1, sh.dims[1])
        H2 = run.ctx[0].rows(bns.BNS_Q_H, 2, sh.dims[2])
        for l, (Hin, Hout) in enumerate([(X, H1), (H1, H2)]):
            zr = z_rows(indptr, indices, lambda g: Hin[g], rows)
            pre = np.concatenate([zr, Hin[rows].astype(np.float64)], 1) @ Ws[l].astype(np.float64)
            h = np.maximum(pre, 0)
            err = np.abs(Hout[rows] - h).max() / np.abs(h).max()
            assert err < 2e-2, (name, l + 1, err)
    finally:
        run.close()


class OracleThread(threading.Thread):
    """One oracle (single-threaded float64, its own weight trajectory) stepping through epochs in the background;
    after each epoch it waits until the test has compared that epoch's tensors (ctypes releases the GIL, so several
    oracles and the GPU runs proceed at the same time on the box's cores)."""

    def __init__(self, orc, W, p, epochs, lr):
        super().__init__(daemon=True)
        self.orc, self.W, self.p, self.epochs, self.lr = orc, W, p, epochs, lr
        self.done = [threading.Event() for _ in range(epochs)]
        self.go = [threading.Event() for _ in range(epochs)]
        self.out, self.err, self.secs = [None] * epochs, None, []

    def run(self):
        import time
        try:
            for e in range(self.epochs):
                t0 = time.time()
                self.orc.sample(self.p, SEED, e)
                lo, ao, Go = self.orc.epoch(self.W, self.lr)
                self.secs.append(time.time() - t0)
                self.out[e] = (lo, ao, Go, [w.copy() for w in self.W], OracleView(self.orc))
                self.done[e].set()
                self.go[e].wait()
        except BaseException as ex:  # noqa: BLE001
            self.err = ex
            for d in self.done:
                d.set()

    def result(self, e):
        self.done[e].wait()
        if self.err is not None:
            raise self.err
        return self.out[e]


def gpu_epochs(indptr, indices, part, m, dims, layer, prec, X, y, p, epochs, lr, light):
    """GPU side of a configuration: per epoch (loss, acc, G, W_new, snapshot) and, in bf16, the layer-local margins
    (the sampled operator from `light`, an oracle holding only the plan and the draw)."""
    L = len(dims) - 1
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y, flags=bns.BNS_RETAIN_GRADS,
                 max_p=0.2 if m > 1 else 0.0)
    W = I.weights(dims, layer)
    out = []
    try:
        for e in range(epochs):
            run.sample(p, SEED, e)
            Ws = [w.copy() for w in W]
            loss, acc, G, Wn = run.epoch(Ws, lr)
            snap = snapshot(run, L)
            light.sample(p, SEED, e)
            op = sampled_operator(light, m, layer, bns.BNS_SAMPLER_BNS, p)
            bf = prec == bns.BNS_BF16
            local = layer_local(op, snap, Ws, G, L, dims, layer, 2e-2 if bf else 1e-5,
                                f"m{m} prec{prec} e{e} layer-local", device="cuda", bf16=bf)
            del op
            out.append(((loss, acc, G, Wn, snap), local))
            W = [w.astype(np.float32) for w in Wn]
        return out, run.tf
    finally:
        run.close()


def test_north_star_full_size(reddit):
    """BASELINE.json north_star Target: Reddit-shaped 4-layer GraphSAGE epoch at p = 0.1 on 8 partitions against the
    oracle (SURVEY.md §8(c) "Large-config parity"), plus the m = 1 bench configuration."""
    import json
    import os
    import time
    sh, indptr, indices, y = reddit
    dims, layer, L, lr = sh.dims, sh.layer, sh.L, 0.1
    X = I.features(np.arange(sh.N, dtype=np.int32), sh.d0)
    zeros = (np.zeros((sh.N, 1), np.float32), np.zeros(sh.N, np.int32))
    configs = [("ldg2", 8, 2), ("random", 8, 2), ("single", 1, 1)]
    threads, parts = {}, {}
    t0 = time.time()
    for name, m, epochs in configs:
        part = np.zeros(sh.N, np.int32) if m == 1 else I.partition(indptr, indices, m, name)
        parts[name] = part
        orc = O.Oracle(indptr, indices, part, m, dims, layer, X, y)
        threads[name] = OracleThread(orc, [w.astype(np.float64) for w in I.weights(dims, layer)], 0.1, epochs, lr)
        threads[name].start()
    report = {"oracle_seconds": {}, "records": []}
    try:
        for name, m, epochs in configs:
            light = O.Oracle(indptr, indices, parts[name], m, [1, 1], 0, *zeros)
            precs = (bns.BNS_BF16,) if m == 1 else (bns.BNS_FP32, bns.BNS_BF16)
            gpu = {prec: gpu_epochs(indptr, indices, parts[name], m, dims, layer, prec, X, y, 0.1, epochs, lr, light)
                   for prec in precs}
            del light
            th = threads[name]
            for e in range(epochs):
                orc_out = th.result(e)
                for prec in precs:
                    (g, local), tf = gpu[prec][0][e], gpu[prec][1]
                    rec = check_epoch(g, orc_out, L, prec, dims, tf, layer, sh.N,
                                      f"{name} m={m} prec={prec} epoch {e}", y,
                                      lambda G_, lo=local: lo)
                    report["records"].append(rec)
                th.go[e].set()
            report["oracle_seconds"][name] = th.secs
            del gpu
    finally:
        for th in threads.values():
            for ev in th.go:
                ev.set()
    report["wall_seconds"] = time.time() - t0
    model = None
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            model = line.split(":", 1)[1].strip()
            break
    report["host"] = {"nproc": os.cpu_count(), "model": model,
                      "note": "each oracle single-threaded (three run concurrently, one per configuration)"}
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "north_star_fullsize.json"), "w") as f:
        json.dump(report, f, indent=1)
