"""Helpers for the GPU parity tests: run m partitions of libbns on one GPU (BNS_TRANSPORT_LOCAL, one host thread
per rank) and compare with the oracle.  No expected value here comes from the CUDA path."""
import threading

import numpy as np

from oracle import oracle as O
from paper_2203_10983_b200 import bns

TOL = {bns.BNS_FP32: 1e-5, bns.BNS_BF16: 2e-2}     # north_star: per-layer activations / gradients
LOSS_TOL = 1e-3


def parallel(m, fn):
    res, errs = [None] * m, [None] * m

    def w(r):
        try:
            res[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    ts = [threading.Thread(target=w, args=(r,)) for r in range(m)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return res


def relerr(a, b):
    """normwise relative error max|a-b| / max|b|."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


# ---------------- epoch parity against the float64 oracle (fp32: 1e-5 everywhere; bf16: see below) ----------------
# bf16 (R19 storage) is compared with the plain float64 definition -- the oracle has no bf16 mode and no knowledge of
# the kernel's evaluation order (transform-first, R42).  A ReLU mask bit is an integer decided by floating point: a
# hidden unit whose pre-activation lies within bf16 rounding of zero takes either branch (R36).  Such a flip leaves the
# forward and every gradient ABOVE its layer unchanged but switches the gradient path below it, by several percent
# normwise at the test widths (16-24 hidden units; measured with any two bf16 evaluation orders, R36).  So
# in bf16: loss, H^l, Z^l, dLogits and the gradients above the highest flipped layer F are held to 2e-2; every flip
# must be ambiguous (|value| <= 2^-6 of the layer maximum on both sides) and flips may touch at most FLIP_SHARE_MAX of
# a layer's units; the gradients at and below F are reported (BF16_REPORT -> gpurun_out/bf16_margins.json) and held
# to 2e-2 by the layer-local check instead: each layer's outputs and gradients recomputed in float64 from that
# layer's own GPU inputs (the H^(l-1) it read, the dH^l it received and its own ReLU mask) and the oracle's sampled
# graph -- no flip can enter there.
FLIP_SHARE_MAX = 5e-3
BF16_REPORT = []


def relu_flips(run, orc, L, prec, tag):
    """Returns (F, flips per hidden layer): F = highest hidden layer with a ReLU flip (0 if none)."""
    F, out = 0, []
    for l in range(1, L):
        g = run.gather(bns.BNS_Q_H, l, run.dims[l])
        o = orc.tensor(O.T_H, l)
        flip = (g > 0) != (o > 0)
        n = int(flip.sum())
        out.append(n)
        if n == 0:
            continue
        assert prec == bns.BNS_BF16, (tag, "ReLU flips in fp32", l, n)
        scale = max(np.abs(o).max(), 1e-30)
        assert n <= FLIP_SHARE_MAX * o.size, (tag, "too many ReLU flips", l, n, o.size)
        assert np.abs(g[flip]).max() <= scale / 64 and np.abs(o[flip]).max() <= scale / 64, (tag, "flip not ambiguous", l)
        F = l
    return F, out


def sampled_operator(orc, m, layer, sampler, q):
    """The epoch's sampled aggregation as one global N x N float64 operator (COO triplets), from the ORACLE's induced
    lists (Alg.1 l.5): row v (inner to rank r) holds c_u / deg_G(v) (SAGE, R1-R3) or c_u / sqrt(d~_v d~_u) +
    [u = v] / d~_v (GCN, App. A); c_u = 1 on inner columns and 1/q on sampled boundary columns (BNS q = p, BES q; R3,
    R41); DropEdge: 1/q on every arc (R41)."""
    N = len(orc.indptr) - 1
    deg = np.diff(orc.indptr).astype(np.float64)
    rows, cols, vals = [], [], []
    for r in range(m):
        V = orc.list(O.V_LIST, r)
        ptr = orc.list(O.INDUCED_PTR, r)
        col = orc.list(O.INDUCED_COL, r)
        v = np.repeat(V, np.diff(ptr))
        inner = orc.part_of[col] == r
        inv = 1.0 / q if q > 0 else 0.0
        c = np.full(len(col), inv) if sampler == bns.BNS_SAMPLER_DROPEDGE else np.where(inner, 1.0, inv)
        if layer == bns.BNS_LAYER_SAGE_MEAN:
            w = c / deg[v]
        else:
            w = c / np.sqrt((deg[v] + 1.0) * (deg[col] + 1.0))
        rows.append(v)
        cols.append(col)
        vals.append(w)
    if layer == bns.BNS_LAYER_GCN:
        rows.append(np.arange(N))
        cols.append(np.arange(N))
        vals.append(1.0 / (deg + 1.0))
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), N


def bf16_round(a):
    import torch
    return torch.tensor(np.asarray(a, np.float32)).bfloat16().double().numpy()


def layer_local(op, snap, Ws, G, L, dims, layer, tol, tag, device="cpu", bf16=True):
    """Every layer against float64 recomputed from its OWN GPU inputs: the H^(l-1) it read, the dH^l it received and
    its own ReLU mask (snap), the weight operands (bf16-rounded in bf16 mode, R19) and the oracle's sampled operator
    (op) -- no ReLU flip can enter.  torch float64 (sparse CSR x dense; cuSPARSE when device = cuda).  Returns the
    margins; asserts <= tol."""
    import torch
    rows, cols, vals, N = op
    dev = torch.device(device)
    A = torch.sparse_coo_tensor(torch.from_numpy(np.stack([rows, cols]).astype(np.int64)), torch.from_numpy(vals),
                                (N, N)).coalesce().to(dev)
    At = A.t().coalesce()
    A, At = A.to_sparse_csr(), At.to_sparse_csr()
    sage = layer == bns.BNS_LAYER_SAGE_MEAN
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(dev)  # noqa: E731
    R = lambda a, b: float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))  # noqa: E731
    out = {}
    for l in range(1, L + 1):
        din = dims[l - 1]
        Wb = T(bf16_round(Ws[l - 1]) if bf16 else Ws[l - 1])   # the GEMM operand (R19: bf16 in bf16 mode)
        X = T(snap[("H", l - 1)])
        AX = A @ X
        pre = AX @ Wb[:din] + X @ Wb[din:] if sage else AX @ Wb
        Hg = T(snap[("H", l)])
        out[f"H{l}"] = e = R(Hg, pre.clamp_min(0) if l < L else pre)
        assert e <= tol, (tag, "layer-local H", l, e)
        dH = T(snap[("dH", l)])
        dpre = dH * (Hg > 0) if l < L else dH
        dW = torch.cat([AX.t() @ dpre, X.t() @ dpre]) if sage else AX.t() @ dpre
        out[f"dW{l}"] = e = R(T(G[l - 1]), dW)
        assert e <= tol, (tag, "layer-local dW", l, e)
        del AX, pre
        if l > 1:
            dX = At @ (dpre @ Wb[:din].t())
            if sage:
                dX = dX + dpre @ Wb[din:].t()
            out[f"dH{l - 1}"] = e = R(T(snap[("dH", l - 1)]), dX)
            assert e <= tol, (tag, "layer-local dH", l - 1, e)
    return out


def snapshot(run, L, what=("H", "Z", "dH")):
    """The GPU's per-layer tensors of the last epoch (inner rows by gid) as float32 -- exact for fp32 / bf16 values."""
    snap = {}
    for l in range(0, L + 1):
        if "H" in what:
            snap[("H", l)] = run.gather(bns.BNS_Q_H, l, run.dims[l]).astype(np.float32)
        if l >= 1 and "dH" in what:
            snap[("dH", l)] = run.gather(bns.BNS_Q_DH, l, run.dims[l]).astype(np.float32)
        if l >= 1 and "Z" in what and not (run.tf >> (l - 1)) & 1 and run.layer != bns.BNS_LAYER_GAT:
            snap[("Z", l)] = run.gather(bns.BNS_Q_Z, l, run.dims[l - 1]).astype(np.float32)
    return snap


class OracleView:
    """The oracle's tensors of its last epoch, read lazily."""

    def __init__(self, orc):
        self.orc = orc

    def get(self, kind, l):
        return self.orc.tensor({"H": O.T_H, "Z": O.T_Z, "dH": O.T_DH}[kind], l)


def check_epoch(gpu, orc_out, L, prec, dims, tf, layer, N, tag, labels, local_fn=None):
    """Parity of one epoch (see the block comment above).  gpu = (loss, acc, G, W_new, snap) with snap from
    snapshot(); orc_out = (loss, acc, G, W_new, OracleView).  local_fn(G) runs the bf16 layer-local check."""
    tol = TOL[prec]
    loss, acc, G, Wn, snap = gpu
    lo, ao, Go, Wd, ov = orc_out
    assert abs(loss - lo) <= LOSS_TOL * max(abs(lo), 1e-12), (tag, loss, lo)
    ntr = max(1, int((labels >= 0).sum()))
    assert abs(acc - ao) <= (0.0 if prec == bns.BNS_FP32 else 0.02) + 2.0 / ntr, (tag, acc, ao)
    # ReLU flips (R36)
    F, flips = 0, []
    for l in range(1, L):
        g, o = snap[("H", l)], ov.get("H", l)
        flip = (g > 0) != (o > 0)
        n = int(flip.sum())
        flips.append(n)
        if n == 0:
            continue
        scale = max(np.abs(o).max(), 1e-30)
        amb = scale / 64 if prec == bns.BNS_BF16 else tol * scale   # bf16: within its rounding; fp32: within 1e-5
        assert n <= (FLIP_SHARE_MAX if prec == bns.BNS_BF16 else 1e-6) * o.size, (tag, "too many ReLU flips", l, n)
        assert np.abs(g[flip]).max() <= amb and np.abs(o[flip]).max() <= amb, (tag, "flip not ambiguous", l, prec)
        F = l
    margins = {"loss": abs(loss - lo) / max(abs(lo), 1e-12)}
    for l in range(1, L + 1):
        if ("Z", l) in snap:
            margins[f"Z{l}"] = e = relerr(snap[("Z", l)], ov.get("Z", l))
            assert e <= tol, (tag, "Z", l, e)
        margins[f"H{l}"] = e = relerr(snap[("H", l)], ov.get("H", l))
        assert e <= tol, (tag, "H", l, e)
        margins[f"dH{l}"] = e = relerr(snap[("dH", l)], ov.get("dH", l))
        assert l < F or e <= tol, (tag, "dH", l, e)
    for l in range(L):
        margins[f"dW{l + 1}"] = e = relerr(G[l], Go[l])
        if l + 1 > F:
            assert e <= tol, (tag, "dW", l, e)
            e = relerr(Wn[l], Wd[l])
            assert e <= max(tol * 0.1, 1e-6), (tag, "W", l, e)
    rec = {"tag": tag, "prec": int(prec), "layer": layer, "F": F, "flips": flips,
           "units": [int(N * dims[l]) for l in range(1, L)], "vs_float64": margins}
    if local_fn is not None:
        rec["layer_local"] = local_fn(G)
    assert F == 0 or "layer_local" in rec or layer == bns.BNS_LAYER_GAT, (tag, "flips need the layer-local check")
    if prec == bns.BNS_BF16:
        BF16_REPORT.append(rec)
    return rec


def compare_epoch(run, orc, L, Ws, Wd, lr, prec, tag="", host=False, local=True):
    """One epoch on both sides (two independent weight trajectories: Ws fp32 on the GPU, Wd float64 in the oracle,
    updated in place / returned) and the parity checks of check_epoch.  Returns the GPU's new weights."""
    loss, acc, G, Wn = run.epoch(Ws, lr, host=host)
    lo, ao, Go = orc.epoch(Wd, lr)
    snap = snapshot(run, L)
    local_fn = None
    if local and run.layer != bns.BNS_LAYER_GAT and run.last_draw is not None:
        op = sampled_operator(orc, run.m, run.layer, *run.last_draw)
        local_fn = lambda G_: layer_local(op, snap, Ws, G_, L, run.dims, run.layer, TOL[prec], tag,  # noqa: E731
                                          bf16=prec == bns.BNS_BF16)
    check_epoch((loss, acc, G, Wn, snap), (lo, ao, Go, Wd, OracleView(orc)), L, prec, run.dims, run.tf, run.layer,
                run.N, tag, orc.labels, local_fn)
    return [w.astype(np.float32) for w in Wn]


class GpuRun:
    def __init__(self, indptr, indices, part, m, dims, layer, prec, X, y, flags=bns.BNS_RETAIN_GRADS, max_p=0.0):
        import torch
        self.torch = torch
        self.m, self.dims, self.layer, self.prec = m, list(dims), layer, prec
        self.part = np.asarray(part, np.int32)
        self.N = len(indptr) - 1
        self.group = bns.bns_group_create(m) if m > 1 else None

        def mk(r):
            inner = np.nonzero(self.part == r)[0]
            return bns.Context(rank=r, world=m, dims=self.dims, layer=layer, precision=prec, indptr=indptr,
                               indices=indices, part_of=self.part, features=np.ascontiguousarray(X[inner]),
                               labels=np.ascontiguousarray(y[inner]), group=self.group, flags=flags, max_p=max_p)

        self.last_draw = None    # (sampler, p or q) of the last draw, for the layer-local check
        self.ctx = parallel(m, mk)
        self.inner = [self.ctx[r].i32(bns.BNS_Q_INNER) for r in range(m)]
        self.tf = 0 if flags & bns.BNS_NO_TRANSFORM_FIRST else tf_rule(self.dims, layer)
        assert all(c.tf_layers() == self.tf for c in self.ctx), "transform-first layers differ from R42's rule"

    def close(self):
        for c in self.ctx:
            c.close()
        if self.group is not None:
            bns.bns_group_destroy(self.group)
            self.group = None

    def sample(self, p, seed, epoch):
        parallel(self.m, lambda r: self.ctx[r].sample_boundary(p, seed, epoch))
        self.last_draw = (bns.BNS_SAMPLER_BNS, p)

    def sample_edges(self, sampler, q, seed, epoch):
        parallel(self.m, lambda r: self.ctx[r].sample_edges(sampler, q, seed, epoch))
        self.last_draw = (sampler, q)

    def epoch(self, Ws, lr, host=False):
        """Ws: list of float32 numpy weights (shared initial value).  Returns (loss, acc, grads, W_new) and checks
        that every rank produced bitwise-identical grads / weights / loss."""
        torch = self.torch
        if host:
            Wr = [[np.array(w, np.float32, copy=True) for w in Ws] for _ in range(self.m)]
            Gr = [[np.zeros_like(w) for w in Ws] for _ in range(self.m)]
        else:
            Wr = [[torch.tensor(w, dtype=torch.float32, device="cuda") for w in Ws] for _ in range(self.m)]
            Gr = [[torch.zeros_like(w) for w in Wr[0]] for _ in range(self.m)]
        out = parallel(self.m, lambda r: self.ctx[r].epoch(Wr[r], lr, Gr[r]))
        if not host:
            torch.cuda.synchronize()
            Wr = [[w.cpu().numpy() for w in ws] for ws in Wr]
            Gr = [[g.cpu().numpy() for g in gs] for gs in Gr]
        for r in range(1, self.m):
            assert out[r] == out[0], "loss/acc differ across ranks"
            for a, b in zip(Gr[r], Gr[0]):
                assert np.array_equal(a, b), "grads differ across ranks"
            for a, b in zip(Wr[r], Wr[0]):
                assert np.array_equal(a, b), "weights differ across ranks"
        return out[0][0], out[0][1], Gr[0], Wr[0]

    def gather(self, what, layer, d):
        g = np.zeros((self.N, d), np.float64)
        for r in range(self.m):
            rows = self.ctx[r].rows(what, layer, d)
            g[self.inner[r]] = rows
        return g


def tf_rule(dims, layer):
    """R42: a GraphSAGE layer runs transform-first iff its 8-padded output is narrower than its input."""
    pad = [(d + 7) // 8 * 8 for d in dims]
    return sum(1 << l for l in range(len(dims) - 1) if layer == bns.BNS_LAYER_SAGE_MEAN and pad[l + 1] < pad[l])


def oracle_for(indptr, indices, part, m, dims, layer, X, y):
    return O.Oracle(indptr, indices, part, m, dims, layer, X, y)
