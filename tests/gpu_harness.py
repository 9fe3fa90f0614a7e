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
