"""ctypes wrapper over oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this module.
The product path (paper_2203_10983_b200.bns over libbns.so) never touches it.  See bns_oracle.cpp's header for
the passages each step follows.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

V_LIST, B_LIST, B_OFF, D_LIST, U_LIST, U_OFF, S_LIST, KEEP, INDUCED_PTR, INDUCED_COL = range(10)
SAMPLER_BES, SAMPLER_DROPEDGE = 1, 2
T_H, T_Z, T_DH = 0, 1, 2


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run make")
        L = ctypes.CDLL(path)
        vp, i64, i32, u64, u32, f64 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64,
                                       ctypes.c_uint32, ctypes.c_double)
        L.orc_philox4x32_10.argtypes = [vp, vp, vp]
        L.orc_draw.restype = u32
        L.orc_draw.argtypes = [u32, u32, u64, u64]
        L.orc_threshold.restype = u64
        L.orc_threshold.argtypes = [f64]
        L.orc_create.restype = vp
        L.orc_create.argtypes = [i64, vp, vp, vp, i32, i32, vp, i32, vp, vp]
        L.orc_destroy.argtypes = [vp]
        L.orc_list.restype = i64
        L.orc_list.argtypes = [vp, i32, i32, i32, vp, i64]
        L.orc_sample.restype = i32
        L.orc_sample.argtypes = [vp, f64, u64, u64]
        L.orc_set_keep.restype = i32
        L.orc_set_keep.argtypes = [vp, f64, i32, vp]
        L.orc_epoch.restype = i32
        L.orc_epoch.argtypes = [vp, vp, f64, vp, vp, vp]
        L.orc_tensor.restype = i64
        L.orc_tensor.argtypes = [vp, i32, i32, vp, i64]
        L.orc_set_training.restype = i32
        L.orc_set_training.argtypes = [vp, i32, f64, f64, f64, f64, u64]
        L.orc_drop_factor.restype = f64
        L.orc_drop_factor.argtypes = [vp, i32, i32, i32]
        L.orc_sample_edges.restype = i32
        L.orc_sample_edges.argtypes = [vp, i32, f64, u64, u64]
        L.orc_arc_keep.restype = i32
        L.orc_arc_keep.argtypes = [vp, i32, i32]
        L.orc_set_multilabel.argtypes = [vp, vp]
        L.orc_rows_sent.restype = i64
        L.orc_rows_sent.argtypes = [vp, i32]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def philox4x32_10(ctr, key):
    c = np.array(ctr, np.uint32)
    k = np.array(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(o))
    return [int(x) for x in o]


def draw(u, i, epoch, seed):
    return int(lib().orc_draw(u, i, epoch, seed))


def threshold(p):
    return int(lib().orc_threshold(p))


class Oracle:
    """All m partitions of Algorithm 1 simulated in one process (double precision)."""

    def __init__(self, indptr, indices, part_of, m, dims, layer, features, labels):
        self.indptr = np.ascontiguousarray(indptr, np.int64)
        self.indices = np.ascontiguousarray(indices, np.int32)
        self.part_of = np.ascontiguousarray(part_of, np.int32)
        self.dims = np.ascontiguousarray(dims, np.int32)
        self.features = np.ascontiguousarray(features, np.float32)
        self.labels = np.ascontiguousarray(labels, np.int32)
        self.N = len(self.indptr) - 1
        self.m, self.L, self.layer = m, len(dims) - 1, layer
        self.h = lib().orc_create(self.N, _p(self.indptr), _p(self.indices), _p(self.part_of), m, self.L,
                                  _p(self.dims), layer, _p(self.features), _p(self.labels))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def set_multilabel(self, targets):
        """f4 / R44: N x C multi-hot targets (global ids); loss -> sigmoid BCE, acc -> F1-micro.  None: back to CE."""
        if targets is None:
            lib().orc_set_multilabel(self.h, None)
            return
        self._targets = np.ascontiguousarray(targets, np.uint8)
        assert self._targets.shape == (self.N, int(self.dims[-1]))
        lib().orc_set_multilabel(self.h, _p(self._targets))

    def set_training(self, optimizer=0, beta1=0.9, beta2=0.999, eps=1e-8, dropout=0.0, dropout_seed=0):
        """f2: optimizer 0 = SGD (Alg.1 l.14), 1 = Adam; dropout rate on every layer input (R38)."""
        rc = lib().orc_set_training(self.h, optimizer, beta1, beta2, eps, dropout, dropout_seed)
        assert rc == 0, rc

    def drop_factor(self, gid, col, layer):
        return float(lib().orc_drop_factor(self.h, gid, col, layer))

    def list(self, what, rank, peer=0):
        n = lib().orc_list(self.h, what, rank, peer, None, 0)
        out = np.zeros(max(n, 0), np.int64)
        lib().orc_list(self.h, what, rank, peer, _p(out), n)
        return out

    def sample(self, p, seed, epoch):
        rc = lib().orc_sample(self.h, p, seed, epoch)
        assert rc == 0, rc

    def sample_edges(self, sampler, q, seed, epoch):
        """f3: BES (sampler 1) or DropEdge (2) with arc keep probability q (R40, R41)."""
        rc = lib().orc_sample_edges(self.h, sampler, q, seed, epoch)
        assert rc == 0, rc

    def arc_keep(self, v, u):
        return bool(lib().orc_arc_keep(self.h, v, u))

    def set_keep(self, p, per_rank_flags):
        for r, f in enumerate(per_rank_flags):
            a = np.ascontiguousarray(f, np.int32)
            lib().orc_set_keep(self.h, p, r, _p(a))

    def epoch(self, weights, lr):
        """weights: list of float64 arrays (updated in place). Returns (loss, acc, grads)."""
        W = [np.ascontiguousarray(w, np.float64) for w in weights]
        G = [np.zeros_like(w) for w in W]
        Wp = (ctypes.c_void_p * self.L)(*[w.ctypes.data for w in W])
        Gp = (ctypes.c_void_p * self.L)(*[g.ctypes.data for g in G])
        loss = ctypes.c_double()
        acc = ctypes.c_double()
        rc = lib().orc_epoch(self.h, Wp, lr, Gp, ctypes.byref(loss), ctypes.byref(acc))
        assert rc == 0, rc
        for w, wn in zip(weights, W):
            w[...] = wn
        return loss.value, acc.value, G

    def tensor(self, what, layer):
        n = lib().orc_tensor(self.h, what, layer, None, 0)
        if n < 0:
            return None
        out = np.zeros(n, np.float64)
        lib().orc_tensor(self.h, what, layer, _p(out), n)
        d = n // self.N if self.N else 0
        return out.reshape(self.N, d)

    def rows_sent(self, layer):
        return int(lib().orc_rows_sent(self.h, layer))
