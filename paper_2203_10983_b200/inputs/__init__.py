"""Seeded synthetic workloads for BNS-GCN (setup only; shared by the oracle-side tests and the CUDA path).

This module holds no arithmetic of the method: it makes graphs, partitions, features, labels and initial
weights.  Shapes follow PAPER.md:375-387 (Table tab:setups) and BASELINE.json ``configs``; the recipe is
SURVEY.md §8(d) "Workload generation" and is restated in DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

SEED_GRAPH, SEED_FEAT, SEED_LABEL, SEED_PART, SEED_WEIGHT = 1, 2, 3, 4, 5
BNS_SEED = 0x0123456789ABCDEF

LAYER_SAGE, LAYER_GCN, LAYER_GAT = 0, 1, 2


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libbnsgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(os.path.dirname(_HERE))}`")
        L = ctypes.CDLL(path)
        i64, i32, u64, f64, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        L.gen_rmat_build.restype = vp
        L.gen_rmat_build.argtypes = [i64, i64, f64, f64, f64, u64]
        L.gen_rmat_nnz.restype = i64
        L.gen_rmat_nnz.argtypes = [vp]
        L.gen_rmat_fetch.argtypes = [vp, vp, vp]
        L.gen_rmat_free.argtypes = [vp]
        L.gen_features.argtypes = [i64, vp, i32, u64, vp]
        L.gen_labels.argtypes = [i64, i32, f64, u64, vp]
        L.gen_weights.argtypes = [i64, i64, i32, u64, vp]
        L.part_random.argtypes = [i64, i32, u64, vp]
        L.part_ldg2.argtypes = [i64, vp, vp, i32, f64, u64, vp]
        _LIB = L
    return _LIB


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def rmat(N: int, target_nnz: int, seed: int = SEED_GRAPH, abc=(0.57, 0.19, 0.19)):
    """Symmetric R-MAT CSR (indptr int64[N+1], indices int32[nnz]); sorted columns, no self loops."""
    L = lib()
    h = L.gen_rmat_build(N, target_nnz, abc[0], abc[1], abc[2], seed)
    nnz = L.gen_rmat_nnz(h)
    indptr = np.empty(N + 1, np.int64)
    indices = np.empty(nnz, np.int32)
    L.gen_rmat_fetch(h, _p(indptr), _p(indices))
    L.gen_rmat_free(h)
    return indptr, indices


def csr_from_edges(N: int, edges) -> tuple[np.ndarray, np.ndarray]:
    """Symmetric, deduplicated, self-loop-free CSR from an undirected edge list (small hand-made graphs)."""
    s = set()
    for u, v in edges:
        if u != v:
            s.add((u, v))
            s.add((v, u))
    arcs = sorted(s)
    indptr = np.zeros(N + 1, np.int64)
    for u, _ in arcs:
        indptr[u + 1] += 1
    indptr = np.cumsum(indptr).astype(np.int64)
    indices = np.array([v for _, v in arcs], np.int32)
    return indptr, indices


def features(gids: np.ndarray, d: int, seed: int = SEED_FEAT) -> np.ndarray:
    gids = np.ascontiguousarray(gids, np.int32)
    out = np.empty((len(gids), d), np.float32)
    lib().gen_features(len(gids), _p(gids), d, seed, _p(out))
    return out


def labels(N: int, C: int, train_frac: float, seed: int = SEED_LABEL) -> np.ndarray:
    out = np.empty(N, np.int32)
    lib().gen_labels(N, C, train_frac, seed, _p(out))
    return out


def multilabels(N: int, C: int, density: float = 0.1, seed: int = 0x5E1B) -> np.ndarray:
    """f4 (Yelp-style multi-label task): N x C multi-hot uint8 targets, each entry an independent
    Bernoulli(density) from a seeded Philox stream (row v depends only on the seed, so every rank slices the same
    global matrix).  The density is an assumption (the paper gives none)."""
    rng = np.random.Generator(np.random.Philox(seed))
    return (rng.random((N, C), dtype=np.float32) < density).astype(np.uint8)


def weights(dims, layer_kind: int, seed: int = SEED_WEIGHT) -> list[np.ndarray]:
    """Glorot-uniform fp32 weights; SAGE W^l is (2 d_{l-1}) x d_l (rows [0,d) multiply z), GCN d_{l-1} x d_l."""
    out = []
    for l in range(len(dims) - 1):
        # SAGE [z-half ; h-half] 2 d; GCN d; GAT [W ; a_l ; a_r] d + 2 (attention vectors Glorot-drawn like W)
        rows = 2 * dims[l] if layer_kind == LAYER_SAGE else dims[l] + 2 if layer_kind == LAYER_GAT else dims[l]
        w = np.empty((rows, dims[l + 1]), np.float32)
        lib().gen_weights(rows, dims[l + 1], l, seed, _p(w))
        out.append(w)
    return out


def partition(indptr, indices, m: int, method: str = "ldg2", seed: int = SEED_PART, slack: float = 0.05):
    N = len(indptr) - 1
    part = np.empty(N, np.int32)
    if m == 1:
        part[:] = 0
    elif method == "random":
        lib().part_random(N, m, seed, _p(part))
    elif method == "ldg2":
        indptr = np.ascontiguousarray(indptr, np.int64)
        indices = np.ascontiguousarray(indices, np.int32)
        lib().part_ldg2(N, _p(indptr), _p(indices), m, slack, seed, _p(part))
    else:
        raise ValueError(method)
    return part


@dataclass
class Shape:
    name: str
    N: int
    nnz: int
    d0: int
    C: int
    L: int
    hidden: int
    layer: int
    train_frac: float
    m: int = 1
    p: float = 0.1

    @property
    def dims(self):
        return [self.d0] + [self.hidden] * (self.L - 1) + [self.C]

    def scaled(self, s: float, name=None) -> "Shape":
        return Shape(name or f"{self.name}/{s:g}", max(int(self.N / s), 16), max(int(self.nnz / s), 16), self.d0,
                     self.C, self.L, self.hidden, self.layer, self.train_frac, self.m, self.p)


# BASELINE.json configs[0..4]; "edges" = arcs of the symmetric CSR
SHAPES = {
    "cora": Shape("cora", 2708, 10556, 1433, 7, 2, 16, LAYER_GCN, 1.0, m=2, p=0.5),
    "reddit": Shape("reddit", 232965, 114_600_000, 602, 41, 4, 256, LAYER_SAGE, 0.66, m=1, p=0.1),
    "products": Shape("products", 2449029, 61_900_000, 100, 47, 3, 128, LAYER_SAGE, 0.08, m=8, p=0.1),
    "yelp": Shape("yelp", 716847, 13_950_000, 300, 100, 4, 512, LAYER_SAGE, 0.75, m=8, p=0.1),
    "papers": Shape("papers", 111_059_956, 1_600_000_000, 128, 172, 3, 128, LAYER_SAGE, 0.78, m=8, p=0.01),
}


@dataclass
class Workload:
    shape: Shape
    indptr: np.ndarray
    indices: np.ndarray
    labels: np.ndarray
    part_of: np.ndarray = field(default=None)
    m: int = 1

    @property
    def N(self):
        return len(self.indptr) - 1

    @property
    def nnz(self):
        return int(self.indptr[-1])

    def inner(self, rank: int) -> np.ndarray:
        return np.nonzero(self.part_of == rank)[0].astype(np.int32)

    def features_of(self, rank: int) -> np.ndarray:
        return features(self.inner(rank), self.shape.d0)

    def labels_of(self, rank: int) -> np.ndarray:
        return np.ascontiguousarray(self.labels[self.part_of == rank])

    def all_features(self) -> np.ndarray:
        return features(np.arange(self.N, dtype=np.int32), self.shape.d0)

    def weights(self):
        return weights(self.shape.dims, self.shape.layer)


def make(shape: Shape, m: int, method: str = "ldg2") -> Workload:
    indptr, indices = rmat(shape.N, shape.nnz)
    y = labels(shape.N, shape.C, shape.train_frac)
    part = partition(indptr, indices, m, method)
    return Workload(shape, indptr, indices, y, part, m)
