"""Thin ctypes binding over libbns.so (include/bns.h) -- argument marshalling only.

Every step of the BNS-GCN hot path runs in the library's sm_100a kernels; this module only converts Python /
numpy / torch arguments to pointers.  There is no fallback: if libbns.so is missing or no GPU is visible the calls
raise.  Names follow the C ABI (bns_setup, bns_sample_boundary, bns_epoch, bns_query, ...); ``Context`` is a small
convenience wrapper around them.
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BNS_LIB") or os.path.join(_HERE, "libbns.so")   # BNS_LIB: A/B builds only

BNS_OK, BNS_ERR_INVALID, BNS_ERR_RUNTIME, BNS_ERR_STATE, BNS_ERR_OOM, BNS_ERR_NONFINITE = range(6)
BNS_LAYER_SAGE_MEAN, BNS_LAYER_GCN, BNS_LAYER_GAT = 0, 1, 2
BNS_FP32, BNS_BF16 = 0, 1
BNS_TRANSPORT_NONE, BNS_TRANSPORT_NCCL, BNS_TRANSPORT_LOCAL, BNS_TRANSPORT_NULL_EMULATE, BNS_TRANSPORT_IPC = 0, 1, 2, 3, 4
BNS_PLAN_ONLY, BNS_DEBUG_EXCHANGE_INDICES, BNS_TIMING, BNS_RETAIN_GRADS, BNS_NO_TRANSFORM_FIRST = 0x1, 0x2, 0x4, 0x8, 0x10
BNS_CACHE_INPUT_HALO = 0x20
BNS_PEER_MEMORY = 0x40   # f1: exchanges fused over peer memory (LOCAL in-process; implied by IPC)
BNS_PREFETCH_DRAW = 0x80   # R48: bns_step enqueues the next epoch's draw before its closing sync
(BNS_Q_COUNTS, BNS_Q_INNER, BNS_Q_BOUNDARY, BNS_Q_BOUNDARY_OFF, BNS_Q_SENDCAND, BNS_Q_SENDCAND_OFF, BNS_Q_MASK,
 BNS_Q_HALO, BNS_Q_HALO_OFF, BNS_Q_SEND, BNS_Q_SEND_OFF, BNS_Q_H, BNS_Q_Z, BNS_Q_DH, BNS_Q_HALO_ROWS, BNS_Q_INDUCED,
 BNS_Q_TIMES, BNS_Q_STATIC_CSR, BNS_Q_MEMORY, BNS_Q_KERNEL_COUNT, BNS_Q_INDUCED_T, BNS_Q_TF_LAYERS,
 BNS_Q_BOUNDARY_ROW) = range(23)
BNS_SAMPLER_BNS, BNS_SAMPLER_BES, BNS_SAMPLER_DROPEDGE = 0, 1, 2
PHASES = ["sample", "induce", "pack", "exchange", "spmm_fwd", "gemm_fwd", "loss", "gemm_bwd", "spmm_bwd",
          "exchange_bwd", "scatter", "allreduce", "update", "epoch_total", "sample_total"]

EXPORTS = ["bns_get_unique_id", "bns_group_create", "bns_group_destroy", "bns_setup", "bns_sample_boundary",
           "bns_sample_edges", "bns_set_multilabel", "bns_epoch", "bns_step", "bns_set_timing", "bns_set_training", "bns_query", "bns_stream", "bns_last_error", "bns_destroy",
           "bns_gemm"]
BNS_OPT_SGD, BNS_OPT_ADAM = 0, 1


class BnsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"bns error {code}: {msg}")
        self.code = code


# bns_allgather_fn: int32 (*)(const void* send, void* recv, int64 bytes, void* user)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)


class bns_config(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("transport", ctypes.c_int32), ("nccl_id", ctypes.c_void_p), ("group", ctypes.c_void_p),
                ("stream", ctypes.c_void_p), ("num_layers", ctypes.c_int32), ("dims", ctypes.c_void_p),
                ("layer", ctypes.c_int32), ("precision", ctypes.c_int32), ("max_p", ctypes.c_double),
                ("flags", ctypes.c_uint32), ("allgather", ALLGATHER_FN), ("allgather_user", ctypes.c_void_p)]


def torch_allgather(world: int, group=None):
    """A bns_allgather_fn over a torch.distributed CPU (gloo) group -- host bytes only (buffer handles, counts)."""
    import torch
    import torch.distributed as dist

    def cb(send, recv, nbytes, user):
        try:
            src = torch.tensor(np.frombuffer(ctypes.string_at(send, nbytes), np.uint8))
            out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(out, src, group=group)
            buf = np.ascontiguousarray(np.concatenate([o.numpy() for o in out]))   # keep it alive during the copy
            ctypes.memmove(recv, buf.ctypes.data, nbytes * world)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
            return 1

    return ALLGATHER_FN(cb)


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing -- build it with `make` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u64, f64, f32 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                       ctypes.c_double, ctypes.c_float)
        L.bns_get_unique_id.argtypes = [vp]
        L.bns_group_create.argtypes = [i32, ctypes.POINTER(vp)]
        L.bns_group_destroy.argtypes = [vp]
        L.bns_setup.argtypes = [ctypes.POINTER(bns_config), i64, vp, vp, vp, vp, vp, ctypes.POINTER(vp)]
        L.bns_sample_boundary.argtypes = [vp, f64, u64, u64]
        L.bns_sample_edges.argtypes = [vp, i32, f64, u64, u64]
        L.bns_set_multilabel.argtypes = [vp, vp]
        L.bns_epoch.argtypes = [vp, vp, f32, vp, ctypes.POINTER(f64), ctypes.POINTER(f64)]
        L.bns_set_training.argtypes = [vp, i32, f64, f64, f64, f64, u64]
        L.bns_step.argtypes = [vp, f64, u64, u64, vp, f32, vp, ctypes.POINTER(f64), ctypes.POINTER(f64)]
        L.bns_set_timing.argtypes = [vp, i32]
        L.bns_query.argtypes = [vp, i32, i32, vp, i64, ctypes.POINTER(i64)]
        L.bns_gemm.argtypes = [i32, i32, i64, i64, i64, vp, vp, i64, vp, i64, vp, i64, vp, i64, i32, vp,
                               ctypes.POINTER(i32)]
        L.bns_stream.restype = vp
        L.bns_stream.argtypes = [vp]
        L.bns_last_error.restype = ctypes.c_char_p
        L.bns_last_error.argtypes = [vp]
        L.bns_destroy.argtypes = [vp]
        for f in ("bns_get_unique_id", "bns_group_create", "bns_setup", "bns_sample_boundary", "bns_sample_edges",
                  "bns_set_multilabel", "bns_epoch", "bns_step", "bns_set_timing",
                  "bns_set_training", "bns_query", "bns_gemm"):
            getattr(L, f).restype = ctypes.c_int
        L.bns_group_destroy.restype = None
        L.bns_destroy.restype = None
        _LIB = L
    return _LIB


def _check(rc, ctx=None):
    if rc != BNS_OK:
        msg = lib().bns_last_error(ctx).decode(errors="replace")
        raise BnsError(rc, msg)


def _ptr(a) -> int:
    """Pointer of a numpy array or torch tensor (contiguous)."""
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    return a.ctypes.data


BNS_GEMM_FWD, BNS_GEMM_WGRAD, BNS_GEMM_WGRAD2, BNS_GEMM_DX = range(4)


def bns_gemm(precision, kind, M, N, K, A0, A1, lda, B, ldb, C, ldc, rowscale=None, scale_cols=0, flags=0,
             stream=None) -> int:
    """One GEMM of the epoch by the epoch's own kernels (bns.h bns_gemm); torch CUDA tensors in, split-K factor out."""
    sp = ctypes.c_int32(0)
    _check(lib().bns_gemm(precision, kind, M, N, K, _ptr(A0), _ptr(A1) if A1 is not None else None, lda, _ptr(B),
                          ldb, _ptr(C), ldc, _ptr(rowscale) if rowscale is not None else None, scale_cols, flags,
                          stream, ctypes.byref(sp)))
    return sp.value


def bns_get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().bns_get_unique_id(buf))
    return bytes(buf)


def bns_group_create(world: int):
    g = ctypes.c_void_p()
    _check(lib().bns_group_create(world, ctypes.byref(g)))
    return g


def bns_group_destroy(g):
    lib().bns_group_destroy(g)


def bns_setup(cfg: bns_config, indptr, indices, part_of, features, labels):
    out = ctypes.c_void_p()
    N = len(indptr) - 1
    rc = lib().bns_setup(ctypes.byref(cfg), N, _ptr(indptr), _ptr(indices), _ptr(part_of),
                         _ptr(features) if features is not None else None,
                         _ptr(labels) if labels is not None else None, ctypes.byref(out))
    _check(rc, None)
    return out


def bns_sample_boundary(ctx, p: float, seed: int, epoch: int):
    _check(lib().bns_sample_boundary(ctx, float(p), int(seed) & (2**64 - 1), int(epoch) & (2**64 - 1)), ctx)


def bns_sample_edges(ctx, sampler: int, q: float, seed: int, epoch: int):
    _check(lib().bns_sample_edges(ctx, int(sampler), float(q), int(seed) & (2**64 - 1), int(epoch) & (2**64 - 1)), ctx)


def bns_set_multilabel(ctx, targets):
    """f4: |V_i| x C multi-hot uint8 targets (None: back to single-label cross entropy)."""
    if targets is None:
        _check(lib().bns_set_multilabel(ctx, None), ctx)
        return
    t = np.ascontiguousarray(targets, np.uint8)
    _check(lib().bns_set_multilabel(ctx, t.ctypes.data_as(ctypes.c_void_p)), ctx)


def bns_epoch(ctx, weights: Sequence, lr: float, grads: Sequence | None = None):
    L = len(weights)
    wp = (ctypes.c_void_p * L)(*[_ptr(w) for w in weights])
    gp = (ctypes.c_void_p * L)(*[_ptr(g) for g in grads]) if grads is not None else None
    loss = ctypes.c_double()
    acc = ctypes.c_double()
    rc = lib().bns_epoch(ctx, wp, ctypes.c_float(lr), gp, ctypes.byref(loss), ctypes.byref(acc))
    _check(rc, ctx)
    return loss.value, acc.value


def bns_step(ctx, p: float, seed: int, epoch: int, weights: Sequence, lr: float, grads: Sequence | None = None):
    """bns_sample_boundary + bns_epoch in one call."""
    L = len(weights)
    wp = (ctypes.c_void_p * L)(*[_ptr(w) for w in weights])
    gp = (ctypes.c_void_p * L)(*[_ptr(g) for g in grads]) if grads is not None else None
    loss = ctypes.c_double()
    acc = ctypes.c_double()
    rc = lib().bns_step(ctx, float(p), int(seed) & (2**64 - 1), int(epoch) & (2**64 - 1), wp, ctypes.c_float(lr), gp,
                        ctypes.byref(loss), ctypes.byref(acc))
    _check(rc, ctx)
    return loss.value, acc.value


def bns_set_training(ctx, optimizer: int = BNS_OPT_SGD, beta1: float = 0.9, beta2: float = 0.999,
                     eps: float = 1e-8, dropout: float = 0.0, dropout_seed: int = 0):
    _check(lib().bns_set_training(ctx, optimizer, beta1, beta2, eps, dropout, int(dropout_seed) & (2**64 - 1)), ctx)


def bns_query(ctx, what: int, layer: int = 0) -> bytes:
    n = ctypes.c_int64()
    _check(lib().bns_query(ctx, what, layer, None, 0, ctypes.byref(n)), ctx)
    buf = (ctypes.c_uint8 * max(n.value, 1))()
    _check(lib().bns_query(ctx, what, layer, buf, n.value, ctypes.byref(n)), ctx)
    return bytes(buf)[: n.value]


def bns_stream(ctx) -> int:
    return lib().bns_stream(ctx) or 0


def bns_destroy(ctx):
    lib().bns_destroy(ctx)


class Context:
    """One partition (rank) of BNS-GCN on one GPU."""

    def __init__(self, *, rank: int, world: int, dims: Sequence[int], layer: int, precision: int, indptr, indices,
                 part_of, features, labels, device: int = 0, transport: int | None = None, nccl_id: bytes | None = None,
                 group=None, max_p: float = 0.0, flags: int = 0, stream: int | None = None, allgather=None):
        self.indptr = np.ascontiguousarray(indptr, np.int64)
        self.indices = np.ascontiguousarray(indices, np.int32)
        self.part_of = np.ascontiguousarray(part_of, np.int32)
        self.features = None if features is None else np.ascontiguousarray(features, np.float32)
        self.labels = None if labels is None else np.ascontiguousarray(labels, np.int32)
        self.dims = np.ascontiguousarray(dims, np.int32)
        self.L = len(dims) - 1
        self.world, self.rank, self.layer = world, rank, layer
        if transport is None:
            transport = BNS_TRANSPORT_NONE if world == 1 else (BNS_TRANSPORT_LOCAL if group else BNS_TRANSPORT_NCCL)
        self._id = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
        self._allgather = allgather   # keep the ctypes callback alive as long as the context
        cfg = bns_config(rank=rank, world=world, device=device, transport=transport,
                         nccl_id=ctypes.addressof(self._id) if self._id else None, group=group, stream=stream,
                         num_layers=self.L, dims=self.dims.ctypes.data, layer=layer, precision=precision,
                         max_p=max_p, flags=flags, allgather=allgather if allgather else ALLGATHER_FN(),
                         allgather_user=None)
        self.h = bns_setup(cfg, self.indptr, self.indices, self.part_of, self.features, self.labels)
        # host inputs are only borrowed during setup
        self.indptr = self.indices = self.part_of = self.features = None

    def close(self):
        if getattr(self, "h", None):
            bns_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def sample_boundary(self, p, seed, epoch):
        bns_sample_boundary(self.h, p, seed, epoch)

    def set_multilabel(self, targets):
        bns_set_multilabel(self.h, targets)

    def sample_edges(self, sampler, q, seed, epoch):
        bns_sample_edges(self.h, sampler, q, seed, epoch)

    def epoch(self, weights, lr, grads=None):
        if weights and hasattr(weights[0], "is_cuda") and weights[0].is_cuda:
            import torch
            torch.cuda.current_stream().synchronize()
        return bns_epoch(self.h, weights, lr, grads)

    def step(self, p, seed, epoch, weights, lr, grads=None):
        if weights and hasattr(weights[0], "is_cuda") and weights[0].is_cuda:
            import torch
            torch.cuda.current_stream().synchronize()
        return bns_step(self.h, p, seed, epoch, weights, lr, grads)

    def set_timing(self, on: bool):
        _check(lib().bns_set_timing(self.h, 1 if on else 0), self.h)

    def set_training(self, optimizer=BNS_OPT_SGD, beta1=0.9, beta2=0.999, eps=1e-8, dropout=0.0, dropout_seed=0):
        bns_set_training(self.h, optimizer, beta1, beta2, eps, dropout, dropout_seed)

    def query(self, what, layer=0):
        return bns_query(self.h, what, layer)

    # typed views
    def counts(self):
        v = np.frombuffer(self.query(BNS_Q_COUNTS), np.int64)
        m = self.world
        return dict(n_in=int(v[0]), n_bd=int(v[1]), n_halo=int(v[2]), n_sent=int(v[3]), nnz=int(v[4]),
                    nnz_kept=int(v[5]), recv=v[6:6 + m].copy(), send=v[6 + m:6 + 2 * m].copy())

    def i32(self, what, layer=0):
        return np.frombuffer(self.query(what, layer), np.int32).copy()

    def i64(self, what, layer=0):
        return np.frombuffer(self.query(what, layer), np.int64).copy()

    def mask(self):
        return np.frombuffer(self.query(BNS_Q_MASK), np.uint8).copy()

    def rows(self, what, layer, d):
        a = np.frombuffer(self.query(what, layer), np.float32)
        return a.reshape(-1, d).copy() if d else a.copy()

    def induced(self, n_in):
        b = self.query(BNS_Q_INDUCED)
        ptr = np.frombuffer(b[: 8 * (n_in + 1)], np.int64).copy()
        col = np.frombuffer(b[8 * (n_in + 1):], np.int32).copy()
        return ptr, col

    def induced_t(self, n_rows):
        """Edge samplers: sampled transposed CSR over rows [inner u ; boundary index b] (n_rows = n_in + n_bd)."""
        b = self.query(BNS_Q_INDUCED_T)
        ptr = np.frombuffer(b[: 8 * (n_rows + 1)], np.int64).copy()
        col = np.frombuffer(b[8 * (n_rows + 1):], np.int32).copy()
        return ptr, col

    def static_csr(self, n_in):
        b = self.query(BNS_Q_STATIC_CSR)
        ptr = np.frombuffer(b[: 8 * (n_in + 1)], np.int64).copy()
        col = np.frombuffer(b[8 * (n_in + 1):], np.int32).copy()
        return ptr, col

    def times(self):
        t = np.frombuffer(self.query(BNS_Q_TIMES), np.float64)
        return dict(zip(PHASES, t.tolist()))

    def tf_layers(self):
        """bit l-1 set <=> layer l runs transform-first (R42)"""
        return int(np.frombuffer(self.query(BNS_Q_TF_LAYERS), np.int32)[0])

    def kernel_count(self):
        return int(np.frombuffer(self.query(BNS_Q_KERNEL_COUNT), np.int64)[0])

    def memory(self):
        v = np.frombuffer(self.query(BNS_Q_MEMORY), np.int64)
        return int(v[0]), int(v[1])

    def stream(self):
        return bns_stream(self.h)
