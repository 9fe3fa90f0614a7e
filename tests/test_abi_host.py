"""CPU tests of the C-ABI library: it loads, exports every symbol include/bns.h declares, validates its inputs, and
its host plan (a0, BNS_PLAN_ONLY -- no device work) equals the oracle's plan (R24)."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2203_10983_b200 import bns
from paper_2203_10983_b200 import inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(bns.LIB_PATH):
        import subprocess
        subprocess.run(["make", "-C", ROOT, "paper_2203_10983_b200/libbns.so"], check=True)


def header_functions():
    src = open(os.path.join(ROOT, "include", "bns.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bns_[a-z_]+)\s*\(", src)))


def test_exports_every_header_symbol():
    L = bns.lib()
    names = header_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(bns.EXPORTS)


def plan_ctx(indptr, indices, part, m, rank, dims=(4, 3), layer=0, labels=None):
    n_in = int((part == rank).sum())
    X = np.zeros((n_in, dims[0]), np.float32)
    y = np.zeros(n_in, np.int32) if labels is None else labels
    return bns.Context(rank=rank, world=m, dims=list(dims), layer=layer, precision=bns.BNS_FP32, indptr=indptr,
                       indices=indices, part_of=part, features=X, labels=y, flags=bns.BNS_PLAN_ONLY)


@pytest.mark.parametrize("seed,N,m", [(1, 40, 2), (2, 120, 3), (3, 300, 5), (4, 64, 1), (5, 500, 8)])
def test_plan_matches_oracle(seed, N, m):
    indptr, indices = I.rmat(N, 8 * N, seed=seed)
    part = I.partition(indptr, indices, m, "random" if seed % 2 else "ldg2")
    orc = O.Oracle(indptr, indices, part, m, [1, 1], 0, np.zeros((N, 1), np.float32), np.zeros(N, np.int32))
    for r in range(m):
        c = plan_ctx(indptr, indices, part, m, r)
        assert list(c.i32(bns.BNS_Q_INNER)) == list(orc.list(O.V_LIST, r))
        assert list(c.i32(bns.BNS_Q_BOUNDARY)) == list(orc.list(O.B_LIST, r))
        assert list(c.i64(bns.BNS_Q_BOUNDARY_OFF)) == list(orc.list(O.B_OFF, r))
        D = c.i32(bns.BNS_Q_SENDCAND)
        Doff = c.i64(bns.BNS_Q_SENDCAND_OFF)
        for j in range(m):
            assert list(D[Doff[j]:Doff[j + 1]]) == list(orc.list(O.D_LIST, r, j))
        # static CSR: full rows of the inner nodes in global order, boundary columns encoded -(b+1)
        V = c.i32(bns.BNS_Q_INNER)
        B = c.i32(bns.BNS_Q_BOUNDARY)
        ptr, col = c.static_csr(len(V))
        for k, v in enumerate(V):
            row = col[ptr[k]:ptr[k + 1]]
            g = [int(V[x]) if x >= 0 else int(B[-x - 1]) for x in row]
            assert g == list(indices[indptr[v]:indptr[v + 1]])
        c.close()


def test_invalid_inputs():
    indptr, indices = I.csr_from_edges(4, [(0, 1), (1, 2), (2, 3)])
    part = np.array([0, 0, 1, 1], np.int32)
    with pytest.raises(bns.BnsError) as e:   # empty partition
        plan_ctx(indptr, indices, np.array([0, 0, 0, 0], np.int32), 2, 0)
    assert e.value.code == bns.BNS_ERR_INVALID and "empty" in str(e.value)
    with pytest.raises(bns.BnsError) as e:   # part id out of range
        plan_ctx(indptr, indices, np.array([0, 0, 2, 1], np.int32), 2, 0)
    assert e.value.code == bns.BNS_ERR_INVALID
    bad = indices.copy()
    bad[0] = 0                               # self loop on node 0
    with pytest.raises(bns.BnsError) as e:
        plan_ctx(indptr, bad, part, 2, 0)
    assert "self loop" in str(e.value)
    bad = indices.copy()
    bad[1], bad[2] = bad[2], bad[1]          # row 1 unsorted
    with pytest.raises(bns.BnsError):
        plan_ctx(indptr, bad, part, 2, 0)
    with pytest.raises(bns.BnsError):        # label >= C
        plan_ctx(indptr, indices, part, 2, 0, dims=(4, 3), labels=np.array([0, 3], np.int32))
    with pytest.raises(bns.BnsError):        # rank >= world
        plan_ctx(indptr, indices, part, 2, 2)
    # asymmetric CSR (bns.h: "symmetric"): arc 3 -> 2 removed, 2 -> 3 kept -- D_{i->j} = B_j ∩ V_i would be wrong
    ip = np.array([0, 1, 3, 5, 5], np.int64)
    ix = np.array([1, 0, 2, 1, 3], np.int32)
    with pytest.raises(bns.BnsError) as e:
        plan_ctx(ip, ix, part, 2, 0)
    assert e.value.code == bns.BNS_ERR_INVALID and "symmetric" in str(e.value)


def test_plan_only_rejects_device_calls():
    indptr, indices = I.csr_from_edges(4, [(0, 1), (1, 2), (2, 3)])
    c = plan_ctx(indptr, indices, np.array([0, 0, 1, 1], np.int32), 2, 0)
    with pytest.raises(bns.BnsError) as e:
        c.sample_boundary(0.5, 1, 0)
    assert e.value.code == bns.BNS_ERR_STATE
    w = [np.zeros((8, 3), np.float32)]
    with pytest.raises(bns.BnsError) as e:
        c.epoch(w, 0.1)
    assert e.value.code == bns.BNS_ERR_STATE
    with pytest.raises(bns.BnsError) as e:
        c.step(0.5, 1, 0, w, 0.1)
    assert e.value.code == bns.BNS_ERR_STATE
    with pytest.raises(bns.BnsError) as e:
        c.set_timing(True)
    assert e.value.code == bns.BNS_ERR_STATE
    c.close()


def test_ipc_transport_needs_allgather():
    indptr, indices = I.csr_from_edges(4, [(0, 1), (1, 2), (2, 3)])
    part = np.array([0, 0, 1, 1], np.int32)
    with pytest.raises(bns.BnsError) as e:
        bns.Context(rank=0, world=2, dims=[1, 2], layer=0, precision=bns.BNS_FP32, indptr=indptr, indices=indices,
                    part_of=part, features=np.zeros((2, 1), np.float32), labels=np.zeros(2, np.int32),
                    transport=bns.BNS_TRANSPORT_IPC)
    assert e.value.code == bns.BNS_ERR_INVALID and "allgather" in str(e.value)


def test_eq3_identity_through_library_plan():
    # Σ_i |B_i| (library) == Σ_{i,j} |D_{i->j}| (library) == Σ_v D(v) edge-wise
    indptr, indices = I.rmat(400, 4000, seed=9)
    part = I.partition(indptr, indices, 4, "ldg2")
    tot_b = tot_d = 0
    for r in range(4):
        c = plan_ctx(indptr, indices, part, 4, r)
        cnt = c.i32(bns.BNS_Q_BOUNDARY)
        tot_b += len(cnt)
        tot_d += len(c.i32(bns.BNS_Q_SENDCAND))
        c.close()
    Dv = sum(len({int(part[u]) for u in indices[indptr[v]:indptr[v + 1]]} - {int(part[v])}) for v in range(400))
    assert tot_b == tot_d == Dv
