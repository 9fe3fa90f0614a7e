"""Oracle pins for the plan (Eq. 3): SPEC hand examples and the Eq. 3 identity
computed by an independent edge-wise path."""
import numpy as np

from oracle import oracle as O
from paper_2203_10983_b200 import inputs as I


def mk(N, edges, part, m, layer=0):
    ip, ix = I.csr_from_edges(N, edges)
    X = np.ones((N, 1), np.float32)
    y = np.zeros(N, np.int32)
    return O.Oracle(ip, ix, np.array(part, np.int32), m, [1, 1], layer, X, y)


def test_p4_plan():
    o = mk(4, [(0, 1), (1, 2), (2, 3)], [0, 0, 1, 1], 2)
    assert list(o.list(O.V_LIST, 0)) == [0, 1] and list(o.list(O.V_LIST, 1)) == [2, 3]
    assert list(o.list(O.B_LIST, 0)) == [2] and list(o.list(O.B_LIST, 1)) == [1]
    assert list(o.list(O.D_LIST, 0, 1)) == [1] and list(o.list(O.D_LIST, 1, 0)) == [2]


def test_m1_no_boundary():
    o = mk(4, [(0, 1), (1, 2), (2, 3)], [0, 0, 0, 0], 1)
    assert len(o.list(O.B_LIST, 0)) == 0


def test_star_plan():  # K1,5 centre in part 0
    o = mk(6, [(0, k) for k in range(1, 6)], [0, 1, 1, 1, 1, 1], 2)
    assert list(o.list(O.B_LIST, 0)) == [1, 2, 3, 4, 5]
    assert list(o.list(O.B_LIST, 1)) == [0]
    assert len(o.list(O.B_LIST, 0)) + len(o.list(O.B_LIST, 1)) == 6   # Eq. 3 total


def test_boundary_order_owner_major():
    ip, ix = I.rmat(300, 2400, seed=5)
    part = I.partition(ip, ix, 4, "random")
    o = O.Oracle(ip, ix, part, 4, [1, 1], 0, np.ones((300, 1), np.float32), np.zeros(300, np.int32))
    for i in range(4):
        B = o.list(O.B_LIST, i)
        off = o.list(O.B_OFF, i)
        keys = [(part[u], u) for u in B]
        assert keys == sorted(keys)
        for j in range(4):
            assert all(part[u] == j for u in B[off[j]:off[j + 1]])


def test_eq3_identity_random_instances():
    # Σ_i |B_i| (boundary sets) == Σ_v D(v) (edge-wise count of other partitions v touches)
    rng = np.random.default_rng(0)
    for t in range(25):
        N = int(rng.integers(10, 80))
        m = int(rng.integers(1, 6))
        ip, ix = I.rmat(N, int(N * rng.integers(2, 8)), seed=100 + t)
        part = rng.integers(0, m, N).astype(np.int32)
        o = O.Oracle(ip, ix, part, m, [1, 1], 0, np.ones((N, 1), np.float32), np.zeros(N, np.int32))
        total_B = sum(len(o.list(O.B_LIST, i)) for i in range(m))
        Dv = 0
        for v in range(N):
            Dv += len({int(part[u]) for u in ix[ip[v]:ip[v + 1]]} - {int(part[v])})
        assert total_B == Dv
        # and the send-candidate lists carry the same total (sent == received)
        assert sum(len(o.list(O.D_LIST, i, j)) for i in range(m) for j in range(m) if i != j) == total_B
