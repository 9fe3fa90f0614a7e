"""R48 (BNS_PREFETCH_DRAW): bns_step(p, seed, e) enqueues the draw of (p, seed, e + 1) after its update kernels and
before its closing sync, so the next step starts its epoch without a host wait for the per-peer counts.

Pins (the draw kernels and the epoch are unchanged, so nothing may move by one bit):
  * a run of steps with the flag gives bitwise the losses, gradients and weights of the same steps without it -- m = 1
    and m = 3 (LOCAL staged and peer-memory transports), fp32 and bf16, including steps whose arguments do not match
    the prefetch (p changes, seed changes, an epoch skipped), which must discard it and draw afresh;
  * after a step the context's draw is the prefetched one: its keep mask and U_i equal the oracle's draw of epoch
    e + 1 (the header's documented behaviour);
  * bns_epoch called right after a prefetching step trains on that draw (bitwise a fresh sample + epoch).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2203_10983_b200 import bns
from paper_2203_10983_b200 import inputs as I

from gpu_harness import GpuRun, parallel
from test_gpu_parity import wl

pytestmark = pytest.mark.gpu
SEED = I.BNS_SEED
SEQ = [(0.1, SEED, 0), (0.1, SEED, 1), (0.1, SEED, 2), (0.3, SEED, 3), (0.3, SEED, 4), (0.3, SEED + 1, 5),
       (0.3, SEED + 1, 7), (0.3, SEED + 1, 8)]


def steps(run, Ws, seq, lr=0.3):
    import torch
    m = run.m
    W = [[torch.tensor(w, device="cuda") for w in Ws] for _ in range(m)]
    G = [[torch.zeros_like(w) for w in W[0]] for _ in range(m)]
    rec = []
    for p, s, e in seq:
        out = parallel(m, lambda r: run.ctx[r].step(p, s, e, W[r], lr, G[r]))
        torch.cuda.synchronize()
        assert all(o == out[0] for o in out)
        rec.append((out[0], [g.cpu().numpy().copy() for g in G[0]], [w.cpu().numpy().copy() for w in W[0]]))
    return rec, W, G


@pytest.mark.parametrize("m,prec,extra", [(1, bns.BNS_FP32, 0), (3, bns.BNS_BF16, 0),
                                          (3, bns.BNS_BF16, bns.BNS_PEER_MEMORY), (3, bns.BNS_FP32, 0)])
def test_prefetch_bitwise_and_current_draw(m, prec, extra):
    indptr, indices, part, X, y = wl(1500, 30000, m, 24, 5, 41, "random")
    dims = [24, 32, 5]
    Ws = I.weights(dims, bns.BNS_LAYER_SAGE_MEAN)
    a = GpuRun(indptr, indices, part, m, dims, bns.BNS_LAYER_SAGE_MEAN, prec, X, y, flags=extra)
    b = GpuRun(indptr, indices, part, m, dims, bns.BNS_LAYER_SAGE_MEAN, prec, X, y, flags=extra | bns.BNS_PREFETCH_DRAW)
    try:
        ra, _, _ = steps(a, Ws, SEQ)
        rb, Wb, Gb = steps(b, Ws, SEQ)
        for k, (x, z) in enumerate(zip(ra, rb)):
            assert x[0] == z[0], (k, x[0], z[0])
            for u, v in zip(x[1] + x[2], z[1] + z[2]):
                assert np.array_equal(u, v), k
        # the prefetching context now holds the draw of (0.3, SEED + 1, 9)
        orc = O.Oracle(indptr, indices, part, m, [1, 1], 0, np.zeros((len(indptr) - 1, 1), np.float32),
                       np.zeros(len(indptr) - 1, np.int32))
        orc.sample(0.3, SEED + 1, 9)
        for r in range(m):
            assert np.array_equal(b.ctx[r].mask(), orc.list(O.KEEP, r).astype(np.uint8)), r
            assert np.array_equal(b.ctx[r].i32(bns.BNS_Q_HALO), orc.list(O.U_LIST, r)), r
        # bns_epoch right after a prefetching step trains on that draw
        import torch
        Wa = [[w.clone() for w in Wb[0]] for _ in range(m)]
        Ga = [[torch.zeros_like(w) for w in Wa[0]] for _ in range(m)]
        a.sample(0.3, SEED + 1, 9)
        oa = parallel(m, lambda r: a.ctx[r].epoch(Wa[r], 0.3, Ga[r]))
        ob = parallel(m, lambda r: b.ctx[r].epoch(Wb[r], 0.3, Gb[r]))
        torch.cuda.synchronize()
        assert oa[0] == ob[0]
        for u, v in zip(Wa[0] + Ga[0], Wb[0] + Gb[0]):
            assert torch.equal(u, v)
    finally:
        a.close()
        b.close()
