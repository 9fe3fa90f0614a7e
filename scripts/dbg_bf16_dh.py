"""Debug: where does the bf16 dH^1 error of the m=1 seed-42 case come from (epoch 1)?"""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from oracle import oracle as O
from paper_2203_10983_b200 import bns
from paper_2203_10983_b200 import inputs as I
from gpu_harness import GpuRun, relerr
from test_gpu_parity import wl

m, dims, lr = 1, [37, 24, 16, 5], 0.5
indptr, indices, part, X, y = wl(3000, 90000, m, dims[0], dims[-1], 42, "random")
deg = np.diff(indptr)
Ws = I.weights(dims, 0)
Wd = [w.astype(np.float64) for w in Ws]
run = GpuRun(indptr, indices, part, m, dims, 0, 1, X, y)
orc = O.Oracle(indptr, indices, part, m, dims, 0, X, y)
orc.set_bf16(True)
for e in range(2):
    run.sample(0.5, I.BNS_SEED, e); orc.sample(0.5, I.BNS_SEED, e)
    loss, acc, G, Wn = run.epoch(Ws, lr)
    lo, ao, Go = orc.epoch(Wd, lr)
    Ws = [w.astype(np.float32) for w in Wn]
    print("epoch", e, "W relerr", [relerr(a, b) for a, b in zip(Wn, Wd)])
    for l in (1, 2, 3):
        g = run.gather(bns.BNS_Q_DH, l, dims[l]); o = orc.tensor(O.T_DH, l)
        d = np.abs(g - o); i = np.unravel_index(np.argmax(d), d.shape)
        print(f" dH{l}: relerr {relerr(g, o):.4g} max|ref| {np.abs(o).max():.4g} at {np.unravel_index(np.argmax(np.abs(o)), o.shape)} "
              f"maxdiff {d.max():.4g} at {i} gpu {g[i]:.5g} orc {o[i]:.5g} deg {deg[i[0]]}")
    for l in (1, 2):
        g = run.gather(bns.BNS_Q_H, l, dims[l]); o = orc.tensor(O.T_H, l)
        flips = np.argwhere((g > 0) != (o > 0))
        print(f" H{l} relu flips {len(flips)}", [(int(r), int(c), float(g[r, c]), float(o[r, c])) for r, c in flips[:5]])
run.close()
