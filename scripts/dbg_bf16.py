import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', 'tests'))
import numpy as np, torch
from oracle import oracle as O
from paper_2203_10983_b200 import bns, inputs as I
from gpu_harness import GpuRun, relerr
def fro(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
dims = [37, 24, 16, 5]; N, nnz, m = 3000, 90000, 1
indptr, indices = I.rmat(N, nnz, seed=22)
part = I.partition(indptr, indices, m, "random")
X = I.features(np.arange(N, dtype=np.int32), dims[0]); y = I.labels(N, dims[-1], 0.7, seed=29)
for rounded in (False, True):
    Ws = I.weights(dims, 0)
    if rounded: Ws = [torch.tensor(w).bfloat16().float().numpy() for w in Ws]
    Wd = [w.astype(np.float64) for w in Ws]
    run = GpuRun(indptr, indices, part, m, dims, 0, 1, X, y)
    orc = O.Oracle(indptr, indices, part, m, dims, 0, X, y)
    run.sample(1.0, 5, 0); orc.sample(1.0, 5, 0)
    loss, acc, G, Wn = run.epoch(Ws, 0.5); lo, ao, Go = orc.epoch(Wd, 0.5)
    print("rounded", rounded, "loss", loss, lo)
    for l in (1, 2, 3):
        a = run.gather(bns.BNS_Q_H, l, dims[l]); b = orc.tensor(O.T_H, l)
        if l < 3: print(f"  l={l} mask flips {int(((a > 0) != (b > 0)).sum())} / {a.size}")
        for nm, q, t, d in (("H", bns.BNS_Q_H, O.T_H, dims[l]), ("dH", bns.BNS_Q_DH, O.T_DH, dims[l])):
            a = run.gather(q, l, d); b = orc.tensor(t, l)
            print(f"  l={l} {nm:2s} max-rel={relerr(a,b):.3e} fro-rel={fro(a,b):.3e}")
    for l in range(3): print(f"  dW{l} max-rel={relerr(G[l], Go[l]):.3e} fro-rel={fro(G[l], Go[l]):.3e}")
    run.close()
