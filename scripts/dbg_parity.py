import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', 'tests'))
import numpy as np
from oracle import oracle as O
from paper_2203_10983_b200 import bns, inputs as I
from gpu_harness import GpuRun, relerr
layer = int(sys.argv[1]) if len(sys.argv) > 1 else 0
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
dims = [37, 24, 16, 5] if layer == 0 else [37, 16, 5]
N, nnz = 3000, 90000
indptr, indices = I.rmat(N, nnz, seed=21 + m)
part = I.partition(indptr, indices, m, "random")
X = I.features(np.arange(N, dtype=np.int32), dims[0]); y = I.labels(N, dims[-1], 0.7, seed=28 + m)
L = len(dims) - 1
deg = np.diff(indptr)
for prec in (0, 1):
    Ws = I.weights(dims, layer); Wd = [w.astype(np.float64) for w in Ws]
    run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y)
    orc = O.Oracle(indptr, indices, part, m, dims, layer, X, y)
    run.sample(p, 5, 0); orc.sample(p, 5, 0)
    loss, acc, G, Wn = run.epoch(Ws, 0.5); lo, ao, Go = orc.epoch(Wd, 0.5)
    print("prec", prec, "loss", loss, lo, "acc", acc, ao)
    for l in range(1, L + 1):
        for nm, q, t, d in (("Z", bns.BNS_Q_Z, O.T_Z, dims[l-1]), ("H", bns.BNS_Q_H, O.T_H, dims[l]), ("dH", bns.BNS_Q_DH, O.T_DH, dims[l])):
            a = run.gather(q, l, d); b = orc.tensor(t, l)
            err = np.abs(a - b).max(1)
            worst = np.argsort(-err)[:3]
            print(f"  l={l} {nm:2s} relerr={relerr(a,b):.3e} max|b|={np.abs(b).max():.3e} worst rows {worst} deg {deg[worst]} err {err[worst]}")
    for l in range(L):
        print(f"  dW{l} relerr={relerr(G[l], Go[l]):.3e}")
    run.close()
