"""Debug: bf16 transform-first (R42) vs the oracle's emulation, per tensor, with ReLU flip counts."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from oracle import oracle as O
from paper_2203_10983_b200 import bns
from paper_2203_10983_b200 import inputs as I
from gpu_harness import GpuRun, relerr
from test_gpu_parity import wl

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dims = [37, 24, 16, 5]
indptr, indices, part, X, y = wl(3000, 90000, m, dims[0], dims[-1], 41 + m, "random")
for tfflag in (0, bns.BNS_NO_TRANSFORM_FIRST):
    for prec in (0, 1):
        Ws = I.weights(dims, 0)
        Wd = [w.astype(np.float64) for w in Ws]
        run = GpuRun(indptr, indices, part, m, dims, 0, prec, X, y, flags=bns.BNS_RETAIN_GRADS | tfflag)
        orc = O.Oracle(indptr, indices, part, m, dims, 0, X, y)
        orc.set_bf16(prec == 1)
        orc.set_transform_first(run.tf)
        run.sample(0.5, I.BNS_SEED, 0); orc.sample(0.5, I.BNS_SEED, 0)
        loss, acc, G, Wn = run.epoch(Ws, 0.5)
        lo, ao, Go = orc.epoch(Wd, 0.5)
        out = {"loss": abs(loss - lo) / abs(lo)}
        for l in range(1, 4):
            g = run.gather(bns.BNS_Q_H, l, dims[l]); o = orc.tensor(O.T_H, l)
            out[f"H{l}"] = relerr(g, o)
            if l < 3:
                out[f"flips{l}"] = int(((g > 0) != (o > 0)).sum())
            out[f"dH{l}"] = relerr(run.gather(bns.BNS_Q_DH, l, dims[l]), orc.tensor(O.T_DH, l))
        for l in range(3):
            out[f"dW{l}"] = relerr(G[l], Go[l])
            # top / bottom halves separately
            d = dims[l]
            out[f"dW{l}top"] = relerr(G[l][:d], Go[l][:d]); out[f"dW{l}bot"] = relerr(G[l][d:], Go[l][d:])
        print("tf" if tfflag == 0 else "noTF", "bf16" if prec else "fp32", {k: (round(v, 5) if isinstance(v, float) else v) for k, v in out.items()})
        run.close()
