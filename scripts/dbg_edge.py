"""Debug: BES at m=1 must equal BNS at m=1 bitwise; print per-tensor errors vs the oracle for both."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from oracle import oracle as O
from paper_2203_10983_b200 import bns
from paper_2203_10983_b200 import inputs as I
from gpu_harness import GpuRun, relerr
from test_gpu_parity import wl

prec = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
m = 1
dims = [37, 24, 16, 5]
indptr, indices, part, X, y = wl(3000, 90000, m, dims[0], dims[-1], 41 + m, "random")
out = {}
for mode in ("bns", "bes"):
    Ws = I.weights(dims, 0)
    Wd = [w.astype(np.float64) for w in Ws]
    run = GpuRun(indptr, indices, part, m, dims, 0, prec, X, y)
    orc = O.Oracle(indptr, indices, part, m, dims, 0, X, y)
    orc.set_bf16(prec == 1)
    for e in range(2):
        if mode == "bns":
            run.sample(0.5, I.BNS_SEED, e); orc.sample(0.5, I.BNS_SEED, e)
        else:
            run.ctx[0].sample_edges(1, 0.5, I.BNS_SEED, e); orc.sample_edges(1, 0.5, I.BNS_SEED, e)
        loss, acc, G, Wn = run.epoch(Ws, lr)
        lo, ao, Go = orc.epoch(Wd, lr)
        errs = {}
        for l in range(1, 4):
            errs[f"Z{l}"] = relerr(run.gather(bns.BNS_Q_Z, l, dims[l - 1]), orc.tensor(O.T_Z, l))
            errs[f"H{l}"] = relerr(run.gather(bns.BNS_Q_H, l, dims[l]), orc.tensor(O.T_H, l))
            errs[f"dH{l}"] = relerr(run.gather(bns.BNS_Q_DH, l, dims[l]), orc.tensor(O.T_DH, l))
        print(mode, e, loss, lo, {k: round(v, 5) for k, v in errs.items()})
        out[(mode, e)] = [run.gather(bns.BNS_Q_DH, l, dims[l]) for l in range(1, 4)]
        Ws = [w.astype(np.float32) for w in Wn]
    run.close()
for e in range(2):
    print("bitwise equal epoch", e, all(np.array_equal(a, b) for a, b in zip(out[("bns", e)], out[("bes", e)])))
