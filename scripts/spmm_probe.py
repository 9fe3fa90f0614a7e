"""Probe: SpMM time on the Reddit shape for an R-MAT graph vs a uniform random graph of the same N / nnz / widths
(is the gather limited by hot L2 slices from hub rows?).  Prints one JSON line per graph."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2203_10983_b200 import bns
    from paper_2203_10983_b200 import inputs as I
    sh = I.SHAPES["reddit"]
    for name, abc in (("rmat", (0.57, 0.19, 0.19)), ("uniform", (0.25, 0.25, 0.25))):
        indptr, indices = I.rmat(sh.N, sh.nnz, abc=abc)
        X = I.features(np.arange(sh.N, dtype=np.int32), sh.d0)
        y = I.labels(sh.N, sh.C, sh.train_frac)
        ctx = bns.Context(rank=0, world=1, dims=sh.dims, layer=sh.layer, precision=bns.BNS_BF16, indptr=indptr,
                          indices=indices, part_of=np.zeros(sh.N, np.int32), features=X, labels=y,
                          flags=bns.BNS_TIMING)
        W = [torch.tensor(w, device="cuda") for w in I.weights(sh.dims, sh.layer)]
        G = [torch.zeros_like(w) for w in W]
        for e in range(3):
            ctx.sample_boundary(0.1, 1, e)
            ctx.epoch(W, 0.0, G)
        t0 = ctx.times()
        for e in range(5):
            ctx.sample_boundary(0.1, 1, 10 + e)
            ctx.epoch(W, 0.0, G)
        t1 = ctx.times()
        ph = {k: round((t1[k] - t0[k]) / 5, 3) for k in t1 if t1[k] > t0[k]}
        deg = np.diff(indptr)
        print(json.dumps({"graph": name, "nnz": int(indptr[-1]), "max_deg": int(deg.max()), "phases_ms": ph}), flush=True)
        ctx.close()
        del indptr, indices, X


if __name__ == "__main__":
    main()
