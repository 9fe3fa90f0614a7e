"""A/B probe: per-phase ms of the Reddit-shaped m=1 bf16 epoch under the current environment (BNS_* knobs).
Usage: BNS_SPMM_N6=0 python scripts/ab_env.py tag"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2203_10983_b200 import bns
    from paper_2203_10983_b200 import inputs as I
    sh = I.SHAPES[os.environ.get("AB_CONFIG", "reddit")]
    indptr, indices = I.rmat(sh.N, sh.nnz)
    X = I.features(np.arange(sh.N, dtype=np.int32), sh.d0)
    y = I.labels(sh.N, sh.C, sh.train_frac)
    ctx = bns.Context(rank=0, world=1, dims=sh.dims, layer=sh.layer, precision=bns.BNS_BF16, indptr=indptr,
                      indices=indices, part_of=np.zeros(sh.N, np.int32), features=X, labels=y, flags=bns.BNS_TIMING)
    W = [torch.tensor(w, device="cuda") for w in I.weights(sh.dims, sh.layer)]
    G = [torch.zeros_like(w) for w in W]
    for e in range(3):
        ctx.sample_boundary(0.1, 1, e)
        ctx.epoch(W, 0.0, G)
    t0 = ctx.times()
    n = 8
    for e in range(n):
        ctx.sample_boundary(0.1, 1, 10 + e)
        loss, _ = ctx.epoch(W, 0.0, G)
    t1 = ctx.times()
    ph = {k: round((t1[k] - t0[k]) / n, 3) for k in t1 if t1[k] > t0[k]}
    print(json.dumps({"tag": sys.argv[1] if len(sys.argv) > 1 else "", "env": {k: v for k, v in os.environ.items()
                      if k.startswith("BNS_")}, "loss": loss, "phases_ms": ph}), flush=True)


main()
