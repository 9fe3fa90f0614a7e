"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck): every kernel of the epoch runs at least
once -- m = 3 LOCAL transport (staged exchange), m = 2 peer memory (device flag barriers, fused pull / scatter, rank-
order all-reduce over peer pointers), bf16 and fp32, SAGE / GCN / GAT, BNS and BES draws.
    compute-sanitizer --tool memcheck python scripts/sanitize_case.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    from gpu_harness import GpuRun
    from paper_2203_10983_b200 import bns
    from paper_2203_10983_b200 import inputs as I
    indptr, indices = I.rmat(1200, 30000, seed=5)
    cases = [(3, bns.BNS_LAYER_SAGE_MEAN, bns.BNS_BF16, 0), (3, bns.BNS_LAYER_GCN, bns.BNS_FP32, 0),
             (2, bns.BNS_LAYER_SAGE_MEAN, bns.BNS_BF16, bns.BNS_PEER_MEMORY),
             (2, bns.BNS_LAYER_GAT, bns.BNS_FP32, bns.BNS_PEER_MEMORY)]
    for m, layer, prec, extra in cases:
        dims = [24, 16, 16, 5] if layer != bns.BNS_LAYER_GCN else [24, 16, 5]
        part = I.partition(indptr, indices, m, "random")
        X = I.features(np.arange(len(indptr) - 1, dtype=np.int32), dims[0])
        y = I.labels(len(indptr) - 1, dims[-1], 0.7)
        run = GpuRun(indptr, indices, part, m, dims, layer, prec, X, y, flags=bns.BNS_RETAIN_GRADS | extra)
        W = I.weights(dims, layer)
        try:
            run.sample(0.3, I.BNS_SEED, 0)
            _, _, _, W = run.epoch(W, 0.1)
            run.sample_edges(bns.BNS_SAMPLER_BES, 0.3, I.BNS_SEED, 1)
            _, _, _, W = run.epoch([w.astype(np.float32) for w in W], 0.1)
            run.sample(1.0, I.BNS_SEED, 2)
            run.epoch([w.astype(np.float32) for w in W], 0.1)
        finally:
            run.close()
        print("case ok", m, layer, prec, extra, flush=True)


if __name__ == "__main__":
    main()
