"""A/B variant of the aggregation (a6 / a10, PAPER.md:100 / :287): rows staged through shared memory by TMA
tile::gather4 (BNS_SPMM_TMA=1, bf16 rows of 256 elements) must give BITWISE the results of the register-gather
SpMM it replaces (same segments, same per-lane edge order, same arithmetic) -- forward (aggregate-first and
transform-first), backward, hub rows split into segments, several partitions."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r'''
import sys, json, hashlib
sys.path[:0] = [%r, %r]
import numpy as np
from gpu_harness import GpuRun
from paper_2203_10983_b200 import bns, inputs as I
indptr, indices = I.rmat(6000, 400000, seed=41)
out = {}
for m, flags in ((1, bns.BNS_RETAIN_GRADS), (3, bns.BNS_RETAIN_GRADS), (3, bns.BNS_RETAIN_GRADS | bns.BNS_NO_TRANSFORM_FIRST)):
    dims = [256, 256, 256, 16]
    part = I.partition(indptr, indices, m, "random")
    X = I.features(np.arange(6000, dtype=np.int32), 256)
    y = I.labels(6000, 16, 0.7)
    run = GpuRun(indptr, indices, part, m, dims, 0, bns.BNS_BF16, X, y, flags=flags)
    W = I.weights(dims, 0)
    h = hashlib.sha256()
    try:
        for e in range(2):
            run.sample(0.3, I.BNS_SEED, e)
            loss, acc, G, W = run.epoch(W, 0.1)
            W = [w.astype(np.float32) for w in W]
            h.update(np.float64(loss).tobytes())
            for g in G: h.update(g.tobytes())
            for l in range(1, 4):
                h.update(run.gather(bns.BNS_Q_H, l, dims[l]).tobytes())
                h.update(run.gather(bns.BNS_Q_DH, l, dims[l]).tobytes())
    finally:
        run.close()
    out["%%d-%%d" %% (m, flags)] = h.hexdigest()
print(json.dumps(out))
''' % (ROOT, os.path.join(ROOT, "tests"))


def run(env):
    r = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, **env))
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_tma_gather4_spmm_is_bitwise_the_register_gather():
    a = run({"BNS_SPMM_TMA": "0"})
    b = run({"BNS_SPMM_TMA": "1"})
    assert a == b
