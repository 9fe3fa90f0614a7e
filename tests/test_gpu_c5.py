"""C5 (BASELINE.json configs[4], papers100M-shaped: 111 M nodes, 1.6 B arcs, SAGE 3 x 128, m = 8, p = 0.01;
PAPER.md:549-563): one rank of the 8-partition job on one B200 -- keep masks / U_i / S_{i,j} bit-exact against the
oracle's plan + sample, 1,000 spot rows of H^1 against float64 from raw neighbours (scripts/c5_papers.py)."""
import os
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))


def test_c5_papers100m_rank0():
    import json

    import c5_papers
    rec = c5_papers.run(ranks=(0,), steps=3, warmup=1)[0]
    assert rec["spot_rows"] >= 1000 and rec["spot_relerr_H1"] < 2e-2
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "c5_papers_rank0.json"), "w") as f:
        json.dump(rec, f, indent=1)
