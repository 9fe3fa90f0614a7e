import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libbns.so on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running statistical / large-size test")
    # the oracle and the input generators are cheap host builds; make sure they exist
    need = [os.path.join(ROOT, "oracle", "liboracle.so"),
            os.path.join(ROOT, "paper_2203_10983_b200", "inputs", "libbnsgen.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-C", ROOT, "oracle/liboracle.so", "paper_2203_10983_b200/inputs/libbnsgen.so"],
                       check=True, stdout=subprocess.DEVNULL)


def pytest_terminal_summary(terminalreporter):
    """bf16 epoch parity report (tests/gpu_harness.py): how many epochs had ReLU flips against the float64 oracle
    (F > 0) and the worst margins, written to gpurun_out/bf16_margins.json for DESIGN.md's measured-gap table."""
    try:
        from gpu_harness import BF16_REPORT
    except Exception:  # noqa: BLE001
        return
    if not BF16_REPORT:
        return
    import json
    n = len(BF16_REPORT)
    nf = sum(1 for r in BF16_REPORT if r["F"] > 0)
    share = max((f / u for r in BF16_REPORT for f, u in zip(r["flips"], r["units"])), default=0.0)
    worst = {}
    for r in BF16_REPORT:
        for part in ("vs_float64", "layer_local"):
            for k, v in r.get(part, {}).items():
                worst[f"{part}:{k}"] = max(worst.get(f"{part}:{k}", 0.0), v)
    terminalreporter.write_line(f"bf16 epochs compared: {n}; with ReLU flips vs float64 (F > 0): {nf}; "
                                f"largest flipped share of a layer's units: {share:.2e}")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "bf16_margins.json"), "w") as f:
        json.dump({"epochs": n, "epochs_with_flips": nf, "max_flip_share": share, "worst": worst,
                   "records": BF16_REPORT}, f, indent=1)
