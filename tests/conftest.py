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
