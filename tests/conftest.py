import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: long CPU test")


def parity_log(**rec):
    """Append one JSON record of realized parity errors / tolerances to $IETI_PARITY_LOG (if set), so
    a GPU run leaves the numbers behind (profiles/r02/parity_*.jsonl), not only pass/fail."""
    path = os.environ.get("IETI_PARITY_LOG")
    if not path:
        return
    import json
    with open(path, "a") as fh:
        fh.write(json.dumps(rec, default=float) + "\n")
