import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size configs (minutes)")
    # Build the in-tree native libraries once per session (no-op when up to date).
    targets = ["gen/libsymmgen.so", "oracle/liboracle.so"]
    if os.path.exists(os.path.join(ROOT, "paper_1907_06487_b200", "csrc", "kernels.cu")):
        targets.append("paper_1907_06487_b200/libsymmspmv.so")
    r = subprocess.run(["make", "-s", "-C", ROOT] + targets, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("native build failed:\n" + r.stdout[-4000:] + r.stderr[-4000:])


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
