import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def parity_log(test, **counts):
    """Record how many cases a parity test actually compared (DESIGN.md §4 quotes these).
    Appends one JSON line to $MPAX_PARITY_LOG when set (the GPU runs point it at
    gpurun_out/), and prints it (visible with pytest -s / -rA)."""
    import json
    conv = lambda v: int(v) if hasattr(v, "__index__") else float(v) if hasattr(v, "__float__") else v  # noqa: E731
    line = json.dumps(dict(test=test, **{k: conv(v) for k, v in counts.items()}))
    print("PARITY", line)
    path = os.environ.get("MPAX_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(line + "\n")
