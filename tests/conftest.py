import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    # GPU tests are never auto-skipped: on the B200 box a missing device or a
    # missing extension must fail, not pass silently.
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
