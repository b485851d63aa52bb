import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "reference: needs /root/reference importable (dev container only)")


REFERENCE_SRC = os.environ.get("PK_REFERENCE_SRC", "/root/reference/pkg/src")


def reference_available() -> bool:
    return Path(REFERENCE_SRC, "pipekrylov", "__init__.py").exists()
