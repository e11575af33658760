import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    # GPU tests are never auto-skipped: on a box without a GPU run -m "not gpu".
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
