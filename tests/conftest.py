import os

# Every node has a main + FRC stream and every NCCL edge its own stream:
# give each its own hardware queue (the default 8 would serialise unrelated
# streams behind spinning P2P kernels). Must precede CUDA initialisation.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun)")
    config.addinivalue_line("markers", "slow: long CPU test")


def pytest_sessionstart(session):
    # A fresh checkout has no libbamboo.so (built artefacts are git-ignored):
    # build it once so the ABI-export and GPU tests load the real library.
    lib = os.path.join(ROOT, "paper_2204_12013_b200", "libbamboo.so")
    if not os.path.exists(lib) and "BB_LIB" not in os.environ:
        import __graft_entry__
        __graft_entry__.build()
