import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def _fill_device_garbage(torch):
    """Fill most free device memory with 0xFF bytes and hand it back to the driver, so every
    later allocation starts from garbage: a buffer read before it is written, or a copy not
    ordered with its consumer, then fails loudly instead of passing on stale-but-right data
    (this caught a stage-ring race and a legacy-stream memset race)."""
    free, _ = torch.cuda.mem_get_info()
    blocks = []
    try:
        for _ in range(int(free * 0.8) // (4 << 30)):
            t = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
            t.fill_(0xFF)
            blocks.append(t)
    except RuntimeError:
        pass
    torch.cuda.synchronize()
    del blocks
    torch.cuda.empty_cache()


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test scheduled on a host without a visible CUDA device")
    if os.environ.get("REATTN_TEST_NO_GARBAGE") is None:
        _fill_device_garbage(torch)
    from paper_2407_15176_b200 import native
    c = native.Context(0)
    yield c
