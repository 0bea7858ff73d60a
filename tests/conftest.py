import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: longer CPU-side checks")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        return np.load(os.path.join(GOLDEN, name), allow_pickle=False)

    return load


@pytest.fixture(autouse=True)
def _poison_recycled_device_memory(request):
    """ITSK_TEST_POISON=1: before every GPU test, fill a spread of freed device
    blocks (small and large pools of torch's caching allocator) with NaN, so a
    kernel that reads a workspace, pad or output it never initialised sees
    NaN instead of whatever the previous test left there (compute-sanitizer's
    initcheck is closed on this pool).  Results of a clean suite must not
    change: run `ITSK_TEST_POISON=1 python -m pytest tests -m gpu`."""
    if os.environ.get("ITSK_TEST_POISON") != "1" or request.node.get_closest_marker("gpu") is None:
        yield
        return
    import torch

    if torch.cuda.is_available():
        free, _ = torch.cuda.mem_get_info()
        sizes = [1 << k for k in range(9, 31, 1)]  # 512 B .. 1 GiB
        blocks = []
        budget = min(free // 4, 24 << 30)
        for rep in range(3):
            for sz in sizes:
                if budget < sz:
                    continue
                budget -= sz
                blocks.append(torch.full((sz // 8,), float("nan"), dtype=torch.float64, device="cuda"))
        torch.cuda.synchronize()
        del blocks
    yield
