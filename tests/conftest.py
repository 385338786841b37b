import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); run with -m gpu")


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(autouse=True)
def _band_width_under_test(monkeypatch):
    """SKV_TEST_BAND_LOG2=n (set by test_step_kernel_selection_paths_subprocess for its child pytest):
    every context the tests create ranks with a selection band of width 2^n (sentencekv_set_band_log2),
    so that narrow or very wide bands drive the step kernel through mode 2, the general path and list
    overflows.  A test hook: the library itself reads no environment."""
    n = os.environ.get("SKV_TEST_BAND_LOG2")
    if n is None:
        yield
        return
    import paper_2504_00970_b200 as skvlib

    init = skvlib.SentenceKV.__init__

    def patched(self, *a, **kw):
        init(self, *a, **kw)
        self.set_band_log2(int(n))

    monkeypatch.setattr(skvlib.SentenceKV, "__init__", patched)
    yield
