import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: multi-second CPU oracle runs")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        return np.load(os.path.join(GOLDEN, name))
    return load

TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


@pytest.fixture(scope="session")
def P():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_09907_b200.multigrid as mg
    import paper_1705_09907_b200.problem as pb
    import paper_1705_09907_b200.trace as tr
    from paper_1705_09907_b200.mesh import build_cartesian

    class NS:
        pass
    ns = NS()
    ns.mg, ns.pb, ns.tr, ns.mesh = mg, pb, tr, build_cartesian
    from paper_1705_09907_b200._lib import check, lib
    ns.lib, ns.lib_check = lib, check
    return ns
