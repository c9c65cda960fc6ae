import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def toy_arrays():
    """(node_ids, src, dst, t) for the Fig.-1 toy graph, ids by first appearance."""
    from paper_2204_09236_b200 import parse_edge_list
    g = parse_edge_list(open(os.path.join(GOLDEN, "toy.txt")).read())
    return g


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def tm():
    import paper_2204_09236_b200 as tm
    return tm


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not has_cuda():
        pytest.skip("no CUDA device")
    import torch
    torch.cuda.set_device(0)
    return True
