import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built libdfx.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden_input(dims, seed):
    """Inputs of tests/golden/make_golden.py: N(0,1) fp32 from default_rng(seed)."""
    n = int(np.prod(dims))
    return np.random.default_rng(seed).standard_normal(n).astype(np.float32)


def corpus_models():
    from paper_2410_21120_b200 import model_io
    out = []
    for i in range(200):
        g = model_io.load_graph(GOLDEN / "models" / f"rm{i:03d}.graph.json")
        w = model_io.load_weights(GOLDEN / "models" / f"rm{i:03d}.weights.fiwt")
        out.append((g, w))
    return out


def zoo_models():
    from paper_2410_21120_b200 import model_io
    data = np.load(GOLDEN / "toy_zoo.npz")
    out = []
    for mid in data["ids"]:
        mid = str(mid)
        g = model_io.load_graph(GOLDEN / "models" / f"zoo_{mid}.graph.json")
        w = model_io.load_weights(GOLDEN / "models" / f"zoo_{mid}.weights.fiwt")
        out.append((g, w))
    return out


@pytest.fixture(scope="session")
def corpus():
    return corpus_models()


@pytest.fixture(scope="session")
def corpus_golden():
    return np.load(GOLDEN / "corpus.npz")


@pytest.fixture(scope="session")
def zoo():
    return zoo_models()


@pytest.fixture(scope="session")
def zoo_golden():
    return np.load(GOLDEN / "toy_zoo.npz")
