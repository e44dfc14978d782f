import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

import paper_1509_01506_b200 as ks  # noqa: E402
from paper_1509_01506_b200 import _native  # noqa: E402

# a fresh checkout: build the C-ABI library (nvcc cross-compiles for sm_100a
# without a GPU) and the oracle before any test loads them
if not _native.LIB_PATH.exists():
    import subprocess

    subprocess.run(["make", "-C", str(REPO / "paper_1509_01506_b200" / "csrc"), "-j8"], check=True,
                   stdout=subprocess.DEVNULL)

TOY_PATTERNS = "acg\ncat\ncta\ntta"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def toy_exprs():
    return ks.parse_expressions(TOY_PATTERNS)


@pytest.fixture(scope="session")
def toy_table(toy_exprs):
    return ks.expand_to_literals(toy_exprs)


@pytest.fixture(scope="session")
def toy_dfa(toy_table):
    return ks.build_dfa(toy_table)


def load_random_cases():
    z = np.load(GOLDEN / "random_cases.npz")
    cases = []
    for i in range(len(z["texts"])):
        def sl(name, i=i):
            off = z[name + "_off"]
            return z[name][off[i]:off[i + 1]]
        t = sl("dfa_t")
        cases.append({
            "text": str(z["texts"][i]),
            "data": sl("data").tobytes(),
            "workers": int(z["workers"][i]),
            "window": int(z["window"][i]),
            "counts": sl("counts"),
            "locs": sl("locs"),
            "meta": json.loads(str(z["meta"][i])),
            "dfa_t": t,
            "dfa_off": z["dfa_off"][z["dfa_off_off"][i]:z["dfa_off_off"][i + 1]],
            "dfa_ids": z["dfa_ids"][z["dfa_ids_off"][i]:z["dfa_ids_off"][i + 1]],
        })
    return cases


def load_config_cases():
    z = np.load(GOLDEN / "configs.npz")
    index = json.loads(str(z["index"]))
    for i, case in enumerate(index):
        case["counts"] = z[f"counts_{i}"]
        case["locs"] = z[f"locs_{i}"] if f"locs_{i}" in z else None
    return index


@pytest.fixture(scope="session")
def random_cases():
    return load_random_cases()


@pytest.fixture(scope="session")
def config_cases():
    return load_config_cases()
