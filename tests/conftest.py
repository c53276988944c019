import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    # a gpu test on a machine without CUDA fails loudly instead of skipping
    # silently only when explicitly selected with -m gpu; otherwise it is
    # deselected by the driver's -m "not gpu".
    pass


def _ref(tok: str) -> int:
    return ~int(tok[1:]) if tok.startswith("~") else int(tok)


def load_fig6():
    d = {"edges": [], "nodes": {}}
    with open(os.path.join(GOLDEN, "fig6.txt")) as f:
        for line in f:
            line = line.split("#")[0].split()
            if not line:
                continue
            k, rest = line[0], line[1:]
            if k in ("weights", "cells", "offsets"):
                d[k] = [int(x) for x in rest]
            elif k == "m":
                d["m"] = int(rest[0])
            elif k == "edge":
                d["edges"].append((rest[0], rest[1]))
            elif k == "node":
                d["nodes"][int(rest[0])] = (_ref(rest[1]), _ref(rest[2]))
            elif k == "table":
                d["table"] = [_ref(x) for x in rest]
    return d


def load_fig9():
    out = {}
    with open(os.path.join(GOLDEN, "fig9_monotone.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            N, i, v = line.split()
            out.setdefault(int(N), {})[int(i)] = float(v)
    return out


@pytest.fixture
def fig6():
    return load_fig6()


@pytest.fixture
def fig9():
    return load_fig9()
