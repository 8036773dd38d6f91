import gzip
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from paper_2506_12204_b200.soa import TraceBatch, tie_ranks  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running parity case")


def has_reference() -> bool:
    return os.path.isdir("/root/reference/pkg/src/semsched")


_GOLDEN = {}


def load_golden(group: str):
    if group not in _GOLDEN:
        path = os.path.join(HERE, "golden", f"golden_{group}.json.gz")
        with gzip.open(path, "rt", encoding="utf-8") as fh:
            _GOLDEN[group] = json.load(fh)
    return _GOLDEN[group]


def golden_cases(group: str):
    return load_golden(group)["cases"]


def case_batch(case) -> TraceBatch:
    inp = case["inputs"]
    n = len(inp["ready"])
    arr = np.array(inp["arrival"], np.float64)
    ids = np.array(inp["ids"], np.int64)
    return TraceBatch(
        offsets=np.array([0, n], np.int64),
        ready=np.array(inp["ready"], np.float64),
        arrival=arr,
        prompt=np.array(inp["prompt"], np.uint32),
        true_out=np.array(inp["true_out"], np.uint32),
        pred_len=np.array(inp["pred_len"], np.uint32),
        pred_urg=np.array(inp["pred_urg"], np.uint8),
        true_urg=np.array(inp["true_urg"], np.uint8),
        tie=tie_ranks(arr, ids) if n else np.zeros(0, np.uint32),
        ids=ids,
        record_pos=np.array(inp["record_pos"], np.int64),
    )


def case_params(case, flags):
    from paper_2506_12204_b200.results import make_params

    p = case["params"]
    return make_params(p["profile"], p["batch_size"], p["memory_capacity"], policy=p["policy"],
                       dependency_rule=p["dependency_rule"], decode_batch_cost=p["decode_batch_cost"],
                       levels=p["levels"], flags=flags, max_rounds=5_000_000)
