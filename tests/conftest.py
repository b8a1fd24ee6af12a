"""Shared test configuration.

``-m gpu`` tests need a B200 (they call the CUDA path through the C-ABI);
everything else runs on CPU.  The oracle (oracle/) is the checker only.
"""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (runs via gpurun)")


def golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_rules(name: str) -> dict:
    from oracle.oracle import RULE_FIELDS
    g = golden(f"rules_{name}.npz")
    if "proto" in g:
        return {f: g[f] for f in RULE_FIELDS}
    from oracle import oracle
    rules = oracle.gen_ruleset(int(g["count"]), int(g["seed"]), float(g["wp"]))
    return rules


def golden_traffic(name: str) -> dict:
    from oracle.oracle import PKT_FIELDS
    g = golden(f"traffic_{name}.npz")
    if "proto" in g:
        return {f: g[f] for f in PKT_FIELDS}
    from oracle import oracle
    return oracle.gen_traffic_uniform(int(g["count"]), int(g["seed"]), int(g["p_proto"]),
                                      int(g["p_src_base"]), int(g["p_src_plen"]),
                                      int(g["p_dst_base"]), int(g["p_dst_plen"]),
                                      int(g["p_sport_lo"]), int(g["p_sport_hi"]),
                                      int(g["p_dport_lo"]), int(g["p_dport_hi"]))


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
