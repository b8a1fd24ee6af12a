"""WORST_CASE traffic generation (traffic.py:161-191) against the reference's
own outputs (tests/golden/worst_case.json, written by make_golden.py from the
unmodified reference): full packet-list equality, including rulesets that
force the uncovered-port fallback.

The CPU test drives the generator's state machine with the oracle as the
candidate classifier (test infrastructure only); the GPU test runs the
product path, where candidate batches are classified by the CUDA scan."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1312_4188_b200 import (CidrMatcher, MatchMode, PortRange, Protocol, Ruleset, TrafficGenerationError,
                                  TrafficProfile, parse_rule)
from paper_1312_4188_b200.classifier import _rule_columns
from paper_1312_4188_b200.traffic import _worst_case


def _cases():
    with open(os.path.join(GOLDEN, "worst_case.json")) as fh:
        return json.load(fh)


CASES = _cases()
NAMES = sorted(k for k in CASES if not k.startswith("_"))


def _setup(name):
    c = CASES[name]
    rs = Ruleset(tuple(parse_rule(line) for line in c["rules"]))
    m = c["profile"]
    prof = TrafficProfile(count=m["count"], seed=m["seed"], proto=Protocol(m["proto"]),
                          src_subnet=CidrMatcher(*m["src"]), dst_subnet=CidrMatcher(*m["dst"]),
                          sport_range=PortRange(*m["sport"]), dport_range=PortRange(*m["dport"]),
                          match_mode=MatchMode.WORST_CASE)
    return rs, prof, c["packets"]


def _oracle_matches(rs):
    from oracle import oracle
    rules = _rule_columns(rs)
    R = len(rs)

    def matches(cands):
        pk = {"proto": np.array([int(p.proto) for p in cands], np.uint8),
              "src_ip": np.array([p.src_ip for p in cands], np.uint32),
              "src_port": np.array([p.src_port for p in cands], np.uint16),
              "dst_ip": np.array([p.dst_ip for p in cands], np.uint32),
              "dst_port": np.array([p.dst_port for p in cands], np.uint16)}
        if not R:
            return np.zeros(len(cands), np.bool_)
        return oracle.scan_range(rules, pk, 0, R) >= 0
    return matches


def _rows(packets):
    return [[p.id, int(p.proto), p.src_ip, p.src_port, p.dst_ip, p.dst_port] for p in packets]


def test_fixture_forces_fallbacks():
    # the fixture really exercises the fallback path (dport 80 / dport 0 packets)
    assert sum(p[5] == 80 for p in CASES["dport_gap_s5"]["packets"]) == 12
    assert sum(p[5] == 0 for p in CASES["src13_s3"]["packets"]) >= 2


@pytest.mark.parametrize("name", NAMES)
def test_worst_case_state_machine_equals_reference(name):
    rs, prof, want = _setup(name)
    got = _worst_case(prof, rs, matches=_oracle_matches(rs))
    assert _rows(got) == want


def test_worst_case_impossible_is_reference_error():
    c = CASES["_impossible"]
    rs = Ruleset(tuple(parse_rule(line) for line in c["rules"]))
    prof = TrafficProfile(3, seed=1, match_mode=MatchMode.WORST_CASE)
    with pytest.raises(TrafficGenerationError) as exc:
        _worst_case(prof, rs, matches=_oracle_matches(rs))
    assert str(exc.value) == c["error"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_worst_case_gpu_equals_reference(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1312_4188_b200 import generate_traffic
    rs, prof, want = _setup(name)
    assert _rows(generate_traffic(prof, rs)) == want
