"""Native readers/writers of the ruleset text and traffic CSV formats
(hostio.cpp via fileio.py) against the reference-compatible Python parsers:
identical columns / records on canonical files, and on every malformed or
non-canonical input the exact reference behaviour (via the Python path)."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1312_4188_b200 import (Packet, Protocol, RuleParseError, RulesetGenParams, TrafficFormatError,
                                  generate_ruleset, load_ruleset, load_traffic, save_ruleset, save_traffic)
from paper_1312_4188_b200.classifier import RULE_COLUMNS, PacketArrays, _rule_columns
from paper_1312_4188_b200.fileio import format_results, load_ruleset_columns, parse_traffic
from paper_1312_4188_b200.rng import Xorshift64Star

sys.path.insert(0, GOLDEN)
from parser_cases import RULE_TEXTS, TRAFFIC_BODIES, TRAFFIC_HEADER  # noqa: E402

with open(os.path.join(GOLDEN, "parsers.json")) as _fh:
    PARSERS = json.load(_fh)  # the reference's load_ruleset / load_traffic on each case (make_golden.py)


def test_rules_native_equals_python(tmp_path):
    rs = generate_ruleset(RulesetGenParams(3000, seed=7, wildcard_probability=0.25))
    path = tmp_path / "r.txt"
    save_ruleset(rs, path)
    got = load_ruleset_columns(path)
    want = _rule_columns(rs)
    for f in RULE_COLUMNS:
        np.testing.assert_array_equal(got[f], want[f])


@pytest.mark.parametrize("text", RULE_TEXTS)
def test_rules_edge_cases_match_python(tmp_path, text):
    path = tmp_path / "r.txt"
    path.write_bytes(text.encode())
    try:
        want = _rule_columns(load_ruleset(path))
    except RuleParseError as exc:
        with pytest.raises(RuleParseError) as got:
            load_ruleset_columns(path)
        assert str(got.value) == str(exc)
        return
    got = load_ruleset_columns(path)
    for f in RULE_COLUMNS:
        np.testing.assert_array_equal(got[f], want[f])


def _packets(n, seed):
    r = Xorshift64Star(seed)
    protos = (Protocol.TCP, Protocol.UDP, Protocol.ICMP)
    return [Packet(r.randbelow(10**6), protos[r.randbelow(3)], r.randbelow(1 << 32), r.randbelow(65536),
                   r.randbelow(1 << 32), r.randbelow(65536)) for _ in range(n)]


def test_traffic_native_equals_python(tmp_path):
    pk = _packets(5000, 3)
    path = tmp_path / "t.csv"
    save_traffic(pk, path)
    ids, rec = parse_traffic(path)
    want = load_traffic(path)
    assert ids.tolist() == [p.id for p in want]
    ref = PacketArrays.pack_host([int(p.proto) for p in want], [p.src_ip for p in want],
                                 [p.src_port for p in want], [p.dst_ip for p in want],
                                 [p.dst_port for p in want])
    np.testing.assert_array_equal(rec, ref)


HDR = TRAFFIC_HEADER


@pytest.mark.parametrize("body", TRAFFIC_BODIES)
def test_traffic_edge_cases_match_python(tmp_path, body):
    path = tmp_path / "t.csv"
    path.write_bytes((HDR + body).encode())
    try:
        want = load_traffic(path)
    except TrafficFormatError as exc:
        with pytest.raises(TrafficFormatError) as got:
            parse_traffic(path)
        assert str(got.value) == str(exc)
        return
    ids, rec = parse_traffic(path)
    assert ids.tolist() == [p.id for p in want]
    assert rec[:, 3].tolist() == [int(p.proto) for p in want]
    assert rec[:, 0].tolist() == [p.src_ip for p in want]
    assert (rec[:, 2] & 0xFFFF).tolist() == [p.dst_port for p in want]


def test_bad_header_is_reference_error(tmp_path):
    path = tmp_path / "t.csv"
    path.write_bytes(b"\xef\xbb\xbf" + HDR.encode() + b"1,tcp,1.2.3.4,5,6.7.8.9,10\n")
    with pytest.raises(TrafficFormatError, match="line 1"):
        parse_traffic(path)


def test_format_results():
    out = format_results(np.array([0, 17, 5]), np.array([3, 0x7FFFFFFF, 0], np.uint32),
                         np.array([1, 0, 0], np.uint8))
    assert out.decode() == "0,ACCEPT,3\n17,DROP,-\n5,DROP,0\n"
    assert format_results(np.zeros(0, np.int64), np.zeros(0, np.uint32), np.zeros(0, np.uint8)) == b""


@pytest.mark.parametrize("k", range(len(RULE_TEXTS)))
def test_rules_edge_cases_equal_reference(tmp_path, k):
    """Python and native readers against the reference's own load_ruleset output."""
    path = tmp_path / "rules.txt"
    path.write_bytes(RULE_TEXTS[k].encode())
    want = PARSERS["rules"][k]
    for load in (lambda q: _rule_columns(load_ruleset(q)), load_ruleset_columns):
        if "error" in want:
            with pytest.raises(RuleParseError) as got:
                load(path)
            assert str(got.value) == want["error"].replace("{path}", str(path))
        else:
            got = load(path)
            for f in RULE_COLUMNS:
                assert np.asarray(got[f]).astype(np.int64).tolist() == want["columns"][f], f


@pytest.mark.parametrize("k", range(len(TRAFFIC_BODIES)))
def test_traffic_edge_cases_equal_reference(tmp_path, k):
    path = tmp_path / "t.csv"
    path.write_bytes((TRAFFIC_HEADER + TRAFFIC_BODIES[k]).encode())
    want = PARSERS["traffic"][k]
    if "error" in want:
        for load in (load_traffic, parse_traffic):
            with pytest.raises(TrafficFormatError) as got:
                load(path)
            assert str(got.value) == want["error"].replace("{path}", str(path))
        return
    got = [[p.id, int(p.proto), p.src_ip, p.src_port, p.dst_ip, p.dst_port] for p in load_traffic(path)]
    assert got == want["packets"]
    ids, rec = parse_traffic(path)
    nat = [[int(i), int(r[3]), int(r[0]), int(r[2] >> 16), int(r[1]), int(r[2] & 0xFFFF)]
           for i, r in zip(ids.tolist(), rec)]
    assert nat == want["packets"]
