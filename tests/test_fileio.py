"""Native readers/writers of the ruleset text and traffic CSV formats
(hostio.cpp via fileio.py) against the reference-compatible Python parsers:
identical columns / records on canonical files, and on every malformed or
non-canonical input the exact reference behaviour (via the Python path)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1312_4188_b200 import (Packet, Protocol, RuleParseError, RulesetGenParams, TrafficFormatError,
                                  generate_ruleset, load_ruleset, load_traffic, save_ruleset, save_traffic)
from paper_1312_4188_b200.classifier import RULE_COLUMNS, PacketArrays, _rule_columns
from paper_1312_4188_b200.fileio import format_results, load_ruleset_columns, parse_traffic
from paper_1312_4188_b200.rng import Xorshift64Star


def test_rules_native_equals_python(tmp_path):
    rs = generate_ruleset(RulesetGenParams(3000, seed=7, wildcard_probability=0.25))
    path = tmp_path / "r.txt"
    save_ruleset(rs, path)
    got = load_ruleset_columns(path)
    want = _rule_columns(rs)
    for f in RULE_COLUMNS:
        np.testing.assert_array_equal(got[f], want[f])


@pytest.mark.parametrize("text", [
    "# header\n\nACCEPT tcp 10.1.2.3/8 * * 80  # web\n  DROP any * * * *\r\nACCEPT udp 1.2.3.4/32 5-6 0.0.0.0/0 00080-65535\n",
    "ACCEPT icmp * 1000 192.168.0.0/16 *",  # no trailing newline
    "ACCEPT tcp +10.0.0.0/8 * * *\n",  # non-canonical -> python path (error)
    "ACCEPT tcp 10.0.0.0/08 * * +80\n",  # '+80' valid for int(): python path accepts
    "ACCEPT tcp 010.0.0.0/8 * * *\n", "ACCEPT tcp 10.0.0.0/33 * * *\n", "ACCEPT tcp * 90-80 * *\n",
    "ACCEPT tcp * * *\n", "PERMIT tcp * * * *\n", "ACCEPT gre * * * *\n", "ACCEPT tcp * 70000 * *\n",
    "ACCEPT tcp * 80- * *\n", "ACCEPT tcp * -5 * *\n", "ACCEPT tcp 1.2.3/8 * * *\n",
    "ACCEPT tcp * * * 80\rDROP any * * * *\n",
])
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


HDR = "id,proto,src_ip,src_port,dst_ip,dst_port\n"


@pytest.mark.parametrize("body", [
    "1,tcp,1.2.3.4,5,6.7.8.9,10\r\n\n2,udp,0.0.0.0,0,255.255.255.255,65535",
    "-3,tcp,1.2.3.4,5,6.7.8.9,10\n",  # negative id: int() accepts -> python path
    " 4,tcp,1.2.3.4, 5,6.7.8.9,10\n",  # spaces: int() accepts -> python path
    '"5",tcp,1.2.3.4,5,6.7.8.9,10\n',  # quoted field: csv accepts -> python path
    "6,any,1.2.3.4,5,6.7.8.9,10\n", "7,tcp,1.2.3.4,70000,6.7.8.9,10\n", "8,tcp,1.2.3,5,6.7.8.9,10\n",
    "9,tcp,1.2.3.4,5,6.7.8.9\n", "x,tcp,1.2.3.4,5,6.7.8.9,10\n", "10,tcp,1.2.3.4,5,6.7.8.9,10,11\n",
])
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
