"""Host-side behaviour of the drop-in API (no GPU): domain types, the ruleset
text format, partitioning / aggregation logic, config validation and the
host PRNG + ruleset generator, each against the reference's KATs
(pkg/tests/test_model.py, test_engines.py) and golden vectors."""
from __future__ import annotations

import ipaddress

import numpy as np
import pytest

from conftest import golden
from paper_1312_4188_b200 import (Action, CidrMatcher, ConfigError, EngineConfig, ExecutionModel,
                                  MatchResult, Packet, PartialMatch, PortRange, Protocol, Rule,
                                  RuleParseError, Ruleset, RulesetGenParams, aggregate, format_rule,
                                  generate_ruleset, load_ruleset, parse_rule, partition_bounds,
                                  partition_rules, rule_matches, save_ruleset)
from paper_1312_4188_b200.classifier import RULE_COLUMNS, _rule_columns
from paper_1312_4188_b200.engines import MAX_NODES
from paper_1312_4188_b200.model import ip_to_text, text_to_ip
from paper_1312_4188_b200.rng import Xorshift64Star, derive_seed


def mk_rule(action=Action.ACCEPT, proto=Protocol.ANY, src="*", sport=None, dst="*", dport=None):
    def cidr(spec):
        if spec == "*":
            return CidrMatcher(0, 0)
        base, _, plen = spec.partition("/")
        return CidrMatcher(int(ipaddress.IPv4Address(base)), int(plen))
    ports = lambda s: PortRange(0, 65535) if s is None else PortRange(*s)  # noqa: E731
    return Rule(action, proto, cidr(src), ports(sport), cidr(dst), ports(dport))


def mk_packet(pid=0, proto=Protocol.TCP, src="10.1.2.3", sport=5555, dst="8.8.8.8", dport=80):
    return Packet(pid, proto, int(ipaddress.IPv4Address(src)), sport, int(ipaddress.IPv4Address(dst)),
                  dport)


# ------------------------------------------------------------------ model KATs (test_model.py)

def test_rule_matches_kats():
    assert rule_matches(mk_rule(Action.ACCEPT, Protocol.TCP, src="10.0.0.0/8", dport=(80, 80)),
                        mk_packet(src="10.1.2.3", dport=80))
    assert not rule_matches(mk_rule(Action.DROP, Protocol.UDP), mk_packet(proto=Protocol.TCP))
    wild = mk_rule()
    for p in (mk_packet(), mk_packet(proto=Protocol.ICMP, src="0.0.0.0", dst="255.255.255.255"),
              mk_packet(sport=0, dport=65535)):
        assert rule_matches(wild, p)


def test_cidr_prefix_equality_vs_stdlib():
    rng = Xorshift64Star(1001)
    for _ in range(2000):
        plen = rng.randint(0, 32)
        m = CidrMatcher(rng.randbelow(1 << 32), plen)
        ip = rng.randbelow(1 << 32)
        expect = True if plen == 0 else (ip >> (32 - plen)) == (m.base >> (32 - plen))
        assert m.matches(ip) == expect
        assert m.matches(ip) == (ipaddress.ip_address(ip) in ipaddress.ip_network((m.base, plen)))


def test_cidr_normalisation_and_wildcard():
    m = CidrMatcher(text_to_ip("10.1.2.3"), 8)
    assert ip_to_text(m.base) == "10.0.0.0" and CidrMatcher(m.base, 8) == m
    z = CidrMatcher(text_to_ip("192.168.1.1"), 0)
    assert z.is_wildcard and z.base == 0 and z.mask == 0 and z.matches(0) and z.matches(0xFFFFFFFF)
    with pytest.raises(RuleParseError):
        CidrMatcher(0, 33)


def test_port_packet_result_invariants():
    with pytest.raises(RuleParseError):
        PortRange(2, 1)
    with pytest.raises(RuleParseError):
        PortRange(0, 70000)
    assert PortRange(0, 65535).is_wildcard and not PortRange(1, 65535).is_wildcard
    with pytest.raises(ValueError):
        Packet(0, Protocol.ANY, 0, 0, 0, 0)
    with pytest.raises(ValueError):
        MatchResult(Action.ACCEPT, None, 0)


@pytest.mark.parametrize("line,fragment", [
    ("ACCEPT tcp * * *", "6 fields"), ("PERMIT tcp * * * *", "field 1"),
    ("ACCEPT gre * * * *", "field 2"), ("ACCEPT tcp 10.0.0.0/40 * * *", "0..32"),
    ("ACCEPT tcp 10.0.0.300/8 * * *", "field 3"), ("ACCEPT tcp 10.0.0.0 * * *", "field 3"),
    ("ACCEPT tcp * 99999 * *", "0..65535"), ("ACCEPT tcp * 90-80 * *", "inverted"),
    ("ACCEPT tcp * * * 80-x", "field 6")])
def test_parse_rule_errors(line, fragment):
    with pytest.raises(RuleParseError) as exc:
        parse_rule(line)
    assert fragment in str(exc.value)


def test_parse_format_round_trip(tmp_path):
    assert parse_rule("ACCEPT tcp 10.0.0.0/8 * * 80-80") == mk_rule(Action.ACCEPT, Protocol.TCP,
                                                                     src="10.0.0.0/8", dport=(80, 80))
    assert parse_rule("DROP any * * * *") == mk_rule(Action.DROP, Protocol.ANY)
    assert ip_to_text(parse_rule("ACCEPT tcp 10.1.2.3/8 * * 80").src.base) == "10.0.0.0"
    assert format_rule(mk_rule()) == "ACCEPT any * * * *"
    r = mk_rule(Action.DROP, Protocol.TCP, "192.168.0.0/16", (1024, 65535), "10.0.0.1/32", (22, 22))
    assert format_rule(r) == "DROP tcp 192.168.0.0/16 1024-65535 10.0.0.1/32 22-22"
    rs = generate_ruleset(RulesetGenParams(count=1000, seed=99, wildcard_probability=0.25))
    for rule in rs:
        assert parse_rule(format_rule(rule)) == rule
    path = tmp_path / "rules.txt"
    save_ruleset(rs, path)
    assert load_ruleset(path) == rs
    (tmp_path / "c.txt").write_text("# c\n\n   \n# d\n")
    assert len(load_ruleset(tmp_path / "c.txt")) == 0
    (tmp_path / "i.txt").write_text("DROP tcp * * * 22  # no ssh\nACCEPT any * * * *\n")
    loaded = load_ruleset(tmp_path / "i.txt")
    assert [r.action for r in loaded] == [Action.DROP, Action.ACCEPT]
    (tmp_path / "b.txt").write_text("ACCEPT any * * * *\nACCEPT bogus * * * *\nDROP any * * * *\n")
    with pytest.raises(RuleParseError, match="line 2"):
        load_ruleset(tmp_path / "b.txt")
    hash(Ruleset((mk_rule(), mk_rule(Action.DROP))))


# ------------------------------------------------------------- engine host logic (test_engines.py)

def test_partition_kats():
    rs = generate_ruleset(RulesetGenParams(count=2048, seed=1))
    parts = partition_rules(rs, 4)
    assert [p.global_offset for p in parts] == [0, 512, 1024, 1536] and all(len(p) == 512 for p in parts)
    rs5 = generate_ruleset(RulesetGenParams(count=5, seed=2))
    assert [(p.global_offset, len(p)) for p in partition_rules(rs5, 2)] == [(0, 3), (3, 2)]
    rs3 = generate_ruleset(RulesetGenParams(count=3, seed=3))
    assert [len(p) for p in partition_rules(rs3, 8)] == [1, 1, 1, 0, 0, 0, 0, 0]
    rs97 = generate_ruleset(RulesetGenParams(count=97, seed=4))
    for nodes in (1, 2, 3, 7, 16, 97, 200):
        parts = partition_rules(rs97, nodes)
        assert [r for p in parts for r in p.rules] == list(rs97)
        sizes = {len(p) for p in parts}
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ConfigError):
        partition_bounds(10, 0)


def test_aggregate_kats():
    r = aggregate([PartialMatch(0, (512, Action.ACCEPT), 513), PartialMatch(1, (1030, Action.DROP), 7)], 2048)
    assert (r.verdict, r.matched_index, r.comparisons) == (Action.ACCEPT, 512, 520)
    r = aggregate([PartialMatch(i, None, 10) for i in range(4)], 40)
    assert r.verdict is Action.DROP and r.matched_index is None
    with pytest.raises(ValueError, match="duplicate"):
        aggregate([PartialMatch(0, None, 1), PartialMatch(0, None, 1)], 8)
    with pytest.raises(ValueError, match="outside"):
        aggregate([PartialMatch(0, (9, Action.ACCEPT), 10)], 8)


def test_config_validation():
    with pytest.raises(ConfigError):
        EngineConfig(model=ExecutionModel.HYBRID, nodes=0)
    with pytest.raises(ConfigError, match="512"):
        EngineConfig(model=ExecutionModel.HYBRID, nodes=MAX_NODES + 1)
    with pytest.raises(ConfigError):
        EngineConfig(model=ExecutionModel.HYBRID, batch_size=0)
    with pytest.raises(ConfigError):
        EngineConfig(model=ExecutionModel.HYBRID, executor="gpu")
    with pytest.raises(ConfigError):
        EngineConfig(model=ExecutionModel.HYBRID, max_workers=0)
    with pytest.raises(ConfigError, match="gpus"):
        EngineConfig(model=ExecutionModel.HYBRID, gpus=0)
    with pytest.raises(ConfigError, match="shard"):
        EngineConfig(model=ExecutionModel.HYBRID, shard="nodes")
    assert EngineConfig(model=ExecutionModel.FUNCTION_PARALLEL, gpus=8, shard="rules").gpus == 8
    with pytest.raises(ConfigError):
        ExecutionModel.from_key("quantum")
    assert ExecutionModel.from_key("hybrid") is ExecutionModel.HYBRID


# ---------------------------------------------------------------- generators vs golden

def test_rng_matches_reference_golden():
    g = golden("rng.npz")
    for seed, stream in zip(g["seeds"].tolist(), g["streams"]):
        r = Xorshift64Star(seed)
        assert [r.next_u64() for _ in range(64)] == stream.tolist()
    for seed, row in zip(g["seeds"].tolist(), g["derive"]):
        assert [derive_seed(seed, k) for k in range(8)] == row.tolist()
    r = Xorshift64Star(99)
    assert [r.randbelow(n) for n in (1, 2, 3, 6, 1000, 65536, 1 << 32, 3 * 10**9) * 8] == g["randbelow"].tolist()
    r = Xorshift64Star(100)
    assert [r.chance(p) for p in (0.0, 0.1, 0.5, 0.15, 0.3, 1.0, 0.999) * 10] == g["chance"].tolist()


@pytest.mark.parametrize("name", ["r1000_s1", "r2048_s21_w15", "r300_s40_w30", "r64_s30_w40"])
def test_generate_ruleset_matches_reference_golden(name):
    g = golden(f"rules_{name}.npz")
    cols = _rule_columns(generate_ruleset(RulesetGenParams(int(g["count"]), int(g["seed"]),
                                                           float(g["wp"]))))
    for f in RULE_COLUMNS:
        np.testing.assert_array_equal(cols[f], g[f])
