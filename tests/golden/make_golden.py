"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED Python reference.

Run ONLY in the build container (it imports the reference package from
/root/reference/pkg/src, which does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture records the reference call that produced it.  The fixtures pin
(a) the oracle restatement in oracle/ and (b) the CUDA path, to the reference:

* rng.npz        -- Xorshift64Star streams / derive_seed   (parafw/rng.py:31-81)
* rules_*.npz    -- CompiledRuleset SoA arrays of generate_ruleset outputs
                    (parafw/classifier.py:120-134, parafw/traffic.py:194-229)
* traffic_*.npz  -- PacketArrays SoA of generate_traffic outputs
                    (parafw/classifier.py:75-83, parafw/traffic.py:117-160)
* scan_*.npz     -- scan_range / classify_batch_sequential first-match indices
                    and ClassifyStats (parafw/classifier.py:146-209)
* engine_*.npz   -- Engine.run per-packet comparisons + stats for the
                    function-parallel / hybrid models (parafw/engines.py:260-369)
* adversarial.npz -- the SURVEY 8(d) adversarial 50K-rule recipe, built with
                    the reference generator, and its first-match indices.
* worst_case.json -- generate_traffic(WORST_CASE) packet lists, including
                    rulesets that force the uncovered-port fallback
                    (parafw/traffic.py:161-191)
* parsers.json    -- load_ruleset / load_traffic on the edge inputs of
                    parser_cases.py: the columns, or the exact error message
                    (parafw/model.py:233-331, parafw/traffic.py:259-297)

    python tests/golden/make_golden.py [--only worst_case,parsers]

Large arrays are stored as sha256 digests plus a head slice so the fixtures
stay small; the oracle regenerates them and compares digests.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from parafw.classifier import PacketArrays, classify_batch_sequential, compile_ruleset  # noqa: E402
from parafw.engines import EngineConfig, ExecutionModel, Engine  # noqa: E402
from parafw.model import Action, CidrMatcher, PortRange, Protocol, Rule, Ruleset  # noqa: E402
from parafw.rng import Xorshift64Star, derive_seed  # noqa: E402
from parafw.traffic import (  # noqa: E402
    MatchMode,
    RulesetGenParams,
    TrafficFormatError,
    TrafficProfile,
    generate_ruleset,
    generate_traffic,
    load_traffic,
)
from parafw.model import RuleParseError, load_ruleset  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import parser_cases  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
RULE_FIELDS = ("proto", "src_base", "src_mask", "sport_lo", "sport_hi",
               "dst_base", "dst_mask", "dport_lo", "dport_hi", "action_accept")
PKT_FIELDS = ("proto", "src_ip", "src_port", "dst_ip", "dst_port")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def rule_arrays(ruleset):
    c = compile_ruleset(ruleset)
    return {f: getattr(c, f) for f in RULE_FIELDS}


def pkt_arrays(packets):
    p = PacketArrays.from_packets(packets)
    return {f: getattr(p, f) for f in PKT_FIELDS}


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path)} bytes")


def gen_rng():
    seeds = np.array([0, 1, 2, 7, 12345, (1 << 64) - 1, 0xDEADBEEF], dtype=np.uint64)
    streams = []
    for s in seeds.tolist():
        r = Xorshift64Star(s)
        streams.append([r.next_u64() for _ in range(64)])
    ds = np.array([[derive_seed(s, k) for k in range(8)] for s in seeds.tolist()], dtype=np.uint64)
    # randbelow / randint / chance on a fixed stream
    r = Xorshift64Star(99)
    rb = np.array([r.randbelow(n) for n in (1, 2, 3, 6, 1000, 65536, 1 << 32, 3 * 10**9) * 8], dtype=np.uint64)
    r = Xorshift64Star(100)
    ch = np.array([r.chance(p) for p in (0.0, 0.1, 0.5, 0.15, 0.3, 1.0, 0.999) * 10], dtype=np.bool_)
    save("rng.npz", seeds=seeds, streams=np.array(streams, dtype=np.uint64), derive=ds,
         randbelow=rb, chance=ch)


# (name, count, seed, wildcard_probability, full arrays?)
RULESETS = [
    ("r1000_s1", 1000, 1, 0.1, True),
    ("r2048_s21_w15", 2048, 21, 0.15, True),
    ("r300_s40_w30", 300, 40, 0.3, True),
    ("r100_s60_w35", 100, 60, 0.35, True),
    ("r503_s24_w30", 503, 24, 0.3, True),
    ("r64_s30_w40", 64, 30, 0.4, True),
    ("r4096_s1", 4096, 1, 0.1, False),
    ("r10000_s1", 10000, 1, 0.1, False),
    ("r100000_s1", 100000, 1, 0.1, False),
]


def gen_rulesets(cache):
    for name, count, seed, wp, full in RULESETS:
        rs = generate_ruleset(RulesetGenParams(count=count, seed=seed, wildcard_probability=wp))
        cache[name] = rs
        arrs = rule_arrays(rs)
        meta = dict(count=np.int64(count), seed=np.int64(seed), wp=np.float64(wp),
                    sha256=np.array(digest(*[arrs[f] for f in RULE_FIELDS])))
        if full:
            save(f"rules_{name}.npz", **meta, **arrs)
        else:
            head = {f"head_{f}": arrs[f][:512] for f in RULE_FIELDS}
            save(f"rules_{name}.npz", **meta, **head)


# (name, profile kwargs, full arrays?)
TRAFFIC = [
    ("t100000_s2", dict(count=100_000, seed=2), False),
    ("t1000_s22", dict(count=1000, seed=22), True),
    ("t10000_s41", dict(count=10_000, seed=41), True),
    ("t150_s61", dict(count=150, seed=61), True),
    ("t600_s25", dict(count=600, seed=25), True),
    ("t2000_s7_dst0_1", dict(count=2000, seed=7, dst_subnet=CidrMatcher(0, 1)), True),
    ("t2000_s8_dst192_2", dict(count=2000, seed=8, dst_subnet=CidrMatcher(0xC0000000, 2)), True),
    ("t5000_s9_ports", dict(count=5000, seed=9, proto=Protocol.UDP,
                            src_subnet=CidrMatcher(0x0A000000, 8),
                            sport_range=PortRange(1000, 2999), dport_range=PortRange(80, 80)), True),
    ("t3000_s11_icmp", dict(count=3000, seed=11, proto=Protocol.ICMP,
                            dport_range=PortRange(7, 65000)), True),
]


def gen_traffic(cache):
    for name, kw, full in TRAFFIC:
        pk = generate_traffic(TrafficProfile(**kw))
        cache[name] = pk
        arrs = pkt_arrays(pk)
        prof = TrafficProfile(**kw)
        meta = dict(
            count=np.int64(prof.count), seed=np.int64(prof.seed), p_proto=np.int64(int(prof.proto)),
            p_src_base=np.int64(prof.src_subnet.base), p_src_plen=np.int64(prof.src_subnet.prefix_len),
            p_dst_base=np.int64(prof.dst_subnet.base), p_dst_plen=np.int64(prof.dst_subnet.prefix_len),
            p_sport_lo=np.int64(prof.sport_range.lo), p_sport_hi=np.int64(prof.sport_range.hi),
            p_dport_lo=np.int64(prof.dport_range.lo), p_dport_hi=np.int64(prof.dport_range.hi),
            sha256=np.array(digest(*[arrs[f] for f in PKT_FIELDS])),
        )
        if full:
            save(f"traffic_{name}.npz", **meta, **arrs)
        else:
            head = {f"head_{f}": arrs[f][:4096] for f in PKT_FIELDS}
            save(f"traffic_{name}.npz", **meta, **head)


def seq_scan(rs, pk):
    t = time.time()
    results, stats = classify_batch_sequential(rs, pk)
    first = np.array([-1 if r.matched_index is None else r.matched_index for r in results], dtype=np.int64)
    verdict = np.array([r.verdict is Action.ACCEPT for r in results], dtype=np.bool_)
    comps = np.array([r.comparisons for r in results], dtype=np.int64)
    print(f"  classify_batch_sequential {len(rs)}x{len(pk)}: {time.time() - t:.1f}s")
    return first, verdict, comps, stats


def gen_scans(rules, traffic):
    pairs = [
        ("oracle_r1000_t100000", "r1000_s1", "t100000_s2"),
        ("r2048_t1000", "r2048_s21_w15", "t1000_s22"),
        ("r300_t10000", "r300_s40_w30", "t10000_s41"),
        ("r64_t600", "r64_s30_w40", "t600_s25"),
        ("r1000_t5000ports", "r1000_s1", "t5000_s9_ports"),
        ("r1000_t3000icmp", "r1000_s1", "t3000_s11_icmp"),
    ]
    for name, rn, tn in pairs:
        first, verdict, comps, st = seq_scan(rules[rn], traffic[tn])
        save(f"scan_{name}.npz", rules=np.array(rn), traffic=np.array(tn),
             first=first.astype(np.int32), verdict=verdict,
             total_comparisons=np.int64(st.total_comparisons),
             max_worker_comparisons=np.int64(st.max_worker_comparisons),
             packets_processed=np.int64(st.packets_processed))

    # data-parallel / grid / function configs sampled at 20K packets (seeds 1/2)
    pk20k = generate_traffic(TrafficProfile(count=20_000, seed=2))
    for rn in ("r4096_s1", "r10000_s1", "r100000_s1"):
        first, verdict, comps, st = seq_scan(rules[rn], pk20k)
        save(f"scan_{rn}_t20000.npz", rules=np.array(rn), traffic=np.array("t20000_s2"),
             first=first.astype(np.int32), verdict=verdict,
             total_comparisons=np.int64(st.total_comparisons),
             max_worker_comparisons=np.int64(st.max_worker_comparisons))

    # scan_range windows (test_classifier.py:94-105)
    c = compile_ruleset(rules["r100_s60_w35"])
    pa = PacketArrays.from_packets(traffic["t150_s61"])
    windows = [(0, 100), (0, 0), (17, 53), (99, 100), (40, 40), (3, 97), (64, 100)]
    out = np.stack([c.scan_range(pa, lo, hi) for lo, hi in windows]).astype(np.int32)
    save("scan_windows_r100_t150.npz", windows=np.array(windows, dtype=np.int64), first=out)


def engine_run(rs, pk, model, nodes, batch=4096):
    cfg = EngineConfig(model=ExecutionModel.from_key(model), nodes=nodes, batch_size=batch,
                       executor="serial")
    with Engine(cfg) as eng:
        results, stats = eng.run(rs, pk)
    first = np.array([-1 if r.matched_index is None else r.matched_index for r in results], dtype=np.int32)
    comps = np.array([r.comparisons for r in results], dtype=np.int64)
    return first, comps, stats


def gen_engines(rules, traffic):
    # function-parallel / hybrid sweeps (test_engines.py:198-230)
    rs, pk = rules["r503_s24_w30"], traffic["t600_s25"]
    out = {}
    for model in ("data", "function", "hybrid"):
        for nodes in (1, 2, 3, 4, 8, 16, 64, 512):
            first, comps, st = engine_run(rs, pk, model, nodes)
            key = f"{model}_{nodes}"
            out[f"{key}_first"] = first
            out[f"{key}_comps"] = comps
            out[f"{key}_stats"] = np.array([st.total_comparisons, st.max_worker_comparisons,
                                            st.packets_processed], dtype=np.int64)
    save("engine_r503_t600.npz", **out)

    # function-parallel at G = 1/2/4/8 on the 100K-rule config (sampled packets)
    rs = rules["r100000_s1"]
    pk = generate_traffic(TrafficProfile(count=2000, seed=2))
    out = {}
    for nodes in (1, 2, 4, 8):
        t = time.time()
        first, comps, st = engine_run(rs, pk, "function", nodes)
        print(f"  function r100000 x 2000 nodes={nodes}: {time.time() - t:.1f}s")
        out[f"function_{nodes}_first"] = first
        out[f"function_{nodes}_comps"] = comps
        out[f"function_{nodes}_stats"] = np.array([st.total_comparisons, st.max_worker_comparisons,
                                                   st.packets_processed], dtype=np.int64)
    save("engine_r100000_t2000.npz", **out)


def adversarial_ruleset(total=50_000) -> Ruleset:
    """SURVEY 8(d) recipe, built from reference primitives."""
    head = Rule(Action.ACCEPT, Protocol.ANY, CidrMatcher(0, 0), PortRange(0, 65535),
                CidrMatcher(0xC0000000, 2), PortRange(0, 65535))
    n_decoy = int(total * 0.9)
    decoys = []
    for r in generate_ruleset(RulesetGenParams(n_decoy, seed=2)):
        if r.dst.prefix_len == 0:
            dst = CidrMatcher(0x80000000, 1)
        else:
            dst = CidrMatcher(r.dst.base | 0x80000000, r.dst.prefix_len)
        decoys.append(Rule(r.action, r.proto, r.src, r.sport, dst, r.dport))
    tail = list(generate_ruleset(RulesetGenParams(total - 1 - n_decoy, seed=1)))
    return Ruleset((head, *decoys, *tail))


def adversarial_traffic(n) -> list:
    n_late = int(n * 0.9)
    late = generate_traffic(TrafficProfile(count=n_late, seed=7, dst_subnet=CidrMatcher(0, 1)))
    early = generate_traffic(TrafficProfile(count=n - n_late, seed=8,
                                            dst_subnet=CidrMatcher(0xC0000000, 2)))
    return late + early


def gen_adversarial():
    rs = adversarial_ruleset()
    pk = adversarial_traffic(20_000)
    arrs = rule_arrays(rs)
    first, verdict, comps, st = seq_scan(rs, pk)
    save("adversarial.npz", rules_sha256=np.array(digest(*[arrs[f] for f in RULE_FIELDS])),
         traffic_sha256=np.array(digest(*[pkt_arrays(pk)[f] for f in PKT_FIELDS])),
         first=first.astype(np.int32), verdict=verdict,
         total_comparisons=np.int64(st.total_comparisons),
         max_worker_comparisons=np.int64(st.max_worker_comparisons))


def _complement_rules(base: int, plen: int, dport: PortRange) -> list:
    """DROP tcp rules whose src prefixes cover every address outside base/plen."""
    out = []
    for k in range(1, plen + 1):
        bit = 1 << (32 - k)
        out.append(Rule(Action.DROP, Protocol.TCP, CidrMatcher((base ^ bit) & ~(bit - 1), k), PortRange(0, 65535),
                        CidrMatcher(0, 0), dport))
    return out


# (name, ruleset builder, profile kwargs)
WORST_CASES = [
    # every TCP candidate matches unless dport == 80: every packet takes the fallback
    ("dport_gap_s5", lambda: Ruleset((
        Rule(Action.ACCEPT, Protocol.TCP, CidrMatcher(0, 0), PortRange(0, 65535), CidrMatcher(0, 0), PortRange(0, 79)),
        Rule(Action.ACCEPT, Protocol.TCP, CidrMatcher(0, 0), PortRange(0, 65535), CidrMatcher(0, 0),
             PortRange(81, 65535)))), dict(count=12, seed=5)),
    # acceptance probability 2^-13: about 30% of packets exhaust 10000 attempts
    ("src13_s3", lambda: Ruleset(tuple(_complement_rules(0x0A000000, 13, PortRange(1, 65535)))),
     dict(count=40, seed=3)),
    ("src13_s11_udp", lambda: Ruleset(tuple(_complement_rules(0x0A000000, 13, PortRange(1, 65535))) + (
        Rule(Action.ACCEPT, Protocol.UDP, CidrMatcher(0, 0), PortRange(0, 65535), CidrMatcher(0, 0),
             PortRange(0, 65535)),)), dict(count=30, seed=11)),
    # random rulesets: rejection only
    ("r2048_s21_w15_s4", lambda: generate_ruleset(RulesetGenParams(2048, seed=21, wildcard_probability=0.15)),
     dict(count=300, seed=4)),
    ("r1000_s1_s9_ports", lambda: generate_ruleset(RulesetGenParams(1000, seed=1)),
     dict(count=200, seed=9, sport_range=PortRange(1000, 2999), dport_range=PortRange(7, 65000))),
]


def _profile_meta(prof):
    return dict(count=prof.count, seed=prof.seed, proto=int(prof.proto),
                src=[prof.src_subnet.base, prof.src_subnet.prefix_len],
                dst=[prof.dst_subnet.base, prof.dst_subnet.prefix_len],
                sport=[prof.sport_range.lo, prof.sport_range.hi], dport=[prof.dport_range.lo, prof.dport_range.hi])


def gen_worst_case():
    import json
    from parafw.model import format_rule
    out = {}
    for name, build, kw in WORST_CASES:
        rs = build()
        prof = TrafficProfile(match_mode=MatchMode.WORST_CASE, **kw)
        t = time.time()
        pk = generate_traffic(prof, rs)
        out[name] = {"rules": [format_rule(r) for r in rs], "profile": _profile_meta(prof),
                     "packets": [[p.id, int(p.proto), p.src_ip, p.src_port, p.dst_ip, p.dst_port] for p in pk]}
        print(f"  worst case {name}: {len(pk)} packets in {time.time() - t:.1f}s")
    # the reference's error when no non-matching packet exists
    rs = Ruleset((Rule(Action.DROP, Protocol.ANY, CidrMatcher(0, 0), PortRange(0, 65535), CidrMatcher(0, 0),
                       PortRange(0, 65535)),))
    try:
        generate_traffic(TrafficProfile(3, seed=1, match_mode=MatchMode.WORST_CASE), rs)
        err = None
    except Exception as exc:  # TrafficGenerationError
        err = str(exc)
    out["_impossible"] = {"rules": [format_rule(r) for r in rs], "error": err}
    path = os.path.join(OUT, "worst_case.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0)
    print(f"wrote worst_case.json: {os.path.getsize(path)} bytes")


def gen_parsers():
    import json
    import tempfile
    res = {"rules": [], "traffic": []}
    with tempfile.TemporaryDirectory() as d:
        for text in parser_cases.RULE_TEXTS:
            path = os.path.join(d, "rules.txt")
            with open(path, "wb") as fh:
                fh.write(text.encode())
            try:
                c = compile_ruleset(load_ruleset(path))
                res["rules"].append({"columns": {f: getattr(c, f).astype(np.int64).tolist() for f in RULE_FIELDS}})
            except RuleParseError as exc:
                res["rules"].append({"error": str(exc).replace(path, "{path}")})
        for body in parser_cases.TRAFFIC_BODIES:
            path = os.path.join(d, "t.csv")
            with open(path, "wb") as fh:
                fh.write((parser_cases.TRAFFIC_HEADER + body).encode())
            try:
                pk = load_traffic(path)
                res["traffic"].append({"packets": [[p.id, int(p.proto), p.src_ip, p.src_port, p.dst_ip, p.dst_port]
                                                   for p in pk]})
            except TrafficFormatError as exc:
                res["traffic"].append({"error": str(exc).replace(path, "{path}")})
    path = os.path.join(OUT, "parsers.json")
    with open(path, "w") as fh:
        json.dump(res, fh)
    print(f"wrote parsers.json: {os.path.getsize(path)} bytes")


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="", help="comma-separated subset: rng,rules,scans,engines,adversarial,"
                                               "worst_case,parsers")
    only = set(filter(None, ap.parse_args().only.split(",")))
    t0 = time.time()
    if not only:
        gen_rng()
        rules, traffic = {}, {}
        gen_rulesets(rules)
        gen_traffic(traffic)
        gen_scans(rules, traffic)
        gen_engines(rules, traffic)
        gen_adversarial()
    if not only or "worst_case" in only:
        gen_worst_case()
    if not only or "parsers" in only:
        gen_parsers()
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
