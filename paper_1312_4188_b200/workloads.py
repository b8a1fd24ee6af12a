"""The BASELINE.json workloads, built with this package's own generators.

Rules: ``generate_ruleset(RulesetGenParams(R, seed=1))``; packets:
``generate_traffic(TrafficProfile(N, seed=2))``, generated
on the device.  The adversarial ruleset follows the SURVEY.md 8(d) recipe.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .classifier import RULE_COLUMNS, PacketArrays, _rule_columns
from .model import CidrMatcher
from .traffic import RulesetGenParams, TrafficProfile, generate_ruleset, generate_traffic_device


@dataclass(frozen=True)
class Workload:
    name: str
    rules: int
    packets: int
    model: str          # data | function | grid (data-parallel scan) | sequential
    description: str


WORKLOADS = {
    "oracle": Workload("oracle", 1000, 100_000, "data",
                       "1,000 rules x 100K packets, sequential first-match (verdict oracle config)"),
    "data": Workload("data", 10_000, 1 << 26, "data",
                     "data-parallel: 10K rules replicated per GPU, 64Mi packets sharded across GPUs"),
    "function": Workload("function", 100_000, 1 << 24, "function",
                         "function-parallel: 100K rules split across GPUs, per-packet min-index allreduce"),
    "grid": Workload("grid", 4096, 1 << 24, "data",
                     "packet x rule grid: 16Mi packets x 4K rules, warp-ballot first-match"),
    "adversarial": Workload("adversarial", 50_000, 1 << 22, "data",
                            "adversarial: 50K rules, 90% of traffic late-matching or default-deny"),
}


def rule_columns(w: Workload) -> dict:
    if w.name == "adversarial":
        return adversarial_rule_columns(w.rules)
    return _rule_columns(generate_ruleset(RulesetGenParams(w.rules, seed=1)))


def adversarial_rule_columns(total: int = 50_000) -> dict:
    """Rule 0 ACCEPT any * * 192.0.0.0/2 *; rules 1..0.9*total: seed-2 random
    rules with every dst forced into 128.0.0.0/1; the rest seed-1 random rules."""
    n_decoy = int(total * 0.9)
    head = {f: np.zeros(1, dtype=np.asarray(0, dtype=t).dtype) for f, t in zip(
        RULE_COLUMNS, (np.uint8, np.uint32, np.uint32, np.uint16, np.uint16, np.uint32, np.uint32,
                       np.uint16, np.uint16, np.bool_))}
    head["dst_base"][0] = head["dst_mask"][0] = 0xC0000000
    head["sport_hi"][0] = head["dport_hi"][0] = 65535
    head["action_accept"][0] = True
    dec = _rule_columns(generate_ruleset(RulesetGenParams(n_decoy, seed=2)))
    wild = dec["dst_mask"] == 0
    dec["dst_base"] = np.where(wild, np.uint32(0x80000000), dec["dst_base"] | np.uint32(0x80000000)).astype(np.uint32)
    dec["dst_mask"] = np.where(wild, np.uint32(0x80000000), dec["dst_mask"]).astype(np.uint32)
    tail = _rule_columns(generate_ruleset(RulesetGenParams(total - 1 - n_decoy, seed=1)))
    return {f: np.concatenate([head[f], dec[f], tail[f]]) for f in RULE_COLUMNS}


def packets(w: Workload, start: int, count: int, device: int) -> PacketArrays:
    """Packets [start, start+count) of the workload's global stream."""
    if w.name != "adversarial":
        return generate_traffic_device(TrafficProfile(w.packets, seed=2), device, start, count)
    import torch
    n_late = int(w.packets * 0.9)
    late = TrafficProfile(n_late, seed=7, dst_subnet=CidrMatcher(0, 1))
    early = TrafficProfile(w.packets - n_late, seed=8, dst_subnet=CidrMatcher(0xC0000000, 2))
    parts = []
    a, b = start, start + count
    if a < n_late:
        parts.append(generate_traffic_device(late, device, a, min(b, n_late) - a).data)
    if b > n_late:
        s = max(a, n_late) - n_late
        parts.append(generate_traffic_device(early, device, s, b - n_late - s).data)
    return PacketArrays(torch.cat(parts) if len(parts) > 1 else parts[0])
