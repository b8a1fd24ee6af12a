"""paper_1312_4188_b200: B200-native first-match packet filtering.

Drop-in for the classify path of the reference ``parafw`` package
(arXiv 1312.4188, "Parallel Firewalls on GPGPU"): the same Rule / Ruleset /
Packet / MatchResult types, the same Engine / EngineConfig / ExecutionModel /
run* API and the same seeded generators, with every rule x packet scan run by
hand-written sm_100a CUDA kernels in ``libpfw.so`` (C-ABI: include/pfw.h).
There is no CPU fallback.
"""

from .model import (Action, CidrMatcher, MatchResult, Packet, PortRange, Protocol, Rule,
                    RuleParseError, Ruleset, format_rule, load_ruleset, parse_rule, rule_matches,
                    save_ruleset)
from .classifier import (ClassifyStats, CompiledRuleset, PacketArrays, classify,
                         classify_batch_sequential, compile_ruleset)
from .engines import (ConfigError, Engine, EngineConfig, EngineResult, ExecutionModel, PartialMatch,
                      RulePartition, aggregate, combine_partition_matches, partition_bounds,
                      partition_rules, run, run_data_parallel, run_function_parallel, run_hybrid,
                      scan_partition)
from .traffic import (MatchMode, RulesetGenParams, TrafficFormatError, TrafficGenerationError,
                      TrafficProfile, generate_ruleset, generate_traffic, generate_traffic_device,
                      load_traffic, save_traffic)


__version__ = "0.2.0"


def __getattr__(name):
    # FirewallClassifier pulls in scikit-learn: import on demand (as the reference does)
    if name == "FirewallClassifier":
        from .estimator import FirewallClassifier
        return FirewallClassifier
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")

__all__ = [
    "FirewallClassifier",
    "Action", "CidrMatcher", "ClassifyStats", "CompiledRuleset", "ConfigError", "Engine",
    "EngineConfig", "EngineResult", "ExecutionModel", "MatchMode", "MatchResult", "Packet",
    "PacketArrays", "PartialMatch", "PortRange", "Protocol", "Rule", "RuleParseError",
    "RulePartition", "Ruleset", "RulesetGenParams", "TrafficFormatError", "TrafficGenerationError",
    "TrafficProfile", "aggregate", "classify", "classify_batch_sequential",
    "combine_partition_matches", "compile_ruleset", "format_rule", "generate_ruleset",
    "generate_traffic", "generate_traffic_device", "load_ruleset", "load_traffic", "parse_rule",
    "partition_bounds", "partition_rules", "rule_matches", "run", "run_data_parallel",
    "run_function_parallel", "run_hybrid", "save_ruleset", "save_traffic", "scan_partition",
]
