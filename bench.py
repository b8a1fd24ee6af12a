#!/usr/bin/env python
"""Benchmark of the B200 packet-filter hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config data|grid|function|adversarial|oracle]
    python bench.py --impl reference ...     # the reference's own Python CPU path (baseline/_ref)

One step = one pass of the hot path over one batch: every packet of this
rank's share of the workload classified (first-match index + verdict +
per-packet comparison count) against the whole ruleset (data-parallel / grid
/ adversarial / oracle configs) or against this rank's rule shard followed by
the per-packet MIN all-reduce (function-parallel).  Inputs are resident in
HBM when the timed region starts; L2 (126 MB) is flushed between timed steps
by writing a 256 MiB buffer.  Each step is timed with CUDA events on the
launching stream; steps are bracketed by a barrier + synchronize; the job
time is the MAX over ranks.  Rank 0 prints ONE JSON line.

``--gpus N`` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one GPU each, NCCL); it fails loudly when
fewer than N GPUs are visible.  The default config is BASELINE.json
configs[1]: 10K rules, 64Mi packets sharded over the GPUs (total work fixed:
"strong" scaling); for N > 1 the line also carries a "weak" record (every
rank scans a full 64Mi shard of an N x 64Mi stream).

The reference arm (``--impl reference``) runs the UNMODIFIED reference package
installed in baseline/_ref (pure Python + numpy) through its own public API:
``Engine(EngineConfig(DATA_PARALLEL, nodes=os.cpu_count(), batch_size=N,
executor="process")).run`` -- the bench.run_point protocol of
parafw/bench.py:103-138 -- on a bounded sample of the same workload (same
generators and seeds), plus single-core ``classify_batch_sequential``.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpackets/sec vs rule count at 1/2/4/8 B200; % of HBM/INT32 roofline"
K_OPS = 10  # int32 ops per rule test: 5 fields x (compare + combine), SURVEY.md 8(d)
INT32_LANES_PER_SM_CLK = 128  # 4 SMSP x 32 lanes, issue bound across ALU + FMA pipes
# algorithmic bytes per packet: uint4 in; uint32 index + u8 verdict + uint32 comparisons out
PKT_BYTES, OUT_BYTES = 16, 9
MS_BYTES_PER_RULE = 0.5       # match-set scan: one bit per rule from each of the 4 rows
# reference-arm samples (packets): ~1-10 s per Engine.run of the Python reference
REF_SAMPLE = {"oracle": 100_000, "data": 100_000, "grid": 100_000, "function": 4_000, "adversarial": 20_000}
SEQ_SAMPLE = {"oracle": 20_000, "data": 10_000, "grid": 10_000, "function": 2_000, "adversarial": 2_000}
# C-port samples: ~10-30 core-seconds of the oracle's scan (~3.3 ns per rule test per core)
PORT_SAMPLE = {"oracle": 100_000, "data": 2_000_000, "grid": 2_000_000, "function": 1_000_000,
               "adversarial": 100_000}


# ------------------------------------------------------------------ peaks

def load_l2_peak():
    """Measured L2 read bandwidth (tools/l2_probe.cu, committed under profiles/):
    (random 128-byte-line ceiling -- the match-set scan's access pattern --,
    streaming ceiling, source)."""
    path = os.path.join(ROOT, "profiles", "l2_peak.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        stream = float(d["l2_read_gbs"])
        return float(d.get("l2_random_line_read_gbs", stream)), stream, d.get("source", path)
    except (OSError, ValueError, KeyError):
        return None, None, None


def probe_l2_live(dev) -> dict | None:
    """The roofline peak measured on this device in this run: random 128-byte
    lines read by 8-lane groups from a 48 MiB L2-resident buffer (the
    match-set scan's access pattern; pfw_probe_l2_lines), 8/16 lines in
    flight per lane x 5/6/8 blocks per SM (the round-1 sweep's best region;
    ~2 ms launches: shorter ones read low), best shape."""
    import torch
    from paper_1312_4188_b200 import _native
    try:
        buf = torch.empty(48 << 20, dtype=torch.uint8, device=dev)
        buf.fill_(1)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        st = torch.cuda.current_stream(dev)
        lib = _native.lib()
        best, shape = 0.0, None
        for occ in (5, 6, 8):
            for k in (8, 16):
                iters = max(128, 66000 // (occ * k))  # ~40 GB of line reads per timed launch (~2 ms)
                _native.check(lib.pfw_probe_l2_lines(buf.data_ptr(), buf.numel(), k, occ, 16, st.cuda_stream),
                              "pfw_probe_l2_lines")
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                _native.check(lib.pfw_probe_l2_lines(buf.data_ptr(), buf.numel(), k, occ, iters, st.cuda_stream),
                              "pfw_probe_l2_lines")
                e1.record(st)
                e1.synchronize()
                gbs = sms * occ * 32 * k * iters * 128 / (e0.elapsed_time(e1) * 1e6)
                if gbs > best:
                    best, shape = gbs, {"blocks_per_sm": occ, "lines_in_flight_per_lane": k}
        del buf
        return {"gbs": round(best, 1), "shape": shape}
    except Exception as e:  # noqa: BLE001 (the file figure is the fallback)
        print(f"bench.py: live L2 probe failed ({e}); using profiles/l2_peak.json", file=sys.stderr)
        return None


def load_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_source": "fallback (B200_PROFILING.md)"}


def measured_traffic(key: str, n: int):
    """dram__bytes_read.sum + dram__bytes_write.sum (and, for the match-set
    scan, the L2 read sectors) of one step, from the committed ncu --set full
    capture (profiles/traffic.json), scaled to n packets."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh).get(key)
    except (OSError, ValueError):
        return None
    if not d:
        return None
    out = {"bytes_per_step": round(d["dram_bytes_per_step"] * n / d["packets"]),
           "bytes_per_packet": round(d["dram_bytes_per_step"] / d["packets"], 1), "source": d["source"]}
    if "l2_read_bytes_per_step" in d:
        out["l2_read_bytes_per_packet"] = round(d["l2_read_bytes_per_step"] / d["packets"], 1)
    return out


class ClockSampler:
    """SM clock + clock-event reasons sampled through NVML every 2 ms while
    the timed region runs (B200_PROFILING.md clocks line)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device: int) -> None:
        self.device = device
        self.sm: list[float] = []
        self.max_mhz = None
        self.reasons: set[str] = set()
        self.stop = threading.Event()
        self.thread = None
        self.source = None

    def _handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        p = torch.cuda.get_device_properties(self.device)
        try:
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(
                f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0")
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)

    def _loop(self, nv, h):
        flags = [(name, getattr(nv, attr, 0)) for name, attr in self.REASONS]
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, bit in flags:
                    if bit and r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self.stop.wait(0.002)

    def __enter__(self):
        try:
            nv, h = self._handle()
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.source = "nvml, 2 ms"
            self.thread = threading.Thread(target=self._loop, args=(nv, h), daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz, "sm_min_mhz": min(self.sm),
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": self.source}


def host_link_peaks(dev) -> dict:
    """Pinned host -> device copy bandwidth on this box (512 MiB, best of 6,
    CUDA events): the ceiling of the e2e path's input stream."""
    import torch
    src = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
    dst = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, src.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return {"h2d_gbs": round(best, 2), "source": "measured: pinned 512 MiB H2D copy, best of 6"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spawn_ranks(n: int) -> int:
    """--gpus N outside torchrun: re-launch this command under
    torch.distributed.run with N local ranks (NCCL, one GPU each)."""
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py --gpus {n}: only {have} CUDA device(s) visible", file=sys.stderr, flush=True)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ------------------------------------------------------------ CPU baselines

def cpu_info() -> dict:
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        import psutil
        physical = psutil.cpu_count(logical=False)
    except Exception:
        physical = None
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"cpu_model": model, "logical_cores": os.cpu_count(), "physical_cores": physical,
            "usable_cores": usable}


def ref_import():
    """The unmodified reference package (pip-installed into baseline/_ref)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "parafw")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import parafw
    return parafw


def ref_workload(name: str, rules: int, n: int):
    """The workload's ruleset and first n packets, built with the reference's
    own generators (the adversarial recipe from reference
    primitives) -- the same inputs the GPU arm generates on the device."""
    from parafw.model import Action, CidrMatcher, PortRange, Protocol, Rule, Ruleset
    from parafw.traffic import RulesetGenParams, TrafficProfile, generate_ruleset, generate_traffic
    if name != "adversarial":
        return (generate_ruleset(RulesetGenParams(rules, seed=1)),
                generate_traffic(TrafficProfile(count=n, seed=2)))
    head = Rule(Action.ACCEPT, Protocol.ANY, CidrMatcher(0, 0), PortRange(0, 65535),
                CidrMatcher(0xC0000000, 2), PortRange(0, 65535))
    n_decoy = int(rules * 0.9)
    decoys = []
    for r in generate_ruleset(RulesetGenParams(n_decoy, seed=2)):
        dst = CidrMatcher(0x80000000, 1) if r.dst.prefix_len == 0 else \
            CidrMatcher(r.dst.base | 0x80000000, r.dst.prefix_len)
        decoys.append(Rule(r.action, r.proto, r.src, r.sport, dst, r.dport))
    tail = list(generate_ruleset(RulesetGenParams(rules - 1 - n_decoy, seed=1)))
    total = 1 << 22  # the workload's 90% / 10% split point is on the full stream
    n_late = int(total * 0.9)
    late = generate_traffic(TrafficProfile(count=min(n, n_late), seed=7, dst_subnet=CidrMatcher(0, 1)))
    early = generate_traffic(TrafficProfile(count=max(0, n - n_late), seed=8,
                                            dst_subnet=CidrMatcher(0xC0000000, 2))) if n > n_late else []
    return Ruleset((head, *decoys, *tail)), late + early


def reference_cpu(name: str, rules: int, model: str, steps: int, warmup: int, sample: int = 0) -> dict:
    """Time the reference's Python path on this host's cores: the
    bench.run_point protocol (parafw/bench.py:103-138) -- a persistent
    Engine(EngineConfig(DATA_PARALLEL [FUNCTION_PARALLEL for the function
    config], nodes=os.cpu_count(), batch_size=N, executor="process")), one
    untimed warm-up run, then ``steps`` timed runs (ClassifyStats.wall_time_ns:
    the reference's own timed region, compile + pack + dispatch + results) --
    and single-core classify_batch_sequential on a smaller sample."""
    parafw = ref_import()
    if parafw is None:
        return {"unavailable": "baseline/_ref/parafw not installed"}
    from parafw.classifier import classify_batch_sequential
    from parafw.engines import MAX_NODES, Engine, EngineConfig, ExecutionModel
    n = sample or REF_SAMPLE[name]
    t0 = time.perf_counter()
    rs, pk = ref_workload(name, rules, n)
    gen_s = time.perf_counter() - t0
    nodes = max(1, min(os.cpu_count() or 1, MAX_NODES))
    em = ExecutionModel.FUNCTION_PARALLEL if model == "function" else ExecutionModel.DATA_PARALLEL
    cfg = EngineConfig(em, nodes=nodes, batch_size=len(pk), executor="process")
    walls, comps = [], None
    with Engine(cfg) as eng:
        for i in range(max(1, warmup) + steps):
            _, st = eng.run(rs, pk)
            if i >= max(1, warmup):
                walls.append(st.wall_time_ns)
                comps = st.total_comparisons
    med = statistics.median(walls)
    ns = SEQ_SAMPLE[name]
    _, sst = classify_batch_sequential(rs, pk[:ns])
    return {"value": len(pk) / (med / 1e9) / 1e6, "unit": "Mpps", "cores": nodes, "kind": "reference",
            "sample": f"{len(pk)} packets x {len(rs)} rules of the {name} workload (reference generators, "
                      f"same seeds); parafw Engine(EngineConfig({em.name}, nodes={nodes}, batch_size={len(pk)}, "
                      f"executor='process')).run, median of {len(walls)} runs after a warm-up (bench.run_point "
                      "protocol)",
            "ms_per_run": med / 1e6, "runs": len(walls), "total_comparisons": comps, "sample_packets": len(pk),
            "sequential_1core": {"value": ns / (sst.wall_time_ns / 1e9) / 1e6, "unit": "Mpps", "packets": ns,
                                 "api": "parafw.classify_batch_sequential"},
            "generation_s": round(gen_s, 2), "source": "baseline/_ref (unmodified parafw 0.1.0, pip-installed)",
            **cpu_info()}


def port_cpu(w, sample: int, threads: int = 0) -> dict:
    """The oracle's C restatement of scan_range (test infrastructure; data-
    parallel over packets on all host threads) on the first ``sample``
    packets of the same workload -- reported beside the reference as
    ``cpu_port``."""
    import numpy as np
    from oracle import oracle
    if w.name == "adversarial":
        rules = oracle.adversarial_rules(w.rules)
        pk = oracle.adversarial_traffic(w.packets)
        pk = {k: v[:sample] for k, v in pk.items()}
    else:
        rules = oracle.gen_ruleset(w.rules, 1)
        pk = oracle.gen_traffic_uniform(sample, 2)
    nthreads = threads or oracle.max_threads()
    t0 = time.perf_counter()
    if w.model == "function":
        first, comps, total, _ = oracle.engine_run(rules, pk, "data", 1, nthreads)
    else:
        first = oracle.scan_range(rules, pk, 0, w.rules, nthreads)
        comps = oracle.sequential_comparisons(first, w.rules)
    dt = time.perf_counter() - t0
    return {"value": sample / dt / 1e6, "unit": "Mpps", "cores": nthreads, "kind": "port",
            "sample": f"{sample} packets of the {w.name} workload x {w.rules} rules "
                      f"(oracle/fw_oracle.c orc_scan_range, pthreads over packets)",
            "seconds": dt, "comparisons": int(np.asarray(comps).sum())}


def reference_subprocess(config: str, timeout: int = 600) -> dict | None:
    """The reference arm in a fresh interpreter (no CUDA context, no host
    threads of ours under the reference's fork-based process pool)."""
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--config", config, "--steps", "3",
           "--warmup", "1", "--no-port"]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout,
                             env={k: v for k, v in os.environ.items()
                                  if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
        line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
        return json.loads(line)
    except Exception as exc:  # the GPU line still prints; say why the baseline is missing
        return {"unavailable": f"reference subprocess failed: {exc!r}"[:300]}


def run_reference(args, w, world, rank) -> int:
    if rank != 0:
        return 0
    ref = reference_cpu(w.name, w.rules, w.model, args.steps, args.warmup, args.cpu_sample)
    if "unavailable" in ref:
        print(json.dumps({"impl": "reference", "unavailable": ref["unavailable"]}), flush=True)
        return 0
    line = {
        "impl": "reference", "metric": METRIC, "value": ref["value"], "unit": "Mpps", "n_gpus": world,
        "steps": ref["runs"], "warmup": max(1, args.warmup), "ms_per_step": ref["ms_per_run"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (reference generators: rules seed 1, packets seed 2)",
        "config": {"workload": w.description, "rules": w.rules, "packets": ref["sample_packets"],
                   "execution_model": w.model, "parallelism": f"{ref['cores']} worker processes (host cores)"},
        "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "reference": ref,
        "e2e": {"value": ref["value"], "unit": "Mpps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_port:
        line["cpu_port"] = {k: v for k, v in port_cpu(w, min(PORT_SAMPLE[w.name], w.packets)).items()
                            if k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- main

def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="data", choices=("data", "grid", "function", "adversarial", "oracle"))
    ap.add_argument("--packets", type=int, default=0, help="override the workload's packet count")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="strong",
                    help="packet-sharded configs: strong = the workload's packets split over the ranks "
                         "(BASELINE.json configs[1], default); weak = every rank scans its own full-size "
                         "shard of an N-times larger global stream")
    ap.add_argument("--cpu-sample", type=int, default=0, help="reference-arm packets per run")
    ap.add_argument("--l2", choices=("flush", "stream"), default="flush",
                    help="between timed steps: flush L2 (256 MiB write), or rely on the packet inputs being "
                         "larger than L2 (the ruleset tables stay resident, as in a deployed filter)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-port", action="store_true", help="skip the C-port CPU figure")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-rule-scan", action="store_true", help="skip the rule-by-rule scan sub-record")
    ap.add_argument("--graph", action="store_true",
                    help="capture one step (all pass launches) in a CUDA graph and replay it")
    ap.add_argument("--e2e-chunk", type=int, default=1 << 23,
                    help="packets per H2D/scan/D2H chunk (ramped down at both ends of the call)")
    ap.add_argument("--algo", type=int, default=-1,
                    help="0 auto (match sets when built), 1 rule-by-rule scan, 2 match sets")
    ap.add_argument("--ms-words", type=int, default=0, help="match-set scan: words per lane per step (1, 2, 4)")
    ap.add_argument("--ms-group", type=int, default=0, help="match-set scan: lanes per packet (8, 16, 32)")
    ap.add_argument("--ms-summary", type=int, default=-1, help="match-set block summaries: 0 off, 1 on, 2 auto")
    ap.add_argument("--ms-compress", type=int, default=-1, help="compressed match-set rows: 0 off, 1 on, 2 auto")
    ap.add_argument("--ms-lean", type=int, default=-1,
                    help="whole-table plain-row scans: 0 general kernel, 1 lean kernel, 2 lean + L1 no-allocate")
    ap.add_argument("--tune", action="append", default=[], metavar="KEY=VALUE",
                    help="any pfw_set_tuning key (repeatable), applied before the ruleset is built")
    ap.add_argument("--ks", type=int, default=0)
    ap.add_argument("--sc", type=int, default=-1, help="warp-level short-circuit of the port tests (0/1)")
    ap.add_argument("--bucket", type=int, default=-1, help="group large batches by protocol (0/1)")
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--first-pass", type=int, default=-1, help="rules in the first pass (0 = single pass)")
    ap.add_argument("--proto-split", action="store_true",
                    help="scan protocol-split rule chains (opt-in algorithmic extension; the "
                         "roofline then over-counts: it charges the reference's comparisons)")
    ap.add_argument("--fused", action="store_true",
                    help="function config: combine fused into the scan epilogue (NVLink atomics via "
                         "CUDA IPC, reduce-scatter result) instead of the NCCL all-reduce")
    args = ap.parse_args()

    from paper_1312_4188_b200 import workloads
    w = workloads.WORKLOADS[args.config]
    if args.packets:
        w = workloads.Workload(w.name, w.rules, args.packets, w.model, w.description)
    world, rank, local = dist_setup()

    if args.impl == "reference":
        return run_reference(args, w, world, rank)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus)
    if world != args.gpus and os.environ.get("PFW_SHARE_GPU") != "1":
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr, flush=True)
        return 2
    return run_ours(args, w, world, rank, local)


def run_ours(args, w, world, rank, local) -> int:
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1312_4188_b200 import _native, parallel, workloads
    from paper_1312_4188_b200.classifier import CompiledRuleset
    from paper_1312_4188_b200.engines import Engine, EngineConfig, ExecutionModel

    # PFW_SHARE_GPU=1: every rank on cuda:0 with gloo collectives on host copies --
    # a functional check of the N-rank path on a 1-GPU box (kernels of
    # different ranks never wait on each other).  Normal runs: one GPU per
    # rank, NCCL over NVLink/NVSwitch.
    share = os.environ.get("PFW_SHARE_GPU") == "1"
    if share:
        local = 0
    if torch.cuda.device_count() <= local:
        print(f"bench.py: rank {rank} needs GPU {local}, {torch.cuda.device_count()} visible", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    tunings = {"algo": args.algo, "ms_words": args.ms_words or -1, "ms_group": args.ms_group or -1,
               "ms_summary": args.ms_summary, "ms_compress": args.ms_compress, "ms_lean": args.ms_lean, "ks": args.ks or -1,
               "short_circuit": args.sc, "bucket": args.bucket, "tile": args.tile or -1,
               "first_pass": args.first_pass, "proto_split": 1 if args.proto_split else -1}
    for k, v in tunings.items():
        if v >= 0:
            _native.set_tuning(k, v)
    for kv in args.tune:
        k, _, v = kv.partition("=")
        _native.set_tuning(k, int(v))
    peaks = load_peaks()
    dev = torch.device(f"cuda:{local}")
    info = parallel.RankInfo(rank, world)

    # ---------------------------------------------------------- workload
    cols = workloads.rule_columns(w)
    R = len(cols["proto"])
    if w.model == "function":
        # rules sharded: this rank uploads only its partition (its own match
        # sets, local windows, global indices)
        r_lo, r_hi = parallel.rule_shard(R, info)
        compiled = CompiledRuleset.from_columns({k: v[r_lo:r_hi] for k, v in cols.items()}, device=local,
                                                shard=(r_lo, R))
    else:
        r_lo, r_hi = 0, R
        compiled = CompiledRuleset.from_columns(cols, device=local)
    ms_bytes = int(_native.lib().pfw_ruleset_matchset_bytes(compiled.handle))
    rule_scan = args.algo == 1 or args.proto_split or args.sc == 1
    algo = "matchset" if ms_bytes and not rule_scan else "rule scan"
    weak = args.scaling == "weak" and w.model != "function"
    total_packets = w.packets * world if weak else w.packets

    def shard_packets(total, start_rank_packets=None):
        """This rank's packets of a global stream of `total` packets."""
        if w.model == "function":
            return workloads.packets(w, 0, w.packets, local)          # packets replicated
        a, b = parallel.packet_shard(total, info)
        wgen = workloads.Workload(w.name, w.rules, total, w.model, w.description)
        return workloads.packets(wgen, a, b - a, local)

    pkts = shard_packets(total_packets)
    n = len(pkts)
    first = torch.empty(n, dtype=torch.int32, device=dev)
    comps = torch.empty(n, dtype=torch.int32, device=dev)
    verdict = torch.empty(n, dtype=torch.uint8, device=dev)
    stats = torch.zeros(2, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_l2 = args.l2 == "flush"
    stream = torch.cuda.current_stream(dev)

    fused = None
    if args.fused and w.model == "function":
        fused = parallel.FusedFunctionParallel(compiled, n, scatter=True, with_comps=True)

    def make_step(batch, out_first, out_comps, out_verdict):
        m = len(batch)

        def step(zero=True):
            # (the timed loop zeroes the stats once before its first step and
            # lets the steps accumulate them: no per-step fill launch)
            if zero:
                stats.zero_()
            if fused is not None:
                fused.run(batch, stats=stats, stream=stream.cuda_stream)
            elif w.model == "function":
                # this rank's shard is ONE partition of the model (engines.py:316-321):
                # its scan writes the shard-local first match (global index) and the
                # per-task comparisons directly (no accumulator pass), then the
                # NCCL MIN / SUM combine across ranks (engines.py:202-212, 359-369)
                compiled.scan_range_device(batch, 0, compiled.num_rules, first=out_first, comps=out_comps,
                                           stats=stats, stream=stream.cuda_stream)
                parallel.function_parallel_combine(out_first, out_comps, None)
            else:
                compiled.scan_range_device(batch, r_lo, r_hi, first=out_first, comps=out_comps,
                                           verdict=out_verdict, stats=stats, stream=stream.cuda_stream)
        return step

    step = make_step(pkts, first, comps, verdict)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            if share:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def timed(run_step, steps, clocks=None):
        """steps timed launches (CUDA events on the launching stream, L2
        flushed before each) -> total ms of this rank.  The steps are queued
        back to back (flush, event, step, event) with one synchronize after the
        last: the host enqueues ahead of the device (each flush alone is ~40 us
        of device time), so an event pair times the step's device execution,
        not the host's launch latency."""
        evs = []
        barrier()
        torch.cuda.synchronize(dev)
        for _ in range(steps):
            if flush_l2:
                flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_step()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize(dev)
        barrier()
        return sum(a.elapsed_time(b) for a, b in evs)

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        parallel.all_reduce(t, dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        parallel.all_reduce(t, dist.ReduceOp.SUM)
        return float(t.item())

    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    barrier()
    run_step = lambda: step(False)  # noqa: E731
    graph_launches = 0  # kernels per replay (replays bypass the library's launch counter)
    if args.graph and fused is None and world == 1:
        # the library launches on the caller's stream, so stream capture
        # records every pass of the multi-pass scan into one graph
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            stream_saved = stream
            stream = cap
            before = _native.launch_count()
            with torch.cuda.graph(g, stream=cap):
                step(False)
            graph_launches = _native.launch_count() - before
            stream = stream_saved
        torch.cuda.synchronize()
        run_step = g.replay
        run_step()
        torch.cuda.synchronize()
    # algorithmic work of one step: sum of this rank's (per-task) comparisons
    stats.zero_()
    run_step()
    local_comps = int(stats[0].item())
    # the match-set scan with block summaries skips blocks: count the blocks it
    # reads in one extra (untimed) step for its roofline
    blocks_read = 0
    if algo == "matchset":
        _native.read_counter("blocks_read")
        _native.set_tuning("count_blocks", 1)
        step()
        torch.cuda.synchronize()
        _native.set_tuning("count_blocks", 0)
        blocks_read = _native.read_counter("blocks_read")

    launches0 = _native.launch_count()
    stats.zero_()
    with ClockSampler(local) as clocks:
        total_ms = timed(run_step, args.steps)
    # every timed step ran the whole scan: the accumulated comparisons say so
    timed_comps = int(stats[0].item())
    if fused is None and timed_comps != local_comps * args.steps:
        raise RuntimeError(f"timed steps accumulated {timed_comps} comparisons, expected "
                           f"{args.steps} x {local_comps}")
    launches = _native.launch_count() - launches0 + graph_launches * args.steps
    job_ms = max_over_ranks(total_ms)
    pk_per_step = w.packets if w.model == "function" else int(sum_over_ranks(float(n)))
    value = pk_per_step * args.steps / (job_ms / 1e3) / 1e6
    ms_per_step = job_ms / args.steps

    # --- roofline for the dominant kernel (the scan), per GPU
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk = float(peaks.get("sm_max_mhz", 1965.0))
    avg_launch_s = (total_ms / args.steps) / 1e3
    hbm_achieved = n * (PKT_BYTES + OUT_BYTES) / avg_launch_s / 1e9
    hbm = {"achieved": round(hbm_achieved, 2), "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
           "frac": round(hbm_achieved / float(peaks.get("hbm_gbs", 6536.4)), 5),
           "bytes_per_packet": PKT_BYTES + OUT_BYTES}
    l2_peak, l2_stream, l2_src = load_l2_peak()
    l2_file = l2_peak
    live = probe_l2_live(dev) if algo == "matchset" else None
    if live:
        l2_peak = live["gbs"]
        l2_src = (f"measured in this run on this device (pfw_probe_l2_lines: random 128-byte lines, 8-lane "
                  f"groups, 48 MiB L2-resident buffer, best of 6 shapes: {live['shape']}); "
                  f"round-1 probe file: {l2_file} GB/s")
    int_peak = sms * INT32_LANES_PER_SM_CLK * clk * 1e6 / 1e12  # T int-ops/s
    int_peak_src = (f"derived: {sms} SMs x {INT32_LANES_PER_SM_CLK} int32 lanes/clk x sm_max_mhz {clk:.0f} "
                    f"({peaks['_source']})")
    if algo == "matchset" and l2_peak:
        if blocks_read:
            # block summaries: the search reads the packet's 4 summary rows
            # (sw words each) and the 4 rows' 128-byte line of every block it
            # visits (counted by the kernel) + the packet in / results out
            wp = -(-(-(-R // 32)) // 128) * 128
            sw = -(-(wp // 32) // 32)
            alg_bytes = blocks_read * 4 * 128 + n * (4 * 4 * sw + PKT_BYTES + OUT_BYTES)
            model = {"bytes_model": "block summaries: 4 rows x 128 B per block read (kernel-counted) + "
                                    f"4 x 4 B x summary words + {PKT_BYTES + OUT_BYTES} B packet in / results out",
                     "blocks_read_per_launch": blocks_read,
                     "blocks_read_per_packet": round(blocks_read / max(n, 1), 2)}
        else:
            # bytes the first-match search must read: one bit per rule resolved
            # from each of the 4 rows (comparisons = the reference's algorithmic
            # work) + the packet in / results out
            alg_bytes = local_comps * MS_BYTES_PER_RULE + n * (PKT_BYTES + OUT_BYTES)
            model = {"bytes_model": f"0.5 B per rule resolved (1 bit x 4 rows) + {PKT_BYTES + OUT_BYTES} B "
                                    "packet in / results out",
                     "bytes_per_rule_resolved": MS_BYTES_PER_RULE, "rules_resolved_per_launch": local_comps}
        achieved = alg_bytes / avg_launch_s / 1e9
        roof = {
            "bound": "l2", "achieved": round(achieved, 1), "peak": l2_peak, "unit": "GB/s",
            "frac": round(achieved / l2_peak, 4), "traffic": measured_traffic(f"{w.name}/matchset", n),
            "algorithmic_bytes_per_launch": round(alg_bytes),
            "algorithmic_bytes_per_packet": round(alg_bytes / max(n, 1), 1), **model,
            "peak_source": "measured L2 read bandwidth for this kernel's access pattern (random 128-byte "
                           f"lines, 8-lane groups; {l2_src})",
            "peak_l2_streaming": l2_stream, "frac_of_streaming_peak": round(achieved / l2_stream, 4),
            "hbm": hbm,
        }
    else:
        achieved = local_comps * K_OPS / avg_launch_s / 1e12
        roof = {
            "bound": "int32", "achieved": round(achieved, 3), "peak": round(int_peak, 3), "unit": "Tops/s",
            "frac": round(achieved / int_peak, 4), "traffic": measured_traffic(w.name, n),
            "ops_per_rule_test": K_OPS, "rule_tests_per_launch": local_comps, "peak_source": int_peak_src,
            "hbm": hbm,
        }

    # --- BASELINE.json north_star figure: Mpps as a fraction of the slower of
    # two rooflines -- HBM for the packet bytes, INT32 for the reference's rule
    # comparisons (K ops each).  The rule-by-rule scan is that formulation; the
    # match-set scan resolves comparisons without evaluating them one by one,
    # so it can exceed it (frac > 1).
    int_peak_ops = int_peak * 1e12
    comps_pp = local_comps / max(n, 1)
    int32_pps = int_peak_ops / (K_OPS * max(comps_pp, 1e-9))
    hbm_pps = float(peaks.get("hbm_gbs", 6536.4)) * 1e9 / (PKT_BYTES + OUT_BYTES)
    per_gpu_pps = n / avg_launch_s
    ns_roof = {"definition": "per-GPU Mpps / min(HBM roofline: packet bytes, INT32 roofline: "
                             f"{K_OPS} int ops per reference comparison)",
               "bound": "int32" if int32_pps < hbm_pps else "hbm",
               "roofline_mpps": round(min(int32_pps, hbm_pps) / 1e6, 1),
               "int32_roofline_mpps": round(int32_pps / 1e6, 1), "hbm_roofline_mpps": round(hbm_pps / 1e6, 1),
               "frac": round(per_gpu_pps / min(int32_pps, hbm_pps), 4)}

    # --- the rule-by-rule scan (the north_star's own formulation: TMA-staged
    # rule tiles, warp-ballot first match, integer ALU) on the same inputs,
    # timed the same way, against the INT32 roofline
    rule_rec = None
    if algo == "matchset" and not args.no_rule_scan and fused is None:
        # on the first 1/8 of this rank's packets (>= 4Mi): the rule scan is
        # ~10x slower per packet, so the whole stream would make it the
        # dominant kernel of the default bench command's launch list (its
        # multi-pass compaction loses a little at smaller batches: 0.676 of
        # the INT32 peak at 64Mi packets, 0.646 at 8Mi)
        m = min(n, max(1 << 22, n // 8))
        sub = pkts.slice(0, m)
        rstep_ = make_step(sub, first[:m], comps[:m], verdict[:m])
        _native.set_tuning("algo", 1)
        try:
            rstep_()
            torch.cuda.synchronize()
            r_comps = int(stats[0].item())  # the sample's comparisons (make_step zeroes stats per step)
            rsteps = max(3, min(args.steps, 5))
            launches_r0 = _native.launch_count()
            with ClockSampler(local) as rclocks:
                r_ms = timed(lambda: rstep_(False), rsteps)
            r_launches = _native.launch_count() - launches_r0
            r_job = max_over_ranks(r_ms)
            r_pk = int(sum_over_ranks(float(m))) if w.model != "function" else m
            r_avg_s = r_ms / rsteps / 1e3
            r_ach = r_comps * K_OPS / r_avg_s / 1e12
            r_int32_pps = int_peak_ops / (K_OPS * max(r_comps / max(m, 1), 1e-9))
            rule_rec = {"value": round(r_pk * rsteps / (r_job / 1e3) / 1e6, 3), "unit": "Mpps",
                        "packets_per_gpu": m, "sample": f"packets [0, {m}) of this rank's stream",
                        "steps": rsteps, "ms_per_step": round(r_job / rsteps, 4),
                        "roofline": {"bound": "int32", "achieved": round(r_ach, 3), "peak": round(int_peak, 3),
                                     "unit": "Tops/s", "frac": round(r_ach / int_peak, 4),
                                     "traffic": measured_traffic(w.name, m), "ops_per_rule_test": K_OPS,
                                     "rule_tests_per_launch": r_comps, "peak_source": int_peak_src},
                        "north_star_frac": round((m / r_avg_s) / min(r_int32_pps, hbm_pps), 4),
                        "clocks": rclocks.summary(), "gpu_launches": r_launches,
                        "kernel": "scan_kernel (rule-by-rule range-test grid, TMA bulk stage ring, ballot/ffs)"}
        finally:
            _native.set_tuning("algo", args.algo if args.algo >= 0 else 0)

    # --- weak scaling (N > 1): every rank scans a full-size shard of an
    # N x larger global stream
    weak_rec = None
    if world > 1 and not weak and w.model != "function":
        wp_ = shard_packets(w.packets * world)
        nw = len(wp_)
        wf = torch.empty(nw, dtype=torch.int32, device=dev)
        wc = torch.empty(nw, dtype=torch.int32, device=dev)
        wv = torch.empty(nw, dtype=torch.uint8, device=dev)
        wstep = make_step(wp_, wf, wc, wv)
        wstep()
        with ClockSampler(local) as wclocks:
            w_ms = timed(lambda: wstep(False), args.steps)
        w_job = max_over_ranks(w_ms)
        w_total = int(sum_over_ranks(float(nw)))
        weak_rec = {"value": round(w_total * args.steps / (w_job / 1e3) / 1e6, 3), "unit": "Mpps",
                    "packets": w_total, "packets_per_gpu": nw, "ms_per_step": round(w_job / args.steps, 4),
                    "clocks": wclocks.summary()}
        del wp_, wf, wc, wv

    # --- end to end through the public API with host buffers:
    # Engine.run_arrays over the reference's PacketArrays columns in host
    # memory (classifier.py:62-95, 13 B/packet); H2D, scans and D2H of the
    # first-match index + verdict inside the timed region
    e2e = None
    fn_e2e = w.model == "function"  # (N = 1 only: ranks hold rule shards, not whole rulesets)
    if not args.no_e2e and (w.model != "function" or (world == 1 and fused is None)):
        hc = pkts.columns()
        pinned = {}
        for f, a in hc.items():
            t = torch.empty(a.shape, dtype={1: torch.uint8, 2: torch.int16, 4: torch.int32}[a.itemsize],
                            pin_memory=True)
            t.numpy().view(a.dtype)[:] = a
            pinned[f] = t.numpy().view(a.dtype)
        eng = Engine(EngineConfig(ExecutionModel.FUNCTION_PARALLEL, nodes=world) if fn_e2e
                     else EngineConfig(ExecutionModel.DATA_PARALLEL), device=local)
        ref_first = first.cpu().numpy()

        def e2e_step(batch):
            return eng.run_arrays(compiled, batch)
        for _ in range(max(1, args.warmup)):
            res = e2e_step(pinned)
        # parity of the e2e path with the device-resident path (bit-exact)
        if not np.array_equal(np.where(res.first < 0, 0x7FFFFFFF, res.first), ref_first):
            raise SystemExit("e2e first-match indices differ from the device path")

        def wall(batch, steps):
            et = []
            for _ in range(steps):
                barrier()
                t0 = time.perf_counter()
                e2e_step(batch)
                et.append(time.perf_counter() - t0)
            return max_over_ranks(sum(et))
        launches_e0 = _native.launch_count()
        e_s = wall(pinned, args.steps)
        e_launches = (_native.launch_count() - launches_e0) // args.steps
        psteps = max(3, min(args.steps, 5))
        e2e_step(hc)  # (the first pageable call allocates the handle's pinned staging ring)
        pg_s = wall(hc, psteps)  # pageable numpy columns: staged through the native pinned ring
        link = host_link_peaks(dev)
        e2e_s = e_s / args.steps
        e2e = {"value": pk_per_step * args.steps / e_s / 1e6, "unit": "Mpps",
               # (one node: the whole-table pipeline, comparisons derived on the host as first + 1
               # or R; several nodes: pfw_classify_host_partitions copies them out too)
               "h2d_bytes_per_step": n * 13, "d2h_bytes_per_step": n * (9 if fn_e2e and world > 1 else 5),
               "api": (f"Engine(EngineConfig(FUNCTION_PARALLEL, nodes={world})).run_arrays(compiled, host_columns) "
                       "-> EngineResult (one node = the sequential scan exactly: the same chunked H2D / scan / "
                       "D2H pipeline, first + verdict copied out, per-packet comparisons derived)" if fn_e2e else
                       "Engine(EngineConfig(DATA_PARALLEL)).run_arrays(compiled, host_columns) -> EngineResult "
                       "(the reference's five PacketArrays columns as numpy arrays in pinned host memory; "
                       "pfw_classify_host_ex: chunked H2D / scan / D2H pipeline, copy-in + 2 compute + copy-out "
                       "streams; results int32 first (-1 = default deny) + bool verdict in pinned memory)"),
               "kernel_launches_per_step": e_launches,
               # the host link bounds this path: H2D of the 13-byte columns
               "h2d_gbs": round(n * 13 / e2e_s / 1e9, 2), "h2d_peak_gbs": link["h2d_gbs"],
               "h2d_frac": round(n * 13 / e2e_s / 1e9 / link["h2d_gbs"], 4),
               "link_peak_source": link["source"],
               "pageable": {"value": pk_per_step * psteps / pg_s / 1e6, "unit": "Mpps", "steps": psteps,
                            "api": "the same call over ordinary (pageable) numpy columns: staged chunk by "
                                   "chunk through the handle's pinned ring by the native host thread pool"}}

    cpu = port = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ref = reference_subprocess(args.config)
        if ref and "reference" in ref:
            r = ref["reference"]
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
            cpu.update({k: r[k] for k in ("sequential_1core", "cpu_model", "logical_cores", "physical_cores",
                                          "usable_cores", "total_comparisons") if k in r})
        else:
            cpu = ref
        if not args.no_port:
            c = port_cpu(w, min(PORT_SAMPLE[w.name], w.packets))
            port = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Mpps", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic: generate_ruleset(RulesetGenParams(R, seed=1)) x generate_traffic("
                    "TrafficProfile(N, seed=2)), generated on the GPU bit-exactly",
            "config": {"workload": w.description, "rules": R, "packets": total_packets,
                       "packets_per_gpu": n, "execution_model": w.model,
                       **({"rules_per_gpu": [r_lo, r_hi]} if w.model == "function" else {}),
                       "parallelism": f"{'rule' if w.model == 'function' else 'packet'}-sharded x{world}"
                                      + (" (fused NVLink-atomic combine)" if fused is not None else
                                         " (NCCL MIN all-reduce)" if w.model == "function" else ""),
                       "l2": ("flushed between timed steps (256 MiB write)" if flush_l2 else
                              f"not flushed: packet inputs ({n * 16 / 2**20:.0f} MiB per GPU) larger than L2, "
                              "ruleset tables resident"),
                       "outputs": "first-match index + verdict + per-packet comparisons + [sum, max] stats",
                       "algorithm": (f"match-set scan (per-field interval bitmaps, {ms_bytes / 2**20:.0f} MiB"
                                     + (", compressed rows" if _native.ruleset_info(compiled.handle, "compressed") else "")
                                     + (", block summaries" if blocks_read else "") + ")"
                                     if algo == "matchset" else "rule-by-rule scan"),
                       "rule_layout": "protocol-split chains" if args.proto_split else "single ordered table",
                       "kernel": _native.version()},
            "roofline": roof,
            "roofline_north_star": ns_roof,
            "rule_scan": rule_rec,
            "weak": weak_rec,
            "cpu_baseline": cpu,
            "cpu_port": port,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "gpu_launches": launches,
            "comparisons_per_packet": round(local_comps / max(n, 1), 2) if w.model != "function" else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
