#!/usr/bin/env python
"""Benchmark of the B200 packet-filter hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config data|grid|function|adversarial|oracle]
    python bench.py --impl reference ...     # the CPU arm (oracle C port, all host cores)

One step = one pass of the hot path over one batch: every packet of this
rank's share of the workload classified (first-match index + verdict +
comparison counters) against the whole ruleset (data-parallel / grid /
adversarial / oracle configs) or against this rank's rule shard followed by
the per-packet MIN all-reduce (function-parallel).  Inputs are resident in
HBM when the timed region starts; L2 (126 MB) is flushed between timed steps
by writing a 256 MiB buffer.  Each step is timed with CUDA events on the
launching stream; steps are bracketed by a barrier + synchronize; the job
time is the MAX over ranks.  Rank 0 prints ONE JSON line.

The default config is BASELINE.json configs[1] (data-parallel, 10K rules,
64Mi packets sharded over the GPUs: total work fixed -> "strong" scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K_OPS = 10  # int32 ops per rule test: 5 fields x (compare + combine), SURVEY.md 8(d)
INT32_LANES_PER_SM_CLK = 128  # 4 SMSP x 32 lanes, issue bound across ALU + FMA pipes
PKT_BYTES, OUT_BYTES = 16, 5  # algorithmic bytes per packet: uint4 in, uint32 index + u8 verdict out
MS_BYTES_PER_RULE = 0.5       # match-set scan: one bit per rule from each of the 4 rows


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


def load_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int) -> None:
        self.device = device
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "20",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self.thread is not None:
                self.thread.join(timeout=2)

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, r[5:9]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


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


def host_link_peaks(dev) -> dict:
    """Pinned host -> device copy bandwidth on this box (512 MiB, best of 5,
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


def cpu_arm(w, sample: int, threads: int = 0) -> dict:
    """The reference path on the host cores: the oracle's C restatement of
    scan_range (data-parallel over packets, all host threads) on the first
    ``sample`` packets of the same workload."""
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


def run_reference(args, w, world, rank) -> None:
    if rank != 0:
        return
    sample = args.cpu_sample or CPU_SAMPLE[w.name]
    sample = min(sample, w.packets)
    runs = []
    for i in range(args.warmup + args.steps):
        r = cpu_arm(w, sample)
        if i >= args.warmup:
            runs.append(r)
    val = statistics.median(r["value"] for r in runs)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "Mpps", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(r["seconds"] for r in runs) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (reference generators: rules seed 1, packets seed 2)",
        "config": {"workload": w.description, "rules": w.rules, "packets": sample,
                   "parallelism": "cpu threads"},
        "cpu_baseline": {k: runs[0][k] for k in ("kind", "cores", "sample")} | {"value": val, "unit": "Mpps"},
        "e2e": {"value": val, "unit": "Mpps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "Mpackets/sec vs rule count at 1/2/4/8 B200; % of HBM/INT32 roofline"
# CPU-arm samples: ~10-30 core-seconds of the oracle's scan (~3.3 ns per rule test per core)
CPU_SAMPLE = {"oracle": 100_000, "data": 2_000_000, "grid": 2_000_000, "function": 1_000_000,
              "adversarial": 100_000}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="data", choices=("data", "grid", "function", "adversarial", "oracle"))
    ap.add_argument("--packets", type=int, default=0, help="override the workload's packet count")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="packet-sharded configs: weak = every rank scans its own full-size shard of "
                         "an N-times larger global stream (default); strong = the workload's packets "
                         "split over the ranks")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
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
        run_reference(args, w, world, rank)
        return 0

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1312_4188_b200 import _native, parallel
    from paper_1312_4188_b200.classifier import CompiledRuleset

    # PFW_SHARE_GPU=1: every rank on cuda:0 with gloo collectives on host copies --
    # a functional check of the N-rank path on a 1-GPU box (kernels of
    # different ranks never wait on each other).  Normal runs: one GPU per
    # rank, NCCL over NVLink/NVSwitch.
    share = os.environ.get("PFW_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    if args.algo >= 0:
        _native.set_tuning("algo", args.algo)
    if args.ms_words:
        _native.set_tuning("ms_words", args.ms_words)
    if args.ms_group:
        _native.set_tuning("ms_group", args.ms_group)
    if args.ms_summary >= 0:
        _native.set_tuning("ms_summary", args.ms_summary)
    if args.ms_compress >= 0:
        _native.set_tuning("ms_compress", args.ms_compress)
    if args.ks:
        _native.set_tuning("ks", args.ks)
    if args.sc >= 0:
        _native.set_tuning("short_circuit", args.sc)
    if args.bucket >= 0:
        _native.set_tuning("bucket", args.bucket)
    if args.tile:
        _native.set_tuning("tile", args.tile)
    if args.first_pass >= 0:
        _native.set_tuning("first_pass", args.first_pass)
    if args.proto_split:
        _native.set_tuning("proto_split", 1)
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
    if w.model == "function":
        p_lo, p_hi = 0, w.packets                       # packets replicated
    else:
        # packets sharded: contiguous partition_bounds shards of the global stream
        p_lo, p_hi = parallel.packet_shard(total_packets, info)
    # the generator draws from the global stream of total_packets packets
    wgen = workloads.Workload(w.name, w.rules, total_packets, w.model, w.description)
    pkts = workloads.packets(wgen, p_lo, p_hi - p_lo, local)
    n = len(pkts)
    first = torch.empty(n, dtype=torch.int32, device=dev)
    comps = torch.empty(n, dtype=torch.int32, device=dev)
    verdict = torch.empty(n, dtype=torch.uint8, device=dev)
    stats = torch.zeros(2, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    fused = None
    if args.fused and w.model == "function":
        fused = parallel.FusedFunctionParallel(compiled, n, scatter=True, with_comps=True)

    def step():
        stats.zero_()
        if fused is not None:
            fused.run(pkts, stats=stats, stream=stream.cuda_stream)
        elif w.model == "function":
            _native.check(_native.lib().pfw_accumulator_init(n, first.data_ptr(), comps.data_ptr(),
                                                             stream.cuda_stream), "init")
            compiled.scan_partition_accumulate(pkts, 0, compiled.num_rules, first, comps, stats,
                                               stream=stream.cuda_stream)
            parallel.function_parallel_combine(first, comps, None)
        else:
            compiled.scan_range_device(pkts, r_lo, r_hi, first=first, verdict=verdict,
                                       stats=stats, stream=stream.cuda_stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            if share:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    barrier()
    run_step = step
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
                step()
            graph_launches = _native.launch_count() - before
            stream = stream_saved
        torch.cuda.synchronize()
        run_step = g.replay
        run_step()
        torch.cuda.synchronize()
    # algorithmic work of one step: sum of this rank's (per-task) comparisons
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

    times = []
    launches0 = _native.launch_count()
    with ClockSampler(local) as clocks:
        barrier()
        for _ in range(args.steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        barrier()
    launches = _native.launch_count() - launches0 + graph_launches * args.steps
    total_ms = sum(times)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    tot = torch.tensor([float(n if w.model != "function" else 0), float(local_comps)],
                       dtype=torch.float64, device=dev)
    parallel.all_reduce(t, dist.ReduceOp.MAX)
    parallel.all_reduce(tot, dist.ReduceOp.SUM)
    job_ms = float(t.item())
    pk_per_step = w.packets if w.model == "function" else int(tot[0].item())
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
    if algo == "matchset" and l2_peak:
        if blocks_read:
            # block summaries: the search reads the packet's 4 summary rows
            # (sw words each) and the 4 rows' 128-byte line of every block it
            # visits (counted by the kernel) + the packet in / results out
            wp = -(-(-(-R // 32)) // 128) * 128
            sw = -(-(wp // 32) // 32)
            alg_bytes = blocks_read * 4 * 128 + n * (4 * 4 * sw + PKT_BYTES + OUT_BYTES)
            model = {"bytes_model": "block summaries: 4 rows x 128 B per block read (kernel-counted) + "
                                    "4 x 4 B x summary words + 21 B packet in / results out",
                     "blocks_read_per_launch": blocks_read,
                     "blocks_read_per_packet": round(blocks_read / max(n, 1), 2)}
        else:
            # bytes the first-match search must read: one bit per rule resolved
            # from each of the 4 rows (comparisons = the reference's algorithmic
            # work) + the packet in / results out
            alg_bytes = local_comps * MS_BYTES_PER_RULE + n * (PKT_BYTES + OUT_BYTES)
            model = {"bytes_model": "0.5 B per rule resolved (1 bit x 4 rows) + 21 B packet in / results out",
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
        int_peak = sms * INT32_LANES_PER_SM_CLK * clk * 1e6 / 1e12  # T int-ops/s
        achieved = local_comps * K_OPS / avg_launch_s / 1e12
        roof = {
            "bound": "int32", "achieved": round(achieved, 3), "peak": round(int_peak, 3), "unit": "Tops/s",
            "frac": round(achieved / int_peak, 4), "traffic": measured_traffic(w.name, n),
            "ops_per_rule_test": K_OPS, "rule_tests_per_launch": local_comps,
            "peak_source": f"derived: {sms} SMs x {INT32_LANES_PER_SM_CLK} int32 lanes/clk x "
                           f"sm_max_mhz {clk:.0f} ({peaks['_source']})",
            "hbm": hbm,
        }

    # --- BASELINE.json north_star figure: Mpps as a fraction of the slower of
    # two rooflines -- HBM for the packet bytes, INT32 for the reference's rule
    # comparisons (K ops each).  The rule-by-rule scan is that formulation; the
    # match-set scan resolves comparisons without evaluating them one by one,
    # so it can exceed it (frac > 1).
    int_peak_ops = sms * INT32_LANES_PER_SM_CLK * clk * 1e6
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

    # --- end to end through the C-ABI with host buffers (pfw_classify_host)
    e2e = None
    if not args.no_e2e and w.model != "function":
        # host input in the reference's own layout: the five PacketArrays columns
        # (classifier.py:62-95, 13 B/packet), pinned; nothing is packed on the host
        hc = pkts.columns()
        dt = {np.dtype(np.uint8): np.uint8, np.dtype(np.uint16): np.int16, np.dtype(np.uint32): np.int32}
        host_cols = [torch.from_numpy(hc[f].view(dt[hc[f].dtype])).pin_memory()
                     for f in ("proto", "src_ip", "src_port", "dst_ip", "dst_port")]
        h_first = torch.empty(n, dtype=torch.int32).pin_memory()
        h_verd = torch.empty(n, dtype=torch.uint8).pin_memory()
        h_stats = torch.zeros(2, dtype=torch.int64)
        lib = _native.lib()

        def e2e_step():
            _native.check(lib.pfw_classify_host_columns(
                compiled.handle, *[t.data_ptr() for t in host_cols], n, h_first.data_ptr(),
                h_verd.data_ptr(), h_stats.data_ptr(), args.e2e_chunk), "pfw_classify_host_columns")
        for _ in range(max(1, args.warmup)):
            e2e_step()
        # parity of the e2e path with the device-resident path (bit-exact)
        if not torch.equal(h_first, first.cpu()):
            raise SystemExit("e2e first-match indices differ from the device path")
        barrier()
        et = []
        for _ in range(args.steps):
            barrier()
            t0 = time.perf_counter()
            e2e_step()
            et.append(time.perf_counter() - t0)
        tt = torch.tensor([sum(et)], dtype=torch.float64, device=dev)
        parallel.all_reduce(tt, dist.ReduceOp.MAX)
        e2e_s = float(tt.item()) / args.steps
        link = host_link_peaks(dev)
        e2e = {"value": pk_per_step * args.steps / float(tt.item()) / 1e6, "unit": "Mpps",
               "h2d_bytes_per_step": n * 13, "d2h_bytes_per_step": n * 5,
               # the host link bounds this path: H2D of the 13-byte columns
               "h2d_gbs": round(n * 13 / e2e_s / 1e9, 2), "h2d_peak_gbs": link["h2d_gbs"],
               "h2d_frac": round(n * 13 / e2e_s / 1e9 / link["h2d_gbs"], 4),
               "link_peak_source": link["source"],
               "api": f"pfw_classify_host_columns (C-ABI, the reference's PacketArrays columns in "
                      f"pinned host memory, {args.e2e_chunk}-packet chunks ramped 1/8-1/4-1/2 at both ends, "
                      "copy-in / 2x compute / "
                      "copy-out streams, 3 slots)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sample = args.cpu_sample or CPU_SAMPLE[w.name]
        c = cpu_arm(w, min(sample, w.packets))
        cpu = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}

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
                       "l2": "flushed between timed steps (256 MiB write)",
                       "algorithm": (f"match-set scan (per-field interval bitmaps, {ms_bytes / 2**20:.0f} MiB"
                                     + (", compressed rows" if _native.ruleset_info(compiled.handle, "compressed") else "")
                                     + (", block summaries" if blocks_read else "") + ")"
                                     if algo == "matchset" else "rule-by-rule scan"),
                       "rule_layout": "protocol-split chains" if args.proto_split else "single ordered table",
                       "kernel": _native.version()},
            "roofline": roof,
            "roofline_north_star": ns_roof,
            "cpu_baseline": cpu,
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
