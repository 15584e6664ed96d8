"""HashGraph build+query throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[4], the weak-scaling sweep, at C=1): every GPU
owns 2^28 uniform uint32 keys drawn from {1..2^28} (SplitMix64 stream seed =
rank, cli.py:101-107) and 2^28 queries (one stream, seed 0x51, rank slice,
cli.py:262-266).  A step = build the table over the GPU's keys + answer its
queries (query-side table + intersect).  N=1 runs the single-shard path; N>1
runs the partitioned path (bin histogram all-reduce, split plan, NCCL
all-to-all, local build; forward/backward query exchange).

`value` = (keys + queries processed by all ranks) / (max-over-ranks device
time), inputs resident in HBM.  `e2e` = the same metric through the public
API from pinned host buffers (H2D of keys+queries and D2H of the uint32
multiplicities inside the timed region).  `--impl reference` times the
reference algorithm's CPU restatement (oracle/, numpy, all host threads) on a
bounded sample of the same workload.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HashGraph build+query keys/sec at 1/2/4/8 B200; achieved HBM & NVLink GB/s"
UNIT = "keys/s"
QUERY_SEED = 0x51

# The oracle's answer for a bench workload, keyed by (log2 keys, k, load
# factor, key bits): the timed step's aggregates must equal it (checked after
# the timed region; tests/test_scale_parity_gpu.py recomputes it with oracle/).
EXPECTED = {
    (28, 28, 1.0, 32): {"matched": 169_672_492, "total": 268_422_361, "comparisons": 517_428_761},
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--log2-keys", type=int, default=28, help="keys (and queries) per GPU = 2^x")
    ap.add_argument("--k", type=int, default=28, help="keys drawn from {1..2^k}")
    ap.add_argument("--load-factor", type=float, default=1.0)
    ap.add_argument("--key-bits", type=int, default=32, choices=[32, 64],
                    help="64: full SplitMix64 words as keys (BASELINE configs[3])")
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--e2e-depth", type=int, default=3, help="e2e steps in flight (one stream and output buffer each)")
    ap.add_argument("--cpu-log2", type=int, default=24, help="CPU baseline sample size 2^x")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels eagerly instead of replaying a CUDA graph")
    ap.add_argument("--dist", action="store_true", help="use the partitioned (torch.distributed) path even at N=1")
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p",
                    help="partitioned path's key exchange: fused peer-memory scatter (p2p) or NCCL alltoallv")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks


class ClockSampler:
    """NVML sampling (in-process thread) of SM clock + throttle reasons during
    the timed region; falls back to an nvidia-smi subprocess."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period_s: float = 0.05):
        self.index = index
        self.period = period_s
        self.samples = []
        self.stop_flag = threading.Event()
        self.thread = None
        self.err = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self.stop_flag.is_set():
                    try:
                        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        reasons = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
                        self.samples.append((mhz, reasons, util))
                    except Exception as e:  # noqa: BLE001
                        self.err = str(e)
                    self.stop_flag.wait(self.period)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"

    def stop(self):
        self.stop_flag.set()
        if self.thread is not None:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"]}
        loaded = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = set()
        for _, r, _ in loaded:
            for name, bit in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in loaded), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples), "samples_under_load": len(loaded)}


# --------------------------------------------------------------------------- roofline bookkeeping


def algorithmic_bytes(name: str, n: int, q: int, v: int, w: int = 4) -> float:
    """Per-launch algorithmic bytes of each kernel (Kernels): the
    HBM bytes its job must move at minimum -- inputs read once, outputs
    written once; scratch such as counters is not counted."""
    table = {
        # direct (Alg. 1) path
        "hg_count": w * n,
        "hg_scan": 4 * v + 4 * (v + 1),
        "hg_place": 2 * w * n,
        "hg_place_pos": 2 * w * q + 4 * q,
        "hg_intersect": 2 * w * q + 4 * q + 4 * q + w * n + 4 * (v + 1),
        # binned path, build side (n keys)
        "hg_hist": w * n,
        "hg_part1": 2 * w * n,
        "hg_part2": 2 * w * n,
        "hg_local_build": 2 * w * n + 4 * (v + 1),
        # binned path, query side (q queries against n table keys)
        "hg_part1_q": 2 * w * q + 2 * q,
        "hg_part2_q": 2 * w * q + 2 * q,
        "hg_local_probe": w * q + w * n + 4 * (v + 1) + 4 * q,
        "hg_unpart2": 4 * q + 2 * q + 4 * q,
        "hg_unpart1": 4 * q + 2 * q + 4 * q,
    }
    return float(table.get(name, 0))


def a_build(n: int, v: int, w: int = 4) -> float:
    """A_build = 3 N w + 4 (V + 1)."""
    return 3.0 * n * w + 4.0 * (v + 1)


def a_query(n: int, q: int, v: int, w: int = 4) -> float:
    """A_query = 4 Q w + 12 Q + N w + 12 (V + 1)."""
    return 4.0 * q * w + 12.0 * q + n * w + 12.0 * (v + 1)


def summarize_kernels(records, steps, n, q, v, peak, w=4):
    agg = {}
    for name, ms in records:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    total = sum(a[1] for a in agg.values()) or 1.0
    rows = []
    for name, (cnt, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        avg = ms / cnt
        ab = algorithmic_bytes(name, n, q, v, w)
        rows.append({"kernel": name, "launches": cnt, "avg_ms": avg, "share": ms / total,
                     "achieved_gbs": (ab / (avg / 1e3) / 1e9) if ab else None})
    top = rows[0] if rows else None
    roof = None
    if top:
        ab = algorithmic_bytes(top["kernel"], n, q, v, w)
        ach = ab / (top["avg_ms"] / 1e3) / 1e9 if ab else None
        roof = {"bound": "hbm", "kernel": top["kernel"], "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": (ach / peak) if ach else None, "traffic": None, "share_of_step": top["share"],
                "algorithmic_bytes_per_launch": ab}
    return rows, roof


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# --------------------------------------------------------------------------- CPU baseline


def host_info() -> dict:
    """CPU model and RAM of the host the CPU arm runs on (BASELINE.md asks for both)."""
    model, ram_gb = "unknown", None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    ram_gb = round(int(line.split()[1]) / (1 << 20), 1)
                    break
    except OSError:
        pass
    return {"cpu_model": model, "ram_gb": ram_gb, "hw_threads": os.cpu_count()}


def cpu_sample(log2: int, k: int, lf: float, workers: int):
    """Reference algorithm (oracle restatement) on a bounded sample: build +
    query of 2^log2 keys / queries of the bench workload's streams."""
    import oracle as O

    n = 1 << log2
    keys = O.generate_keys(k, n, 0)
    queries = O.generate_keys(k, n, QUERY_SEED)
    v = O.hash_range_for(n, lf)
    t0 = time.perf_counter()
    off, placed, _ = O.build_csr(keys, v, workers=workers)
    t1 = time.perf_counter()
    O.query(off, placed, queries, workers=workers)
    t2 = time.perf_counter()
    return 2 * n / (t2 - t0), (t1 - t0), (t2 - t1)


# --------------------------------------------------------------------------- reference arm


def workload_name(args, kb: int = 32) -> str:
    """The workload both arms report (BASELINE configs[4], one point of the sweep)."""
    return (f"C5 weak scaling: 2^{args.log2_keys} uint{kb} keys + 2^{args.log2_keys} queries per GPU, "
            + (f"keys from {{1..2^{args.k}}}" if kb == 32 else "full 64-bit SplitMix64 words") + f", C={args.load_factor}")


def run_reference(args, rank, world):
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    log2 = min(args.cpu_log2, 22)
    for _ in range(args.warmup):
        cpu_sample(log2, args.k, args.load_factor, workers)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_sample(log2, args.k, args.load_factor, workers)[0])
    elapsed = time.perf_counter() - t0
    value = (2 << log2) * args.steps / elapsed
    sample = (f"per step: build+query of 2^{log2} uint32 keys and 2^{log2} queries (k={args.k}, C={args.load_factor}) "
              f"with the reference algorithm's numpy restatement (oracle/), worker_count={workers}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": workload_name(args), "keys_per_gpu": 1 << args.log2_keys,
                   "queries_per_gpu": 1 << args.log2_keys,
                   "sample": f"each step times 2^{log2} keys + 2^{log2} queries of the same streams on the host"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port", "sample": sample,
                         "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- B200 arm


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch

    import paper_2104_00792_b200 as hg
    from paper_2104_00792_b200 import _lib

    torch.cuda.set_device(local)
    dist = None
    use_dist = world > 1 or args.dist
    if use_dist:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = 1 << args.log2_keys
    q = n
    spec = hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, args.k, n, rank)
    qspec = hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, args.k, q * world, QUERY_SEED)
    kb = args.key_bits
    keys = hg.generate_device(spec, 0, n, key_bits=kb)
    queries = hg.generate_device(qspec, rank * q, q, key_bits=kb)
    torch.cuda.synchronize()

    if use_dist:
        from paper_2104_00792_b200 import distributed as hd

        cfg = hd.DistConfig(load_factor=args.load_factor, key_bits=kb, transport=args.transport)

        def step():
            table = hd.build_distributed(keys, cfg)
            res = hd.query_distributed(table, queries)
            return table, res
    else:
        def step():
            table = hg.build(keys, args.load_factor, key_bits=kb)
            res = hg.intersect(table, queries)
            return table, res

    v = hg.hash_range_for(n, args.load_factor)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    # N=1: the whole step (15 kernels) is captured once into a CUDA graph and
    # replayed, so host launch jitter cannot leave the GPU idle; the per-launch
    # timing events are captured with it (they hold the last replay's times).
    # N>1 steps contain host-synchronising collectives and run eagerly.
    use_graph = not use_dist and not args.no_graph
    timing = not os.environ.get("HG_BENCH_NO_TIMING")
    graph = None
    launches_per_step = None
    if use_graph:
        _lib.timing_enable(timing)
        _lib.timing_collect()
        l0 = _lib.launch_count()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            table, res = step()
        launches_per_step = _lib.launch_count() - l0
        _lib.timing_enable(False)
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()

    sampler = ClockSampler(local) if rank == 0 and not os.environ.get("HG_BENCH_NO_CLOCKS") else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if not use_graph:
        _lib.timing_enable(timing)
        _lib.timing_collect()
    launches0 = _lib.launch_count()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            table, res = step()
    e1.record()
    torch.cuda.synchronize()
    launches = (launches_per_step * args.steps) if use_graph else (_lib.launch_count() - launches0)
    records = _lib.timing_collect(1 << 16)
    _lib.timing_enable(False)
    clocks = sampler.stop() if sampler else None
    elapsed_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([elapsed_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
        dist.barrier()
    total_units = (n + q) * world * args.steps
    value = total_units / (elapsed_ms / 1e3)

    # the timed step's answer against the oracle's (EXPECTED; N=1 single-shard)
    check = None
    if not use_dist:
        exp = EXPECTED.get((args.log2_keys, args.k, float(args.load_factor), kb)) if kb == 32 else None
        got = {"matched": res.matched_positions, "total": res.total_matches, "comparisons": res.comparisons}
        check = {"step_aggregates": got, "expected": exp, "ok": (got == exp) if exp else None}
        if exp and got != exp:
            print(f"bench: timed step's aggregates {got} differ from the oracle's {exp}", file=sys.stderr)
            sys.exit(3)

    # build and query timed apart (graph replays, same inputs): the SURVEY
    # 8(d3) fractions of the whole build, the whole query and the step
    phases = None
    if use_graph:
        gb, gq = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gb):
            tb = hg.build(keys, args.load_factor, key_bits=kb)
        with torch.cuda.graph(gq):
            hg.intersect(tb, queries)
        gb.replay()
        gq.replay()
        reps = max(3, args.steps // 2)
        ms = {}
        for name, g in (("build", gb), ("query", gq)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(reps):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            ms[name] = a.elapsed_time(b) / reps
        del gb, gq, tb
        phases = {"build_ms": ms["build"], "query_ms": ms["query"], "replays": reps}

    peak, peak_kind = measured_peak()
    kernels, roof = summarize_kernels(records, args.steps, n, q, v, peak, kb // 8)
    if roof:
        roof["peak_source"] = f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else "fallback"
        roof["traffic"] = load_traffic(roof["kernel"])
        w = kb // 8
        ab, aq = a_build(n, v, w), a_query(n, q, v, w)
        step_ms = elapsed_ms / args.steps
        roof["step_frac"] = (ab + aq) / (step_ms / 1e3) / (peak * 1e9)
        roof["algorithmic_bytes"] = {"build": ab, "query": aq, "formula": "SURVEY 8(d3): 3Nw+4(V+1); 4Qw+12Q+Nw+12(V+1)"}
        if phases:
            roof["build_frac"] = ab / (phases["build_ms"] / 1e3) / (peak * 1e9)
            roof["query_frac"] = aq / (phases["query_ms"] / 1e3) / (peak * 1e9)
            roof.update({"build_ms": phases["build_ms"], "query_ms": phases["query_ms"]})

    # end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        sdt = torch.int32 if kb == 32 else torch.int64
        hk = torch.empty(n, dtype=sdt, pin_memory=True)
        hq = torch.empty(q, dtype=sdt, pin_memory=True)
        hk.copy_(keys.cpu())
        hq.copy_(queries.cpu())
        # `depth` steps in flight, one stream each (a serving loop): step
        # i+1's H2D overlaps step i's kernels and D2H; PCIe is full duplex, so
        # the step rate is bounded by the 2 GiB of inputs per step.  The host consumes
        # every step's result (waits for its D2H, reads it) before reusing
        # that step's output buffer.
        depth = args.e2e_depth
        streams = [torch.cuda.Stream() for _ in range(depth)]
        outs = [torch.empty(q, dtype=torch.int32, pin_memory=True) for _ in range(depth)]
        done = [None] * depth
        checksum = 0

        def e2e_step(i):
            nonlocal checksum
            slot = i % depth
            if done[slot] is not None:
                done[slot].synchronize()
                checksum ^= int(outs[slot][0])  # the host reads the previous result of this slot
            with torch.cuda.stream(streams[slot]):
                if use_dist:
                    table = hd.build_distributed(hk, cfg)
                    res = hd.query_distributed(table, hq)
                else:
                    table = hg.build(hk, args.load_factor, key_bits=kb)
                    res = hg.intersect(table, hq)
                outs[slot].copy_(res.multiplicities_device, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
                done[slot] = ev
            return res

        for i in range(depth):
            e2e_step(i)
        torch.cuda.synchronize()
        done = [None] * depth
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(args.e2e_steps):
            e2e_step(i)
            if os.environ.get("HG_E2E_TRACE"):
                print(f"e2e step {i} enqueued at {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        if dist:
            t = torch.tensor([e2e_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": (n + q) * world * args.e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": (kb // 8) * (n + q), "d2h_bytes_per_step": 4 * q,
               "ms_per_step": e2e_s / args.e2e_steps * 1e3,
               "pipeline": f"{depth} steps in flight on {depth} streams; host waits for and reads each result before reusing its buffer"}
        e2e["link"] = pcie_link(hk, outs[0], e2e)

    # end to end as a caller of the reference API sees it: numpy keys and
    # queries in, build + intersect, then the int64 multiplicities and the
    # aggregates read back (pageable host memory, one step at a time)
    e2e_ref = None
    if not args.no_e2e and not use_dist and world == 1:
        npk = keys.cpu().numpy().view(np.uint32 if kb == 32 else np.uint64)
        npq = queries.cpu().numpy().view(np.uint32 if kb == 32 else np.uint64)

        def ref_step():
            t_ = hg.build(npk, args.load_factor, key_bits=kb)
            r_ = hg.intersect(t_, npq)
            m_ = r_.multiplicities
            return int(m_[-1]) + r_.matched_positions + r_.total_matches + r_.comparisons

        ref_step()
        torch.cuda.synchronize()
        reps = max(2, args.e2e_steps // 2)
        t0 = time.perf_counter()
        for _ in range(reps):
            ref_step()
        e2e_ref_s = (time.perf_counter() - t0) / reps
        e2e_ref = {"value": (n + q) / e2e_ref_s, "unit": UNIT, "h2d_bytes_per_step": (kb // 8) * (n + q),
                   "d2h_bytes_per_step": 8 * q + 24, "ms_per_step": e2e_ref_s * 1e3,
                   "api": "hg.build(numpy keys); hg.intersect(table, numpy queries).multiplicities (int64) + "
                          "matched_positions/total_matches/comparisons; pageable host memory, one step at a time"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        val, tb, tq = cpu_sample(args.cpu_log2, args.k, args.load_factor, workers)
        cpu = {"value": val, "unit": UNIT, "cores": workers, "kind": "port", "host": host_info(),
               "sample": (f"2^{args.cpu_log2} keys + 2^{args.cpu_log2} queries of the same streams (k={args.k}, "
                          f"C={args.load_factor}); build {tb:.2f} s + query {tq:.2f} s with the numpy restatement "
                          f"of the reference (oracle/), worker_count={workers}")}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": f"u{kb}", "data": "synthetic",
        "config": {"workload": workload_name(args, kb),
                   "keys_per_gpu": n, "queries_per_gpu": q, "hash_range_per_gpu": v,
                   "l2": "inputs (1 GiB per array) larger than the 126 MB L2",
                   "parallelism": "single-shard" if not use_dist else f"partitioned over {world} GPU(s) ({'fused peer-memory exchange' if args.transport == 'p2p' else 'NCCL alltoallv'})",
                   "launch": "cuda_graph (one step captured, replayed per step)" if use_graph else "eager"},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "e2e_reference_api": e2e_ref, "gpu_launches": launches,
        "clocks": clocks, "check": check, "kernels": kernels,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def pcie_link(h_in, h_out, e2e):
    """The host link's own copy rates, measured here (pinned buffers, CUDA
    events, best of 3): H2D alone, D2H alone, and one step's copies with
    nothing else running -- its input bytes H2D on one stream while its
    result bytes go D2H on another.  That duplex time is the floor of a
    serving loop whose compute hides under the copies; `frac` = floor / the
    measured e2e step."""
    import torch

    d_in = torch.empty(h_in.numel(), dtype=h_in.dtype, device="cuda")
    d_out = torch.empty(h_out.numel(), dtype=h_out.dtype, device="cuda")
    in_b, out_b = h_in.numel() * h_in.element_size(), h_out.numel() * h_out.element_size()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    reps_in = max(1, round(e2e["h2d_bytes_per_step"] / in_b))  # copies of h_in per step's inputs
    reps_out = max(1, round(e2e["d2h_bytes_per_step"] / out_b))

    def timed(fn):
        best = float("inf")
        for _ in range(3):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s_in.wait_stream(torch.cuda.current_stream())
            s_out.wait_stream(torch.cuda.current_stream())
            fn()
            torch.cuda.current_stream().wait_stream(s_in)
            torch.cuda.current_stream().wait_stream(s_out)
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    def up():
        with torch.cuda.stream(s_in):
            for _ in range(reps_in):
                d_in.copy_(h_in, non_blocking=True)

    def down():
        with torch.cuda.stream(s_out):
            for _ in range(reps_out):
                h_out.copy_(d_out, non_blocking=True)

    t_up, t_down = timed(up), timed(down)
    t_both = timed(lambda: (up(), down()))
    return {"h2d_GBps": reps_in * in_b / t_up / 1e6, "d2h_GBps": reps_out * out_b / t_down / 1e6,
            "step_copies_alone_ms": t_both, "frac": t_both / e2e["ms_per_step"]}


def load_traffic(kernel: str):
    """dram bytes per launch from a committed `ncu --set full` capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


if __name__ == "__main__":
    main()
