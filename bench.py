#!/usr/bin/env python
"""Benchmark of the Parallel Space Saving hot path on B200 (one JSON line on rank 0).

A step is one pass of the whole hot path over the workload:
pss_summarize (K1) -> pss_merge (K2) -> pss_prune (K3) -> pss_verify (K4) -> pss_report (K5),
all through the C-ABI of libpss.so, inputs resident in HBM. Default workload: the metric's
configuration (BASELINE.json "metric": n = 2^29 uint32 Zipf(1.1), k = 1000), P = 8192.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload H] [--impl ours|reference]

N > 1 runs under torchrun (one process per GPU, NCCL): every rank owns an equal shard of one
longer stream (weak scaling); the rank-local subtree roots are all-gathered and the top levels of
the same fixed tree are finished on every rank, then exact counts are all-reduced
(paper_1606_04669_b200/dist.py). `--impl reference` times the CPU oracle instead (the reference
arm of this tier): a bounded sample of the same workload per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gitems/s for summarize+merge (and verify) at n=2^29, k=1000; % of HBM roofline"
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="H")
    ap.add_argument("--P", type=int, default=0, help="override the number of partitions")
    # a custom synthetic workload: any of these overrides the named workload's field
    ap.add_argument("--n", type=int, default=0, help="override the number of keys (per GPU)")
    ap.add_argument("--k", type=int, default=0, help="override the number of counters")
    ap.add_argument("--zipf-s", type=float, default=0.0, help="override the Zipf skew")
    ap.add_argument("--universe", type=float, default=0.0, help="override the universe size")
    ap.add_argument("--seed", type=int, default=-1, help="override the generator seed")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0, help="default: min(steps, 5)")
    ap.add_argument("--no-e2e", action="store_true",
                    help="profiling runs only: skip the end-to-end leg (e2e is then null)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    ap.add_argument("--no-stream", action="store_true", help="skip the on-line stream leg (f2)")
    ap.add_argument("--stream-passes", type=int, default=4,
                    help="stream leg: the workload's array fed this many times (one stream)")
    return ap.parse_args()


def workload_of(args):
    """The named BASELINE workload with the command line's overrides (a 'custom' workload)."""
    import dataclasses

    import inputs
    w = inputs.WORKLOADS[args.workload]
    ov = {}
    if args.n:
        ov["n"] = args.n
    if args.k:
        ov["k"] = args.k
    if args.P:
        ov["P"] = args.P
    if args.zipf_s:
        ov["s"] = args.zipf_s
    if args.universe:
        ov["universe"] = args.universe
    if args.seed >= 0:
        ov["seed"] = args.seed
    if set(ov) - {"P"}:
        ov["name"] = w.name + "-custom"
    return dataclasses.replace(w, **ov) if ov else w


# ------------------------------------------------------------------------------ helpers
def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy kernel, read+write)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def ncu_traffic(workload: str):
    """dram bytes of one summarize+merge (K1 + tree + root COMBINE) from committed ncu captures."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(workload, {}).get("summarize_merge_dram_bytes_per_launch")
    return float(v) if v is not None else None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------------------ oracle arms
def oracle_sample(w, seconds: float, threads: int, A_host=None):
    """Time the oracle, as it stands, on the first S blocks of the workload (S sized so one run
    takes about `seconds`). Returns (items/s, description, threads)."""
    import numpy as np

    import inputs
    import oracle

    chunk = w.n // w.P
    A1 = A_host[:chunk] if A_host is not None else w.generate(chunk)
    t0 = time.perf_counter()
    oracle.space_saving(A1, w.k)
    t1 = max(time.perf_counter() - t0, 1e-4)
    S = int(max(1, min(w.P, threads * max(1, math.floor(seconds * 0.8 / t1)))))
    S = 1 << int(math.log2(S)) if S > 1 else 1
    m = S * chunk
    A = A_host[:m] if A_host is not None else w.generate(m)
    t0 = time.perf_counter()
    pl = oracle.pipeline(np.ascontiguousarray(A), w.k, S, threads=threads)
    dt = time.perf_counter() - t0
    desc = (f"first {S} of {w.P} blocks ({m} keys, {100.0 * m / w.n:.2f}% of n), k={w.k}: "
            f"leaves + fixed tree + prune + verify + report, oracle/pss_oracle.c via ctypes, "
            f"leaves on {threads} threads of {cpu_model()}; one core: {chunk / t1 / 1e6:.1f} "
            f"Mitems/s (Space Saving on one block)")
    del pl
    return m / dt, desc, threads, dt


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def run_reference(args):
    """--impl reference: the CPU oracle timed on this box's host cores (the tier's reference arm)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import inputs

    w = workload_of(args)
    T = host_threads()
    budget = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    chunk = w.n // w.P
    rates = []
    desc = ""
    for i in range(args.warmup + args.steps):
        rate, desc, cores, dt = oracle_sample(w, budget, T)
        if i >= args.warmup:
            rates.append(rate)
    v = statistics.median(rates) / 1e9
    line = {"metric": METRIC, "value": v, "unit": "Gitems/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_of(w),
            "data": "synthetic", "impl": "reference",
            "config": config_of(w, w.P, args.gpus),
            "cpu_baseline": {"value": v, "unit": "Gitems/s", "cores": T, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": v, "unit": "Gitems/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def dtype_of(w):
    return "u32" if w.key_bytes == 4 else "u64"


def config_of(w, P, gpus):
    d = w.describe()
    d["P"] = P
    d["global_n"] = w.n * gpus
    d["parallelism"] = f"dp{gpus}" if gpus > 1 else "1gpu"
    if l2_flush_needed(w):
        d["l2"] = (f"inputs of {w.n * w.key_bytes / 2**20:.0f} MiB/GPU could stay in the 126 MB L2: "
                   f"{L2_FLUSH_BYTES >> 20} MiB written between timed steps (outside the timed spans)")
    else:
        d["l2"] = (f"inputs larger than L2 ({w.n * w.key_bytes / 2**30:.1f} GiB/GPU streamed per "
                   f"pass vs 126 MB L2), no flush needed")
    return d


L2_FLUSH_BYTES = 256 << 20


def l2_flush_needed(w) -> bool:
    """Inputs of up to twice the L2 size are flushed out of it between timed steps."""
    return w.n * w.key_bytes <= 2 * 126 * 10**6


# ------------------------------------------------------------------------------ accuracy (f3)
def accuracy_leg(pss, runner, d_A, n, k):
    """The paper's accuracy metrics of the last timed step's answer, against the exact
    k-majority set computed without Space Saving (pss_exact_kmajority, timed here with CUDA
    events: a second exact method, two passes over A). Not part of the timed step."""
    import torch
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        _, _, n_true, over = pss.pss_exact_kmajority(d_A, k)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    cand, n_cand = runner.cand
    rep = pss.pss_accuracy(runner.top, n, n_cand, runner.exact, n_true).as_dict()
    rep["exact_kmajority_ms"] = round(min(ts), 3)
    rep["exact_kmajority_overflow"] = int(over.item())
    return rep


# ------------------------------------------------------------------------------ stream leg (f2)
def stream_leg(pss, w, P, h_A, d_A, passes, dev):
    """On-line ingestion (pss_stream_*): one stream of passes * n keys (the
    workload's array fed `passes` times), leaves of n/P keys, then its root and the on-line
    candidates (pss_prune; no verification pass in the on-line setting). Timed with CUDA events on
    the stream, once from device memory (K1 + incremental merges) and once from pinned host memory
    (pieces of batch_leaves leaves copied on a private stream, overlapped with the kernels); the
    host leg is bound by the host->device link, measured here with a plain pinned copy."""
    import torch
    n, kb = w.n, w.key_bytes
    kt = pss.KEY_U32 if kb == 4 else pss.KEY_U64
    st_dev = torch.cuda.current_stream()
    out = {}
    # device feeds: one K1 launch per P leaves (a full GPU); host feeds: pieces of P/4 leaves, so
    # that only a quarter of the last piece's copy-to-kernel latency is not overlapped
    batches = {"device": P, "host": max(1, P // 4)}
    for src_name, src in (("device", d_A), ("host", h_A)):
        ts = []
        for rep in range(2):  # the first run warms up
            st = pss.Stream(w.k, n // P, kt, batch_leaves=batches[src_name])
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(st_dev)
            for _ in range(passes):
                st.feed(src)
            root = st.root()
            cand, n_cand = pss.pss_prune(root, st.n_seen)
            b.record(st_dev)
            torch.cuda.synchronize()
            if rep:
                ts.append(a.elapsed_time(b))
            del st
        ms = min(ts)
        out[src_name] = {"value": round(passes * n / (ms * 1e-3) / 1e9, 3), "unit": "Gitems/s",
                         "ms": round(ms, 3), "n_cand": int(n_cand.item())}
    # the link's own bandwidth: one pinned host -> device copy of the same bytes
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st_dev)
    d_A.copy_(h_A, non_blocking=True)
    b.record(st_dev)
    torch.cuda.synchronize()
    h2d = n * kb / (a.elapsed_time(b) * 1e-3) / 1e9
    host_gbs = passes * n * kb / (out["host"]["ms"] * 1e-3) / 1e9
    out["host"]["roofline"] = {"bound": "h2d", "achieved": round(host_gbs, 2),
                               "peak": round(h2d, 2), "unit": "GB/s",
                               "frac": round(host_gbs / h2d, 4),
                               "peak_source": "pinned torch copy of the same bytes, this run"}
    out["items"] = passes * n
    out["leaf_len"] = n // P
    out["batch_leaves"] = batches
    return out


# ------------------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch

    import inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD

    import paper_1606_04669_b200 as pss
    from paper_1606_04669_b200 import dist as pdist

    w = workload_of(args)
    n, k = w.n, w.k
    P = w.P
    kb = w.key_bytes
    kt = pss.KEY_U32 if kb == 4 else pss.KEY_U64

    # this rank's shard: positions [rank*n, (rank+1)*n) of one stream (weak scaling)
    h_A = torch.empty((n,), dtype=torch.uint32 if kb == 4 else torch.uint64, pin_memory=True)
    w.generate(n, out=h_A.numpy(), start=rank * n)
    d_A = h_A.to(dev)

    runner = pdist.Runner(n, k, P, kt, dev, world=world, rank=rank, group=pg)
    stream = torch.cuda.current_stream()

    def step(A, ev=None):
        return runner.step(A, ev)

    for _ in range(args.warmup):
        step(d_A)
    torch.cuda.synchronize()

    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if pg is not None:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    flush = (torch.empty((L2_FLUSH_BYTES,), dtype=torch.uint8, device=dev)
             if l2_flush_needed(w) else None)
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for i in range(K):
            if flush is not None:
                flush.fill_(i & 0xff)  # small inputs: push them out of L2 (not timed)
            step(d_A, evs[i])
        t_end.record(stream)
        torch.cuda.synchronize()
    if pg is not None:
        torch.distributed.barrier()
    # K back-to-back steps; with the L2 flush between steps, the sum of the steps' own spans
    ms = (t_start.elapsed_time(t_end) if flush is None
          else sum(e[0].elapsed_time(e[3]) for e in evs))
    # summarize_merge: pss_summarize_merge (K1 with the tree kernel overlapping its last wave);
    # exchange: the all-gather of the rank roots and the top levels (N > 1); tail: a5..a7
    per = {"summarize_merge": [], "exchange": [], "tail": []}
    for e in evs:
        per["summarize_merge"].append(e[0].elapsed_time(e[1]))
        per["exchange"].append(e[1].elapsed_time(e[2]))
        per["tail"].append(e[2].elapsed_time(e[3]))
    if pg is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / K
    value = world * n / (ms_step * 1e-3) / 1e9

    # correctness of the last step against a brute-force-free invariant: the answer is sorted
    # and every reported count reaches the threshold (full parity lives in tests/)
    res_items, res_counts, res_len = runner.result()
    ln = int(res_len.item())
    thr = world * n // k + 1
    counts = res_counts[:ln].cpu().numpy()
    assert (counts >= thr).all() and (np.diff(counts.astype(np.int64)) <= 0).all()

    # ---- end to end: host (pinned) keys -> H2D -> path -> D2H of the answer, every step
    E = 0 if args.no_e2e else (args.e2e_steps or min(K, 5))
    e2e_ms = []
    for i in range(E + 1 if E else 0):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        if pg is not None:
            torch.distributed.barrier()
        a.record(stream)
        out = runner.step_host(h_A, d_A)
        b.record(stream)
        torch.cuda.synchronize()
        if i > 0:
            e2e_ms.append(a.elapsed_time(b))
    e2e = statistics.median(e2e_ms) if e2e_ms else float("nan")
    if pg is not None:
        t = torch.tensor([e2e], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e = float(t.item())
    h2d = n * kb
    d2h = k * kb + k * 8 + 4

    # ---- roofline of the dominant launch pair (K1 summarize with the tree kernel overlapping
    # its last wave; CUDA events on their stream around pss_summarize_merge): algorithmic bytes =
    # n * key bytes (one read of A; the leaves and the tree are method overhead, not credited)
    peak, peak_src = measured_peaks()
    t_sm = statistics.mean(per["summarize_merge"])
    achieved = n * kb / (t_sm * 1e-3) / 1e9
    traffic = ncu_traffic(w.name)  # null for a custom workload (no ncu capture of it)
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "kernel": "ss_summarize_kernel + tree_kernel (programmatic dependent launch)",
            "algorithmic_bytes_per_launch": n * kb, "peak_source": peak_src,
            "ms_per_launch": round(t_sm, 4)}

    if rank != 0:
        return
    line = {"metric": METRIC, "value": round(value, 3), "unit": "Gitems/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_of(w),
            "data": "synthetic", "config": config_of(w, P, world),
            "phases_ms": {p: round(statistics.mean(v), 4) for p, v in per.items()},
            "summarize_merge_gitems_s": round(n / (t_sm * 1e-3) / 1e9, 3),
            "hbm_frac_of_8TBs_summarize_merge": round(n * kb / (t_sm * 1e-3) / 8e12, 4),
            "roofline": roof,
            "e2e": None if not e2e_ms else {
                "value": round(world * n / (e2e * 1e-3) / 1e9, 3), "unit": "Gitems/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": round(e2e, 3), "api": runner.host_api},
            "gpu_launches": runner.launches_per_step * K,
            "clocks": clk.summary(),
            "result_len": ln}
    # K6: the attainable HBM read bandwidth on the same array (128-bit streaming reads)
    probe_ms = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        pss.pss_read_probe(d_A)
        b.record(stream)
        torch.cuda.synchronize()
        probe_ms.append(a.elapsed_time(b))
    read_gbs = n * kb / (min(probe_ms[1:]) * 1e-3) / 1e9
    roof["read_probe_gbs"] = round(read_gbs, 1)
    roof["frac_of_read_probe"] = round(achieved / read_gbs, 4)
    if world == 1:
        line["accuracy"] = accuracy_leg(pss, runner, d_A, n, k)
    if world == 1 and not args.no_stream:
        line["stream"] = stream_leg(pss, w, P, h_A, d_A, args.stream_passes, dev)
    if world == 1 and not args.no_cpu_baseline:
        rate, desc, cores, dt = oracle_sample(w, args.cpu_seconds, host_threads(), h_A.numpy())
        line["cpu_baseline"] = {"value": round(rate / 1e9, 6), "unit": "Gitems/s", "cores": cores,
                                "kind": "oracle", "sample": desc, "seconds": round(dt, 2)}
    print(json.dumps(line), flush=True)
    if pg is not None:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
