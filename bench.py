#!/usr/bin/env python
"""bench.py -- one JSON line for the greedy binary-code construction on B200.

A STEP is one whole construction (every row of SURVEY.md Sec. 8(a): candidate
generation, windowed screen, in-tile resolve, commit) for the workload
(n, d, ordering).  Default workload: n=28, d=3, lexicographic (BASELINE.json
configs[4], the config BASELINE's metric is quoted on at 1/2/4/8 GPUs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload 28,3,lex] [--impl b200|reference]

metric: candidate-codeword distance checks per second, counted DEFINITIONALLY as the
paper's kernel performs them (every candidate against every codeword accepted before it,
PAPER.md:73): W_def = sum_j (2^n - 1 - rank_j).  value = W_def / (device time per step).
ms_per_step is the wall (device) time of one construction.  The executed checks
(W_exec, after early exit) and the POPC-pipe roofline of the screen kernel are reported
beside it.

N > 1: launched by torch.distributed.run, one process per GPU; each rank screens 1/N of
every tile (gc_generate_rank over an NCCL communicator).  Strong scaling: the same
construction at every N.
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
from workloads import parse_workload, seq_digest, set_digest  # noqa: E402  (inputs + fingerprints only)

# measured check rates (checks/clk/SM), profiles/r01_popc_peak.txt: the arithmetic the
# kernel uses for each d (d <= 4: half of the checks in the ALU bit-clearing form)
CHECK_PEAK_PER_CLK_SM = {"popc": 15.49, 2: 23.62, 3: 19.18, 4: 16.66}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                clk, mx, util = float(r[1]), float(r[2]), float(r[9])
            except Exception:
                continue
            smax = mx
            if util > 0:
                sm.append(clk)
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(self.rows), "samples_under_load": len(sm)}


def load_ncu_summary():
    """Key counters of the dominant kernel from the committed ncu --set full summary of the same
    workload (profiles/k_pipeline_ncu_summary.json, tools/ncu_summary.py), or {}."""
    p = os.path.join(ROOT, "profiles", "k_pipeline_ncu_summary.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


# ------------------------------------------------------------------ CPU oracle

def host_cpu():
    """(threads this process may use, CPU model) of the host the bench runs on."""
    cores = len(os.sched_getaffinity(0))
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return cores, model


def golden_row(workload: str):
    """Expected output of a bench workload (tests/golden/bench_golden.json, written by
    tools/gen_bench_golden.py from oracle O2 alone), or None."""
    try:
        rows = json.load(open(os.path.join(ROOT, "tests", "golden", "bench_golden.json")))["rows"]
    except Exception:
        return None
    for r in rows:
        if r["workload"] == workload:
            return r
    return None


def o2_full(n, d, o, ex):
    """The oracle's exact greedy (O2, ball marking, one thread) on the WHOLE workload."""
    import oracle as O
    t = time.perf_counter()
    w = O.greedy_ball_ex(n, d, o, **ex) if ex else O.greedy_ball(n, d, o)
    return time.perf_counter() - t, w


def o1_prefix(n, d, o, threads, budget_s, start_log2=16):
    """The oracle's plain greedy (O1: Fig. 2(a) with threads == 1, the Fig. 2(b) thread
    sections otherwise) on a bounded PREFIX of the workload's scan: the first
    2^k ranks, k grown while the budget allows.  Returns (W_def of the prefix / s, text)."""
    import numpy as np
    import oracle as O
    k = min(start_log2, n)
    spent, best = 0.0, None
    full = O.order_table(o, n) if o not in ("lex", "gray") else None
    while True:
        nranks = 1 << k
        # the first 2^k ranks of the n-bit lex / reflected Gray order are the k-bit order
        table = O.order_table(o, k) if full is None else full[:nranks].copy()
        t = time.perf_counter()
        if threads == 1:
            w = O.greedy_plain(n, d, o, nranks=nranks, table=table)
        else:
            w = O.greedy_plain_mt(n, d, o, threads=threads, nranks=nranks, table=table)
        dt = time.perf_counter() - t
        spent += dt
        inv = np.argsort(table)
        ranks = inv[np.searchsorted(np.sort(table), w)]
        wdef = int((nranks - 1 - ranks.astype(np.int64)).sum())
        best = (wdef / dt, f"O1{'' if threads == 1 else '_mt'} on ranks [0, 2^{k}) of ({n},{d},{o}): M={len(w)}, "
                           f"W_def={wdef:.4g} in {dt:.2f} s, {threads} thread(s)")
        if spent + 4 * dt > budget_s or k >= n:
            return best
        k += 1


def cpu_baseline(n, d, o, ex, w_def, budget_s):
    """The oracle timed on this host: O2 on the whole workload (value; the same config as the
    GPU line), plus O1 single-threaded and O1 over all host threads on a bounded prefix."""
    cores, model = host_cpu()
    dt, w = o2_full(n, d, o, ex)
    out = {"value": (w_def / dt) if w_def else None, "unit": "checks/s", "cores": 1, "kind": "oracle",
           "sample": f"O2 (oracle/greedy_oracle.c or_greedy_ball: exact greedy by Hamming-ball marking) on the "
                     f"whole workload ({n},{d},{o}), 1 thread: {dt:.2f} s per construction, M={len(w)}",
           "seconds_per_construction": dt, "host_threads": cores, "cpu_model": model}
    if not ex:
        v1, s1 = o1_prefix(n, d, o, 1, budget_s / 2)
        vm, sm = o1_prefix(n, d, o, cores, budget_s / 2)
        out["o1_1thread"] = {"value": v1, "unit": "checks/s", "cores": 1, "sample": s1}
        out["o1_threads"] = {"value": vm, "unit": "checks/s", "cores": cores, "sample": sm}
    return out


def run_reference(args):
    """The reference arm: the oracle as it stands (O2, exact, one host thread) on the SAME
    workload as the B200 arm, one whole construction per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, d, o, ex = parse_workload(args.workload)
    g = golden_row(args.workload)
    w_def = g.get("w_def") if g else None
    for _ in range(args.warmup):
        o2_full(n, d, o, ex)
    tot = 0.0
    for _ in range(args.steps):
        dt, w = o2_full(n, d, o, ex)
        tot += dt
    ms = 1e3 * tot / args.steps
    if w_def is None and not ex:
        import oracle as O
        import numpy as np
        table = O.order_table(o, n)
        inv = np.empty(1 << n, dtype=np.uint32)
        inv[table] = np.arange(1 << n, dtype=np.uint32)
        w_def = int(((1 << n) - 1 - inv[w].astype(np.int64)).sum())
    val = (w_def / (ms * 1e-3)) if w_def else 1e3 / ms
    unit = "checks/s" if w_def else "constructions/s"
    cores, model = host_cpu()
    sample = (f"O2 (oracle/, exact greedy by Hamming-ball marking) on the whole workload ({n},{d},{o}) per step, "
              f"1 thread of {cores} ({model})")
    line = {
        "impl": "reference", "metric": "candidate-codeword distance checks/sec (definitional W_def)",
        "value": val, "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (the whole space F_2^n, no dataset)",
        "config": {"workload": args.workload, "M": len(w), "w_def": w_def, "sample": sample},
        "cpu_baseline": {"value": val, "unit": unit, "cores": 1, "kind": "oracle", "sample": sample,
                         "host_threads": cores, "cpu_model": model},
        "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ B200 arm

def run_b200(args):
    import torch
    import torch.distributed as dist
    import paper_1507_05398_b200 as gc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        print(f"--gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n, d, o, ex = parse_workload(args.workload)
    from paper_1507_05398_b200 import dist as gdist
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    comm = gdist.comm_from_group()

    cap = gc.gc_capacity_bound(n, d)
    codebook = torch.empty(cap, dtype=torch.int32, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    opts = {"flags": gc.GC_FLAG_KERNEL_TIMING}

    def construct():
        if ex:
            return gc.gc_construct_device(n, d, codebook, count, ordering=o, stream=stream, options=opts,
                                          stats=True, **ex)
        return gc.gc_generate_rank(n, d, o, comm, codebook, count, stream=stream, options=opts)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        flush.zero_()
        construct()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    stats = []
    dev_ms = 0.0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()                      # L2 flushed between timed steps (outside the events)
        ev[k][0].record(stream)
        st = construct()                   # synchronises the stream at the end
        ev[k][1].record(stream)
        stats.append(st)
    barrier()
    sampler.stop()
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    max_ms = gdist.max_over_ranks(dev_ms) if world > 1 else dev_ms
    ms_per_step = max_ms / args.steps
    M = int(count.item())
    w_def = stats[-1]["w_def"]
    # parity gate (outside the timed region): the constructed code against the oracle's
    # (tests/golden/bench_golden.json, O2); a mismatch is not reported as a number
    parity = "unchecked (no golden row for this workload)"
    g = golden_row(args.workload)
    if g is not None and rank == 0:
        words = codebook[:M].cpu().numpy().view("uint32")
        got = {"M": M, "seq_digest": format(seq_digest(words), "016x"), "set_digest": format(set_digest(words), "016x")}
        want = {k: g[k] for k in got}
        if not ex and "w_def" in g:
            got["w_def"], want["w_def"] = int(w_def), g["w_def"]
        if got != want:
            print(json.dumps({"error": "parity gate: output differs from the oracle", "workload": args.workload,
                              "got": got, "want": want}), flush=True)
            return 3
        parity = "O2-equal (M, sequence and set digests" + (", W_def" if "w_def" in got else "") + \
                 " vs tests/golden/bench_golden.json)"
    value = w_def / (ms_per_step * 1e-3)
    if ex:
        # filtered problems have no definitional count over all ranks: report executed checks/s
        value = stats[-1]["checks_exec"] / (ms_per_step * 1e-3)

    # e2e through the public API: host buffers, device->host copy of the code inside the region
    e2e_val, d2h = None, 0
    if world == 1 and ex:
        e2e_val = None            # the host-buffer entry for extended problems is gc_construct
        gc.gc_construct(n, d, ordering=o, **ex)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ds = torch.cuda.default_stream(dev)
        tot = 0.0
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            e0.record(ds)
            w, _ = gc.gc_construct(n, d, ordering=o, **ex)
            e1.record(ds)
            torch.cuda.synchronize(dev)
            tot += e0.elapsed_time(e1)
            d2h = w.nbytes
        e2e_val = (tot / args.steps)
    elif world == 1:
        gc.gc_generate(n, d, o)       # warm (allocations)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ds = torch.cuda.default_stream(dev)
        tot = 0.0
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            e0.record(ds)
            w = gc.gc_generate(n, d, o)
            e1.record(ds)
            torch.cuda.synchronize(dev)
            tot += e0.elapsed_time(e1)
            d2h = w.nbytes
        e2e_val = w_def / (tot / args.steps * 1e-3)
    else:
        # each rank constructs; rank 0 reads the code back to the host
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0.record(stream)
            construct()
            host = codebook[:M].cpu() if rank == 0 else None
            e1.record(stream)
            barrier()
            tot += e0.elapsed_time(e1)
            if rank == 0:
                d2h = host.numel() * 4 + 8
        e2e_val = w_def / (gdist.max_over_ranks(tot) / args.steps * 1e-3)

    if ex and e2e_val is not None:
        e2e_val = stats[-1]["checks_exec"] / (e2e_val * 1e-3)     # e2e_val held ms per step

    # roofline of the dominant kernel (k_pipeline, the whole construction in one launch): executed
    # checks / its device time, against the measured rate of the check arithmetic
    checks = sum(s["checks_exec"] for s in stats)
    tests = sum(s["bound_tests"] for s in stats)
    screen_ms = sum(s["screen_ms"] for s in stats)
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz") or 1965.0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    per_clk = CHECK_PEAK_PER_CLK_SM.get(d, CHECK_PEAK_PER_CLK_SM["popc"])
    peak = sms * per_clk * sm_max * 1e6
    achieved = checks / (screen_ms * 1e-3) if screen_ms > 0 else 0.0
    achieved_tests = (checks + tests) / (screen_ms * 1e-3) if screen_ms > 0 else 0.0
    clocks = sampler.summary()
    ncu = load_ncu_summary()

    if rank == 0:
        line = {
            "metric": "candidate-codeword distance checks/sec (definitional W_def)",
            "value": value, "unit": "checks/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (the whole space F_2^n in the chosen ordering; no dataset)",
            "config": {"workload": args.workload, "M": M, "w_def": w_def,
                       "parallelism": (f"tile screens partitioned over {world} GPUs (peer stores of the mask "
                                       "words, replicated codebook and resolve)") if world > 1 else "1 GPU",
                       "l2": "flushed between timed steps (512 MiB write)"},
            "w_exec": checks / args.steps,
            "w_exec_per_s": (checks / args.steps) / (ms_per_step * 1e-3),
            "roofline": {"bound": "alu", "kernel": "k_pipeline (persistent: screen levels, preparation, resolve)",
                         "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tchecks/s",
                         "frac": achieved / peak if peak else None,
                         "traffic": ncu.get("dram_bytes_per_launch") if ncu.get("workload") == args.workload else None,
                         "peak_basis": f"{sms} SM x {per_clk} checks/clk/SM x {sm_max:.0f} MHz (check "
                                       f"arithmetic for d={d} measured by tools/popc_peak.cu, "
                                       "profiles/r01_popc_peak.txt)",
                         "bound_tests_per_step": tests / args.steps,
                         "frac_with_bound_tests": achieved_tests / peak if peak else None,
                         "ncu": {k: ncu.get(k) for k in ("pipes_pct_of_peak_active", "source", "workload")} if ncu else None,
                         "screen_share_of_step": (screen_ms / args.steps) / ms_per_step,
                         "screen_launches_per_step": stats[-1]["screen_launches"],
                         "regime": "latency-bound: the block bound leaves W_exec ~1e-4 of W_def, so a step is "
                                   "a chain of dependent tile resolves (one resolving CTA), overlapped with the "
                                   "screen of later tiles and their preparation; frac is the executed-check "
                                   "rate against the check-arithmetic peak (frac_with_bound_tests also counts "
                                   "the block-summary tests as one unit each)"},
            "latency": {"tiles_per_step": stats[-1]["tiles"], "levels_per_step": stats[-1]["phases"],
                        "us_per_tile": 1e3 * ms_per_step / max(1, stats[-1]["tiles"]),
                        "resolver_busy_ms": stats[-1]["resolve_busy_ms"],
                        "resolver_wait_ms": stats[-1]["resolve_wait_ms"],
                        "tiles_prepared": stats[-1]["prep_used"],
                        "pipeline_depth": stats[-1]["pipeline_depth"]},
            "e2e": {"value": e2e_val, "unit": "checks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(sum(s["launches"] for s in stats)),
            "clocks": clocks,
        }
        if ex:
            line["metric"] = "executed candidate-codeword checks/sec (W_exec; constrained problem)"
        line["parity"] = parity
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(n, d, o, ex, w_def if not ex else None, args.cpu_budget)
        print(json.dumps(line), flush=True)
    comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="28,3,lex")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
