"""Benchmark: scheduler decisions/s on BASELINE.json config B (headline) and
the other named workloads.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload A|B|C|D|E|audit]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...     # the CPU reference arm

A step = one pass of the scheduler hot path over the whole synthetic batch:
every round of every trace. B and D are weak-scaled (4,096 traces x 1,000
requests per GPU); E is ONE job of 65,536 traces x 2,000 requests split over
the ranks (strong scaling); A (one medical trace) and C (one 1M-request
pool) are single traces (replicas only). ``value`` is device-timed with
inputs resident in HBM (L2 flushed between steps; NCCL all-gather of the
per-trace statistics inside the step at N > 1); ``e2e`` is the same work
through the C-ABI host-buffer entry (``ss_run_traces_host``: H2D inputs,
kernels, D2H results, host clock).

CPU legs (test infrastructure, never the measured product): the C
restatement of the reference scheduler (``oracle/``, all host threads) on a
bounded sample of the same traces -- the ``cpu_baseline`` here and the
``--impl reference`` arm, warmed and timed the same way; its digests double
as a full-size parity check. The reference arm additionally times the
UNMODIFIED Python reference ``Simulator`` (``baseline/_ref``, installed from
/root/reference) with ``multiprocessing.Pool(os.cpu_count())`` on a sample.
The reference arm never loads this package's CUDA library: its inputs come
from the reference's own ``generate`` + ``predictor_pipeline``.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
REF_PKG = os.path.join(REPO, "baseline", "_ref")

METRIC = "scheduler decisions/sec"
UNIT = "decisions/s"

WORKLOADS = {
    "A": dict(desc="config A: one medical-emergency trace, 1,000 requests, 3 uniform urgency levels, Poisson arrivals "
                   "(rate 15/s, seed 0), fixed KV budget 4,096 slots, b=16, a100_qwen7b",
              traces=1, requests=1000, capacity=4096, profile="a100_qwen7b", levels=3, scaling="replicas only"),
    "B": dict(desc="config B: 4,096 independent traces x 1,000 requests (generate(WorkloadSpec(total_requests=1000, "
                   "seed=s))), b=16, ample KV (1e9 slots), a100_qwen7b, exact predictors",
              traces=4096, requests=1000, capacity=10**9, profile="a100_qwen7b", levels=5, scaling="weak"),
    "C": dict(desc="config C: one pool of 1,000,000 requests all at t=0 (WorkloadSpec(total_requests=N, "
                   "concurrent=N, concurrent_mode='fixed', seed=1)), b=16, ample KV, a100_qwen7b; steady-state "
                   "per-step time from runs capped at 1 and 1+S rounds",
              traces=1, requests=1_000_000, capacity=10**9, profile="a100_qwen7b", levels=5, scaling="replicas only"),
    "D": dict(desc="config D shape at scale: 4,096 traces x 1,000 requests, 3 levels, KV budget 2,295 slots "
                   "(25% of the seed-1 ample peak), a100_qwen7b (offload), heavy eviction",
              traces=4096, requests=1000, capacity=2295, profile="a100_qwen7b", levels=3, scaling="weak"),
    "E": dict(desc="config E: ONE job of 65,536 traces x 2,000 requests (generate(WorkloadSpec(total_requests=2000, "
                   "seed=s)), s = 0..65535), block-partitioned over the GPUs, b=16, ample KV, a100_qwen7b",
              traces=65536, requests=2000, capacity=10**9, profile="a100_qwen7b", levels=5, scaling="strong"),
}
# traces of the bounded CPU sample per step (C port, all host threads): ~2-3 s per run on 16
# threads, i.e. ~30-45 s of CPU work per run; cpu_baseline = 1 warm-up + 2 timed runs
CPU_SAMPLE = {"A": 1, "B": 1024, "D": 512, "E": 256}
# traces of the Python-reference sample (one multiprocessing pool run)
PY_SAMPLE = {"A": 1, "B": 16, "D": 16, "E": 16}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.p is None:
            return False
        time.sleep(0.2)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)
        return False

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- inputs ----

def job_layout(wl, world, rank, traces_override=None):
    """(seeds of this rank, traces per rank, traces in the whole job)."""
    from paper_2506_12204_b200.dist import job_seeds, shard_seeds

    T = traces_override or wl["traces"]
    if wl["scaling"] == "strong":
        if T % world:
            raise SystemExit(f"config E: {T} traces do not split evenly over {world} ranks")
        seeds = job_seeds(T, world, rank)
        return seeds, T // world, T
    seeds = shard_seeds(T, rank)
    return seeds, T, T * world


def workload_config(name, wl, world, per_rank, total):
    """The `config` object, identical in both arms."""
    return {"workload": wl["desc"], "name": name, "traces_per_gpu": per_rank, "traces_total": total,
            "requests_per_trace": wl["requests"], "batch_size": 16, "memory_capacity": wl["capacity"],
            "profile": wl["profile"], "levels": wl["levels"], "parallelism": f"traces sharded x{world}",
            "l2": "flushed (256 MiB write) between timed steps"}


def scenario(name, wl, seed=0):
    from paper_2506_12204_b200.engine import ScenarioConfig
    from paper_2506_12204_b200.workload import WorkloadSpec

    return ScenarioConfig(workload=WorkloadSpec(total_requests=wl["requests"], levels=wl["levels"], seed=seed),
                          memory_capacity=wl["capacity"], profile=wl["profile"], seed=seed)


def native_batch(name, wl, seeds, pinned=True):
    """This package's inputs (the native generator; config A's Poisson arrivals
    through the Python predictor pipeline)."""
    from paper_2506_12204_b200.tracegen import generate_batch
    from paper_2506_12204_b200.workload import WorkloadSpec

    if name == "A":
        from paper_2506_12204_b200.scenarios import medical_arrivals
        from paper_2506_12204_b200.soa import prepare_trace

        return prepare_trace(medical_arrivals(seed=0, n=wl["requests"]), scenario(name, wl))[0]
    spec = WorkloadSpec(total_requests=wl["requests"], levels=wl["levels"])
    return generate_batch(spec, seeds, pinned=pinned)


REF_SRC = "/root/reference/pkg/src"  # build container only (absent on the GPU box)


def _ref_semsched():
    """The unmodified reference package (baseline/_ref, else its source tree
    when this is the build container) or None."""
    for root in (REF_PKG, REF_SRC):
        if os.path.isdir(os.path.join(root, "semsched")):
            if root not in sys.path:
                sys.path.insert(0, root)
            import semsched  # noqa: F401

            return semsched
    return None


def reference_batch(name, wl, seeds):
    """Reference-arm inputs WITHOUT this package's CUDA library: the
    reference's own generate + predictor_pipeline (baseline/_ref) laid out
    as the oracle's SoA."""
    import random

    from paper_2506_12204_b200.soa import TraceBatch, from_prepared

    ref = _ref_semsched()
    if ref is None:
        raise SystemExit("reference arm: the reference package is not installed (baseline/_ref)")
    from semsched.predictors import PredictorConfig, predictor_pipeline
    from semsched.requests import Request, UrgencyLevel
    from semsched.workload import WorkloadSpec, generate

    parts = []
    for s in seeds:
        if name == "A":
            from paper_2506_12204_b200.scenarios import medical_arrivals

            arr = [Request(id=r.id, arrival_time=r.arrival_time, prompt_len=r.prompt_len,
                           true_output_len=r.true_output_len, true_urgency=UrgencyLevel(r.true_urgency.rank, 3))
                   for r in medical_arrivals(seed=0, n=wl["requests"])]
        else:
            arr = generate(WorkloadSpec(total_requests=wl["requests"], levels=wl["levels"], seed=int(s)))
        ready = predictor_pipeline(arr, PredictorConfig(), random.Random(0 if name == "A" else int(s)),
                                   levels=wl["levels"])
        parts.append(from_prepared(arr, ready))
    return TraceBatch.concat(parts)


VARIANT = os.environ.get("SS_BENCH_VARIANT", "auto")  # dev: force a scheduler variant


def params_for(wl, flags=None):
    from paper_2506_12204_b200 import _abi as A
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params

    force = {"auto": 0, "chunked": A.SS_FLAG_FORCE_CHUNKED, "perround": A.SS_FLAG_FORCE_PERROUND}[VARIANT]
    dflt = 0 if os.environ.get("SS_BENCH_NODIGEST") else A.SS_FLAG_DIGEST  # dev: cost of the digest
    return make_params(get_profile(wl["profile"]), 16, wl["capacity"], levels=wl["levels"],
                       flags=(dflt if flags is None else flags) | force)


# ------------------------------------------------------------- CPU legs -----

def time_cpu_port(pf, batch, sample, threads, warmup, steps):
    """The C restatement of the reference scheduler (test infrastructure) on
    the first `sample` traces: `warmup` untimed runs, then `steps` timed ones.
    Returns (decisions/s, seconds per step, last result)."""
    from oracle_binding import run_oracle

    sub = batch.subset(range(min(sample, batch.n_traces)))
    for _ in range(warmup):
        run_oracle(pf(), sub, threads=threads)
    ts, res = [], None
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        res = run_oracle(pf(), sub, threads=threads)
        ts.append(time.perf_counter() - t0)
    dec = int(res.stats["rounds"].sum())
    return dec * len(ts) / sum(ts), sum(ts) / len(ts), res


def _py_one(job):
    """One trace through the UNMODIFIED Python reference Simulator (worker)."""
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    from semsched.engine import ScenarioConfig, Simulator
    from semsched.requests import Request, UrgencyLevel
    from semsched.workload import WorkloadSpec

    cfg = ScenarioConfig(workload=WorkloadSpec(total_requests=job["requests"], levels=job["levels"],
                                               seed=job["seed"]),
                         memory_capacity=job["capacity"], profile=job["profile"], seed=job["seed"])
    arrivals = None
    if job.get("rows"):
        arrivals = [Request(id=i, arrival_time=a, prompt_len=p, true_output_len=o,
                            true_urgency=UrgencyLevel(u, job["levels"])) for i, a, p, o, u in job["rows"]]
    sim = Simulator(cfg)
    rounds = [0]
    execute = sim._execute

    def counted(batch):  # one decision = one _schedule + _execute round (engine.py:215-224)
        rounds[0] += 1
        return execute(batch)

    sim._execute = counted
    t0 = time.perf_counter()
    sim.run(arrivals)
    return rounds[0], time.perf_counter() - t0


def time_python_reference(name, wl, seeds):
    """Python reference Simulator over a sample, all host cores."""
    import multiprocessing as mp

    if _ref_semsched() is None:
        return {"unavailable": "baseline/_ref not installed"}
    rows = None
    if name == "A":
        from paper_2506_12204_b200.scenarios import medical_arrivals

        rows = [(r.id, r.arrival_time, r.prompt_len, r.true_output_len, r.true_urgency.rank)
                for r in medical_arrivals(seed=0, n=wl["requests"])]
    jobs = [dict(requests=wl["requests"], levels=wl["levels"], capacity=wl["capacity"], profile=wl["profile"],
                 seed=0 if name == "A" else int(s), rows=rows) for s in seeds]
    procs = min(os.cpu_count() or 1, len(jobs))
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(abs, range(procs))  # workers up before the clock starts
        t0 = time.perf_counter()
        res = pool.map(_py_one, jobs)
        wall = time.perf_counter() - t0
    dec = sum(r for r, _ in res)
    busy = sum(t for _, t in res)
    import semsched

    return {"value": dec / wall, "unit": UNIT, "cores": procs, "per_core": dec / busy, "kind": "reference",
            "sample": f"{len(jobs)} traces of the same workload, unmodified semsched {semsched.__version__} "
                      f"Simulator (baseline/_ref), multiprocessing.Pool({procs}), {wall:.1f} s wall",
            "python": platform.python_version(), "cpu": _cpu_model(), "host_threads": os.cpu_count()}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or platform.machine()


def _loaded_libs():
    try:
        with open("/proc/self/maps") as fh:
            return sorted({ln.split()[-1] for ln in fh if ln.rstrip().endswith(".so") and REPO in ln})
    except OSError:
        return []


def reference_arm(args, name, wl):
    """The reference's CPU scheduler on this box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    seeds, per_rank, total = job_layout(wl, world, 0, args.traces)
    threads = os.cpu_count() or 1
    sample = min(per_rank, CPU_SAMPLE[name])
    t0 = time.perf_counter()
    batch = reference_batch(name, wl, seeds[:sample])
    gen_s = time.perf_counter() - t0
    value, sec, res = time_cpu_port(lambda: params_for(wl), batch, sample, threads, args.warmup, args.steps)
    py = None if args.no_python else time_python_reference(name, wl, seeds[:min(sample, PY_SAMPLE[name])])
    libs = _loaded_libs()
    assert not any("libsemsched_b200" in x for x in libs), libs
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sec, "higher_is_better": True, "scaling": wl["scaling"],
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": workload_config(name, wl, world, per_rank, total),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"first {sample} of {per_rank} traces per step (oracle/semsched_oracle.c, "
                                       f"the C restatement of the reference scheduler), {threads} threads; inputs "
                                       f"from the reference's own generate + predictor_pipeline ({gen_s:.1f} s)"},
            "python_reference": py,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "traces_per_s": sample / sec, "decisions_per_step": int(res.stats["rounds"].sum()),
            "native_so_loaded": libs}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- roofline ----

def algorithmic_bytes(stats, n_req):
    """B_decision summed over rounds + per-trace load/store."""
    s = lambda k: float(stats[k].astype(np.float64).sum())
    rounds = s("rounds")
    per_round = (16 * s("sum_pool") + 16 * s("sum_resident_evict") + 84 * (s("sum_granted") + s("sum_victims"))
                 + 4 * s("sum_granted") + 4 * s("completed") + 32 * s("sum_victims") + 32 * rounds)
    return per_round + (28 + 16) * n_req + 80 * len(stats)


def roofline(name, k_ms, decisions, n_traces, clk):
    """The dominant kernel against what binds it: instruction issue.

    achieved = warp instructions the scheduler kernel executes per launch
    (ncu smsp__inst_executed.sum of the same workload at HEAD, committed in
    profiles/ncu_issue_<W>.json) / this run's live kernel time; peak = 4 issue
    slots per SM per cycle x 148 SMs x the SM clock sampled under load. The
    HBM view (ncu DRAM bytes / kernel time vs the measured copy bandwidth) and
    SURVEY §8(d)'s pool-scan byte model are reported beside it."""
    peaks, src = measured_peaks()
    prof = None
    path = os.path.join(REPO, "profiles", f"ncu_issue_{name}.json")
    if os.path.exists(path):
        with open(path) as fh:
            prof = json.load(fh)
        if prof.get("decisions") != decisions or prof.get("traces") != n_traces:
            prof = None  # profiled on another workload size
    mhz = (clk or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    peak = 4 * 148 * mhz * 1e6
    out = {"bound": "issue", "unit": "warp-instr/s", "peak": peak, "achieved": None, "frac": None,
           "traffic": None, "kernel_ms": k_ms,
           "peak_note": f"4 warp-instr/cycle/SM x 148 SMs x {mhz:.0f} MHz (SM clock sampled under load)"}
    if prof:
        inst = float(prof["inst_executed"])
        out.update(achieved=inst / (k_ms / 1e3), frac=inst / (k_ms / 1e3) / peak, traffic=prof["dram_bytes"],
                   inst_per_launch=inst, warp_instr_per_decision=inst / decisions,
                   ncu_source=os.path.relpath(path, REPO), ncu_kernel=prof.get("kernel"),
                   ncu_issue_active_pct=prof.get("issue_active_pct"))
        gbs = prof["dram_bytes"] / (k_ms / 1e3) / 1e9
        out["hbm"] = {"achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"],
                      "peak_source": src}
    return out


# ------------------------------------------------------------ config C ------

def pool_bench(args, wl):
    """Config C: per-step latency of one million-request pool (replicas only)."""
    from paper_2506_12204_b200 import _abi as A
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.workload import WorkloadSpec

    N = args.traces or wl["requests"]
    spec = WorkloadSpec(total_requests=N, concurrent=N, concurrent_mode="fixed", seed=1)
    S = args.pool_steps
    prof = get_profile(wl["profile"])
    pf = lambda cap_rounds: make_params(prof, 16, wl["capacity"], levels=5, flags=A.SS_FLAG_DIGEST,
                                        max_rounds=cap_rounds)
    cfg = {"workload": wl["desc"], "name": "C", "requests": N, "batch_size": 16, "memory_capacity": wl["capacity"],
           "profile": wl["profile"], "parallelism": "replicas only"}
    metric = "scheduler decisions/sec (one 1M-request pool, steady state)"
    if args.impl == "reference":
        from oracle_binding import run_oracle
        from paper_2506_12204_b200.soa import prepare_trace
        from paper_2506_12204_b200.engine import ScenarioConfig
        from paper_2506_12204_b200.workload import generate

        batch = prepare_trace(generate(spec), ScenarioConfig(workload=spec, seed=1))[0]
        S = 10 * S  # the port's per-step cost is small next to its 1M-request setup
        t = {}
        for r in (1, 1 + S):
            ts = []
            for _ in range(max(1, args.steps)):
                t0 = time.perf_counter()
                run_oracle(pf(r), batch)
                ts.append(time.perf_counter() - t0)
            t[r] = min(ts)
        per = (t[1 + S] - t[1]) / S
        line = {"metric": metric, "value": 1.0 / per, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
                "scaling": "replicas only", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "impl": "reference", "config": cfg,
                "cpu_baseline": {"value": 1.0 / per, "unit": UNIT, "cores": 1, "kind": "port",
                                 "sample": f"{S} steady-state steps of the 1M pool, oracle port, 1 thread; "
                                           f"first step {t[1]:.2f} s"},
                "e2e": {"value": 1.0 / per, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "native_so_loaded": _loaded_libs()}
        print(json.dumps(line), flush=True)
        return
    import torch
    from paper_2506_12204_b200 import native
    from paper_2506_12204_b200.tracegen import generate_batch

    batch = generate_batch(spec, [1], pinned=True)
    dev = torch.device("cuda", 0)
    dbatch = native.DeviceBatch(batch, dev)
    douts = native.DeviceOutputs(batch.n_requests, 1, dev, with_state=False)
    ws = native.Workspace(pf(1), 1, batch.n_requests, dev)
    for _ in range(args.warmup):
        native.run_device(pf(1 + S), dbatch, douts, ws, time_kernel=True)
    t = {}
    with ClockSampler(0) as clk:
        for r in (1, 1 + S):
            t[r] = min(native.run_device(pf(r), dbatch, douts, ws, time_kernel=True)
                       for _ in range(max(1, args.steps)))
    native.run_device(pf(1), dbatch, douts, ws, time_kernel=True)
    prepass_ms = native.last_timings()[0]  # grid-wide init + radix sort of the 1M bulk admission
    per_ms = (t[1 + S] - t[1]) / S
    native.run_device(pf(1 + S), dbatch, douts, ws)  # the state the parity check compares
    st = douts.stats_numpy()
    cfg.update(pool_steps=S, prepass_ms=prepass_ms, first_step_ms=prepass_ms + t[1], first_step_kernels_ms=t[1],
               capped_run_ms=t[1 + S], rounds_run=int(st["rounds"][0]))
    line = {"metric": metric, "value": 1e3 / per_ms, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_ms, "higher_is_better": True, "scaling": "replicas only",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg, "clocks": clk.summary(),
            "gpu_launches": native.launches_per_run(pf(1))}
    if not args.no_cpu:
        from oracle_binding import run_oracle

        tc = {}
        S2 = 10 * S
        for r in (1, 1 + S, 1 + S2):
            t0 = time.perf_counter()
            res = run_oracle(pf(r), batch)
            tc[r] = time.perf_counter() - t0
            if r == 1 + S:
                match = bool(res.stats["digest"][0] == st["digest"][0] and res.stats["rounds"][0] == st["rounds"][0])
        line["cpu_baseline"] = {"value": S2 / (tc[1 + S2] - tc[1]), "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"{S2} steady-state steps, oracle port 1 thread, first step "
                                          f"{tc[1]:.2f} s"}
        line["parity"] = {"digest_and_rounds_match_after_steps": match}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- audit ------

def audit_bench(args):
    """Eq. 2 constraint audit (metrics.py:59-91) of every trace of config B's
    schedule: pairs examined per second (the reference's n(n-1)/2 per trace)."""
    from paper_2506_12204_b200 import _abi as A

    base = WORKLOADS["B"]
    T = args.traces or base["traces"]
    if args.impl == "reference":
        from oracle_binding import audit_oracle, run_oracle

        batch = reference_batch("B", base, range(min(T, 16)))
        fin = run_oracle(params_for(base, 0), batch, threads=os.cpu_count() or 1).finish_time
        done = np.add.reduceat(~np.isnan(fin), batch.offsets[:-1])
        pairs = float((done.astype(np.float64) * (done - 1) / 2).sum())
        ts = []
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            audit_oracle(batch.offsets, fin, batch.arrival, batch.true_urg)
            ts.append(time.perf_counter() - t0)
        v = pairs / float(np.mean(ts))
        line = {"metric": "constraint-audit pairs/sec", "value": v, "unit": "pairs/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": {"workload": f"Eq. 2 audit of {batch.n_traces} config-B traces", "pairs_per_step": pairs},
                "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": 1, "kind": "port",
                                 "sample": f"{batch.n_traces} traces, oracle so_audit (C restatement), 1 thread"},
                "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "native_so_loaded": _loaded_libs()}
        print(json.dumps(line), flush=True)
        return
    from paper_2506_12204_b200 import native
    from paper_2506_12204_b200.metrics import _audit_call

    batch = native_batch("B", base, np.arange(T), pinned=False)
    res = native.run_host(params_for(base), batch)
    fin = res.finish_time
    done = np.add.reduceat(~np.isnan(fin), batch.offsets[:-1])
    pairs = float((done.astype(np.float64) * (done - 1) / 2).sum())
    rank = batch.true_urg
    for _ in range(args.warmup):
        _audit_call(batch.offsets, fin, batch.arrival, rank, batch.ids, False)
    kms, ems = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        viol, comp, _ = _audit_call(batch.offsets, fin, batch.arrival, rank, batch.ids, False)
        ems.append(time.perf_counter() - t0)
        kms.append(_audit_call.kernel_ms)
    k_ms = float(np.mean(kms))
    cpu = parity = None
    if not args.no_cpu:
        from oracle_binding import audit_oracle

        S = min(T, 64)
        sub_off = batch.offsets[: S + 1]
        n_s = int(sub_off[-1])
        t0 = time.perf_counter()
        cv, cc = audit_oracle(sub_off, fin[:n_s], batch.arrival[:n_s], rank[:n_s])
        dt = time.perf_counter() - t0
        sp = float((done[:S].astype(np.float64) * (done[:S] - 1) / 2).sum())
        cpu = {"value": sp / dt, "unit": "pairs/s", "cores": 1, "kind": "port",
               "sample": f"first {S} of {T} traces, oracle so_audit (C restatement of metrics.py:59-91), 1 thread"}
        parity = {"traces_checked": S, "violations_and_comparable_match": bool(np.array_equal(cv, viol[:S]) and
                                                                              np.array_equal(cc, comp[:S]))}
    h2d = int(batch.offsets.nbytes + fin.nbytes + batch.arrival.nbytes + 4 * len(fin))
    line = {"metric": "constraint-audit pairs/sec", "value": pairs / (k_ms / 1e3), "unit": "pairs/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": k_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"Eq. 2 audit (true ranks) of the config-B schedule: {T} traces x "
                                   f"{base['requests']} requests", "pairs_per_step": pairs,
                       "violations": int(viol.sum()), "comparable": int(comp.sum())},
            "cpu_baseline": cpu, "parity": parity,
            "e2e": {"value": pairs / float(np.mean(ems)), "unit": "pairs/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 16 * T, "ms_per_step": 1e3 * float(np.mean(ems))},
            "gpu_launches": args.steps}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ main arm ------

def dry_run(args, name, wl):
    """The multi-rank plumbing without a GPU: gloo, each rank generates its
    shard, fills one ss_trace_stats record per trace with a checksum of the
    trace's inputs (no scheduling) and the records are all-gathered exactly as
    the timed step gathers them. Rank 0 prints the gathered count and a
    checksum that must equal a single-process dry run's."""
    import hashlib

    import torch
    import torch.distributed as dist

    from paper_2506_12204_b200 import _abi as A
    from paper_2506_12204_b200.dist import all_gather_stats, stats_of

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    seeds, T, total = job_layout(wl, world, rank, args.traces)
    batch = native_batch(name, wl, seeds, pinned=False)
    rec = np.zeros(T, A.stats_dtype())
    for t in range(T):
        sl = batch.trace_slice(t)
        rec["rounds"][t] = sl.stop - sl.start
        rec["digest"][t] = int(np.bitwise_xor.reduce(batch.ready[sl].view(np.uint64) ^
                                                     batch.prompt[sl].astype(np.uint64)))
        rec["completed"][t] = int(seeds[t]) if name != "A" else 0
    local = torch.from_numpy(rec.view(np.uint8).copy())
    got = stats_of(all_gather_stats(local, world))
    if rank == 0:
        print(json.dumps({"dry": True, "workload": name, "world": world, "gathered_traces": int(len(got)),
                          "traces_total": total, "seeds_in_order": bool(np.array_equal(got["completed"],
                                                                                       np.arange(total))),
                          "checksum": hashlib.sha256(got.tobytes()).hexdigest()}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="B", choices=sorted(WORKLOADS) + ["audit"])
    ap.add_argument("--traces", type=int, default=None, help="override traces per rank (E: per job)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-python", action="store_true", help="reference arm: skip the Python Simulator leg")
    ap.add_argument("--pool-steps", type=int, default=20000, help="config C: steady-state steps per sample")
    ap.add_argument("--dry", action="store_true", help="CPU/gloo check of sharding + gather (no scheduler)")
    args = ap.parse_args()
    if args.workload == "audit":
        return audit_bench(args)
    name = args.workload
    wl = WORKLOADS[name]
    if name == "C":
        return pool_bench(args, wl)
    if args.impl == "reference":
        return reference_arm(args, name, wl)
    if args.dry:
        return dry_run(args, name, wl)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:  # the driver checks the communicator size in NCCL's init log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import torch
    import torch.distributed as dist

    from paper_2506_12204_b200 import _abi as A
    from paper_2506_12204_b200 import native
    from paper_2506_12204_b200.dist import all_gather_stats, job_summary, stats_of

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    seeds, T, total = job_layout(wl, world, rank, args.traces)
    t0 = time.perf_counter()
    batch = native_batch(name, wl, seeds)
    host_gen_s = time.perf_counter() - t0
    log(f"[rank {rank}] traces {T} x {wl['requests']} prepared in {host_gen_s:.2f} s")
    tracegen = {"host_ms": 1e3 * host_gen_s, "host_threads": os.cpu_count(),
                "note": "input preparation (generate + predictor_pipeline), outside the timed step"}
    if name != "A":  # the same inputs generated on the device (one thread per trace, straight into HBM)
        from paper_2506_12204_b200.tracegen import generate_batch_device
        from paper_2506_12204_b200.workload import WorkloadSpec

        gspec = WorkloadSpec(total_requests=wl["requests"], levels=wl["levels"])
        generate_batch_device(gspec, seeds[:64], device=dev)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gdb = generate_batch_device(gspec, seeds, device=dev)
        tracegen["device_ms"] = 1e3 * (time.perf_counter() - t0)
        tracegen["device_matches_host"] = bool(
            torch.equal(gdb.t["ready"][: batch.n_requests].cpu(), torch.from_numpy(batch.ready)) and
            torch.equal(gdb.t["prompt"][: batch.n_requests].cpu(), torch.from_numpy(batch.prompt.view(np.int32))))
        del gdb
    pf = lambda: params_for(wl)
    dbatch = native.DeviceBatch(batch, dev)
    douts = native.DeviceOutputs(batch.n_requests, T, dev, with_state=False)
    ws = native.Workspace(pf(), T, batch.n_requests, dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    gathered = torch.empty(world * T * C.sizeof(A.ss_trace_stats), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        native.run_device(pf(), dbatch, douts, ws, stream=stream)
        all_gather_stats(douts.t["stats"], world, gathered)  # the one collective (a copy at N = 1)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stats = douts.stats_numpy()
    job = job_summary(stats_of(gathered))
    assert job["traces"] == total, (job, total)
    bad = int((stats["status"] != 0).sum())
    decisions = int(stats["rounds"].sum())
    cfgk = native.kernel_config(pf(), T)

    # ---- timed region: device events per step, L2 flushed between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = [a.elapsed_time(b) for a, b in ev]
    ms_step = float(np.mean(ms))
    t_total = torch.tensor([sum(ms)], dtype=torch.float64, device=dev)
    dec_t = torch.tensor([decisions * args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_total, op=dist.ReduceOp.MAX)
        dist.all_reduce(dec_t, op=dist.ReduceOp.SUM)
    value = float(dec_t.item()) / (float(t_total.item()) / 1e3)
    traces_s = total * args.steps / (float(t_total.item()) / 1e3)
    clocks = clk.summary()

    # kernel-only duration (the scheduler launch after the prepass) on the same stream
    kms = []
    for _ in range(3):
        flush.zero_()
        kms.append(native.run_device(pf(), dbatch, douts, ws, stream=stream, time_kernel=True))
    k_ms = float(np.mean(kms))
    n_req = batch.n_requests

    # ---- end to end through the C-ABI host entry (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        from paper_2506_12204_b200.results import alloc_host_outputs

        hb = native.host_batch(batch)
        outs = alloc_host_outputs(n_req, T)
        pin = lambda a: torch.from_numpy(a.view(np.uint8)).pin_memory().numpy().view(a.dtype) if a.size else a
        outs = {k: pin(v) for k, v in outs.items()}
        o = A.ss_outputs()
        o.req = A.ss_request_out(outs["first_scheduled"].ctypes.data, outs["finish_time"].ctypes.data,
                                 outs["generated"].ctypes.data, outs["evictions"].ctypes.data, None, None)
        o.stats = outs["stats"].ctypes.data
        o.unservable_slots = outs["unservable"].ctypes.data
        h2d = batch.nbytes_inputs()
        d2h = n_req * (8 + 8 + 4 + 4 + 4) + T * C.sizeof(A.ss_trace_stats)
        L = native.lib()
        st = C.c_void_p(stream.cuda_stream)
        for _ in range(2):
            L.ss_run_traces_host(C.byref(pf()), C.byref(hb), C.byref(o), st, None)
        if world > 1:
            dist.barrier()
        et = []
        for _ in range(args.steps):
            t1 = time.perf_counter()
            rc = L.ss_run_traces_host(C.byref(pf()), C.byref(hb), C.byref(o), st, None)
            et.append(time.perf_counter() - t1)
            # traces the reference itself fails on report SS_ERR_TRACE_FAILED (stats carry them)
            assert rc in (A.SS_OK, A.SS_ERR_TRACE_FAILED), native.last_error()
        e_tot = torch.tensor([sum(et)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_tot, op=dist.ReduceOp.MAX)
        e2e = {"value": float(dec_t.item()) / float(e_tot.item()), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * float(e_tot.item()) / args.steps}

    # ---- CPU baseline (C port, warmed and timed like the reference arm); digests = parity check
    cpu = parity = None
    if rank == 0 and not args.no_cpu:
        threads = os.cpu_count() or 1
        sample = min(T, CPU_SAMPLE[name])
        v, sec, res = time_cpu_port(pf, batch, sample, threads, 1, 2)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"first {sample} of {T} traces of the same workload, oracle/semsched_oracle.c "
                         f"(C restatement of the reference scheduler), {threads} threads, 1 warm-up + 2 timed runs, "
                         f"{sec:.2f} s each"}
        # status and rounds on every sampled trace; the digest where the trace
        # finished (a reference exception ends a trace mid-round)
        ok = res.stats["status"] == 0
        obs = ok | (res.stats["status"] == A.SS_TRACE_REF_ERROR)
        match = bool(np.array_equal(res.stats["status"], stats["status"][:sample]) and
                     np.array_equal(res.stats["rounds"][obs], stats["rounds"][:sample][obs]) and
                     np.array_equal(res.stats["digest"][ok], stats["digest"][:sample][ok]))
        parity = {"traces_checked": sample, "digest_and_rounds_match": match,
                  "reference_error_traces": int((~ok).sum())}

    if rank == 0:
        rl = roofline(name, k_ms, decisions, T, clocks)
        rl["model_bytes"] = algorithmic_bytes(stats, n_req)
        rl["model_note"] = ("SURVEY.md §8(d) pool-scan byte model (every live key re-read each round); this kernel "
                            "keeps queue fronts, ongoing sets and stretch state on chip, so its DRAM traffic is far "
                            "below the model and instruction issue / latency bind it")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": wl["scaling"],
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(name, wl, world, T, total),
            "kernel": {"blocks": cfgk["blocks"], "warps_per_block": cfgk["warps_per_block"],
                       "smem_per_block": cfgk["smem_per_block"]},
            "traces_per_s": traces_s, "tracegen": tracegen, "decisions_per_step": int(dec_t.item()) // args.steps,
            "roofline": rl, "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "clocks": clocks,
            "comm": {"backend": "nccl" if world > 1 else None, "world_size": world,
                     "collective": "all_gather_into_tensor of per-trace ss_trace_stats records" if world > 1
                     else None, "gathered_traces": job["traces"]},
            "job": job,
            "gpu_launches": args.steps * native.launches_per_run(pf(), dbatch.max_trace_len),
            "failed_traces": bad,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()  # rank 0 finishes its CPU baseline and report first
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
