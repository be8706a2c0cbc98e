"""bench.py — fact rows/s of the covariance batch (BASELINE.json configs[1]) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]
  (N > 1: one process per GPU over NCCL — either launched by torch.distributed.run, or,
  when WORLD_SIZE is unset, bench.py launches N ranks itself the same way)

A step is one lmfao_run over the whole batch (view build (b), fused root scan
(c)+(d), dimension-side finishing, NCCL all-reduce when N > 1) with the
relations already resident in HBM.  Each rank keeps a contiguous shard of the
sorted fact (domain parallelism): per-GPU work is fixed = 1/N of the fact
(the fact is the same 10M rows at every N) -> "strong" scaling.  Timed with CUDA
events on the launching stream, barrier + synchronize on both sides, max over
ranks.  Inputs (760 MB fact) exceed the 126 MB L2, so no explicit flush.

e2e: the same metric through the public API with HOST buffers: every step copies
the relations from pinned host memory (add_relation), prepares (sort), plans,
runs and fetches the 780 results to the host.

--impl reference: the CPU oracle (oracle/, the reference arm for this tier) on a
bounded sample of the same workload, rank 0 only.
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

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "fact rows/s for covariance batch and % of HBM roofline at 1/2/4/8 B200"
BYTES_PER_ROW = {"C1": 3 * 8 + 2 * 4, "C2": 8 * 8 + 3 * 4, "C5": 8 * 8 + 4 * 4}


def workload(name):
    return {"C1": synth.config1, "C2": synth.config2, "C5": synth.config5}[name]()


def dim_feature_bytes(w):
    """Algorithmic bytes of the dimension feature tables the scan reads (PK dims)."""
    tot = 0
    for r in w.db.relations:
        if r.name == w.db.root:
            continue
        nf = sum(1 for c in r.cols if c in w.meta["features"])
        tot += nf * 8 * r.nrows
    return tot


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def committed_traffic(config):
    """dram bytes per launch of the scan kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_scan_summary.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if d.get("config") == config:
            return d.get("dram_bytes_per_launch")
    return None


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(w, max_rows, threads=0):
    """The oracle as it stands (oracle/, OpenMP over contiguous fact-row chunks with private
    accumulators merged in chunk order) on the first `max_rows` fact rows,
    on every host core (threads=0)."""
    import oracle
    db = w.db
    F = db.rel(db.root)
    n = min(max_rows, F.nrows)
    cores = oracle.host_cores() if threads == 0 else threads
    t0 = time.perf_counter()
    oracle.evaluate(db, w.batch, root_range=(0, n), threads=cores)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "rows/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(), "nproc": os.cpu_count(), "wall_s": round(dt, 3),
            "sample": f"first {n} of {F.nrows} fact rows of {w.name} (all dims, whole batch), "
                      f"{cores} OpenMP threads, {dt:.1f} s"}


REF_BUDGET_S = 150.0  # --impl reference: CPU seconds the timed steps may take in total


def run_reference(args, rank, world):
    if rank != 0:
        return
    w = workload(args.config)
    per_step = []
    rows = args.ref_rows
    if rows <= 0:  # auto: size each step's sample so the whole run takes about REF_BUDGET_S of CPU
        probe = cpu_baseline(w, 50_000)
        rows = int(probe["value"] * REF_BUDGET_S / (args.warmup + args.steps))
        rows = max(2_000, min(400_000, rows))
    for i in range(args.warmup + args.steps):
        b = cpu_baseline(w, rows)
        if i >= args.warmup:
            per_step.append(rows / b["value"])
    cores = b["cores"]
    N = w.db.rel(w.db.root).nrows
    t = sum(per_step)
    value = rows * args.steps / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            # the own arm's workload, named the same way; each step evaluates a bounded sample of it
            "config": {"workload": f"{args.config}: {w.batch[0].name if w.batch else ''} batch, "
                                   f"{N} fact rows, {synth.n_aggregates(w.batch)} aggregates",
                       "fact_rows": N, "aggregates": synth.n_aggregates(w.batch),
                       "sample": f"first {rows} of {N} fact rows per step"},
            "cpu_baseline": {"value": value, "unit": "rows/s", "cores": cores, "kind": "oracle",
                             "cpu_model": b.get("cpu_model"),
                             "sample": f"first {rows} fact rows of {args.config} per step, {cores} OpenMP threads"},
            "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C5"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-rows", type=int, default=4_000_000)
    ap.add_argument("--ref-rows", type=int, default=0, help="rows per reference step (0: sized to the run)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: launch the N ranks the way the driver does (torch.distributed.run)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}", file=sys.stderr)

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1906_08687_b200 import lmfao

    torch.cuda.set_device(local)
    # a dedicated (non-default) stream: lmfao_run and the CUDA events share it
    torch.cuda.set_stream(torch.cuda.Stream())
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workload(args.config)

    def new_engine():
        uid = None
        if world > 1:
            t = torch.zeros(lmfao.UNIQUE_ID_BYTES, dtype=torch.uint8, device="cuda")
            if rank == 0:
                t.copy_(torch.frombuffer(bytearray(lmfao.lmfao_unique_id()), dtype=torch.uint8))
            dist.broadcast(t, 0)
            uid = bytes(t.cpu().numpy().tobytes())
        return lmfao.Engine(device=local, rank=rank, world=world, unique_id=uid)

    eng = new_engine()
    t_load = time.perf_counter()
    qids = lmfao.load(eng, w.db, w.batch)
    torch.cuda.synchronize()
    t_plan = time.perf_counter()
    eng.plan()
    torch.cuda.synchronize()
    load_s = time.perf_counter() - t_load
    plan_s = time.perf_counter() - t_plan
    info = eng.plan_info()
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    for _ in range(args.warmup):
        eng.run(sptr)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            eng.run(sptr)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    info = eng.plan_info()
    # dominant kernel: CUDA events around the root-scan launches (eager runs, same stream)
    eng.profile(True)
    for _ in range(min(args.steps, 200)):
        eng.run(sptr)
    scan_ms, scan_n = eng.profile_read()
    collective = None
    if world > 1:  # the all-reduce of the partial results, timed on the run stream
        ci = eng.plan_info()
        if "collective_ms" in ci:
            collective = {"ms_per_step": ci["collective_ms"], "bytes_per_step": ci["collective_bytes"],
                          "backend": "nccl"}
    eng.profile(False)
    launches_per_run = info.get("launches_last_run", 0)
    if world > 1:
        t = torch.tensor([ms, scan_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, scan_ms = float(t[0]), float(t[1])
    N = w.db.rel(w.db.root).nrows
    value = N * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (root scan) on this rank's shard
    peak, peak_kind = measured_peak()
    rows_rank = info["root_rows"]
    alg_bytes = BYTES_PER_ROW[args.config] * rows_rank + dim_feature_bytes(w)
    scan_avg_s = (scan_ms / max(scan_n, 1)) / 1e3
    achieved = alg_bytes / scan_avg_s / 1e9 if scan_n else None
    # the committed ncu capture is of the 1-GPU launch; a shard's launch has no capture
    traffic = committed_traffic(args.config) if world == 1 else None

    # result check (cheap): the count equals the fact rows
    keys, vals, counts = eng.fetch(qids[0])
    assert int(counts[0]) == N, (int(counts[0]), N)
    res_bytes = sum(vals.nbytes if q == qids[0] else 0 for q in qids) + 8

    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        pinned = {}
        for r in w.db.relations:
            pinned[r.name] = {c: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for c, v in r.cols.items()}
        h2d = sum(t.numel() * t.element_size() for d in pinned.values() for t in d.values())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times = []
        phases = {k: [] for k in ("create", "add_relation", "prepare", "plan", "run", "fetch")}
        for i in range(args.e2e_steps + 1):
            barrier()
            t = [time.perf_counter()]
            e = new_engine()
            t.append(time.perf_counter())
            for r in w.db.relations:
                e.add_relation(r.name, pinned[r.name])
            t.append(time.perf_counter())
            e.set_join_tree(w.db.root, list(w.db.edges))
            e.prepare()
            t.append(time.perf_counter())
            qids_e = [e.add_query(list(q.groupby), list(q.udafs)) for q in w.batch]
            e.plan()
            t.append(time.perf_counter())
            e.run(sptr)
            torch.cuda.current_stream().synchronize()
            t.append(time.perf_counter())
            k, v, c = e.fetch(qids_e[0])
            barrier()
            t.append(time.perf_counter())
            if i > 0:
                times.append(t[-1] - t[0])
                for name, a, b in zip(phases, t[:-1], t[1:]):
                    phases[name].append(1e3 * (b - a))
            e.close()
        tt = max(times) if world == 1 else None
        if world > 1:
            t = torch.tensor([sum(times)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tt = float(t[0]) / len(times)
        else:
            tt = sum(times) / len(times)
        e2e = {"value": N / tt, "unit": "rows/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(res_bytes),
               "s_per_step": tt, "what": "add_relation from pinned host + prepare (sort) + plan + run + fetch",
               "phases_ms": {k: round(statistics.median(v), 2) for k, v in phases.items()}}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, args.cpu_rows)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {w.batch[0].name if w.batch else ''} batch, "
                                   f"{N} fact rows, {synth.n_aggregates(w.batch)} aggregates",
                       "fact_rows": N, "aggregates": synth.n_aggregates(w.batch),
                       "parallelism": f"fact row-sharded x{world}, dims replicated",
                       "l2": "inputs (fact 760 MB) larger than L2 (126 MB); no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "peak_kind": peak_kind, "kernel": "root scan (c)+(d)",
                         "alg_bytes_per_launch": alg_bytes, "kernel_ms_avg": scan_avg_s * 1e3},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches_per_run) * args.steps,
            **({"collective": collective} if collective else {}),
            "clocks": clk.summary(), "load_s": load_s,
            # plan time (not in value): the planner incl. the scan layout of the root (a second,
            # re-laid-out copy of the fact: x in DMMA lane order + run-flagged keys, 76 B/row) and
            # the static cost-balanced chunking
            "plan_s": plan_s, "plan": info.get("fast_path"),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
