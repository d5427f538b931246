"""Benchmark: HBP fitness evaluation of a GA population on B200 (one JSON line).

Default workload (N=1): BASELINE.json config 4's single-GPU shape, "syn20k" --
synthetic Euclidean n = m = 20000, p = 200, a 4096-chromosome population
evaluated per step.  A step = one evaluation of the whole
population (the batch evolve_block hands to fitness(), ga.cpp:147).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config syn20k|syn5k|sweep:P|pmed40]
  python bench.py --impl reference ...   # the reference's own fitness() on the host cores

Under torchrun (N>1) the BASELINE population is split contiguously over the
ranks (BASELINE configs 3-4: one batch, strong scaling), every rank evaluates
its shard against locally built, replicated tables, and the costs are
all-gathered (NCCL) inside the timed step; `--scaling weak` gives every rank a
whole population of its own instead.

Timing: W warm-up steps, then K steps; before every timed step a 512 MiB
buffer is written to flush L2; each step is bracketed by CUDA events on the
stream the kernels run on; the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fitness evals/s & GA gens/s (pmed40; synthetic n=m=20000,p=200), % HBM roofline"
CONFIGS = {
    "syn20k": dict(npts=20000, p=200, count=4096,
                   workload="syn20k: synthetic Euclidean n=m=20000, p=200, 4096-chromosome fitness batch"),
    "syn5k": dict(npts=5000, p=50, count=1024,
                  workload="syn5k: synthetic Euclidean n=m=5000, p=50, 1024-chromosome fitness batch"),
    "pmed40": dict(npts=900, p=90, count=15360,
                   workload="pmed40-shape: synthetic Euclidean n=m=900, p=90, 60x256 population "
                            "(OR-Library pmed40 file absent offline)"),
}


def config_for(name: str) -> dict:
    if name.startswith("sweep:"):
        p = int(name.split(":")[1])
        return dict(npts=10000, p=p, count=4096,
                    workload=f"sweep: synthetic Euclidean n=m=10000, p={p}, 4096-chromosome fitness batch")
    return dict(CONFIGS[name])


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock and throttle reasons sampled every ~2 ms through NVML during the
    timed region (the profiling recipe's clocks line, at a rate that sees
    millisecond-scale regions)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

            def sample():
                try:
                    self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for bit, name in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(name)
                except Exception:
                    pass

            def run():
                while not self._stop.is_set():
                    sample()
                    time.sleep(0.002)

            self._sample = sample
            sample()  # the region's start, even when it is shorter than a tick

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *exc):
        if getattr(self, "_sample", None):
            self._sample()  # the region's end, even when it was shorter than a tick
        self._stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# PMB_DIST_BACKEND=gloo and PMB_DEVICE=<d> let a multi-rank run share one GPU
# for plumbing tests (host-side collectives only; no kernel waits on another rank).
BACKEND = os.environ.get("PMB_DIST_BACKEND", "nccl")


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("PMB_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(BACKEND)
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allgather_into(dst, src):
    """dst (world * len(src)) <- every rank's src, in rank order.  NCCL on the
    device tensors; over gloo (CPU plumbing tests) through host copies."""
    import torch
    import torch.distributed as dist
    if BACKEND == "nccl":
        dist.all_gather_into_tensor(dst, src)
        return
    parts = [torch.empty_like(src, device="cpu") for _ in range(dist.get_world_size())]
    dist.all_gather(parts, src.cpu())
    dst.copy_(torch.cat(parts))


def shard(count: int, world: int, rank: int):
    """The strong split (BASELINE configs 3-4): rank r evaluates the contiguous
    chromosomes [r * count / world, (r + 1) * count / world) of the one batch."""
    if count % world:
        raise ValueError(f"strong scaling needs the population ({count}) divisible by {world}")
    per = count // world
    return rank * per, (rank + 1) * per


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def load_synth():
    """paper_1610_10061_b200/synth.py loaded by path: the reference arm must not
    import the package (whose __init__ maps libpmedian_b200.so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("pmb_synth", os.path.join(ROOT, "paper_1610_10061_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def source_hash(*rel):
    import hashlib
    h = hashlib.sha256()
    for r in rel:
        with open(os.path.join(ROOT, r), "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def ncu_record(config: str, kernel: str):
    """The committed ncu --set full summary of the dominant kernel
    (profiles/ncu_<kernel>_<config>.json, tools/ncu_to_json.py), stamped with the
    hash of the kernel source it was captured from; `stale` when the source
    changed since."""
    path = os.path.join(ROOT, "profiles", f"ncu_{kernel}_{config}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        rec = json.load(f)
    src = rec.get("source_file", "paper_1610_10061_b200/csrc/fitness.cu")
    rec["stale"] = rec.get("source_sha16") != source_hash(src)
    rec["file"] = os.path.relpath(path, ROOT)
    return rec


def cpu_reference_sample(costs_host, n, m, p, words, gpu_costs, budget_s=10.0):
    """The reference's own build_ordering + fitness() (oracle/_ref, compiled from
    /root/reference sources) on all host threads over a bounded sample of the
    same population, on the reference's OWN tables (so the GPU costs are checked
    end to end: K1 and K2)."""
    from oracle.oracle import RefLib
    if not RefLib.available():
        return None
    ref = RefLib()
    t0 = time.perf_counter()
    ri = ref.create(n, m, p, costs_host)  # Instance + build_ordering (single thread, ordering.cpp:10-38)
    build_s = time.perf_counter() - t0
    threads = len(os.sched_getaffinity(0))
    probe = words[:threads]
    t0 = time.perf_counter()
    rc, pc, _ = ri.evaluate(probe, threads)
    dt = time.perf_counter() - t0
    per_eval = dt / max(1, probe.shape[0]) * threads  # single-thread seconds per eval
    count = int(max(threads, min(words.shape[0], budget_s * threads / max(per_eval, 1e-9))))
    count = max(threads, count // threads * threads)
    sample = words[:count]
    t0 = time.perf_counter()
    rc, costs, _ = ri.evaluate(sample, threads)
    dt = time.perf_counter() - t0
    parity = bool(rc == 0 and (costs == gpu_costs[:count]).all())
    # one worker too, ~2 s of work
    one = int(max(1, min(count, 2.0 / max(per_eval, 1e-9))))
    t0 = time.perf_counter()
    ri.evaluate(words[:one], 1)
    dt1 = time.perf_counter() - t0
    return {"value": count / dt, "unit": "evals/s", "cores": threads, "kind": "reference",
            "sample": f"first {count} of the {words.shape[0]} chromosomes of the same population, reference "
                      f"fitness() (proj/src/ordering.cpp:40-59) on the reference's own build_ordering tables, "
                      f"{threads} host threads, {dt:.1f} s",
            "bit_exact_vs_gpu": parity, "single_thread_value": one / dt1,
            "reference_build_ordering_s": round(build_s, 2), "cpu_model": cpu_model()}


def workload_config(cfg, n, m, p, world, scaling):
    """The `config` object: workload-defining keys only, identical in both arms."""
    count = cfg["count"]
    total = count if scaling == "strong" else count * world
    return {"workload": cfg["workload"], "n": n, "m": m, "p": p, "population": total,
            "scaling": scaling, "instance_seed": 12345, "population_seed": 7}


def run_ours(args):
    import torch

    import paper_1610_10061_b200 as pm
    from paper_1610_10061_b200 import synth

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = config_for(args.config)
    n = m = cfg["npts"]
    p, count = cfg["p"], cfg["count"]
    wp = (m + 63) // 64
    scaling = args.scaling
    if scaling == "strong" and count % world:
        raise SystemExit(f"strong scaling needs the population ({count}) divisible by {world}")

    ctx = pm.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream)
    if args.kernel != "auto":
        ctx.set_eval_kernel({"scan": pm.EVAL_SCAN, "gather": pm.EVAL_GATHER}[args.kernel])

    costs = synth.euclid_costs(n, 12345, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.set_instance(costs, n, m, p)
    build_s = time.perf_counter() - t0
    del costs
    torch.cuda.empty_cache()

    # strong: one global population (seed 7), contiguous shard per rank, costs
    # all-gathered back; weak: every rank its own population of `count`
    if scaling == "strong":
        pop_all = synth.random_population(m, p, count, seed=7)
        lo, hi = shard(count, world, rank)
        per = hi - lo
        pop = pop_all[lo:hi]
    else:
        pop_all = None
        per = count
        pop = synth.random_population(m, p, count, seed=7 + 1000 * rank)
    words_host = torch.from_numpy(np.ascontiguousarray(pop).view(np.int64)).pin_memory()
    words = words_host.to(dev)
    out = torch.empty(per, dtype=torch.int64, device=dev)
    gathered = torch.empty(per * world, dtype=torch.int64, device=dev) if scaling == "strong" else None
    sumk = torch.empty(per, dtype=torch.int64, device=dev)
    ctx.scan_depths_device(words, sumk, per, wp)
    algo_bytes = 12 * int(sumk.sum().item()) + 8 * wp * per  # SURVEY.md 8(d) B_eval x shard
    ti = ctx.table_info()
    col_bytes = ti.site_bytes + ti.dist_bytes
    gsum = torch.zeros((per + 31) // 32, dtype=torch.int64, device=dev)
    cmax = torch.zeros(n, dtype=torch.int32, device=dev)
    ctx.scan_walks_device(words, gsum, cmax, per, wp)
    group_stream_bytes = int(gsum.sum().item()) * col_bytes
    ts = (m + 2) // 2 * 2
    dram_floor_bytes = int(cmax.to(torch.int64).sum().item()) * col_bytes + ((per + 63) // 64) * ts * 8 + per * 8
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def gather_costs():
        if gathered is not None and world > 1:
            allgather_into(gathered, out)

    for _ in range(args.warmup):
        ctx.evaluate_device(words, out, per, wp, check=False)
        gather_costs()
    ctx.check_errors()
    gpu_costs = out.cpu().numpy()
    if scaling == "strong":
        # the split is exact: the gathered costs equal one evaluation of the whole batch
        full = torch.empty(count, dtype=torch.int64, device=dev)
        wfull = torch.from_numpy(np.ascontiguousarray(pop_all).view(np.int64)).to(dev)
        ctx.evaluate_device(wfull, full, count, wp, check=True)
        if world > 1:
            assert torch.equal(gathered, full), "strong split: gathered costs differ from the whole-batch result"
        del wfull

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ctx.profile_read()
    ctx.set_profiling(True)
    launches0 = ctx.kernel_launches
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            flush.zero_()
            starts[s].record(stream)
            ctx.evaluate_device(words, out, per, wp, check=False)
            gather_costs()
            ends[s].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = ctx.kernel_launches - launches0
    ctx.set_profiling(False)
    kern_ms, kern_n = ctx.profile_read()
    ctx.check_errors()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    total_ms = max_over_ranks(float(sum(step_ms)), world)
    units = count if scaling == "strong" else count * world
    value = units * args.steps / (total_ms / 1e3)

    # e2e: the public host-buffer call (pm_evaluate) with the H2D of this rank's
    # chromosomes from pinned memory and the D2H of its costs (and, strong, the
    # all-gather of the costs) inside a host wall-clock bracket per step
    host_pop = words_host.numpy().view(np.uint64)
    for _ in range(2):
        ctx.evaluate(host_pop)
    e2e_s = []
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk2:
        for s in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = ctx.evaluate(host_pop)
            if scaling == "strong" and world > 1:
                g = torch.empty(per * world, dtype=torch.int64, device=dev)
                allgather_into(g, torch.from_numpy(res).to(dev))
                res_all = g.cpu().numpy()
                assert res_all.shape[0] == count
            e2e_s.append(time.perf_counter() - t0)
    barrier(world)
    assert (res == gpu_costs).all()
    e2e_total = max_over_ranks(float(sum(e2e_s)), world)
    e2e_value = units * args.steps / e2e_total

    peak, peak_src = peaks()
    avg_kernel_s = kern_ms / max(1, kern_n) / 1e3
    achieved = algo_bytes / avg_kernel_s / 1e9
    kname = "k_scan" if (ctx.auto_eval_kernel() == 1 and args.kernel == "auto") or args.kernel == "scan" \
        else "k_gather"
    kernel_name = {"k_scan": "k_scan (K2, bit-sliced scan)", "k_gather": "k_gather (K2b, gather-min)"}[kname]
    ncu = ncu_record(args.config, kname)
    physical = {
        "group_stream_bytes": group_stream_bytes,
        "group_stream_gbs": group_stream_bytes / avg_kernel_s / 1e9,
        "dram_floor_bytes": dram_floor_bytes,
        "dram_floor_gbs": dram_floor_bytes / avg_kernel_s / 1e9,
        "dram_floor_frac": dram_floor_bytes / avg_kernel_s / 1e9 / peak,
        "definition": "measured in this run (pm_scan_walks_device): group_stream = sum over 32-chromosome "
                      "groups and clients of the walk max_{c in group} k*_ic x (site+dist bytes) -- the row "
                      "prefixes K2 must stream from L2; dram_floor = sum over clients of the longest walk x "
                      "(site+dist bytes) + transposed masks + population + costs -- bytes that must come from "
                      "DRAM at least once per launch",
    }
    if ncu:
        physical["ncu_dram_bytes"] = ncu.get("dram_bytes")
        physical["ncu_dram_frac"] = (ncu["dram_bytes"] / avg_kernel_s / 1e9 / peak) if ncu.get("dram_bytes") else None
        physical["binding"] = {k: ncu.get(k) for k in ("l1tex_throughput_pct", "issue_active_pct",
                                                         "sm_throughput_pct", "lts_throughput_pct",
                                                         "dram_throughput_pct", "warp_instructions",
                                                         "duration_ms")}
        physical["ncu_source"] = {k: ncu.get(k) for k in ("file", "source_file", "source_sha16", "stale", "commit",
                                                           "captured")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        costs_host = synth.euclid_costs(n, 12345)
        cpu = cpu_reference_sample(costs_host, n, m, p, pop, gpu_costs, budget_s=args.cpu_seconds)
        del costs_host

    ga = None if args.no_ga else bench_ga(ctx, args, world, rank, local, n, m, p)
    evolved = None
    if rank == 0 and world == 1 and not args.no_ga and count % 256 == 0:
        evolved = evolved_population(ctx, pop, n, wp, stream, flush, args.steps, peak)

    clocks = clk.summary()
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "evals/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic (seeded Euclidean instance, uniform random p-subset population)",
        "config": workload_config(cfg, n, m, p, world, scaling),
        "details": {"per_gpu_chromosomes": per,
                    "parallelism": (f"one {count}-chromosome batch split contiguously over {world} GPU(s), "
                                    "costs all-gathered (NCCL) inside the step" if scaling == "strong" else
                                    f"{count} chromosomes per GPU, tables replicated, no data-path collective"),
                    "l2": "flushed before every timed step (512 MiB write)",
                    "kernel": kernel_name, "build_ordering_s": round(build_s, 3)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu.get("dram_bytes") if ncu else None,
                     "kernel": kernel_name, "avg_kernel_ms": avg_kernel_s * 1e3,
                     "algorithmic_bytes_per_launch": algo_bytes,
                     "bytes_definition": "SURVEY.md 8(d): B_eval = 12*sum_i k*_i + 8*ceil(m/64) per "
                                         "chromosome (reference layout, no reuse); effective-bandwidth "
                                         "figure, may exceed 1.0 -- see `physical` for the reuse-aware floors "
                                         "and the ncu-measured DRAM traffic and binding units",
                     "physical": physical,
                     "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": per * wp * 8,
                "d2h_bytes_per_step": per * 8,
                "call": "pm_evaluate (C ABI, host buffers; population from pinned memory); host wall clock "
                        "around each synchronous call" + (", plus the cost all-gather" if world > 1 and
                                                          scaling == "strong" else ""),
                "bytes_note": "per GPU per step"},
        "gpu_launches": launches,
        "clocks": clocks,
        "clocks_e2e": clk2.summary(),
        "ga": ga,
        "evolved_population": evolved,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


GA_GENS = 20


def bench_ga(ctx, args, world, rank, local, n, m, p):
    """GA gens/s (BASELINE metric's second half).  One generation = one run_ga
    loop iteration (ga.cpp:246-299).  Timed end to end on the host around
    pm_run_ga (device work, host population draw, stop test, migration)."""
    import paper_1610_10061_b200 as pm
    from paper_1610_10061_b200 import synth
    out = {}
    # syn20k-shape island GA (BASELINE config 4): 16 blocks x 256 = 4096
    # chromosomes in total, split over the ranks as islands (strong; weak: 16
    # blocks per GPU); the reference's exact population draw (device rank draw
    # + unranking over a 0.87 GB Pascal table), then the device draw (same
    # distribution)
    nb = 16 * world if args.scaling == "weak" else 16
    ag = None
    if world > 1 and BACKEND == "nccl":
        # the library's own NCCL exchange (pm_nccl_*); torch.distributed only
        # distributes the communicator's unique id
        import torch.distributed as dist
        box = [pm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        ag = pm.NcclComm(box[0], rank, world, local)
    elif world > 1:
        ag = pm.torch_allgather()  # gloo (CPU test runs)
    for pop_mode, key in (("reference", "islands"), ("device", "islands_device_population")):
        cfg = pm.ga_config(nb=nb, nt=256, evolve_limit=GA_GENS, saturation=GA_GENS + 1, seed=1,
                           population=pop_mode)
        warm = pm.ga_config(nb=nb, nt=256, evolve_limit=1, saturation=1, seed=2, population=pop_mode)
        ctx.run_ga(warm, rank=rank, world=world, allgather=ag)  # kernels loaded, Pascal table resident
        ctx.profile_read()
        ctx.set_profiling(True)  # CUDA events around every fitness-kernel launch of the run
        r = ctx.run_ga(cfg, rank=rank, world=world, allgather=ag)
        ctx.set_profiling(False)
        eval_ms, eval_launches = ctx.profile_read()
        out[key] = {"config": f"n=m={n}, p={p}, nb={nb} ({nb // world} per GPU), nt=256, {pop_mode} population draw",
                    "gens_per_s": r["kernels_executed"] / r["wall_time"], "generations": r["kernels_executed"],
                    "fitness_kernel_share_of_wall": eval_ms / 1e3 / r["wall_time"],
                    "fitness_kernel_launches": eval_launches,
                    "best_cost": r["best_cost"], "evals_per_gen_reference_semantics":
                        r["evaluations"] / r["kernels_executed"],
                    "device_evals_per_gen": r["device_evaluations"] / r["kernels_executed"],
                    "exchange": "none (1 island)" if world == 1 else (
                        "pm_nccl_allgather_device (library NCCL communicator, device buffers)" if BACKEND == "nccl"
                        else "torch.distributed gloo allgather")}
    if isinstance(ag, pm.NcclComm):
        ag.close()
    if world == 1 and args.orlib_dir:
        # BASELINE configs 1-2 on the real OR-Library files when supplied (tools/orlib_run.py)
        import subprocess
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "orlib_run.py"), "--orlib-dir",
                            args.orlib_dir, "--instances", "pmed1,pmed40"], capture_output=True, text=True)
        out["orlib"] = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    if world == 1 and rank == 0:
        # the paper's Table-1 shape (nb=60, nt=256) on a pmed40-sized synthetic instance
        import paper_1610_10061_b200 as pm2
        c2 = pm2.Context(local)
        c2.set_instance(synth.euclid_costs(900, 12345), 900, 900, 90)
        for pop_mode in ("reference", "device"):
            cfg = pm.ga_config(nb=60, nt=256, evolve_limit=GA_GENS, saturation=GA_GENS + 1, seed=1,
                               population=pop_mode)
            c2.run_ga(pm.ga_config(nb=60, nt=256, evolve_limit=1, saturation=1, seed=2, population=pop_mode))
            r = c2.run_ga(cfg)
            out[f"pmed40_shape_{pop_mode}_population"] = {
                "config": "synthetic Euclidean n=m=900, p=90, nb=60, nt=256 (OR-Library pmed40 absent)",
                "gens_per_s": r["kernels_executed"] / r["wall_time"], "generations": r["kernels_executed"],
                "best_cost": r["best_cost"],
                "evals_per_gen_reference_semantics": r["evaluations"] / r["kernels_executed"]}
        # full runs at the paper's Table-1 settings (evolve_limit=100, saturation=10,
        # acceptance.cpp:323-328), reference-exact population draw
        full = pm.ga_config(nb=60, nt=256, evolve_limit=100, saturation=10, seed=1)
        r = c2.run_ga(full)
        out["pmed40_shape_full_run"] = {
            "config": "synthetic Euclidean n=m=900, p=90, nb=60, nt=256, evolve_limit=100, saturation=10, seed 1",
            "generations": r["kernels_executed"], "kernel_of_best": r["kernel_of_best"],
            "best_cost": r["best_cost"], "wall_s": r["wall_time"]}
        c2.close()
        c3 = pm2.Context(local)
        c3.set_instance(synth.euclid_costs(100, 12345), 100, 100, 5)
        opt, nsub, t_ex = exhaustive_optimum(c3, 100, 5)
        r = c3.run_ga(full)
        out["pmed1_shape_full_run"] = {
            "config": "synthetic Euclidean n=m=100, p=5, nb=60, nt=256, evolve_limit=100, saturation=10, seed 1",
            "generations": r["kernels_executed"], "kernel_of_best": r["kernel_of_best"],
            "best_cost": r["best_cost"], "wall_s": r["wall_time"], "optimum": opt,
            "optimal": r["best_cost"] == opt,
            "optimum_by": f"device evaluation of all {nsub} p-subsets ({t_ex:.1f} s incl. host enumeration)"}
        c3.close()
    return out


def evolved_population(ctx, pop, n, wp, stream, flush, steps, peak):
    """SURVEY.md 8(d) secondary report: the same batch after 3 reference
    evolve_block generations (nt=256); evolved chromosomes keep clients near
    an open site, so k* is shorter than for uniform random subsets."""
    import torch

    import paper_1610_10061_b200 as pm
    count = pop.shape[0]
    cfg = pm.ga_config(nb=count // 256, nt=256, seed=1)
    ev = pop
    for kern in range(3):
        ev, _, _ = ctx.evolve_blocks(ev, cfg, kern)
    w = torch.from_numpy(np.ascontiguousarray(ev).view(np.int64)).cuda()
    out = torch.empty(count, dtype=torch.int64, device="cuda")
    sumk = torch.empty(count, dtype=torch.int64, device="cuda")
    ctx.scan_depths_device(w, sumk, count, wp)
    ks = int(sumk.sum().item())
    for _ in range(3):
        ctx.evaluate_device(w, out, count, wp, check=False)
    ctx.profile_read()
    ctx.set_profiling(True)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    torch.cuda.synchronize()
    for s in range(steps):
        flush.zero_()
        ev0[s].record(stream)
        ctx.evaluate_device(w, out, count, wp, check=False)
        ev1[s].record(stream)
    torch.cuda.synchronize()
    ctx.set_profiling(False)
    kern_ms, kern_n = ctx.profile_read()
    ctx.check_errors()
    ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1)) / steps
    kern_s = kern_ms / max(1, kern_n) / 1e3
    achieved = (12 * ks + 8 * wp * count) / kern_s / 1e9
    return {"config": f"the benchmark batch after 3 evolve_block generations (nb={count // 256}, nt=256, seed 1)",
            "evals_per_s": count / (ms / 1e3), "mean_k_star": ks / (count * n),
            "roofline_frac": achieved / peak}


def exhaustive_optimum(ctx, m, p):
    """min over every p-subset of range(m), each evaluated by the device path."""
    import torch

    from paper_1610_10061_b200 import synth
    t0 = time.perf_counter()
    best, total = None, 0
    for chunk in synth.all_subsets(m, p):
        w = torch.from_numpy(chunk.view(np.int64)).cuda()
        out = torch.empty(chunk.shape[0], dtype=torch.int64, device="cuda")
        ctx.evaluate_device(w, out, chunk.shape[0], chunk.shape[1], check=True)
        v = int(out.min().item())
        best = v if best is None else min(best, v)
        total += chunk.shape[0]
    return best, total, time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the reference's own CPU build_ordering + fitness()
    (oracle/_ref, compiled from /root/reference/proj/src) on all host cores, on
    the SAME workload as the GPU arm: every step evaluates the whole
    population.  Never imports the product package."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.oracle import RefLib
    synth = load_synth()
    cfg = config_for(args.config)
    n = m = cfg["npts"]
    p, count = cfg["p"], cfg["count"]
    if not RefLib.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpmref.so not built"}))
        return
    ref = RefLib()
    costs = synth.euclid_costs(n, 12345)
    t0 = time.perf_counter()
    ri = ref.create(n, m, p, costs)  # the reference's Instance + build_ordering (single thread)
    build_s = time.perf_counter() - t0
    del costs
    threads = len(os.sched_getaffinity(0))
    total = count if args.scaling == "strong" else count * world
    sample = min(total, args.ref_sample) if args.ref_sample else total
    pop = synth.random_population(m, p, sample, seed=7)
    for _ in range(args.warmup):
        ri.evaluate(pop, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rc, _, _ = ri.evaluate(pop, threads)
        times.append(time.perf_counter() - t0)
        assert rc == 0
    value = sample * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded Euclidean instance, uniform random p-subset population)",
        "config": workload_config(cfg, n, m, p, world, args.scaling),
        "details": {"parallelism": f"{threads} host threads (std::thread slices, ga.cpp:253-277)",
                    "build_ordering_s": round(build_s, 2),
                    "step": f"reference fitness() over {sample} chromosomes of the population",
                    "cpu_model": cpu_model()},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "reference",
                         "sample": f"{sample} chromosomes per step (the whole workload), {args.steps} steps"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    del ri
    if not args.no_ga:
        # the reference run_ga (ga.cpp:219-303) at the paper's Table-1 shape, all host threads
        ri = ref.create(900, 900, 90, synth.euclid_costs(900, 12345))
        rc, r = ri.run_ga(60, 256, 2, 10, 1, workers=threads)
        line["ga"] = {"pmed40_shape_reference_population": {
            "config": "synthetic Euclidean n=m=900, p=90, nb=60, nt=256; reference run_ga, "
                      f"{threads} worker threads",
            "gens_per_s": r["kernels_executed"] / r["wall_time"], "generations": r["kernels_executed"],
            "best_cost": r["best_cost"]}}
        # a full Table-1 run on the pmed1 shape (the 900/90 one would take minutes here)
        ri = ref.create(100, 100, 5, synth.euclid_costs(100, 12345))
        rc, r = ri.run_ga(60, 256, 100, 10, 1, workers=threads)
        line["ga"]["pmed1_shape_full_run"] = {
            "config": "synthetic Euclidean n=m=100, p=5, nb=60, nt=256, evolve_limit=100, saturation=10, seed 1; "
                      f"reference run_ga, {threads} worker threads",
            "generations": r["kernels_executed"], "kernel_of_best": r["kernel_of_best"],
            "best_cost": r["best_cost"], "wall_s": r["wall_time"]}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="syn20k")
    ap.add_argument("--kernel", default="auto", choices=["auto", "scan", "gather"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-sample", type=int, default=0)
    ap.add_argument("--no-ga", action="store_true")
    ap.add_argument("--orlib-dir", default=os.environ.get("PMB_ORLIB_DIR", ""),
                    help="OR-Library pmed files + pmedopt: adds BASELINE configs 1-2 (pmed1, pmed40) to `ga`")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default): the BASELINE population split over the GPUs; weak: per GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
