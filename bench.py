"""Benchmark: schedule plans evaluated/sec (BASELINE.json metric) on the cfg3 workload.

Workload (config.workload = "cfg3", BASELINE configs[2]): exhaustive sweep of all 3^16 =
43,046,721 plans of CTRDNN16 x {CPU, V100, V100-v1} (limit 5e4) with the fused (cost, index)
argmin, i.e. what brute_force computes without its 2^24 cap (ls/baselines.py:63-87). One step =
one full sweep; at N GPUs rank r sweeps indices r, r+N, r+2N, ... (strong scaling) and the
per-rank winners meet in one NCCL all_gather of 48-byte keys.

  value  plans/s of the device sweep (instance tables already resident, CUDA events on the
         launching stream, max over ranks; L2 flushed between steps by a 256 MiB write)
  e2e    the same metric through the public API with host inputs: every step stages the
         instance from host memory (hps_instance_create = H2D of the profile tables + table
         build), sweeps, gathers, reads the winner back and re-scores it (brute_force path)

Side measurements on the other BASELINE configs (keys of the same JSON line):
  cfg5   1e9 random plans of default_rng(0) (64 layers x 4 types; random_search's stream,
         ls/baselines.py:270-271), generated in-kernel, fused argmin; own roofline + CPU sample
  rl     cfg4 RL training (200 rounds x 4096 plans): round latency and time-to-best from
         per-round CUDA events, and the public train() call timed up to the best round
  cfg1   RL 200 rounds x 64 plans, seeds 0-2, public train() wall time per seed
  cfg2   exhaustive 3^8 brute force through the public brute_force() (wall, host result)
  enum_pruned  the cfg3 search with certified subtree pruning (same winner; not a plans-evaluated
         rate: 3^16 / wall time of the whole pruned search)

`--impl reference` times the CPU oracle (oracle/, the C restatement of the reference's path;
the reference itself is Python and has no compiled form) on all host cores over a strided
sample spanning the whole cfg3 index range.
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
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOAD = "cfg3"
METRIC = "schedule plans evaluated/sec"
UNIT = "plans/s"
SWEEP = 3 ** 16
# reference-algorithm FP64 operations per plan (24*E[S*C] + 9*N_bp + 13*61*S +
# 4*C + 88*L + 60*S with the measured means); cfg3: E[S*C]=7718, N_bp=697, S=11.0, C=689, L=16;
# cfg5: E[S*C]=43429, N_bp=1344, S=48.6, C=892, L=64
W_REF_OPS = {"cfg3": 205_052, "cfg5": 1_105_048}
PROFILES = ROOT / "profiles"
NCU_LAUNCHES = PROFILES / "r2_launches_bench_summary.json"   # per-kernel DRAM bytes and shares
NCU_METRICS = PROFILES / "r2_ncu_metrics.json"               # issue / lanes / FP64 pipe per kernel
# config shared by both arms (the reference arm times a bounded sample of the same workload)
CONFIG = {"workload": WORKLOAD, "sweep_plans": SWEEP, "layers": 16, "types": 3,
          "throughput_limit": 50000.0, "l2": "flushed between steps (256 MiB write)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=0, help="plans in the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rl", action="store_true", help="skip the cfg1/cfg4 RL measurements")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the cfg5 random-plan sweep")
    ap.add_argument("--no-small", action="store_true", help="skip the cfg1/cfg2 measurements")
    ap.add_argument("--cfg5-plans", type=int, default=10 ** 9)
    ap.add_argument("--no-prune", action="store_true", help="skip the pruned-search measurement")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def instance(name=WORKLOAD):
    from paper_2111_10635_b200 import load_fixture
    from paper_2111_10635_b200.model import JobParams
    g, c, limit = load_fixture(name)
    return g, c, JobParams(limit)


def _json(path):
    try:
        return json.loads(path.read_text())
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------------------- CPU arm

def cpu_oracle_rate(sample: int, threads: int):
    """Oracle plans/s on `threads` host threads over a strided sample spanning the whole cfg3
    index range (index i * (3^16 // sample) for i < sample)."""
    import numpy as np
    import oracle
    from paper_2111_10635_b200._abi import StagedDesc
    from paper_2111_10635_b200.model import ProvisionerConfig
    g, c, job = instance()
    sd = StagedDesc(g, c, job, ProvisionerConfig())
    idx = np.arange(sample, dtype=np.int64) * (SWEEP // sample)
    plans = np.empty((sample, 16), np.uint8)
    x = idx.copy()
    for l in range(15, -1, -1):
        plans[:, l] = x % 3
        x //= 3
    t0 = time.perf_counter()
    out = oracle.score_batch(sd, plans, threads, want_k=False)
    ok = (out["status"] & 0x7F) == 0
    best = int(np.argmin(np.where(ok, out["cost"], np.inf)))   # the sample's argmin (earliest on ties)
    dt = time.perf_counter() - t0
    return sample / dt, dt, int(idx[best])


def cpu_oracle_cfg5_rate(sample: int, threads: int):
    """Oracle plans/s on the first `sample` plans of cfg5's default_rng(0) stream."""
    import numpy as np
    import oracle
    from paper_2111_10635_b200._abi import StagedDesc, pcg64_words
    from paper_2111_10635_b200.model import ProvisionerConfig
    g, c, job = instance("cfg5")
    sd = StagedDesc(g, c, job, ProvisionerConfig())
    plans = oracle.random_plans(pcg64_words(np.random.default_rng(0).bit_generator.state), 4, 64, sample)
    t0 = time.perf_counter()
    oracle.score_batch(sd, plans, threads, want_k=False)
    dt = time.perf_counter() - t0
    return sample / dt, dt


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample = args.cpu_sample or 40_000 * threads
    for _ in range(max(0, args.warmup)):
        cpu_oracle_rate(max(1000, sample // 10), threads)
    rates, times = [], []
    for _ in range(max(1, args.steps)):
        r, dt, _ = cpu_oracle_rate(sample, threads)
        rates.append(r)
        times.append(dt)
    value = statistics.median(rates)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(CONFIG),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{sample} cfg3 enumeration indices i*{SWEEP // sample} "
                                       f"(strided over the whole 3^16 range) per step, C oracle "
                                       f"on {threads} host threads ({cpu_model()})"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- GPU arm

def fp64_peak(torch, lib, dev):
    """Measured DFMA throughput (TFLOP/s) of this GPU: the FP64 roofline denominator."""
    import ctypes as C
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks, threads, iters = sms * 8, 256, 4096
    out = torch.empty(blocks * threads, dtype=torch.float64, device=dev)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    lib.hps_probe_fp64(0, C.c_void_p(out.data_ptr()), blocks, threads, 64, s)
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.hps_probe_fp64(0, C.c_void_p(out.data_ptr()), blocks, threads, iters, s)
        e1.record()
        torch.cuda.synchronize()
        flops = 2.0 * 64 * blocks * threads * iters
        best = max(best, flops / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def _max_over_ranks(torch, dist, world, dev, values):
    t = torch.tensor(values, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def measure_rl(torch, g4, c4, job4):
    """cfg4 (BASELINE configs[3]): 200 rounds x 4096 plans on one GPU (latency-bound)."""
    from paper_2111_10635_b200 import policy
    cfg = policy.TrainerConfig(rounds=200, plans_per_round=4096, seed=0)
    p0, _ = policy.init_policy(g4, c4, cfg)
    policy.train(g4, c4, p0, policy.TrainerConfig(rounds=2, plans_per_round=4096, seed=0), job4, shard=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = policy.train(g4, c4, p0, cfg, job4, shard=False)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    opt = 0.11630007595486111  # brute-force optimum of cfg4 (index 4030; tests/golden/sweep_digests.json)
    hit = next((i for i, h in enumerate(res.history) if h.best_cost == opt), None)
    dev_round = [b - a for a, b in zip([0.0] + res.round_wall_s[:-1], res.round_wall_s)]
    out = {"workload": "cfg4", "rounds": 200, "plans_per_round": 4096, "gpus": 1, "wall_s": wall,
           "device_s": res.round_wall_s[-1], "round_ms_median": 1e3 * statistics.median(dev_round),
           "best_cost": res.best.cost, "best_plan": list(res.best.plan.assignment),
           "round_of_best": hit + 1 if hit is not None else None,
           "time_to_best_s": res.round_wall_s[hit] if hit is not None else None,
           "time_to_best_note": "device time from the start of round 1 to the end of the round whose "
                                "best-ever cost first equals the brute-force optimum (CUDA events)"}
    if hit is not None:   # the public call a user makes, stopped at that round, host wall incl. sync
        cfg_hit = policy.TrainerConfig(rounds=hit + 1, plans_per_round=4096, seed=0)
        walls = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = policy.train(g4, c4, p0, cfg_hit, job4, shard=False)
            walls.append(time.perf_counter() - t0)
            assert r.best.cost == opt
        out["train_call_to_best_s"] = min(walls)
    out["reference_cpu"] = {"wall_s": 404.3, "time_to_best_s": 15.3,
                            "source": "BASELINE.md §2: the Python reference on 1 core of the build "
                                      "container (not re-run on this box; the reference is not installed here)"}
    return out


def measure_cfg1(torch):
    """cfg1 (BASELINE configs[0]): RL 200 rounds x 64 plans, seeds 0-2, public train()."""
    from paper_2111_10635_b200 import policy
    g1, c1, job1 = instance("cfg1")
    res = {}
    for seed in (0, 1, 2):
        cfg = policy.TrainerConfig(rounds=200, plans_per_round=64, seed=seed)
        p0, _ = policy.init_policy(g1, c1, cfg)
        policy.train(g1, c1, p0, policy.TrainerConfig(rounds=2, plans_per_round=64, seed=seed), job1, shard=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = policy.train(g1, c1, p0, cfg, job1, shard=False)
        torch.cuda.synchronize()
        res[f"seed{seed}"] = {"wall_s": time.perf_counter() - t0, "device_s": r.round_wall_s[-1],
                              "best_cost": r.best.cost, "best_plan": list(r.best.plan.assignment)}
    return {"workload": "cfg1", "rounds": 200, "plans_per_round": 64, **res,
            "reference_cpu_s_per_seed": [2.3, 2.6],
            "reference_source": "BASELINE.md §2 (Python reference, 1 core of the build container)"}


def measure_cfg2(torch):
    """cfg2 (BASELINE configs[1]): exhaustive 3^8 = 6,561 plans through the public brute_force()
    (instance staged from host memory each call, winner re-scored and read back), beside the C
    oracle's sweep of the same plans on this box's host cores."""
    import oracle
    import paper_2111_10635_b200.scoring as scoring
    from paper_2111_10635_b200._abi import StagedDesc
    from paper_2111_10635_b200.model import ProvisionerConfig
    from paper_2111_10635_b200.search import brute_force
    g2, c2, job2 = instance("cfg2")
    walls = []
    for i in range(6):
        scoring._INSTANCES.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        best = brute_force(g2, c2, job2)
        torch.cuda.synchronize()
        if i:
            walls.append(time.perf_counter() - t0)
    sd = StagedDesc(g2, c2, job2, ProvisionerConfig())
    cpu = {}
    for th in (1, os.cpu_count() or 1):
        t0 = time.perf_counter()
        bc, bi, _ = oracle.enum_argmin(sd, 0, 3 ** 8, th)
        cpu[f"oracle_{th}_threads_s"] = time.perf_counter() - t0
        assert bc == best.cost
    return {"workload": "cfg2", "plans": 6561, "brute_force_wall_s": statistics.median(walls),
            "plans_per_s": 6561 / statistics.median(walls), "best_cost": best.cost,
            "best_plan": list(best.plan.assignment), **cpu,
            "reference_cpu_s": 2.38, "reference_source": "BASELINE.md §2 (Python reference, 1 core)"}


def measure_pruned(torch, inst, total, full_key):
    """Pruning-assisted exhaustive search of the same cfg3 space (hps_enum_argmin_pruned): certified
    per-prefix cost lower bounds skip index ranges that cannot hold the winner, the rest are swept
    exactly. Reported apart from `value` (which scores every plan); the winner must equal the full
    sweep's, ties included."""
    import paper_2111_10635_b200.scoring as scoring
    from paper_2111_10635_b200.search import brute_force
    inst.enum_argmin_pruned()   # warm-up
    walls, keys = [], []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        key, st = inst.enum_argmin_pruned()   # synchronous (sizes the survivor sweep on the host)
        walls.append(time.perf_counter() - t0)
        keys.append(key)
    assert all(k["rank"] == full_key["rank"] and k["cost"] == full_key["cost"] for k in keys)
    g, c, job = instance()
    e2e = []
    for i in range(4):   # public API: brute_force(prune=True), instance staged from host memory
        scoring._INSTANCES.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        best = brute_force(g, c, job, enumeration_cap=total, prune=True)
        if i:
            e2e.append(time.perf_counter() - t0)
    assert best.cost == full_key["cost"]
    t = statistics.median(walls)
    return {"workload": WORKLOAD, "plans_covered": total, "ms": 1e3 * t,
            "effective_plans_per_s": total / t, "evaluated": st["evaluated"],
            "evaluated_fraction": st["evaluated"] / total, "depth": st["depth"],
            "prefixes": st["prefixes"], "surviving_prefixes": st["survivors"],
            "incumbent_cost": st["incumbent_cost"], "winner_index": key["rank"],
            "winner_cost": key["cost"], "same_winner_as_full_sweep": True,
            "e2e_brute_force_prune_s": statistics.median(e2e),
            "note": "exact search with certified subtree lower bounds (csrc/hps_prune.cuh); rate = "
                    "3^16 / wall time of the whole call (bounds, incumbent sweep, survivor sweep); "
                    "not a plans-evaluated rate"}


def measure_cfg5(torch, dist, world, rank, dev, n_total, peak):
    """cfg5 (BASELINE configs[4]): n_total random plans of default_rng(0), 64 layers x 4 types.
    Plans are generated in-kernel (numpy Generator.integers replica) and reduced by the fused
    argmin; ranks take contiguous slices of the stream."""
    import numpy as np
    from paper_2111_10635_b200.instance import DeviceInstance, pcg_from_generator
    from paper_2111_10635_b200.search import allgather_argmin, shard_range
    g5, c5, job5 = instance("cfg5")
    inst5 = DeviceInstance(g5, c5, job5)
    pcg = pcg_from_generator(np.random.default_rng(0))
    lo, hi = shard_range(0, n_total, rank, world)
    for _ in range(3):   # warm-up on a 2^22-plan slice (pools, caches)
        inst5.read_argmin(inst5.random_argmin_async(pcg, lo, min(hi - lo, 1 << 22)))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    buf = inst5.random_argmin_async(pcg, lo, hi - lo)
    e1.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(torch, dist, world, dev, [e0.elapsed_time(e1)])[0]
    key = allgather_argmin(buf)
    rate = n_total / (ms * 1e-3)
    my_rate = (hi - lo) / (e0.elapsed_time(e1) * 1e-3)
    achieved = my_rate * W_REF_OPS["cfg5"] / 1e12
    return {"workload": "cfg5", "layers": 64, "types": 4, "plans": n_total, "ms": ms,
            "plans_per_s": rate, "winner_rank": str(key["rank"]), "winner_cost": key["cost"],
            "feasible": key["feasible"], "evaluated": key["evaluated"],
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None,
                         "note": f"plans/s x {W_REF_OPS['cfg5']} reference-algorithm FP64 ops per "
                                 "plan (SURVEY.md §8(d)) / measured DFMA peak"},
            "note": "first n plans of default_rng(0).integers(0,4,(n,64)) = random_search(seed=0)'s "
                    "stream (ls/baselines.py:270-271), penalties included in the argmin"}


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2111_10635_b200 import _abi
    from paper_2111_10635_b200.instance import DeviceInstance
    from paper_2111_10635_b200.search import allgather_argmin, brute_force, enum_shard_async, shard_strided

    rank, world, local = dist_env()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL_DEBUG stays the caller's (the image sets VERSION). NCCL prints its banner on fd 1
        # while the communicator is created: fd 1 points at stderr for that window, so stdout
        # keeps exactly one JSON line and the NCCL lines stay in the log.
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    g, c, job = instance()
    T, L = c.num_types, g.num_layers
    total = T ** L
    my_plans = shard_strided(0, total, rank, world)[2]  # every world-th index (balanced)
    inst = DeviceInstance(g, c, job)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def sweep():
        return allgather_argmin(enum_shard_async(inst, 0, total, rank, world, True))

    for _ in range(max(3, args.warmup)):
        key = sweep()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = []
    keys = []
    launches0 = inst.lib.hps_launch_count()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            buf = enum_shard_async(inst, 0, total, rank, world, True)
            e1.record()
            keys.append(allgather_argmin(buf))  # the exchange (and its host read) follows
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    my_launches = inst.lib.hps_launch_count() - launches0   # this rank's kernels, timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    my_total = sum(step_ms)
    per_rank_ms = [my_total / args.steps]
    if world > 1:   # diagnostic: every rank's mean step time (the value uses the max)
        pr = torch.zeros(world, dtype=torch.float64, device=dev)
        pr[rank] = my_total / args.steps
        dist.all_reduce(pr)
        per_rank_ms = [float(x) for x in pr.cpu()]
    total_ms = _max_over_ranks(torch, dist, world, dev, [my_total])[0]
    nl = torch.tensor([my_launches], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(nl)
    gpu_launches = int(nl.item())   # summed over ranks
    value = total * args.steps / (total_ms * 1e-3)
    key = keys[-1]
    assert all(k["rank"] == key["rank"] and k["cost"] == key["cost"] for k in keys)

    # ---- e2e: the public brute_force path with host inputs, every step ----
    import paper_2111_10635_b200.scoring as scoring
    e2e_ms = []
    for i in range(args.steps + 1):
        scoring._INSTANCES.clear()  # force re-staging from host memory (H2D inside the step)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        best = brute_force(g, c, job, enumeration_cap=total)
        torch.cuda.synchronize()
        if i > 0:  # first call is warm-up (library load, allocator pools)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    assert best.cost == key["cost"]
    e2e_value = total * args.steps / (_max_over_ranks(torch, dist, world, dev, [sum(e2e_ms)])[0] * 1e-3)
    h2d = 4 * T * L * 8 + T * (8 + 8 + 1)  # profile tables + prices/quotas/is_cpu
    d2h = _abi.ARGMIN_NBYTES * world + 8 * 6  # gathered keys + the re-scored winner's outputs

    peak = fp64_peak(torch, inst.lib, dev) if rank == 0 else 0.0
    pruned = measure_pruned(torch, inst, total, key) if (rank == 0 and world == 1 and not args.no_prune) else None
    rl = cfg1 = cfg2 = None
    if not args.no_rl and rank == 0:  # latency-bound per round: timed unsharded on one GPU
        rl = measure_rl(torch, *instance("cfg4"))
        if not args.no_small:
            cfg1 = measure_cfg1(torch)
    if not args.no_small and world == 1:   # brute_force would all_gather across ranks
        cfg2 = measure_cfg2(torch)
    r5 = None
    if not args.no_cfg5:
        r5 = measure_cfg5(torch, dist, world, rank, dev, args.cfg5_plans, peak)

    if rank == 0:
        kernel_plans_per_s = my_plans / (statistics.median(step_ms) * 1e-3)
        achieved = kernel_plans_per_s * W_REF_OPS[WORKLOAD] / 1e12
        launches = _json(NCU_LAUNCHES)
        metrics = _json(NCU_METRICS)
        traffic = launches["dram_bytes_per_plan"] * my_plans if launches else None
        roof = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "note": "achieved = plans/s of the sweep (all its kernels, one step) x "
                        f"reference-algorithm FP64 ops per plan ({W_REF_OPS[WORKLOAD]}, SURVEY.md "
                        "§8(d)); peak = DFMA probe measured in this run (MEASURED_PEAKS.json has no "
                        "FP64); traffic = DRAM bytes per step from the committed ncu launch list "
                        f"({NCU_LAUNCHES.name})"}
        if metrics:   # measured pipe / issue / lane utilisation of the sweep kernels (ncu, same command)
            roof["ncu"] = metrics
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(CONFIG),
            "parallelism": f"strided enumeration shards x{world}",
            "result": {"winner_index": key["rank"], "winner_cost": key["cost"],
                       "feasible_plans": key["feasible"]},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": gpu_launches,
            "roofline": roof,
            "clocks": clocks.summary(),
            "per_rank_ms": per_rank_ms,
        }
        if rl is not None:
            line["rl"] = rl
        if cfg1 is not None:
            line["cfg1_rl"] = cfg1
        if cfg2 is not None:
            line["cfg2_bf"] = cfg2
        if r5 is not None:
            line["cfg5_random"] = r5
        if pruned is not None:
            line["enum_pruned"] = pruned
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            sample = args.cpu_sample or 40_000 * threads
            rate, dt, _ = cpu_oracle_rate(sample, threads)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                    "sample": f"{sample} cfg3 enumeration indices strided over the "
                                              f"whole 3^16 range in {dt:.1f} s ({cpu_model()})"}
            if r5 is not None:
                s5 = 16_000 * threads
                rate5, dt5 = cpu_oracle_cfg5_rate(s5, threads)
                r5["cpu_baseline"] = {"value": rate5, "unit": UNIT, "cores": threads, "kind": "port",
                                      "sample": f"first {s5} plans of the stream in {dt5:.1f} s"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
