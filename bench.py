"""Benchmark: schedule plans evaluated/sec (BASELINE.json metric) on the cfg3 workload.

Workload (config.workload = "cfg3"): exhaustive sweep of all 3^16 = 43,046,721 plans of
CTRDNN16 x {CPU, V100, V100-v1} (limit 5e4) with the fused (cost, index) argmin, i.e. what
brute_force computes without its 2^24 cap (ls/baselines.py:63-87). One step = one full sweep;
at N GPUs the index range is split into N contiguous shards (strong scaling) and the per-rank
winners meet in one NCCL all_gather of 48-byte keys.

  value  plans/s of the device sweep (instance tables already resident, CUDA events, max
         over ranks; L2 flushed between steps)
  e2e    the same metric through the public API with host inputs: every step stages the
         instance from host memory (hps_instance_create = H2D of the profile tables + table
         build), sweeps, gathers, reads the winner back and re-scores it (brute_force path)

`--impl reference` times the CPU oracle (oracle/, the C restatement of the reference's path;
the reference itself is Python and has no compiled form) on all host cores over a bounded
index range of the same sweep.
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
# reference-algorithm FP64 operations per plan on cfg3 (24*E[S*C] + 9*N_bp +
# 13*61*S + 4*C + 88*L + 60*S with the measured means E[S*C]=7718, N_bp=697, S=11, C=689)
W_REF_OPS = 205_052
TRAFFIC_BYTES_PER_PLAN = 2098  # ncu dram__bytes_{read,write}.sum over a cfg3 sweep / plans (v36)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=0, help="plans in the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rl", action="store_true", help="skip the cfg4 RL time-to-best measurement")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the cfg5 random-plan measurements")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def instance():
    from paper_2111_10635_b200 import load_fixture
    from paper_2111_10635_b200.model import JobParams
    g, c, limit = load_fixture(WORKLOAD)
    return g, c, JobParams(limit)


# ----------------------------------------------------------------------------- CPU arm

def cpu_oracle_rate(sample: int, threads: int):
    """Oracle plans/s on `threads` host threads over a bounded index range of the sweep."""
    import oracle
    from paper_2111_10635_b200._abi import StagedDesc
    from paper_2111_10635_b200.model import ProvisionerConfig
    g, c, job = instance()
    sd = StagedDesc(g, c, job, ProvisionerConfig())
    begin = 3 ** 16 // 2  # middle of the enumeration (mixed CPU/GPU plans)
    t0 = time.perf_counter()
    oracle.enum_argmin(sd, begin, begin + sample, threads)
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
    sample = args.cpu_sample or 80_000 * threads
    for _ in range(max(0, args.warmup)):
        cpu_oracle_rate(max(1000, sample // 10), threads)
    rates, times = [], []
    for _ in range(max(1, args.steps)):
        r, dt = cpu_oracle_rate(sample, threads)
        rates.append(r)
        times.append(dt)
    value = statistics.median(rates)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "plans_per_step": sample,
                       "parallelism": f"host threads x{threads}"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{sample} consecutive enumeration indices from 3^16/2 "
                                       f"of the cfg3 sweep per step ({cpu_model()})"},
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


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2111_10635_b200 import _abi
    from paper_2111_10635_b200.instance import DeviceInstance
    from paper_2111_10635_b200.search import (allgather_argmin, brute_force, enum_shard_async,
                                              merge_keys, shard_range, shard_strided)

    rank, world, local = dist_env()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "WARN"   # NCCL's banner goes to stdout: keep ONE JSON line
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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
    t = torch.tensor([my_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
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
    t = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = total * args.steps / (float(t.item()) * 1e-3)
    h2d = 4 * T * L * 8 + T * (8 + 8 + 1)  # profile tables + prices/quotas/is_cpu
    d2h = _abi.ARGMIN_NBYTES * world + 8 * 6  # gathered keys + the re-scored winner's outputs

    # ---- RL scheduler, cfg4 (BASELINE configs[3]): 200 rounds x 4096 plans, time-to-best ----
    rl = None
    if not args.no_rl and rank == 0:  # latency-bound per round: timed unsharded on one GPU
        from paper_2111_10635_b200 import load_fixture, policy
        from paper_2111_10635_b200.model import JobParams
        g4, c4, lim4 = load_fixture("cfg4")
        job4 = JobParams(lim4)
        cfg = policy.TrainerConfig(rounds=200, plans_per_round=4096, seed=0)
        p0, _ = policy.init_policy(g4, c4, cfg)
        policy.train(g4, c4, p0, policy.TrainerConfig(rounds=2, plans_per_round=4096, seed=0), job4,
                     shard=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = policy.train(g4, c4, p0, cfg, job4, shard=False)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        opt = 0.11630007595486111  # brute-force optimum of cfg4 (index 4030)
        hit = next((i for i, h in enumerate(res.history) if h.best_cost == opt), None)
        rl = {"workload": "cfg4", "rounds": 200, "plans_per_round": 4096, "gpus": 1, "wall_s": wall,
              "rounds_per_s": 200 / wall, "best_cost": res.best.cost,
              "best_plan": list(res.best.plan.assignment),
              "time_to_best_s": res.round_wall_s[hit] if hit is not None else None,
              "round_of_best": hit + 1 if hit is not None else None,
              "reference_cpu": {"wall_s": 404.3, "time_to_best_s": 15.3,
                                "source": "SURVEY.md §6 (reference, 1 core, measured in the build container)"}}

    # ---- cfg5 (BASELINE configs[4]): 64 layers x 4 types, random plans of default_rng(0) ----
    #   batch: hps_score_plans with every plan's outputs (cost, status, gap, ps, k) from a device
    #          batch of 2^20 plans;  sweep: plans generated in-kernel + fused argmin
    r5 = None
    if not args.no_cfg5:
        from paper_2111_10635_b200 import load_fixture
        from paper_2111_10635_b200.instance import pcg_from_generator
        from paper_2111_10635_b200.model import JobParams
        import numpy as np
        g5, c5, lim5 = load_fixture("cfg5")
        inst5 = DeviceInstance(g5, c5, JobParams(lim5))
        pcg = pcg_from_generator(np.random.default_rng(0))
        nb = 1 << 20
        plo, phi = shard_range(0, nb, rank, world)
        plans5 = inst5.random_plans(pcg, plo, phi - plo)
        inst5.score(plans5)   # warm-up at full size (scratch pools sized for 2^20-plan chunks)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out5 = inst5.score(plans5)
        e1.record()
        torch.cuda.synchronize()
        bms = e0.elapsed_time(e1)
        e0.record()
        key5 = inst5.read_argmin(inst5.random_argmin_async(pcg, plo, phi - plo))
        e1.record()
        torch.cuda.synchronize()
        sms = e0.elapsed_time(e1)
        t5 = torch.tensor([bms, sms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t5, op=dist.ReduceOp.MAX)
        feas = int(((out5["status"] & 0x7F) == 0).sum().item())
        r5 = {"workload": "cfg5", "layers": 64, "types": 4, "plans": nb,
              "batch_plans_per_s": nb / (float(t5[0]) * 1e-3),
              "sweep_plans_per_s": nb / (float(t5[1]) * 1e-3),
              "feasible_fraction": feas / (phi - plo),
              "note": "first 2^20 plans of default_rng(0).integers(0,4,64) per call (ls/baselines.py:270-271)"}

    if rank == 0:
        peak = fp64_peak(torch, inst.lib, dev)
        kernel_plans_per_s = my_plans / (statistics.median(step_ms) * 1e-3)
        achieved = kernel_plans_per_s * W_REF_OPS / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "plans_per_step": total, "layers": L, "types": T,
                       "throughput_limit": job.throughput_limit,
                       "parallelism": f"enumeration shards x{world}",
                       "l2": "flushed between steps (256 MiB write)",
                       "winner_index": key["rank"], "winner_cost": key["cost"],
                       "feasible_plans": key["feasible"]},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": gpu_launches,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": TRAFFIC_BYTES_PER_PLAN * my_plans,
                         "note": "achieved = plans/s of the sweep (stage + prep + candidate + slow "
                                 "kernels, one step) x reference-algorithm FP64 ops per plan "
                                 f"({W_REF_OPS}, SURVEY.md §8(d)); peak = DFMA probe measured in "
                                 "this run (MEASURED_PEAKS.json has no FP64); traffic = DRAM "
                                 f"bytes per step at {TRAFFIC_BYTES_PER_PLAN} B/plan from the ncu "
                                 "launch list (profiles/r1_launches_bench_v36_summary.txt): "
                                 "the split kernels' per-plan state round trips, ~1.4% of HBM "
                                 "bandwidth at this rate"},
            "clocks": clocks.summary(),
            "per_rank_ms": per_rank_ms,
        }
        if rl is not None:
            line["rl"] = rl
        if r5 is not None:
            line["cfg5_random"] = r5
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            sample = args.cpu_sample or 80_000 * threads
            rate, dt = cpu_oracle_rate(sample, threads)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                    "sample": f"{sample} consecutive cfg3 enumeration indices "
                                              f"from 3^16/2 in {dt:.1f} s ({cpu_model()})"}
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
