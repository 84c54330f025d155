"""Per-rank phase timing of the public brute_force path (bench.py's e2e step) under torchrun:
instance staging, the sharded sweep + all_gather, and the winner re-score. Not a bench."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    from paper_2111_10635_b200 import load_fixture
    from paper_2111_10635_b200.model import JobParams, ProvisionerConfig, SchedulingPlan
    import paper_2111_10635_b200.scoring as scoring
    from paper_2111_10635_b200.search import enumerate_argmin, decode_index
    g, c, limit = load_fixture("cfg3")
    job = JobParams(limit)
    total = 3 ** 16
    for step in range(4):
        scoring._INSTANCES.clear()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        inst = scoring.device_instance(g, c, job, ProvisionerConfig())
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        key = enumerate_argmin(g, c, job, 0, total, True, ProvisionerConfig())
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        best = scoring.PlanScorer(g, c, job, ProvisionerConfig())(SchedulingPlan(decode_index(key["rank"], 3, 16)))
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"rank {rank} step {step}: stage {1e3*(t1-t0):.1f} ms, sweep+gather {1e3*(t2-t1):.1f} ms, "
              f"rescore {1e3*(t3-t2):.1f} ms", flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
