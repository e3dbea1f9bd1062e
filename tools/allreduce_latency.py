"""Latency of one small NCCL all-reduce over NVLink (the per-round exchange an
op-range-sharded multi-GPU TAC would need, SURVEY §8e option 1), against the
single-GPU TAC round times in DESIGN.md §3.3.

    torchrun --nproc-per-node 2 tools/allreduce_latency.py
"""
import json
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = {"world": world}
    for n in (2, 1024, 100_000):  # P/M+ vectors of R_t int64 entries
        x = torch.ones(n, dtype=torch.int64, device="cuda")
        for _ in range(50):
            dist.all_reduce(x)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 2000
        a.record()
        for _ in range(iters):
            dist.all_reduce(x)
        b.record()
        torch.cuda.synchronize()
        us = torch.tensor([a.elapsed_time(b) * 1000.0 / iters], device="cuda")
        dist.all_reduce(us, op=dist.ReduceOp.MAX)
        out[f"int64x{n}_us"] = round(us.item(), 2)
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
