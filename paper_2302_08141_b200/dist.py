"""Multi-process plumbing: one process per GPU launched by torchrun.

torch.distributed (gloo, CPU tensors) carries only the bootstrap — the NCCL unique id for the
executor's own communicators — and the max-over-ranks reduction of timings.  All device work and
all resharding traffic go through librhino_exec.so.
"""
import os


def env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def init_process_group():
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("gloo")
    return dist


def exchange_uid(make_uid):
    """Rank 0 creates the id (`make_uid()`), every rank returns it."""
    dist = init_process_group()
    obj = [make_uid() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(x):
    import torch
    world, _, _ = env()
    if world == 1:
        return float(x)
    dist = init_process_group()
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    world, _, _ = env()
    if world > 1:
        init_process_group().barrier()


def make_runtime():
    """Runtime for this process: all-local on cuda:0 when not under torchrun, else one rank of
    the torchrun world on cuda:LOCAL_RANK."""
    from . import runtime
    world, rank, local = env()
    if world == 1:
        return runtime.Runtime(devices=[0])
    uid = exchange_uid(runtime.unique_id)
    return runtime.Runtime(dist=(world, rank, local, uid))
