"""One process per GPU: rank/world plumbing for sharded sweeps and the bench.

No collective ever touches the GEMM data path -- shapes are independent.
torch.distributed (NCCL on GPUs, gloo on CPU) is used only to agree on
timings (max over ranks) and to gather per-shape results for reporting.
"""

import os


def env_rank_world():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", os.environ.get("RANK", "0"))))


def init(backend: str | None = None):
    """Initialise the default group when launched under torchrun; returns (rank, world, local_rank)."""
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank_world()
    ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # AG_DIST_BACKEND=gloo lets several ranks share one GPU (a functional
        # check of the N > 1 path on a 1-GPU box; NCCL refuses duplicate GPUs)
        backend = backend or os.environ.get("AG_DIST_BACKEND") or ("nccl" if ndev else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
        elif ndev:
            torch.cuda.set_device(local % ndev)
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    elif ndev:
        torch.cuda.set_device(local % ndev)
    return rank, world, local


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def reduce_max(values: list, device=None) -> list:
    """Element-wise max over ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return list(values)
    if dist.get_backend() != "nccl":
        device = None  # gloo reduces host tensors
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def gather_objects(obj) -> list:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def shard(items: list, rank: int, world: int, cost) -> list:
    """This rank's LPT share of independent work items."""
    from .sharding import lpt_partition
    return lpt_partition(items, world, cost)[rank]


def finalize():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
