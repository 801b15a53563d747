"""Multi-process plumbing of the sharded sweep / bench on CPU (gloo, world_size 2).

The GPU path shards independent shapes over one process per GPU with no
collective on the data path; here two gloo ranks check that the LPT shards
are disjoint and complete, that timing agreement is a max over ranks, and
that the CLI's worker-process tune sharding assigns every shape once.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1806_07060_b200 import distributed, sharding
    from paper_1806_07060_b200.dataset import gen_po2

    r, w, _ = distributed.init(backend="gloo")
    shapes = [s.mnk for s in gen_po2(64, 4096)]
    mine = distributed.shard(shapes, r, w, lambda t: sharding.sweep_cost(t, 778))
    everyone = distributed.gather_objects(mine)
    # per-rank "timings": the agreed value must be the max over ranks
    agreed = distributed.reduce_max([float(r + 1), 10.0 - r])
    distributed.barrier()
    q.put((r, everyone, agreed, len(mine)))
    distributed.finalize()


def test_gloo_world2_sharding_and_max_reduce():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1806_07060_b200.dataset import gen_po2
    shapes = [s.mnk for s in gen_po2(64, 4096)]
    for r, everyone, agreed, n in results:
        flat = [tuple(x) for part in everyone for x in part]
        assert sorted(flat) == sorted(shapes) and len(set(flat)) == len(shapes)
        assert agreed == [2.0, 10.0]
    assert results[0][1] == results[1][1]


def test_cli_worker_binding_round_robins_gpus(monkeypatch):
    from multiprocessing import get_context

    from paper_1806_07060_b200 import cli
    monkeypatch.setenv("CUDA_VISIBLE_DEVICES", "")  # restored at teardown
    slots = get_context("spawn").Value("i", 0)
    seen = []
    for _ in range(5):
        cli._bind_gpu(slots, ["3", "5"])
        seen.append(os.environ["CUDA_VISIBLE_DEVICES"])
    assert seen == ["3", "5", "3", "5", "3"]
    monkeypatch.setenv("CUDA_VISIBLE_DEVICES", "0,1,2")
    assert cli._visible_gpus() == ["0", "1", "2"]
