"""Host-side logic of the multi-process path on CPU (gloo, world_size 2): the NCCL-unique-id
bootstrap, max-over-ranks timing and barriers used by bench.py / the dist runtime, plus the mesh
rank/coordinate/group convention (row-major, axis 0 slowest: proj/src/planner.cpp:58-63)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2302_08141_b200.abi import rank_coords


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    from paper_2302_08141_b200 import dist as D
    uid = D.exchange_uid(lambda: bytes(range(128)))
    m = D.max_over_ranks(1.5 + rank)
    D.barrier()
    q.put((rank, uid == bytes(range(128)), m, D.env()))
    D.init_process_group().destroy_process_group()


def test_gloo_bootstrap_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, uid_ok, m, env in res:
        assert uid_ok, "every rank must receive rank 0's NCCL unique id"
        assert m == 2.5, "timings are reported as the max over ranks"
        assert env == (world, rank, rank)


@pytest.mark.parametrize("mesh", [[4], [2, 2], [2, 4], [8]])
def test_rank_coordinates(mesh):
    world = 1
    for d in mesh:
        world *= d
    seen = set()
    for r in range(world):
        c = rank_coords(r, mesh)
        flat = 0
        for a, d in enumerate(mesh):
            assert 0 <= c[a] < d
            flat = flat * d + c[a]
        assert flat == r
        seen.add(tuple(c))
    assert len(seen) == world
    if len(mesh) == 2:  # machines x gpus: consecutive ranks share a machine (axis 0 slowest)
        assert rank_coords(1, mesh) == [0, 1]
