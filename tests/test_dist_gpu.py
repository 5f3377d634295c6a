"""The sharded path of dist.Runner on a real GPU: two ranks (gloo, both on cuda:0 -- a functional
check of the exchange, their kernels never wait on each other) must give the same answer as one
rank over the whole stream, and the same as the oracle's k-majority set."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_local, k, P, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import inputs
        import paper_1606_04669_b200 as pss
        from paper_1606_04669_b200 import dist as pdist
        A = inputs.zipf(n_local, 1.1, 1e6, seed=33, start=rank * n_local)
        r = pdist.Runner(n_local, k, P, pss.KEY_U32, "cuda:0", world=world, rank=rank,
                         group=dist.group.WORLD)
        items, counts, ln = r.step(torch.from_numpy(A).cuda())
        torch.cuda.synchronize()
        m = int(ln.item())
        q.put((rank, items[:m].cpu().numpy().tolist(), counts[:m].cpu().numpy().tolist(),
               r.top.host(0)))
    finally:
        dist.destroy_process_group()


def test_two_ranks_match_one(pss_lib=None):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from conftest import build_lib
    build_lib()
    import torch.multiprocessing as mp

    import inputs
    import oracle
    import paper_1606_04669_b200 as pss
    from paper_1606_04669_b200 import dist as pdist

    world, n_local, k, P = 2, 1 << 20, 200, 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_local, k, P, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1:] == res[1][1:]
    A = inputs.zipf(world * n_local, 1.1, 1e6, seed=33)
    one = pdist.Runner(world * n_local, k, world * P, pss.KEY_U32, "cuda:0")
    items, counts, ln = one.step(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    m = int(ln.item())
    assert res[0][1] == items[:m].cpu().numpy().tolist()
    assert res[0][2] == counts[:m].cpu().numpy().tolist()
    ref = oracle.pipeline(A, k, world * P, threads=8)
    assert res[0][1] == ref.result[0].tolist() and res[0][2] == ref.result[1].tolist()
    # the gathered top of the tree (wide summaries) on every rank is the oracle's root
    for r in res:
        assert r[3] == ref.root.as_tuples()
