"""The multi-GPU exchange logic (paper_1606_04669_b200/dist.py) on CPU: world_size 2, gloo.

Each rank owns one shard of one stream. Its subtree root (computed here with the oracle, as the
GPU kernels need a GPU) is all-gathered with dist.gather_summaries and the top level of the fixed
tree is finished from the gathered batch; verification counts are all-reduced with
dist.allreduce_counts. The result must be bit-identical to the single-process tree over all
leaves of the whole stream.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _summ_to_tensors(S, k):
    from paper_1606_04669_b200 import Summaries
    it = torch.zeros((1, k), dtype=torch.uint32)
    c = torch.zeros((1, k), dtype=torch.uint32)
    e = torch.zeros((1, k), dtype=torch.uint32)
    n = len(S)
    it[0, :n] = torch.from_numpy(S.items.astype(np.uint32))
    c[0, :n] = torch.from_numpy(S.counts.astype(np.uint32))
    e[0, :n] = torch.from_numpy(S.errs.astype(np.uint32))
    return Summaries(it, c, e, torch.tensor([n], dtype=torch.uint32))


def _worker(rank, world, port, n_total, k, P_per, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import inputs
        import oracle
        from paper_1606_04669_b200 import dist as pdist

        lo, hi = pdist.shard(n_total, world, rank)
        A = inputs.zipf(hi - lo, 1.1, 1e6, seed=21, start=lo)
        local_root = oracle.tree(oracle.leaves(A, k, P_per), k)
        gathered = pdist.gather_summaries(_summ_to_tensors(local_root, k))
        roots = []
        for g in range(world):
            ng = int(gathered.sizes[g])
            roots.append(oracle.Summary(gathered.items[g, :ng].numpy().astype(np.uint64),
                                        gathered.counts[g, :ng].numpy().astype(np.uint64),
                                        gathered.errs[g, :ng].numpy().astype(np.uint64)))
        top = oracle.tree(roots, k)
        cand = oracle.prune(top, n_total, k)
        exact = torch.from_numpy(oracle.verify(A, cand).astype(np.uint64))
        pdist.allreduce_counts(exact)
        out_q.put((rank, top.as_tuples(), cand.tolist(), exact.numpy().tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,P_per", [(2, 4), (4, 2), (8, 1), (8, 2)])
def test_sharded_tree_is_bit_identical(world, P_per):
    from conftest import build_lib
    build_lib()
    import inputs
    import oracle

    n_total, k = 80_000, 50
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, k, P_per, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = inputs.zipf(n_total, 1.1, 1e6, seed=21)
    ref = oracle.pipeline(A, k, world * P_per)
    for rank, top, cand, exact in res:
        assert top == ref.root.as_tuples(), rank
        assert cand == ref.cand.tolist()
        assert exact == ref.exact.tolist()


def test_shard_bounds():
    from conftest import build_lib
    build_lib()
    from paper_1606_04669_b200 import dist as pdist
    assert [pdist.shard(12, 3, r) for r in range(3)] == [(0, 4), (4, 8), (8, 12)]
    with pytest.raises(ValueError):
        pdist.shard(10, 3, 0)
