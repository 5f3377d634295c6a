"""Runner for one pass of the hot path, on one GPU or sharded over several (one process per GPU).

Single GPU: pss_summarize -> pss_merge -> pss_prune -> pss_verify -> pss_report, all C-ABI calls
on the current stream.

Several GPUs (the paper's hybrid MPI/OpenMP structure):
rank g owns the contiguous shard [g*n, (g+1)*n) of one stream of world*n keys and the blocks
[g*P, (g+1)*P) of the global decomposition into world*P blocks. With equal shards those are
exactly the rank-local blocks (floor(r*n/P) offsets), and with world and P powers of two they
form one complete subtree of the fixed binary tree (R6). Each rank reduces its subtree to a root;
ONE all-gather moves the world roots (k counters each) over NVLink, and every rank finishes the
top log2(world) levels of the same tree in the same order, so the global root is bit-identical to
the single-GPU one. Those top levels run on wide summaries (64-bit counts, pss_merge_wide): each
rank's shard holds at most 2^31 keys, but world shards together may exceed 2^31 (weak scaling of
the 2^29-key workload to 8 GPUs is 2^32 keys), beyond reading R9's u32 bound. Verification counts
the local shard and ONE all-reduce(sum) adds the exact (uint64) counts. The collectives are
torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import math

import os

import torch

from . import (KEY_U32, OP_MERGE_WIDE, OP_SUMMARIZE_MERGE, OP_VERIFY, Summaries, _key_dtype,
               pss_merge_wide, pss_prune, pss_prune_wide, pss_query_host, pss_report,
               pss_summarize_merge, pss_verify, pss_widen, pss_workspace_bytes)


def shard(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Positions of rank's shard; shards must be equal so block boundaries line up."""
    if n_total % world:
        raise ValueError("the stream length must be a multiple of the number of ranks")
    m = n_total // world
    return rank * m, (rank + 1) * m


def _as_signed(t: torch.Tensor) -> torch.Tensor:
    """Bit-preserving view with a dtype every backend can move (gloo/NCCL lack uint32)."""
    m = {torch.uint32: torch.int32, torch.uint64: torch.int64}
    return t.view(m[t.dtype]) if t.dtype in m else t


def gather_summaries(root: Summaries, group=None) -> Summaries:
    """All-gather one summary per rank into a batch ordered by rank (the next tree level)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = Summaries(torch.empty((world, root.k), dtype=root.items.dtype, device=root.items.device),
                    torch.empty((world, root.k), dtype=root.counts.dtype, device=root.items.device),
                    torch.empty((world, root.k), dtype=root.errs.dtype, device=root.items.device),
                    torch.empty((world,), dtype=root.sizes.dtype, device=root.items.device))
    host = _host_staged(root.items, group)
    for src, dst in ((root.items, out.items), (root.counts, out.counts), (root.errs, out.errs),
                     (root.sizes, out.sizes)):
        d = dst.cpu() if host else dst
        parts = list(_as_signed(d).reshape(world, -1).unbind(0))
        dist.all_gather(parts, _as_signed(src.cpu() if host else src).reshape(-1), group=group)
        if host:
            dst.copy_(d)
    return out


def _host_staged(t: torch.Tensor, group) -> bool:
    """gloo moves host tensors only: device tensors are staged through host memory (tests)."""
    import torch.distributed as dist

    return t.is_cuda and dist.get_backend(group) == "gloo"


def allreduce_counts(exact: torch.Tensor, group=None) -> torch.Tensor:
    import torch.distributed as dist

    if _host_staged(exact, group):
        h = exact.cpu()
        dist.all_reduce(_as_signed(h), op=dist.ReduceOp.SUM, group=group)
        exact.copy_(h)
        return exact
    dist.all_reduce(_as_signed(exact), op=dist.ReduceOp.SUM, group=group)
    return exact


def _merge_launches(P: int, k: int, kb: int) -> int:
    """Kernels pss_merge launches (csrc/merge.cu): the root COMBINE, plus one persistent launch
    for all internal levels when a COMBINE's working set fits shared memory (else one per level)."""
    if P <= 2:
        return 1
    levels, c = 0, P
    while (c + 1) // 2 > 1:
        c = (c + 1) // 2
        levels += 1
    NP = max(256, 1 << (2 * k - 1).bit_length())
    work = 2 * k * (kb + 8) + k + 4 * (1 << (2 * k - 1).bit_length()) + NP * (8 + kb)
    return 1 + (1 if work <= 227 * 1024 - 2048 else levels)


class Runner:
    """Preallocated buffers + one step of the path (see module docstring)."""

    def __init__(self, n: int, k: int, P: int, key_type: int, device, world: int = 1,
                 rank: int = 0, group=None):
        if world > 1 and (world & (world - 1) or P & (P - 1)):
            raise ValueError("sharded runs need power-of-two ranks and blocks per rank")
        self.n, self.k, self.P, self.kt = n, k, P, key_type
        self.world, self.rank, self.group = world, rank, group
        self.dev = torch.device(device)
        kb = 4 if key_type == KEY_U32 else 8
        if n > (1 << 31):
            raise ValueError("a rank's shard holds at most 2^31 keys (u32 leaf counters, R9)")
        self.leaves = Summaries.empty(P, k, key_type, self.dev)
        self.root = Summaries.empty(1, k, key_type, self.dev)
        if world > 1:  # the top levels over the ranks' roots: 64-bit counts (wide summaries)
            self.gathered_w = Summaries.empty(world, k, key_type, self.dev, wide=True)
            self.top = Summaries.empty(1, k, key_type, self.dev, wide=True)
        else:
            self.top = self.root
        ws = max(pss_workspace_bytes(OP_SUMMARIZE_MERGE, n, k, P, key_type),
                 pss_workspace_bytes(OP_MERGE_WIDE, 0, k, world, key_type),
                 pss_workspace_bytes(OP_VERIFY, n, k, 1, key_type))
        self.ws = torch.empty((ws,), dtype=torch.uint8, device=self.dev)
        self.exact = torch.zeros((k,), dtype=torch.uint64, device=self.dev)
        self.cand = (torch.empty((k,), dtype=_key_dtype(key_type), device=self.dev),
                     torch.empty((1,), dtype=torch.uint32, device=self.dev))
        kd = _key_dtype(key_type)
        self.out = (torch.empty((k,), dtype=kd, device=self.dev),
                    torch.empty((k,), dtype=torch.uint64, device=self.dev),
                    torch.zeros((1,), dtype=torch.uint32, device=self.dev))
        self.host_out = tuple(torch.empty_like(t, device="cpu").pin_memory() for t in self.out)
        # K1 (+ the histogram kernel when 40 k >= block length), the tree, [widen + one wide
        # COMBINE launch per top level], prune, verify (setup, the scan for <= 75 candidates and,
        # when k allows more, the general scan, finalize), report
        top_levels = (world - 1).bit_length() if world > 1 else 0
        hist = 1 if 40 * k >= -(-n // P) and -(-n // P) <= (1 << 17) else 0
        # the frequent-key sample K0 and the bypass kernel K1b in front of K1 (csrc/summarize.cu,
        # ss_plan: u32 keys, packed counters, blocks of 2^13..2^16 keys, 128 <= k <= 4094)
        lmax = -(-n // P)
        cb = max(1, lmax.bit_length())
        packed = cb < 30 and lmax // k < (1 << (30 - cb))
        bypass = 2 if (kb == 4 and packed and 8192 <= lmax <= 65536 and 128 <= k <= 4094 and
                       os.environ.get("PSS_BYPASS", "1") != "0") else 0
        verify = 4  # setup, the tagged scan, the general scan (one of the two returns), finalize
        self.launches_per_step = (1 + hist + bypass + _merge_launches(P, k, kb) +
                                  (1 + top_levels if world > 1 else 0) + 1 + verify + 1)
        self.host_api = "pss_query_host" if world == 1 else "H2D copy + step + D2H (torch)"
        self._kb = kb

    def step(self, A: torch.Tensor, ev=None):
        s = torch.cuda.current_stream()
        if ev is not None:
            ev[0].record(s)
        # leaves and this rank's subtree root; the tree kernel overlaps the leaf kernel's last wave
        pss_summarize_merge(A, self.k, self.P, leaves=self.leaves, root=self.root,
                            workspace=self.ws)
        if ev is not None:
            ev[1].record(s)
        n_global = self.n * self.world
        if self.world > 1:
            gathered = gather_summaries(self.root, self.group)
            pss_widen(gathered, out=self.gathered_w)
            pss_merge_wide(self.gathered_w, out=self.top, workspace=self.ws)
        if ev is not None:
            ev[2].record(s)
        if self.world > 1:
            cand, n_cand = pss_prune_wide(self.top, n_global, out=self.cand)
        else:
            cand, n_cand = pss_prune(self.top, n_global, out=self.cand)
        exact = pss_verify(A, cand, n_cand, out=self.exact, workspace=self.ws)
        if self.world > 1:
            allreduce_counts(self.exact, self.group)
        pss_report(cand, exact, n_global, self.k, n_cand=n_cand, out=self.out)
        if ev is not None:
            ev[3].record(s)
        return self.out

    def result(self):
        return self.out

    def step_host(self, h_A: torch.Tensor, d_A: torch.Tensor):
        """End to end from pinned host keys: H2D, the whole path, D2H of the answer."""
        if self.world == 1:
            return pss_query_host(h_A, self.k, self.P, d_A=d_A, workspace=None, out=self.host_out,
                                  sync=False)
        d_A.copy_(h_A, non_blocking=True)
        self.step(d_A)
        for h, d in zip(self.host_out, self.out):
            h.copy_(d, non_blocking=True)
        return self.host_out
