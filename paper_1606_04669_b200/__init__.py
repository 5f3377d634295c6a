"""pss-b200: the data-parallel hot path of Parallel Space Saving (arXiv 1606.04669) on one B200.

A thin Python binding over the C-ABI library ``libpss.so`` (include/pss.h). Every function here
only marshals arguments: tensors are passed as device pointers, the current torch stream as the
CUDA stream, and every step of the method runs in the CUDA kernels of ``csrc/``. There is no CPU
fallback: importing this package fails loudly if ``libpss.so`` has not been built
(``python -c "import __graft_entry__ as g; g.build()"``).

Names mirror the C functions: pss_summarize, pss_merge, pss_combine, pss_prune, pss_verify,
pss_query, pss_query_host, pss_workspace_bytes.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

__all__ = ["Summaries", "PssError", "pss_workspace_bytes", "pss_summarize", "pss_summarize_merge",
           "OP_SUMMARIZE_MERGE", "pss_merge", "pss_combine", "pss_prune", "pss_verify",
           "pss_report", "pss_query", "pss_query_host", "lib_path",
           "KEY_U32", "KEY_U64", "OP_SUMMARIZE", "OP_MERGE", "OP_COMBINE", "OP_VERIFY", "OP_QUERY",
           "EXPORTED_SYMBOLS"]

_PKG = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("PSS_LIB") or os.path.join(_PKG, "libpss.so")  # PSS_LIB: dev builds

KEY_U32, KEY_U64 = 0, 1
OP_SUMMARIZE, OP_MERGE, OP_COMBINE, OP_VERIFY, OP_QUERY = range(5)
OP_SUMMARIZE_MERGE = 6
OP_COMBINE_WIDE, OP_MERGE_WIDE = 7, 8
STATUS = {0: "PSS_OK", 1: "PSS_ERR_INVALID_ARG", 2: "PSS_ERR_UNSUPPORTED",
          3: "PSS_ERR_CAPACITY_MISMATCH", 4: "PSS_ERR_WORKSPACE_TOO_SMALL", 5: "PSS_ERR_CUDA"}
EXPORTED_SYMBOLS = ["pss_workspace_bytes", "pss_summarize", "pss_summarize_merge", "pss_merge",
                    "pss_combine",
                    "pss_prune", "pss_verify", "pss_report", "pss_query", "pss_query_host",
                    "pss_widen", "pss_combine_wide", "pss_merge_wide", "pss_prune_wide",
                    "pss_status_string", "pss_version"]


class PssError(RuntimeError):
    def __init__(self, fn: str, status: int):
        super().__init__(f"{fn} returned {STATUS.get(status, status)}")
        self.status = status


class _Summ(ctypes.Structure):
    _fields_ = [("key_type", ctypes.c_int32), ("k", ctypes.c_uint32), ("count", ctypes.c_uint32),
                ("items", ctypes.c_void_p), ("counts", ctypes.c_void_p), ("errs", ctypes.c_void_p),
                ("sizes", ctypes.c_void_p)]


if not os.path.exists(lib_path):
    raise ImportError(f"{lib_path} is missing: build it first (__graft_entry__.build()); "
                      "there is no CPU fallback")
_lib = ctypes.CDLL(lib_path)
_vp, _u64, _u32, _i32, _sz = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                              ctypes.c_size_t)
_SP = ctypes.POINTER(_Summ)
_lib.pss_workspace_bytes.argtypes = [_i32, _u64, _u32, _u32, _i32]
_lib.pss_workspace_bytes.restype = _sz
_lib.pss_summarize.argtypes = [_vp, _u64, _i32, _u32, _u32, _SP, _vp, _sz, _vp]
_lib.pss_merge.argtypes = [_SP, _SP, _vp, _sz, _vp]
_lib.pss_summarize_merge.argtypes = [_vp, _u64, _i32, _u32, _u32, _SP, _SP, _vp, _sz, _vp]
_lib.pss_combine.argtypes = [_SP, _SP, _SP, _vp, _sz, _vp]
_lib.pss_prune.argtypes = [_SP, _u64, _vp, _vp, _vp]
_lib.pss_verify.argtypes = [_vp, _u64, _i32, _vp, _u32, _vp, _vp, _vp, _sz, _vp]
_lib.pss_report.argtypes = [_vp, _u32, _vp, _vp, _i32, _u64, _u32, _vp, _vp, _vp, _vp]
_lib.pss_query.argtypes = [_vp, _u64, _i32, _u32, _u32, _vp, _vp, _vp, _vp, _sz, _vp]
_lib.pss_query_host.argtypes = [_vp, _vp, _u64, _i32, _u32, _u32, _vp, _vp, _vp, _vp, _sz, _vp]
# wide summaries (include/pss.h pss_wsummaries) share pss_summaries' layout: 64-bit counts/errs
_lib.pss_widen.argtypes = [_SP, _SP, _vp]
_lib.pss_combine_wide.argtypes = [_SP, _SP, _SP, _vp, _sz, _vp]
_lib.pss_merge_wide.argtypes = [_SP, _SP, _vp, _sz, _vp]
_lib.pss_prune_wide.argtypes = [_SP, _u64, _vp, _vp, _vp]
for _f in ("pss_summarize", "pss_summarize_merge", "pss_merge", "pss_combine", "pss_prune",
           "pss_verify", "pss_report", "pss_query", "pss_query_host", "pss_widen",
           "pss_combine_wide", "pss_merge_wide", "pss_prune_wide"):
    getattr(_lib, _f).restype = _i32
_lib.pss_status_string.argtypes = [_i32]
_lib.pss_status_string.restype = ctypes.c_char_p
_lib.pss_version.restype = ctypes.c_char_p


def version() -> str:
    return _lib.pss_version().decode()


def _check(fn: str, st: int):
    if st != 0:
        raise PssError(fn, st)


def _key_type(t: torch.Tensor) -> int:
    if t.dtype in (torch.uint32, torch.int32):
        return KEY_U32
    if t.dtype in (torch.uint64, torch.int64):
        return KEY_U64
    raise TypeError(f"keys must be uint32/uint64 (or int32/int64 bit patterns), got {t.dtype}")


def _key_dtype(kt: int):
    return torch.uint32 if kt == KEY_U32 else torch.uint64


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev_keys(A: torch.Tensor) -> torch.Tensor:
    if not A.is_cuda:
        raise ValueError("A must be a CUDA tensor (use pss_query_host for host buffers)")
    if not A.is_contiguous():
        raise ValueError("A must be contiguous")
    return A


def _ws(nbytes: int, ws: torch.Tensor | None, device, stream=None) -> torch.Tensor:
    """The caller's workspace if large enough, else a temporary. A temporary is marked as in use
    on `stream` (record_stream): the call only enqueues work, so without it the caching
    allocator could hand the block to a new allocation while the kernels still use it."""
    if ws is not None and ws.numel() * ws.element_size() >= nbytes:
        return ws.view(torch.uint8) if ws.dtype != torch.uint8 else ws
    t = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
    if stream is not None:
        t.record_stream(stream)
    return t


def pss_workspace_bytes(op: int, n: int, k: int, P: int, key_type: int) -> int:
    return int(_lib.pss_workspace_bytes(op, n, k, P, key_type))


@dataclass
class Summaries:
    """`count` summaries of capacity k (device tensors, structure of arrays; include/pss.h)."""
    items: torch.Tensor   # [count, k] uint32|uint64
    counts: torch.Tensor  # [count, k] uint32
    errs: torch.Tensor    # [count, k] uint32
    sizes: torch.Tensor   # [count] uint32

    @staticmethod
    def empty(count: int, k: int, key_type: int, device="cuda", wide: bool = False) -> "Summaries":
        """wide: 64-bit counts and errors (pss_wsummaries, the tree above the leaves)."""
        ct = torch.uint64 if wide else torch.uint32
        return Summaries(torch.empty((count, k), dtype=_key_dtype(key_type), device=device),
                         torch.empty((count, k), dtype=ct, device=device),
                         torch.empty((count, k), dtype=ct, device=device),
                         torch.zeros((count,), dtype=torch.uint32, device=device))

    @property
    def wide(self) -> bool:
        return self.counts.dtype == torch.uint64

    @property
    def k(self) -> int:
        return int(self.items.shape[1])

    @property
    def count(self) -> int:
        return int(self.items.shape[0])

    @property
    def key_type(self) -> int:
        return _key_type(self.items)

    def _c(self) -> _Summ:
        return _Summ(self.key_type, self.k, self.count, self.items.data_ptr(),
                     self.counts.data_ptr(), self.errs.data_ptr(), self.sizes.data_ptr())

    def host(self, i: int = 0):
        """Summary i as host lists [(item, count, err)] (items as unsigned ints)."""
        n = int(self.sizes[i].item())
        it = self.items[i, :n].cpu().numpy().astype("uint64").tolist()
        c = self.counts[i, :n].cpu().numpy().astype("uint64").tolist()
        e = self.errs[i, :n].cpu().numpy().astype("uint64").tolist()
        return list(zip(it, c, e))


def pss_summarize(A: torch.Tensor, k: int, P: int, out: Summaries | None = None,
                  workspace: torch.Tensor | None = None, stream=None) -> Summaries:
    """Per-block Space Saving leaves (Alg. 1 l.3-5): see include/pss.h."""
    A = _dev_keys(A)
    kt = _key_type(A)
    out = out or Summaries.empty(P, k, kt, A.device)
    ws = _ws(pss_workspace_bytes(OP_SUMMARIZE, A.numel(), k, P, kt), workspace, A.device, stream)
    c = out._c()
    _check("pss_summarize", _lib.pss_summarize(A.data_ptr(), A.numel(), kt, k, P, ctypes.byref(c),
                                               ws.data_ptr(), ws.numel(), _stream(stream)))
    return out


def pss_summarize_merge(A: torch.Tensor, k: int, P: int, leaves: Summaries | None = None,
                        root: Summaries | None = None, workspace: torch.Tensor | None = None,
                        stream=None) -> tuple[Summaries, Summaries]:
    """pss_summarize + pss_merge in one call, the tree overlapping the leaves (include/pss.h)."""
    A = _dev_keys(A)
    kt = _key_type(A)
    leaves = leaves or Summaries.empty(P, k, kt, A.device)
    root = root or Summaries.empty(1, k, kt, A.device)
    ws = _ws(pss_workspace_bytes(OP_SUMMARIZE_MERGE, A.numel(), k, P, kt), workspace, A.device, stream)
    a, b = leaves._c(), root._c()
    _check("pss_summarize_merge", _lib.pss_summarize_merge(
        A.data_ptr(), A.numel(), kt, k, P, ctypes.byref(a), ctypes.byref(b), ws.data_ptr(),
        ws.numel(), _stream(stream)))
    return leaves, root


def pss_merge(leaves: Summaries, out: Summaries | None = None,
              workspace: torch.Tensor | None = None, stream=None) -> Summaries:
    """Fixed binary COMBINE tree over the leaves (Alg. 1 l.7, Alg. 2) -> root (canonical)."""
    out = out or Summaries.empty(1, leaves.k, leaves.key_type, leaves.items.device)
    ws = _ws(pss_workspace_bytes(OP_MERGE, 0, leaves.k, leaves.count, leaves.key_type), workspace,
             leaves.items.device, stream)
    a, b = leaves._c(), out._c()
    _check("pss_merge", _lib.pss_merge(ctypes.byref(a), ctypes.byref(b), ws.data_ptr(), ws.numel(),
                                       _stream(stream)))
    return out


def pss_combine(a: Summaries, b: Summaries, out: Summaries | None = None,
                workspace: torch.Tensor | None = None, stream=None) -> Summaries:
    """out[i] = COMBINE(a[i], b[i]) (Alg. 2), canonical order."""
    out = out or Summaries.empty(a.count, a.k, a.key_type, a.items.device)
    ws = _ws(pss_workspace_bytes(OP_COMBINE, 0, a.k, a.count, a.key_type), workspace, a.items.device, stream)
    ca, cb, co = a._c(), b._c(), out._c()
    _check("pss_combine", _lib.pss_combine(ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co),
                                           ws.data_ptr(), ws.numel(), _stream(stream)))
    return out


def _need(S: Summaries, wide: bool, fn: str):
    if S.wide != wide:
        raise TypeError(f"{fn}: {'wide' if wide else 'narrow'} summaries expected")


def pss_widen(S: Summaries, out: Summaries | None = None, stream=None) -> Summaries:
    """The same summaries with 64-bit counts and errors (include/pss.h pss_widen)."""
    _need(S, False, "pss_widen")
    out = out or Summaries.empty(S.count, S.k, S.key_type, S.items.device, wide=True)
    a, b = S._c(), out._c()
    _check("pss_widen", _lib.pss_widen(ctypes.byref(a), ctypes.byref(b), _stream(stream)))
    return out


def pss_combine_wide(a: Summaries, b: Summaries, out: Summaries | None = None,
                     workspace: torch.Tensor | None = None, stream=None) -> Summaries:
    """out[i] = COMBINE(a[i], b[i]) (Alg. 2) with 64-bit counts, canonical order."""
    _need(a, True, "pss_combine_wide")
    out = out or Summaries.empty(a.count, a.k, a.key_type, a.items.device, wide=True)
    ws = _ws(pss_workspace_bytes(OP_COMBINE_WIDE, 0, a.k, a.count, a.key_type), workspace,
             a.items.device, stream)
    ca, cb, co = a._c(), b._c(), out._c()
    _check("pss_combine_wide", _lib.pss_combine_wide(ctypes.byref(ca), ctypes.byref(cb),
                                                     ctypes.byref(co), ws.data_ptr(), ws.numel(),
                                                     _stream(stream)))
    return out


def pss_merge_wide(nodes: Summaries, out: Summaries | None = None,
                   workspace: torch.Tensor | None = None, stream=None) -> Summaries:
    """The fixed binary tree (R6) over wide summaries -> wide root (canonical)."""
    _need(nodes, True, "pss_merge_wide")
    out = out or Summaries.empty(1, nodes.k, nodes.key_type, nodes.items.device, wide=True)
    ws = _ws(pss_workspace_bytes(OP_MERGE_WIDE, 0, nodes.k, nodes.count, nodes.key_type),
             workspace, nodes.items.device, stream)
    a, b = nodes._c(), out._c()
    _check("pss_merge_wide", _lib.pss_merge_wide(ctypes.byref(a), ctypes.byref(b), ws.data_ptr(),
                                                 ws.numel(), _stream(stream)))
    return out


def pss_prune_wide(root: Summaries, n: int, stream=None, out=None):
    """pss_prune on a wide root (any n < 2^63)."""
    _need(root, True, "pss_prune_wide")
    if out is not None:
        cand, n_cand = out
    else:
        cand = torch.empty((root.k,), dtype=root.items.dtype, device=root.items.device)
        n_cand = torch.empty((1,), dtype=torch.uint32, device=root.items.device)
    c = root._c()
    _check("pss_prune_wide", _lib.pss_prune_wide(ctypes.byref(c), n, cand.data_ptr(),
                                                 n_cand.data_ptr(), _stream(stream)))
    return cand, n_cand


def pss_prune(root: Summaries, n: int, stream=None, out=None):
    """Pruned(global, n, k) (Alg. 1 l.8-9): (candidates[k] device keys, n_cand[1] device uint32).
    `out` = preallocated (cand, n_cand); the kernel writes n_cand, so neither needs clearing."""
    if out is not None:
        cand, n_cand = out
    else:
        cand = torch.empty((root.k,), dtype=root.items.dtype, device=root.items.device)
        n_cand = torch.empty((1,), dtype=torch.uint32, device=root.items.device)
    c = root._c()
    _check("pss_prune", _lib.pss_prune(ctypes.byref(c), n, cand.data_ptr(), n_cand.data_ptr(),
                                       _stream(stream)))
    return cand, n_cand


def pss_verify(A: torch.Tensor, cand: torch.Tensor, n_cand: torch.Tensor | None = None,
               out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
    """Exact counts of the candidates over A. Returns uint64[len(cand)] on the device."""
    A = _dev_keys(A)
    kt = _key_type(A)
    if _key_type(cand) != kt:
        raise TypeError("candidate and key types differ")
    cap = cand.numel()
    out = out if out is not None else torch.zeros((max(cap, 1),), dtype=torch.uint64, device=A.device)
    ws = _ws(pss_workspace_bytes(OP_VERIFY, A.numel(), cap, 1, kt), workspace, A.device, stream)
    _check("pss_verify", _lib.pss_verify(A.data_ptr(), A.numel(), kt, cand.data_ptr(), cap,
                                         n_cand.data_ptr() if n_cand is not None else None,
                                         out.data_ptr(), ws.data_ptr(), ws.numel(),
                                         _stream(stream)))
    return out[:cap]


def pss_report(cand: torch.Tensor, exact: torch.Tensor, n: int, k: int,
               n_cand: torch.Tensor | None = None, out=None, stream=None):
    """The verified k-majority answer: (items, counts uint64, length[1]) on the device."""
    kt = _key_type(cand)
    cap = cand.numel()
    if out is None:
        out = (torch.empty((max(cap, 1),), dtype=cand.dtype, device=cand.device),
               torch.empty((max(cap, 1),), dtype=torch.uint64, device=cand.device),
               torch.zeros((1,), dtype=torch.uint32, device=cand.device))
    oi, oc, ol = out
    _check("pss_report", _lib.pss_report(cand.data_ptr(), cap,
                                         n_cand.data_ptr() if n_cand is not None else None,
                                         exact.data_ptr(), kt, n, k, oi.data_ptr(), oc.data_ptr(),
                                         ol.data_ptr(), _stream(stream)))
    return oi, oc, ol


def pss_query(A: torch.Tensor, k: int, P: int, workspace: torch.Tensor | None = None, stream=None):
    """The k-majority set of A: (items[k], counts[k] uint64, length[1]) device tensors."""
    A = _dev_keys(A)
    kt = _key_type(A)
    items = torch.empty((k,), dtype=_key_dtype(kt), device=A.device)
    counts = torch.empty((k,), dtype=torch.uint64, device=A.device)
    length = torch.zeros((1,), dtype=torch.uint32, device=A.device)
    ws = _ws(pss_workspace_bytes(OP_QUERY, A.numel(), k, P, kt), workspace, A.device, stream)
    _check("pss_query", _lib.pss_query(A.data_ptr(), A.numel(), kt, k, P, items.data_ptr(),
                                       counts.data_ptr(), length.data_ptr(), ws.data_ptr(),
                                       ws.numel(), _stream(stream)))
    return items, counts, length


def pss_query_host(A_host: torch.Tensor, k: int, P: int, d_A: torch.Tensor | None = None,
                   workspace: torch.Tensor | None = None, out=None, stream=None, sync=True):
    """End-to-end query from a HOST tensor (pinned recommended): H2D copy, the whole path, D2H of
    the result -- all inside the C call. Returns (items, counts) host tensors of the result."""
    if A_host.is_cuda:
        raise ValueError("A_host must be a host tensor")
    kt = _key_type(A_host)
    n = A_host.numel()
    dev = torch.device("cuda", torch.cuda.current_device())
    if d_A is None:
        d_A = torch.empty((max(n, 1),), dtype=A_host.dtype, device=dev)
        if stream is not None:
            d_A.record_stream(stream)
    ws = _ws(pss_workspace_bytes(OP_QUERY, n, k, P, kt), workspace, dev, stream)
    if out is None:
        pin = torch.cuda.is_available()
        out = (torch.empty((k,), dtype=_key_dtype(kt), pin_memory=pin),
               torch.empty((k,), dtype=torch.uint64, pin_memory=pin),
               torch.zeros((1,), dtype=torch.uint32, pin_memory=pin))
    oi, oc, ol = out
    _check("pss_query_host", _lib.pss_query_host(A_host.data_ptr(), d_A.data_ptr(), n, kt, k, P,
                                                 oi.data_ptr(), oc.data_ptr(), ol.data_ptr(),
                                                 ws.data_ptr(), ws.numel(), _stream(stream)))
    if sync:
        (stream or torch.cuda.current_stream()).synchronize()
        ln = int(ol[0].item())
        return oi[:ln], oc[:ln]
    return out


# ---- on-line ingestion (include/pss.h: pss_stream_*) ---------------------------------------
class _Stream(ctypes.Structure):
    _fields_ = [("key_type", ctypes.c_int32), ("k", ctypes.c_uint32), ("leaf_len", ctypes.c_uint32),
                ("batch_leaves", ctypes.c_uint32), ("n_seen", ctypes.c_uint64),
                ("d_ws", ctypes.c_void_p), ("ws_bytes", ctypes.c_size_t)]


_STP = ctypes.POINTER(_Stream)
_lib.pss_stream_workspace_bytes.argtypes = [_i32, _u32, _u32, _u32]
_lib.pss_stream_workspace_bytes.restype = _sz
_lib.pss_stream_init.argtypes = [_STP, _i32, _u32, _u32, _u32, _vp, _sz]
_lib.pss_stream_feed.argtypes = [_STP, _vp, _u64, _vp]
_lib.pss_stream_feed_host.argtypes = [_STP, _vp, _u64, _vp]
_lib.pss_stream_root.argtypes = [_STP, _SP, _vp]
_lib.pss_stream_root_wide.argtypes = [_STP, _SP, _vp]
for _f in ("pss_stream_init", "pss_stream_feed", "pss_stream_feed_host", "pss_stream_root",
           "pss_stream_root_wide"):
    getattr(_lib, _f).restype = _i32
EXPORTED_SYMBOLS += ["pss_stream_workspace_bytes", "pss_stream_init", "pss_stream_feed",
                     "pss_stream_feed_host", "pss_stream_root", "pss_stream_root_wide"]
__all__ += ["Stream", "pss_stream_workspace_bytes"]


def pss_stream_workspace_bytes(key_type: int, k: int, leaf_len: int, batch_leaves: int) -> int:
    return int(_lib.pss_stream_workspace_bytes(key_type, k, leaf_len, batch_leaves))


class Stream:
    """On-line Space Saving over a stream fed in pieces (pss_stream_*): leaves of `leaf_len`
    items, summary = the fixed binary COMBINE tree over the leaves so far (include/pss.h)."""

    def __init__(self, k: int, leaf_len: int, key_type: int = KEY_U32, batch_leaves: int = 1024,
                 device="cuda"):
        nb = pss_stream_workspace_bytes(key_type, k, leaf_len, batch_leaves)
        if nb == 0:
            raise PssError("pss_stream_workspace_bytes", 1)
        self.ws = torch.empty((nb,), dtype=torch.uint8, device=device)
        self._st = _Stream()
        _check("pss_stream_init", _lib.pss_stream_init(ctypes.byref(self._st), key_type, k, leaf_len,
                                                       batch_leaves, self.ws.data_ptr(), nb))

    @property
    def n_seen(self) -> int:
        return int(self._st.n_seen)

    @property
    def k(self) -> int:
        return int(self._st.k)

    @property
    def key_type(self) -> int:
        return int(self._st.key_type)

    def _check_keys(self, chunk: torch.Tensor):
        if _key_type(chunk) != self.key_type:
            raise TypeError("chunk key type differs from the stream's")
        if not chunk.is_contiguous():
            raise ValueError("chunk must be contiguous")

    def feed(self, chunk: torch.Tensor, stream=None) -> "Stream":
        """Append a DEVICE or HOST (pinned recommended) tensor of keys."""
        self._check_keys(chunk)
        fn = _lib.pss_stream_feed if chunk.is_cuda else _lib.pss_stream_feed_host
        _check("pss_stream_feed", fn(ctypes.byref(self._st), chunk.data_ptr() if chunk.numel() else None,
                                     chunk.numel(), _stream(stream)))
        return self

    def root(self, out: Summaries | None = None, stream=None, wide: bool = False) -> Summaries:
        """The summary of the stream so far, canonical order (one summary); wide = 64-bit
        counts (required once n_seen + n_seen / k reaches 2^32)."""
        out = out or Summaries.empty(1, self.k, self.key_type, self.ws.device, wide=wide)
        c = out._c()
        fn = _lib.pss_stream_root_wide if out.wide else _lib.pss_stream_root
        _check("pss_stream_root", fn(ctypes.byref(self._st), ctypes.byref(c), _stream(stream)))
        return out


# ---- accuracy (include/pss.h: pss_exact_kmajority, pss_accuracy) ----------------------------
OP_EXACT = 5


class AccuracyReport(ctypes.Structure):
    _fields_ = [("n_reported", ctypes.c_uint64), ("n_reported_true", ctypes.c_uint64),
                ("n_true", ctypes.c_uint64), ("precision", ctypes.c_double),
                ("recall", ctypes.c_double), ("are_reported", ctypes.c_double),
                ("are_true", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib.pss_exact_kmajority.argtypes = [_vp, _u64, _i32, _u32, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
_lib.pss_exact_kmajority.restype = _i32
_lib.pss_accuracy.argtypes = [_SP, _u64, _vp, _vp, _vp, _vp, _vp]
_lib.pss_accuracy.restype = _i32
EXPORTED_SYMBOLS += ["pss_exact_kmajority", "pss_accuracy"]
__all__ += ["OP_EXACT", "AccuracyReport", "pss_exact_kmajority", "pss_accuracy"]


def pss_exact_kmajority(A: torch.Tensor, k: int, workspace: torch.Tensor | None = None,
                        stream=None):
    """The k-majority set of A computed without Space Saving (local heavy hitters + exact counts):
    (items[k], counts[k] uint64, length[1], overflow[1]) device tensors, (f desc, x asc)."""
    A = _dev_keys(A)
    kt = _key_type(A)
    items = torch.empty((k,), dtype=_key_dtype(kt), device=A.device)
    counts = torch.empty((k,), dtype=torch.uint64, device=A.device)
    length = torch.zeros((1,), dtype=torch.uint32, device=A.device)
    overflow = torch.zeros((1,), dtype=torch.uint32, device=A.device)
    ws = _ws(pss_workspace_bytes(OP_EXACT, A.numel(), k, 0, kt), workspace, A.device, stream)
    _check("pss_exact_kmajority", _lib.pss_exact_kmajority(
        A.data_ptr(), A.numel(), kt, k, items.data_ptr(), counts.data_ptr(), length.data_ptr(),
        overflow.data_ptr(), ws.data_ptr(), ws.numel(), _stream(stream)))
    return items, counts, length, overflow


def pss_accuracy(root: Summaries, n: int, n_cand: torch.Tensor, exact: torch.Tensor,
                 n_true: torch.Tensor, stream=None) -> AccuracyReport:
    """Precision, recall and ARE of the root's pruned candidates (synchronises)."""
    out = torch.zeros((ctypes.sizeof(AccuracyReport),), dtype=torch.uint8, device=root.items.device)
    c = root._c()
    _check("pss_accuracy", _lib.pss_accuracy(ctypes.byref(c), n, n_cand.data_ptr(), exact.data_ptr(),
                                             n_true.data_ptr(), out.data_ptr(), _stream(stream)))
    return AccuracyReport.from_buffer_copy(bytes(out.cpu().numpy()))


# ---- hybrid decomposition (include/pss.h: pss_*_hybrid) ------------------------------------
_lib.pss_hybrid_workspace_bytes.argtypes = [_u64, _u32, _u32, _u32, _i32]
_lib.pss_hybrid_workspace_bytes.restype = _sz
_lib.pss_summarize_hybrid.argtypes = [_vp, _u64, _i32, _u32, _u32, _u32, _SP, _vp, _sz, _vp]
_lib.pss_summarize_hybrid.restype = _i32
_lib.pss_merge_hybrid.argtypes = [_SP, _u32, _SP, _vp, _sz, _vp]
_lib.pss_merge_hybrid.restype = _i32
EXPORTED_SYMBOLS += ["pss_hybrid_workspace_bytes", "pss_summarize_hybrid", "pss_merge_hybrid"]
__all__ += ["pss_hybrid_workspace_bytes", "pss_summarize_hybrid", "pss_merge_hybrid"]


def pss_hybrid_workspace_bytes(n: int, k: int, Pp: int, T: int, key_type: int) -> int:
    return int(_lib.pss_hybrid_workspace_bytes(n, k, Pp, T, key_type))


def pss_summarize_hybrid(A: torch.Tensor, k: int, Pp: int, T: int, out: Summaries | None = None,
                         workspace: torch.Tensor | None = None, stream=None) -> Summaries:
    """Leaves of the two-level (processes x threads) decomposition: leaf p*T + t."""
    A = _dev_keys(A)
    kt = _key_type(A)
    out = out or Summaries.empty(Pp * T, k, kt, A.device)
    ws = _ws(pss_hybrid_workspace_bytes(A.numel(), k, Pp, T, kt), workspace, A.device, stream)
    c = out._c()
    _check("pss_summarize_hybrid", _lib.pss_summarize_hybrid(
        A.data_ptr(), A.numel(), kt, k, Pp, T, ctypes.byref(c), ws.data_ptr(), ws.numel(),
        _stream(stream)))
    return out


def pss_merge_hybrid(leaves: Summaries, T: int, out: Summaries | None = None,
                     workspace: torch.Tensor | None = None, stream=None) -> Summaries:
    """Per-process fixed trees over groups of T leaves, then the fixed tree over the roots."""
    out = out or Summaries.empty(1, leaves.k, leaves.key_type, leaves.items.device)
    ws = _ws(pss_hybrid_workspace_bytes(0, leaves.k, leaves.count // max(T, 1), T, leaves.key_type),
             workspace, leaves.items.device, stream)
    a, b = leaves._c(), out._c()
    _check("pss_merge_hybrid", _lib.pss_merge_hybrid(ctypes.byref(a), T, ctypes.byref(b),
                                                     ws.data_ptr(), ws.numel(), _stream(stream)))
    return out


# ---- leaf kernel routing (include/pss.h: pss_leaf_kernels) ----------------------------------
_lib.pss_leaf_kernels.argtypes = [_u64, _u32, _u32, _i32]
_lib.pss_leaf_kernels.restype = _i32
LEAF_K1, LEAF_K1E, LEAF_K1H = 1, 2, 4
EXPORTED_SYMBOLS += ["pss_leaf_kernels"]
__all__ += ["pss_leaf_kernels", "epoch_used", "LEAF_K1", "LEAF_K1E", "LEAF_K1H"]


def pss_leaf_kernels(n: int, k: int, P: int, key_type: int) -> int:
    """Bit flags of the kernels that summarize the leaves of this shape (LEAF_K1/K1E/K1H)."""
    return int(_lib.pss_leaf_kernels(n, k, P, key_type))


def epoch_used(n: int, k: int, P: int, key_bytes: int = 4) -> bool:
    return bool(pss_leaf_kernels(n, k, P, KEY_U32 if key_bytes == 4 else KEY_U64) & LEAF_K1E)


# ---- K6 read-bandwidth probe (include/pss.h: pss_read_probe) -------------------------------
_lib.pss_read_probe.argtypes = [_vp, _u64, _i32, _vp, _vp]
_lib.pss_read_probe.restype = _i32
EXPORTED_SYMBOLS += ["pss_read_probe"]
__all__ += ["pss_read_probe"]


def pss_read_probe(A: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Reads A once with 128-bit loads (the attainable HBM read bandwidth); returns the fold."""
    A = _dev_keys(A)
    out = out if out is not None else torch.zeros((1,), dtype=torch.uint32, device=A.device)
    _check("pss_read_probe", _lib.pss_read_probe(A.data_ptr(), A.numel(), _key_type(A),
                                                 out.data_ptr(), _stream(stream)))
    return out
