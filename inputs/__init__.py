"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds no arithmetic of the method (no Space Saving, no COMBINE, no counting). It
only generates the input arrays A and names the workloads of BASELINE.json (configs C1-C5 and the
headline H). The generator is plain C (``inputs/zipfgen.c``), compiled
with gcc into ``inputs/libpssgen.so`` by :func:`build` and called through ctypes. The recipe is in
DESIGN.md ("Input recipe") and in the C file's header.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "zipfgen.c")
_LIB = os.path.join(_HERE, "libpssgen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the generator with gcc (plain C, -O2, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.pssgen_zipf.restype = ctypes.c_int
        lib.pssgen_zipf.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_uint64, ctypes.c_double, ctypes.c_int,
                                    ctypes.c_int]
        lib.pssgen_zipf_range.restype = ctypes.c_int
        lib.pssgen_zipf_range.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_uint64, ctypes.c_double, ctypes.c_int,
                                          ctypes.c_int]
        lib.pssgen_mix32.restype = ctypes.c_uint32
        lib.pssgen_mix32.argtypes = [ctypes.c_uint32]
        lib.pssgen_mix64.restype = ctypes.c_uint64
        lib.pssgen_mix64.argtypes = [ctypes.c_uint64]
        _lib = lib
    return _lib


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def zipf(n: int, s: float, universe: float, seed: int, key_bytes: int = 4,
         tail_frac: float = 0.0, hash_ids: bool = True, threads: int | None = None,
         out: np.ndarray | None = None, start: int = 0) -> np.ndarray:
    """Positions [start, start + n) of the i.i.d. Zipf(s) stream over `universe` ranks (hashed
    ids), as a numpy u32/u64 array. `out` may be a preallocated (e.g. pinned) contiguous array.
    """
    dt = np.uint32 if key_bytes == 4 else np.uint64
    if out is None:
        out = np.empty(int(n), dtype=dt)
    assert out.dtype == dt and out.size == n and out.flags["C_CONTIGUOUS"]
    rc = _load().pssgen_zipf_range(out.ctypes.data if n else None, int(start), int(n), key_bytes,
                                   float(s), float(universe), int(seed), float(tail_frac),
                                   int(hash_ids), int(threads or host_threads()))
    if rc != 0:
        raise ValueError("pssgen_zipf rejected its arguments")
    return out


def mix32(r: int) -> int:
    return int(_load().pssgen_mix32(r))


def mix64(r: int) -> int:
    return int(_load().pssgen_mix64(r))


@dataclass(frozen=True)
class Workload:
    """One synthetic workload of BASELINE.json."""
    name: str
    n: int
    key_bytes: int
    s: float
    universe: float
    seed: int
    k: int
    P: int
    tail_frac: float = 0.0
    verify: bool = True
    note: str = field(default="", compare=False)

    def generate(self, n: int | None = None, out=None, threads=None, start: int = 0) -> np.ndarray:
        """Keys [start, start + n) (default: the whole workload) of this workload's stream."""
        return zipf(self.n if n is None else n, self.s, self.universe, self.seed, self.key_bytes,
                    self.tail_frac, True, threads, out, start)

    def describe(self) -> dict:
        return {"workload": self.name, "n": self.n, "key": "u32" if self.key_bytes == 4 else "u64",
                "zipf_s": self.s, "universe": self.universe, "seed": self.seed, "k": self.k,
                "P": self.P, "tail_frac": self.tail_frac}


def _c3(s):
    return Workload(f"C3-s{s}", 1 << 29, 4, s, 1e8, 3, 2000, 8192, note="BASELINE.json configs[2]")


def _c4(k):
    return Workload(f"C4-k{k}", 1 << 28, 4, 1.5, float(1 << 32), 4, k, 4096, verify=False,
                    note="BASELINE.json configs[3]")


WORKLOADS: dict[str, Workload] = {
    w.name: w for w in [
        Workload("C1", 1_000_000, 4, 1.1, float(1 << 20), 1, 100, 64, note="BASELINE.json configs[0]"),
        Workload("C2", 1 << 28, 4, 1.1, 1e8, 2, 1000, 4096, note="BASELINE.json configs[1]"),
        *[_c3(s) for s in (0.5, 1.0, 1.5, 2.0, 3.0)],
        *[_c4(k) for k in (200, 1000, 5000, 20000)],
        Workload("C5", 1 << 31, 8, 1.8, float(1 << 40), 5, 2000, 32768, tail_frac=0.01,
                 note="BASELINE.json configs[4]"),
        # Headline: the metric's n=2^29, k=1000 (BASELINE.json "metric"); seed 2 so its first
        # 2^28 keys are C2's array; P=8192 (chunks of 65 536 keys).
        Workload("H", 1 << 29, 4, 1.1, 1e8, 2, 1000, 8192, note="BASELINE.json metric"),
    ]
}
