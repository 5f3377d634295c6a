"""CPU-side checks of the boundary: libpss.so loads, exports every symbol include/pss.h declares,
sizes workspaces, and rejects bad arguments before launching anything (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pss():
    from conftest import build_lib
    build_lib()
    import paper_1606_04669_b200 as p
    return p


def header_functions():
    src = open(os.path.join(ROOT, "include", "pss.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(pss_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ["pss_summarize", "pss_merge", "pss_combine", "pss_prune", "pss_verify", "pss_query",
              "pss_query_host", "pss_workspace_bytes", "pss_status_string", "pss_version"]:
        assert f in fns


def test_library_exports_every_declared_symbol(pss):
    lib = ctypes.CDLL(pss.lib_path)
    for f in header_functions():
        assert hasattr(lib, f), f
    assert set(header_functions()) == set(pss.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", pss.lib_path], capture_output=True,
                         text=True).stdout
    for f in header_functions():
        assert re.search(rf"\bT {f}$", out, re.M), f


def test_sm100a_code_only(pss):
    out = subprocess.run(["cuobjdump", "--list-elf", pss.lib_path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_status_strings_and_version(pss):
    lib = pss._lib
    assert lib.pss_status_string(0) == b"PSS_OK"
    assert lib.pss_status_string(4) == b"PSS_ERR_WORKSPACE_TOO_SMALL"
    assert b"sm_100a" in lib.pss_version()


def test_workspace_bytes_monotone(pss):
    for kt in (pss.KEY_U32, pss.KEY_U64):
        q1 = pss.pss_workspace_bytes(pss.OP_QUERY, 1 << 20, 100, 64, kt)
        q2 = pss.pss_workspace_bytes(pss.OP_QUERY, 1 << 20, 1000, 64, kt)
        q3 = pss.pss_workspace_bytes(pss.OP_QUERY, 1 << 20, 1000, 4096, kt)
        assert 0 < q1 < q2 < q3
        assert pss.pss_workspace_bytes(pss.OP_MERGE, 0, 1000, 8192, kt) > 0
        assert pss.pss_workspace_bytes(pss.OP_VERIFY, 0, 1000, 1, kt) > 0
    assert pss.pss_workspace_bytes(pss.OP_QUERY, 10, 10, 1, 7) == 0  # bad key type


def test_validation_before_launch(pss):
    """Bad arguments return status codes without touching the device."""
    lib = pss._lib
    S = pss._Summ
    dummy = ctypes.c_void_p(0x1000)
    leaves = S(0, 10, 4, 0x1000, 0x1000, 0x1000, 0x1000)
    by = ctypes.byref
    # k < 2
    assert lib.pss_summarize(dummy, 100, 0, 1, 4, by(leaves), dummy, 1 << 20, None) == 1
    # P == 0
    assert lib.pss_summarize(dummy, 100, 0, 10, 0, by(leaves), dummy, 1 << 20, None) == 1
    # bad key type
    assert lib.pss_summarize(dummy, 100, 3, 10, 4, by(leaves), dummy, 1 << 20, None) == 1
    # n > 2^31
    assert lib.pss_summarize(dummy, (1 << 31) + 1, 0, 10, 4, by(leaves), dummy, 1 << 20, None) == 2
    # mismatched capacity / key type / count
    assert lib.pss_summarize(dummy, 100, 0, 11, 4, by(leaves), dummy, 1 << 20, None) == 3
    assert lib.pss_summarize(dummy, 100, 1, 10, 4, by(leaves), dummy, 1 << 20, None) == 3
    assert lib.pss_summarize(dummy, 100, 0, 10, 5, by(leaves), dummy, 1 << 20, None) == 3
    # null leaves / null A
    assert lib.pss_summarize(dummy, 100, 0, 10, 4, None, dummy, 1 << 20, None) == 1
    assert lib.pss_summarize(None, 100, 0, 10, 4, by(leaves), dummy, 1 << 20, None) == 1
    # merge: root must have count 1 and the same k/type
    root = S(0, 10, 2, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_merge(by(leaves), by(root), dummy, 1 << 30, None) == 3
    root = S(1, 10, 1, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_merge(by(leaves), by(root), dummy, 1 << 30, None) == 3
    # combine: mismatched k
    b = S(0, 12, 4, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_combine(by(leaves), by(b), by(leaves), dummy, 1 << 30, None) == 3
    # query: k < 2, P == 0, null outputs
    assert lib.pss_query(dummy, 100, 0, 1, 4, dummy, dummy, dummy, dummy, 1 << 30, None) == 1
    assert lib.pss_query(dummy, 100, 0, 10, 0, dummy, dummy, dummy, dummy, 1 << 30, None) == 1
    assert lib.pss_query(dummy, 100, 0, 10, 4, None, dummy, dummy, dummy, 1 << 30, None) == 1
    # verify: null candidates with n_cand > 0
    assert lib.pss_verify(dummy, 100, 0, None, 5, None, dummy, dummy, 1 << 20, None) == 1


def test_workspace_too_small_is_reported(pss):
    lib = pss._lib
    S = pss._Summ
    dummy = ctypes.c_void_p(0x1000)
    leaves = S(0, 1000, 4096, 0x1000, 0x1000, 0x1000, 0x1000)
    root = S(0, 1000, 1, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_merge(ctypes.byref(leaves), ctypes.byref(root), dummy, 1024, None) == 4
    assert lib.pss_query(dummy, 1 << 20, 0, 1000, 4096, dummy, dummy, dummy, dummy, 1024, None) == 4


def test_product_path_does_not_import_the_oracle():
    """The product package must not reference oracle/ (parity would be void)."""
    pkg = os.path.join(ROOT, "paper_1606_04669_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\boracle\b", src.replace("oracle/", "")), f


def test_stream_validation_before_launch(pss):
    """pss_stream_*: bad arguments return status codes; init launches nothing (include/pss.h)."""
    lib = pss._lib
    st = pss._Stream()
    by = ctypes.byref
    dummy = ctypes.c_void_p(0x1000)
    nb = pss.pss_stream_workspace_bytes(pss.KEY_U32, 1000, 65536, 16)
    assert nb > 16 * 65536 * 4 * 2 and pss.pss_stream_workspace_bytes(pss.KEY_U32, 1, 10, 1) == 0
    assert pss.pss_stream_workspace_bytes(7, 10, 10, 1) == 0
    assert lib.pss_stream_init(None, 0, 10, 100, 4, dummy, 1 << 30) == 1
    assert lib.pss_stream_init(by(st), 0, 1, 100, 4, dummy, 1 << 30) == 1       # k < 2
    assert lib.pss_stream_init(by(st), 0, 10, 0, 4, dummy, 1 << 30) == 1        # leaf_len 0
    assert lib.pss_stream_init(by(st), 0, 10, 100, 0, dummy, 1 << 30) == 1      # batch 0
    assert lib.pss_stream_init(by(st), 3, 10, 100, 4, dummy, 1 << 30) == 1      # key type
    assert lib.pss_stream_init(by(st), 0, 70000, 100, 4, dummy, 1 << 30) == 2   # k > PSS_MAX_K
    assert lib.pss_stream_init(by(st), 0, 10, 1 << 20, 1 << 12, dummy, 1 << 40) == 2  # batch > 2^31
    assert lib.pss_stream_init(by(st), 0, 10, 100, 4, dummy, 1024) == 4         # workspace
    need = pss.pss_stream_workspace_bytes(pss.KEY_U32, 10, 100, 4)
    assert lib.pss_stream_init(by(st), 0, 10, 100, 4, dummy, need) == 0
    assert (st.k, st.leaf_len, st.batch_leaves, st.n_seen) == (10, 100, 4, 0)
    # feeds: null chunk with len > 0; a stream longer than 2^63 items (64-bit counts above the
    # blocks) or one whose length wraps
    assert lib.pss_stream_feed(by(st), None, 5, None) == 1
    assert lib.pss_stream_feed(by(st), dummy, (1 << 63) + 1, None) == 2
    assert lib.pss_stream_feed_host(by(st), dummy, (1 << 64) - 1, None) == 2
    assert st.n_seen == 0
    # the narrow root is refused once N + N/k could exceed a u32 counter (R9); the wide one is not
    big = pss._Stream.from_buffer_copy(st)
    big.n_seen = 1 << 32
    root = pss._Summ(0, 10, 1, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_stream_root(by(big), by(root), None) == 2
    assert lib.pss_stream_root_wide(by(big), by(pss._Summ(0, 11, 1, 0x1000, 0x1000, 0x1000,
                                                             0x1000)), None) == 3
    # root: capacity mismatch
    root = pss._Summ(0, 11, 1, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_stream_root(by(st), by(root), None) == 3
    root = pss._Summ(1, 10, 1, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_stream_root(by(st), by(root), None) == 3


def test_accuracy_validation_before_launch(pss):
    lib = pss._lib
    dummy = ctypes.c_void_p(0x1000)
    ws = pss.pss_workspace_bytes(pss.OP_EXACT, 1 << 29, 1000, 0, pss.KEY_U32)
    assert ws > (1 << 24) * 4
    assert lib.pss_exact_kmajority(dummy, 100, 0, 1, dummy, dummy, dummy, None, dummy, ws, None) == 1
    assert lib.pss_exact_kmajority(dummy, 100, 5, 10, dummy, dummy, dummy, None, dummy, ws, None) == 1
    assert lib.pss_exact_kmajority(dummy, 100, 0, 10, None, dummy, dummy, None, dummy, ws, None) == 1
    assert lib.pss_exact_kmajority(dummy, (1 << 31) + 1, 0, 10, dummy, dummy, dummy, None, dummy,
                                   1 << 40, None) == 2
    assert lib.pss_exact_kmajority(dummy, 100, 0, 10, dummy, dummy, dummy, None, dummy, 64, None) == 4
    root = pss._Summ(0, 10, 1, 0x1000, 0x1000, 0x1000, 0x1000)
    by = ctypes.byref
    assert lib.pss_accuracy(by(root), 100, None, dummy, dummy, dummy, None) == 1
    assert lib.pss_accuracy(by(root), 100, dummy, dummy, dummy, None, None) == 1
    two = pss._Summ(0, 10, 2, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_accuracy(by(two), 100, dummy, dummy, dummy, dummy, None) == 1
    assert ctypes.sizeof(pss.AccuracyReport) == 56


def test_hybrid_validation_before_launch(pss):
    lib = pss._lib
    by = ctypes.byref
    dummy = ctypes.c_void_p(0x1000)
    S = pss._Summ
    assert pss.pss_hybrid_workspace_bytes(1 << 20, 100, 4, 3, pss.KEY_U32) > 0
    assert pss.pss_hybrid_workspace_bytes(1 << 20, 100, 0, 3, pss.KEY_U32) == 0
    leaves = S(0, 10, 12, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_summarize_hybrid(dummy, 100, 0, 10, 0, 3, by(leaves), dummy, 1 << 30, None) == 1
    assert lib.pss_summarize_hybrid(dummy, 100, 0, 10, 4, 0, by(leaves), dummy, 1 << 30, None) == 1
    assert lib.pss_summarize_hybrid(dummy, 100, 0, 10, 4, 4, by(leaves), dummy, 1 << 30, None) == 3
    assert lib.pss_summarize_hybrid(dummy, 100, 0, 10, 4, 3, by(leaves), dummy, 16, None) == 4
    root = S(0, 10, 1, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_merge_hybrid(by(leaves), 5, by(root), dummy, 1 << 30, None) == 1  # 12 % 5
    assert lib.pss_merge_hybrid(by(leaves), 0, by(root), dummy, 1 << 30, None) == 1
    bad = S(1, 10, 1, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_merge_hybrid(by(leaves), 3, by(bad), dummy, 1 << 30, None) == 3


def test_read_probe_validation(pss):
    lib = pss._lib
    assert lib.pss_read_probe(ctypes.c_void_p(0x1004), 10, 0, ctypes.c_void_p(0x1000), None) == 1
    assert lib.pss_read_probe(ctypes.c_void_p(0x1000), 10, 0, None, None) == 1
    assert lib.pss_read_probe(ctypes.c_void_p(0x1000), 10, 9, ctypes.c_void_p(0x1000), None) == 1


def test_wide_validation_before_launch(pss):
    """The wide-summary calls (64-bit counts) validate like their narrow twins."""
    lib = pss._lib
    S = pss._Summ
    dummy = ctypes.c_void_p(0x1000)
    by = ctypes.byref
    a = S(0, 10, 4, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_widen(None, by(a), None) == 1
    assert lib.pss_widen(by(a), by(S(0, 11, 4, 0x1000, 0x1000, 0x1000, 0x1000)), None) == 3
    assert lib.pss_combine_wide(by(a), by(S(1, 10, 4, 0x1000, 0x1000, 0x1000, 0x1000)), by(a),
                                dummy, 1 << 30, None) == 3
    assert lib.pss_combine_wide(by(a), by(a), by(a), None, 1 << 30, None) == 1
    assert lib.pss_merge_wide(by(a), by(S(0, 10, 2, 0x1000, 0x1000, 0x1000, 0x1000)), dummy,
                              1 << 30, None) == 3
    assert lib.pss_merge_wide(by(a), by(S(0, 10, 1, 0x1000, 0x1000, 0x1000, 0x1000)), dummy,
                              16, None) == 4
    root = S(0, 10, 1, 0x1000, 0x1000, 0x1000, 0x1000)
    assert lib.pss_prune_wide(by(a), 100, dummy, dummy, None) == 1  # count != 1
    assert lib.pss_prune_wide(by(root), 1 << 63, dummy, dummy, None) == 2
    assert lib.pss_prune_wide(by(root), 100, None, dummy, None) == 1
