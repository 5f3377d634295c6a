#!/usr/bin/env python
"""Time K4 (pss_verify) alone on a BASELINE workload, with the candidates the path produces.

  python tools/verify_time.py [--workload H] [--reps 10] [--libs a.so b.so ...]

Each --libs entry is an experiment build of libpss.so (tools/variant.sh), timed in a child
process with PSS_LIB pointing at it; without --libs the in-tree library is timed.
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(a):
    import torch

    import inputs
    import paper_1606_04669_b200 as pss

    w = inputs.WORKLOADS[a.workload]
    A = torch.from_numpy(w.generate(w.n)).cuda()
    kt = pss.KEY_U32 if w.key_bytes == 4 else pss.KEY_U64
    leaves = pss.pss_summarize(A, w.k, w.P)
    root = pss.pss_merge(leaves)
    cand, n_cand = pss.pss_prune(root, w.n)
    ws = torch.empty((pss.pss_workspace_bytes(pss.OP_VERIFY, w.n, w.k, 1, kt),), dtype=torch.uint8,
                     device="cuda")
    out = torch.empty((w.k,), dtype=torch.uint64, device="cuda")
    for _ in range(3):
        pss.pss_verify(A, cand, n_cand, out=out, workspace=ws)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pss.pss_verify(A, cand, n_cand, out=out, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[len(ts) // 2]
    nb = w.n * w.key_bytes
    print(f"{os.environ.get('PSS_LIB', 'in-tree')}: {a.workload} n_cand={int(n_cand.item())} "
          f"verify {t * 1e3:.1f} us  {nb / t / 1e6:.1f} GB/s")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="H")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--libs", nargs="*", default=[])
    a = ap.parse_args()
    if not a.libs:
        run(a)
        return
    for lib in a.libs:
        env = dict(os.environ, PSS_LIB=os.path.abspath(lib))
        subprocess.run([sys.executable, __file__, "--workload", a.workload, "--reps", str(a.reps)],
                       env=env, check=False)


if __name__ == "__main__":
    main()
