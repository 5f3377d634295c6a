"""Mutation check of the oracle's pins (not collected by pytest; run by hand:
`python tests/oracle_mutations.py`). Each plausible mistake below is patched into
oracle/pss_oracle.c in turn and tests/test_oracle_pins.py must fail; the file is restored after.
Last run: every mutation CAUGHT ("Oracle pins")."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.chdir(ROOT)
SRC = os.path.join('oracle', 'pss_oracle.c')
orig = open(SRC).read()
muts = {
 'evict_highest': ('while (counts[v] != m) ++v;', 'v = k - 1; while (counts[v] != m) --v;'),
 'err_off': ('errs[v] = m;', 'errs[v] = m + 1;'),
 'swap_m': ('sc[nc++] = (counter_t){it1[i], c1[i] + m2, e1[i] + m2};', 'sc[nc++] = (counter_t){it1[i], c1[i] + m1, e1[i] + m1};'),
 'R4_dropped': ('if (size < k) return 0;', 'if (size == 0) return 0;'),
 'tie_desc': ('return x->item < y->item ? -1 : 1;', 'return x->item > y->item ? -1 : 1;'),
 'matched_err': ('c1[i] + c2[j], e1[i] + e2[j]}', 'c1[i] + c2[j], e1[i]}'),
 'no_carry': ('if (cur & 1u) {', 'if (0) {'),
 'thr': ('return n / k + 1;', 'return n / k;'),
 'bounds': ('*hi = (uint64_t)(((unsigned __int128)(r + 1u) * n) / p);', '*hi = (uint64_t)(((unsigned __int128)(r + 1u) * n + p - 1) / p);'),
}
for name, (a, b) in muts.items():
    assert a in orig, name
    open(SRC, 'w').write(orig.replace(a, b))
    r = subprocess.run([sys.executable, '-m', 'pytest', 'tests/test_oracle_pins.py', '-x', '-q', '-p', 'no:cacheprovider'], capture_output=True, text=True)
    print(name, 'CAUGHT' if r.returncode else 'MISSED', r.stdout.strip().splitlines()[-1])
open(SRC, 'w').write(orig)
subprocess.run([sys.executable, '-c', 'import oracle; oracle.build(force=True)'])
