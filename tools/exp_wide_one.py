"""One wide automaton (> 32767 states) over 256 MiB: count a few times (ncu target)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_01506_b200 as ks  # noqa: E402
from paper_1509_01506_b200 import _native, workloads  # noqa: E402

nlit, length = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (12000, 20)
rng = np.random.default_rng(7)
w = workloads.make(3, 1 << 28)
ctx = _native.context(0)
sh = ctx.upload_ascii(w.ascii)
lits = set()
while len(lits) < nlit:
    lits.add("".join(rng.choice(list("acgt"), size=length)))
dfa = ks.build_dfa(ks.expand_to_literals(ks.parse_expressions("\n".join(sorted(lits)) + "\n")))
dh = ctx.dfa(dfa)
for _ in range(3):
    c = ctx.count(dh, sh)
print(f"|Q|={dfa.state_count} scan {ctx.stats()['scan_ms']:.3f} ms, matches {int(c.sum())}")
