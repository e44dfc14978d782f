"""Scan throughput for automata beyond the fast kernel (|Q| >= 4096)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_01506_b200 as ks  # noqa: E402
from paper_1509_01506_b200 import _native, workloads  # noqa: E402
from oracle import oracle as O  # noqa: E402

rng = np.random.default_rng(7)
w = workloads.make(3, 1 << 28)
ctx = _native.context(0)
sh = ctx.upload_ascii(w.ascii)
sym = None
sizes = [(400, 12), (1000, 14), (2000, 14), (2600, 13), (6000, 14), (12000, 16)]
if len(sys.argv) > 1 and sys.argv[1] == "mid":    # 16-bit automata whose table exceeds shared memory
    sizes = [(2800, 14), (3200, 14), (3600, 14), (3900, 14)]
if len(sys.argv) > 1 and sys.argv[1] == "wide":   # automata above 32767 states
    sizes = [(4000, 14), (8000, 16), (5000, 24), (12000, 20)]
for nlit, length in sizes:
    lits = set()
    while len(lits) < nlit:
        lits.add("".join(rng.choice(list("acgt"), size=length)))
    dfa = ks.build_dfa(ks.expand_to_literals(ks.parse_expressions("\n".join(sorted(lits)) + "\n")))
    dh = ctx.dfa(dfa)
    c = ctx.count(dh, sh)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.count(dh, sh)
        ts.append(time.perf_counter() - t0)
    st = ctx.stats()
    info = dh.info
    print(f"|Q|={dfa.state_count} K={info['stride']} smem={info['tables_in_smem']} table={info['table_bytes']} "
          f"scan {st['scan_ms']:.3f} ms -> {w.n / st['scan_ms'] / 1e6:.0f} GB/s, matches {int(c.sum())}", flush=True)
    if nlit == 400:
        if sym is None:
            sym = ks.encode_bytes(w.ascii[: 1 << 22].tobytes())
        small = ctx.upload_codes(sym)
        assert ctx.count(dh, small).tolist() == O.ref_sequential_count(dfa, sym)[0].tolist()
