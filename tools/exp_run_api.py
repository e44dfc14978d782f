import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1509_01506_b200 as ks
from paper_1509_01506_b200 import workloads
for cfg in (3, 4, 5):
    w = workloads.make(cfg)
    seq = ks.Sequence(ks.encode_bytes(w.ascii.tobytes())) if cfg != 4 else None
    if seq is None:
        seq = ks.Sequence(ks.encode_bytes(w.ascii.tobytes()))
    for mode in ("count",) if cfg != 4 else ("count", "locate"):
        for rep in range(2):
            t0 = time.perf_counter()
            r = ks.run(w.dfa, seq, ks.EngineConfig(mode=mode))
            t = time.perf_counter() - t0
        print(f"C{cfg} run({mode}) {t*1e3:.1f} ms  total {r.total_count}  meta keys {sorted(r.metadata)[:4]}", flush=True)
