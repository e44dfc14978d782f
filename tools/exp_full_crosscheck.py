"""Full-size cross-checks of independent kernel paths (no oracle at this size):
C4 locate through the lean log kernel vs the per-step log kernel vs the
two-pass (rows + emit) form; C4 count lean vs ring."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_01506_b200 import _native, workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
t0 = time.time()
w = workloads.make(cfg)
print(f"C{cfg} generated in {time.time() - t0:.0f}s", flush=True)
results = {}
for name, env in (("default", {}), ("ring", {"KS_LEAN": "0"}), ("lean", {"KS_LEAN": "1"}),
                  ("two-sync", {"KS_LOCATE_TWO_SYNC": "1"})):
    for k, v in env.items():
        os.environ[k] = v
    ctx = _native.DeviceContext(0)
    dh = ctx.dfa(w.dfa)
    sh = ctx.upload_ascii(w.ascii)
    c = ctx.count(dh, sh)
    lc, rows = ctx.locate(dh, sh)
    results[name] = (c, lc, rows)
    print(f"{name}: total {int(c.sum())} rows {rows.shape[0]} sorted "
          f"{bool(np.all(np.diff(rows[:, 0] * 1000 + rows[:, 1]) >= 0)) if rows.shape[0] else True}", flush=True)
    for k in env:
        del os.environ[k]
    del sh, dh, ctx
base = results["default"]
for name, (c, lc, rows) in results.items():
    ok = np.array_equal(c, base[0]) and np.array_equal(lc, base[1]) and np.array_equal(rows, base[2])
    print(f"{name} == default: {ok}")
