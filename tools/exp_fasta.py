"""End-to-end count of a FASTA rendering of C3 (60-column lines, a header
every 16 MiB) through ks_count_host_bytes; checks against the oracle."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_01506_b200 as ks  # noqa: E402
from paper_1509_01506_b200 import _native, workloads  # noqa: E402
from oracle import oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
w = workloads.make(3, n)
body = w.ascii
lines = body[: n - n % 60].reshape(-1, 60)
fa = np.empty((lines.shape[0], 61), dtype=np.uint8)
fa[:, :60] = lines
fa[:, 60] = ord("\n")
flat = fa.reshape(-1)
hdr = np.frombuffer(b">chrN synthetic header line\n", dtype=np.uint8)
step = ((16 << 20) // 61) * 61   # headers start lines
parts = []
for i in range(0, flat.size, step):
    parts += [hdr, flat[i:i + step]]
data = np.concatenate(parts)
pinned = torch.empty(data.size, dtype=torch.uint8, pin_memory=True)
pinned.numpy()[:] = data
ctx = _native.context(0)
dh = ctx.dfa(w.dfa)
want = O.ref_sequential_count(w.dfa, ks.encode_bytes(body[: n - n % 60].tobytes()))[0]
got = ctx.count_host_ascii(dh, pinned.numpy(), fasta=True)
assert got.tolist() == want.tolist(), "fasta e2e mismatch"
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.count_host_ascii(dh, pinned.numpy(), fasta=True)
    ts.append(time.perf_counter() - t0)
st = ctx.stats()
t = float(np.median(ts))
print(f"fasta e2e: {data.size / t / 1e9:.1f} GB/s of file bytes, {(n - n % 60) / t / 1e9:.1f} Gbases/s, "
      f"{t * 1e3:.1f} ms, h2d {st['h2d_bytes']} launches {st['kernel_launches']}")
