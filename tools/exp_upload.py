"""Codes upload (ks_seq_upload_codes) time, host-packed vs device-packed
(KS_DEVICE_PACK_CODES=1), pageable numpy input (gpurun)."""
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_01506_b200 as ks  # noqa: E402
from paper_1509_01506_b200 import _native, workloads  # noqa: E402

w = workloads.make(3, int(os.environ.get("N", str(1 << 30))))
codes = ks.encode_bytes(w.ascii.tobytes())
ctx = _native.context(0)
for v in ("host", "device", "host", "device"):
    if v == "device":
        os.environ["KS_DEVICE_PACK_CODES"] = "1"
    else:
        os.environ.pop("KS_DEVICE_PACK_CODES", None)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        sh = ctx.upload_codes(codes)
        ts.append(time.perf_counter() - t0)
        sh.free()
    print(f"{v}: {statistics.median(ts) * 1e3:.1f} ms for {codes.size} symbols "
          f"({codes.size / statistics.median(ts) / 1e9:.1f} Gsym/s)", flush=True)
