"""Golden CLI transcripts produced by the REAL reference CLI (`kmerscan.cli`).

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_cli_golden.py [/root/reference/pkg/src]

Inputs are small seeded FASTA/raw files and pattern files written next to the
transcripts; every case records argv, exit code, stdout and stderr in
tests/golden/cli/cases.json.  The drop-in CLI must reproduce stdout and the
exit code byte for byte (tests/test_cli_bench.py).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "cli"
REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"


def write_inputs() -> None:
    HERE.mkdir(exist_ok=True)
    rng = np.random.default_rng(1509)
    body = bytes(np.frombuffer(b"acgtACGTnN", dtype=np.uint8)[rng.integers(0, 10, 20_000)])
    lines = [body[i:i + 60] for i in range(0, len(body), 60)]
    fasta = b">chr1 synthetic\n" + b"\n".join(lines[:150]) + b"\n>chr2\r\n" + b"\r\n".join(lines[150:]) + b"\r\n"
    (HERE / "seq.fa").write_bytes(fasta)
    (HERE / "seq.txt").write_bytes(body[:5000])
    (HERE / "pats.txt").write_text("acg\ncat\ncta\ntta\n")
    (HERE / "classes.txt").write_text("ac(g|t)t\n(a|c)(g|t)ga\ntt\nggg(a|t)\n")
    (HERE / "bad.txt").write_text("ac(g\n")


CASES = [
    ["count", "--patterns", "pats.txt", "--input", "seq.fa"],
    ["count", "--patterns", "classes.txt", "--input", "seq.fa", "--workers", "7", "--output-format", "json"],
    ["locate", "--patterns", "pats.txt", "--input", "seq.txt", "--workers", "3"],
    ["locate", "--patterns", "classes.txt", "--input", "seq.fa", "--output-format", "json", "--window", "0"],
    ["count", "--patterns", "pats.txt", "--input", "seq.fa", "--format", "raw"],
    ["dump-dfa", "--patterns", "classes.txt"],
    ["dump-dfa", "--patterns", "pats.txt", "--minimized"],
    ["count", "--patterns", "bad.txt", "--input", "seq.fa"],
    ["count", "--patterns", "pats.txt", "--input", "missing.fa"],
    ["bench", "--patterns", "pats.txt", "--synthetic-size", "64K", "--workers", "1,3", "--repeat", "2",
     "--pattern-based"],
    ["bench", "--patterns", "classes.txt", "--input", "seq.fa", "--workers", "2", "--repeat", "1",
     "--output-format", "json"],
]


def main() -> None:
    write_inputs()
    env = dict(os.environ, PYTHONPATH=REF, PYTHONDONTWRITEBYTECODE="1",
               NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/numba_cache"))
    out = []
    for argv in CASES:
        p = subprocess.run([sys.executable, "-c", "import sys; from kmerscan.cli import main; sys.exit(main())", *argv], cwd=HERE, env=env, capture_output=True,
                           text=True)
        out.append({"argv": argv, "code": p.returncode, "stdout": p.stdout, "stderr": p.stderr})
        print(argv[0], p.returncode, len(p.stdout))
    (HERE / "cases.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
