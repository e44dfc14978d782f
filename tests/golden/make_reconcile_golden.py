"""Fixture generator: the REAL reference's exhaustive reconciliation check on
the toy automaton (reference tests/conftest.py TOY_PATTERNS), lengths 1..12
with window 10 and length 3 with window 0 (reference
tests/test_acceptance.py:169-181, tests/test_oracle_bench.py:62-73).

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \\
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_reconcile_golden.py

Writes tests/golden/reconcile_toy.json (per-length speculative/converged runs
and mismatch counts).  Run in the build container only (the reference does
not travel to the GPU box)."""

import json
from pathlib import Path

import kmerscan as ref

TOY_PATTERNS = "acg\ncat\ncta\ntta"


def main():
    dfa = ref.build_dfa(ref.expand_to_literals(ref.parse_expressions(TOY_PATTERNS)))
    out = {"patterns": TOY_PATTERNS, "window10": [], "window0_len3": None}
    for length in range(1, 13):
        r = ref.exhaustive_reconciliation_check(dfa, length, window=10)
        out["window10"].append({k: int(v) for k, v in r.items()})
        print(r, flush=True)
    r = ref.exhaustive_reconciliation_check(dfa, 3, window=0)
    out["window0_len3"] = {k: int(v) for k, v in r.items()}
    Path(__file__).with_name("reconcile_toy.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
