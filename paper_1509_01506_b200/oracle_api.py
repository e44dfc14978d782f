"""The reference's public oracle functions (`kmerscan/oracle.py:24-116`),
kept for API compatibility.  ``naive_count`` is the reference's brute-force
literal matcher (host numpy, shares no code with any automaton);
``pattern_parallel_count`` and ``exhaustive_reconciliation_check`` run their
scans on the GPU engine.  (This module is part of the product API; it is
unrelated to the repository's test oracle under ``oracle/``.)
"""

from __future__ import annotations

import itertools

import numpy as np

from .alphabet import BASE_CODES, N_SYMBOLS
from .automaton import Dfa, build_dfa
from .engine import possible_starting_states, sequential_count
from .ingest import Sequence
from .patterns import ExpressionSet, LiteralTable, expand_to_literals


def naive_count(table: LiteralTable, seq: Sequence) -> tuple[np.ndarray, np.ndarray]:
    """Every literal checked at every start position; overlaps count, OTHER
    matches nothing.  Returns (counts, rows sorted by (end offset, id))."""
    sym = np.asarray(seq.symbols)
    n = sym.shape[0]
    counts = np.zeros(table.n_expressions, dtype=np.int64)
    parts = []
    for literal, expr_id in table.literals:
        codes = [BASE_CODES[c] for c in literal]
        k = len(codes)
        if k > n:
            continue
        hit = np.ones(n - k + 1, dtype=bool)
        for j, c in enumerate(codes):
            hit &= sym[j:n - k + 1 + j] == c
        pos = np.flatnonzero(hit)
        counts[expr_id] += pos.size
        if pos.size:
            parts.append(np.column_stack([pos + k, np.full(pos.size, expr_id)]).astype(np.int64))
    rows = np.concatenate(parts) if parts else np.empty((0, 2), dtype=np.int64)
    return counts, rows[np.lexsort((rows[:, 1], rows[:, 0]))]


def pattern_parallel_count(exprs: ExpressionSet, seq: Sequence, workers: int) -> np.ndarray:
    """Expressions partitioned round-robin into `workers` automata, each
    scanning the whole sequence (the paper's Fig. 1b alternative)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    table = expand_to_literals(exprs)
    groups: list[list[tuple[str, int]]] = [[] for _ in range(workers)]
    for literal, expr_id in table.literals:
        groups[expr_id % workers].append((literal, expr_id))
    total = np.zeros(table.n_expressions, dtype=np.int64)
    for g in groups:
        if g:
            total += sequential_count(build_dfa(LiteralTable(tuple(g), table.n_expressions)), seq)
    return total


def exhaustive_reconciliation_check(dfa: Dfa, length: int, window: int) -> dict:
    """All 4**length base words x every border symbol: each converged
    speculative run's reconciled counts and final state must equal a full
    scan from its own start state (reference oracle.py:94-116).  The words
    are laid end to end in one device sequence; ``ks_speculate`` runs the
    speculative lanes and ``ks_scan_range`` the full scans."""
    from . import _native

    ctx = _native.context(0)
    pss_sets = [possible_starting_states(dfa, b, 0) for b in range(N_SYMBOLS)]
    if length <= 13 and dfa.n_expressions <= 16 and dfa.state_count <= 1024:
        # one device thread per (word, border): ks_reconciliation_sweep
        r = ctx.reconciliation_sweep(dfa, pss_sets, length, window)
        return {"length": length, "speculative_runs": int(r[0]), "converged_runs": int(r[1]),
                "count_mismatches": int(r[2]), "final_state_mismatches": int(r[3])}
    # larger automata: words laid end to end, ks_speculate + ks_scan_range per word
    dh = ctx.dfa(dfa)
    words = np.array(list(itertools.product(range(4), repeat=length)), dtype=np.uint8).reshape(-1)
    n_words = 4 ** length
    sh = ctx.upload_codes(words)
    runs = converged = bad_counts = bad_state = 0
    for pss in pss_sets:
        begins = np.arange(n_words, dtype=np.int64) * length
        ends = begins + length
        offs = np.arange(n_words + 1, dtype=np.int64) * pss.size
        data = np.tile(pss, n_words)
        conv, delta = ctx.speculate(dh, sh, begins, ends, offs, data, window, with_delta=True)
        for k in range(n_words):
            b, e = int(begins[k]), int(ends[k])
            c0, last0, _ = ctx.scan_range(dh, sh, b, e, int(pss[0]))
            for i in range(1, pss.size):
                runs += 1
                j = int(conv[offs[k] + i])
                if j < 0:
                    continue
                converged += 1
                full, last, _ = ctx.scan_range(dh, sh, b, e, int(pss[i]))
                if not np.array_equal(full, c0 + delta[offs[k] + i]):
                    bad_counts += 1
                if last != last0:
                    bad_state += 1
    return {"length": length, "speculative_runs": runs, "converged_runs": converged,
            "count_mismatches": bad_counts, "final_state_mismatches": bad_state}
