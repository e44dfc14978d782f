"""Exhaustive reconciliation sweep on the device (ks_reconciliation_sweep)
against the REAL reference's results on the toy automaton
(tests/golden/reconcile_toy.json from tests/golden/make_reconcile_golden.py;
reference tests/test_acceptance.py:169-181 -- chunk lengths 1-12,
178,956,960 speculative runs, 178,956,956 converged, 0 mismatches,
pkg/test_output.txt:22 -- and tests/test_oracle_bench.py:62-73)."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_1509_01506_b200 as ks
from paper_1509_01506_b200 import _native

pytestmark = pytest.mark.gpu
GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "reconcile_toy.json").read_text())


def test_fixture_totals():
    runs = sum(r["speculative_runs"] for r in GOLDEN["window10"])
    conv = sum(r["converged_runs"] for r in GOLDEN["window10"])
    assert (runs, conv) == (178_956_960, 178_956_956)


@pytest.mark.parametrize("length", range(1, 13))
def test_sweep_matches_reference(toy_dfa, length):
    r = ks.exhaustive_reconciliation_check(toy_dfa, length, window=10)
    assert r == GOLDEN["window10"][length - 1]


def test_sweep_window_zero(toy_dfa):
    assert ks.exhaustive_reconciliation_check(toy_dfa, 3, window=0) == GOLDEN["window0_len3"]


def test_sweep_all_states_as_candidates(toy_dfa):
    """Every state as a candidate for every border (a superset of the
    reference's sets): every run is counted, reconciliation still exact."""
    ctx = _native.context(0)
    pss_all = [np.arange(toy_dfa.state_count)] * 5
    r = ctx.reconciliation_sweep(toy_dfa, pss_all, 5, 10)
    assert r[0] == 5 * (toy_dfa.state_count - 1) * 4**5
    assert 0 < r[1] <= r[0] and r[2] == 0 and r[3] == 0


def test_sweep_permutation_automaton_never_converges():
    """C5's G-counter: candidate runs never meet R0 within the window."""
    from paper_1509_01506_b200 import workloads

    perm = workloads.permutation_dfa(64)
    r = ks.exhaustive_reconciliation_check(perm, 6, window=10)
    assert r["speculative_runs"] == 4 * 63 * 4**6 and r["converged_runs"] == 0
