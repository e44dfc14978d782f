"""Benchmark harness with checksum guards (drop-in for ``kmerscan.bench``).

Same protocol as the reference (`kmerscan/bench.py:68-106`): every scenario
runs one untimed warm-up that pins the counts checksum, then `repetitions`
timed calls; any checksum divergence -- across repetitions, or between
scenarios of one comparison group -- raises ``BenchChecksumError`` before a
single number is reported.  Scenario bodies call the GPU engine.
"""

from __future__ import annotations

import hashlib
import statistics
import time
from dataclasses import dataclass
from typing import Callable

import numpy as np

from .alphabet import OTHER
from .automaton import Dfa
from .engine import EngineConfig, run
from .ingest import Sequence
from .patterns import ExpressionSet

DEFAULT_REPETITIONS = 20


class BenchChecksumError(RuntimeError):
    """Counts diverged between repetitions or between paired scenarios."""


@dataclass(frozen=True)
class Scenario:
    name: str
    workers: int
    fn: Callable[[], np.ndarray]
    group: str = ""


@dataclass(frozen=True)
class BenchResult:
    scenario: str
    workers: int
    repetitions: int
    seconds: tuple[float, ...]
    median_seconds: float
    min_seconds: float
    checksum: str


def counts_checksum(counts) -> str:
    """First 16 hex digits of sha256 over the comma-joined decimal counts."""
    text = ",".join(str(int(c)) for c in counts)
    return hashlib.sha256(text.encode()).hexdigest()[:16]


def synthetic_sequence(length: int, seed: int = 42, other_rate: float = 0.0) -> Sequence:
    """Seeded uniform acgt codes with an optional OTHER admixture (same draws
    as the reference generator, so checksums agree)."""
    rng = np.random.default_rng(seed)
    sym = rng.integers(0, 4, size=length, dtype=np.uint8)
    if other_rate > 0.0:
        sym[rng.random(length) < other_rate] = OTHER
    return Sequence(sym, source_name=f"synthetic(seed={seed},n={length},other={other_rate})")


def bench(scenarios: list[Scenario], repetitions: int = DEFAULT_REPETITIONS) -> list[BenchResult]:
    if repetitions < 1:
        raise ValueError("repetitions must be >= 1")
    out: list[BenchResult] = []
    pinned: dict[str, tuple[str, str]] = {}
    for sc in scenarios:
        expect = counts_checksum(sc.fn())
        times = []
        for rep in range(repetitions):
            t0 = time.perf_counter()
            got = counts_checksum(sc.fn())
            times.append(time.perf_counter() - t0)
            if got != expect:
                raise BenchChecksumError(f"{sc.name}: repetition {rep} checksum {got} != {expect}")
        if sc.group:
            first = pinned.setdefault(sc.group, (sc.name, expect))
            if first[1] != expect:
                raise BenchChecksumError(
                    f"group {sc.group!r}: {sc.name} checksum {expect} != {first[0]} checksum {first[1]}")
        out.append(BenchResult(sc.name, sc.workers, repetitions, tuple(times), statistics.median(times),
                               min(times), expect))
    return out


def input_scan_scenario(dfa: Dfa, seq: Sequence, workers: int, window: int, group: str = "") -> Scenario:
    cfg = EngineConfig(workers=workers, window=window)
    return Scenario(f"input-based/w{workers}", workers, lambda: run(dfa, seq, cfg).per_expression_counts,
                    group)


def pattern_scan_scenario(exprs: ExpressionSet, seq: Sequence, workers: int, group: str = "") -> Scenario:
    from .oracle_api import pattern_parallel_count

    return Scenario(f"pattern-based/w{workers}", workers,
                    lambda: pattern_parallel_count(exprs, seq, workers), group)
