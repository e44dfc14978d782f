"""Chunked DFA scan engine -- the drop-in for ``kmerscan.engine``.

Public names and semantics follow the reference (`kmerscan/engine.py:1-237`);
the work runs on the GPU through the C ABI (``_native``), never on the CPU:

* ``run`` -> one ``ks_count`` / ``ks_locate`` call over the device-resident
  packed sequence.  Results (counts, sorted ``[end offset, id]`` rows) are
  bit-identical to the reference and independent of ``workers``/``window``,
  as the reference's are (SPEC: "results independent of workers/window").
* ``metadata`` reproduces the reference's keys and values for the requested
  worker plan: its speculative runs are executed by ``ks_speculate`` (warp
  lanes = candidate start states, convergence by ``__match_any_sync``), so
  ``pss_sizes``/``convergence_steps`` are the reference's own numbers.
  Device-side figures are reported separately in ``MatchReport.device_stats``.
* ``match_chunk`` / ``reduce`` / ``possible_starting_states`` keep the
  reference's per-chunk API (used by tests and diagnostics).
"""

from __future__ import annotations

import time
from collections import Counter
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import ReductionChainError
from .alphabet import N_SYMBOLS
from .automaton import START, Dfa
from .ingest import ChunkPlan, Sequence, plan_chunks

DEFAULT_WINDOW = 10

__all__ = [
    "DEFAULT_WINDOW", "EngineConfig", "ChunkResult", "MatchReport", "ReductionChainError",
    "possible_starting_states", "match_chunk", "reduce", "run", "scan_bytes", "sequential_count",
]


@dataclass(frozen=True)
class EngineConfig:
    """``workers``/``window``/``mode`` as in the reference (`engine.py:38-50`);
    ``device`` selects the CUDA device of this process; ``devices`` (a tuple
    of device ids) shards the sequence over several GPUs of this process --
    the reference's workers spread over devices (ks_open_multi: NCCL between
    distinct devices)."""

    workers: int = 1
    window: int = DEFAULT_WINDOW
    mode: str = "count"  # "count" or "locate"
    device: int = 0
    devices: tuple[int, ...] | None = None

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.window < 0:
            raise ValueError("window must be >= 0")
        if self.mode not in ("count", "locate"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.device < 0:
            raise ValueError("device must be >= 0")
        if self.devices is not None:
            if len(self.devices) == 0 or min(int(d) for d in self.devices) < 0:
                raise ValueError("devices must be a non-empty tuple of device ids >= 0")
            object.__setattr__(self, "devices", tuple(int(d) for d in self.devices))


@dataclass(frozen=True)
class ChunkResult:
    """One run over one chunk (reference `engine.py:53-69`)."""

    init_state: int
    last_state: int
    counts: np.ndarray
    converged_at: int | None = None
    locations: np.ndarray | None = None


@dataclass(frozen=True)
class MatchReport:
    per_expression_counts: np.ndarray
    total_count: int
    locations: np.ndarray | None
    metadata: dict = field(default_factory=dict)
    device_stats: dict = field(default_factory=dict)


def possible_starting_states(dfa: Dfa, prev_last: int, first: int) -> np.ndarray:
    """Image of ``prev_last`` over all states, sorted and deduplicated
    (`engine.py:80-91`); OTHER collapses to [START] for built automata."""
    for sym in (prev_last, first):
        if not 0 <= sym < N_SYMBOLS:
            raise ValueError(f"symbol {sym} out of range")
    return np.unique(np.asarray(dfa.transitions)[:, prev_last]).astype(np.int64)


def _ctx(cfg: EngineConfig) -> _native.DeviceContext:
    return _native.context(cfg.device)


def _speculation_metadata(ctx, dh, sh, dfa, seq, plan: ChunkPlan, cfg: EngineConfig) -> dict:
    """Reference metadata (`engine.py:178-203`) for the worker plan, computed
    by the device speculation kernel."""
    pss_sizes = [1]
    steps: Counter = Counter()
    speculative = unconverged = 0
    if plan.worker_count > 1:
        begins, ends, offs, data = [], [], [0], []
        for i in range(1, plan.worker_count):
            prev_last, first = plan.boundary_symbols[i]
            pss = possible_starting_states(dfa, prev_last, first)
            pss_sizes.append(int(pss.size))
            begins.append(plan.bounds[i][0])
            ends.append(plan.bounds[i][1])
            data.append(pss)
            offs.append(offs[-1] + int(pss.size))
        conv, _ = ctx.speculate(dh, sh, begins, ends, offs, np.concatenate(data), cfg.window)
        offs_a = np.asarray(offs, dtype=np.int64)
        spec = np.ones(conv.size, dtype=bool)
        spec[offs_a[:-1]] = False            # R0 (pss[0]) of every chunk is not speculative
        runs = np.asarray(conv)[spec]
        speculative = int(runs.size)
        unconverged = int(np.count_nonzero(runs < 0))
        vals, cnts = np.unique(runs[runs >= 0], return_counts=True)
        steps.update({int(v): int(c) for v, c in zip(vals, cnts)})
    return {
        "input_length": plan.bounds[-1][1],
        "workers": cfg.workers,
        "effective_workers": plan.worker_count,
        "window": cfg.window,
        "mode": cfg.mode,
        "pss_sizes": pss_sizes,
        "speculative_runs": speculative,
        "converged_runs": speculative - unconverged,
        "unconverged_runs": unconverged,
        "convergence_steps": dict(sorted(steps.items())),
    }


def _speculation_metadata_windows(ctx, dfa, seq, plan: ChunkPlan, cfg: EngineConfig) -> dict:
    """The same metadata when the sequence lives sharded over several devices:
    the speculative runs only read the first min(window, chunk length)
    symbols of each chunk, so those windows are uploaded to one device."""
    sym = np.asarray(seq.symbols)
    parts, bounds, pos = [], [(0, 0)], 0
    for i in range(1, plan.worker_count):
        b, e = plan.bounds[i]
        w = sym[b:b + min(cfg.window, e - b)]
        parts.append(w)
        bounds.append((pos, pos + w.size))
        pos += w.size
    if plan.worker_count == 1:
        return _speculation_metadata(ctx, None, None, dfa, seq, plan, cfg)
    sh = ctx.upload_codes(np.concatenate(parts) if pos else np.zeros(0, np.uint8))
    compact = ChunkPlan(plan.worker_count, tuple(bounds), plan.boundary_symbols)
    meta = _speculation_metadata(ctx, ctx.dfa(dfa), sh, dfa, seq, compact, cfg)
    meta["input_length"] = plan.bounds[-1][1]
    return meta


def _run_multi(dfa: Dfa, seq: Sequence, cfg: EngineConfig, plan: ChunkPlan, t0: float) -> MatchReport:
    m = _native.multi_context(cfg.devices)
    dh = m.dfa(dfa)
    key = ("multi",) + cfg.devices
    cache = getattr(seq, "_device", None)
    sh = cache.get(key) if isinstance(cache, dict) else None
    if sh is None:
        sh = m.upload_codes(seq.symbols)
        if isinstance(cache, dict):
            cache[key] = sh
    if cfg.mode == "locate":
        counts, locations = m.locate(dh, sh)
    else:
        counts, locations = m.count(dh, sh), None
    total = int(counts.sum())
    if locations is not None and locations.shape[0] != total:
        raise ReductionChainError(f"{locations.shape[0]} rows for {total} matches")
    dstats = {"devices": list(cfg.devices), "nccl": m.uses_nccl}
    metadata = _speculation_metadata_windows(_native.context(cfg.devices[0]), dfa, seq, plan, cfg)
    metadata["input_name"] = getattr(seq, "source_name", "")
    metadata["elapsed_seconds"] = time.perf_counter() - t0
    return MatchReport(counts, total, locations, metadata, dstats)


def run(dfa: Dfa, seq: Sequence, cfg: EngineConfig = EngineConfig()) -> MatchReport:
    """Scan the whole sequence on the GPU and report counts (and rows)."""
    t0 = time.perf_counter()
    plan = plan_chunks(seq, cfg.workers)
    if cfg.devices is not None:
        return _run_multi(dfa, seq, cfg, plan, t0)
    ctx = _ctx(cfg)
    dh = ctx.dfa(dfa)
    sh = ctx.seq(seq)
    if cfg.mode == "locate":
        counts, locations = ctx.locate(dh, sh)
    else:
        counts, locations = ctx.count(dh, sh), None
    dstats = ctx.stats()
    dstats.update(strategy=dh.info["strategy_name"], stride=dh.info["stride"],
                  sync_depth=dh.info["sync_depth"], monoid_size=dh.info["monoid_size"],
                  device=cfg.device)
    total = int(counts.sum())
    if locations is not None and locations.shape[0] != total:
        raise ReductionChainError(f"{locations.shape[0]} rows for {total} matches")
    metadata = _speculation_metadata(ctx, dh, sh, dfa, seq, plan, cfg)
    metadata["input_name"] = getattr(seq, "source_name", "")
    metadata["elapsed_seconds"] = time.perf_counter() - t0
    return MatchReport(counts, total, locations, metadata, dstats)


def scan_bytes(dfa: Dfa, data, mode: str = "count", device: int = 0, fmt: str = "raw"):
    """Raw or FASTA file bytes (host buffer) -> (counts, rows | None) with the
    ingest on the device: the same result as ``run(dfa, seq)`` for the
    Sequence ``load_sequence`` would build (`ingest.py:54-70`), without the
    host encode.  Counts stream the input through ks_count_host_bytes."""
    if mode not in ("count", "locate"):
        raise ValueError(f"unknown mode {mode!r}")
    if fmt not in ("raw", "fasta"):
        raise ValueError(f"unknown format {fmt!r}")
    ctx = _native.context(device)
    dh = ctx.dfa(dfa)
    if mode == "count":  # pipelined host->device copy, encode and scan
        return ctx.count_host_ascii(dh, data, fasta=fmt == "fasta"), None
    sh = ctx.upload_ascii(data, fasta=fmt == "fasta")
    try:
        return ctx.locate(dh, sh)
    finally:
        sh.free()


def sequential_count(dfa: Dfa, seq: Sequence, device: int = 0) -> np.ndarray:
    """Counts of one pass from the start state (`oracle.py:56-61`)."""
    ctx = _native.context(device)
    return ctx.count(ctx.dfa(dfa), ctx.seq(seq))


def match_chunk(dfa: Dfa, chunk: np.ndarray, global_offset: int, pss,
                cfg: EngineConfig) -> list[ChunkResult]:
    """Full run from pss[0] plus speculative runs from pss[1:]
    (`engine.py:94-134` / `_kernels.py:43-113`), on the device.

    Converged runs carry R0's counts plus the device-computed prefix
    correction and R0's final state; their rows stop at the convergence
    position.  Unconverged runs are full scans from their own start state.
    """
    pss = np.ascontiguousarray(np.asarray(pss, dtype=np.int64))
    if pss.size == 0:
        raise ValueError("pss must be non-empty")
    ctx = _ctx(cfg)
    dh = ctx.dfa(dfa)
    sh = ctx.upload_codes(np.asarray(chunk, dtype=np.uint8))
    m = sh.length
    locate = cfg.mode == "locate"
    counts0, last0, rows0 = ctx.scan_range(dh, sh, 0, m, int(pss[0]), global_offset, locate)
    conv, delta = ctx.speculate(dh, sh, [0], [m], [0, int(pss.size)], pss, cfg.window, with_delta=True)
    results = [ChunkResult(int(pss[0]), last0, counts0, None, rows0)]
    for i in range(1, int(pss.size)):
        j = int(conv[i])
        if j >= 0:
            rows = None
            if locate:
                _, _, rows = ctx.scan_range(dh, sh, 0, j + 1, int(pss[i]), global_offset, True)
            results.append(ChunkResult(int(pss[i]), last0, counts0 + delta[i], j, rows))
        else:
            c, last, rows = ctx.scan_range(dh, sh, 0, m, int(pss[i]), global_offset, locate)
            results.append(ChunkResult(int(pss[i]), last, c, None, rows))
    return results


def reduce(dfa: Dfa, plan: ChunkPlan, per_chunk: list[list[ChunkResult]],
           cfg: EngineConfig) -> MatchReport:
    """Chain per-chunk results into one report (`engine.py:137-204`): chunk
    i's selected run starts where chunk i-1's selected run ended; a converged
    run contributes its prefix rows plus R0's rows past the convergence."""
    if len(per_chunk) != plan.worker_count:
        raise ValueError("per_chunk does not match the plan")
    locate = cfg.mode == "locate"
    counts = np.zeros(dfa.n_expressions, dtype=np.int64)
    parts: list[np.ndarray] = []
    want = START
    for i, results in enumerate(per_chunk):
        if i:
            want = chosen.last_state
        chosen = next((r for r in results if r.init_state == want), None)
        if chosen is None:
            raise ReductionChainError(
                f"chunk {i}: no run starting from state {want} "
                f"(have {[r.init_state for r in results]})")
        counts += chosen.counts
        if locate:
            parts.append(chosen.locations)
            if chosen.converged_at is not None:
                r0 = results[0].locations
                border = plan.bounds[i][0] + chosen.converged_at + 1
                parts.append(r0[r0[:, 0] > border])
    locations = None
    if locate:
        locations = np.concatenate(parts) if parts else np.empty((0, 2), dtype=np.int64)
        locations = locations[np.lexsort((locations[:, 1], locations[:, 0]))]
    total = int(counts.sum())
    assert locations is None or locations.shape[0] == total

    steps: Counter = Counter()
    speculative = unconverged = 0
    for results in per_chunk:
        for r in results[1:]:
            speculative += 1
            if r.converged_at is None:
                unconverged += 1
            else:
                steps[r.converged_at] += 1
    metadata = {
        "input_length": plan.bounds[-1][1],
        "workers": cfg.workers,
        "effective_workers": plan.worker_count,
        "window": cfg.window,
        "mode": cfg.mode,
        "pss_sizes": [len(results) for results in per_chunk],
        "speculative_runs": speculative,
        "converged_runs": speculative - unconverged,
        "unconverged_runs": unconverged,
        "convergence_steps": dict(sorted(steps.items())),
    }
    return MatchReport(counts, total, locations, metadata)
