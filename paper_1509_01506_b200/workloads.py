"""Seeded synthetic workloads C1..C5 (BASELINE.json configs).

The paper's GenBank genomes are not available; these generators stand in with
the configs' shapes, sizes and value distributions.  Every config k draws its
sequence from ``default_rng([1509, k, 0])`` and its patterns from
``default_rng([1509, k, 1])``; ``n`` may be reduced for tests (same
distributions, shorter draw).  Sequences are returned as raw ASCII bytes
(uppercase bases, lowercase = soft-masked, 'N' runs), i.e. the form the device
encoder consumes.

C1  1 MiB uniform ACGT; 4 distinct 4-mers.
C2  64 MiB, GC 0.41, 5% soft-mask runs (mean 300); 32 distinct 8-mers.
C3  1 GiB, GC 0.41, 1% N runs (mean 10,000); 256 expressions of length 6-12
    with 1-2 positions replaced by a 2-base class.
C4  3.2e9, order-3 Markov chain (GC 0.405-0.415), 2% N runs (mean 50,000),
    50% soft-mask runs (mean 1,000); 64 distinct 12-mers.
C5  256 MiB uniform ACGT; hand-built 1024-state "G count mod 1024" DFA.
"""

from __future__ import annotations

import itertools
import os
from dataclasses import dataclass

import numpy as np

from .automaton import Dfa, build_dfa
from .patterns import expand_to_literals, parse_expressions

FULL_SIZES = {1: 1 << 20, 2: 64 << 20, 3: 1 << 30, 4: 3_200_000_000, 5: 256 << 20}
ASCII_UPPER = np.frombuffer(b"ACGT", dtype=np.uint8)
_BLOCK = 64 << 20


@dataclass
class Workload:
    config: int
    n: int
    dfa: Dfa
    pattern_text: str | None
    ascii: np.ndarray          # uint8 raw bytes (no whitespace)
    description: str


def _rng(k: int, stream: int) -> np.random.Generator:
    return np.random.default_rng([1509, k, stream])


def _iid_codes(rng, n: int, gc: float | None) -> np.ndarray:
    """i.i.d. base codes 0..3 (uniform, or GC-biased: P(C)=P(G)=gc/2)."""
    out = np.empty(n, dtype=np.uint8)
    if gc is None:
        for lo in range(0, n, _BLOCK):
            hi = min(n, lo + _BLOCK)
            out[lo:hi] = rng.integers(0, 4, hi - lo, dtype=np.uint8)
        return out
    probs = np.array([(1 - gc) / 2, gc / 2, gc / 2, (1 - gc) / 2])
    lut = np.searchsorted(np.cumsum(probs) * 65536, np.arange(65536), side="right").astype(np.uint8)
    lut = np.minimum(lut, 3)
    for lo in range(0, n, _BLOCK):
        hi = min(n, lo + _BLOCK)
        out[lo:hi] = lut[rng.integers(0, 65536, hi - lo, dtype=np.uint16)]
    return out


def _to_ascii(codes: np.ndarray) -> np.ndarray:
    """codes 0..3 -> b"ACGT" (threaded gather in 64 MiB pieces)."""
    from concurrent.futures import ThreadPoolExecutor

    out = np.empty(codes.size, dtype=np.uint8)

    def piece(lo):
        np.take(ASCII_UPPER, codes[lo:lo + _BLOCK], out=out[lo:lo + _BLOCK])

    with ThreadPoolExecutor(min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(piece, range(0, codes.size, _BLOCK)))
    return out


def _runs(rng, n: int, frac: float, mean: float) -> list[tuple[int, int]]:
    """Alternating renewal process: geometric gaps (mean mean*(1-f)/f) and
    runs (mean `mean`) covering about `frac` of [0, n)."""
    gap_mean = mean * (1 - frac) / frac
    est = int(n / (mean + gap_mean) * 1.3) + 16
    spans: list[tuple[int, int]] = []
    pos = 0
    while pos < n:
        gaps = rng.geometric(1.0 / gap_mean, est)
        lens = rng.geometric(1.0 / mean, est)
        starts = pos + np.cumsum(gaps) + np.concatenate([[0], np.cumsum(lens)[:-1]])
        ends = starts + lens
        keep = starts < n
        for s, e in zip(starts[keep], ends[keep]):
            spans.append((int(s), int(min(e, n))))
        pos = int(ends[-1]) if keep.all() else n
    return spans


def _apply_spans(buf: np.ndarray, spans, fn) -> None:
    for s, e in spans:
        buf[s:e] = fn(buf[s:e])


def _distinct_kmers(rng, count: int, k: int) -> list[str]:
    seen: list[str] = []
    have = set()
    while len(seen) < count:
        kmer = "".join("acgt"[int(x)] for x in rng.integers(0, 4, k))
        if kmer not in have:
            have.add(kmer)
            seen.append(kmer)
    return seen


def config3_patterns(rng) -> str:
    """256 expressions, L ~ U{6..12}, 1-2 positions replaced by a 2-base class."""
    pairs = list(itertools.combinations("acgt", 2))
    lines = []
    for _ in range(256):
        L = int(rng.integers(6, 13))
        atoms = ["acgt"[int(x)] for x in rng.integers(0, 4, L)]
        k = int(rng.integers(1, 3))
        for p in rng.choice(L, size=k, replace=False):
            a, b = pairs[int(rng.integers(0, 6))]
            atoms[int(p)] = f"({a}|{b})"
        lines.append("".join(atoms))
    return "\n".join(lines) + "\n"


def permutation_dfa(n_states: int = 1024) -> Dfa:
    """C5: A/C/T keep the state, G advances it mod n_states, OTHER resets;
    state 0 emits expression 0 every time it is entered."""
    s = np.arange(n_states, dtype=np.int32)
    trans = np.stack([s, s, (s + 1) % n_states, s, np.zeros_like(s)], axis=1).astype(np.int32)
    off = np.ones(n_states + 1, dtype=np.int32)
    off[0] = 0
    return Dfa(transitions=trans, out_offsets=off, out_ids=np.zeros(1, dtype=np.int32),
               labels=tuple(str(i) for i in range(n_states)), n_expressions=1)


def _markov3(rng, n: int) -> np.ndarray:
    """Order-3 Markov chain with Dirichlet(20*[.295,.205,.205,.295]) rows,
    redrawn until the stationary GC is within [0.405, 0.415]."""
    alpha = 20 * np.array([0.295, 0.205, 0.205, 0.295])
    while True:
        P = rng.dirichlet(alpha, size=64)
        M = np.zeros((64, 64))
        for ctx in range(64):
            for b in range(4):
                M[ctx, ((ctx << 2) | b) & 63] = P[ctx, b]
        w, v = np.linalg.eig(M.T)
        pi = np.real(v[:, np.argmin(np.abs(w - 1))])
        pi = pi / pi.sum()
        gc = sum(pi[c] * (P[c, 1] + P[c, 2]) for c in range(64))
        if 0.405 <= gc <= 0.415:
            break
    cdf = np.cumsum(P, axis=1)
    out = np.empty(n, dtype=np.uint8)
    try:  # compiled loop when numba is present (it is in this image)
        from numba import njit

        @njit(cache=False, nogil=True)
        def walk(u, cdf, out, ctx):
            # b = first index with r < cdf[ctx, b] (cdf rows are increasing),
            # counted branch-free
            for i in range(u.shape[0]):
                r = u[i]
                b = (r >= cdf[ctx, 0]) + (r >= cdf[ctx, 1]) + (r >= cdf[ctx, 2])
                out[i] = b
                ctx = ((ctx << 2) | b) & 63
            return ctx

        from concurrent.futures import ThreadPoolExecutor

        # the next block's uniforms are drawn (numpy releases the GIL) while
        # the compiled walk consumes this one; the stream is consumed in order
        ctx = 0
        blocks = [(lo, min(n, lo + _BLOCK)) for lo in range(0, n, _BLOCK)]
        with ThreadPoolExecutor(1) as ex:
            nxt = ex.submit(rng.random, blocks[0][1] - blocks[0][0]) if blocks else None
            for i, (lo, hi) in enumerate(blocks):
                u = nxt.result()
                if i + 1 < len(blocks):
                    nxt = ex.submit(rng.random, blocks[i + 1][1] - blocks[i + 1][0])
                ctx = walk(u, cdf, out[lo:hi], ctx)
    except ImportError:  # pragma: no cover
        ctx = 0
        u = rng.random(n)
        for i in range(n):
            b = int(np.searchsorted(cdf[ctx], u[i], side="right"))
            out[i] = min(b, 3)
            ctx = ((ctx << 2) | out[i]) & 63
    return out


def make(k: int, n: int | None = None, shard: int = 0) -> Workload:
    """Build workload C<k> (optionally with a shorter sequence of length n).

    ``shard`` > 0 draws another independent slice of the same distribution
    (sequence stream ``[1509, k, 0, shard]``; the patterns are shared) -- the
    per-rank slices of the weak-scaling multi-GPU runs.
    """
    n = FULL_SIZES[k] if n is None else int(n)
    srng = _rng(k, 0) if shard == 0 else np.random.default_rng([1509, k, 0, shard])
    prng = _rng(k, 1)
    text = None
    if k == 1:
        codes = _iid_codes(srng, n, None)
        text = "\n".join(_distinct_kmers(prng, 4, 4)) + "\n"
        desc = "1 MiB uniform ACGT, 4 distinct 4-mers"
    elif k == 2:
        codes = _iid_codes(srng, n, 0.41)
        text = "\n".join(_distinct_kmers(prng, 32, 8)) + "\n"
        desc = "64 MiB GC 0.41, 5% soft-mask runs (mean 300), 32 distinct 8-mers"
    elif k == 3:
        codes = _iid_codes(srng, n, 0.41)
        text = config3_patterns(prng)
        desc = "1 GiB GC 0.41, 1% N runs (mean 10k), 256 class patterns of length 6-12"
    elif k == 4:
        codes = _markov3(srng, n)
        text = "\n".join(_distinct_kmers(prng, 64, 12)) + "\n"
        desc = "3.2e9 order-3 Markov GC~0.41, 2% N runs (mean 50k), 50% soft-mask (mean 1k), 64 12-mers"
    elif k == 5:
        codes = _iid_codes(srng, n, None)
        desc = "256 MiB uniform ACGT, 1024-state permutation DFA"
    else:
        raise ValueError("config must be 1..5")
    ascii_ = _to_ascii(codes)
    del codes
    if k == 2:
        _apply_spans(ascii_, _runs(srng, n, 0.05, 300), lambda b: b | 0x20)
    elif k == 3:
        _apply_spans(ascii_, _runs(srng, n, 0.01, 10_000), lambda b: np.full_like(b, ord("N")))
    elif k == 4:
        _apply_spans(ascii_, _runs(srng, n, 0.50, 1_000), lambda b: b | 0x20)
        _apply_spans(ascii_, _runs(srng, n, 0.02, 50_000), lambda b: np.full_like(b, ord("N")))
    dfa = permutation_dfa() if k == 5 else build_dfa(expand_to_literals(parse_expressions(text)))
    return Workload(k, n, dfa, text, ascii_, desc)
