"""Dense failure-free Aho-Corasick automaton (host side).

``build_dfa`` produces a table bit-identical to the reference builder
(`kmerscan/automaton.py:54-135`):

* state ids are the distinct literal prefixes in breadth-first order with
  children visited a < c < g < t -- i.e. sorted by (length, string); the
  root (empty prefix) is ``START = 0``;
* ``transitions`` is ``int32[|Q|, 5]`` (columns a, c, g, t, OTHER); a missing
  trie edge is densified through the failure link, and the OTHER column
  always returns to START;
* outputs are suffix-closed *multisets* of expression ids in CSR form
  (``out_offsets``/``out_ids``), sorted per state, multiplicity kept.

The automaton is built once on the host (milliseconds).  Its device form --
renumbered, multi-symbol stride tables and the synchronisation analysis -- is
compiled natively by ``ks_dfa_upload`` (csrc/dfa_compile.cpp).
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass

import numpy as np

from .alphabet import BASE_CODES, N_SYMBOLS, OTHER
from .patterns import LiteralTable

START = 0


@dataclass(frozen=True)
class Dfa:
    """Immutable total automaton over the 5-symbol alphabet (start = 0).

    transitions: (state_count, 5) int32, columns a, c, g, t, OTHER.
    out_offsets / out_ids: CSR output multisets (ids sorted per state).
    labels: trie prefix per state (diagnostic only).
    """

    transitions: np.ndarray
    out_offsets: np.ndarray
    out_ids: np.ndarray
    labels: tuple[str, ...]
    n_expressions: int

    start: int = START

    @property
    def state_count(self) -> int:
        return int(self.transitions.shape[0])

    def __post_init__(self):
        for arr in (self.transitions, self.out_offsets, self.out_ids):
            arr.setflags(write=False)


def _csr(lists: list[list[int]]) -> tuple[np.ndarray, np.ndarray]:
    sizes = np.fromiter((len(x) for x in lists), dtype=np.int64, count=len(lists))
    offsets = np.zeros(len(lists) + 1, dtype=np.int32)
    np.cumsum(sizes, out=offsets[1:])
    flat = np.fromiter((e for x in lists for e in x), dtype=np.int32, count=int(sizes.sum()))
    return offsets, flat


def build_dfa(table: LiteralTable) -> Dfa:
    """Literal table -> dense suffix-closed automaton."""
    if not table.literals:
        raise ValueError("cannot build an automaton from an empty literal table")

    # Validate and collect every prefix; endings keyed by the full literal.
    prefixes: set[str] = {""}
    endings: dict[str, list[int]] = {}
    for literal, expr_id in table.literals:
        if not literal:
            raise ValueError("empty literal")
        for ch in literal:
            if ch not in BASE_CODES:
                raise ValueError(f"literal {literal!r} contains non-base character {ch!r}")
        for k in range(1, len(literal) + 1):
            prefixes.add(literal[:k])
        endings.setdefault(literal, []).append(expr_id)

    # BFS order with a<c<g<t children == sort by (depth, string).
    labels = sorted(prefixes, key=lambda p: (len(p), p))
    index = {p: i for i, p in enumerate(labels)}
    n = len(labels)

    trans = np.zeros((n, N_SYMBOLS), dtype=np.int32)
    fail = np.zeros(n, dtype=np.int64)
    # One pass in id order: fail[s] < s, so its row is already dense.
    for s, label in enumerate(labels):
        for code, ch in enumerate("acgt"):
            child = index.get(label + ch)
            if child is None:
                trans[s, code] = trans[fail[s], code] if s else START
            else:
                trans[s, code] = child
                fail[child] = trans[fail[s], code] if s else START
    trans[:, OTHER] = START

    outputs: list[list[int]] = [[] for _ in range(n)]
    for s in range(1, n):
        outputs[s] = sorted(endings.get(labels[s], []) + outputs[fail[s]])

    offsets, ids = _csr(outputs)
    return Dfa(transitions=trans, out_offsets=offsets, out_ids=ids,
               labels=tuple(labels), n_expressions=table.n_expressions)


def step(dfa: Dfa, state: int, symbol: int) -> int:
    """Total transition function with range checks."""
    if not 0 <= state < dfa.state_count:
        raise ValueError(f"state {state} out of range")
    if not 0 <= symbol < N_SYMBOLS:
        raise ValueError(f"symbol {symbol} out of range")
    return int(dfa.transitions[state, symbol])


def outputs_at(dfa: Dfa, state: int) -> tuple[int, ...]:
    """Sorted expression-id multiset emitted on entering ``state``."""
    if not 0 <= state < dfa.state_count:
        raise ValueError(f"state {state} out of range")
    lo, hi = int(dfa.out_offsets[state]), int(dfa.out_offsets[state + 1])
    return tuple(int(e) for e in dfa.out_ids[lo:hi])


def minimize(dfa: Dfa) -> Dfa:
    """Merge output-equivalent states (coarsest stable partition).

    Moore-style refinement reaches the same unique coarsest partition as the
    reference's Hopcroft loop (`kmerscan/automaton.py:162-250`); blocks are
    then renumbered breadth-first from the start block (symbols in column
    order, representative = smallest member), as the reference does.
    """
    n = dfa.state_count
    trans = np.asarray(dfa.transitions, dtype=np.int64)
    keys: dict[tuple[int, ...], int] = {}
    cls = np.fromiter((keys.setdefault(outputs_at(dfa, s), len(keys)) for s in range(n)),
                      dtype=np.int64, count=n)
    n_cls = len(keys)
    while True:
        sig = np.concatenate([cls[:, None], cls[trans]], axis=1)
        _, new_cls = np.unique(sig, axis=0, return_inverse=True)
        new_cls = new_cls.reshape(-1)
        n_new = int(new_cls.max()) + 1
        if n_new == n_cls:
            break
        cls, n_cls = new_cls, n_new

    rep = np.full(n_cls, n, dtype=np.int64)
    np.minimum.at(rep, cls, np.arange(n))
    block_id = {int(cls[START]): 0}
    order = [int(cls[START])]
    queue = deque(order)
    while queue:
        b = queue.popleft()
        r = rep[b]
        for code in range(N_SYMBOLS):
            nb = int(cls[trans[r, code]])
            if nb not in block_id:
                block_id[nb] = len(order)
                order.append(nb)
                queue.append(nb)
    m = len(order)
    new_trans = np.zeros((m, N_SYMBOLS), dtype=np.int32)
    out_lists: list[list[int]] = []
    labels: list[str] = []
    for b in order:
        r = int(rep[b])
        new_trans[block_id[b]] = [block_id[int(cls[trans[r, c]])] for c in range(N_SYMBOLS)]
        out_lists.append(list(outputs_at(dfa, r)))
        labels.append(dfa.labels[r])
    offsets, ids = _csr(out_lists)
    return Dfa(transitions=new_trans, out_offsets=offsets, out_ids=ids,
               labels=tuple(labels), n_expressions=dfa.n_expressions)


def dump_dfa(dfa: Dfa) -> str:
    """TSV: state, label, five targets (a,c,g,t,OTHER), comma-joined outputs."""
    rows = []
    for s in range(dfa.state_count):
        targets = "\t".join(str(int(t)) for t in dfa.transitions[s])
        outs = ",".join(str(e) for e in outputs_at(dfa, s))
        rows.append(f"{s}\t{dfa.labels[s]}\t{targets}\t{outs}")
    return "\n".join(rows) + "\n"
