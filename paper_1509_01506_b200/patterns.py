"""Motif expression dialect: parsing and literal expansion (host side).

Same grammar, ids, expansion order, error classes and error positions as the
reference (`kmerscan/patterns.py:1-260`)::

    expr   := branch ('|' branch)*
    branch := atom+
    atom   := base | '(' base ('|' base)+ ')'
    base   := a | c | g | t          (case-insensitive)

One expression per line; '#' lines and blank lines are skipped; spaces/tabs
are allowed around '|' and at line edges.  Class choices expand in sorted
base order; a branch expanding past the cap raises ``ExpansionLimitError``;
duplicate literals inside one expression are rejected.

The regex-dna motif set the reference compiles in is *not* reproduced in this
repository: ``builtin_expression_set()`` loads it at run time from the file
named by ``$KMERSCAN_BUILTIN_PATTERNS`` or from an importable reference
``kmerscan`` package, and raises ``LookupError`` when neither exists.
"""

from __future__ import annotations

import itertools
import math
import os
from dataclasses import dataclass
from functools import lru_cache

from .alphabet import BASES

DEFAULT_EXPANSION_CAP = 4096

# The reference's informational state count for the regex-dna set built by
# another construction (`kmerscan/patterns.py:42-45`); never asserted.
BUILTIN_DFA_REFERENCE_STATES = 137

_INLINE_WS = " \t"


class PatternSyntaxError(ValueError):
    """Text outside the grammar; ``line``/``column`` are 1-based."""

    def __init__(self, message: str, line: int, column: int):
        super().__init__(f"line {line}, column {column}: {message}")
        self.line = line
        self.column = column


class ExpansionLimitError(ValueError):
    """A single branch would expand to more literals than the cap."""


@dataclass(frozen=True)
class Branch:
    """One alternative: a tuple of atoms, each a string of distinct bases
    in source order (length 1 = plain base, >= 2 = class)."""

    atoms: tuple[str, ...]

    def product_size(self) -> int:
        return math.prod(len(atom) for atom in self.atoms)

    def literals(self):
        choices = [sorted(atom) for atom in self.atoms]
        for combo in itertools.product(*choices):
            yield "".join(combo)


@dataclass(frozen=True)
class Expression:
    id: int
    source: str
    branches: tuple[Branch, ...]


@dataclass(frozen=True)
class ExpressionSet:
    expressions: tuple[Expression, ...]

    def __len__(self) -> int:
        return len(self.expressions)


@dataclass(frozen=True)
class LiteralTable:
    """Flat ``(literal, expression id)`` pairs in expansion order."""

    literals: tuple[tuple[str, int], ...]
    n_expressions: int

    def __len__(self) -> int:
        return len(self.literals)


class _Cursor:
    """Position-tracking reader over one lowercased line."""

    __slots__ = ("text", "lineno", "i")

    def __init__(self, text: str, lineno: int):
        self.text = text
        self.lineno = lineno
        self.i = 0

    def fail(self, message: str, at: int | None = None):
        raise PatternSyntaxError(message, self.lineno, (self.i if at is None else at) + 1)

    def current(self) -> str | None:
        return self.text[self.i] if self.i < len(self.text) else None

    def skip_blanks(self) -> None:
        n = len(self.text)
        while self.i < n and self.text[self.i] in _INLINE_WS:
            self.i += 1


def _read_class(cur: _Cursor) -> str:
    opened_at = cur.i
    cur.i += 1  # '('
    members: list[str] = []
    while True:
        cur.skip_blanks()
        ch = cur.current()
        if ch is None:
            cur.fail("unterminated class", opened_at)
        if ch not in BASES:
            cur.fail(f"unexpected {ch!r} in class, expected a base a/c/g/t")
        if ch in members:
            cur.fail(f"duplicate base {ch!r} in class")
        members.append(ch)
        cur.i += 1
        cur.skip_blanks()
        ch = cur.current()
        if ch == "|":
            cur.i += 1
            continue
        if ch == ")":
            cur.i += 1
            break
        cur.fail("unterminated class" if ch is None else "expected '|' or ')' in class")
    if len(members) < 2:
        cur.fail("class needs at least 2 bases", opened_at)
    return "".join(members)


def _read_branch(cur: _Cursor) -> Branch:
    cur.skip_blanks()
    began = cur.i
    atoms: list[str] = []
    while True:
        ch = cur.current()
        if ch is None or ch == "|" or ch in _INLINE_WS:
            break
        if ch == "(":
            atoms.append(_read_class(cur))
        elif ch in BASES:
            atoms.append(ch)
            cur.i += 1
        else:
            cur.fail(f"unexpected {ch!r}, expected a base a/c/g/t or '('")
    if not atoms:
        cur.fail("empty branch", began)
    return Branch(tuple(atoms))


def _read_expression(line: str, lineno: int) -> tuple[Branch, ...]:
    cur = _Cursor(line, lineno)
    branches = [_read_branch(cur)]
    while True:
        cur.skip_blanks()
        ch = cur.current()
        if ch is None:
            return tuple(branches)
        if ch != "|":
            cur.fail(f"unexpected {ch!r}, expected '|' or end of line")
        cur.i += 1
        branches.append(_read_branch(cur))


def _reject_duplicate_literals(branches: tuple[Branch, ...], lineno: int) -> None:
    if any(b.product_size() > DEFAULT_EXPANSION_CAP for b in branches):
        return  # expand_to_literals refuses the expression anyway
    seen: set[str] = set()
    for lit in itertools.chain.from_iterable(b.literals() for b in branches):
        if lit in seen:
            raise PatternSyntaxError(f"duplicate literal {lit!r} in expression", lineno, 1)
        seen.add(lit)


def parse_expressions(text: str) -> ExpressionSet:
    """Pattern-file text -> ExpressionSet (ids in file order, 0-based)."""
    out: list[Expression] = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        body = raw.strip()
        if not body or body.startswith("#"):
            continue
        line = raw.lower()
        branches = _read_expression(line, lineno)
        _reject_duplicate_literals(branches, lineno)
        out.append(Expression(len(out), line.strip(), branches))
    return ExpressionSet(tuple(out))


def expand_to_literals(exprs: ExpressionSet, cap: int = DEFAULT_EXPANSION_CAP) -> LiteralTable:
    """Cartesian expansion: expressions by id, branches in source order,
    class choices sorted.  Raises ``ExpansionLimitError`` past ``cap``."""
    pairs: list[tuple[str, int]] = []
    for expr in exprs.expressions:
        seen: set[str] = set()
        for branch in expr.branches:
            size = branch.product_size()
            if size > cap:
                raise ExpansionLimitError(
                    f"expression {expr.id} ({expr.source!r}): branch expands to "
                    f"{size} literals, cap is {cap}")
            for lit in branch.literals():
                if lit in seen:
                    raise ValueError(f"expression {expr.id}: duplicate literal {lit!r}")
                seen.add(lit)
                pairs.append((lit, expr.id))
    return LiteralTable(tuple(pairs), len(exprs))


def render_expression(expr: Expression) -> str:
    def atom_text(atom: str) -> str:
        return atom if len(atom) == 1 else "(" + "|".join(atom) + ")"

    return " | ".join("".join(atom_text(a) for a in b.atoms) for b in expr.branches)


def render_expression_set(exprs: ExpressionSet) -> str:
    return "\n".join(render_expression(e) for e in exprs.expressions) + "\n"


def _load_builtin_text() -> str:
    path = os.environ.get("KMERSCAN_BUILTIN_PATTERNS")
    if path:
        with open(path, encoding="utf-8") as fh:
            return fh.read()
    try:  # an importable reference package (never shipped with this repo)
        import kmerscan.patterns as _ref_patterns  # type: ignore
        return _ref_patterns.BUILTIN_PATTERN_TEXT
    except Exception as exc:  # pragma: no cover - environment dependent
        raise LookupError(
            "built-in regex-dna pattern set is not bundled; set "
            "KMERSCAN_BUILTIN_PATTERNS to a pattern file") from exc


def __getattr__(name: str):
    if name == "BUILTIN_PATTERN_TEXT":
        return _load_builtin_text()
    raise AttributeError(name)


@lru_cache(maxsize=1)
def builtin_expression_set() -> ExpressionSet:
    """The regex-dna 8-mer set (9 expressions, 50 literals), loaded at run time."""
    return parse_expressions(_load_builtin_text())
