"""Host-side API parity (no GPU): alphabet, patterns, automaton, ingest,
engine helpers.  Mirrors the reference's unit tests (pkg/tests/test_ingest.py,
test_patterns.py, test_automaton.py, host parts of test_engine.py) and checks
the automaton builder bit-for-bit against tables produced by the reference
(tests/golden/dfas.npz)."""

import itertools

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_1509_01506_b200 as ks
from paper_1509_01506_b200 import patterns as P
from paper_1509_01506_b200.alphabet import BYTE_CODES, DROP, OTHER, encode_bytes
from paper_1509_01506_b200.automaton import START

from conftest import GOLDEN


def dfa_from(text):
    return ks.build_dfa(ks.expand_to_literals(ks.parse_expressions(text)))


# ------------------------------------------------------------------ alphabet

class TestAlphabet:
    def test_byte_classification_exhaustive(self):
        for byte in range(256):
            ch = chr(byte)
            code = BYTE_CODES[byte]
            if ch.lower() in "acgt":
                assert code == "acgt".index(ch.lower())
            elif byte in b" \t\r\n":
                assert code == DROP
            else:
                assert code == OTHER

    def test_encode_drops_whitespace(self):
        assert encode_bytes(b"a c\tg\nt\r").tolist() == [0, 1, 2, 3]

    def test_ambiguity_and_non_ascii(self):
        assert ks.encode("acgtNnxu7").tolist() == [0, 1, 2, 3, 4, 4, 4, 4, 4]
        assert ks.encode("aég").tolist() == [0, OTHER, 2]

    def test_decode(self):
        assert ks.decode(ks.encode("acgtn")) == "acgt?"

    def test_table_immutable(self):
        with pytest.raises(ValueError):
            BYTE_CODES[0] = 0


# ------------------------------------------------------------------ ingest

class TestIngest:
    def test_detect_format(self):
        assert ks.detect_format("genome.fa") == "fasta"
        assert ks.detect_format("GENOME.FASTA") == "fasta"
        assert ks.detect_format("genome.txt") == "raw"

    def test_fasta_drops_headers(self, tmp_path):
        p = tmp_path / "x.fa"
        p.write_bytes(b">chr1 test\nacgt\r\nACGT\r>chr2\nnn\n")
        seq = ks.load_sequence(p, "fasta")
        assert seq.symbols.tolist() == [0, 1, 2, 3, 0, 1, 2, 3, 4, 4]
        assert seq.source_name == str(p)

    def test_raw_keeps_header_bytes_as_other(self, tmp_path):
        p = tmp_path / "x.txt"
        p.write_bytes(b">a\ncg\n")
        assert ks.load_sequence(p, "raw").symbols.tolist() == [OTHER, 0, 1, 2]

    def test_empty_and_bad_format(self, tmp_path):
        p = tmp_path / "e.fa"
        p.write_bytes(b"")
        assert ks.load_sequence(p).length == 0
        with pytest.raises(ValueError):
            ks.load_sequence(p, "fastq")

    def test_symbols_read_only(self):
        seq = ks.sequence_from_text("acgt")
        with pytest.raises(ValueError):
            seq.symbols[0] = 3

    def test_chunk_plans(self):
        assert ks.plan_chunks(ks.sequence_from_text("acgtacgtac"), 4).bounds == \
            ((0, 2), (2, 4), (4, 6), (6, 10))
        plan = ks.plan_chunks(ks.sequence_from_text("acg"), 16)
        assert plan.worker_count == 3 and plan.bounds == ((0, 1), (1, 2), (2, 3))
        plan = ks.plan_chunks(ks.sequence_from_text(""), 7)
        assert plan.worker_count == 1 and plan.bounds == ((0, 0),) and plan.boundary_symbols == (None,)
        assert ks.plan_chunks(ks.sequence_from_text("acgtn"), 2).boundary_symbols == (None, (1, 2))
        with pytest.raises(ValueError):
            ks.plan_chunks(ks.sequence_from_text("acgt"), 0)

    @given(st.integers(0, 300), st.integers(1, 40), st.randoms())
    @settings(max_examples=60, deadline=None)
    def test_partition_invariants(self, n, workers, rnd):
        seq = ks.sequence_from_text("".join(rnd.choice("acgtn") for _ in range(n)))
        plan = ks.plan_chunks(seq, workers)
        assert plan.bounds[0][0] == 0 and plan.bounds[-1][1] == n
        for (a0, a1), (b0, b1) in zip(plan.bounds, plan.bounds[1:]):
            assert a1 == b0 and a1 > a0
        for i in range(1, plan.worker_count):
            lo = plan.bounds[i][0]
            assert plan.boundary_symbols[i] == (seq.symbols[lo - 1], seq.symbols[lo])


# ------------------------------------------------------------------ patterns

class TestPatterns:
    def test_parse_basics(self):
        e = ks.parse_expressions("c(a|t)t | agg").expressions[0]
        assert [b.atoms for b in e.branches] == [("c", "at", "t"), ("a", "g", "g")]
        assert ks.parse_expressions("(t|a)c").expressions[0].branches[0].atoms == ("ta", "c")
        exprs = ks.parse_expressions("acg\n\n# c\ncat\n")
        assert [x.id for x in exprs.expressions] == [0, 1]
        assert [x.source for x in exprs.expressions] == ["acg", "cat"]
        assert len(ks.parse_expressions("# only\n\n")) == 0

    @pytest.mark.parametrize("text,fragment", [
        ("acg|", "empty branch"), ("|acg", "empty branch"),
        ("ac g", "expected '|' or end of line"), ("axg", "expected a base"),
        ("a(g)t", "class needs at least 2 bases"), ("a(g|g)t", "duplicate base"),
        ("a(g|c", "unterminated class"), ("a(g|x)t", "in class"), ("a()t", "in class"),
        ("aa|aa", "duplicate literal"), ("(a|c)t|at", "duplicate literal"),
    ])
    def test_syntax_errors(self, text, fragment):
        with pytest.raises(ks.PatternSyntaxError) as exc:
            ks.parse_expressions(text)
        assert fragment in str(exc.value)

    def test_error_position(self):
        with pytest.raises(ks.PatternSyntaxError) as exc:
            ks.parse_expressions("acg\ncat\ncxt\n")
        assert (exc.value.line, exc.value.column) == (3, 2)

    def test_expansion(self):
        table = ks.expand_to_literals(ks.parse_expressions("aggg(a|c|g)aaa|ttt(c|g|t)ccct"))
        assert [lit for lit, _ in table.literals] == [
            "agggaaaa", "agggcaaa", "aggggaaa", "tttcccct", "tttgccct", "ttttccct"]
        table = ks.expand_to_literals(ks.parse_expressions("acg\nc(a|t)t\n"))
        assert table.literals == (("acg", 0), ("cat", 1), ("ctt", 1)) and table.n_expressions == 2
        exprs = ks.parse_expressions("(a|c)(a|c)|(a|g)")
        with pytest.raises(ks.ExpansionLimitError):
            ks.expand_to_literals(exprs, cap=2)
        assert len(ks.expand_to_literals(exprs, cap=4)) == 6
        assert len(ks.expand_to_literals(ks.parse_expressions("(a|c|g|t)" * 6))) == 4096
        with pytest.raises(ks.ExpansionLimitError):
            ks.expand_to_literals(ks.parse_expressions("(a|c|g|t)" * 7))

    def test_render_round_trip(self):
        text = "c(t|a)t | agg\n(a|c|g)gggtaaa\n"
        exprs = ks.parse_expressions(text)
        assert P.render_expression(exprs.expressions[0]) == "c(t|a)t | agg"
        again = ks.parse_expressions(ks.render_expression_set(exprs))
        assert [e.branches for e in again.expressions] == [e.branches for e in exprs.expressions]


# ------------------------------------------------------------------ automaton

def golden_dfas():
    z = np.load(GOLDEN / "dfas.npz")
    for i, text in enumerate(z["texts"]):
        yield str(text), {k: z[f"{k}_{i}"] for k in ("t", "off", "ids", "labels", "min_t", "min_ids", "dump")}


class TestAutomaton:
    def test_matches_reference_tables(self):
        n = 0
        for text, g in golden_dfas():
            d = dfa_from(text)
            assert np.array_equal(d.transitions, g["t"]), text
            assert np.array_equal(d.out_offsets, g["off"]), text
            assert np.array_equal(d.out_ids, g["ids"]), text
            assert list(d.labels) == [str(x) for x in g["labels"]]
            assert ks.dump_dfa(d) == str(g["dump"])
            m = ks.minimize(d)
            assert np.array_equal(m.transitions, g["min_t"]) and np.array_equal(m.out_ids, g["min_ids"])
            n += 1
        assert n >= 10

    def test_structure(self, toy_dfa, toy_table):
        prefixes = {lit[:k] for lit, _ in toy_table.literals for k in range(1, len(lit) + 1)}
        assert toy_dfa.state_count == 1 + len(prefixes) == 12
        assert list(toy_dfa.labels[1:4]) == ["a", "c", "t"]
        assert (toy_dfa.transitions[:, OTHER] == START).all()
        with pytest.raises(ValueError):
            toy_dfa.transitions[0, 0] = 1
        with pytest.raises(ValueError):
            ks.build_dfa(ks.LiteralTable((), 0))

    def test_longest_suffix_rule(self, toy_dfa):
        idx = {label: s for s, label in enumerate(toy_dfa.labels)}
        for s, label in enumerate(toy_dfa.labels):
            for code, ch in enumerate("acgt"):
                word = label + ch
                expect = next(word[i:] for i in range(len(word) + 1) if word[i:] in idx)
                assert ks.step(toy_dfa, s, code) == idx[expect]

    def test_outputs_multiset(self):
        d = dfa_from("a|aa")
        idx = {label: s for s, label in enumerate(d.labels)}
        assert ks.outputs_at(d, idx["aa"]) == (0, 0)
        d = dfa_from("aa\na")
        idx = {label: s for s, label in enumerate(d.labels)}
        assert ks.outputs_at(d, idx["aa"]) == (0, 1)

    def test_step_range_checks(self, toy_dfa):
        for bad in ((-1, 0), (toy_dfa.state_count, 0), (0, 5)):
            with pytest.raises(ValueError):
                ks.step(toy_dfa, *bad)

    def test_dump_golden(self):
        assert ks.dump_dfa(dfa_from("a")) == "0\t\t1\t0\t0\t0\t0\t\n1\ta\t1\t0\t0\t0\t0\t0\n"

    @given(st.lists(st.text(alphabet="acgt", min_size=1, max_size=6), min_size=1, max_size=6, unique=True))
    @settings(max_examples=40, deadline=None)
    def test_minimize_idempotent(self, lits):
        d = dfa_from("\n".join(lits))
        m = ks.minimize(d)
        assert ks.minimize(m).state_count == m.state_count <= d.state_count


# ------------------------------------------------------------------ engine host parts

class TestEngineHost:
    def test_config(self):
        cfg = ks.EngineConfig()
        assert (cfg.workers, cfg.window, cfg.mode) == (1, 10, "count")
        for kwargs in ({"workers": 0}, {"window": -1}, {"mode": "stream"}, {"device": -1}):
            with pytest.raises(ValueError):
                ks.EngineConfig(**kwargs)

    def test_pss(self, toy_dfa):
        for sym in range(4):
            assert ks.possible_starting_states(toy_dfa, sym, 0).tolist() == \
                sorted(set(int(s) for s in toy_dfa.transitions[:, sym]))
        assert ks.possible_starting_states(toy_dfa, OTHER, 0).tolist() == [START]
        labels = [toy_dfa.labels[s] for s in ks.possible_starting_states(toy_dfa, 2, 0)]
        assert labels == ["", "acg"]
        with pytest.raises(ValueError):
            ks.possible_starting_states(toy_dfa, 5, 0)

    def test_reduce_chain_break(self, toy_dfa):
        seq = ks.sequence_from_text("aaaa")
        plan = ks.plan_chunks(seq, 2)
        cfg = ks.EngineConfig(workers=2)
        z = np.zeros(4, dtype=np.int64)
        good = [ks.ChunkResult(0, 1, z)]
        bad = [ks.ChunkResult(5, 5, z)]
        with pytest.raises(ks.ReductionChainError):
            ks.reduce(toy_dfa, plan, [good, bad], cfg)

    def test_reduce_splice(self, toy_dfa):
        # chunk 1's selected run converged at 0: its prefix rows + R0's later rows
        seq = ks.sequence_from_text("acgacg")
        plan = ks.plan_chunks(seq, 2)
        cfg = ks.EngineConfig(workers=2, mode="locate")
        c = lambda *v: np.array(v, dtype=np.int64)
        r0_0 = ks.ChunkResult(0, 7, c(1, 0, 0, 0), None, np.array([[3, 0]]))
        r1_0 = ks.ChunkResult(0, 9, c(1, 0, 0, 0), None, np.array([[6, 0]]))
        r1_7 = ks.ChunkResult(7, 9, c(1, 0, 0, 0), 0, np.empty((0, 2), np.int64))
        rep = ks.reduce(toy_dfa, plan, [[r0_0], [r1_0, r1_7]], cfg)
        assert rep.per_expression_counts.tolist() == [2, 0, 0, 0]
        assert rep.locations.tolist() == [[3, 0], [6, 0]]
        assert rep.metadata["convergence_steps"] == {0: 1}


def test_engine_config_devices_validation():
    with pytest.raises(ValueError):
        ks.EngineConfig(devices=())
    with pytest.raises(ValueError):
        ks.EngineConfig(devices=(0, -1))
    assert ks.EngineConfig(devices=[1, 0]).devices == (1, 0)
