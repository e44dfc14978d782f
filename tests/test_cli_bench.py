"""Drop-in CLI and bench harness (reference pkg/tests/test_cli.py,
test_oracle_bench.py).  Harness-logic tests run on CPU; anything that scans
runs on the GPU (marked)."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_1509_01506_b200 as ks
from paper_1509_01506_b200 import cli

TOY = "acg\ncat\ncta\ntta\n"


@pytest.fixture()
def files(tmp_path):
    pats = tmp_path / "pats.txt"
    pats.write_text(TOY)
    fa = tmp_path / "tiny.fa"
    fa.write_text(">s1 demo\nctacat\n")
    return {"patterns": str(pats), "fasta": str(fa), "dir": tmp_path}


def run_cli(capsys, argv):
    code = cli.main(argv)
    cap = capsys.readouterr()
    return code, cap.out, cap.err


# ------------------------------------------------------------------ CPU

def constant(name="s", workers=1, value=7, group=""):
    return ks.Scenario(name, workers, lambda: np.array([value]), group)


class TestHarness:
    def test_shape_and_median(self):
        (r,) = ks.bench([constant()], repetitions=5)
        assert r.repetitions == 5 and len(r.seconds) == 5
        assert min(r.seconds) <= r.median_seconds <= max(r.seconds) and r.min_seconds == min(r.seconds)

    def test_warmup_not_timed(self):
        calls = []
        ks.bench([ks.Scenario("s", 1, lambda: (calls.append(1), np.array([1]))[1])], repetitions=3)
        assert len(calls) == 4

    def test_unstable_and_group_mismatch_rejected(self):
        state = {"n": 0}

        def flaky():
            state["n"] += 1
            return np.array([state["n"]])

        with pytest.raises(ks.BenchChecksumError):
            ks.bench([ks.Scenario("flaky", 1, flaky)], repetitions=3)
        with pytest.raises(ks.BenchChecksumError):
            ks.bench([constant("a", value=1, group="g"), constant("b", value=2, group="g")], repetitions=1)
        with pytest.raises(ValueError):
            ks.bench([constant()], repetitions=0)

    def test_checksum(self):
        a = ks.counts_checksum(np.array([1, 2, 3]))
        assert a == ks.counts_checksum(np.array([1, 2, 3], dtype=np.int32))
        assert a != ks.counts_checksum(np.array([1, 2, 4]))
        assert ks.counts_checksum([2056, 6144, 6194, 6145, 6224, 5951, 6078, 6289, 6156]) == "65ef91881aebcb08"

    def test_synthetic_sequence(self):
        a = ks.synthetic_sequence(10_000, seed=1)
        assert (a.symbols == ks.synthetic_sequence(10_000, seed=1).symbols).all()
        assert a.symbols.max() <= 3
        share = (ks.synthetic_sequence(5_000, seed=9, other_rate=0.5).symbols == 4).mean()
        assert 0.4 < share < 0.6


class TestNaive:
    def test_overlaps_and_order(self):
        table = ks.expand_to_literals(ks.parse_expressions("aca"))
        counts, loc = ks.naive_count(table, ks.sequence_from_text("acaca"))
        assert counts.tolist() == [2] and loc.tolist() == [[3, 0], [5, 0]]
        table = ks.expand_to_literals(ks.parse_expressions("ta\ncta"))
        assert ks.naive_count(table, ks.sequence_from_text("cta"))[1].tolist() == [[3, 0], [3, 1]]
        counts, loc = ks.naive_count(table, ks.sequence_from_text(""))
        assert counts.tolist() == [0, 0] and loc.shape == (0, 2)


class TestCliParsing:
    def test_sizes(self):
        assert cli.parse_size("64") == 64 and cli.parse_size("2k") == 2048
        assert cli.parse_size("64M") == 64 << 20 and cli.parse_size("1G") == 1 << 30
        with pytest.raises(Exception):
            cli.parse_size("64Q")

    def test_usage_errors_exit_2(self, files):
        for argv in (["count", "--input", files["fasta"]],
                     ["count", "--patterns", files["patterns"], "--builtin-patterns", "--input", files["fasta"]],
                     ["count", "--patterns", files["patterns"], "--input", files["fasta"], "--workers", "0"]):
            with pytest.raises(SystemExit) as exc:
                cli.main(argv)
            assert exc.value.code == 2

    def test_bad_pattern_file_exit_1(self, capsys, files):
        bad = files["dir"] / "bad.txt"
        bad.write_text("ac(g\n")
        code, out, err = run_cli(capsys, ["count", "--patterns", str(bad), "--input", files["fasta"]])
        assert code == 1 and out == "" and "line 1" in err

    def test_missing_input_exit_1(self, capsys, files):
        code, out, err = run_cli(capsys, ["count", "--patterns", files["patterns"], "--input", "/no/such"])
        assert code == 1 and out == "" and "kmerscan:" in err

    def test_dump_dfa(self, capsys, files):
        code, out, _ = run_cli(capsys, ["dump-dfa", "--patterns", files["patterns"]])
        assert code == 0 and "# dfa_states\t12" in out and "reference_states" not in out
        assert len(out.splitlines()) == 4 + 12


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
class TestCliScans:
    def test_count_tsv_golden(self, capsys, files):
        code, out, err = run_cli(capsys, ["count", "--patterns", files["patterns"], "--input", files["fasta"],
                                          "--workers", "4"])
        assert code == 0 and err == ""
        assert out == ("expression_index\texpression_source\tcount\n0\tacg\t0\n1\tcat\t1\n2\tcta\t1\n"
                       "3\ttta\t0\nTOTAL\t\t2\n")

    def test_count_json(self, capsys, files):
        code, out, _ = run_cli(capsys, ["count", "--patterns", files["patterns"], "--input", files["fasta"],
                                        "--output-format", "json"])
        doc = json.loads(out)
        assert doc["total"] == 2 and [e["count"] for e in doc["expressions"]] == [0, 1, 1, 0]
        assert doc["metadata"]["input_length"] == 6 and "elapsed_seconds" not in doc["metadata"]
        assert "locations" not in doc

    def test_locate(self, capsys, files):
        code, out, _ = run_cli(capsys, ["locate", "--patterns", files["patterns"], "--input", files["fasta"],
                                        "--workers", "2"])
        counts, matches = out.split("\n\n")
        assert counts.endswith("TOTAL\t\t2") and matches == "offset\texpression_index\n3\t2\n6\t1\n"
        code, out, _ = run_cli(capsys, ["locate", "--patterns", files["patterns"], "--input", files["fasta"],
                                        "--output-format", "json"])
        assert json.loads(out)["locations"] == [{"expression": 2, "offset": 3}, {"expression": 1, "offset": 6}]

    def test_raw_and_determinism(self, capsys, files):
        raw = files["dir"] / "body.txt"
        raw.write_text("ctacat")
        code, out, _ = run_cli(capsys, ["count", "--patterns", files["patterns"], "--input", str(raw)])
        assert "TOTAL\t\t2" in out
        argv = ["locate", "--patterns", files["patterns"], "--input", files["fasta"], "--workers", "8",
                "--output-format", "json"]
        assert run_cli(capsys, argv)[1] == run_cli(capsys, argv)[1]

    def test_bench(self, capsys, files):
        code, out, _ = run_cli(capsys, ["bench", "--patterns", files["patterns"], "--synthetic-size", "32K",
                                        "--workers", "1,2", "--repeat", "3"])
        assert code == 0
        lines = out.splitlines()
        assert len([l for l in lines if not l.startswith("#") and not l.startswith("scenario")]) == 6
        assert len({l.split("\t")[2] for l in lines if l.startswith("# checksum")}) == 1
        code, out, _ = run_cli(capsys, ["bench", "--patterns", files["patterns"], "--synthetic-size", "32K",
                                        "--workers", "2", "--repeat", "1", "--pattern-based",
                                        "--output-format", "json"])
        doc = json.loads(out)
        assert [r["scenario"] for r in doc["results"]] == ["input-based/w2", "pattern-based/w2"]
        assert len({r["checksum"] for r in doc["results"]}) == 1


@pytest.mark.gpu
def test_pattern_parallel_and_exhaustive(toy_exprs, toy_dfa):
    seq = ks.sequence_from_text("ttacatctacgtttacta" * 9)
    expect = ks.sequential_count(toy_dfa, seq)
    for workers in (1, 2, 3, 4, 9):
        assert ks.pattern_parallel_count(toy_exprs, seq, workers).tolist() == expect.tolist()
    for length in (1, 2, 3):
        r = ks.exhaustive_reconciliation_check(toy_dfa, length, window=10)
        assert r["count_mismatches"] == 0 and r["final_state_mismatches"] == 0
        assert 0 < r["converged_runs"] <= r["speculative_runs"]
    r = ks.exhaustive_reconciliation_check(toy_dfa, 3, window=0)
    assert r["converged_runs"] == 0


# ------------------------------------------------------------ reference transcripts
# tests/golden/cli/cases.json: argv, exit code and stdout of the REAL reference
# CLI (tests/golden/make_cli_golden.py).  The drop-in must match byte for byte.

GOLDEN_CLI = Path(__file__).resolve().parent / "golden" / "cli"


def _cli_cases(pred):
    cases = json.loads((GOLDEN_CLI / "cases.json").read_text())
    return [c for c in cases if pred(c)]


def _run_case(case, capsys, monkeypatch):
    monkeypatch.chdir(GOLDEN_CLI)
    code = cli.main(case["argv"])
    cap = capsys.readouterr()
    return code, cap.out, cap.err


@pytest.mark.parametrize("case", _cli_cases(lambda c: c["argv"][0] == "dump-dfa" or c["code"] != 0),
                         ids=lambda c: " ".join(c["argv"][:3]))
def test_cli_matches_reference_transcript_cpu(case, capsys, monkeypatch):
    """dump-dfa and the error paths never touch the GPU."""
    code, out, err = _run_case(case, capsys, monkeypatch)
    assert code == case["code"] and out == case["stdout"]
    if case["code"]:
        assert err == case["stderr"]


def _untimed(argv, text: str):
    """bench output without its timings (everything else must match)."""
    if argv[0] != "bench":
        return text
    if "--output-format" in argv:
        doc = json.loads(text)
        for r in doc["results"]:
            for k in ("seconds", "median_seconds", "min_seconds"):
                r.pop(k)
        return doc
    keep = []
    for line in text.splitlines():
        f = line.split("\t")
        keep.append(f[:2] if line.startswith("# median") else f[:3] if len(f) == 4 and not line.startswith("#") else f)
    return keep


@pytest.mark.gpu
@pytest.mark.parametrize("case", _cli_cases(lambda c: c["argv"][0] in ("count", "locate", "bench") and c["code"] == 0),
                         ids=lambda c: " ".join(c["argv"]))
def test_cli_matches_reference_transcript_gpu(case, capsys, monkeypatch):
    code, out, err = _run_case(case, capsys, monkeypatch)
    assert code == 0 and err == ""
    assert _untimed(case["argv"], out) == _untimed(case["argv"], case["stdout"])


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the reference algorithm's C port on the host
    cores) prints one JSON line with the contract's keys -- runs on CPU."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(repo / "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "1", "--bases", str(1 << 18)],
                         capture_output=True, text=True, timeout=600, cwd=repo)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    for key in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config"):
        assert key in line
    assert {"value", "unit", "cores", "kind", "sample"} <= set(line["cpu_baseline"])
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_bench_gpus_self_launch_on_cpu():
    """`bench.py --gpus 2` outside torchrun re-launches itself with two ranks
    (torch.distributed.run, rendezvous on 127.0.0.1); the reference arm's
    rank 0 prints n_gpus 2 and the other rank exits 0 -- runs on CPU."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in __import__("os").environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(repo / "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--config", "1", "--steps", "1", "--warmup", "3", "--bases", str(1 << 16)],
                         capture_output=True, text=True, timeout=600, cwd=repo, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def test_bench_world_size_mismatch_fails():
    """Under a launcher whose world size differs from --gpus, bench.py refuses."""
    import subprocess
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parents[1]
    env = dict(__import__("os").environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(repo / "bench.py"), "--impl", "reference", "--gpus", "4",
                          "--config", "1", "--steps", "1", "--bases", "4096"],
                         capture_output=True, text=True, timeout=300, cwd=repo, env=env)
    assert out.returncode == 2 and "WORLD_SIZE" in out.stderr
