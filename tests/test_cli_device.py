"""CLI (paper_2408_04343_b200.cli) against the reference CLI's recorded
outputs (tests/golden/cli.json, make_cli_golden.py) and the reference's
pkg/tests/test_cli.py cases.  `run` / `bench` execute the CUDA engine and
are marked gpu; argument handling, generate and size run on CPU."""

import csv
import io
import re

import pytest

import paper_2408_04343_b200 as snp
from paper_2408_04343_b200.bench import CSV_HEADER
from paper_2408_04343_b200.cli import main
from conftest import golden_json

GOLD = golden_json("cli.json")


def run_cli(*argv):
    return main(list(argv))


# -- CPU ------------------------------------------------------------------------------

@pytest.mark.parametrize("case", range(len(GOLD["generate"])))
def test_generate_matches_reference(case, tmp_path, capsys):
    g = GOLD["generate"][case]
    path = tmp_path / "m.snp"
    assert run_cli(*g["argv"], "-o", str(path)) == g["rc"] == 0
    assert path.read_text() == g["model"]
    assert capsys.readouterr().out.replace(str(path), "<out>") == g["stdout"]


@pytest.mark.parametrize("case", range(len(GOLD["size"])))
def test_size_matches_reference(case, capsys):
    s = GOLD["size"][case]
    assert run_cli(*s["argv"]) == s["rc"]
    assert capsys.readouterr().out == s["stdout"]


def test_size_empty_model_and_single_format(tmp_path, capsys):
    empty = tmp_path / "empty.snp"
    empty.write_text("snp 1\nneurons 0\nspikes\n")
    assert run_cli("size", "--model", str(empty)) == 0
    for line in capsys.readouterr().out.splitlines():
        assert "elements=1 " in line
    assert run_cli("size", "--family", "sort", "-n", "100", "--format", "compressed") == 0
    assert capsys.readouterr().out.strip().startswith("compressed elements=71301")


def test_usage_errors_exit_1(tmp_path, capsys):
    assert run_cli() == 1
    assert "generate" in capsys.readouterr().out
    assert run_cli("generate", "--family", "sort", "-n", "0", "-o", str(tmp_path / "x.snp")) == 1
    assert not (tmp_path / "x.snp").exists()
    assert run_cli("generate", "-o", str(tmp_path / "x.snp")) == 1
    assert run_cli("run", "--family", "sort", "-n", "3", "--format", "dense") == 1
    err = capsys.readouterr().err
    assert all(f in err for f in ("sparse", "ell", "compressed", "oracle"))
    assert run_cli("run", "--model", "/nonexistent.snp", "--format", "sparse") == 1
    assert run_cli("run", "--family", "sort", "-n", "3", "--format", "oracle") == 1
    assert run_cli("bench", "--family", "sort", "--sizes", "3", "--reps", "0") == 1
    assert run_cli("bench", "--family", "sort", "--sizes", "3", "--formats", "oracle") == 1
    assert run_cli("bench", "--family", "sort", "--sizes", "0") == 1


def test_invalid_model_file_exit_2(tmp_path, capsys):
    bad = tmp_path / "bad.snp"
    bad.write_text("snp 1\nneurons 1\nspikes 0\nsynapse 1 1\n")
    assert run_cli("run", "--model", str(bad), "--format", "sparse") == 2
    assert "model error" in capsys.readouterr().err
    bad.write_text("snp 1\nneurons 1\nspikes 0\nbogus\n")
    assert run_cli("size", "--model", str(bad)) == 2


def test_generate_synth_roundtrip(tmp_path, capsys):
    path = tmp_path / "synth.snp"
    assert run_cli("generate", "--family", "synth", "-n", "5000", "--delays", "-o", str(path)) == 0
    assert "q=5000 m=20000 max_out_degree=16" in capsys.readouterr().out
    a = snp.load_model(path)
    b = snp.synth_v1(5000, with_delays=True)
    assert (a.adj_targets == b.adj_targets).all() and (a.rules.delay == b.rules.delay).all()


# -- GPU ------------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(GOLD["run"])))
def test_run_trace_matches_reference(case, tmp_path, capsys):
    r = GOLD["run"][case]
    path = tmp_path / "t.trace"
    assert run_cli(*r["argv"], "--trace-out", str(path)) == r["rc"] == 0
    assert path.read_text() == r["trace"]
    summary = re.sub(r" (wall_ms|build_ms)=[0-9.]+", "", capsys.readouterr().out.strip())
    assert summary == r["summary"]


@pytest.mark.gpu
def test_run_formats_and_variants_identical(tmp_path):
    model = tmp_path / "m.snp"
    run_cli("generate", "--family", "sort", "-n", "6", "-o", str(model))
    blobs = []
    for fmt, var in [("sparse", "auto"), ("ell", "auto"), ("compressed", "tiled"), ("compressed", "pull"),
                     ("compressed", "push")]:
        trace = tmp_path / f"{fmt}-{var}.trace"
        assert run_cli("run", "--model", str(model), "--format", fmt, "--variant", var, "--steps", "50",
                       "--seed", "9", "--trace-out", str(trace)) == 0
        blobs.append(trace.read_bytes())
    assert all(b == blobs[0] for b in blobs)


@pytest.mark.gpu
def test_run_negative_spikes_exit_3(tmp_path, capsys):
    bad = tmp_path / "neg.snp"
    bad.write_text("snp 1\nneurons 1\nspikes 1\nrule 1 ge 1 2 1 0\n")
    assert run_cli("run", "--model", str(bad), "--format", "ell") == 3
    assert "simulation error" in capsys.readouterr().err


@pytest.mark.gpu
def test_run_final_only_synth(capsys):
    assert run_cli("run", "--family", "synth", "-n", "100000", "--format", "compressed", "--steps", "20",
                   "--final-only") == 0
    assert "halt=step_limit steps=20 format=compressed" in capsys.readouterr().out


@pytest.mark.gpu
def test_bench_csv(tmp_path, capsys):
    out = tmp_path / "bench.csv"
    assert run_cli("bench", "--family", "sort", "--sizes", "3,5", "--formats", "sparse,ell,compressed",
                   "--reps", "3", "--csv-out", str(out)) == 0
    text = out.read_text()
    lines = text.splitlines()
    assert lines[0] == CSV_HEADER and len(lines) == 1 + 2 * 3 * 3
    for row in csv.DictReader(io.StringIO(text)):
        system = snp.gen_sort(snp.SortInstance(int(row["size"])))
        assert int(row["elements"]) == snp.storage_elements(snp.Format(row["format"]), system)
        assert row["halt"] == "no_applicable_rules" and float(row["wall_ms"]) >= 0.0
    assert "build_ms" in capsys.readouterr().out
    assert run_cli("bench", "--family", "subsetsum", "--sizes", "3", "--formats", "compressed") == 0
    assert CSV_HEADER in capsys.readouterr().out


@pytest.mark.gpu
def test_run_digest_out_matches_trace(tmp_path):
    trace = tmp_path / "t.trace"
    digs = tmp_path / "t.dig"
    assert run_cli("run", "--family", "sort", "-n", "12", "--format", "compressed", "--trace-out", str(trace)) == 0
    assert run_cli("run", "--family", "sort", "-n", "12", "--format", "compressed", "--digest-out", str(digs)) == 0
    rows = [[int(v) for v in line.split()] for line in trace.read_text().splitlines()]
    assert digs.read_text().split() == [f"{snp.row_digest(r):016x}" for r in rows]
