"""Model files (modelfile.py / csrc/snp_modelio.cpp) against the reference's
own behaviour (tests/golden/modelfile.json, made by make_modelfile_golden.py)
and the reference's tests (pkg/tests/test_modelfile.py)."""

import numpy as np
import pytest

import paper_2408_04343_b200 as snp
from paper_2408_04343_b200 import modelfile as mf
from conftest import golden_json

GOLD = golden_json("modelfile.json")


def _families():
    systems = {
        "sort5": snp.gen_sort(snp.SortInstance(5)),
        "sort5v": snp.gen_sort(snp.SortInstance(5, (4, 1, 3, 7, 2))),
        "subset": snp.gen_subset_sum(snp.SubsetSumInstance((1, 0, 3), 4)),
    }
    for seed in range(12):
        systems[f"random{seed}"] = snp.gen_random(30, 4, 8, 20, 3, seed)
    return systems


def _same_arrays(a, b):
    for x, y in [(a.initial, b.initial), (a.rule_map.offsets, b.rule_map.offsets), (a.adj_offsets, b.adj_offsets),
                 (a.adj_targets, b.adj_targets)]:
        np.testing.assert_array_equal(np.asarray(x, np.int64), np.asarray(y, np.int64))
    for f in ("threshold", "is_exact", "consumed", "produced", "delay", "neuron"):
        np.testing.assert_array_equal(getattr(a.rules, f), getattr(b.rules, f))
    assert a.output_neuron == b.output_neuron


@pytest.mark.parametrize("name", sorted(GOLD["serialized"]))
def test_serialize_matches_reference(name, tmp_path):
    system = _families()[name]
    want = GOLD["serialized"][name]
    assert snp.serialize_model(system) == want
    assert snp.parse_model(want) == system
    # native writer: same bytes; native parser: same arrays
    path = tmp_path / "m.snp"
    mf.save_model(path, system)
    assert path.read_text() == want
    _same_arrays(mf.load_model(path), snp.system_arrays(system))


@pytest.mark.parametrize("case", range(len(GOLD["bad"])))
def test_malformed_and_invalid_texts(case):
    bad = GOLD["bad"][case]
    for parse in (snp.parse_model, mf.parse_model_arrays):
        with pytest.raises(Exception) as info:
            parse(bad["text"])
        assert type(info.value).__name__ == bad["type"], parse
        assert str(info.value) == bad["message"], parse
        assert isinstance(info.value, snp.ModelError)


@pytest.mark.parametrize("case", range(len(GOLD["good"])))
def test_good_texts(case):
    good = GOLD["good"][case]
    system = snp.parse_model(good["text"])
    assert snp.serialize_model(system) == good["serialized"]
    _same_arrays(mf.parse_model_arrays(good["text"]), snp.system_arrays(system))


def test_reference_roundtrip_cases():
    # pkg/tests/test_modelfile.py: empty system, output neuron, 1-based indices
    empty = snp.SNPSystem().validate()
    assert snp.parse_model(snp.serialize_model(empty)) == empty
    s = snp.SNPSystem()
    a, b = s.add_neuron(2), s.add_neuron(0)
    s.add_rule(a, snp.at_least(1), 1, 1, 0)
    s.add_synapse(a, b)
    s.output_neuron = b
    text = snp.serialize_model(s.validate())
    assert text.startswith("snp 1\n") and "rule 1 ge 1 1 1 0" in text and "synapse 1 2" in text
    assert "output 2" in text
    assert snp.parse_model(text).output_neuron == 1
    with pytest.raises(snp.ModelFileError, match="line 4"):
        snp.parse_model("snp 1\nneurons 1\nspikes 0\nbogus\n")


def test_native_roundtrip_synthetic(tmp_path):
    """A 200k-neuron synthetic system through the native writer and parser."""
    arrays = snp.synth_v1(200_000, with_delays=True)
    path = tmp_path / "synth.snp"
    mf.save_model(path, arrays)
    _same_arrays(mf.load_model(path), arrays)


def test_missing_file_is_oserror(tmp_path):
    with pytest.raises(OSError):
        mf.load_model(tmp_path / "nope.snp")


def test_native_trace_writer_matches_format_trace(tmp_path):
    rng = np.random.default_rng(3)
    rows = [rng.integers(-5, 10**12, size=37) for _ in range(9)]
    tr = snp.Trace(configs=rows, halt_reason=snp.HaltReason.STEP_LIMIT)
    path = tmp_path / "t.trace"
    mf.write_trace(path, tr)
    assert path.read_text() == snp.format_trace(tr)
    mf.write_trace(path, rows[:2], append=True)  # segment-by-segment writing
    assert path.read_text() == snp.format_trace(tr) + "".join(" ".join(map(str, r)) + "\n" for r in rows[:2])
    empty = snp.Trace(configs=[np.zeros(0, np.int64)] * 3, halt_reason=snp.HaltReason.STEP_LIMIT)
    mf.write_trace(path, empty)
    assert path.read_text() == snp.format_trace(empty) == "\n\n\n"


def _corrupt_cases(text):
    """Errors planted at several places of a valid model text: format, index,
    reflexive, rule-validation and directive errors, mixed line breaks."""
    lines = text.split("\n")
    n = len(lines)
    cases = []
    for frac, bad in [(0.95, "rule 1 ge x 1 1 0"), (0.5, "synapse 1 999999999"), (0.3, "synapse 2 2"),
                      (0.7, "rule 1 ge 1 1 2 0"), (0.8, "neurons 4"), (0.6, "bogus 1"), (0.99, "spikes 1")]:
        ls = list(lines)
        ls[int(n * frac)] = bad
        cases.append("\n".join(ls))
    # the first of two errors wins, whichever chunk it lands in
    ls = list(lines)
    ls[int(n * 0.9)] = "synapse 0 1"
    ls[int(n * 0.4)] = "rule 1 eq 0 1 1 0"
    cases.append("\n".join(ls))
    # \r\n, lone \r, \f and \v as line breaks (str.splitlines) before the error
    mixed = text.replace("\n", "\r\n", 200).replace("\n", "\r", 50)
    ls = mixed.split("\n")
    ls[int(len(ls) * 0.75)] = "\f\vsynapse 3 3"
    cases.append("\n".join(ls))
    return cases


@pytest.mark.parametrize("chunk", ["64", "1000", "1048576"])
def test_native_chunked_parse_matches_python(chunk, monkeypatch):
    """The native parser splits the rule/synapse section into chunks parsed on
    several threads; arrays, the first error (file order) and its line number
    must equal the sequential Python parser's."""
    monkeypatch.setenv("SNPIO_PARSE_CHUNK_BYTES", chunk)
    s = snp.SNPSystem()
    rng = np.random.default_rng(11)
    ids = [s.add_neuron(int(rng.integers(0, 5))) for _ in range(60)]
    for i in ids:
        for k in range(int(rng.integers(1, 4))):
            s.add_rule(i, snp.at_least(k + 1), k + 1, int(rng.integers(1, k + 2)), int(rng.integers(0, 2)))
        for j in rng.choice(len(ids), size=5, replace=False):
            if int(j) != i:
                s.add_synapse(i, ids[int(j)])
    s.output_neuron = ids[7]
    text = snp.serialize_model(s.validate())
    text += "output 3\n# trailing comment\nsynapse 4 5\n"  # later output wins
    want = snp.system_arrays(snp.parse_model(text))
    _same_arrays(mf.parse_model_arrays(text), want)
    _same_arrays(mf.parse_model_arrays(text.replace("\n", "\r\n")), want)
    for bad in _corrupt_cases(text):
        with pytest.raises(snp.ModelError) as py_err:
            snp.parse_model(bad)
        with pytest.raises(snp.ModelError) as native_err:
            mf.parse_model_arrays(bad)
        assert type(native_err.value) is type(py_err.value)
        assert str(native_err.value) == str(py_err.value)
