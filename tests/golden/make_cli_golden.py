"""Record the reference CLI's outputs (run in the build container, where
/root/reference exists):  python tests/golden/make_cli_golden.py

Writes tests/golden/cli.json: for each `run` case the trace file bytes and
the summary line without its timing fields; for `generate` the model-file
text; for `size` the printed lines (pkg/src/snpsim/cli.py:117-191)."""

import contextlib
import io
import json
import re
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from snpsim.cli import main  # noqa: E402

OUT = Path(__file__).resolve().parent / "cli.json"
RUNS = [
    ["run", "--family", "sort", "-n", "4", "--format", "compressed", "--steps", "50", "--seed", "9"],
    ["run", "--family", "sort", "-n", "10", "--format", "ell"],
    ["run", "--family", "sort", "--values", "5,1,4,2", "--format", "sparse"],
    ["run", "--family", "sort", "-n", "3", "--format", "sparse", "--steps", "1"],
    ["run", "--family", "subsetsum", "--values", "1,0,3", "--target", "4", "--format", "compressed", "--seed", "3"],
    ["run", "--family", "random", "-n", "40", "--seed", "11", "--format", "ell", "--steps", "30"],
]
GENERATE = [
    ["generate", "--family", "sort", "-n", "3"],
    ["generate", "--family", "subsetsum", "-n", "6", "--seed", "1"],
    ["generate", "--family", "random", "-n", "20", "--seed", "5"],
]
SIZE = [["size", "--family", "sort", "-n", "100"], ["size", "--family", "random", "-n", "30", "--seed", "2"]]


def capture(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = main(argv)
    return rc, buf.getvalue()


def main_():
    out = {"run": [], "generate": [], "size": []}
    with tempfile.TemporaryDirectory() as d:
        for argv in RUNS:
            path = Path(d) / "t.trace"
            rc, text = capture(argv + ["--trace-out", str(path)])
            summary = re.sub(r" (wall_ms|build_ms)=[0-9.]+", "", text.strip())
            out["run"].append({"argv": argv, "rc": rc, "summary": summary, "trace": path.read_text()})
        for argv in GENERATE:
            path = Path(d) / "m.snp"
            rc, text = capture(argv + ["-o", str(path)])
            out["generate"].append({"argv": argv, "rc": rc, "stdout": text.replace(str(path), "<out>"),
                                    "model": path.read_text()})
        for argv in SIZE:
            rc, text = capture(argv)
            out["size"].append({"argv": argv, "rc": rc, "stdout": text})
    OUT.write_text(json.dumps(out, indent=1))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main_()
