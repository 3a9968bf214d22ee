"""Record the reference's model-file behaviour (run in the build container,
where /root/reference exists):

    python tests/golden/make_modelfile_golden.py

Writes tests/golden/modelfile.json: serialize_model text of family and
random systems, and for malformed / invalid texts the exception type and
message parse_model raises (pkg/src/snpsim/modelfile.py:40-167).
"""

import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import snpsim  # noqa: E402

OUT = Path(__file__).resolve().parent / "modelfile.json"

BAD = [
    "",
    "   \n# only a comment\n",
    "snp 2\nneurons 1\nspikes 0\n",
    "snp x\n",
    "snp\n",
    "neurons 1\nspikes 0\n",
    "snp 1\nneurons 1\n",
    "snp 1\nspikes 0\n",
    "snp 1\nneurons 2\nspikes 1\n",
    "snp 1\nneurons -1\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 gte 1 1 1 0\n",
    "snp 1\nneurons 1\nspikes 0\nrule 2 ge 1 1 1 0\n",
    "snp 1\nneurons 1\nspikes 0\nrule 0 ge 1 1 1 0\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 ge 1 1 1\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 ge x 1 1 0\n",
    "snp 1\nneurons 1\nspikes 0\nwibble 3\n",
    "snp 1\nneurons 1\nspikes x\n",
    "snp 1\nneurons 2\nspikes 0 0\nsynapse 1\n",
    "snp 1\nneurons 2\nspikes 0 0\nsynapse 0 1\n",
    "snp 1\nneurons 1\nspikes 0\nneurons 1\n",
    "snp 1\nneurons 1\nspikes 0\nspikes 0\n",
    "snp 1\nneurons 1\nrule 1 ge 1 1 1 0\n",
    "snp 1\nneurons 1\nspikes 0\nsynapse 1 1\n",
    "snp 1\nneurons 1\nspikes -3\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 ge -1 1 1 0\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 eq 0 1 1 0\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 ge 1 0 0 0\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 ge 1 1 -1 0\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 ge 1 1 1 -2\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 eq 2 2 0 1\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 ge 2 2 0 0\n",
    "snp 1\nneurons 1\nspikes 0\nrule 1 ge 1 1 2 0\n",
    "snp 1\nneurons 2\nspikes 0 0\noutput 3\n",
    "snp 1\nneurons 1\nspikes 0 # c\nbogus 'q'\n",
    "garbage\tline 'x'\n",
    "snp 1\r\nneurons 1\r\nspikes 0\r\nbogus\r\n",
]

GOOD = [
    "# a model\n\nsnp 1\nneurons 1\nspikes 4  # initial\n",
    "snp 1 extra\nneurons 2 9\nspikes 1_0 +2\nrule 2 ge 1 1 1 0\nrule 1 eq 3 3 0 0\nrule 1 ge 1 1 1 2\n"
    "synapse 1 2\nsynapse 1 2\nsynapse 2 1\noutput 2 7\n",
    "snp 1\nneurons 0\nspikes\n",
]


def main():
    systems = {
        "sort5": snpsim.gen_sort(snpsim.SortInstance(5)),
        "sort5v": snpsim.gen_sort(snpsim.SortInstance(5, (4, 1, 3, 7, 2))),
        "subset": snpsim.gen_subset_sum(snpsim.SubsetSumInstance((1, 0, 3), 4)),
    }
    for seed in range(12):
        systems[f"random{seed}"] = snpsim.gen_random(30, 4, 8, 20, 3, seed)
    out = {"serialized": {k: snpsim.serialize_model(v) for k, v in systems.items()}, "bad": [], "good": []}
    for text in BAD:
        try:
            snpsim.parse_model(text)
            out["bad"].append({"text": text, "type": None, "message": None})
        except Exception as exc:  # noqa: BLE001 - record whatever the reference raises
            out["bad"].append({"text": text, "type": type(exc).__name__, "message": str(exc)})
    for text in GOOD:
        out["good"].append({"text": text, "serialized": snpsim.serialize_model(snpsim.parse_model(text))})
    OUT.write_text(json.dumps(out, indent=1))
    print(f"wrote {OUT}: {len(systems)} systems, {len(BAD)} bad, {len(GOOD)} good texts")


if __name__ == "__main__":
    main()
