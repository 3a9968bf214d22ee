"""Turn gpurun_out/ captures into committed summaries under profiles/."""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import summary  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "profiles"
GP = ROOT / "gpurun_out"
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"


def stall_top(rep, n=15):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    hdr, data = rows[1], rows[2:]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    tot = sum(float(r[si] or 0) for r in data) or 1.0
    top = sorted(enumerate(data), key=lambda x: -float(x[1][si] or 0))[:n]
    return [f"{float(r[si]) / tot * 100:5.1f}%  sass#{i:<5d} exec={r[ie]:>9}  {r[1].strip()[:90]}" for i, r in top]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0, []])
    for r in data:
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] in ("ns", "nsecond") else (v * 1000 if r[ui] in ("ms", "msecond") else v)
        a = agg[r[ki].split("(")[0]]
        a[0] += 1
        a[1] += v
        a[2].append(v)
    setup_marks = ("ingest_", "cub::", "tp_", "fill_", "indeg", "transpose", "build_", "digest_u32", "load_state",
                   "widen_", "ds_to_delay")
    step = {k: v for k, v in agg.items() if not any(m in k for m in setup_marks)}
    setup = {k: v for k, v in agg.items() if k not in step}
    tot = sum(a[1] for a in step.values()) or 1.0
    lines = ["per-step kernels (share of per-step kernel time):",
             "kernel | launches | total_us | share | per-launch us (each)"]
    for name, (c, t, each) in sorted(step.items(), key=lambda x: -x[1][1]):
        lines.append(f"{name} | {c} | {t:.1f} | {t / tot * 100:.1f}% | " + " ".join(f"{x:.1f}" for x in each))
    lines += ["", "engine-creation / host-API kernels (not per step):", "kernel | launches | total_us"]
    for name, (c, t, _) in sorted(setup.items(), key=lambda x: -x[1][1]):
        lines.append(f"{name} | {c} | {t:.1f}")
    return lines


def main():
    OUT.mkdir(exist_ok=True)
    traffic = {}
    tf = OUT / "traffic_bytes.json"
    if tf.exists():
        traffic = json.loads(tf.read_text())
    for rep, key, title in [("prof_k3.ncu-rep", "k3/compressed/tiled/first", "K3 synth q=1e7, tiled step kernel"),
                            ("prof_k4.ncu-rep", "k4/compressed/tiled/first", "K4 synth q=1e7 + delays, tiled step kernel"),
                            ("prof_k2.ncu-rep", "k2/compressed/tiled/first", "K2 sort n=4096, tiled step kernel")]:
        p = GP / rep
        if not p.exists():
            continue
        s = summary(str(p))[0]
        rd = float(s["dram__bytes_read.sum"].split()[0]) * (1e9 if "Gbyte" in s["dram__bytes_read.sum"] else 1e6)
        wr = float(s["dram__bytes_write.sum"].split()[0]) * (1e9 if "Gbyte" in s["dram__bytes_write.sum"] else 1e6)
        traffic[key] = rd + wr
        lines = [f"# {title} -- ncu --set full --clock-control none (one launch, cold cache, serialised)", ""]
        lines += [f"{k:80s} {v}" for k, v in s.items()]
        lines += ["", f"dram traffic per launch (read+write): {rd + wr:.4e} bytes", "", "top warp-stall SASS lines:"]
        lines += stall_top(p)
        (OUT / f"{tag}_ncu_{key.split('/')[0]}_tiled.txt").write_text("\n".join(lines) + "\n")
    tf.write_text(json.dumps(traffic, indent=1) + "\n")
    if (GP / "launches.csv").exists():
        (OUT / f"{tag}_launches_bench.txt").write_text(
            "# ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 5 --warmup 3 --no-cpu\n"
            "# (cold-cache, serialised launches: compare shares, not absolutes; early-exit launches are the\n"
            "#  graph slots past the segment end and the e2e snp_run calls)\n" + "\n".join(launches(GP / "launches.csv")) + "\n")
    if (GP / "bench_full.json").exists():
        (OUT / f"{tag}_bench_k3.json").write_text((GP / "bench_full.json").read_text())


if __name__ == "__main__":
    main()
