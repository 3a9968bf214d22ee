"""Turn the round-2 captures (gpurun_out/r2f, tools/capture_r2.sh) into the
committed summaries under profiles/ (r2_*)."""
import json
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from write_profiles import launches  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
GP = ROOT / "gpurun_out" / "r2f"
OUT = ROOT / "profiles"

CAPS = [("k3_tiled", "k3/compressed/tiled/first", "K3 synth q=1e7, Optimized (tiled) step kernel"),
        ("k4_tiled", "k4/compressed/tiled/first", "K4 synth q=1e7 + delays 0-3, tiled step kernel"),
        ("k2_tiled", "k2/compressed/tiled/first", "K2 sort n=4096, tiled step kernel"),
        ("k5_tiled", "k5/compressed/tiled/first", "K5 synth q=1e8 on one GPU, tiled step kernel"),
        ("k3_ell", "k3/ell/tiled/first", "K3 synth q=1e7, ELL (Alg. 4) binned push step kernel"),
        ("k3_push", "k3/compressed/push/first", "K3 synth q=1e7, COMPRESSED push (Alg. 5) binned step kernel"),
        ("k3_pull", "k3/compressed/pull/first", "K3 synth q=1e7, COMPRESSED CSR-pull step kernel"),
        ("sort100_small", "sort100/compressed/small/first", "sort n=100, small-system kernel (one launch = 6 steps)"),
        ("k3_tiled2_pass1", "k3tp/compressed/tiled2/pass1", "K3, two-pass receive (variant tiled2): pass 1 per source window"),
        ("k3_tiled2_tiles", "k3tp/compressed/tiled2/tiles", "K3, two-pass receive (variant tiled2): the tile kernel"),
        ("sort2048_dense", "sort2048/sparse/dense", "sort n=2048, SPARSE (dense GEMV over fired rows, Alg. 3)"),
        ("sort2048_dense_step", "sort2048/sparse/step", "sort n=2048, SPARSE: the fused finish/select step kernel")]


def dram_bytes(summary: str) -> float:
    tot = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        m = re.search(key + r"\s+([\d.]+)\s+(\w+)", summary)
        if m:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(m.group(2), 1)
            tot += float(m.group(1)) * scale
    return tot


def main():
    OUT.mkdir(exist_ok=True)
    tf = OUT / "traffic_bytes.json"
    traffic = json.loads(tf.read_text()) if tf.exists() else {}
    for name, key, title in CAPS:
        sp, so = GP / f"{name}.summary.txt", GP / f"{name}.source.txt"
        if not sp.exists():
            continue
        summ = sp.read_text()
        if "gpu__time_duration" not in summ:
            continue
        b = dram_bytes(summ)
        if key.startswith(("k2/", "k3/", "k4/", "k5/")):
            traffic[key] = b
        log = (GP / f"{name}.log").read_text() if (GP / f"{name}.log").exists() else ""
        info = [l for l in log.splitlines() if "ms/step" in l]
        lines = [f"# {title} -- ncu --set full --import-source on --clock-control none (one launch, cold cache,",
                 "# serialised; shares and counters, not absolute times)", ""]
        lines += [l for l in summ.splitlines() if l.strip()]
        lines += ["", f"dram traffic per launch (read+write): {b:.4e} bytes"]
        if info:
            lines += ["", "engine (profile_step.py, not a bench value): " + info[-1]]
        if so.exists():
            lines += ["", "source lines by warp-level instructions executed (tools/ncu_source.py):"]
            lines += so.read_text().splitlines()
        (OUT / f"r2_ncu_{name}.txt").write_text("\n".join(lines) + "\n")
    tf.write_text(json.dumps(traffic, indent=1) + "\n")
    if (GP / "launches.csv").exists():
        (OUT / "r2_launches_bench.txt").write_text(
            "# ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 5 --warmup 3 --no-cpu\n"
            "# (cold-cache, serialised launches: compare shares, not absolutes; early-exit launches are the\n"
            "#  graph slots past the segment end and the e2e snp_run calls)\n" + "\n".join(launches(GP / "launches.csv")) + "\n")
    for f in ("bench_k3", "bench_k4", "bench_k2", "bench_k5", "bench_reference"):
        p = GP / f"{f}.json"
        if p.exists():
            last = [l for l in p.read_text().splitlines() if l.strip().startswith("{")]
            if last:
                (OUT / f"r2_{f}.json").write_text(last[-1] + "\n")
    if (GP / "formats.json").exists():
        d = json.loads((GP / "formats.json").read_text())
        (OUT / "r2_formats.json").write_text(json.dumps(d, indent=1) + "\n")
        rows = ["| workload | format | variant | ms/step (device, run to halt or 20 steps) | step-kernel ms | "
                "alg. GB/s | frac of %.0f GB/s | device MB |" % d["hbm_gbs"], "|---|---|---|---|---|---|---|---|"]
        for r in d["rows"]:
            rows.append(f"| {r['workload']} | {r['format']} | {r['variant']} | {r['ms_per_step']:.4f} | "
                        f"{r['step_kernel_ms']:.4f} | {r['alg_GBps']:.1f} | {r['frac']:.3f} | {r['device_MB']:.0f} |")
        (OUT / "r2_formats.md").write_text("# Format comparison on one B200 (tools/bench_formats.py)\n\n" +
                                           "\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
