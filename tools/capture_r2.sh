#!/bin/bash
# Round-2 evidence, run on the GPU box (gpurun -- 'bash tools/capture_r2.sh'):
# bench lines, the bench launch list, ncu --set full captures of every step
# kernel (summaries and source-line breakdowns written on the box, so only
# text comes back), and the format comparison.  Then: python tools/write_profiles_r2.py
set -x
O=gpurun_out/r2f
mkdir -p $O
timeout 900 python bench.py > $O/bench_k3.json 2> $O/bench_k3.err
timeout 600 python bench.py --workload k4 --no-cpu > $O/bench_k4.json 2> $O/bench_k4.err
timeout 600 python bench.py --workload k2 --no-cpu > $O/bench_k2.json 2> $O/bench_k2.err
timeout 900 python bench.py --workload k5 --no-cpu --steps 20 > $O/bench_k5.json 2> $O/bench_k5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu > $O/bench_under_ncu.log 2>&1
cap() {
  n=$1; k=$2; shift 2
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$k" -s ${SKIP:-3} -c 1 -o $O/$n \
      python tools/profile_step.py --steps 6 "$@" > $O/$n.log 2>&1
  python tools/ncu_summary.py $O/$n.ncu-rep > $O/$n.summary.txt 2>&1
  python tools/ncu_source.py $O/$n.ncu-rep --top 25 > $O/$n.source.txt 2>&1
}
cap k3_tiled tiled_step_kernel
cap k4_tiled tiled_step_kernel --workload k4
cap k2_tiled tiled_step_kernel --workload k2
cap k3_ell ell_bin_step_kernel --format ell
cap k3_push ell_bin_step_kernel --variant push
cap k3_pull '^(snp::)?step_kernel' --variant pull
cap k5_tiled tiled_step_kernel --q 100000000
SKIP=0 cap sort100_small small_run_kernel --sort 100 --variant small
timeout 1800 python tools/bench_formats.py --out $O/formats.json > $O/formats.log 2>&1
for f in $O/*.ncu-rep; do case $f in *k3_tiled.ncu-rep|*k3_ell.ncu-rep) ;; *) rm -f $f;; esac; done
ls -la $O
