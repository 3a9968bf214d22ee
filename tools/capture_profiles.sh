#!/bin/bash
# Run on the GPU box (gpurun): bench line + ncu launch list + full captures.
# gpurun copies back at most 64 MiB of gpurun_out/, and each --set full report
# is ~22 MB, so the captures come in two calls:
#   gpurun -- 'bash tools/capture_profiles.sh 1'   # bench --extra, launch list, K3 report
#   gpurun -- 'bash tools/capture_profiles.sh 2'   # K4 and K2 reports
# (move gpurun_out/prof_k3.ncu-rep aside between the calls), then
#   python tools/write_profiles.py r1
set -x
mkdir -p gpurun_out
part=${1:-1}
if [ "$part" = "1" ]; then
  timeout 600 python bench.py --extra > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:tiled_step_kernel -s 3 -c 1 \
      -o gpurun_out/prof_k3 python tools/profile_step.py --steps 5 > gpurun_out/ncu_k3.log 2>&1
else
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 3 -c 1 \
      -o gpurun_out/prof_k4 python tools/profile_step.py --steps 5 --workload k4 > /dev/null 2>&1
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 3 -c 1 \
      -o gpurun_out/prof_k2 python tools/profile_step.py --steps 5 --workload k2 > /dev/null 2>&1
fi
ls -la gpurun_out
