b() { timeout 600 python bench.py --no-cpu --steps 300 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; }
for i in 1 2; do
for env in "X=0" "SNPB200_TILES_PER_SM=3" "SNPB200_TILES_PER_SM=1" "SNPB200_RING=3" "SNPB200_PDL=0"; do
  echo "$env k3 $(env $env bash -c "$(declare -f b); b --workload k3")"
done; done
