b() { timeout 600 python bench.py --no-cpu --steps 50 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4))"; }
for i in 1 2; do
echo "gu6 $(b --workload k3 --format ell) $(b --workload k4 --format ell)"
for gu in 4 8; do echo "gu$gu $(SNPB200_LIB=tools/ab/libsnpb200_gu$gu.so b --workload k3 --format ell) $(SNPB200_LIB=tools/ab/libsnpb200_gu$gu.so b --workload k4 --format ell)"; done
done
