b() { timeout 600 python bench.py --no-cpu --steps 50 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; }
for i in 1 2; do
echo "768 ell $(b --workload k3 --format ell) push $(b --workload k3 --variant push)"
for bt in 512 1024; do echo "$bt ell $(SNPB200_LIB=tools/ab/libsnpb200_bin$bt.so b --workload k3 --format ell) push $(SNPB200_LIB=tools/ab/libsnpb200_bin$bt.so b --workload k3 --variant push)"; done
done
