b() { timeout 600 python bench.py --no-cpu --steps 300 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; }
p() { timeout 600 python tools/profile_step.py --steps 50 "$@" 2>&1 | grep ms/step | sed 's/.*ring=/ring=/' | cut -c1-60; }
for i in 1 2; do
  echo "48 k3 $(b --workload k3) $(p)"
  echo "52 k3 $(SNPB200_LIB=tools/ab/libsnpb200_stage52.so b --workload k3) $(SNPB200_LIB=tools/ab/libsnpb200_stage52.so p)"
  echo "40 k3 $(SNPB200_LIB=tools/ab/libsnpb200_stage40.so b --workload k3) $(SNPB200_LIB=tools/ab/libsnpb200_stage40.so p)"
done
echo "48 k4 $(b --workload k4)"
echo "52 k4 $(SNPB200_LIB=tools/ab/libsnpb200_stage52.so b --workload k4)"
echo "40 k4 $(SNPB200_LIB=tools/ab/libsnpb200_stage40.so b --workload k4)"
