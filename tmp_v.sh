timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "binned or push_step or ell or scenarios or corpus or full_size or negative or huge or edge or sort" 2>&1 | tail -2
b() { timeout 600 python bench.py --no-cpu --steps 50 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; }
echo "ell k3 $(b --workload k3 --format ell) k4 $(b --workload k4 --format ell) push k3 $(b --workload k3 --variant push)"
