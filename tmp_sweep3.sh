b() { timeout 600 python bench.py --no-cpu --steps 300 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; }
echo "default k3 $(b --workload k3)"
echo "default k4 $(b --workload k4)"
for tps in 4 2 1; do echo "tps=$tps k2 $(SNPB200_TILES_PER_SM=$tps b --workload k2)"; done
cat > /tmp/ma.py <<'PY'
import sys, time; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2408_04343_b200 as snp
from conftest import multi_amount_system
a = multi_amount_system(5_000_000, int(sys.argv[1]))
prep = snp.prepare(a, snp.Format.COMPRESSED, variant="tiled")
prep.engine.begin(); tot, k, _ = prep.engine.time_steps(50, snp.FirstApplicable(), per_kernel=True)
print("multi-amount 5e6 pmax", sys.argv[1], round(tot / 50, 4), prep.engine.info["counter_bits"], prep.engine.info["tile"], prep.engine.info["ring_stages"])
PY
for tps in 2 1; do SNPB200_TILES_PER_SM=$tps timeout 600 python /tmp/ma.py 300 2>&1 | tail -1; done
timeout 3000 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
