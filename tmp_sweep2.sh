b() { timeout 600 python bench.py --no-cpu --steps 300 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; }
p() { timeout 600 python tools/profile_step.py --steps 100 "$@" 2>&1 | grep ms/step | cut -c1-120; }
for tps in 2 1; do
  export SNPB200_TILES_PER_SM=$tps
  echo "tps=$tps k4 $(b --workload k4)"
  echo "tps=$tps k3 seeded $(b --workload k3 --policy seeded)"
  echo "tps=$tps q=3e6: $(p --q 3000000)"
  echo "tps=$tps q=1e6: $(p --q 1000000)"
  echo "tps=$tps q=3e5: $(p --q 300000)"
done
unset SNPB200_TILES_PER_SM
cat > /tmp/ma.py <<'PY'
import sys, time; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2408_04343_b200 as snp
from conftest import multi_amount_system
a = multi_amount_system(5_000_000, 3)
prep = snp.prepare(a, snp.Format.COMPRESSED, variant="tiled")
prep.engine.begin(); tot, k, _ = prep.engine.time_steps(50, snp.FirstApplicable(), per_kernel=True)
print("multi-amount 5e6", round(tot / 50, 4), prep.engine.info["counter_bits"], prep.engine.info["tile"], prep.engine.info["ring_stages"])
PY
for tps in 2 1; do SNPB200_TILES_PER_SM=$tps timeout 600 python /tmp/ma.py 2>&1 | tail -1; done
