timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_sharded.py -x -q -m gpu -k "not corpus and not full_size" 2>&1 | tail -2
for T in 16896 22528; do echo -n "T=$T: "; SNPB200_TILE=$T timeout 60 python tools/profile_step.py --steps 30; done
timeout 60 python tools/profile_step.py --steps 20 --workload k2
timeout 60 python tools/profile_step.py --steps 20 --workload k4
timeout 60 python tools/profile_step.py --steps 20 --policy seeded
