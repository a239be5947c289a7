set -x
timeout 120 python tools/profile_run.py --config c3_prefix 2>&1 | tail -3
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in c1 c2 c3 c4 c2_prefix c2_decode c3_chunks; do timeout 120 python tools/profile_run.py --config $c 2>&1 | tail -1; done
