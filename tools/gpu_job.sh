#!/bin/bash
# Round-end style validation on one B200 (run through gpurun): GPU tests, smoke,
# bench lines for every config + the reference arm, launch lists and ncu summaries.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py 2>&1 | tail -1 | tee -a gpurun_out/bench.jsonl
for c in c3 c4 c1; do timeout 300 python bench.py --config $c 2>&1 | tail -1 | tee -a gpurun_out/bench.jsonl; done
timeout 300 python bench.py --config c5 --steps 20 --no-e2e 2>&1 | tail -1 | tee -a gpurun_out/bench.jsonl
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 | tee -a gpurun_out/bench.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for c in c2 c3 c4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:psa_v2 -s 3 -c 1 -f \
    -o /tmp/${c}_full python tools/profile_run.py --config $c > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/${c}_full.ncu-rep "$c" > gpurun_out/ncu_sum_$c.txt 2>&1
done
