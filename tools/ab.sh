#!/bin/bash
# A/B driver (diagnostics): tools/ab.sh "CONFIGS" "ENV_A" "ENV_B" [...]  -> one line per run
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
cfgs=$1; shift
for c in $cfgs; do
  for rep in 1 2; do
    for e in "$@"; do
      r=$(env $e timeout 400 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d.get('parity',{}).get('ok'), d.get('device_error_bits'))" 2>&1 | tail -1)
      echo "$c [$e] $r" | tee -a gpurun_out/ab.txt
    done
  done
done
