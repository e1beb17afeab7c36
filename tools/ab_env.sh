#!/bin/bash
# A/B of library environment knobs on one GPU box:
#   tools/ab_env.sh "WORKLOAD[:ARGS]..." "ENV_A" "ENV_B" [reps]
# e.g. tools/ab_env.sh "config4 config3-default" "QTN_LEVEL_STREAMS=0" "QTN_LEVEL_STREAMS=1" 2
# Prints value and ms_per_step per (workload, env, rep), alternating A and B.
cd "$(dirname "$0")/.."
WL="$1"; A="$2"; B="$3"; REPS="${4:-2}"
for w in $WL; do
  name="${w%%:*}"; extra=""; [[ "$w" == *:* ]] && extra="${w#*:}"; extra="${extra//,/ }"
  for r in $(seq 1 "$REPS"); do
    for e in "$A" "$B"; do
      out=$(env $e timeout 300 python bench.py --workload "$name" --steps 20 --warmup 5 \
            --no-cpu-baseline --no-records $extra 2>&1 | tail -n 1)
      echo "$name [$e] rep$r: $(echo "$out" | python -c 'import json,sys
try:
    d=json.loads(sys.stdin.read()); print(round(d["value"],1), "contr/s", round(d["ms_per_step"],4), "ms", "frac", round(d["roofline"]["frac"],3) if d.get("roofline") else None)
except Exception as ex: print("ERR", ex)')"
    done
  done
done
