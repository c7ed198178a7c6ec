#!/bin/bash
# A/B of an environment knob on the C2 bench: scripts/ab_env.sh VAR v1 v2 ...  ("-" = unset)
var=$1; shift
for v in "$@"; do
  for rep in 1 2; do
    if [ "$v" = "-" ]; then unset $var; else export $var=$v; fi
    timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 300 > gpurun_out/abenv.json 2>/dev/null
    python - "$var=$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/abenv.json").readline())
p = d["phases_ms_per_step"]
print(f"{sys.argv[1]:22s} C2 {d['value']:.0f}/s {d['ms_per_step']:.4f} ms fwd {p['rec_fwd01']:.4f} bwd {p['rec_bwd01']:.4f}")
PY
  done
done
