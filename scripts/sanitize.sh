#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small steps of every device program
# (3 steps each: the second and third use the commit-refreshed bf16 copies)
for tool in memcheck racecheck synccheck; do
  for wl in c1 c2small c2v c3small c3rnn; do
    echo "== san_${tool}_${wl}"
    timeout 900 compute-sanitizer --tool $tool python scripts/run_c2.py 3 $wl 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|COMPUTE-SANITIZER|Invalid|Race|Error" | head -8
  done
done
