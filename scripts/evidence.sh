#!/bin/bash
# Round evidence on one GPU box: full GPU suite, the bench line, the ncu launch list of the bench
# command and one ncu --set full capture of a C2 step (every launch of step 3).
# usage: scripts/evidence.sh TAG   (outputs under gpurun_out/TAG_*)
tag=${1:-r2}
o=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > $o/${tag}_gputest.log 2>&1; echo "gpu tests rc=$?: $(tail -1 $o/${tag}_gputest.log)"
timeout 900 python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > $o/${tag}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --launch-skip 24 --launch-count 12 \
  -o $o/${tag}_c2_full -f python scripts/run_c2.py 3 > $o/${tag}_ncu_full.log 2>&1; echo "ncu full rc=$?"
# the dominant kernel alone (small report, committed): rec_bwd of step 3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_rec_bwd --launch-skip 2 --launch-count 1 \
  -o $o/${tag}_rec_bwd -f python scripts/run_c2.py 3 > $o/${tag}_ncu_recbwd.log 2>&1; echo "ncu rec_bwd rc=$?"
# C3 B=25 launch list
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_tree_launches.csv \
  python scripts/run_c2.py 3 c3 > /dev/null 2>&1; echo "tree launch list rc=$?"
