#!/bin/bash
# A/B of dev kernel variants (paper_1812_01329_b200/build.py JANUS_VARIANT): parity subset + the
# C2 / C3 bench numbers per variant. usage: scripts/ab_variants.sh "" nmw1 nmw2 ...
out=gpurun_out/ab
mkdir -p $out
for v in "$@"; do
  tag=${v:-base}
  JANUS_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_lm.py tests/test_gpu_tree.py -x -q > $out/test_$tag.log 2>&1
  echo "$tag tests: $(tail -1 $out/test_$tag.log)"
  for rep in 1 2; do
    JANUS_VARIANT=$v timeout 300 python bench.py --no-cpu-baseline --steps 200 > $out/bench_$tag.json 2>/dev/null
    python - "$out/bench_$tag.json" "$tag" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).readline())
p = d["phases_ms_per_step"]
t = d.get("treelstm_b25", {}); t2 = d.get("treelstm_b256", {}); r = d.get("treernn_b25", {})
print(f"{sys.argv[2]:8s} C2 {d['value']:.0f}/s {d['ms_per_step']:.4f} ms fwd {p['rec_fwd01']:.4f} bwd {p['rec_bwd01']:.4f} "
      f"gemm {p['gemm_dec']+p['gemm_in0']+p['gemm_dh']+p['gemm_wgrad']:.4f} | tree25 {t.get('ms_per_step',0):.4f} "
      f"(fwd {t.get('phases_ms_per_step',{}).get('tree_fwd',0):.4f} bwd {t.get('phases_ms_per_step',{}).get('tree_bwd',0):.4f}) "
      f"tree256 {t2.get('ms_per_step',0):.4f} rnn25 {r.get('ms_per_step',0):.4f} clk {d['clocks']['sm_mhz']}")
PY
  done
done
