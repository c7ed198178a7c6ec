#!/bin/bash
# GEMM epilogue / pairing modes on the C2 shapes (scripts/gemm_ref.py), one process per mode
for mode in "" "JANUS_GEMM_NOSTREAM=1" "" "JANUS_GEMM_NOSTREAM=1"; do
  echo "== ${mode:-default}"
  env $mode timeout 120 python scripts/gemm_ref.py 2>&1 | grep -v "^big"
done
