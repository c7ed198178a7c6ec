#!/bin/bash
# Microbenchmarks of the recurrent step's building blocks (run on the GPU box; binaries built here).
for cfg in "64 64 0 1" "64 64 0 4" "128 64 0 1" "128 64 0 4" "128 64 1 1" "128 64 1 4" "64 64 1 1" "128 128 0 1" "128 128 1 1" "64 64 2 0" "16 16 2 0" "32 32 2 0"; do
  timeout 30 ./scripts/bm.bin $cfg
done
timeout 120 ./scripts/bx.bin
