"""GEMM throughput vs K for the decoder shape: separates mainloop throughput from per-tile costs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import torch
from scripts.gemm_check import run
for K in (704, 2048, 4096, 8192):
    run(2240, 10000, K, 0, 0, 1, reps=10)
for M, N in ((2240, 2560), (4480, 10240), (1280, 5120)):
    run(M, N, 704, 0, 0, 1, reps=10)
