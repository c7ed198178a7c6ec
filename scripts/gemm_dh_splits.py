import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, os.getcwd())
from scripts.gemm_check import run
for s in (1, 2, 3, 4):
    run(2240, 650, 10000, 0, 1, s)
for s in (1, 2):
    run(2240, 650, 2600, 0, 1, s)
