"""Timing of the step's GEMM shapes, unsplit (run once with JANUS_GEMM_CM=1 and once with =2)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_check import run
shapes = [(2240, 10000, 704, 0, 0), (2240, 2600, 656, 0, 0), (10000, 651, 2240, 1, 1), (2240, 650, 10000, 0, 1),
          (2600, 651, 2240, 1, 1), (2240, 650, 2600, 0, 1), (8192, 8192, 8192, 0, 0), (300, 650, 1000, 0, 0)]
print("JANUS_GEMM_CM =", os.environ.get("JANUS_GEMM_CM", "default"))
for sh in shapes:
    run(*sh, 1)
