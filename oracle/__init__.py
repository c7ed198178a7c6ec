"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what JANUS's speculative graph path computes
(the graph path must reach the imperative result, or report the broken assumption and
change nothing). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import it. It shares no code with the CUDA path (paper_1812_01329_b200/).
"""
from .interp import run_graph_step, run_imperative_step, run_dp_step, tree_schedule, Result  # noqa
