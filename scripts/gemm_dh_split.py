"""dh_top = dy . W_dec at C2 (M = T*B = 2240, N = 656, K = V = 10000; W_dec MN-major as in the
step): time and check split-K x tile width x CTA pair (JANUS_GEMM_BN / JANUS_GEMM_PAIR are read
once per process, so the caller runs one process per setting). usage: gemm_dh_split.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1812_01329_b200 import janus as J  # noqa: E402

M, N, K = 2240, 656, 10000
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randn(M, K, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
B = (torch.randn(K, N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)  # [K][N]: b_mn = 1
ref = A.float() @ B.float()


def t_us(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


tag = " ".join(f"{k}={os.environ[k]}" for k in ("JANUS_GEMM_BN", "JANUS_GEMM_PAIR", "JANUS_GEMM_SPLIT_ADD") if k in os.environ)
for splits in ((1, 2) if os.environ.get("JANUS_GEMM_SPLIT_ADD") else (1, 2, 3, 4)):
    C = torch.zeros(M, N, device="cuda")
    fn = lambda: J.dev_gemm_bf16_splitk(M, N, K, A, K, 0, B, N, 1, C, N, splits=splits)  # noqa: E731
    us = t_us(lambda: (C.zero_(), fn()))
    C.zero_()
    fn()
    err = ((C - ref).abs().max() / ref.abs().max()).item()
    print(f"{tag or 'default'} splits={splits}: {us:6.1f} us ({2 * M * N * K / us / 1e6:6.0f} TF/s) rel err {err:.2e}",
          flush=True)
