"""Our tcgen05 GEMM vs cuBLAS (torch.matmul, bf16 in, fp32 out via a bf16 product + cast is not
comparable, so cuBLAS is timed with bf16 output) on the C2 step's GEMM shapes; L2-warm, 50 reps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1812_01329_b200 import janus as J  # noqa: E402


def t_ms(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, M, N, K in [("dec", 2240, 10000, 656), ("in0", 2240, 2600, 656), ("dh", 2240, 656, 10000),
                      ("wgrad_dWdec", 10000, 656, 2240)] + ([("big", 8192, 8192, 8192)] if os.environ.get("GEMM_BIG") else []):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.zeros(M, N, device="cuda")
    ours = t_ms(lambda: J.dev_gemm_bf16(M, N, K, A, K, 0, B, K, 0, C, N))
    cub = t_ms(lambda: torch.matmul(A, B.T))
    f = 2.0 * M * N * K
    print(f"{name:12s} M={M} N={N} K={K}: ours {ours*1e3:7.1f} us ({f/ours/1e9:6.0f} TF/s)  "
          f"cuBLAS(bf16 out) {cub*1e3:7.1f} us ({f/cub/1e9:6.0f} TF/s)", flush=True)
