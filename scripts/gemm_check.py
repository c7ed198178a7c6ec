"""Error and timing of the tcgen05 GEMM (dev hook) for the C2 step's shapes, per split count."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1812_01329_b200 import janus as J

def run(M, N, K, a_mn, b_mn, splits, reps=20):
    g = torch.Generator(device="cuda").manual_seed(0)
    r8 = lambda x: (x + 7) // 8 * 8
    lda = r8(M) if a_mn else r8(K)
    ldb = r8(N) if b_mn else r8(K)
    A = (torch.rand((K, lda) if a_mn else (M, lda), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    B = (torch.rand((K, ldb) if b_mn else (N, ldb), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    ldc = (N + 3) // 4 * 4
    C = torch.zeros((M, ldc), device="cuda")
    Am = (A[:, :M].T if a_mn else A[:, :K]).double()
    Bm = (B[:, :N].T if b_mn else B[:, :K]).double()
    ref = Am @ Bm.T
    J.dev_gemm_bf16_splitk(M, N, K, A, lda, a_mn, B, ldb, b_mn, C, ldc, None, None, False, splits)
    torch.cuda.synchronize()
    err = ((C[:, :N].double() - ref).abs().max() / ref.abs().max()).item()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        J.dev_gemm_bf16_splitk(M, N, K, A, lda, a_mn, B, ldb, b_mn, C, ldc, None, None, False, splits)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 2.0 * M * N * K / ms / 1e9
    print(f"M={M:5d} N={N:5d} K={K:5d} a_mn={a_mn} b_mn={b_mn} splits={splits}: err {err:.2e}  {ms*1000:8.1f} us  {tf:7.1f} TFLOP/s", flush=True)

if __name__ == "__main__":
    shapes = [(2240, 10000, 704, 0, 0), (2240, 2600, 656, 0, 0), (10000, 651, 2240, 1, 1), (2240, 650, 10000, 0, 1),
              (2600, 651, 2240, 1, 1), (2240, 650, 2600, 0, 1)]
    for sh in shapes:
        for s in (1, 0, 2):
            run(*sh, s)
