"""tcgen05 GEMM vs the oracle's contraction (fp64 of the same bf16-rounded operands): every output
element within the fp32 summation bound gamma_K * sum_k |a_k b_k|, plus the relative-norm check."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.numerics import rb  # noqa: E402


def _run(M, N, K, a_mn, b_mn, bias=None, acc=False, seed=0, splits=None, ret_out=False):
    from paper_1812_01329_b200 import janus as J
    g = np.random.default_rng(seed)
    A = rb(g.uniform(-1, 1, (M, K)))
    B = rb(g.uniform(-1, 1, (N, K)))
    r8 = lambda x: (x + 7) // 8 * 8
    lda = r8(M) if a_mn else r8(K) + 8
    ldb = r8(N) if b_mn else r8(K) + 8
    At = np.zeros((K, lda) if a_mn else (M, lda))
    Bt = np.zeros((K, ldb) if b_mn else (N, ldb))
    if a_mn:
        At[:, :M] = A.T
    else:
        At[:, :K] = A
    if b_mn:
        Bt[:, :N] = B.T
    else:
        Bt[:, :K] = B
    dA = torch.tensor(At, dtype=torch.bfloat16, device="cuda")
    dB = torch.tensor(Bt, dtype=torch.bfloat16, device="cuda")
    ldc = (N + 3) // 4 * 4
    C0 = g.uniform(-1, 1, (M, ldc)) if acc else np.zeros((M, ldc))
    dC = torch.tensor(C0, dtype=torch.float32, device="cuda")
    bcol = torch.tensor(g.uniform(-1, 1, N), dtype=torch.float32, device="cuda") if bias == "col" else None
    brow = torch.tensor(g.uniform(-1, 1, M), dtype=torch.float32, device="cuda") if bias == "row" else None
    if splits is None:
        J.dev_gemm_bf16(M, N, K, dA, lda, a_mn, dB, ldb, b_mn, dC, ldc, bcol, brow, acc)
    else:
        J.dev_gemm_bf16_splitk(M, N, K, dA, lda, a_mn, dB, ldb, b_mn, dC, ldc, bcol, brow, acc, splits)
    torch.cuda.synchronize()
    ref = A @ B.T
    if bcol is not None:
        ref += bcol.cpu().double().numpy()[None, :]
    if brow is not None:
        ref += brow.cpu().double().numpy()[:, None]
    if acc:
        ref += np.asarray(C0, np.float32)[:, :N]
    got = dC.cpu().double().numpy()[:, :N]
    # element-wise: bf16 x bf16 products are exact in fp32, so each output differs from the fp64
    # reference by at most the fp32 summation error, |err| <= gamma_n * sum_k |a_k b_k| (+ the
    # rounding of the bias / old C terms), gamma_n ~ n u with n = K + 2 terms, u = 2^-24; a factor
    # two of slack for the split / tile summation order
    absref = np.abs(A) @ np.abs(B).T
    if bcol is not None:
        absref += np.abs(bcol.cpu().double().numpy())[None, :]
    if brow is not None:
        absref += np.abs(brow.cpu().double().numpy())[:, None]
    if acc:
        absref += np.abs(np.asarray(C0, np.float32)[:, :N])
    bound = 2.0 * (K + 2) * 2.0 ** -24 * absref + 1e-30
    worst = (np.abs(got - ref) / bound).max()
    assert worst <= 1.0, f"element-wise fp32 summation bound exceeded by {worst:.3g}x"
    err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30)
    return (err, got) if ret_out else err


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (200, 136, 650), (2240, 2600, 650), (300, 1100, 2240)])
def test_gemm_layouts(M, N, K, a_mn, b_mn):
    assert _run(M, N, K, a_mn, b_mn) < 1e-5


def test_gemm_bias_and_accumulate():
    assert _run(333, 260, 130, 0, 0, bias="col") < 1e-5
    assert _run(333, 260, 130, 0, 1, bias="row", acc=True) < 1e-5


@pytest.mark.parametrize("splits", [0, 1, 2, 3, 5])
@pytest.mark.parametrize("M,N,K,a_mn,b_mn", [(2240, 650, 10000, 0, 1), (2600, 651, 2240, 1, 1), (200, 136, 650, 0, 0)])
def test_gemm_splitk(M, N, K, a_mn, b_mn, splits):
    """K split across CTAs, partial sums added in split order (SURVEY §8(a) H10 dgrad/wgrad)."""
    # fp32 accumulation over K = 10^4 terms: the error bound grows with K
    assert _run(M, N, K, a_mn, b_mn, splits=splits) < 1e-5 * max(1.0, K / 4096)


def test_gemm_splitk_bias_accumulate_and_empty_splits():
    # bias and the old C enter exactly once; more splits than k-blocks leaves empty splits
    assert _run(333, 260, 130, 0, 0, bias="col", acc=True, splits=4) < 1e-5
    assert _run(333, 260, 130, 0, 1, bias="row", acc=True, splits=3) < 1e-5
    assert _run(130, 300, 64, 0, 0, bias="col", splits=4) < 1e-5


def test_gemm_splitk_deterministic():
    e1, o1 = _run(2240, 650, 10000, 0, 1, splits=4, ret_out=True)
    e2, o2 = _run(2240, 650, 10000, 0, 1, splits=4, ret_out=True)
    assert e1 < 1e-5 and np.array_equal(o1, o2)


@pytest.mark.parametrize("M,N,K,a_mn,b_mn,bias", [(2240, 650, 10000, 0, 1, None), (300, 1100, 2240, 0, 0, "col"),
                                                  (2240, 650, 10000, 1, 0, "row")])
def test_gemm_split_add_two_halves(monkeypatch, M, N, K, a_mn, b_mn, bias):
    """GemmOp::split_add (the dh_top launch): the two K halves reduce-add into the zeroed C
    through the TMA store; bias added once; same bits on every run (two addends onto zero)."""
    monkeypatch.setenv("JANUS_GEMM_SPLIT_ADD", "1")
    e1, o1 = _run(M, N, K, a_mn, b_mn, bias=bias, splits=2, ret_out=True)
    e2, o2 = _run(M, N, K, a_mn, b_mn, bias=bias, splits=2, ret_out=True)
    assert e1 < 1e-5 * max(1.0, K / 4096) and np.array_equal(o1, o2)
