"""tcgen05 bf16 GEMM and fp32 SIMT GEMM vs a plain torch fp32 reference (all three operand-major combos)."""
import ctypes

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def run(bf16, A, a_mn, B, b_mn, M, N, K, alpha=1.0, acc=False, C=None):
    from paper_2510_17519_b200._lib import lib
    if C is None:
        C = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    rc = lib().mgv_dev_gemm(1 if bf16 else 0, A.data_ptr(), A.shape[1], 1 if a_mn else 0, B.data_ptr(), B.shape[1],
                            1 if b_mn else 0, M, N, K, C.data_ptr(), C.shape[1], alpha, 1 if acc else 0,
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    return C


@pytest.mark.parametrize("mode", [1, 0])
@pytest.mark.parametrize("bf16", [True, False])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 520, 200), (1000, 96, 3456), (64, 700, 4096), (777, 333, 96),
                                   (4096, 3456, 3456)])
def test_gemm(mode, bf16, a_mn, b_mn, M, N, K):
    """mode 1: CTA-pair (cta_group::2) kernel; mode 0: 1-CTA kernel with weight-tile multicast."""
    from paper_2510_17519_b200._lib import lib
    if not bf16 and mode == 0:
        pytest.skip("fp32 path has a single kernel")
    lib().mgv_dev_set_gemm_mode(mode)
    torch.manual_seed(M * 7 + N + K)
    dt = torch.bfloat16 if bf16 else torch.float32
    # storage shapes: K-major (rows, K) ; MN-major (K, rows); pad ld to a multiple of 8
    def make(rows, mn):
        shape = (K, rows) if mn else (rows, K)
        ld = (shape[1] + 7) // 8 * 8
        t = torch.randn(shape[0], ld, device="cuda").to(dt)
        return t, (t[:, :shape[1]].float().t() if mn else t[:, :shape[1]].float())
    A, Af = make(M, a_mn)
    B, Bf = make(N, b_mn)
    ref = Af @ Bf.t()
    C = run(bf16, A, a_mn, B, b_mn, M, N, K)
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < (2e-5 if bf16 else 1e-5), err
    # accumulate + alpha
    C2 = run(bf16, A, a_mn, B, b_mn, M, N, K, alpha=0.5, acc=True, C=C.clone())
    err2 = (C2 - 1.5 * ref).abs().max().item() / ref.abs().max().item()
    assert err2 < 3e-5, err2
