"""GEMM engines in isolation (tcgen05 3xTF32 and SIMT FP32) against an fp64 NumPy product,
through hmc_debug_gemm.  Tolerance: |C - C64| <= 4e-6 * (|A| |B|)_ij (fp32 accumulation over K
plus the 3xTF32 split error ~2^-22 relative per product)."""
import numpy as np
import pytest

from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu

CASES = [
    # (a_kmajor, b_kmajor, M, N, K, batch)
    (True, True, 256, 256, 256, 3),
    (True, True, 300, 200, 100, 2),     # ragged M, N, K (K-major both)
    (True, True, 512, 2048, 256, 1),    # combine shape
    (True, False, 2048, 256, 256, 2),   # input-gradient shape (B N-major)
    (True, False, 512, 256, 2048, 1),   # dB shape
    (False, False, 2048, 256, 512, 1),  # dT shape (A M-major)
    (False, False, 256, 256, 2048, 2),  # weight-gradient shape
    (False, False, 96, 64, 77, 2),      # ragged K, small
    (False, True, 128, 96, 64, 2),
]


def _layout(X, kmajor_rows, rows, cols):
    """Store logical X (rows x cols) as row-major (kmajor_rows) or transposed."""
    return np.ascontiguousarray(X if kmajor_rows else X.T)


@pytest.mark.parametrize("case", CASES, ids=[f"{'K' if c[0] else 'M'}{'K' if c[1] else 'N'}-{c[2]}x{c[3]}x{c[4]}x{c[5]}" for c in CASES])
@pytest.mark.parametrize("engine", [0, 1], ids=["simt", "tcgen05"])
def test_engine_matches_fp64(case, engine):
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    akm, bkm, M, N, K, batch = case
    g = np.random.default_rng(M * 7 + N * 3 + K)
    A = g.normal(size=(batch, M, K)).astype(np.float32)
    B = g.normal(size=(batch, K, N)).astype(np.float32)
    # device layouts
    if akm:
        Ad, lda = A, K                                   # A[m*K + k]
    else:
        Ad, lda = np.ascontiguousarray(A.transpose(0, 2, 1)), M   # A[k*M + m]
    if bkm:
        Bd, ldb = np.ascontiguousarray(B.transpose(0, 2, 1)), K   # B[n*K + k]
    else:
        Bd, ldb = B, N                                   # B[k*N + n]
    tA = torch.as_tensor(Ad, device="cuda").contiguous()
    tB = torch.as_tensor(Bd, device="cuda").contiguous()
    tC = torch.zeros(batch, M, N, dtype=torch.float32, device="cuda")
    try:
        abi.hmc_debug_gemm(engine, akm, bkm, M, N, K, batch, tA, lda, M * K, tB, ldb, K * N, tC, N, M * N)
    except abi.HmcError as e:
        if engine == 1 and e.code == abi.HMC_E_CONFIG:
            pytest.skip("shape not taken by the tcgen05 engine")
        raise
    torch.cuda.synchronize()
    C = tC.cpu().numpy().astype(np.float64)
    ref = np.einsum("bmk,bkn->bmn", A.astype(np.float64), B.astype(np.float64))
    scale = np.einsum("bmk,bkn->bmn", np.abs(A.astype(np.float64)), np.abs(B.astype(np.float64)))
    err = np.abs(C - ref) / scale
    assert err.max() <= 4e-6, (err.max(), np.unravel_index(err.argmax(), err.shape))


def test_tcgen05_engine_takes_the_wide_shapes():
    """The shapes the cfg5 hot path needs must run on the tensor-core engine."""
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    for akm, bkm, M, N, K, batch in CASES[:7]:
        A = torch.zeros(batch * M * K, device="cuda")
        B = torch.zeros(batch * K * N, device="cuda")
        C = torch.zeros(batch * M * N, device="cuda")
        lda = K if akm else M
        ldb = K if bkm else N
        abi.hmc_debug_gemm(1, akm, bkm, M, N, K, batch, A, lda, M * K, B, ldb, K * N, C, N, M * N)
    torch.cuda.synchronize()
