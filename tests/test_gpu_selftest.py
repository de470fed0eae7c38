"""tcgen05 / SW128 descriptor self-test: one UMMA tile per operand-major combination the
GLA kernels use, checked against a float32 torch matmul of the same bf16 values."""

import pytest
import torch

pytestmark = pytest.mark.gpu

# (M, N, K, a_mn, b_mn, lane_off): every (shape, major) pair used by fast_fwd.cu / fast_bwd.cu
CASES = [
    (128, 128, 64, 1, 1, 0),   # K^T V state contribution (both MN-major)
    (64, 64, 128, 0, 0, 0),    # Q K^T scores (both K-major), M=64
    (64, 64, 128, 0, 0, 16),   # same, second half-subpartition tile
    (64, 128, 64, 0, 1, 0),    # A V  (A K-major, V MN-major)
    (64, 128, 128, 0, 0, 0),   # Q S  (S stored [dv][dk], K-major)
    (64, 128, 128, 0, 1, 0),   # Q S  (S stored [dk][dv], MN-major)
    (64, 128, 64, 1, 1, 0),    # A^T dO (both MN-major), M=64
    (128, 64, 64, 1, 1, 0),    # dk^T = Qh^T dPm, dv^T = dO^T Am
    (128, 64, 64, 1, 0, 0),    # dq^T = Kh^T dPm^T
    (128, 64, 128, 0, 0, 0),   # dq^T += S' dO^T, dk^T += D' V^T
    (128, 64, 128, 1, 0, 0),   # dv^T += D'^T Kh^T
    (128, 128, 128, 0, 0, 0),
]


@pytest.mark.parametrize("M,N,K,a_mn,b_mn,lane_off", CASES)
def test_umma_tile(M, N, K, a_mn, b_mn, lane_off):
    from paper_2507_01004_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K + a_mn * 2 + b_mn + lane_off)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
    a_store = A.t().contiguous() if a_mn else A.contiguous()      # MN-major: [K][M]
    b_store = B.contiguous() if b_mn else B.t().contiguous()      # MN-major: [K][N], K-major: [N][K]
    D = ops.selftest_mma(a_store, b_store, M, N, K, a_mn, b_mn, lane_off)
    ref = A.float() @ B.float()
    err = (D - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), f"max abs err {err}"
