"""GLA model wrapper: geometry and parameter count of the 1.3B configuration (no GPU work)."""

import torch

from paper_2507_01004_b200.layer import GLA_1P3B, GLAModel, model_flops_per_token, num_params


def test_gla_1p3b_geometry_on_meta_device():
    m = GLAModel(GLA_1P3B, device="meta")
    n = num_params(m)
    assert 1.3e9 < n < 1.5e9, n
    assert GLA_1P3B.hidden // GLA_1P3B.heads == 128  # the fused tcgen05 head size
    blk = m.blocks[0].attn
    assert tuple(blk.w_qkvr.shape) == (2048, 4 * 2048) and blk.bg.dtype == torch.float32
    assert model_flops_per_token(GLA_1P3B) > 6 * 1.2e9
