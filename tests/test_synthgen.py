"""The shared input generator: deterministic, shard-consistent, right distribution, RNE bf16."""
import torch

import synthgen as g


def test_shard_equals_slice_of_full_and_head_rows():
    shape = (2, 64, 6, 8)
    full = g.gen_qkv_shard(3, g.TENSOR_K, shape, 0, 64)
    part = g.gen_qkv_shard(3, g.TENSOR_K, shape, 16, 48)
    assert torch.equal(full[:, 16:48].view(torch.int16), part.view(torch.int16))
    rows = g.gen_head_rows(3, g.TENSOR_K, shape, 1, 4, tokens=torch.tensor([0, 5, 63]))
    assert torch.equal(rows.view(torch.int16), full[1, [0, 5, 63], 4].view(torch.int16))


def test_deterministic_and_streams_differ():
    shape = (1, 32, 2, 16)
    a = g.gen_qkv_shard(0, g.TENSOR_Q, shape, 0, 32).view(torch.int16)
    b = g.gen_qkv_shard(0, g.TENSOR_Q, shape, 0, 32).view(torch.int16)
    c = g.gen_qkv_shard(1, g.TENSOR_Q, shape, 0, 32).view(torch.int16)
    d = g.gen_qkv_shard(0, g.TENSOR_V, shape, 0, 32).view(torch.int16)
    assert torch.equal(a, b) and not torch.equal(a, c) and not torch.equal(a, d)


def test_moments_and_distributions():
    shape = (1, 512, 4, 64)
    x = g.gen_qkv_shard(0, g.TENSOR_Q, shape, 0, 512).double()
    assert abs(x.mean().item()) < 0.02 and abs(x.std().item() - 1.0) < 0.02
    assert x.abs().max().item() <= 2 * 3 ** 0.5 + 1e-6          # Irwin-Hall support
    q1 = g.gen_qkv_shard(0, g.TENSOR_Q, shape, 0, 512, dist="D1").double()
    assert abs(q1.std().item() - 4.0) < 0.1
    assert (g.gen_qkv_shard(0, g.TENSOR_Q, shape, 0, 512, dist="D2").double() == 0).all()
    assert (g.gen_qkv_shard(0, g.TENSOR_V, shape, 0, 512, dist="D3").double() == 1).all()
    k4 = g.gen_qkv_shard(0, g.TENSOR_K, shape, 0, 512, dist="D4").double()
    q0 = g.gen_qkv_shard(0, g.TENSOR_Q, shape, 0, 512, dist="D4").double()
    assert abs((k4 - q0).std().item() - 0.5) < 0.02


def test_bf16_rounding_is_rne():
    x = torch.randn(100_000, dtype=torch.float64) * 3
    mine = g.bf16_bits_from_f64(x)
    ref = x.to(torch.float32).to(torch.bfloat16).view(torch.int16)
    assert torch.equal(mine, ref)
    assert torch.equal(g.bf16_bits_to_f64(mine), ref.view(torch.bfloat16).double())


def test_token_counts():
    assert g.tokens_for_video(640, 480, 93) == 28_800
    assert g.tokens_for_video(1024, 576, 129) == 76_032
    assert g.tokens_for_video(1280, 720, 129) == 118_800
