"""Large-config encoder (ViT-L size: S=384, p=16, D=1024,
16 heads) on the tcgen05 path: flash attention alone against a float64
reference, and the 2-layer encoder against the reference's golden rows
(tools/make_golden.py "c4.l2.feats_rows", Decoder.encode decoder.py:231)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# bf16 operands (LN output, q/k/v, P, context, MLP hidden) against the
# reference's fp32: relative L2 error of the final features
VIT_REL_L2 = 2e-2


def _vitl(layers=2):
    from paper_2603_15603_b200 import decoder as dc

    return dc.DecoderConfig(crop_size=384, patch=16, dim=1024, heads=16, enc_layers=layers, body_layers=1,
                            hand_layers=1)


def _attention_ref(qkv, crops, T, D, H):
    out = np.empty((crops * T, D))
    dh = D // H
    for c in range(crops):
        r = slice(c * T, (c + 1) * T)
        for h in range(H):
            q = qkv[r, h * dh:(h + 1) * dh]
            k = qkv[r, D + h * dh:D + (h + 1) * dh]
            v = qkv[r, 2 * D + h * dh:2 * D + (h + 1) * dh]
            s = q @ k.T / np.sqrt(dh)
            p = np.exp(s - s.max(axis=1, keepdims=True))
            out[r, h * dh:(h + 1) * dh] = (p / p.sum(axis=1, keepdims=True)) @ v
    return out


@pytest.mark.parametrize("crops,T,D", [(1, 128, 128), (2, 200, 128), (2, 576, 256), (1, 576, 1024)])
def test_flash_attention(crops, T, D):
    import torch

    from paper_2603_15603_b200 import runtime as rt

    H = D // 64
    rng = np.random.default_rng(T + D)
    x = (rng.standard_normal((crops * T, 3 * D)) * 1.5).astype(np.float32)
    bits = rt.to_bf16_bits(x)
    ref = _attention_ref(rt.bf16_bits_to_f32(bits).astype(np.float64), crops, T, D, H)
    lib = ctypes.CDLL(rt.LIB_PATH)
    P = ctypes.c_void_p
    lib.fsb_debug_attention.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P]
    dq = torch.from_numpy(bits.view(np.int16)).cuda()
    out = torch.zeros((crops * T, D), dtype=torch.int16, device="cuda")
    assert lib.fsb_debug_attention(dq.data_ptr(), crops, T, D, H, out.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    got = rt.bf16_bits_to_f32(out.cpu().numpy().view(np.uint16)).astype(np.float64)
    err = np.abs(got - ref).max()
    assert err < 2e-2 * np.abs(ref).max() + 1e-2, err


@pytest.fixture(scope="module")
def vit_ctx():
    from paper_2603_15603_b200 import runtime as rt
    from paper_2603_15603_b200 import synth

    cfg = _vitl(2)
    ctx = rt.Context()
    ctx.load_decoder(cfg, synth.decoder_weights(cfg, 40, encoder_only=True))
    return ctx, cfg


def _encode(ctx, crops):
    import torch

    from paper_2603_15603_b200 import runtime as rt

    x = torch.from_numpy(np.ascontiguousarray(crops, np.float32)).cuda()
    out = torch.empty((crops.shape[0], 576, 1024), dtype=torch.float32, device="cuda")
    ctx.check(ctx.lib.fsb_encode(ctx.h, rt.ptr(x), crops.shape[0], rt.ptr(out), rt.PRECISIONS["bf16"], ctx.stream),
              "encode")
    torch.cuda.synchronize()
    return out.cpu().numpy()


def test_vitl_two_layers_golden(vit_ctx, golden):
    ctx, _ = vit_ctx
    crop = np.random.default_rng(0).random((1, 384, 384, 3)).astype(np.float32)
    got = _encode(ctx, crop)[0, ::36]
    want = golden["c4.l2.feats_rows"].astype(np.float64)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert np.isfinite(got).all()
    assert rel < VIT_REL_L2, rel


def test_vitl_batch_independence(vit_ctx):
    """A crop's features do not depend on what else is in the batch."""
    ctx, _ = vit_ctx
    rng = np.random.default_rng(5)
    crops = rng.random((3, 384, 384, 3)).astype(np.float32)
    many = _encode(ctx, crops)
    one = _encode(ctx, crops[1:2])
    assert np.array_equal(many[1], one[0])


def test_vitl_chunk_boundary(vit_ctx):
    """More crops than one encoder pass (fsb_capi.cu kVitChunk = 256): crops on
    both sides of the pass boundary and in the ragged last pass equal solo runs."""
    import torch

    from paper_2603_15603_b200 import runtime as rt

    ctx, _ = vit_ctx
    n = 260
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.rand((n, 384, 384, 3), generator=g, device="cuda")
    out = torch.empty((n, 576, 1024), dtype=torch.float32, device="cuda")
    ctx.check(ctx.lib.fsb_encode(ctx.h, rt.ptr(x), n, rt.ptr(out), rt.PRECISIONS["bf16"], ctx.stream), "encode")
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    for i in (0, 255, 256, n - 1):
        one = _encode(ctx, x[i:i + 1].cpu().numpy())
        assert np.array_equal(out[i].cpu().numpy(), one[0]), i


def test_vitl_fp32_reference_precision(vit_ctx, golden):
    """precision='fp32' runs the large config on the CUDA cores in fp32
    (k_enc_f32.cu): the reference's arithmetic type, held to the fp32 bar."""
    import torch

    from paper_2603_15603_b200 import runtime as rt

    ctx, _ = vit_ctx
    crop = np.random.default_rng(0).random((1, 384, 384, 3)).astype(np.float32)
    x = torch.from_numpy(crop).cuda()
    out = torch.empty((1, 576, 1024), dtype=torch.float32, device="cuda")
    ctx.check(ctx.lib.fsb_encode(ctx.h, rt.ptr(x), 1, rt.ptr(out), rt.PRECISIONS["fp32"], ctx.stream), "encode")
    torch.cuda.synchronize()
    got = out.cpu().numpy()[0, ::36]
    want = golden["c4.l2.feats_rows"]
    err = np.abs(got.astype(np.float64) - want).max() / np.abs(want).max()
    assert err <= 1e-4, err


@pytest.mark.parametrize("cfgkw", [dict(crop_size=32, patch=8, dim=32, heads=2, enc_layers=2),
                                   dict(crop_size=48, patch=16, dim=96, heads=3, enc_layers=1),
                                   dict(crop_size=64, patch=8, dim=128, heads=1, enc_layers=1)])
def test_any_config_fp32_encoder(cfgkw):
    """Decoder.encode at fp32 for configurations outside the fused default
    kernels (reference decoder.py:231-260 accepts any DecoderConfig), against
    the oracle on the same seeded weights."""
    import oracle as orc
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import synth

    cfg = dc.DecoderConfig(body_layers=1, hand_layers=1, **cfgkw)
    dec = dc.Decoder(synth.make_toy_models(0, 252, 168)[1], cfg, seed=40)
    crops = np.random.default_rng(3).random((5, cfg.crop_size, cfg.crop_size, 3)).astype(np.float32)
    got = dec.encode(crops, precision="fp32")
    want = orc.encode(dec.weights, cfg, crops)
    err = np.abs(got.astype(np.float64) - want).max() / np.abs(want).max()
    assert err <= 1e-4, err
