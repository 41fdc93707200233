"""Small invocation of every kernel family for compute-sanitizer:
    compute-sanitizer --tool memcheck python tools/sanitize_run.py
(K1 device + host frames, K2/K3 fp32 + bf16, K4 tail, C4 GEMM + attention +
LayerNorm, denoise, fit, barycentric search; round 2: the tcgen05 projector
kernels at small and large batches -- transposed, persistent, split-bf16 --
with the compacted-corner LBS and multi-mesh bridge, the single-frame API and
the host-read peak kernel)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import projection as pj
    from paper_2603_15603_b200 import runtime as rt
    from paper_2603_15603_b200 import synth

    mhr, smpl, gt = synth.make_toy_models(0, 1200, 600)
    proj = pj.init_projector(pj.make_subsample(600, 150), (64, 32), seed=0)
    scenes = [synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512)) for i in range(5)]
    imgs = np.stack([synth.render_scene(s, smpl) for s in scenes])
    kps = np.stack([s.keypoints2d for s in scenes])
    for prec in ("fp32", "bf16"):
        pipe = pl.Pipeline(dc.Decoder(smpl, dc.DecoderConfig(), seed=40), mhr=mhr, bmap=gt, projector=proj,
                           precision=prec)
        pipe.context().set_graphs(False)
        out = pipe.run_batch(imgs, kps)
        pipe.run_batch(imgs[:1], kps[:1])  # one HBM frame: boxes derived inside the crop CTAs
        out = pipe.run_batch(torch.from_numpy(imgs).pin_memory(), torch.from_numpy(kps).pin_memory())
        torch.cuda.synchronize()
        print(prec, "frame batch ok", out["theta"].shape)
    # hand decoder in both schedules: one-tile CTAs whose two thread groups
    # split the cross-attention keys (10 hands) and two-tile CTAs that run
    # the halves in sequence (80 hands)
    feats = np.random.default_rng(9).normal(size=(80, 64, 64)).astype(np.float32)
    for n in (10, 80):
        pipe.decoder.decode_hand(feats[:n], (), precision="bf16")
    torch.cuda.synchronize()
    print("hand schedules ok")
    # C4 pipeline: 2 layers, 2 crops (SANITIZE_ATTN_ONLY=1: the attention
    # kernel alone, without the GEMMs)
    if os.environ.get("SANITIZE_ATTN_ONLY"):
        import ctypes

        lib = ctypes.CDLL(rt.LIB_PATH)
        P = ctypes.c_void_p
        lib.fsb_debug_attention.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P]
        q = (torch.randn((2 * 576, 3 * 256), device="cuda") * 0.5).to(torch.bfloat16)
        o = torch.empty((2 * 576, 256), dtype=torch.bfloat16, device="cuda")
        assert lib.fsb_debug_attention(q.data_ptr(), 2, 576, 256, 4, o.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
        print("attention ok")
    # round 2: tensor-core projector (hidden 512 / 256) at B = 5 (transposed
    # tile GEMM) and B = 1200 (persistent tile GEMM, 4 meshes per bridge
    # CTA), bf16 and fp32 (split-bf16); single-frame API; host-read kernel
    if not os.environ.get("SANITIZE_SKIP_R2"):
        proj2 = pj.init_projector(pj.make_subsample(600, 300), (512, 256), seed=0)
        nb = 1200
        rng = np.random.default_rng(3)
        p = np.zeros((nb, 76), np.float32)
        p[:, :66] = rng.normal(0.0, 0.2, size=(nb, 66))
        p[:, 66:] = rng.normal(0.0, 0.45, size=(nb, 10))
        for prec in ("bf16", "fp32"):
            pipe = pl.Pipeline(dc.Decoder(smpl, dc.DecoderConfig(), seed=40), mhr=mhr, bmap=gt, projector=proj2,
                               precision=prec)
            c2 = pipe.context()
            c2.set_graphs(False)
            pipe.run_batch(imgs, kps)
            c2.reserve(nb)
            poses = torch.from_numpy(p).cuda()
            v = torch.empty((nb, mhr.num_vertices, 3), device="cuda")
            th = torch.empty((nb, 76), device="cuda")
            j = torch.empty((nb, 22, 3), device="cuda")
            c2.check(c2.lib.fsb_skin_project(c2.h, rt.ptr(poses), nb, rt.ptr(v), rt.ptr(th), rt.ptr(j), None,
                                             rt.PRECISIONS[prec], c2.stream))
            torch.cuda.synchronize()
            c2.check_finite("sanitize c3")
            pipe.run_smpl(imgs[0], scenes[0])
            print(prec, "projector kernels ok")
        import ctypes

        lib = ctypes.CDLL(rt.LIB_PATH)
        lib.fsb_debug_host_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int,
                                            ctypes.c_void_p]
        hb = torch.arange(1 << 18, dtype=torch.float32).pin_memory()
        db = torch.empty_like(hb, device="cuda")
        assert lib.fsb_debug_host_read(hb.data_ptr(), hb.numel() * 4, db.data_ptr(), 8,
                                       torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
        assert torch.equal(db.cpu(), hb)
        print("host read ok")
    cfg = dc.DecoderConfig(crop_size=384, patch=16, dim=1024, heads=16, enc_layers=2, body_layers=1, hand_layers=1)
    ctx = rt.Context()
    ctx.load_decoder(cfg, synth.decoder_weights(cfg, 40, encoder_only=True))
    x = torch.rand((2, 384, 384, 3), device="cuda")
    f = torch.empty((2, 576, 1024), device="cuda")
    if not os.environ.get("SANITIZE_ATTN_ONLY"):
        ctx.check(ctx.lib.fsb_encode(ctx.h, rt.ptr(x), 2, rt.ptr(f), rt.PRECISIONS["bf16"], ctx.stream))
        torch.cuda.synchronize()
        print("vit ok")
    w = pj.DenoiserWeights(*(np.random.default_rng(1).normal(size=s).astype(np.float32) * 0.1
                             for s in ((63, 32), (32,), (32, 63), (63,))))
    pj.denoise(w, np.zeros((5, 63), np.float32))
    v = np.stack([mhr.vertices_rest] * 2)
    pj.fit_batch(v, gt, smpl, pj.FitConfig(steps=3))
    pj.precompute_bary(mhr, smpl)
    torch.cuda.synchronize()
    print("aux ok")
