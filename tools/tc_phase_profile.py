"""Cycle attribution of CTA 0 of the tcgen05 encoder / decoder kernels (needs
a library built with FSB_PROFILE=1): total, MMA waits, weight waits, issue
barriers and LayerNorm exchange barriers for thread 0 (the MMA / TMA issuer)
and thread 255; the remainder is the thread's own work (epilogues)."""

import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import priors as pr
    from paper_2603_15603_b200 import runtime

    pipe, (mhr, smpl, gt, dec, proj) = bench.build_models("bf16")
    ctx = pipe.context()
    ctx.set_graphs(False)
    scenes = bench.make_scenes(smpl, bench.frame_seeds(0, 32))
    images = pr.render_scenes(scenes)
    kps = torch.from_numpy(np.stack([s.keypoints2d for s in scenes])).cuda()
    outs = pipe.allocate_outputs(32, tail=True)
    for _ in range(3):
        pipe.launch(images, kps, outs, pl.fast_config())
    torch.cuda.synchronize()
    lib = ctypes.CDLL(runtime.LIB_PATH)
    buf = (ctypes.c_ulonglong * 96)()
    rc = lib.fsb_debug_tc_profile(buf)
    names = ["total", "mma_wait", "weight_wait", "issue_bar", "xch_bar"]
    for role, tag in ((0, "encoder"), (1, "body decoder"), (2, "hand decoder")):
        for th, tname in ((0, "t0"), (1, "t255")):
            v = [buf[role * 32 + th * 16 + i] for i in range(16)]
            rest = v[0] - sum(v[1:5])
            print(tag, tname, "rc", rc,
                  " ".join("%s=%d(%.1f%%)" % (n, x, 100.0 * x / max(v[0], 1)) for n, x in zip(names, v)),
                  "work=%d(%.1f%%)" % (rest, 100.0 * rest / max(v[0], 1)))
            if role == 0:
                print("   encoder: setup+patchify+embed=%d [start->patchified=%d embed wait+GEMM=%d] self-attn=%d "
                      "mlp=%d final-LN+out=%d kv-projection=%d" % (v[8], v[10], v[11], v[5], v[7], v[9], v[6]))
            if role >= 1:
                other = v[0] - v[5] - v[6] - v[7]
                print("   sub-layers: self=%d cross=%d mlp=%d other=%d [setup+final=%d pos+params=%d heads=%d fk=%d]"
                      % (v[5], v[6], v[7], other, v[8], v[9], v[10], v[11]))
            print("   self-attn: LN=%d QKV gemm+wait=%d drains=%d attn_core=%d out_proj=%d"
                  % (v[12], v[13], v[14], v[15], v[5] - v[12] - v[13] - v[14] - v[15]))


if __name__ == "__main__":
    main()
