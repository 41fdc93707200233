"""Run the C3 LBS + projector microbench kernels a few times (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    import bench

    pipe, _ = bench.build_models(sys.argv[1] if len(sys.argv) > 1 else "bf16")
    ctx = pipe.context()
    print(bench.c3_microbench(torch, pipe, ctx, meshes=4096, reps=2))
