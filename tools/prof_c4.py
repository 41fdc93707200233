"""Run the C4 ViT-L-sized encoder a few times (for ncu): python tools/prof_c4.py [crops] [layers]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    import bench

    crops = int(sys.argv[1]) if len(sys.argv) > 1 else 768
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    print(bench.c4_microbench(torch, crops=crops, reps=1, layers=layers))
