import os,sys
sys.path.insert(0,'.')
import torch, bench
pipe,_=bench.build_models("bf16"); ctx=pipe.context()
print(bench.c3_microbench(torch,pipe,ctx,meshes=4096,reps=20))
