"""B200-native (sm_100a) implementation of the Fast SAM 3D Body accelerated
inference path, keeping the reference ``fsb`` package's Python API.

Modules mirror the reference layout (pkg/src/fsb/):

  numkit      error types, FSB1 files, stand-alone bilinear sampling
  bodymodel   templates, FK and LBS (GPU)
  priors      keypoint stub, body/hand boxes, crop grids (GPU, bit-exact)
  decoder     frozen encoder + pruned body/hand decoders (GPU)
  projection  barycentric bridge and MHR -> SMPL projector (GPU)
  pipeline    plans, Pipeline.run / run_fast / run_batch (+ SMPL tail)

``import paper_2603_15603_b200 as fsb`` gives a drop-in for the fast path.
The compute runs in ``lib/libfsb_b200.so`` (csrc/, C ABI in
include/fsb_b200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"
