"""Error types, array conventions and the FSB1 array-file format.

Mirrors the public surface of the reference ``fsb.numkit`` that callers of the
hot path touch (reference pkg/src/fsb/numkit.py:31-71 for the error classes
and array helpers, :247-276 for FSB1).  The numeric kernels themselves
(matmul, bilinear_sample, layer_norm, softmax) run on the GPU inside the fused
stage kernels in ``csrc/``; ``bilinear_sample`` below is the stand-alone entry
the reference exposes (numkit.py:136) and dispatches to the CUDA gather.
"""

from __future__ import annotations

import struct

import numpy as np

DTYPE = np.float32


class ShapeError(ValueError):
    """Operand dimensions do not match the kernel contract (numkit.py:33)."""


class NumericError(ArithmeticError):
    """Non-finite values reached a kernel boundary (numkit.py:37)."""


class UsageError(RuntimeError):
    """API misuse or malformed inputs (numkit.py:41)."""


def asarray(x) -> np.ndarray:
    """C-contiguous float32 view/copy, the reference array convention."""
    return np.ascontiguousarray(x, dtype=DTYPE)


def check_finite(arr, op):
    if not np.all(np.isfinite(arr)):
        raise NumericError("%s: non-finite values in operand" % op)


def bilinear_sample(image, grid):
    """Edge-clamped bilinear lookup of image (H, W, C) at grid (..., 2).

    Same contract as numkit.bilinear_sample (numkit.py:136-154): taps are
    floor/clamped exactly, each product and sum is rounded separately, and a
    lattice grid reduces to an exact gather.  Runs the CUDA gather kernel.
    """
    from . import runtime

    image = asarray(image)
    grid = asarray(grid)
    if image.ndim != 3 or grid.ndim < 1 or grid.shape[-1] != 2 or grid.size == 0:
        raise ShapeError("bilinear_sample: image %r, grid %r" % (image.shape, grid.shape))
    check_finite(image, "bilinear_sample")
    check_finite(grid, "bilinear_sample")
    return runtime.bilinear_sample(image, grid)


# ---------------------------------------------------------------------------
# FSB1: b'FSB1' | u32 rank | u32 dims[rank] | little-endian float32 payload

FSB1_MAGIC = b"FSB1"


def write_fsb1(path, arr):
    a = np.ascontiguousarray(arr, dtype="<f4")
    head = FSB1_MAGIC + struct.pack("<I", a.ndim) + struct.pack("<%dI" % a.ndim, *a.shape)
    with open(path, "wb") as fh:
        fh.write(head)
        fh.write(a.tobytes())


def read_fsb1(path) -> np.ndarray:
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < 8 or blob[:4] != FSB1_MAGIC:
        raise UsageError("%s: not an FSB1 file" % path)
    (rank,) = struct.unpack_from("<I", blob, 4)
    if rank > 32:
        raise UsageError("%s: implausible rank %d" % (path, rank))
    off = 8 + 4 * rank
    if len(blob) < off:
        raise UsageError("%s: truncated FSB1 header" % path)
    dims = struct.unpack_from("<%dI" % rank, blob, 8)
    count = int(np.prod(dims, dtype=np.int64)) if rank else 1
    if len(blob) != off + 4 * count:
        raise UsageError("%s: payload size mismatch" % path)
    return np.frombuffer(blob, dtype="<f4", count=count, offset=off).reshape(dims).astype(DTYPE)
