"""Numerics of the drop-in boundary (F/numerics.py): counter RNG, seeds, fp16.

The RNG is the reference's splitmix64 over (seed, index), evaluated on the
GPU by libls2 (bit-identical to F/numerics.py:139-155); seed derivation is a
host-side integer function because it feeds kernel arguments.
"""

from __future__ import annotations

import math
import struct

import numpy as np
import torch

from . import _lib

_MASK64 = (1 << 64) - 1
_PHI = 0x9E3779B97F4A7C15


def _finalize(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def derive_seed(base: int, *tags: int) -> int:
    """Per-site stream seed (F/numerics.py:158-163)."""
    h = base & _MASK64
    for t in tags:
        h = _finalize((h + _PHI + (t & _MASK64)) & _MASK64)
    return h


def rand_uniform(seed: int, index: int) -> float:
    """Scalar draw, host side (F/numerics.py:139-142)."""
    return (_finalize((seed + index * _PHI) & _MASK64) >> 11) / float(1 << 53)


def rand_uniform_array(seed: int, start: int, count: int, device=None) -> torch.Tensor:
    """float64 draws for indices start..start+count-1, generated on the GPU."""
    ctx = _lib.context(device)
    out = torch.empty(count, dtype=torch.float64, device=ctx.device)
    _lib.call("ls2_rand_uniform", out.data_ptr(), seed & _MASK64, start, count,
              _lib.stream_handle())
    return out


def keep_threshold(p: float) -> int:
    """keep iff (mix >> 11) >= ceil(p * 2^53)  <=>  rand >= p (exact)."""
    return int(math.ceil(p * float(1 << 53)))


def narrow_f32(x) -> torch.Tensor:
    """binary32 -> binary16, RNE (F/numerics.py:115-121)."""
    x = torch.as_tensor(x)
    return x.to(torch.float32).to(torch.float16)


def widen_f16(x) -> torch.Tensor:
    """binary16 -> binary32, exact (F/numerics.py:124-126)."""
    return torch.as_tensor(x).to(torch.float16).to(torch.float32)


def b32_to_b16_bits(x: float) -> int:
    """Host scalar conversion returning the binary16 bit pattern."""
    return int(np.array([x], dtype=np.float32).astype(np.float16).view(np.uint16)[0])


def b16_bits_to_b32(bits: int) -> float:
    return float(np.array([bits], dtype=np.uint16).view(np.float16).astype(np.float32)[0])


def f32(x: float) -> float:
    """Round a Python float to binary32 (numpy's np.float32(x))."""
    return struct.unpack("<f", struct.pack("<f", x))[0]
