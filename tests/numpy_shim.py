"""numpy <-> CUDA shim for the reference's unit tests (SURVEY §8(b) "what calls it").

The reference's tests call `ftrain.kernels` / `ftrain.gradients` with numpy
arrays and compare numpy results.  The mirror modules accept numpy inputs
(they are uploaded to the device) but return CUDA tensors; `NumpyAPI(module)`
wraps every function of a mirror module so that

  * numpy arrays passed as `out=`, `accumulate_into=` or any `*_out=` argument
    are replaced by device tensors for the call and written back in place
    afterwards (the reference's in-place output contract);
  * every torch tensor in the result (also inside tuples and cache / mask
    objects) comes back as a numpy array, one array per distinct tensor, so
    identity checks such as `cache.probs is y` keep their meaning.

Test infrastructure only: tests/test_gpu_reftests.py uses it to restate the
reference's test_kernels.py / test_gradients.py / test_trainer.py against the
CUDA path.
"""

from __future__ import annotations

import copy
import dataclasses

import numpy as np
import torch


def _is_out_name(name: str) -> bool:
    return name in ("out", "accumulate_into") or name.endswith("_out")


class _Converter:
    def __init__(self):
        self.memo: dict = {}

    def __call__(self, x):
        if isinstance(x, torch.Tensor):
            key = (x.data_ptr(), tuple(x.shape), x.dtype)
            if key not in self.memo:
                self.memo[key] = x.detach().cpu().numpy()
            return self.memo[key]
        if isinstance(x, tuple):
            return tuple(self(v) for v in x)
        if isinstance(x, list):
            return [self(v) for v in x]
        if dataclasses.is_dataclass(x) and not isinstance(x, type):
            y = copy.copy(x)
            for f in dataclasses.fields(x):
                setattr(y, f.name, self(getattr(x, f.name)))
            return y
        if hasattr(x, "keep") and hasattr(x, "p") and hasattr(x, "bitmask"):   # DropoutMask
            return _HostMask(x, self(x.keep))
        return x


class _HostMask:
    """A DropoutMask seen from the test: numpy `keep`; handed back to the mirror
    it unwraps to the device mask it came from."""

    def __init__(self, dev_mask, keep):
        self._ls2_orig = dev_mask
        self.keep = keep
        self.p = dev_mask.p


def _unwrap(v):
    return getattr(v, "_ls2_orig", v)


def wrap(fn):
    def call(*args, **kwargs):
        back = []
        for k, v in list(kwargs.items()):
            if _is_out_name(k) and isinstance(v, np.ndarray):
                t = torch.from_numpy(np.ascontiguousarray(v)).cuda()
                kwargs[k] = t
                back.append((v, t))
        args = tuple(_unwrap(a) for a in args)
        kwargs = {k: _unwrap(v) for k, v in kwargs.items()}
        res = fn(*args, **kwargs)
        conv = _Converter()
        for arr, t in back:
            host = t.detach().cpu().numpy()
            arr[...] = host.reshape(arr.shape)
            conv.memo[(t.data_ptr(), tuple(t.shape), t.dtype)] = arr
        return conv(res)
    call.__name__ = getattr(fn, "__name__", "call")
    call.__doc__ = getattr(fn, "__doc__", None)
    return call


class NumpyAPI:
    """Attribute access to a mirror module with numpy in / numpy out functions."""

    def __init__(self, module):
        self._m = module

    def __getattr__(self, name):
        v = getattr(self._m, name)
        if callable(v) and not isinstance(v, type) and getattr(v, "__module__", "") == self._m.__name__:
            return wrap(v)
        return v


def host(x) -> np.ndarray:
    """A device tensor (or anything array-like) as a numpy array."""
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)
