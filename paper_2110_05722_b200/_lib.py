"""ctypes binding of the C-ABI library (include/ls2.h) and per-device context.

The product path has no CPU fallback: if libls2.so is missing or no CUDA
device is present, every operator raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import STATUS_TO_ERROR, DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libls2.so")

F16, BF16, F32, F64 = 0, 1, 2, 3
MASK_NONE, MASK_CAUSAL, MASK_PADDING, MASK_DENSE = 0, 1, 2, 3

_TORCH_CODE = {torch.float16: F16, torch.bfloat16: BF16, torch.float32: F32, torch.float64: F64}
I32 = 4             # collectives only (LS2_I32)

P = ctypes.c_void_p
I = ctypes.c_int
L = ctypes.c_int64
U = ctypes.c_uint64
D = ctypes.c_double
Fl = ctypes.c_float

# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGS = {
    "ls2_last_error": [],
    "ls2_version": [],
    "ls2_copy_spans": [P, P, P, I, P],
    "ls2_num_kernels_launched": [P],
    "ls2_rand_uniform": [P, U, L, L, P],
    "ls2_dropout_bits": [P, L, U, P, U, P],
    "ls2_dropout_bits_multi": [P, I, L, P, P, U, P, P, P],
    "ls2_dropout_bits_multi_ex": [P, I, L, P, P, U, P, P, I, P],
    "ls2_bits_to_dense": [P, P, I, L, P],
    "ls2_dense_to_bits": [P, I, P, L, P],
    "ls2_bias_dropout_residual_fwd": [P, P, P, P, P, L, L, I, I, U, P, U, D, I, I, P],
    "ls2_bias_dropout_residual_bwd": [P, P, P, P, I, I, P, L, L, I, D, I, I, P],
    "ls2_bias_relu_dropout_fwd": [P, P, P, P, P, L, L, I, I, U, P, U, D, I, I, P],
    "ls2_bias_relu_dropout_bwd": [P, P, P, P, P, I, I, P, L, L, I, D, I, I, P],
    "ls2_colsum_ws_bytes": [L, L],
    "ls2_colsum": [P, I, P, I, I, P, L, L, P],
    "ls2_bias_add": [P, P, L, L, I, P],
    "ls2_layernorm_fwd": [P, P, P, P, P, P, P, L, L, D, I, I, I, P],
    "ls2_layernorm_bwd_ws_bytes": [L, L],
    "ls2_layernorm_bwd": [P, P, P, P, P, P, P, P, P, I, I, P, L, L, I, I, I, P],
    "ls2_bdr_layernorm_fwd": [P, P, P, P, P, P, P, P, P, P, L, L, D, I, U, P, U, D, I, I, I, P],
    "ls2_layernorm_bwd_bdr": [P, P, P, P, P, P, P, P, P, I, D, P, P, P, I, I, P, L, L, I, I, I, P],
    "ls2_softmax_fwd": [P, P, L, L, I, L, L, P, P, D, P, I, I, P],
    "ls2_softmax_bwd": [P, P, P, L, L, D, I, I, P],
    "ls2_log_softmax_fwd": [P, P, L, L, I, I, P],
    "ls2_softmax_fwd_strategy": [P, P, L, L, I, L, L, P, P, D, P, I, I, I, P],
    "ls2_log_softmax_fwd_strategy": [P, P, L, L, I, I, I, P],
    "ls2_ls_ce_fwd": [P, P, P, P, P, L, L, D, L, I, I, P],
    "ls2_ls_ce_bwd": [P, P, P, P, L, L, D, L, I, D, I, I, P],
    "ls2_criterion_fused": [P, P, P, P, P, P, P, L, L, D, L, I, D, I, P],
    "ls2_criterion_fused_ld": [P, L, P, P, P, P, P, L, L, D, L, I, D, I, P],
    "ls2_attention_supported": [L, L, L, I],
    "ls2_attention_fwd": [P, L, P, L, P, L, P, P, L, L, L, L, L, L, I, P, D, P],
    "ls2_attention_bwd": [P, L, P, L, P, L, P, P, L, P, L, P, L, P, L, L, L, L, L, L, D, P],
    "ls2_attention_bwd_bias": [P, L, P, L, P, L, P, P, L, P, L, P, L, P, L, L, L, L, L, L, D,
                               P, L, P, L, P, L, P],
    "ls2_attention_tc_supported": [L, L, L, I],
    "ls2_attention_tc_trace": [P],
    "ls2_attention_tc_fwd": [P, L, P, L, P, L, P, P, L, L, L, L, L, L, I, P, D, P],
    "ls2_attention_tc_bwd": [P, L, P, L, P, L, P, P, L, P, L, P, L, P, L, L, L, L, L, L, I, P, D,
                             P, L, P, L, P, L, P],
    "ls2_attention_tc_bwd_o": [P, L, P, L, P, L, P, L, P, P, L, P, L, P, L, P, L, L, L, L, L, L, I,
                               P, D, P, L, P, L, P, L, P],
    "ls2_embedding_fwd": [P, P, P, P, P, P, L, L, L, L, D, I, I, U, P, U, D, I, I, P],
    "ls2_embedding_bwd": [P, P, P, P, P, I, I, L, L, L, L, D, I, D, I, P],
    "ls2_adam": [P, P, P, P, L, P, P, L, L, P, P, P, P],
    "ls2_adam_spans": [P, P, P, P, P, L, L, P, P, L, L, P, P, P, P],
    "ls2_sgd": [P, P, P, L, P, P, P, P],
    "ls2_step_commit": [P, P, P, P, P],
    "ls2_step_report": [P, P, P, P, P],
    "ls2_scale_narrow": [P, P, L, D, P, L, Fl, P, P],
    "ls2_count_nonfinite_f16": [P, L, P, P],
    "ls2_finish_narrow": [P, P, L, P, P, D, P, L, Fl, P, P],
    "ls2_finish_acc32": [P, P, L, P, P, P],
    "ls2_colsum_nblk": [L, L, I],
    "ls2_layernorm_bwd_nblk": [L, L],
    "ls2_blas_create": [],
    "ls2_blas_destroy": [P],
    "ls2_gemm": [P, I, I, L, L, L, D, P, L, L, L, P, L, L, L, D, P, L, L, L, L, L, I, I, P, I, P],
    "ls2_gemm_list": [P, I, I, L, L, L, D, P, L, P, L, D, P, L, I, I, I, P, I, P],
    "ls2_gemm_lt": [P, I, I, L, L, L, D, P, L, P, L, D, P, L, P, I, I, P],
    "ls2_gemm_lt_bgrad": [P, I, I, L, L, L, D, P, L, P, L, D, P, L, P, I, I, I, P],
    "ls2_gemm_scratch_bytes": [L, L],
    "ls2_gemm_tc_supported": [I, I, L, L, L, P, L, P, L, D, P, L, I, I],
    "ls2_gemm_tc": [I, I, L, L, L, D, P, L, P, L, D, P, L, P, I, I, I, P],
    "ls2_wgrad_tc_split": [L, L, L],
    "ls2_wgrad_tc": [P, L, P, L, P, L, L, L, L, I, P],
    "ls2_comm_load": [ctypes.c_char_p],
    "ls2_comm_version": [P],
    "ls2_comm_unique_id": [P],
    "ls2_comm_init": [P, I, I, P, I],
    "ls2_comm_allreduce": [P, P, P, L, I, P],
    "ls2_comm_reduce_scatter": [P, P, P, L, I, P],
    "ls2_comm_all_gather": [P, P, P, L, I, P],
    "ls2_comm_destroy": [P],
}
_RESTYPES = {"ls2_last_error": ctypes.c_char_p, "ls2_blas_create": P, "ls2_blas_destroy": None,
             "ls2_colsum_ws_bytes": L, "ls2_layernorm_bwd_ws_bytes": L,
             "ls2_attention_supported": ctypes.c_int,
             "ls2_attention_tc_supported": ctypes.c_int, "ls2_colsum_nblk": ctypes.c_int,
             "ls2_layernorm_bwd_nblk": ctypes.c_int, "ls2_wgrad_tc_split": ctypes.c_int,
             "ls2_gemm_tc_supported": ctypes.c_int,
             "ls2_gemm_scratch_bytes": L}

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load libls2.so (torch is imported first so its CUDA libraries win)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(f"native library missing: {path} (run python -m "
                              "paper_2110_05722_b200.build)")
        lib = ctypes.CDLL(path)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
        return lib


def exported_symbols():
    return list(_SIGS)


def call(name: str, *args):
    """Invoke an ls2_* entry point; raise the mapped exception on failure."""
    lib = _lib or load_library()
    rc = getattr(lib, name)(*args)
    if rc:
        msg = lib.ls2_last_error().decode(errors="replace")
        raise STATUS_TO_ERROR.get(rc, DeviceError)(f"{name}: {msg}")
    return rc


def call_i64(name: str, *args) -> int:
    """Invoke a size-query entry point returning int64."""
    lib = _lib or load_library()
    return int(getattr(lib, name)(*args))


def dtype_code(t) -> int:
    dt = t.dtype if isinstance(t, torch.Tensor) else t
    try:
        return _TORCH_CODE[dt]
    except KeyError:
        raise STATUS_TO_ERROR[7](f"unsupported dtype {dt}") from None


def ptr(t):
    return None if t is None else t.data_ptr()


def stream_handle():
    return torch.cuda.current_stream().cuda_stream


def launches() -> int:
    v = ctypes.c_int64(0)
    (_lib or load_library()).ls2_num_kernels_launched(ctypes.byref(v))
    return v.value


class DeviceContext:
    """Per-device native state: cuBLAS handle and reusable scratch buffers.

    Scratch buffers are shared by consecutive kernels on the compute stream
    (stream order makes the reuse safe) and only ever grow, so a captured
    CUDA graph keeps valid addresses.
    """

    def __init__(self, device: torch.device):
        load_library()
        self.device = device
        with torch.cuda.device(device):
            self.blas = _lib.ls2_blas_create()
        if not self.blas:
            raise DeviceError("cuBLAS init failed: " + _lib.ls2_last_error().decode())
        self._scratch: dict[str, torch.Tensor] = {}
        self._keep: list[torch.Tensor] = []
        self.ptr_cache: dict = {}        # pointer arrays of pointer-array GEMM batches
        self.lt_unsupported: set = set()  # cuBLASLt keys that fell back
        # side lane for off-critical-path work (weight-gradient GEMMs): lowest
        # priority, its own cuBLAS handle + workspace so the two streams never
        # share a GEMM workspace
        # (torch clamps out-of-range priorities: +100 -> lowest, -100 -> highest)
        self.side_stream = torch.cuda.Stream(device=device, priority=100)
        self.compute_stream = torch.cuda.Stream(device=device, priority=-100)
        self._blas_side = None

    @property
    def blas_side(self):
        if self._blas_side is None:
            with torch.cuda.device(self.device):
                self._blas_side = _lib.ls2_blas_create()
            if not self._blas_side:
                raise DeviceError("cuBLAS init failed: " + _lib.ls2_last_error().decode())
        return self._blas_side

    def blas_handle(self):
        """cuBLAS plan/workspace handle for the current stream."""
        if torch.cuda.current_stream(self.device) == self.side_stream:
            return self.blas_side
        return self.blas

    def scratch(self, name: str, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        buf = self._scratch.get(name)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                self._keep.append(buf)   # may still be referenced by a captured graph
            buf = torch.empty(nbytes + (nbytes >> 2), dtype=torch.uint8, device=self.device)
            self._scratch[name] = buf
        return buf


_contexts: dict[int, DeviceContext] = {}


def context(device=None) -> DeviceContext:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       torch.device(device).index or 0)
    ctx = _contexts.get(dev.index)
    if ctx is None:
        ctx = _contexts[dev.index] = DeviceContext(dev)
    return ctx
