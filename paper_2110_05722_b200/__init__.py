"""B200-native (sm_100a) LightSeq2 training hot path.

Drop-in for the reference `ftrain` operator API (F/__init__.py:9-18):
fused non-GEMM kernels, embedding, criterion and workspace trainer in a C-ABI
CUDA library (include/ls2.h, lib/libls2.so), GEMMs on cuBLAS, Python host
layer mirroring the reference modules.
"""

__version__ = "0.1.0"

_LAZY = {
    "Batch": "model", "ModelConfig": "model", "Transformer": "model",
    "transformer_forward_backward": "model", "OptimConfig": "trainer", "Workspace": "trainer",
    "workspace_pack": "trainer", "RunConfig": "config", "TrainingEngine": "engine",
}

__all__ = sorted(_LAZY)


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f"{__name__}.{mod}"), name)
