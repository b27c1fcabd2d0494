"""Checkpoint interoperability fixtures written by the REFERENCE (LSF2, F/checkpoint.py).

Run in the build container (needs /root/reference, read-only):

    python tests/golden/make_golden_ckpt.py

Writes
  * ref_ckpt_step40.lsf2 — the reference engine's own checkpoint (F/engine.py:189-208)
    of the default copy-task job (p_drop 0.1) after 40 training steps;
  * ref_ckpt_tail.npz    — that job's uninterrupted losses for steps 40..47, its
    params16 after step 47, and the reference's applied-step count;
  * ref_ckpt_format.lsf2 — a small checkpoint of fixed tensors (f16 and f32, ranks
    0..3, an empty tensor), written by the reference's save_checkpoint, so the CPU
    tests can check this repo's writer byte for byte against the reference's.
The GPU box never has /root/reference; tests read only these files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
RESUME_AT, TAIL = 40, 8


def format_tensors():
    """The fixed tensors of ref_ckpt_format.lsf2 (shared with the CPU test)."""
    rng = np.random.default_rng(5)
    return [("params16", rng.normal(size=37).astype(np.float16)),
            ("moments_m", rng.normal(size=(3, 5)).astype(np.float32)),
            ("scalar", np.array(2.5, dtype=np.float32)),
            ("cube", rng.normal(size=(2, 3, 4)).astype(np.float16)),
            ("empty", np.zeros((0, 4), dtype=np.float32)),
            ("applied_steps", np.array([7.0], dtype=np.float32))]


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    from ftrain import checkpoint as C
    from ftrain.config import RunConfig
    from ftrain.engine import TrainingEngine

    C.save_checkpoint(os.path.join(OUT, "ref_ckpt_format.lsf2"), 123456789, format_tensors())

    run = RunConfig()
    run.train.p_drop = 0.1
    eng = TrainingEngine(run)
    eng.setup_arena()
    for s in range(RESUME_AT):
        eng.train_step(s)
    eng.save(os.path.join(OUT, f"ref_ckpt_step{RESUME_AT}.lsf2"), RESUME_AT)
    tail = [eng.train_step(s).loss for s in range(RESUME_AT, RESUME_AT + TAIL)]
    np.savez_compressed(os.path.join(OUT, "ref_ckpt_tail.npz"), losses=np.array(tail),
                        params16=eng.ws.params16.copy(),
                        applied=np.array([eng.applied_steps]))
    print("wrote checkpoint fixtures under", OUT)


if __name__ == "__main__":
    main()
