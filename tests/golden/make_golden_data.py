"""Golden batches of the reference's data path (F/data.py): the token-file task
(FileTask: truncation, length ordering, bucketed greedy grouping, copy objective)
and the synthetic copy / reverse tasks, written to tests/golden/data.npz.

Runs in the build container only (imports the reference read-only from
/root/reference/pkg/src); the committed fixture is what the tests read.
    python tests/golden/make_golden_data.py
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"


def token_lines(seed: int = 5, n: int = 37, vocab: int = 50, max_len: int = 30):
    rng = np.random.default_rng(seed)
    lines = []
    for i in range(n):
        L = int(rng.integers(1, max_len + 6))        # some longer than max_len: truncated
        lines.append(" ".join(str(int(t)) for t in rng.integers(0, vocab, L)))
        if i % 9 == 4:
            lines.append("")                         # blank lines are skipped
    return "\n".join(lines) + "\n"


def main():
    sys.path.insert(0, REF)
    from ftrain.config import RunConfig
    from ftrain.data import FileTask, SyntheticTask
    out = {}
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "tokens.txt")
        with open(path, "w") as fh:
            fh.write(token_lines())
        out["file_text"] = np.frombuffer(token_lines().encode(), dtype=np.uint8)
        run = RunConfig()
        run.model.vocab, run.model.max_len = 50, 24
        run.train.batch_tokens = 96
        run.data.task, run.data.path = "file", path
        ft = FileTask(run)
        out["file_n"] = np.array([len(ft.batches)])
        for i, b in enumerate(ft.batches):
            for k in ("src", "tgt_in", "tgt_out", "src_len"):
                out[f"file_{i}_{k}"] = np.asarray(getattr(b, k))
    for task in ("copy", "reverse"):
        run = RunConfig()
        run.data.task = task
        st = SyntheticTask(run)
        for step in (0, 1, 7):
            b = st.batch(step)
            for k in ("src", "tgt_in", "tgt_out", "src_len"):
                out[f"{task}_{step}_{k}"] = np.asarray(getattr(b, k))
    np.savez_compressed(os.path.join(OUT, "data.npz"), **out)
    print("wrote", os.path.join(OUT, "data.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
