"""Token batches (F/data.py): synthetic copy/reverse tasks as pure functions of
(seed, step), length bucketing to multiples of 4, and a fixed-shape synthetic
WMT-like task for benchmarking.  Host-side numpy (the batch is uploaded by the
engine through pinned buffers)."""

from __future__ import annotations

import numpy as np

from .errors import DataError, ParseError, TokenOutOfRange
from .model import Batch
from .numerics import derive_seed, _finalize, _PHI, _MASK64

LEN_BUCKET = 4


def _uniform(seed: int, n: int) -> np.ndarray:
    """Host splitmix64 draws (same stream as the device RNG)."""
    i = np.arange(n, dtype=np.uint64)
    z = np.uint64(seed & _MASK64) + i * np.uint64(_PHI)
    z ^= z >> np.uint64(30)
    z *= np.uint64(0xBF58476D1CE4E5B9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return (z >> np.uint64(11)).astype(np.float64) / float(1 << 53)


def bucket_len(m: int, max_len: int) -> int:
    """Padded length of a batch whose longest sequence is m (F/data.py:46-48):
    the next multiple of LEN_BUCKET while that fits max_len, otherwise
    max_len itself (or m, for an over-long sequence)."""
    up = LEN_BUCKET * ((m + LEN_BUCKET - 1) // LEN_BUCKET)
    return up if up <= max_len else max(m, max_len)


def bos_id(pad_id: int, vocab: int) -> int:
    """Beginning-of-sequence id: the id after pad, wrapping at vocab."""
    return (pad_id + 1) % vocab


def payload_range(pad_id: int, vocab: int) -> list:
    """Ids a synthetic sequence may contain: all but pad and bos, ascending."""
    ids = np.arange(vocab)
    keep = (ids != pad_id) & (ids != bos_id(pad_id, vocab))
    return ids[keep].tolist()


def _parse_line(path: str, lineno: int, text: str, vocab: int):
    toks = text.split()
    if not toks:
        return None
    try:
        ids = list(map(int, toks))
    except ValueError:
        raise ParseError(f"{path}:{lineno}: non-integer token") from None
    lo, hi = min(ids), max(ids)
    if lo < 0:
        raise ParseError(f"{path}:{lineno}: negative token id")
    if hi >= vocab:
        raise TokenOutOfRange(f"{path}:{lineno}: token id >= vocab ({vocab})")
    return ids


def load_token_file(path: str, vocab: int) -> list:
    """Sequences of a token file (F/data.py:22-43): one per non-blank line,
    whitespace-separated ids in [0, vocab); same exceptions and messages."""
    try:
        text = open(path).read()
    except OSError as exc:
        raise DataError(f"cannot read {path}: {exc}") from exc
    parsed = (_parse_line(path, n, line, vocab) for n, line in enumerate(text.splitlines(), 1))
    return [ids for ids in parsed if ids is not None]


class SyntheticTask:
    """copy / reverse batches as a pure function of (seed, step) (F/data.py:61-102).

    Lengths come from counter-RNG stream 101, payload symbols from stream 102
    (one draw per padded cell, row-major); the batch is assembled with
    whole-array index arithmetic rather than a per-sequence loop.
    """

    def __init__(self, run_cfg):
        model, train, data = run_cfg.model, run_cfg.train, run_cfg.data
        if model.vocab < 4:
            raise DataError("synthetic tasks need vocab >= 4")
        self.task = data.task
        self.pad_id = data.pad_id
        self.bos = bos_id(data.pad_id, model.vocab)
        self.symbols = np.asarray(payload_range(data.pad_id, model.vocab))
        self.min_len = max(1, data.min_len)
        self.max_len = model.max_len
        self.batch_size = max(1, train.batch_tokens // model.max_len)
        self.seed = train.seed

    def possible_shapes(self) -> list:
        lens = range(self.min_len, self.max_len + 1)
        return [(self.batch_size, L) for L in sorted(set(bucket_len(n, self.max_len) for n in lens))]

    def batch(self, step: int) -> Batch:
        nseq = self.batch_size
        nlen = self.max_len - self.min_len + 1
        lens = self.min_len + np.floor(_uniform(derive_seed(self.seed, step, 101), nseq) * nlen).astype(np.int64)
        width = bucket_len(int(lens.max()), self.max_len)
        draw = _uniform(derive_seed(self.seed, step, 102), nseq * width)
        payload = self.symbols[np.floor(draw * len(self.symbols)).astype(np.int64)].reshape(nseq, width)
        col = np.arange(width)[None, :]
        inside = col < lens[:, None]
        if self.task == "copy":
            target = payload
        else:                                  # position j reads payload[n - 1 - j]
            target = np.take_along_axis(payload, np.where(inside, lens[:, None] - 1 - col, 0), 1)
        src = np.where(inside, payload, self.pad_id).astype(np.int64)
        tgt_out = np.where(inside, target, self.pad_id).astype(np.int64)
        shifted = np.concatenate([np.full((nseq, 1), self.bos), target[:, :-1]], axis=1)
        tgt_in = np.where(inside, shifted, self.pad_id).astype(np.int64)
        return Batch(src=src, tgt_in=tgt_in, tgt_out=tgt_out, src_len=lens, pad_id=self.pad_id)


class FixedShapeTask:
    """Benchmark batches: B x L tokens uniform in [2, V), full-length sequences
    (4096 target tokens for 64 x 64), a pure function of (seed, step)."""

    def __init__(self, batch: int, length: int, vocab: int, seed: int = 0, pad_id: int = 0):
        self.b, self.l, self.v, self.seed, self.pad_id = batch, length, vocab, seed, pad_id
        self.bos = bos_id(pad_id, vocab)

    def possible_shapes(self) -> list:
        return [(self.b, self.l)]

    def batch(self, step: int) -> Batch:
        u = _uniform(derive_seed(self.seed, step, 7), 2 * self.b * self.l)
        tok = (2 + (u * (self.v - 2)).astype(np.int64)).reshape(2, self.b, self.l)
        src, tgt = tok[0], tok[1]
        tgt_in = np.concatenate([np.full((self.b, 1), self.bos, np.int64), tgt[:, :-1]], axis=1)
        return Batch(src=src, tgt_in=tgt_in, tgt_out=tgt.copy(),
                     src_len=np.full(self.b, self.l, np.int64), pad_id=self.pad_id)


class MLMTask:
    """Masked-LM batches for the BERT-shaped encoder (BASELINE.json configs[3]):
    B x L ids uniform in [2, V); each position is an MLM position with
    probability `mask_prob` (counter RNG), its input replaced by `mask_id` and
    its target the original id; every other target is pad.  A pure function of
    (seed, step)."""

    def __init__(self, batch: int, length: int, vocab: int, seed: int = 0, pad_id: int = 0,
                 mask_prob: float = 0.15, mask_id: int = 1):
        self.b, self.l, self.v, self.seed, self.pad_id = batch, length, vocab, seed, pad_id
        self.mask_prob, self.mask_id = mask_prob, mask_id

    def possible_shapes(self) -> list:
        return [(self.b, self.l)]

    def batch(self, step: int) -> Batch:
        n = self.b * self.l
        u = _uniform(derive_seed(self.seed, step, 11), 2 * n)
        tok = (2 + (u[:n] * (self.v - 2)).astype(np.int64)).reshape(self.b, self.l)
        mlm = (u[n:] < self.mask_prob).reshape(self.b, self.l)
        src = np.where(mlm, self.mask_id, tok)
        tgt = np.where(mlm, tok, self.pad_id)
        return Batch(src=src, tgt_in=src.copy(), tgt_out=tgt,
                     src_len=np.full(self.b, self.l, np.int64), pad_id=self.pad_id)


class FileTask:
    """Copy objective over the sequences of a token file (F/data.py:105-155):
    sequences truncated to max_len, ordered by length (stable), grouped greedily
    so a group padded to its bucketed length stays within batch_tokens; the
    batches are precomputed and step s takes batch s mod count."""

    def __init__(self, run_cfg):
        m, t, d = run_cfg.model, run_cfg.train, run_cfg.data
        self.pad_id = d.pad_id
        self.bos = bos_id(d.pad_id, m.vocab)
        seqs = [s[:m.max_len] for s in load_token_file(d.path, m.vocab) if s]
        if not seqs:
            raise DataError(f"no usable sequences in {d.path}")
        self.batches = self._group(seqs, t.batch_tokens, m.max_len)

    def _group(self, seqs, batch_tokens: int, max_len: int) -> list:
        out, cur, longest = [], [], 0
        for i in sorted(range(len(seqs)), key=lambda j: len(seqs[j])):
            s = seqs[i]
            lb = bucket_len(max(longest, len(s)), max_len)
            if cur and lb * (len(cur) + 1) > batch_tokens:
                out.append(self._pack(cur, max_len))
                cur, longest = [], 0
            cur.append(s)
            longest = max(longest, len(s))
        if cur:
            out.append(self._pack(cur, max_len))
        return out

    def _pack(self, group, max_len: int) -> Batch:
        lb = bucket_len(max(len(s) for s in group), max_len)
        b = len(group)
        src = np.full((b, lb), self.pad_id, dtype=np.int64)
        tgt_in = src.copy()
        tgt_out = src.copy()
        lens = np.array([len(s) for s in group], dtype=np.int64)
        for i, s in enumerate(group):
            n = len(s)
            src[i, :n] = s
            tgt_out[i, :n] = s
            tgt_in[i, 0] = self.bos
            tgt_in[i, 1:n] = s[:n - 1]
        return Batch(src=src, tgt_in=tgt_in, tgt_out=tgt_out, src_len=lens, pad_id=self.pad_id)

    def possible_shapes(self) -> list:
        return sorted({tuple(np.asarray(b.src).shape) for b in self.batches})

    def batch(self, step: int) -> Batch:
        return self.batches[step % len(self.batches)]


class WmtShapedTask:
    """Synthetic WMT-shaped batches: per step, a bucket length is
    drawn with the counter RNG (lengths 8..max_len, bucketed to multiples of 4,
    F/data.py:19,46-48) and the batch packs as many sequences of that bucket as fit
    batch_tokens (the FileTask grouping rule); real lengths inside a batch vary,
    the rest is padding.  A pure function of (seed, step), so resume is exact."""

    def __init__(self, batch_tokens: int, max_len: int, vocab: int, seed: int = 0,
                 pad_id: int = 0, min_len: int = 8):
        self.tokens, self.max_len, self.v, self.seed = batch_tokens, max_len, vocab, seed
        self.pad_id, self.bos = pad_id, bos_id(pad_id, vocab)
        self.min_len = min_len
        self.buckets = sorted({bucket_len(m, max_len) for m in range(min_len, max_len + 1)})

    def possible_shapes(self) -> list:
        return [(max(1, self.tokens // lb), lb) for lb in self.buckets]

    def batch(self, step: int) -> Batch:
        u = _uniform(derive_seed(self.seed, step, 9), 1)[0]
        lb = self.buckets[min(int(u * len(self.buckets)), len(self.buckets) - 1)]
        b = max(1, self.tokens // lb)
        r = _uniform(derive_seed(self.seed, step, 10), b * (lb + 1))
        lens = np.maximum(lb - 3, 1) + (r[:b] * min(4, lb)).astype(np.int64)
        lens = np.minimum(lens, lb)
        tok = 2 + (r[b:] * (self.v - 2)).astype(np.int64).reshape(b, lb)
        src = np.full((b, lb), self.pad_id, dtype=np.int64)
        tgt_in, tgt_out = src.copy(), src.copy()
        for i in range(b):
            n = int(lens[i])
            src[i, :n] = tok[i, :n]
            tgt_out[i, :n] = tok[i, :n]
            tgt_in[i, 0] = self.bos
            tgt_in[i, 1:n] = tok[i, :n - 1]
        return Batch(src=src, tgt_in=tgt_in, tgt_out=tgt_out, src_len=lens, pad_id=self.pad_id)


def make_task(run_cfg):
    if run_cfg.data.task == "file":
        return FileTask(run_cfg)
    if run_cfg.data.task == "fixed":
        m = run_cfg.model
        return FixedShapeTask(max(1, run_cfg.train.batch_tokens // m.max_len), m.max_len, m.vocab,
                              run_cfg.train.seed, run_cfg.data.pad_id)
    return SyntheticTask(run_cfg)
