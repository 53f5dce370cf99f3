"""Per-rank batch sampling (reference pkg/src/faultsim/data.py).

`ShardedSampler` mirrors data.py:58-116: contiguous corpus shards (or
seeded-bigram teacher streams) per DP rank and one PCG64 stream per rank
seeded with SeedSequence((seed, 0xDA7A, rank)) (data.py:95-98). The window
starts are drawn by the native stream (`pcg.Pcg64Generator`,
libmecefo_ctl.so), so batches are bit-identical to the reference's for the
same seed. The reference's embedded corpus asset (data.py:20-24) is not
shipped: pass `corpus_path` (or `text`) for the corpus source.
"""

from __future__ import annotations

import os

import numpy as np

from .errors import ConfigError
from .pcg import Pcg64Generator

SOURCE_CORPUS = "corpus"
SOURCE_TEACHER = "teacher"


def load_corpus(path: str | None = None) -> str:
    """data.py:20-24. The reference reads its embedded asset
    (faultsim/assets/corpus.txt); this package does not ship a copy, so a
    missing path resolves, in order, to $MECEFO_CORPUS or the asset of an
    installed `faultsim` package, else raises ConfigError (exit code 2)."""
    if path is None:
        path = os.environ.get("MECEFO_CORPUS")
    if path is None:
        try:
            from importlib import resources

            return resources.files("faultsim").joinpath("assets/corpus.txt").read_text("utf-8")
        except Exception:
            raise ConfigError("data.source 'corpus' needs data.path (or $MECEFO_CORPUS): the reference's embedded "
                              "corpus asset is not shipped with this package") from None
    if not os.path.exists(path):
        raise ConfigError(f"dataset path does not exist: {path}")
    with open(path, "r", encoding="utf-8") as f:
        return f.read()


def build_char_vocab(text: str, vocab_size: int) -> dict:
    """data.py:27-33: the corpus's distinct characters in code-point order -> ids."""
    alphabet = sorted(set(text))
    if len(alphabet) > vocab_size:
        raise ConfigError(f"corpus has {len(alphabet)} distinct characters, vocab is {vocab_size}")
    return dict(zip(alphabet, range(len(alphabet))))


def encode(text: str, vocab: dict) -> np.ndarray:
    """data.py:36-40, as one table lookup over the UTF-32 code points."""
    cps = np.frombuffer(text.encode("utf-32-le"), dtype=np.uint32)
    keys = np.array([ord(c) for c in vocab], dtype=np.uint32)
    vals = np.array(list(vocab.values()), dtype=np.int64)
    order = np.argsort(keys)
    keys, vals = keys[order], vals[order]
    pos = np.clip(np.searchsorted(keys, cps), 0, max(len(keys) - 1, 0))
    miss = (keys[pos] != cps) if len(keys) else np.ones(len(cps), bool)
    if miss.any():
        raise ConfigError(f"character {chr(int(cps[np.argmax(miss)]))!r} not in vocabulary")
    return vals[pos]


def teacher_stream(vocab_size: int, length: int, seed: int) -> np.ndarray:
    """data.py:43-55: a walk on a frozen random bigram chain. Draw order on the
    PCG64(seed) stream: V x V Gaussian logits (x2), `length` uniforms, then the
    first token. The table is host init data drawn with numpy (like
    init_weights); each step inverts the row's CDF at the pre-drawn uniform."""
    g = np.random.Generator(np.random.PCG64(seed))
    z = 2.0 * g.normal(size=(vocab_size, vocab_size))
    w = np.exp(z - z.max(axis=1)[:, None])
    cdf = np.cumsum(w / w.sum(axis=1)[:, None], axis=1)
    u = g.random(length)
    tok = np.empty(length, dtype=np.int64)
    tok[0] = g.integers(vocab_size)
    prev = int(tok[0])
    for t in range(1, length):
        prev = int(np.searchsorted(cdf[prev], u[t]))
        tok[t] = prev
    return tok


class ShardedSampler:
    """data.py:58-116 (same constructor arguments and batch semantics)."""

    def __init__(self, n_ranks: int, seq_len: int, vocab_size: int, seed: int, source: str = SOURCE_CORPUS,
                 corpus_path: str | None = None, teacher_tokens_per_rank: int = 20000, text: str | None = None):
        self.seq_len = seq_len
        self.n_ranks = n_ranks
        if source == SOURCE_CORPUS:
            if text is None:
                text = load_corpus(corpus_path)
            self.vocab = build_char_vocab(text, vocab_size)
            tokens = encode(text, self.vocab)
            per = len(tokens) // n_ranks
            self.shards = [tokens[i * per:(i + 1) * per] for i in range(n_ranks)]
        elif source == SOURCE_TEACHER:
            self.vocab = None
            self.shards = [teacher_stream(vocab_size, teacher_tokens_per_rank, seed * 7919 + 13 * i)
                           for i in range(n_ranks)]
        else:
            raise ConfigError(f"unknown data source {source!r}")
        if any(len(s) < seq_len + 2 for s in self.shards):
            raise ConfigError("shard too short for the sequence length")
        self.rngs = [Pcg64Generator((seed, 0xDA7A, i)) for i in range(n_ranks)]

    def _windows(self, shard: np.ndarray, starts: np.ndarray):
        idx = starts[:, None] + np.arange(self.seq_len + 1)[None, :]
        win = shard[idx]
        return win[:, :-1], win[:, 1:]

    def batch(self, rank: int, batch_size: int):
        """data.py:100-107: next (inputs, targets), each (batch, seq_len)."""
        shard = self.shards[rank]
        starts = self.rngs[rank].integers(0, len(shard) - self.seq_len - 1, size=batch_size)
        return self._windows(shard, starts)

    def eval_windows(self, rank: int, count: int):
        """data.py:109-116: evenly spaced fixed windows."""
        shard = self.shards[rank]
        starts = np.linspace(0, len(shard) - self.seq_len - 1, num=count, dtype=np.int64)
        return self._windows(shard, starts)
