"""Golden batches from the REFERENCE sampler (faultsim.data.ShardedSampler).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sampler_golden.py

Writes tests/golden/sampler.json and weights_manifest.json (C0 final_weights.json
of the reference dump_weights). sampler.json: for the teacher source and for a corpus
source over a synthetic text (written to a temp file, so the reference's
embedded asset is not needed), three batch() calls per rank plus
eval_windows(). Nothing at test time imports the reference.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from faultsim import data  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def synthetic_text() -> str:
    words = ["node", "failure", "neighbour", "gradient", "rank", "low", "skip", "recompute", "ffn", "step"]
    return " ".join(words[(i * 7 + i // 3) % len(words)] + (".\n" if i % 11 == 10 else "") for i in range(900))


def record(sampler, n_ranks, sizes):
    calls = []
    for bs in sizes:
        for r in range(n_ranks):
            x, y = sampler.batch(r, bs)
            calls.append({"rank": r, "batch": bs, "inputs": x.tolist(), "targets": y.tolist()})
    ev = sampler.eval_windows(0, 5)
    return {"calls": calls, "eval": {"inputs": ev[0].tolist(), "targets": ev[1].tolist()}}


def main():
    out = {}
    args = dict(n_ranks=2, seq_len=12, vocab_size=16, seed=3)
    out["teacher"] = {"args": {**args, "source": "teacher", "teacher_tokens_per_rank": 400},
                      **record(data.ShardedSampler(**args, source="teacher", teacher_tokens_per_rank=400), 2,
                               [4, 1, 7])}
    text = synthetic_text()
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False, encoding="utf-8") as f:
        f.write(text)
    cargs = dict(n_ranks=3, seq_len=10, vocab_size=64, seed=5)
    out["corpus"] = {"args": {**cargs, "source": "corpus"}, "text": text,
                     **record(data.ShardedSampler(**cargs, source="corpus", corpus_path=f.name), 3, [3, 5])}
    os.unlink(f.name)
    with open(os.path.join(OUT, "sampler.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()


def weights_manifest():
    """final_weights.json of the reference dump for C0 init weights (seed 0),
    plus sha256 of the dumped blob rounded to float32 (the engine's master
    precision): tests/golden/weights_manifest.json."""
    import hashlib

    import numpy as np

    from faultsim import harness, model as mdl

    cfg = mdl.ModelConfig(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=2, seq_len=64, rope=True)
    with tempfile.TemporaryDirectory() as d:
        harness.dump_weights(mdl.init_weights(cfg, seed=0), d)
        manifest = json.load(open(os.path.join(d, "final_weights.json")))
        blob = np.fromfile(os.path.join(d, "final_weights.bin"), dtype="<f8")
    manifest["sha256_f32"] = hashlib.sha256(blob.astype("<f4").tobytes()).hexdigest()
    with open(os.path.join(OUT, "weights_manifest.json"), "w") as fh:
        json.dump(manifest, fh)


if __name__ == "__main__":
    weights_manifest()
