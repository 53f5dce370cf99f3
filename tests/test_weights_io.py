"""final_weights.bin/.json wire format (reference harness.py:635-665 dump_weights
/ load_weights; test_harness.py:153-165 round trip). CPU: the packer against the
reference's own C0 manifest (tests/golden/weights_manifest.json, made by
tests/golden/make_sampler_golden.py). GPU: device dump -> load round trip."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import model_ref as R
from paper_2510_16415_b200 import errors, harness, model as mdl

G = os.path.join(os.path.dirname(__file__), "golden")
C0 = mdl.ModelConfig(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=2, seq_len=64)


def _host_store():
    layout, total = mdl._param_layout(C0)
    W = R.init_params(R.Dims(64, 128, 4, 344, 2, 64), 0)
    host = np.full(total, np.nan, dtype=np.float32)  # padding must never reach the blob
    for name, shape, off in layout:
        host[off: off + int(np.prod(shape))] = np.asarray(W[name], dtype=np.float32).reshape(-1)
    return layout, total, host


def test_pack_matches_reference_manifest_and_blob():
    ref = json.load(open(os.path.join(G, "weights_manifest.json")))
    layout, total, host = _host_store()
    blob, manifest = harness.pack_weights(layout, host)
    assert manifest["dtype"] == ref["dtype"] and manifest["total_elems"] == ref["total_elems"]
    assert manifest["params"] == ref["params"]
    assert blob.dtype == np.dtype("<f8") and blob.size == ref["total_elems"]
    assert hashlib.sha256(blob.astype("<f4").tobytes()).hexdigest() == ref["sha256_f32"]


def test_unpack_inverts_pack_and_checks_contract():
    layout, total, host = _host_store()
    blob, manifest = harness.pack_weights(layout, host)
    back = harness.unpack_weights(layout, total, blob, manifest)
    for name, shape, off in layout:
        n = int(np.prod(shape))
        assert np.array_equal(back[off: off + n], host[off: off + n]), name
    bad = json.loads(json.dumps(manifest))
    bad["params"][1]["shape"] = [1, 2]
    with pytest.raises(errors.ContractViolation):
        harness.unpack_weights(layout, total, blob, bad)
    with pytest.raises(errors.ContractViolation):
        harness.unpack_weights(layout, total, blob[:-5], manifest)
    short = dict(manifest, params=manifest["params"][:-1])
    with pytest.raises(errors.ContractViolation):
        harness.unpack_weights(layout, total, blob, short)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_device_dump_load_round_trip(tmp_path, precision):
    ref = json.load(open(os.path.join(G, "weights_manifest.json")))
    w = mdl.init_weights(C0, 0, precision=precision)
    harness.dump_weights(w, str(tmp_path))
    blob = np.fromfile(os.path.join(tmp_path, "final_weights.bin"), dtype="<f8")
    assert hashlib.sha256(blob.astype("<f4").tobytes()).hexdigest() == ref["sha256_f32"]
    assert os.path.getsize(os.path.join(tmp_path, "final_weights.bin")) == 8 * ref["total_elems"]
    back = harness.load_weights(C0, str(tmp_path), precision=precision)
    for name, arr in w.named():
        assert bool((arr == back.get(name)).all()), name
    if precision == "bf16":
        assert bool((w.shadow == back.shadow).all())
