"""`python -m paper_2510_16415_b200 train` mirrors `faultsim train`
(reference cli.py:36-165): outputs and exit codes 0/2/3/4."""

import json
import os

import numpy as np
import pytest

from paper_2510_16415_b200 import cli, harness

C0 = {"model": {"vocab": 64, "hidden": 128, "heads": 4, "ffn_intermediate": 344, "layers": 2, "seq_len": 64},
      "cluster": {"dp": 2, "pp": 2, "layers": 2},
      "scenario": {"kind": "per_iteration", "probability": 1.0, "recovery_iterations": 1000000000,
                   "victims": [[0, 1]]},
      "run": {"iterations": 3, "global_batch": 4, "seed": 0, "r": 32, "tau": 100, "probe_interval": 0},
      "data": {"source": "teacher"}}


def _write(tmp_path, cfg):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(cfg))
    return str(p)


def test_config_errors_exit_2(tmp_path, capsys):
    assert cli.main(["train", "--config", str(tmp_path / "missing.json"), "--quiet"]) == cli.EXIT_CONFIG
    bad = dict(C0, bogus={})
    assert cli.main(["train", "--config", _write(tmp_path, bad), "--quiet"]) == cli.EXIT_CONFIG
    bad = json.loads(json.dumps(C0))
    bad["run"]["global_batch"] = 3  # not divisible by dp
    assert cli.main(["train", "--config", _write(tmp_path, bad), "--quiet"]) == cli.EXIT_CONFIG
    assert "config error" in capsys.readouterr().err


def test_seed_override_reseeds_failure_stream(tmp_path):
    args = cli.build_parser().parse_args(["train", "--config", _write(tmp_path, C0), "--seed", "5"])
    cfg = cli.load_run_config(args)
    assert cfg.run.seed == 5 and cfg.scenario.seed == 5 * 31 + 7
    assert harness.config_from_dict(C0).scenario.seed == 7


def test_make_sampler_selects_reference_sampler():
    from paper_2510_16415_b200 import data

    assert isinstance(harness.make_sampler(harness.config_from_dict(C0)), data.ShardedSampler)
    syn = json.loads(json.dumps(C0))
    syn["data"]["source"] = "synthetic"
    assert isinstance(harness.make_sampler(harness.config_from_dict(syn)), harness.SyntheticSampler)


@pytest.mark.gpu
def test_train_writes_reference_outputs(tmp_path):
    out = tmp_path / "run"
    assert cli.main(["train", "--config", _write(tmp_path, C0), "--out", str(out), "--quiet"]) == cli.EXIT_OK
    lines = (out / "metrics.csv").read_text().splitlines()
    assert lines[0] == harness.METRICS_HEADER and len(lines) == 1 + C0["run"]["iterations"]
    events = [json.loads(x) for x in (out / "events.jsonl").read_text().splitlines()]
    assert events and events[0]["kind"] == "fail" and events[0]["node"] == [0, 1]
    manifest = json.loads((out / "final_weights.json").read_text())
    blob = np.fromfile(out / "final_weights.bin", dtype="<f8")
    assert manifest["dtype"] == "<f8" and blob.size == manifest["total_elems"] and np.isfinite(blob).all()


@pytest.mark.gpu
def test_unrecoverable_cluster_exit_4(tmp_path, capsys):
    cfg = json.loads(json.dumps(C0))
    cfg["cluster"] = {"dp": 1, "pp": 2, "layers": 2}
    cfg["run"]["global_batch"] = 2
    cfg["scenario"] = {"kind": "per_iteration", "probability": 1.0, "recovery_iterations": 1000000000}
    assert cli.main(["train", "--config", _write(tmp_path, cfg), "--quiet"]) == cli.EXIT_UNRECOVERABLE
    assert "unrecoverable" in capsys.readouterr().err


def test_data_defaults_follow_reference(tmp_path, monkeypatch):
    """harness.py:54-56: the default source is the corpus; harness.py:74-75:
    a configured data.path must exist (ConfigError -> exit 2)."""
    assert harness.DataSettings().source == "corpus"
    bad = json.loads(json.dumps(C0))
    bad["data"] = {"source": "corpus", "path": str(tmp_path / "nope.txt")}
    with pytest.raises(harness.ConfigError):
        harness.config_from_dict(bad)
    assert cli.main(["train", "--config", _write(tmp_path, bad), "--quiet"]) == cli.EXIT_CONFIG
    # corpus without a path and no asset available: explicit ConfigError, not a traceback
    from paper_2510_16415_b200 import data

    monkeypatch.delenv("MECEFO_CORPUS", raising=False)
    monkeypatch.setattr("importlib.resources.files", lambda pkg: (_ for _ in ()).throw(ModuleNotFoundError(pkg)))
    with pytest.raises(harness.ConfigError, match="data.path"):
        data.load_corpus(None)
