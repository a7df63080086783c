"""The command line end to end on the GPU path (reference cli.py:50-283):
gen -> train (split-and-merge) -> eval -> denoise, with the reference's
file formats, report and manifest. The CLI's dictionary equals the Python
API's for the same inputs (exact mode), bit for bit."""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gen_train_eval_denoise(tmp_path, capsys):
    import paper_1403_4781_b200 as sdb
    from paper_1403_4781_b200 import cli, storage
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps({"m": 16, "K": 32, "N": 600, "s": 3, "seed": 4}))
    assert cli.main(["gen", "--config", str(spec), "--out", str(tmp_path / "g")]) == 0
    Y = storage.load_dataset(tmp_path / "g" / "training_set.sdata")
    assert Y.shape == (16, 600)
    cfg = tmp_path / "train.json"
    conf = {"K": 32, "s": 6, "iterations": 3, "seed": 1, "mode": "split-merge", "L": 2, "K1": 32,
            "s1": 3, "s2": 2}
    cfg.write_text(json.dumps(conf))
    assert cli.main(["train", "--data", str(tmp_path / "g" / "training_set.sdata"), "--config", str(cfg),
                     "--out", str(tmp_path / "t")]) == 0
    D = storage.load_dictionary(tmp_path / "t" / "dictionary.sdict")
    rep = json.loads((tmp_path / "t" / "report.json").read_text())
    assert set(rep) == {"config", "report"} and len(rep["report"]["local_wall_times_s"]) == 2
    assert json.loads((tmp_path / "t" / "manifest.json").read_text())["command"] == "train"
    D2, _ = sdb.train_split_merge(Y, sdb.TrainConfig.from_dict(dict(conf)))
    assert np.array_equal(D, D2)
    capsys.readouterr()
    assert cli.main(["eval", "--dict", str(tmp_path / "t" / "dictionary.sdict"), "--truth-dict",
                     str(tmp_path / "g" / "truth_dictionary.sdict"), "--data",
                     str(tmp_path / "g" / "training_set.sdata"), "--sparsity", "3"]) == 0
    res = json.loads(capsys.readouterr().out)
    assert "atom_recovery_pct" in res and "mse_db" in res
    # denoise a small synthetic image with an overcomplete DCT dictionary
    rng = np.random.default_rng(0)
    clean = np.clip(128 + 60 * np.sin(np.arange(40)[None, :] / 5.0) + np.zeros((36, 40)), 0, 255)
    storage.save_pgm(sdb.GrayImage(clean), tmp_path / "clean.pgm")
    storage.save_pgm(sdb.GrayImage(clean + rng.normal(0, 10, clean.shape)), tmp_path / "noisy.pgm")
    storage.save_dictionary(tmp_path / "dct.sdict", sdb.overcomplete_dct(8, 256))
    assert cli.main(["denoise", "--in", str(tmp_path / "noisy.pgm"), "--dict", str(tmp_path / "dct.sdict"),
                     "--sigma", "10", "--out", str(tmp_path / "den" / "out.pgm"), "--reference",
                     str(tmp_path / "clean.pgm")]) == 0
    out = capsys.readouterr().out
    assert "output PSNR" in out
    a = float(out.split("input PSNR")[1].split("dB")[0])
    b = float(out.split("output PSNR")[1].split("dB")[0])
    assert b > a
