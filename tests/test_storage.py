"""SDICT / SDATA / PGM formats (reference storage.py:1-110,
denoising.py:78-106) and the CLI's validation-before-compute (cli.py:277-279);
host-only, no GPU."""

import json
import struct

import numpy as np
import pytest

from paper_1403_4781_b200 import storage
from paper_1403_4781_b200.exceptions import FormatError


def test_sdict_layout_and_round_trip(tmp_path):
    D = np.arange(12, dtype=np.float64).reshape(3, 4) / 7.0
    p = tmp_path / "d.sdict"
    storage.save_dictionary(p, D)
    blob = p.read_bytes()
    magic, r, c = struct.unpack("<8sII", blob[:16])
    assert magic == b"SDICT\x00v1" and (r, c) == (3, 4)
    assert np.array_equal(np.frombuffer(blob[16:], "<f8"), D.ravel(order="F"))
    assert np.array_equal(storage.load_dictionary(p), D)
    with pytest.raises(FormatError):
        storage.load_dataset(p)                    # wrong magic


def test_sdata_truncated_and_short_header(tmp_path):
    p = tmp_path / "y.sdata"
    storage.save_dataset(p, np.ones((2, 5)))
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(FormatError):
        storage.load_dataset(p)
    p.write_bytes(b"SDATA")
    with pytest.raises(FormatError):
        storage.load_dataset(p)
    with pytest.raises(FormatError):
        storage.save_dataset(p, np.ones(3))


def test_pgm_round_trip_clamps_and_rounds(tmp_path):
    from paper_1403_4781_b200.denoising import GrayImage
    img = GrayImage(np.array([[-3.0, 0.5, 1.49], [254.5, 300.0, 128.0]]))
    p = tmp_path / "a.pgm"
    storage.save_pgm(img, p)
    assert p.read_bytes().startswith(b"P5\n3 2\n255\n")
    back = storage.load_pgm(p)
    assert np.array_equal(back.pixels, [[0, 1, 1], [255, 255, 128]])
    p.write_bytes(b"P5\n# comment\n3 2\n255\n" + bytes(6))
    assert storage.load_pgm(p).pixels.shape == (2, 3)
    p.write_bytes(b"P2\n3 2\n255\n")
    with pytest.raises(FormatError):
        storage.load_pgm(p)
    p.write_bytes(b"P5\n3 2\n65535\n" + bytes(12))
    with pytest.raises(FormatError):
        storage.load_pgm(p)


def test_manifest_fields(tmp_path):
    path = storage.write_manifest(tmp_path, "train", seed=5, config_path="c.json", inputs=["y"],
                                  outputs=["d"], extra={"threads": 2})
    m = json.loads(path.read_text())
    assert {"command", "config", "seed", "inputs", "outputs", "tool_version", "timestamp", "threads"} <= set(m)


def test_cli_rejects_bad_config_before_compute(tmp_path, capsys):
    from paper_1403_4781_b200 import cli
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"K": 8, "s": 2, "bogus": 1}))
    data = tmp_path / "y.sdata"
    storage.save_dataset(data, np.ones((4, 10)))
    rc = cli.main(["train", "--data", str(data), "--config", str(cfg), "--out", str(tmp_path / "o")])
    assert rc == 1 and "bogus" in capsys.readouterr().err
    spec = tmp_path / "g.json"
    spec.write_text(json.dumps({"m": 4, "K": 8, "N": 20, "s": 9}))
    assert cli.main(["gen", "--config", str(spec), "--out", str(tmp_path / "g")]) == 1
