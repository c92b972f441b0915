"""Output formats beside the path (reference densefield.py:202-251): MRDF
field files and the node CSV, byte-identical to what the reference writes
(tests/golden/formats.npz holds the reference's own bytes).  Host I/O only."""
import os

import numpy as np
import pytest

import paper_1411_2141_b200 as mrb
from conftest import golden


def test_mrdf_bytes_and_roundtrip(tmp_path):
    g, f = golden("gen64"), golden("formats")
    field = mrb.DenseField(g["ux"], g["uy"])
    path = tmp_path / "f.mrdf"
    mrb.save_field(field, str(path))
    assert path.read_bytes() == f["mrdf"].tobytes()
    back = mrb.load_field(str(path))
    assert back.shape == field.shape
    assert np.array_equal(back.ux, g["ux"].astype(np.float32).astype(np.float64))
    assert np.array_equal(back.uy, g["uy"].astype(np.float32).astype(np.float64))


def test_mrdf_errors(tmp_path):
    good = golden("formats")["mrdf"].tobytes()
    cases = {"trunc": (good[:10], "truncated field file"),
             "magic": (b"XXXX" + good[4:], "bad field magic"),
             "version": (good[:4] + (2).to_bytes(4, "little") + good[8:],
                         "unsupported field version 2"),
             "size": (good + b"\0", f"has {len(good) + 1} bytes, expected {len(good)}")}
    for name, (blob, msg) in cases.items():
        p = tmp_path / f"{name}.mrdf"
        p.write_bytes(blob)
        with pytest.raises(mrb.FileFormatError, match=msg):
            mrb.load_field(str(p))
    assert issubclass(mrb.FileFormatError, ValueError)


def test_node_csv_matches_reference(tmp_path):
    g, f = golden("gen64"), golden("formats")

    class M:  # duck-typed mesh: only .vertices is read
        vertices = g["V"]

    p = tmp_path / "u.csv"
    mrb.save_node_displacements_csv(M, g["u"], str(p))
    assert p.read_text(encoding="ascii") == str(f["csv"])


def test_difference_image():
    a = mrb.ImageGrid(3, 2, np.arange(6.0))
    b = mrb.ImageGrid(3, 2, np.full(6, 2.5))
    d = mrb.difference_image(a, b)
    assert np.array_equal(d.data, np.abs(np.arange(6.0) - 2.5).reshape(2, 3))
    with pytest.raises(ValueError, match="dimension mismatch"):
        mrb.difference_image(a, mrb.ImageGrid(2, 3, np.zeros(6)))
