"""Vector files (reference storage.py:170-186) — host only."""

import os

import numpy as np
import pytest

import paper_1502_01379_b200 as bf
from conftest import GOLDEN


def test_vector_round_trip_and_reference_file(tmp_path):
    g = bf.read_vector(os.path.join(GOLDEN, "g128.vec"))
    assert g.shape == (128,) and g.dtype == np.complex128
    out = tmp_path / "g.vec"
    bf.write_vector(out, g)
    assert open(out, "rb").read() == open(os.path.join(GOLDEN, "g128.vec"), "rb").read()
    with pytest.raises(ValueError):
        bf.write_vector(out, np.zeros((2, 2)))
    out.write_bytes(open(os.path.join(GOLDEN, "g128.vec"), "rb").read() + b"x")
    with pytest.raises(bf.FormatError):
        bf.read_vector(out)
