"""The .bfac path (bf_plan_load_bfac / bf_plan_save_bfac) against files written
by the reference's own storage.py (tests/golden/*.bfac, oracle/gen_golden.py):
byte-identical round trips, apply after reload, and FormatError offsets
(pkg/tests/test_storage.py:18-75)."""

import os
import shutil

import numpy as np
import pytest

import paper_1502_01379_b200 as bf
from conftest import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FILES = ["fio_n128_r4_leaf025.bfac", "fio_n1024_r8_leaf16.bfac"]


@pytest.mark.parametrize("name", FILES)
def test_load_save_byte_identical(name, tmp_path):
    src = os.path.join(GOLDEN, name)
    f = bf.load_factors(src)
    out = tmp_path / "again.bfac"
    bf.save_factors(f, out)
    assert open(src, "rb").read() == open(out, "rb").read()


def test_apply_after_load_matches_reference():
    f = bf.load_factors(os.path.join(GOLDEN, "fio_n128_r4_leaf025.bfac"))
    g = bf.read_vector(os.path.join(GOLDEN, "g128.vec"))
    want = bf.read_vector(os.path.join(GOLDEN, "u128.vec"))
    got = f.apply(g)
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


def test_save_gpu_built_factors_round_trip(tmp_path):
    p = bf.make_partition(256, 1)
    f = bf.factorize(bf.FioKernel(256), p, 4, seed=5)
    path = tmp_path / "f.bfac"
    bf.save_factors(f, path)
    f2 = bf.load_factors(path)
    assert bf.factors_equal(f, f2)
    path2 = tmp_path / "f2.bfac"
    bf.save_factors(f2, path2)
    assert open(path, "rb").read() == open(path2, "rb").read()


def test_format_errors(tmp_path):
    src = os.path.join(GOLDEN, "fio_n128_r4_leaf025.bfac")
    data = open(src, "rb").read()
    bad = tmp_path / "bad.bfac"
    bad.write_bytes(b"XFAC" + data[4:])
    with pytest.raises(bf.FormatError) as e:
        bf.load_factors(bad)
    assert e.value.offset == 0
    bad.write_bytes(data[:1000])
    with pytest.raises(bf.FormatError) as e:
        bf.load_factors(bad)
    assert 0 < e.value.offset <= 1000
    bad.write_bytes(data + b"\0")
    with pytest.raises(bf.FormatError) as e:
        bf.load_factors(bad)
    assert e.value.offset == len(data)
    # corrupt the column offset of the first block of the first factor: header at 28+13
    corrupt = bytearray(data)
    corrupt[28 + 13 + 8] ^= 0x01
    bad.write_bytes(bytes(corrupt))
    with pytest.raises(bf.FormatError) as e:
        bf.load_factors(bad)
    assert e.value.offset == 28 + 13 + 24


def test_save_rejects_quadtree_chain(tmp_path):
    """The .bfac header carries no branching field (storage.py:65-93): a quadtree chain
    is refused at save time instead of writing a file that cannot be read back."""
    from paper_1502_01379_b200.synthetic import synthetic_chain
    f = synthetic_chain(bf.make_quadtree_partition(32, 2), 4, seed=1)
    with pytest.raises(ValueError, match="binary-tree"):
        bf.save_factors(f, tmp_path / "q.bfac")
    assert not (tmp_path / "q.bfac").exists()
