"""ANMG container round trips and compatibility with the reference's own
Field.dump/load (field.py:81-108)."""
import os
import sys

import numpy as np
import pytest

from paper_1307_2036_b200 import fieldio

REF = "/root/reference/pkg/src"


def test_round_trip(tmp_path):
    a = np.random.default_rng(0).standard_normal((8, 8, 3))
    p = tmp_path / "f.bin"
    fieldio.dump_array(p, a)
    assert np.array_equal(fieldio.load_array(p), a)
    halo = np.zeros((10, 10, 3))
    halo[1:-1, 1:-1] = a
    fieldio.dump_array(p, halo, has_halo=True)
    assert np.array_equal(fieldio.load_array(p), a)


def test_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"XXXX" + bytes(16))
    with pytest.raises(ValueError):
        fieldio.load_array(p)
    fieldio.dump_array(p, np.ones((2, 2, 2)))
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(ValueError):
        fieldio.load_array(p)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_compatible_with_reference_field(tmp_path):
    sys.path.insert(0, REF)
    from panelmg.field import Field
    a = np.random.default_rng(1).standard_normal((4, 4, 5))
    p1 = tmp_path / "ours.bin"
    fieldio.dump_array(p1, a)
    assert np.array_equal(Field.load(p1).owned, a)
    p2 = tmp_path / "theirs.bin"
    Field.from_owned(a).dump(p2, include_halo=True)
    assert np.array_equal(fieldio.load_array(p2), a)
