"""Instance formats (ref tests/test_data.py): Dataset contract and FVEC."""

import numpy as np
import pytest

from paper_1212_2287_b200 import (DataFormatError, Dataset, as_feature_vector, read_fvec,
                                  read_fvec_into, write_fvec)


def test_dataset_contract():
    d = Dataset([[1, 2], [3, 4]])
    assert d.matrix.dtype == np.float32 and d.matrix.flags.c_contiguous
    assert (d.count, d.num_features, len(d)) == (2, 2, 2)
    with pytest.raises(ValueError):
        Dataset([[np.nan, 1.0]])
    with pytest.raises(ValueError):
        Dataset([1.0, 2.0])
    with pytest.raises(ValueError):
        as_feature_vector([1.0, np.inf])
    with pytest.raises(ValueError):
        as_feature_vector([1.0, 2.0], 3)


def test_fvec_round_trip_and_windows(tmp_path):
    m = np.random.default_rng(0).random((37, 5), dtype=np.float32)
    p = tmp_path / "x.fvec"
    write_fvec(p, Dataset(m))
    raw = p.read_bytes()
    assert raw[:4] == b"FVEC" and len(raw) == 12 + m.size * 4
    assert np.array_equal(read_fvec(p).matrix, m)
    buf = np.zeros((10, 5), np.float32)
    assert read_fvec_into(p, buf, 30) == 7
    assert np.array_equal(buf[:7], m[30:])
    assert read_fvec_into(p, buf, 37) == 0


def test_fvec_errors(tmp_path):
    p = tmp_path / "bad.fvec"
    p.write_bytes(b"FVE")
    with pytest.raises(DataFormatError):
        read_fvec(p)
    p.write_bytes(b"XVEC" + b"\0" * 8)
    with pytest.raises(DataFormatError):
        read_fvec(p)
    m = np.ones((2, 2), np.float32)
    write_fvec(p, m)
    p.write_bytes(p.read_bytes()[:-1])
    with pytest.raises(DataFormatError):
        read_fvec(p)
    m[0, 0] = np.nan
    write_fvec(p, m)
    with pytest.raises(DataFormatError):
        read_fvec(p)
