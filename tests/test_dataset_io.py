"""Feature-map files (src/dataset.cpp:115-247): the product's
FMAP / CSV reader and writer (csrc/host/dataset.cpp, host-only C ABI) against
the reference's save / load -- byte-identical files, bit-identical maps, the
same error classes -- and the batched loader that feeds the GPU entries."""
import os

import numpy as np
import pytest


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("ext", [".fmap", ".csv"])
def test_roundtrip_and_reference_bytes(sc, orc, ref, tmp_path, ext):
    m = orc.generate(7, 9, 3, 0.6, 11) - np.float32(0.3)  # negatives, zeros, fractions
    m[0, 0, 0] = -0.0
    fm = sc.FeatureMap(3, 7, 9, m.reshape(-1))
    ours, theirs = tmp_path / ("ours" + ext), tmp_path / ("theirs" + ext)
    sc.save(fm, ours)
    ref.save_map(m, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    back = sc.load(theirs)
    assert (back.channels, back.height, back.width) == (3, 7, 9)
    assert np.array_equal(bits(back.values), bits(m.reshape(-1)))
    assert np.array_equal(bits(ref.load_map(ours)), bits(m))


def test_errors_match_reference(sc, ref, tmp_path):
    from oracle.oracle import OracleError
    bad = tmp_path / "bad.fmap"
    bad.write_bytes(b"NOPE" + bytes(16))
    with pytest.raises(sc.FormatError, match="bad magic"):
        sc.load(bad)
    with pytest.raises(OracleError):
        ref.load_map(bad)
    trunc = tmp_path / "t.fmap"
    sc.save(sc.FeatureMap(1, 2, 2, np.ones(4, np.float32)), trunc)
    trunc.write_bytes(trunc.read_bytes()[:-3])
    with pytest.raises(sc.FormatError, match="truncated payload"):
        sc.load(trunc)
    with pytest.raises(sc.IoError):
        sc.load(tmp_path / "missing.fmap")
    csv = tmp_path / "b.csv"
    csv.write_text("channels,height,width\n1,1,2\n1.5,abc\n")
    with pytest.raises(sc.FormatError, match="bad value"):
        sc.load(csv)


def test_load_batch(sc, orc, tmp_path):
    paths = []
    want = []
    for i in range(5):
        m = orc.generate(6, 8, 2, 0.7, 100 + i)
        p = tmp_path / f"m{i}.fmap"
        sc.save(sc.FeatureMap(2, 6, 8, m.reshape(-1)), p)
        paths.append(p)
        want.append(m)
    got = sc.load_batch(paths, threads=3)
    assert np.array_equal(bits(got), bits(np.stack(want)))
    odd = tmp_path / "odd.fmap"
    sc.save(sc.FeatureMap(1, 6, 8, np.zeros(48, np.float32)), odd)
    with pytest.raises(sc.ShapeError):
        sc.load_batch(paths + [odd])
