"""Flat binary series I/O (series.cpp:262-284; format series.hpp:93) -- CPU."""
import struct

import numpy as np
import pytest


def test_bin_round_trip_and_layout(tmp_path):
    import paper_2112_12994_b200 as tf
    v = np.array([1.5, -2.25, 3.0e300, 0.0])
    p = str(tmp_path / "s.bin")
    tf.save_series_bin(tf.TimeSeries(v), p)
    raw = open(p, "rb").read()
    assert len(raw) == 8 + 8 * v.size
    assert struct.unpack("<Q", raw[:8])[0] == v.size            # uint64 LE count
    assert struct.unpack("<4d", raw[8:]) == tuple(v)               # f64 LE payload
    back = tf.load_series_bin(p)
    assert np.array_equal(back.values(), v)


def test_bin_errors(tmp_path):
    import paper_2112_12994_b200 as tf
    with pytest.raises(tf.DataError, match="cannot open"):
        tf.load_series_bin(str(tmp_path / "missing.bin"))
    p = tmp_path / "short.bin"
    p.write_bytes(b"\x01\x02")
    with pytest.raises(tf.DataError, match="truncated header"):
        tf.load_series_bin(str(p))
    p.write_bytes(struct.pack("<Q", 3) + struct.pack("<2d", 1.0, 2.0))
    with pytest.raises(tf.DataError, match="truncated payload"):
        tf.load_series_bin(str(p))
    p.write_bytes(struct.pack("<Q", 2) + struct.pack("<2d", 1.0, float("nan")))
    with pytest.raises(tf.DataError, match="not finite"):          # TimeSeries validation
        tf.load_series_bin(str(p))


@pytest.mark.gpu
def test_bin_pinned_load_fits_identically(tmp_path):
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import build, gen
    build.build()
    y = gen.simulate_roots(gen.ar_roots(6, 1.2, 3.0, 3), 40000, 3)
    p = str(tmp_path / "y.bin")
    tf.save_series_bin(tf.TimeSeries(y), p)
    a = tf.lsar_fit(tf.load_series_bin(p, pinned=True), 12, 500, 7)
    b = tf.lsar_fit(tf.TimeSeries(y), 12, 500, 7)
    assert a.pacf.taus == b.pacf.taus and a.p_star == b.p_star
