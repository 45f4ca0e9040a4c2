""".rti image sink (ingest.hpp:105-126, ingest.cpp:240-320): files
written by the library's sink are read by the reference's RtiReader and files written by
the reference's RtiWriter match ours byte for byte. Host code only: runs on the CPU."""
import os

import numpy as np
import pytest

HEADER = [1, 12, 8, 5, 3, 4, 2, 1, 24]  # version, N, channels, spokes, turns, frames, slices, mode, samples


def _images(n, N, seed=5):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, N, N)).astype(np.float32)


def test_sink_files_are_read_by_the_reference(ref, tmp_path):
    import paper_1701_08361_b200 as pb
    px = _images(5, 12)
    recs = [(0, 0, "magnitude"), (0, 1, "magnitude"), (1, 0, "magnitude"), (1, 1, "phase_difference"),
            (3, 0, "magnitude")]
    path = tmp_path / "ours.rti"
    with pb.RtiSink(path, HEADER) as sink:
        for (f, sl, k), p in zip(recs, px):
            sink.write(f, sl, k, p)
        assert sink.count == 5
    h, got, gpx = ref.rti_read(path)
    assert h == HEADER
    assert got == [(f, sl, 1 if k == "phase_difference" else 0) for f, sl, k in recs]
    assert np.array_equal(gpx, px)
    # the reference's writer produces the identical bytes (header text, payload, index)
    theirs = tmp_path / "theirs.rti"
    ref.rti_write(theirs, HEADER, [(f, sl, 1 if k == "phase_difference" else 0) for f, sl, k in recs], px)
    assert path.read_bytes() == theirs.read_bytes()
    assert (tmp_path / "ours.rti.idx").read_text() == (tmp_path / "theirs.rti.idx").read_text()


def test_sink_enforces_the_delivery_contract(tmp_path):
    import paper_1701_08361_b200 as pb
    px = _images(1, 12)[0]
    with pb.RtiSink(tmp_path / "a.rti", HEADER) as sink:
        sink.write(2, 0, "magnitude", px)
        with pytest.raises(pb.UsageError):
            sink.write(2, 0, "magnitude", px)  # frame indices increase strictly per slice
        with pytest.raises(pb.UsageError):
            sink.write(3, 2, "magnitude", px)  # slice id out of range
        sink.write(1, 1, "magnitude", px)  # another slice has its own order
    with pb.RtiSink(tmp_path / "b.rti", HEADER, strict_order=False) as sink:
        sink.write(2, 0, "magnitude", px)
        sink.write(1, 0, "magnitude", px)
    bad = list(HEADER)
    bad[5] = 0
    with pytest.raises(pb.DataError):
        pb.RtiSink(tmp_path / "c.rti", bad)
    flow_odd = list(HEADER)
    flow_odd[7], flow_odd[5] = 2, 3
    with pytest.raises(pb.DataError):
        pb.RtiSink(tmp_path / "d.rti", flow_odd)
    with pytest.raises(pb.DataError):
        pb.RtiSink(os.path.join(str(tmp_path), "missing_dir", "e.rti"), HEADER)
