"""TFFT1 signal files (reference tests/test_cli.py:23-57 restated): round trip
in both precisions, malformed headers / payloads, unsupported sizes. CPU only."""

import numpy as np
import pytest

from conftest import gaussian


def _io():
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import signal_io
    return tf, signal_io


@pytest.mark.parametrize("precision", ["single", "double"])
def test_signal_file_roundtrip(tmp_path, precision):
    tf, sio = _io()
    batch = tf.SignalBatch(gaussian(16, 3, precision, seed=1))
    path = tmp_path / "sig.tfft"
    tf.write_signal_file(path, batch)
    back = tf.read_signal_file(path)
    assert back.precision == precision
    assert np.array_equal(back.data, batch.data)
    raw = path.read_bytes()
    assert raw[:5] == b"TFFT1" and raw[5] == 1 and raw[6] == (1 if precision == "single" else 2)
    assert len(raw) == sio.HEADER.size + batch.data.nbytes


def test_signal_file_malformed(tmp_path):
    tf, sio = _io()
    path = tmp_path / "bad.tfft"
    cases = [
        b"XXXXX" + b"\0" * 18,                                      # bad magic
        b"TF",                                                      # short header
        sio.HEADER.pack(b"TFFT1", 1, 1, 8, 1) + b"\0" * 10,        # truncated payload
        sio.HEADER.pack(b"TFFT1", 1, 1, 8, 1) + b"\0" * 65,        # trailing bytes
        sio.HEADER.pack(b"TFFT1", 1, 9, 8, 1) + b"\0" * 64,        # unknown dtype code
        sio.HEADER.pack(b"TFFT1", 7, 1, 8, 1) + b"\0" * 64,        # unknown version
    ]
    for raw in cases:
        path.write_bytes(raw)
        with pytest.raises(tf.SignalFileError):
            tf.read_signal_file(path)


def test_signal_file_unsupported_size(tmp_path):
    tf, sio = _io()
    path = tmp_path / "n12.tfft"
    path.write_bytes(sio.HEADER.pack(b"TFFT1", 1, 1, 12, 1) + b"\0" * (12 * 8))
    with pytest.raises(tf.UnsupportedSizeError):
        tf.read_signal_file(path)
