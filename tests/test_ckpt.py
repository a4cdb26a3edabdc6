"""CPU: the DSIMCKPT container (checkpoint_io.hpp:20-111) -- byte layout,
exact round trip of u64 bit patterns, and the reference's error texts."""
import struct

import numpy as np
import pytest

from paper_2412_12089_b200 import ckpt


def test_byte_layout(tmp_path):
    p = str(tmp_path / "a.ckpt")
    ckpt.save_checkpoint({"zeta": np.array([1.5]), "alpha": np.array([2.0, -3.0])}, p)
    raw = open(p, "rb").read()
    want = (b"DSIMCKPT" + struct.pack("<II", 1, 2) +
            struct.pack("<I", 5) + b"alpha" + struct.pack("<Q", 2) + struct.pack("<2d", 2.0, -3.0) +
            struct.pack("<I", 4) + b"zeta" + struct.pack("<Q", 1) + struct.pack("<d", 1.5))
    assert raw == want  # entries in std::map (name) order, little-endian


def test_round_trip_exact(tmp_path):
    p = str(tmp_path / "b.ckpt")
    words = [0, 1, 0x9E3779B97F4A7C15, 0xFFFFFFFFFFFFFFFF, 0x7FF8000000000001]  # incl. NaN payloads
    arr = {"rng": np.array([ckpt.pack_u64(w) for w in words]), "empty": np.zeros(0),
           "x": np.random.default_rng(0).standard_normal(1000)}
    ckpt.save_checkpoint(arr, p)
    c = ckpt.load_checkpoint(p)
    assert [ckpt.unpack_u64(v) for v in c["rng"]] == words
    assert c["empty"].size == 0 and np.array_equal(c["x"], arr["x"])


def test_errors(tmp_path):
    p = str(tmp_path / "c.ckpt")
    with pytest.raises(ckpt.CheckpointError, match="cannot open checkpoint"):
        ckpt.load_checkpoint(str(tmp_path / "missing"))
    open(p, "wb").write(b"NOTACKPT" + b"\0" * 8)
    with pytest.raises(ckpt.CheckpointError, match="not a checkpoint file"):
        ckpt.load_checkpoint(p)
    open(p, "wb").write(b"DSIMCKPT" + struct.pack("<II", 2, 0))
    with pytest.raises(ckpt.CheckpointError, match="unsupported checkpoint version 2"):
        ckpt.load_checkpoint(p)
    ckpt.save_checkpoint({"a": np.arange(4.0)}, p)
    open(p, "ab").truncate(len(open(p, "rb").read()) - 8)
    with pytest.raises(ckpt.CheckpointError, match="truncated checkpoint"):
        ckpt.load_checkpoint(p)
    c = {"a": np.arange(3.0)}
    with pytest.raises(ckpt.CheckpointError, match="missing entry 'b'"):
        ckpt.expect(c, "b", 3)
    with pytest.raises(ckpt.CheckpointError, match="entry 'a' has 3 values, model needs 4"):
        ckpt.expect(c, "a", 4)
