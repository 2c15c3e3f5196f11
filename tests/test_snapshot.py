"""SPHK snapshots: the reference-written golden file (tests/golden/
make_snapshot_golden.py) parsed by the repo's reader, re-encoded byte for
byte, and the reference's error types on damaged files (snapshot.py:34-67 of
the reference).  The device streaming path is in tests/test_gpu_parity.py."""
import os
import struct

import numpy as np
import pytest

from paper_1612_06090_b200 import snapshot as S
from paper_1612_06090_b200 import workload

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "snap_uniform3000_k32.sphk")


def test_reads_reference_snapshot():
    sec = S.load(GOLD)
    assert set(sec) == {"meta", "particles"}
    p = S.decode_particles(sec["particles"])
    pos = workload.uniform_box(3000, 17, 1.0)  # the reference UniformBox stream, seed 17
    assert np.array_equal(p["x"], pos[:, 0]) and np.array_equal(p["z"], pos[:, 2])
    assert np.array_equal(p["id"], np.arange(3000))
    g = np.load(os.path.join(HERE, "golden", "snap_uniform3000_k32.npz"))
    assert np.all(p["smoothing_length"] == p["smoothing_length"][0])  # the reference's initial h rule
    assert f"{S.checksum64(sec['particles']):016x}" == str(g["particles_checksum"])


def test_writer_reproduces_reference_bytes(tmp_path):
    sec = S.load(GOLD)
    p = S.decode_particles(sec["particles"])
    assert S.encode_particles(p) == sec["particles"]
    out = tmp_path / "copy.sphk"
    S.dump(out, {"meta": sec["meta"], "particles": S.encode_particles(p)})
    assert open(out, "rb").read() == open(GOLD, "rb").read()


def test_damaged_files_raise_reference_errors(tmp_path):
    raw = bytearray(open(GOLD, "rb").read())
    bad = tmp_path / "bad.sphk"
    bad.write_bytes(b"XXXX" + bytes(raw[4:]))
    with pytest.raises(S.BadMagicError):
        S.load(bad)
    bad.write_bytes(bytes(raw[:4]) + struct.pack("<I", 2) + bytes(raw[8:]))
    with pytest.raises(S.VersionError):
        S.load(bad)
    bad.write_bytes(bytes(raw[:-100]))
    with pytest.raises(S.TruncatedError):
        S.load(bad)
    flip = bytearray(raw)
    flip[len(flip) // 2] ^= 0x40
    bad.write_bytes(bytes(flip))
    with pytest.raises(S.ChecksumError) as ei:
        S.load(bad)
    assert ei.value.section == "particles"
    with pytest.raises(S.SnapshotIOError):
        S.load(tmp_path / "missing.sphk")
