"""Checkpoint container (reference pkg/tests/test_output.py:86-197) and its
compatibility with files written by the reference's own writer."""
import json
import os

import numpy as np
import pytest

from paper_2207_07098_b200.checkpoint import read_checkpoint, write_checkpoint
from paper_2207_07098_b200.errors import CheckpointError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ref_state.ckpt")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def test_reads_reference_file_and_rewrites_it_byte_for_byte(tmp_path):
    arrays, meta = read_checkpoint(GOLDEN)
    assert meta["case"] == "golden" and meta["projections"]["p"] == {"count": 2, "solves": 7}
    assert arrays["vel_0"].shape == (3, 2, 3, 3, 3) and arrays["scalar"].shape == ()
    out = tmp_path / "again.ckpt"
    write_checkpoint(str(out), arrays, meta)
    assert out.read_bytes() == open(GOLDEN, "rb").read()


def test_roundtrip_is_bitwise(tmp_path, rng):
    arrays = {"vel": rng.standard_normal((3, 2, 3, 3, 3)), "prs": rng.standard_normal((2, 3, 3, 3)) * 1e-300,
              "scalar": np.array(np.pi)}
    meta = {"time": 0.125, "nsteps": 10, "name": "case", "nested": {"a": [1, 2]}}
    path = tmp_path / "state.ckpt"
    write_checkpoint(str(path), arrays, meta)
    back, meta2 = read_checkpoint(str(path))
    assert set(back) == set(arrays) and meta2 == meta
    for name in arrays:
        assert back[name].dtype == np.float64 and np.array_equal(back[name], arrays[name])


def test_torch_tensors_accepted(tmp_path, rng):
    import torch

    a = rng.standard_normal((2, 5))
    write_checkpoint(str(tmp_path / "t.ckpt"), {"a": torch.from_numpy(a)}, {})
    back, _ = read_checkpoint(str(tmp_path / "t.ckpt"))
    assert np.array_equal(back["a"], a)


def test_header_layout(tmp_path):
    path = tmp_path / "layout.ckpt"
    write_checkpoint(str(path), {"x": np.zeros(2)}, {"m": 3})
    blob = path.read_bytes()
    assert blob[:8] == b"SEMFCKPT"
    assert int(np.frombuffer(blob[8:12], dtype="<u4")[0]) == 1
    hlen = int(np.frombuffer(blob[12:20], dtype="<u8")[0])
    header = json.loads(blob[20:20 + hlen].decode("utf-8"))
    assert header == {"arrays": [{"name": "x", "shape": [2]}], "meta": {"m": 3}}
    assert len(blob) == 20 + hlen + 16


def test_rejects_non_float64(tmp_path):
    with pytest.raises(CheckpointError, match="float64"):
        write_checkpoint(str(tmp_path / "bad.ckpt"), {"x": np.zeros(3, dtype=np.float32)}, {})


def test_bad_magic_and_version(tmp_path):
    p = tmp_path / "bad.ckpt"
    p.write_bytes(b"NOTMAGIC" + b"\x00" * 32)
    with pytest.raises(CheckpointError, match="magic") as exc:
        read_checkpoint(str(p))
    assert exc.value.offset == 0 and exc.value.section == "magic"
    good = tmp_path / "good.ckpt"
    write_checkpoint(str(good), {"x": np.zeros(1)}, {})
    blob = bytearray(good.read_bytes())
    blob[8:12] = np.uint32(9).tobytes()
    p.write_bytes(bytes(blob))
    with pytest.raises(CheckpointError, match="version 9") as exc:
        read_checkpoint(str(p))
    assert exc.value.section == "version"


def test_truncation_header_and_trailer(tmp_path):
    good = tmp_path / "good.ckpt"
    write_checkpoint(str(good), {"field": np.arange(16.0)}, {"a": 1})
    blob = good.read_bytes()
    p = tmp_path / "x.ckpt"
    p.write_bytes(blob[:-8])
    with pytest.raises(CheckpointError, match="truncated") as exc:
        read_checkpoint(str(p))
    assert exc.value.section == "field"
    p.write_bytes(blob[:10])
    with pytest.raises(CheckpointError, match="truncated") as exc:
        read_checkpoint(str(p))
    assert exc.value.section == "version"
    bad = bytearray(blob)
    bad[21] = 0xFF
    p.write_bytes(bytes(bad))
    with pytest.raises(CheckpointError, match="header") as exc:
        read_checkpoint(str(p))
    assert exc.value.section == "header"
    p.write_bytes(blob + b"\x00\x01\x02")
    with pytest.raises(CheckpointError, match="trailing") as exc:
        read_checkpoint(str(p))
    assert exc.value.section == "trailer"


def test_empty(tmp_path):
    p = tmp_path / "empty.ckpt"
    write_checkpoint(str(p), {}, {})
    assert read_checkpoint(str(p)) == ({}, {})


def test_diagnostics_csv_row_matches_reference_runner():
    from paper_2207_07098_b200.checkpoint import DIAG_HEADER, diag_row
    from paper_2207_07098_b200.timestep import StepDiagnostics

    with open(os.path.join(os.path.dirname(__file__), "golden", "diag_row.txt")) as fh:
        header, row = fh.read().splitlines()
    d = StepDiagnostics(step=7, time=0.07000000000000001, cfl=0.2012345678901234, div_norm=1.25e-5,
                        p_iterations=33, p_residual=9.87654321e-6, v_iterations=(4, 4, 3),
                        v_residual=(1e-9, 2.5e-9, 3.333e-9), wall_time=0.0123)
    assert DIAG_HEADER == header and diag_row(d) == row
