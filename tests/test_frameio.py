"""Frame ingest host API (§8f #4; reference frameio.py): CPU-only.

Every reader branch against the outcomes recorded by running the reference's
own ``load_frames`` on the same bytes (tests/golden/golden_frameio.json), plus
the write / round-trip behaviours of the reference's test_frameio.py.
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2604_24391_b200 import frameio
from paper_2604_24391_b200.types import FrameParseError

GOLD = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLD))
from cases import fhash, frameio_cases  # noqa: E402


def test_readers_match_reference_outcomes(tmp_path):
    gold = {g["name"]: g for g in json.loads((GOLD / "golden_frameio.json").read_text())}
    for name, suffix, data in frameio_cases():
        p = tmp_path / f"{name}{suffix}"
        p.write_bytes(data)
        g = gold[name]
        if "error" in g:
            with pytest.raises(FrameParseError) as err:
                frameio.load_frames(p)
            assert err.value.offset == g["offset"], name
            assert str(err.value).replace(str(p), "<path>") == g["message"], name
        else:
            frs = frameio.load_frames(p)
            assert [fhash(f) for f in frs] == g["frames"], name
            assert list(frs[0].shape) == g["shape"]


def test_pgm_write_read_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    img = rng.random((7, 9))
    frameio.write_pgm(tmp_path / "a.pgm", img)
    back = frameio.read_netpbm(tmp_path / "a.pgm")
    assert np.max(np.abs(back - img)) <= 0.5 / 255 + 1e-12
    u8 = rng.integers(0, 256, (3, 4), dtype=np.uint8)
    frameio.write_pgm(tmp_path / "b.pgm", u8)
    assert np.array_equal(np.round(frameio.read_netpbm(tmp_path / "b.pgm") * 255).astype(np.uint8), u8)
    with pytest.raises(ValueError):
        frameio.write_pgm(tmp_path / "c.pgm", np.zeros((2, 2, 2)))


def test_rawf32_round_trip_bit_identical(tmp_path):
    rng = np.random.default_rng(2)
    frames = [rng.random((5, 6)).astype(np.float32).astype(np.float64) for _ in range(3)]
    frameio.save_rawf32(tmp_path / "s.raw", frames)
    back = frameio.load_rawf32(tmp_path / "s.raw")
    assert all(np.array_equal(a, b) for a, b in zip(frames, back))
    with pytest.raises(ValueError):
        frameio.save_rawf32(tmp_path / "t.raw", [np.full((2, 2), np.nan)])


def test_load_frames_auto_and_directories(tmp_path):
    d = tmp_path / "seq"
    d.mkdir()
    for i in range(3):
        frameio.write_pgm(d / f"f{i:02d}.pgm", np.full((4, 4), i / 4))
    (d / "notes.txt").write_text("ignored")
    frs = frameio.load_frames(d)
    assert [f[0, 0] for f in frs] == [np.round(i / 4 * 255) / 255 for i in range(3)]
    (tmp_path / "empty").mkdir()
    with pytest.raises(FrameParseError):
        frameio.load_frames(tmp_path / "empty")
    with pytest.raises(ValueError):
        frameio.load_frames(d, fmt="tiff")


def test_energy_heatmap(tmp_path):
    class _E:
        energies = np.array([[0.0, 1.0], [2.0, 4.0]])
    frameio.export_energy_heatmap(_E(), tmp_path / "h.pgm")
    px, ch = frameio.read_netpbm_payload(tmp_path / "h.pgm")
    assert ch == 1 and px[1, 1] == 255 and px[0, 0] == 0
    _E.energies = np.zeros((2, 2))
    frameio.export_energy_heatmap(_E(), tmp_path / "z.pgm")
    assert (frameio.read_netpbm_payload(tmp_path / "z.pgm")[0] == 0).all()
