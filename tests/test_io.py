"""Volume I/O (reference E/io.py) on the host: golden files written by the
reference's own writer (tests/golden/make_io.py) are read back value for
value and rewritten byte for byte; the error cases of the reference's
tests/test_volume_io.py:96-231 raise the same exception types."""

import os

import numpy as np
import pytest

from paper_2504_19930_b200 import (CorruptHeader, InternalError, Sequence4, TruncatedData,
                                   UnsupportedFormat, Volume3)
from paper_2504_19930_b200.io import (read_volume, read_volume_device, write_u8_nifti,
                                      write_volume)

from .conftest import golden

CASES = {"f32_3d": (".nii", "float32"), "f32_4d": (".nii", "float32"),
         "mask_u8": (".nii", "uint8"), "raw_4d": (".raw", None)}


def _frames(v):
    return v.frames if isinstance(v, Sequence4) else [v]


def _materialise(g, name, tmp_path):
    ext = CASES[name][0]
    path = str(tmp_path / (name + ext))
    g[f"{name}.file"].tofile(path)
    if ext == ".raw":
        g[f"{name}.json"].tofile(path[:-4] + ".json")
    return path


@pytest.mark.parametrize("name", sorted(CASES))
def test_reads_reference_written_files(name, tmp_path):
    g = golden("io.npz")
    back = read_volume(_materialise(g, name, tmp_path))
    fr = _frames(back)
    assert np.array_equal(np.stack([f.data for f in fr]), g[f"{name}.data"])
    assert np.array_equal(np.array([*fr[0].spacing, *fr[0].origin]), g[f"{name}.geom"])
    rate, ed = g[f"{name}.seq"]
    if rate < 0:
        assert isinstance(back, Volume3)
    else:
        assert back.frame_rate == rate and back.ed_index == ed


@pytest.mark.parametrize("name", sorted(CASES))
def test_writer_matches_reference_bytes(name, tmp_path):
    g = golden("io.npz")
    ext, dtype = CASES[name]
    geom = g[f"{name}.geom"]
    frames = [Volume3(d, tuple(geom[:3]), tuple(geom[3:])) for d in g[f"{name}.src"]]
    rate, ed = g[f"{name}.seq"]
    v = frames[0] if rate < 0 else Sequence4(frames, frame_rate=float(rate), ed_index=int(ed))
    path = str(tmp_path / ("ours" + ext))
    if dtype:
        write_volume(v, path, dtype=dtype)
    else:
        write_volume(v, path)
    assert np.array_equal(np.fromfile(path, np.uint8), g[f"{name}.file"])
    if ext == ".raw":
        assert np.array_equal(np.fromfile(path[:-4] + ".json", np.uint8), g[f"{name}.json"])


def test_u8_grey_nifti_roundtrip_is_an_8bit_codec_volume(tmp_path):
    rng = np.random.default_rng(5)
    raws = [rng.integers(0, 256, (7, 5, 9), dtype=np.uint8) for _ in range(3)]
    seq = Sequence4([Volume3.from_u8(r, (0.87, 1.08, 0.73), (1.0, 2.0, 3.0)) for r in raws],
                    frame_rate=30.0)
    path = str(tmp_path / "echo.nii")
    write_u8_nifti(seq, path)
    assert os.path.getsize(path) == 352 + 3 * 7 * 5 * 9
    back = read_volume(path)
    assert len(back) == 3 and back.frame_rate == pytest.approx(30.0, rel=1e-6)
    for r, f in zip(raws, back.frames):
        assert f.codec is not None and f.codec.identity
        assert np.array_equal(f.codec.raw, r) and np.array_equal(f.data, r.astype(np.float64))
    with pytest.raises(ValueError):
        write_u8_nifti(Volume3(np.full((2, 2, 2), 0.5)), str(tmp_path / "x.nii"))


def test_error_types_match_the_reference(tmp_path):
    rng = np.random.default_rng(0)
    v = Volume3(rng.random((4, 4, 4), dtype=np.float32).astype(np.float64))
    with pytest.raises(ValueError):  # test_volume_io.py:136-140
        write_volume(v, str(tmp_path / "x.nii"), dtype="uint8")
    path = str(tmp_path / "v.nii")
    write_volume(v, path)
    blob = bytearray(open(path, "rb").read())
    bad = bytearray(blob)
    bad[344:348] = b"ni1\x00"
    (tmp_path / "m.nii").write_bytes(bytes(bad))
    with pytest.raises(UnsupportedFormat):  # :142-149
        read_volume(str(tmp_path / "m.nii"))
    (tmp_path / "s.nii").write_bytes(bytes(blob[:100]))
    with pytest.raises(CorruptHeader):  # :151-155
        read_volume(str(tmp_path / "s.nii"))
    (tmp_path / "t.nii").write_bytes(bytes(blob[:-5]))
    with pytest.raises(TruncatedData):  # :157-163
        read_volume(str(tmp_path / "t.nii"))
    bad = bytearray(blob)
    bad[70:72] = np.int16(64).tobytes()
    (tmp_path / "d.nii").write_bytes(bytes(bad))
    with pytest.raises(UnsupportedFormat):  # :165-172
        read_volume(str(tmp_path / "d.nii"))
    bad = bytearray(blob)
    bad[40:42] = np.int16(5).tobytes()
    (tmp_path / "n.nii").write_bytes(bytes(bad))
    with pytest.raises(CorruptHeader):
        read_volume(str(tmp_path / "n.nii"))
    with pytest.raises(UnsupportedFormat):  # :174-176
        read_volume(str(tmp_path / "vol.dcm"))
    (tmp_path / "x.json").write_text('{"spacing": [1, 1, 1]}')
    with pytest.raises(CorruptHeader):  # :219-223
        read_volume(str(tmp_path / "x.raw"))
    (tmp_path / "r.json").write_text('{"dims": [2, 2, 2], "spacing": [1, 1, 1]}')
    (tmp_path / "r.raw").write_bytes(b"\x00" * 31)
    with pytest.raises(TruncatedData):  # :225-231
        read_volume(str(tmp_path / "r.raw"))


def test_device_ingest_fails_loudly_without_cuda(tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    path = str(tmp_path / "e.nii")
    write_u8_nifti(Volume3.from_u8(np.zeros((4, 4, 4), np.uint8)), path)
    with pytest.raises(InternalError):
        read_volume_device(path)
