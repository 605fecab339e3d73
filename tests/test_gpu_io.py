"""Device ingest of 8-bit NIfTI volumes (er_ingest_u8; reference E/io.py:
124-187 + the z-score of E/volume.py:119-130): read_volume_device returns
the same volumes as the host reader (itself pinned to the reference's files
by tests/test_io.py), with each frame's histogram counted in the same pass
and its device copy already resident."""

import ctypes

import numpy as np
import pytest

from paper_2504_19930_b200 import (ConstantVolume, SmcConfig, Sequence4, Volume3, normalize_zscore,
                                   register_smc)
from paper_2504_19930_b200 import _lib
from paper_2504_19930_b200.device import _U8_STORE, ptr, stream_ptr
from paper_2504_19930_b200.io import read_volume, read_volume_device, write_u8_nifti, write_volume

pytestmark = pytest.mark.gpu

DIMS = [((1, 1, 1), 1), ((3, 5, 7), 2), ((64, 64, 64), 1), ((65, 63, 130), 3),
        ((128, 7, 68), 2), ((176, 176, 208), 2), ((200, 3, 1), 4)]


def _frames(v):
    return v.frames if isinstance(v, Sequence4) else [v]


def _grey_file(tmp_path, dims, nf, seed):
    rng = np.random.default_rng(seed)
    raws = [rng.integers(0, 256, dims, dtype=np.uint8) for _ in range(nf)]
    # a skewed, clustered distribution as well (shared-memory bin contention)
    raws[-1][..., ::2] = 7
    vols = [Volume3.from_u8(r, (0.87, 1.08, 0.73), (1.0, -2.0, 0.5)) for r in raws]
    v = Sequence4(vols, frame_rate=25.0) if nf > 1 else vols[0]
    path = str(tmp_path / f"g{seed}.nii")
    write_u8_nifti(v, path)
    return path, raws


@pytest.mark.parametrize("dims,nf", DIMS)
def test_device_ingest_equals_host_reader(tmp_path, dims, nf):
    import torch

    path, raws = _grey_file(tmp_path, dims, nf, seed=sum(dims) + nf)
    host, dev = read_volume(path), read_volume_device(path)
    assert type(host) is type(dev)
    if nf > 1:
        assert dev.frame_rate == host.frame_rate and dev.ed_index == host.ed_index
    for r, h, d in zip(raws, _frames(host), _frames(dev)):
        assert d.dims == h.dims == dims
        assert d.spacing == h.spacing and d.origin == h.origin
        assert np.array_equal(d.codec.raw, r) and np.array_equal(h.codec.raw, r)
        sh = _U8_STORE[(id(d.codec.raw), torch.cuda.current_device())]
        assert sh.raw_ref() is d.codec.raw
        assert np.array_equal(sh.hist, np.bincount(r.ravel(), minlength=256))
        assert np.array_equal(sh.storage.cpu().numpy(), r.ravel())  # the resident copy
        if r.min() == r.max():  # constant frame: the z-score raises (volume.py:126-128)
            with pytest.raises(ConstantVolume):
                normalize_zscore(d)
            continue
        zh, zd = normalize_zscore(h), normalize_zscore(d)
        assert zd.codec.mean == zh.codec.mean and zd.codec.std == zh.codec.std
        assert np.array_equal(zd.data, zh.data)


def test_binary_mask_file_and_float32_file(tmp_path):
    rng = np.random.default_rng(3)
    m = Volume3((rng.random((33, 17, 9)) > 0.4).astype(np.float64))
    write_volume(m, str(tmp_path / "m.nii"), dtype="uint8")
    d = read_volume_device(str(tmp_path / "m.nii"))
    assert np.array_equal(d.data, m.data)
    f = Volume3(rng.random((5, 6, 7), dtype=np.float32).astype(np.float64))
    write_volume(f, str(tmp_path / "f.nii"))
    assert np.array_equal(read_volume_device(str(tmp_path / "f.nii")).data, f.data)


def test_word_and_byte_paths_on_unaligned_buffers():
    """The kernel takes 32-bit words only when rows are 4-byte aligned; an
    offset payload or output pointer must take the byte path, same result."""
    import torch

    nx, ny, nz, nf = 68, 5, 72, 2
    rng = np.random.default_rng(11)
    disk = rng.integers(0, 256, nf * nx * ny * nz, dtype=np.uint8)
    want = disk.reshape(nf, nz, ny, nx).transpose(0, 3, 2, 1).reshape(nf, -1)
    for off_in, off_out in ((0, 0), (1, 0), (0, 3), (2, 1)):
        d_in = torch.zeros(disk.size + 8, dtype=torch.uint8, device="cuda")
        d_in[off_in:off_in + disk.size] = torch.from_numpy(disk).cuda()
        out = torch.zeros(nf * nx * ny * nz + 8, dtype=torch.uint8, device="cuda")
        hist = torch.empty((nf, 256), dtype=torch.int64, device="cuda")
        p_in = ctypes.c_void_p(d_in.data_ptr() + off_in)
        p_out = ctypes.c_void_p(out.data_ptr() + off_out)
        _lib.call("er_ingest_u8", p_in, nx, ny, nz, nf, p_out, ptr(hist), stream_ptr())
        got = out[off_out:off_out + want.size].cpu().numpy().reshape(nf, -1)
        assert np.array_equal(got, want), (off_in, off_out)
        for f in range(nf):
            assert np.array_equal(hist[f].cpu().numpy(), np.bincount(want[f], minlength=256))
        # no histogram requested: the reorder alone
        out.zero_()
        _lib.call("er_ingest_u8", p_in, nx, ny, nz, nf, p_out, None, stream_ptr())
        assert np.array_equal(out[off_out:off_out + want.size].cpu().numpy().reshape(nf, -1),
                              want)


def test_ingest_abi_rejects_bad_arguments():
    import torch

    lib = _lib.load()
    a = torch.zeros(64, dtype=torch.uint8, device="cuda")
    b = torch.zeros(64, dtype=torch.uint8, device="cuda")
    s = stream_ptr()
    assert lib.er_ingest_u8(None, 4, 4, 4, 1, ptr(b), None, s) != 0
    assert lib.er_ingest_u8(ptr(a), 0, 4, 4, 1, ptr(b), None, s) != 0
    assert lib.er_ingest_u8(ptr(a), 4, 4, 4, 1, ptr(a), None, s) != 0  # in place
    assert lib.er_ingest_u8(ptr(a), 4, 4, 4, 70000, ptr(b), None, s) != 0
    assert lib.er_ingest_u8(ptr(a), 4, 4, 4, 0, ptr(b), None, s) == 0


def test_registration_from_device_ingested_files_is_identical(tmp_path):
    """read_volume_device -> normalize_zscore -> register_smc gives the same
    estimate as the in-memory volumes the files were written from."""
    from paper_2504_19930_b200.phantom import echo_case

    case = echo_case(dims=(40, 40, 48), frames=1)
    write_u8_nifti(case.target.frames[0], str(tmp_path / "t.nii"))
    write_u8_nifti(case.source.frames[0], str(tmp_path / "s.nii"))
    cfg = SmcConfig(mode="image", n_particles=300, n_iterations=8, seed=1)
    want, _ = register_smc(normalize_zscore(case.target.frames[0]),
                           normalize_zscore(case.source.frames[0]), cfg)
    t = read_volume_device(str(tmp_path / "t.nii"))
    s = read_volume_device(str(tmp_path / "s.nii"))
    got, _ = register_smc(normalize_zscore(t), normalize_zscore(s), cfg)
    assert got == want
