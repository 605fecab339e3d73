"""Parity of the sm_100a measurement kernel (the hot path) against the
reference's own outputs (golden vectors) and the bit-exact C oracle.

Tolerances (written here, per BASELINE north star): in-bounds voxel counts
and degenerate flags bit-exact; per-particle squared NCC within 1e-4
relative for the fp32-lerp mode, 1e-6 for fp64 lerps on the fixed-point fast
path and 1e-10 relative for the reference-order fp64 mode (only the
summation order differs from the reference there), each with an absolute
floor of 1e-12 for numerically-zero likelihoods (see ATOL).
"""

import math

import numpy as np
import pytest

from oracle import kernels as ok

from .conftest import golden, golden_kernel_cases

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

# f64 on 8-bit sources runs the fast path (Q24.40 fixed-point coordinates):
# per-voxel coordinate error <= 2^-41 (k+1) voxels, visible only through the
# sts^2 cancellation of near-zero likelihoods -> 1e-6 relative.
RTOL = {"f32": 1e-4, "f64": 1e-6, "exact": 1e-10}
CASES = golden_kernel_cases()


def _vol(data, spacing, origin):
    from paper_2504_19930_b200 import Volume3

    return Volume3(np.asarray(data), tuple(spacing), tuple(origin))


def _measure(tgt, src, a, b, overlap, precision):
    from paper_2504_19930_b200 import ops
    from paper_2504_19930_b200.device import device_volume, require_cuda

    dev = require_cuda()
    A = torch.as_tensor(np.ascontiguousarray(a).reshape(-1, 9), device=dev)
    B = torch.as_tensor(np.ascontiguousarray(b).reshape(-1, 3), device=dev)
    z, d, n = ops.measure(device_volume(tgt, dev), device_volume(src, dev), A, B, overlap,
                          precision)
    return z.cpu().numpy(), d.cpu().numpy().astype(bool), n.cpu().numpy()


# Absolute floor for likelihoods that are numerically zero: z ~ 1e-12 (no
# overlap structure at all) is ill-conditioned through the sts^2
# cancellation, and an error of 1e-12 moves exp(beta z) by 5e-11 relative.
ATOL = 1e-12


def _close(got, want, rtol, atol=ATOL):
    got, want = np.asarray(got), np.asarray(want)
    scale = np.maximum(np.abs(want), 1e-300)
    bad = np.abs(got - want) > rtol * scale + atol
    # exact zeros (degenerate) must stay exact zeros
    bad |= (want == 0.0) != (got == 0.0)
    return not bad.any(), float(np.max(np.abs(got - want) / scale))


@pytest.mark.parametrize("precision", ["f32", "f64", "exact"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_measure_matches_reference_goldens(name, precision):
    c = CASES[name]
    tgt = _vol(c["tgt"], c["tgt_spacing"], c["tgt_origin"])
    src = _vol(c["src"], c["src_spacing"], c["src_origin"])
    for overlap, key in ((False, "full"), (True, "overlap")):
        z, d, n = _measure(tgt, src, c["a"], c["b"], overlap, precision)
        ok_, err = _close(z, c[f"ncc_{key}"], RTOL[precision])
        assert ok_, (name, key, precision, err)
        assert np.array_equal(d, c[f"degen_{key}"]), (name, key)
        assert np.array_equal(n, c["n_in"]), (name, key)


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_executor_seam_matches_reference(precision):
    from paper_2504_19930_b200 import Executor

    c = CASES["cube10"]
    tgt = _vol(c["tgt"], c["tgt_spacing"], c["tgt_origin"])
    src = _vol(c["src"], c["src_spacing"], c["src_origin"])
    z, d = Executor(precision=precision).measure_ncc(tgt, src, c["mats"], False)
    assert _close(z, c["ncc_full"], RTOL[precision])[0]
    assert np.array_equal(d, c["degen_full"])


def _c1():
    g = golden("smc.npz")
    dims = tuple(int(x) for x in g["c1_dims"])
    n = int(np.prod(dims))
    t = np.unpackbits(g["c1_target_bits"])[:n].reshape(dims).astype(np.float64)
    s = np.unpackbits(g["c1_source_bits"])[:n].reshape(dims).astype(np.float64)
    return g, t, s


@pytest.mark.parametrize("precision", ["f32", "f64", "exact"])
def test_c1_lockstep_iteration0(precision):
    """C1 (64^3 masks, 500 particles): the reference's iteration-0 batch."""
    g, t, s = _c1()
    z, d, n = _measure(_vol(t, (1, 1, 1), (0, 0, 0)), _vol(s, (1, 1, 1), (0, 0, 0)),
                       g["c1_a_it0"], g["c1_b_it0"], False, precision)
    ok_, err = _close(z, g["c1_z"][0], RTOL[precision])
    assert ok_, err
    assert np.array_equal(d, g["c1_degen"][0])
    # overlap counts against the bit-exact oracle
    _, _, n_or = ok.ncc_measure_batch(t, s, g["c1_a_it0"], g["c1_b_it0"], True,
                                      return_counts=True)
    assert np.array_equal(n, n_or)


def test_sharding_is_bitwise_invariant():
    """Any split of the particle set gives bit-identical results (the
    reference's worker-count invariance, tests/test_kernels.py:106-116)."""
    g, t, s = _c1()
    tv, sv = _vol(t, (1, 1, 1), (0, 0, 0)), _vol(s, (1, 1, 1), (0, 0, 0))
    a, b = g["c1_a_it0"], g["c1_b_it0"]
    full = _measure(tv, sv, a, b, False, "f64")[0]
    for parts in (2, 3, 7):
        cuts = np.linspace(0, a.shape[0], parts + 1).astype(int)
        got = np.concatenate([_measure(tv, sv, a[lo:hi], b[lo:hi], False, "f64")[0]
                              for lo, hi in zip(cuts[:-1], cuts[1:])])
        assert np.array_equal(got, full)


def test_identity_scores_one_and_out_of_frame_degenerate():
    from paper_2504_19930_b200 import Executor, RigidParams, Volume3, to_matrix

    rng = np.random.default_rng(3)
    v = Volume3(rng.random((7, 7, 7), dtype=np.float32).astype(np.float64))
    # fp64 modes: 1 to 1e-12; the default fp32 mode (quad layout, fp32 row
    # partials) to its 1e-4 bar -- at identity the samples are exact and only
    # the fp32 partial sums round
    for prec, tol in (("f64", 1e-12), ("exact", 1e-12), ("f32", 1e-6)):
        z, d = Executor(precision=prec).measure_ncc(v, v, np.eye(4)[np.newaxis])
        assert z[0] == pytest.approx(1.0, abs=tol) and not d[0], prec
    gone = to_matrix(RigidParams(tx=1e5))
    z, d = Executor().measure_ncc(v, v, gone[np.newaxis])
    assert z[0] == 0.0 and d[0]


def _echo_pair(dims=(176, 176, 208), seed=0):
    """uint8 echo-like pair on a C2-shaped grid (host construction, small cost)."""
    rng = np.random.default_rng(seed)
    nx, ny, nz = dims
    x = (np.arange(nx) - nx / 2)[:, None, None] / (0.35 * nx)
    y = (np.arange(ny) - ny / 2)[None, :, None] / (0.30 * ny)
    z = (np.arange(nz) - nz / 2)[None, None, :] / (0.40 * nz)
    r = x * x + y * y + z * z
    base = np.where(r <= 1.0, 200.0, 40.0) * np.where(r <= 0.45, 0.2, 1.0)
    speck = np.exp(0.3 * rng.standard_normal(dims))
    raw = np.clip(np.round(base * speck), 0, 255)
    raw2 = np.roll(raw, (2, -3, 1), axis=(0, 1, 2))
    return raw, raw2


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_c2_shaped_uint8_codec_vs_oracle(precision):
    """176x176x208 raw uint8 images, z-scored (codec path: 1-byte gathers with
    the affine folded in) against the C oracle on the normalised fp64 data."""
    from paper_2504_19930_b200 import Volume3, normalize_zscore
    from paper_2504_19930_b200.geometry import index_affine_batch, to_matrix, RigidParams

    raw_t, raw_s = _echo_pair()
    sp = (0.87, 1.08, 0.73)
    tv = normalize_zscore(Volume3(raw_t, sp))
    sv = normalize_zscore(Volume3(raw_s, sp))
    assert tv.codec is not None and sv.codec is not None
    rng = np.random.default_rng(1)
    mats = np.stack([to_matrix(RigidParams(*rng.uniform(-0.26, 0.26, 3),
                                           *rng.uniform(-20, 20, 3)), tv.physical_center())
                     for _ in range(12)])
    a, b = index_affine_batch(mats, sp, (0, 0, 0), sp, (0, 0, 0))
    for overlap in (False, True):
        z, d, n = _measure(tv, sv, a, b, overlap, precision)
        zo, do, no = ok.ncc_measure_batch(tv.data, sv.data, a, b, overlap, return_counts=True)
        ok_, err = _close(z, zo, 1e-4 if precision == "f32" else 1e-6)
        assert ok_, (overlap, err)
        assert np.array_equal(d, do)
        assert np.array_equal(n, no)


def test_resample_bit_exact_vs_reference():
    from paper_2504_19930_b200 import kernels_sm100

    for name in ("cube10", "ragged", "flat", "mask12", "tiny_src"):
        c = CASES[name]
        for p in range(c["resampled"].shape[0]):
            out = kernels_sm100.resample_trilinear(c["src"], c["a"][p], c["b"][p],
                                                   c["tgt"].shape)
            assert np.array_equal(out, c["resampled"][p]), (name, p)


def test_kernel_module_seam_host_buffers():
    from paper_2504_19930_b200 import kernels_sm100

    c = CASES["ragged"]
    z, d = kernels_sm100.ncc_measure_batch(c["tgt"], c["src"], c["a"], c["b"], True)
    # the seam measures in the default fp32-lerp mode (quad layout for these
    # f32-valued volumes): the north star's per-particle fp32 bar
    assert _close(z, c["ncc_overlap"], RTOL["f32"])[0]
    assert np.array_equal(d, c["degen_overlap"])
    assert math.isfinite(float(z.sum()))


def _zscored_bytes(dims, seed):
    """The reference's normalize_zscore of 8-bit data (volume.py:119-130) as
    the plain fp64 array its kernel-module seam receives."""
    raw = np.random.default_rng(seed).integers(0, 256, dims).astype(np.float64)
    return (raw - raw.mean()) / raw.std()


def _near_identity_affines(n, seed, shift=2.0):
    g = np.random.default_rng(seed)
    a = np.eye(3)[None] + g.uniform(-0.05, 0.05, (n, 3, 3))
    b = g.uniform(-shift, shift, (n, 3))
    return a, b


def test_kernel_module_seam_recovers_zscored_bytes():
    """z-scored 8-bit volumes reach the seam as fp64; they are recognised as an
    affine image of bytes (stored u8, oct fast path) and measure like the
    reference (f32 tolerance), and the next call reuses the device copies."""
    from paper_2504_19930_b200 import _lib, kernels_sm100

    t = _zscored_bytes((40, 36, 44), 3)
    s = _zscored_bytes((40, 36, 44), 4)
    a, b = _near_identity_affines(24, 5)
    for overlap in (False, True):
        z, d = kernels_sm100.ncc_measure_batch(t, s, a, b, overlap)
        zo, do = ok.ncc_measure_batch(t, s, a, b, overlap)
        assert _close(z, zo, RTOL["f32"])[0], overlap
        assert np.array_equal(d, do)
    dvs = [dv for ref, _fp, dv in kernels_sm100._CACHE.values() if ref() is t]
    assert dvs and all(dv.dtype_code == _lib.ER_U8 for dv in dvs)
    assert abs(dvs[0].desc.alpha * 255 + dvs[0].desc.gamma - t.max()) < 1e-12
    n_cached = len(kernels_sm100._CACHE)
    kernels_sm100.ncc_measure_batch(t, s, a, b, False)
    assert len(kernels_sm100._CACHE) == n_cached
    assert [dv for ref, _fp, dv in kernels_sm100._CACHE.values() if ref() is t][0] is dvs[0]


def test_kernel_module_seam_revalidates_mutated_volumes():
    from paper_2504_19930_b200 import _lib, kernels_sm100

    t = _zscored_bytes((30, 20, 26), 7)
    s = _zscored_bytes((30, 20, 26), 8)
    a, b = _near_identity_affines(12, 9)
    kernels_sm100.ncc_measure_batch(t, s, a, b, False)
    t[0, 0, 0] += 1.0          # off the byte lattice; index 0 is fingerprinted
    z, d = kernels_sm100.ncc_measure_batch(t, s, a, b, False)
    zo, do = ok.ncc_measure_batch(t, s, a, b, False)
    assert _close(z, zo, RTOL["f32"])[0]
    assert np.array_equal(d, do)
    dvs = [dv for ref, _fp, dv in kernels_sm100._CACHE.values() if ref() is t]
    assert [dv.dtype_code for dv in dvs] == [_lib.ER_F64]   # re-uploaded, exact storage


def test_kernel_module_seam_sees_any_in_place_edit():
    """The device copies are validated against the FULL content of the host
    arrays (Volume3.data is writable, /root/reference/pkg/src/echoreg/volume.py:
    32-47): an edit of one interior voxel of either volume -- on the byte
    lattice, so the storage type does not change -- and of the warp's source
    must show up in the next call's results."""
    from paper_2504_19930_b200 import kernels_sm100

    t = _zscored_bytes((30, 20, 26), 17)
    s = _zscored_bytes((30, 20, 26), 18)
    a, b = _near_identity_affines(12, 19, shift=0.5)
    z_prev, _ = kernels_sm100.ncc_measure_batch(t, s, a, b, False)
    # one byte step of each volume's lattice (taken before any edit)
    steps = {id(v): float(np.min(np.diff(np.unique(v)))) for v in (t, s)}
    for vol, idx in ((s, (17, 11, 13)), (t, (13, 7, 19)), (s, (12, 9, 8))):
        step = steps[id(vol)]
        vol[idx] += step if vol[idx] < vol.max() else -step
        z, d = kernels_sm100.ncc_measure_batch(t, s, a, b, False)
        # bitwise what a fresh upload of the edited arrays gives, and not the
        # stale result
        z_fresh, d_fresh = kernels_sm100.ncc_measure_batch(t.copy(), s.copy(), a, b, False)
        assert np.array_equal(z, z_fresh) and np.array_equal(d, d_fresh), idx
        assert not np.array_equal(z, z_prev), idx
        zo, do = ok.ncc_measure_batch(t, s, a, b, False)
        assert _close(z, zo, RTOL["f32"])[0], idx
        assert np.array_equal(d, do)
        z_prev = z
    w = np.arange(30 * 20 * 26, dtype=np.float64).reshape(30, 20, 26)
    eye, zero = np.eye(3), np.zeros(3)
    kernels_sm100.resample_trilinear(w, eye, zero, w.shape)
    w[21, 9, 4] = -5.0
    assert np.array_equal(kernels_sm100.resample_trilinear(w, eye, zero, w.shape), w)


def test_lattice_recognition_rejects_other_data():
    from paper_2504_19930_b200 import _lib
    from paper_2504_19930_b200.device import device_volume_from_array

    g = np.random.default_rng(1)
    for data in (g.standard_normal((20, 20, 20)),                       # continuous
                 np.round(g.standard_normal((20, 20, 20)) * 200) / 7.0,  # > 256 levels
                 _zscored_bytes((20, 20, 20), 2) + 1e-9 * g.standard_normal((20, 20, 20))):
        dv = device_volume_from_array(data, lattice=True)
        assert dv.dtype_code == _lib.ER_F64
    dv = device_volume_from_array(_zscored_bytes((20, 20, 20), 2), lattice=True)
    assert dv.dtype_code == _lib.ER_U8


def _nearest_ncc_numpy(tgt, src, a, b, overlap):
    """Test-only: the reference _ncc_kernel (kernels_numba.py:116-189) with the
    trilinear sample replaced by the nearest corner of the same clamped cell
    (fraction >= 0.5 -> upper) -- the opt-in ER_LERP_NEAREST semantics."""
    nx, ny, nz = tgt.shape
    sx, sy, sz = src.shape
    i, j, k = np.meshgrid(np.arange(nx, dtype=np.float64), np.arange(ny, dtype=np.float64),
                          np.arange(nz, dtype=np.float64), indexing="ij")
    out = np.zeros(a.shape[0])
    for p in range(a.shape[0]):
        A, B = a[p], b[p]
        u = (A[0, 0] * i + A[0, 1] * j + B[0]) + A[0, 2] * k
        v = (A[1, 0] * i + A[1, 1] * j + B[1]) + A[1, 2] * k
        w = (A[2, 0] * i + A[2, 1] * j + B[2]) + A[2, 2] * k
        inb = (u >= 0) & (u <= sx - 1) & (v >= 0) & (v <= sy - 1) & (w >= 0) & (w <= sz - 1)

        def near(c, n):
            c0 = np.clip(np.floor(c), 0, None).astype(np.int64)
            c1 = c0 + 1
            over = c1 > n - 1
            c1 = np.where(over, n - 1, c1)
            c0 = np.where(over, np.maximum(c1 - 1, 0), c0)
            return np.where(c - c0 >= 0.5, c1, c0)

        x = np.zeros_like(u)
        x[inb] = src[near(u[inb], sx), near(v[inb], sy), near(w[inb], sz)]
        t = tgt
        if overlap:
            t, x = t[inb], x[inb]
        n = t.size
        st, ss = t.sum(), x.sum()
        sst = (t * t).sum() - st * st / n
        sss = (x * x).sum() - ss * ss / n
        sts = (t * x).sum() - st * ss / n
        out[p] = 0.0 if sst / n < 1e-12 or sss / n < 1e-12 else sts * sts / (sst * sss)
    return out


@pytest.mark.parametrize("kind", ["mask", "u8", "f64"])
@pytest.mark.parametrize("overlap", [False, True])
def test_nearest_sampling_opt_in(kind, overlap):
    """Executor(precision="nearest"): the north star's nearest-neighbour
    sampling (opt-in; the reference samples trilinearly) on the bit-oct mask
    path, the 8-bit oct path and the generic fp64-storage path."""
    from paper_2504_19930_b200 import Executor, Volume3
    from paper_2504_19930_b200.device import device_volume

    g = np.random.default_rng(11)
    dims = (22, 19, 26)
    if kind == "mask":
        tgt = (g.random(dims) > 0.6).astype(np.float64)
        src = (g.random(dims) > 0.5).astype(np.float64)
    elif kind == "u8":
        tgt = g.integers(0, 256, dims).astype(np.float64)
        src = g.integers(0, 256, dims).astype(np.float64)
    else:
        tgt, src = g.standard_normal(dims), g.standard_normal(dims)
    a, b = _near_identity_affines(16, 12, shift=3.0)
    mats = np.zeros((16, 4, 4))
    mats[:, :3, :3], mats[:, :3, 3], mats[:, 3, 3] = a, b, 1.0   # unit grids: index affine = matrix
    tv, sv = Volume3(tgt), Volume3(src)
    z, d = Executor(precision="nearest").measure_ncc(tv, sv, mats, overlap)
    want = _nearest_ncc_numpy(tgt, src, a, b, overlap)
    assert _close(z, want, 1e-4)[0], (kind, z[:4], want[:4])
    expect_code = {"mask": 0, "u8": 0, "f64": 2}[kind]
    assert device_volume(sv).dtype_code == expect_code
