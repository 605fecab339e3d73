"""The single-CTA device update (er_smc_update) against the reference's
numpy semantics (echoreg/smc.py:203-259): best tracking, update_weights,
ess, resample_systematic with stream (seed, 2, k, 0), estimate, trace row.

The device normaliser and cumulative sum are fixed-order block reductions,
not numpy's pairwise sum / sequential cumsum, so weights agree to ~1e-15
relative; resampling indices, the fired flag and the best index are exact
(SURVEY.md Appendix A.6 found these reorderings parity-safe)."""

import numpy as np
import pytest

from oracle import smc as osmc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _run_update(z, w, states, beta, ess_frac, seed, k, best=-1.0, est_best=False):
    from paper_2504_19930_b200 import _lib
    from paper_2504_19930_b200.device import ptr, require_cuda, stream_ptr
    from paper_2504_19930_b200.smc import _u64

    dev = require_cuda()
    n = z.size
    f64 = dict(dtype=torch.float64, device=dev)
    zt = torch.as_tensor(z, **f64)
    dg = torch.zeros(n, dtype=torch.uint8, device=dev)
    wt = torch.as_tensor(w, **f64)
    st = torch.as_tensor(states, **f64)
    so = torch.empty_like(st)
    zo = torch.empty_like(zt)
    scratch = torch.empty_like(zt)
    trace = torch.zeros(_lib.ER_TRACE_STRIDE, **f64)
    ctl = _lib.ErSmcCtl()
    ctl.best_measurement = best
    ctl_t = torch.frombuffer(bytearray(bytes(memoryview(ctl))), dtype=torch.uint8).to(dev)
    _lib.call("er_smc_update", ptr(zt), ptr(dg), ptr(wt), ptr(st), ptr(so), ptr(zo),
              ptr(scratch), n, float(beta), float(ess_frac), _u64(seed), int(k),
              int(est_best), ptr(ctl_t), ptr(trace), stream_ptr(dev))
    ctl_out = _lib.ErSmcCtl.from_buffer_copy(bytes(ctl_t.cpu().numpy().tobytes()))
    return (wt.cpu().numpy(), so.cpu().numpy(), zo.cpu().numpy(), trace.cpu().numpy(), ctl_out)


def _reference_update(z, w, states, beta, ess_frac, seed, k):
    w2 = osmc.update_weights(w, z, beta)
    ess = float(1.0 / (w2 @ w2))
    fire = ess < ess_frac * z.size
    if fire:
        u0 = osmc.stream(seed, 2, k, 0).uniform(0.0, 1.0 / z.size)
        idx = osmc.resample_indices(w2, u0)
        return np.full(z.size, 1.0 / z.size), states[idx], z[idx], ess, fire
    return w2, states, z, ess, fire


@pytest.mark.parametrize("n", [1, 2, 3, 7, 500, 2000, 4099, 65536])
@pytest.mark.parametrize("beta", [0.0, 20.0, 50.0, 400.0])
def test_update_matches_reference(n, beta):
    rng = np.random.default_rng(n * 31 + int(beta))
    z = rng.random(n) ** 3
    w = rng.random(n)
    w /= w.sum()
    states = rng.normal(size=(n, 6))
    seed, k = 11, 7
    gw, gs, gz, tr, ctl = _run_update(z, w, states, beta, 0.5, seed, k)
    rw, rs, rz, ress, rfire = _reference_update(z, w, states, beta, 0.5, seed, k)
    assert bool(tr[10]) == rfire
    np.testing.assert_allclose(tr[9], ress, rtol=1e-12)
    np.testing.assert_allclose(gw, rw, rtol=1e-12, atol=1e-300)
    assert np.array_equal(gs, rs)        # resampled states: exact gather
    assert np.array_equal(gz, rz)
    top = int(np.argmax(z))
    assert ctl.best_measurement == z[top]
    assert np.array_equal(np.array(ctl.best_state[:]), states[top])
    np.testing.assert_allclose(tr[:6], rw @ rs, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(tr[6], rz.mean(), rtol=1e-12)
    assert tr[7] == rz.max()


def test_reference_hand_cases():
    """The reference's fixtures: weights (0.8, 0.2) for z = (1, 0), beta = ln 4
    (tests/test_smc.py:119-124); ESS 8/3 (tests/test_smc.py:150-153)."""
    gw, _, _, tr, _ = _run_update(np.array([1.0, 0.0]), np.array([0.5, 0.5]),
                                  np.zeros((2, 6)), np.log(4.0), 1e-9, 0, 0)
    np.testing.assert_allclose(gw, [0.8, 0.2], atol=1e-15)
    w = np.array([0.5, 0.25, 0.25])
    gw, _, _, tr, _ = _run_update(np.zeros(3), w, np.zeros((3, 6)), 0.0, 1e-9, 0, 0)
    assert tr[9] == pytest.approx(8.0 / 3.0, rel=1e-15)


def test_uniform_weight_reset_on_underflow():
    """A vanished normaliser resets to uniform (smc.py:219-221)."""
    z = np.array([0.0, 0.0, 0.0])
    w = np.array([0.0, 0.0, 0.0])
    gw, _, _, tr, _ = _run_update(z, w, np.zeros((3, 6)), 1.0, 1e-9, 0, 0)
    np.testing.assert_allclose(gw, np.full(3, 1 / 3), rtol=1e-15)


def test_best_tracking_strict_greater():
    z = np.array([0.2, 0.7, 0.7, 0.1])
    st = np.arange(24, dtype=float).reshape(4, 6)
    _, _, _, _, ctl = _run_update(z, np.full(4, 0.25), st, 1.0, 1e-9, 0, 0, best=0.7)
    assert ctl.has_best == 0          # 0.7 is not > 0.7
    _, _, _, _, ctl = _run_update(z, np.full(4, 0.25), st, 1.0, 1e-9, 0, 0, best=0.5)
    assert np.array_equal(np.array(ctl.best_state[:]), st[1])   # first max wins


def _multi_case(n, beta, seed=5):
    rng = np.random.default_rng(n + int(beta))
    z = rng.random(n) ** 3
    w = rng.random(n)
    w /= w.sum()
    states = rng.normal(size=(n, 6))
    degen = (rng.random(n) < 0.01).astype(np.uint8)
    return z, w, states, degen


def _run_update_both(z, w, states, degen, beta, world=2):
    """er_smc_update on contiguous arrays and er_smc_update_gathered on a
    packed world-rank buffer ([z shard | flags shard | pad] per rank)."""
    from paper_2504_19930_b200 import _lib
    from paper_2504_19930_b200.device import ptr, require_cuda, stream_ptr
    from paper_2504_19930_b200.smc import _u64

    dev = require_cuda()
    n = z.size
    f64 = dict(dtype=torch.float64, device=dev)
    out = []
    for gathered in (False, True):
        zt = torch.as_tensor(z, **f64)
        dg = torch.as_tensor(degen, device=dev)
        wt = torch.as_tensor(w, **f64)
        st = torch.as_tensor(states, **f64)
        so, zo, scratch = torch.empty_like(st), torch.empty_like(zt), torch.empty_like(zt)
        trace = torch.zeros(_lib.ER_TRACE_STRIDE, **f64)
        ctl = _lib.ErSmcCtl()
        ctl.best_measurement = -1.0
        ctl_t = torch.frombuffer(bytearray(bytes(memoryview(ctl))), dtype=torch.uint8).to(dev)
        tail = (ptr(wt), ptr(st), ptr(so), ptr(zo), ptr(scratch), n, float(beta), 0.5,
                _u64(3), 7, 0, ptr(ctl_t), ptr(trace), stream_ptr(dev))
        if gathered:
            shard = -(-n // world)
            block = ((9 * shard + 7) // 8) * 8
            buf = torch.zeros(world * block, dtype=torch.uint8, device=dev)
            zp = np.zeros(world * shard)
            zp[:n] = z
            dp = np.zeros(world * shard, dtype=np.uint8)
            dp[:n] = degen
            for r in range(world):
                seg = np.concatenate([zp[r * shard:(r + 1) * shard].view(np.uint8),
                                      dp[r * shard:(r + 1) * shard]])
                buf[r * block:r * block + seg.size] = torch.as_tensor(seg, device=dev)
            _lib.call("er_smc_update_gathered", ptr(buf), shard, block, *tail)
        else:
            _lib.call("er_smc_update", ptr(zt), ptr(dg), *tail)
        torch.cuda.synchronize()
        out.append(np.concatenate([wt.cpu().numpy(), so.cpu().numpy().ravel(),
                                   zo.cpu().numpy(), trace.cpu().numpy(),
                                   np.frombuffer(ctl_t.cpu().numpy().tobytes(), np.float64)]))
    return out


_SINGLE_SCRIPT = """
import sys, numpy as np
sys.path.insert(0, {root!r})
from tests.test_gpu_update import _multi_case, _run_update_both
z, w, s, d = _multi_case({n}, {beta})
a, b = _run_update_both(z, w, s, d, {beta})
np.save({path!r}, np.stack([a, b]))
"""


@pytest.mark.parametrize("n", [16384, 65537, 262144])
@pytest.mark.parametrize("beta", [0.0, 50.0])
def test_multi_cta_update_bit_identical(n, beta, tmp_path):
    """At n >= 16384 the update runs as a chain of whole-GPU kernels (13
    launches, same per-chunk loops and reduction trees); it must reproduce the
    single-CTA kernel (forced with ER_SMC_UPDATE_SINGLE=1 in a subprocess)
    bit for bit, contiguous and gathered, with and without resampling."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    z, w, s, d = _multi_case(n, beta)
    multi = np.stack(_run_update_both(z, w, s, d, beta))
    path = str(tmp_path / "single.npy")
    env = dict(os.environ, ER_SMC_UPDATE_SINGLE="1")
    subprocess.run([sys.executable, "-c", _SINGLE_SCRIPT.format(root=root, n=n, beta=beta,
                                                                path=path)],
                   check=True, env=env, cwd=root)
    single = np.load(path)
    assert np.array_equal(multi.view(np.uint64), single.view(np.uint64))
    assert np.array_equal(multi[0], multi[1])          # gathered == contiguous
