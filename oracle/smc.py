"""numpy restatement of the reference SMC loop -- TEST INFRASTRUCTURE ONLY.

Follows /root/reference/pkg/src/echoreg/smc.py and geometry.py line by line
(cited per function) with the measurement done by the C oracle
(``oracle.kernels``).  Randomness is numpy's Philox exactly as the reference
draws it (smc.py:38-42), so this is the reference algorithm on the reference
RNG.  Pinned by tests/test_oracle.py against tests/golden/smc.npz, which was
produced by the real reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import kernels

ROLE_INIT, ROLE_PREDICT, ROLE_RESAMPLE = 0, 1, 2  # smc.py:31-33


def stream(seed, role, step, index):
    """smc.py:38-42"""
    return np.random.Generator(np.random.Philox(key=seed, counter=[0, role, step, index]))


def rotation_xyz(rx, ry, rz):
    """geometry.py:76-84"""
    cx, sx = math.cos(rx), math.sin(rx)
    cy, sy = math.cos(ry), math.sin(ry)
    cz, sz = math.cos(rz), math.sin(rz)
    rmx = np.array([[1.0, 0.0, 0.0], [0.0, cx, -sx], [0.0, sx, cx]])
    rmy = np.array([[cy, 0.0, sy], [0.0, 1.0, 0.0], [-sy, 0.0, cy]])
    rmz = np.array([[cz, -sz, 0.0], [sz, cz, 0.0], [0.0, 0.0, 1.0]])
    return rmz @ rmy @ rmx


def to_matrix(state, center):
    """geometry.py:87-99"""
    c = np.asarray(center, dtype=np.float64)
    t = np.array(state[3:6], dtype=np.float64)
    r = rotation_xyz(*state[:3])
    m = np.eye(4)
    m[:3, :3] = r
    m[:3, 3] = r @ (t - c) + c
    return m


def index_affine(m, src_spacing, src_origin, ref_spacing, ref_origin):
    """geometry.py:136-152"""
    r = m[:3, :3]
    t = m[:3, 3]
    st = np.asarray(ref_spacing, dtype=np.float64)
    ss = np.asarray(src_spacing, dtype=np.float64)
    ot = np.asarray(ref_origin, dtype=np.float64)
    os_ = np.asarray(src_origin, dtype=np.float64)
    return (r * st[np.newaxis, :]) / ss[:, np.newaxis], (r @ ot + t - os_) / ss


def physical_center(dims, spacing, origin):
    """volume.py:58-63"""
    return tuple(o + 0.5 * (n - 1) * s for o, n, s in zip(origin, dims, spacing))


@dataclass(frozen=True)
class Cfg:
    """SmcConfig defaults (smc.py:50-62)."""

    n_particles: int = 256
    n_iterations: int = 50
    t_limit: float = 20.0
    r_limit: float = 15.0
    sigma0_t: float = 2.0
    sigma0_r: float = 2.0
    anneal_gamma: float = 0.95
    beta: float = 50.0
    ess_fraction: float = 0.5
    seed: int = 0
    mode: str = "image"
    estimate: str = "weighted_mean"
    ncc_region: str = "full"

    def state_limits(self):
        r = math.radians(self.r_limit)
        return np.array([r, r, r, self.t_limit, self.t_limit, self.t_limit])

    def state_sigma0(self):
        sr = math.radians(self.sigma0_r)
        return np.array([sr, sr, sr, self.sigma0_t, self.sigma0_t, self.sigma0_t])


def init_states(cfg):
    """smc.py:145-157"""
    lim = cfg.state_limits()
    return stream(cfg.seed, ROLE_INIT, 0, 0).uniform(-lim, lim, size=(cfg.n_particles, 6))


def predict(states, k, cfg):
    """smc.py:160-174"""
    sigma = cfg.state_sigma0() * (cfg.anneal_gamma ** k)
    lim = 2.0 * cfg.state_limits()
    out = states.copy()
    for i in range(out.shape[0]):
        out[i] += sigma * stream(cfg.seed, ROLE_PREDICT, k, i).standard_normal(6)
    np.clip(out, -lim, lim, out=out)
    return out


def affines_for(states, tgt_geom, src_geom):
    """smc.py:188-191 + backend.py:87-94 (tgt_geom/src_geom = (dims, spacing, origin))."""
    center = physical_center(*tgt_geom)
    a = np.empty((states.shape[0], 3, 3))
    b = np.empty((states.shape[0], 3))
    for i, row in enumerate(states):
        a[i], b[i] = index_affine(to_matrix(row, center), src_geom[1], src_geom[2],
                                  tgt_geom[1], tgt_geom[2])
    return a, b


def update_weights(weights, z, beta):
    """smc.py:210-224"""
    logw = beta * z
    w = weights * np.exp(logw - logw.max())
    total = float(w.sum())
    if not math.isfinite(total) or total <= 0.0:
        return np.full(z.shape[0], 1.0 / z.shape[0])
    return w / total


def resample_indices(weights, u0):
    """smc.py:232-248 (index part; u0 drawn by the caller)."""
    n = weights.shape[0]
    positions = u0 + np.arange(n) / n
    cumw = np.cumsum(weights)
    return np.minimum(np.searchsorted(cumw, positions, side="right"), n - 1)


@dataclass
class Trace:
    estimates: list = field(default_factory=list)
    mean_measurement: list = field(default_factory=list)
    max_measurement: list = field(default_factory=list)
    best_measurement: list = field(default_factory=list)
    ess: list = field(default_factory=list)
    resampled: list = field(default_factory=list)
    z: list = field(default_factory=list)
    best_particle: np.ndarray | None = None


def register(tgt, src, tgt_geom, src_geom, cfg, workers=0, measure=None):
    """smc.py:325-373 (without the optional Dice trace).

    ``measure(a, b, overlap) -> (z, degen)`` defaults to the C oracle; the
    multi-rank host-logic tests substitute a sharded variant.
    """
    if measure is None:
        def measure(a, b, overlap):
            return kernels.ncc_measure_batch(tgt, src, a, b, overlap, workers)
    n = cfg.n_particles
    states = init_states(cfg)
    weights = np.full(n, 1.0 / n)
    best_m, best_s = -1.0, None
    tr = Trace()
    for k in range(cfg.n_iterations):
        states = predict(states, k, cfg)
        a, b = affines_for(states, tgt_geom, src_geom)
        z, _ = measure(a, b, cfg.ncc_region == "overlap")
        tr.z.append(z.copy())
        top = int(np.argmax(z))
        if float(z[top]) > best_m:
            best_m, best_s = float(z[top]), states[top].copy()
        weights = update_weights(weights, z, cfg.beta)
        ess = float(1.0 / (weights @ weights))
        fire = ess < cfg.ess_fraction * n
        if fire:
            u0 = stream(cfg.seed, ROLE_RESAMPLE, k, 0).uniform(0.0, 1.0 / n)
            idx = resample_indices(weights, u0)
            states = states[idx].copy()
            z = z[idx].copy()
            weights = np.full(n, 1.0 / n)
        if cfg.estimate == "best_particle" and best_s is not None:
            est = best_s.copy()
        else:
            est = weights @ states
        tr.estimates.append(est)
        tr.mean_measurement.append(float(z.mean()))
        tr.max_measurement.append(float(z.max()))
        tr.best_measurement.append(best_m)
        tr.ess.append(ess)
        tr.resampled.append(bool(fire))
    tr.best_particle = best_s
    return tr.estimates[-1], tr


def ncc_full(t, s):
    """metrics.py:49-68 (value only; None when degenerate)."""
    td, sd = t.ravel(), s.ravel()
    n = td.size
    dt, ds = td - td.mean(), sd - sd.mean()
    sst, sss = float(dt @ dt), float(ds @ ds)
    if sst / n < 1e-12 or sss / n < 1e-12:
        return None
    sts = float(dt @ ds)
    return min(max((sts * sts) / (sst * sss), 0.0), 1.0)


def dice(a, b):
    """metrics.py:71-85"""
    sa, sb = float(a.sum()), float(b.sum())
    if sa == 0.0 and sb == 0.0:
        return 1.0
    return 2.0 * float((a * b).sum()) / (sa + sb)


def dice_under_transform(a, b, m, a_geom, b_geom):
    """metrics.py:88-93: warp mask a onto b's grid, cut at > 0.5."""
    A, bb = index_affine(m, a_geom[1], a_geom[2], b_geom[1], b_geom[2])
    moved = (kernels.resample_trilinear(a, A, bb, b.shape) > 0.5).astype(np.float64)
    return dice(moved, b)
