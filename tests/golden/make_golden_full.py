"""Full-scale golden fixtures from the REAL reference package: BASELINE C2
(image-mode SMC, 2000 particles x 50 iterations on the 176x176x208 8-bit echo
pair) and C3 (mask-mode register_sequence over a 30-frame 4D cycle of the
same grid).  Run in the build container only (/root/reference does not exist
on the GPU box); about an hour of CPU at 8 numba threads:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_full.py [c2] [c3] [c2o] [c2s:<seed> ...] [c3s:<seed> ...] [c2os:<seed> ...]

Inputs are built with the reference's own generator (echoreg.phantom
make_phantom / make_pair, phantom.py:61-166) on the echo grid of BASELINE
C2 (semi-axes scaled by extent/64, spacing 0.87 x 1.08 x 0.73 mm), then
quantised to 8 bit as clip(round(x * 255 / p99.9(frame 0)), 0, 255) -- the
same recipe as paper_2504_19930_b200.phantom.echo_case and
oracle.phantom.echo_case.  The fixtures store SHA-256 digests of the input
bytes, so a GPU test can prove it measured the identical pair before
comparing trajectories.  Everything else is the reference's output:
register_smc (smc.py:325-373) through Executor/kernels_numba, and
register_sequence (pipeline.py:155-216).
"""

from __future__ import annotations

import hashlib
import math
import os
import sys
import time

os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count() or 8))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from echoreg import smc  # noqa: E402
from echoreg.backend import Executor  # noqa: E402
from echoreg.geometry import RigidParams  # noqa: E402
from echoreg.phantom import PhantomSpec, make_pair, make_phantom  # noqa: E402
from echoreg.pipeline import register_sequence  # noqa: E402
from echoreg.volume import Sequence4, Volume3, binarize, normalize_zscore  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
DIMS = (176, 176, 208)
SPACING = (0.87, 1.08, 0.73)
TRUTH = RigidParams(math.radians(5.0), math.radians(-8.0), math.radians(4.0), 6.0, -4.0, 3.0)


def echo_spec(frames):
    ext = [d * s for d, s in zip(DIMS, SPACING)]
    f = [e / 64.0 for e in ext]
    return PhantomSpec(dims=DIMS, spacing=SPACING,
                       outer_semiaxes=tuple(a * k for a, k in zip((22.0, 18.0, 26.0), f)),
                       inner_semiaxes=tuple(a * k for a, k in zip((14.0, 11.0, 17.0), f)),
                       speckle_sigma=0.3, amplitude=0.25, frames=frames, seed=0)


def echo_case(frames):
    seq, masks = make_phantom(echo_spec(frames))
    case = make_pair(seq, masks, TRUTH)
    scale = 255.0 / float(np.percentile(seq.frames[0].data, 99.9))

    def q(v):
        return Volume3(np.clip(np.round(v.data * scale), 0.0, 255.0), v.spacing, v.origin)

    tq = Sequence4([q(f) for f in case.target.frames], frame_rate=seq.frame_rate,
                   ed_index=seq.ed_index)
    sq = Sequence4([q(f) for f in case.source.frames], frame_rate=seq.frame_rate,
                   ed_index=seq.ed_index)
    return tq, sq, case.target_masks, case.source_masks


def digest(vols):
    h = hashlib.sha256()
    for v in vols:
        h.update(np.ascontiguousarray(v.data).astype(np.uint8).tobytes())
    return h.hexdigest()


class RecordingExecutor(Executor):
    """Keeps the first and last measured batch (reference seam backend.py:78-108)."""

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        object.__setattr__(self, "log", [])

    def measure_ncc(self, target, source, mats, overlap_only=False):
        out = super().measure_ncc(target, source, mats, overlap_only)
        self.log.append((out[0].copy(), out[1].copy()))
        if len(self.log) > 2:
            del self.log[1]
        return out


def trace_arrays(est, trace):
    return {
        "estimate": est.to_array(),
        "estimates": np.stack([e.to_array() for e in trace.estimates]),
        "mean_measurement": np.array(trace.mean_measurement),
        "max_measurement": np.array(trace.max_measurement),
        "best_measurement": np.array(trace.best_measurement),
        "ess": np.array(trace.ess),
        "resampled": np.array(trace.resampled),
        "best_particle": trace.best_particle.to_array(),
    }


def c2():
    tq, sq, _, _ = echo_case(1)
    t = normalize_zscore(tq.frames[0])
    s = normalize_zscore(sq.frames[0])
    cfg = smc.SmcConfig(mode="image", n_particles=2000, n_iterations=50, seed=0)
    rec = RecordingExecutor(workers=int(os.environ["NUMBA_NUM_THREADS"]))
    t0 = time.perf_counter()
    est, trace = smc.register_smc(t, s, cfg, rec)
    wall = time.perf_counter() - t0
    out = {f"c2_{k}": v for k, v in trace_arrays(est, trace).items()}
    out["c2_z_first"], out["c2_degen_first"] = rec.log[0]
    out["c2_z_last"], out["c2_degen_last"] = rec.log[-1]
    out["c2_target_sha256"] = np.array(digest([tq.frames[0]]))
    out["c2_source_sha256"] = np.array(digest([sq.frames[0]]))
    out["c2_zscore"] = np.array([t.data.mean(), t.data.std(), s.data.mean(), s.data.std()])
    out["c2_cpu_s"] = np.array(wall)
    np.savez_compressed(os.path.join(OUT, "full_c2.npz"), **out)
    print("full_c2.npz", wall, "s; estimate deg", np.degrees(est.to_array()[:3]),
          est.to_array()[3:], flush=True)


def c2os(seed):
    """c2o at another SMC seed (full_c2o_seed<seed>.npz)."""
    c2o(int(seed))


def c2o(seed=3):
    """C2 in the overlap region (SmcConfig.ncc_region="overlap",
    kernels_numba.py:172-189 overlap branch): fewer iterations (20), same
    pair, seed 3."""
    tq, sq, _, _ = echo_case(1)
    t = normalize_zscore(tq.frames[0])
    s = normalize_zscore(sq.frames[0])
    cfg = smc.SmcConfig(mode="image", n_particles=2000, n_iterations=20, seed=seed,
                        ncc_region="overlap")
    rec = RecordingExecutor(workers=int(os.environ["NUMBA_NUM_THREADS"]))
    t0 = time.perf_counter()
    est, trace = smc.register_smc(t, s, cfg, rec)
    wall = time.perf_counter() - t0
    out = {f"c2o_{k}": v for k, v in trace_arrays(est, trace).items()}
    out["c2o_z_first"], out["c2o_degen_first"] = rec.log[0]
    out["c2o_z_last"], out["c2o_degen_last"] = rec.log[-1]
    out["c2o_target_sha256"] = np.array(digest([tq.frames[0]]))
    out["c2o_source_sha256"] = np.array(digest([sq.frames[0]]))
    out["c2o_cpu_s"] = np.array(wall)
    name = "full_c2o.npz" if seed == 3 else f"full_c2o_seed{seed}.npz"
    out["c2o_seed"] = np.array(seed)
    np.savez_compressed(os.path.join(OUT, name), **out)
    print(name, wall, "s; estimate deg", np.degrees(est.to_array()[:3]),
          est.to_array()[3:], flush=True)


def c2s(seed):
    """C2 (image mode, 2000 x 50) at another SMC seed, same pair: the
    trajectory, resampling flags, ESS and the first iteration's likelihoods
    (full_c2_seed<seed>.npz)."""
    seed = int(seed)
    tq, sq, _, _ = echo_case(1)
    t = normalize_zscore(tq.frames[0])
    s = normalize_zscore(sq.frames[0])
    cfg = smc.SmcConfig(mode="image", n_particles=2000, n_iterations=50, seed=seed)
    rec = RecordingExecutor(workers=int(os.environ["NUMBA_NUM_THREADS"]))
    t0 = time.perf_counter()
    est, trace = smc.register_smc(t, s, cfg, rec)
    wall = time.perf_counter() - t0
    out = {f"c2_{k}": v for k, v in trace_arrays(est, trace).items()}
    out["c2_z_first"], out["c2_degen_first"] = rec.log[0]
    out["c2_target_sha256"] = np.array(digest([tq.frames[0]]))
    out["c2_source_sha256"] = np.array(digest([sq.frames[0]]))
    out["c2_seed"] = np.array(seed)
    out["c2_cpu_s"] = np.array(wall)
    np.savez_compressed(os.path.join(OUT, f"full_c2_seed{seed}.npz"), **out)
    print(f"full_c2_seed{seed}.npz", wall, "s; estimate deg", np.degrees(est.to_array()[:3]),
          est.to_array()[3:], flush=True)


def c3s(seed):
    """C3 at another SMC seed (full_c3_seed<seed>.npz, no report file)."""
    c3(int(seed))


def c3(seed=0):
    tq, sq, tm, sm = echo_case(30)
    cfg = smc.SmcConfig(mode="mask", n_particles=2000, n_iterations=50, seed=seed)
    ex = Executor(workers=int(os.environ["NUMBA_NUM_THREADS"]))
    t0 = time.perf_counter()
    rep = register_sequence(tq, sq, tm, sm, cfg, ex, case_id="c3")
    wall = time.perf_counter() - t0
    keys = ("rx_deg", "ry_deg", "rz_deg", "tx_mm", "ty_mm", "tz_mm")
    tr = rep.trace
    out = {
        "c3_estimate_deg_mm": np.array([rep.estimate_deg_mm[k] for k in keys]),
        "c3_best_deg_mm": np.array([rep.best_estimate_deg_mm[k] for k in keys]),
        "c3_ncc_before": np.array(rep.ncc_before), "c3_ncc_after": np.array(rep.ncc_after),
        "c3_dsc_before": np.array(rep.dsc_before), "c3_dsc_after": np.array(rep.dsc_after),
        "c3_ess": np.array(tr["ess"]), "c3_resampled": np.array(tr["resampled"]),
        "c3_trace_dsc": np.array(tr["dsc"], dtype=np.float64),
        "c3_mean_measurement": np.array(tr["mean_measurement"]),
        "c3_estimates_deg_mm": np.array([[e[k] for k in keys] for e in tr["estimates_deg_mm"]]),
        "c3_target_sha256": np.array(digest(tq.frames)),
        "c3_source_sha256": np.array(digest(sq.frames)),
        "c3_target_masks_sha256": np.array(digest(tm)),
        "c3_source_masks_sha256": np.array(digest(sm)),
        "c3_cpu_s": np.array(wall),
    }
    if seed:
        out["c3_seed"] = np.array(seed)
        np.savez_compressed(os.path.join(OUT, f"full_c3_seed{seed}.npz"), **out)
    else:
        np.savez_compressed(os.path.join(OUT, "full_c3.npz"), **out)
        rep.save(os.path.join(OUT, "full_c3_report.json"))
    print(f"full_c3_seed{seed}.npz" if seed else "full_c3.npz", wall, "s; estimate",
          rep.estimate_deg_mm, flush=True)


if __name__ == "__main__":
    for w in sys.argv[1:] or ["c2", "c3", "c2o"]:
        name, _, arg = w.partition(":")   # c2s:<seed>
        globals()[name](*([arg] if arg else []))
