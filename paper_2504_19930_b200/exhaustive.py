"""Exhaustive 6-DOF grid search on the device (reference exhaustive.py).

Node states are generated on the device straight from the flat
lexicographic index (last axis fastest, exhaustive.py:71-75) and turned into
index affines there (er_grid_to_affine); chunks are measured with the same
kernel as the SMC and folded into a running first-max with a strict '>'
(er_argmax_update), so the lowest node index wins ties exactly as in
exhaustive.py:106-109.  With world_size > 1 each rank scans a contiguous
node range and the (value, index) pairs are all-gathered and reduced with
the same tie-break.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib, dist, ops
from .backend import Executor
from .device import device_volume, ptr, require_cuda, stream_ptr, torch
from .errors import BadConfig
from .geometry import RigidParams
from .metrics import MetricValue
from .volume import Volume3

CHUNK = 4096            # the reference's batch size (exhaustive.py:22)
DEVICE_CHUNK = 65536    # nodes per device launch (result independent of chunking)


@dataclass(frozen=True)
class GridSpec:
    """Per-axis half counts and steps, axis order (rx, ry, rz, tx, ty, tz)
    (exhaustive.py:25-68)."""

    half_counts: tuple = (4, 4, 4, 4, 4, 4)
    step_t: float = 2.5
    step_r: float = 2.0

    def validate(self):
        if len(self.half_counts) != 6 or any(m < 0 for m in self.half_counts):
            raise BadConfig(f"half counts must be six integers >= 0, got {self.half_counts}")
        if any(self.half_counts[:3]) and self.step_r <= 0:
            raise BadConfig(f"step_r must be positive, got {self.step_r}")
        if any(self.half_counts[3:]) and self.step_t <= 0:
            raise BadConfig(f"step_t must be positive, got {self.step_t}")

    @property
    def n_nodes(self) -> int:
        return int(np.prod([2 * m + 1 for m in self.half_counts]))

    def axis_steps(self) -> list:
        return [math.radians(self.step_r)] * 3 + [self.step_t] * 3

    def axis_values(self) -> list:
        return [np.arange(-m, m + 1, dtype=np.float64) * s
                for m, s in zip(self.half_counts, self.axis_steps())]

    def node_state(self, index: int) -> np.ndarray:
        axes = self.axis_values()
        sizes = [len(a) for a in axes]
        out = np.empty(6)
        rest = index
        for axis in range(5, -1, -1):
            rest, pos = divmod(rest, sizes[axis])
            out[axis] = axes[axis][pos]
        return out


def _node_states(g: GridSpec) -> np.ndarray:
    axes = g.axis_values()
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1)


def register_exhaustive(target: Volume3, source: Volume3, g: GridSpec,
                        executor: Executor | None = None, ncc_region: str = "full"):
    """Highest-NCC grid node and its score (exhaustive.py:78-113)."""
    g.validate()
    if ncc_region not in ("full", "overlap"):
        raise BadConfig(f"ncc_region must be full or overlap, got {ncc_region!r}")
    executor = executor or Executor()
    if type(executor).measure_ncc is not Executor.measure_ncc:
        return _register_exhaustive_via_seam(target, source, g, executor, ncc_region)
    dev = require_cuda(executor.device)
    t = torch()
    tdv, sdv = device_volume(target, dev), device_volume(source, dev)
    n_nodes = g.n_nodes
    w, r, _ = dist.world()
    per = -(-n_nodes // w)
    lo, hi = min(n_nodes, r * per), min(n_nodes, (r + 1) * per)
    f64 = dict(dtype=t.float64, device=dev)
    best = t.tensor([-1.0, -1.0], **f64)
    chunk = min(DEVICE_CHUNK, max(hi - lo, 1))
    A = t.empty((chunk, 9), **f64)
    B = t.empty((chunk, 3), **f64)
    out = (t.empty(chunk, **f64), t.empty(chunk, dtype=t.uint8, device=dev),
           t.empty(chunk, dtype=t.int64, device=dev))
    center = target.physical_center()
    half = _lib.i6(g.half_counts)
    steps = _lib.d6(g.axis_steps())
    st = stream_ptr(dev)
    for start in range(lo, hi, chunk):
        cnt = min(chunk, hi - start)
        _lib.call("er_grid_to_affine", start, cnt, half, steps, _lib.d3(center),
                  _lib.d3(target.spacing), _lib.d3(target.origin), _lib.d3(source.spacing),
                  _lib.d3(source.origin), None, ptr(A), ptr(B), st)
        z, _, _ = ops.measure(tdv, sdv, A[:cnt], B[:cnt], ncc_region == "overlap",
                              executor.precision, out=tuple(o[:cnt] for o in out))
        _lib.call("er_argmax_update", ptr(z), cnt, start, ptr(best), st)
    if w > 1:
        allb = t.empty(2 * w, **f64)
        dist.allgather_tensor(best, allb)
        pairs = allb.view(w, 2).cpu().numpy()
        best_value, best_index = -1.0, -1
        for v, i in pairs:  # ranks hold increasing node ranges: strict '>' keeps lowest
            if v > best_value:
                best_value, best_index = float(v), int(i)
    else:
        best_value, best_index = (float(x) for x in best.cpu().numpy())
        best_index = int(best_index)
    return (RigidParams.from_array(g.node_state(best_index)),
            MetricValue(best_value, "NCC"))


def _register_exhaustive_via_seam(target, source, g, executor, ncc_region):
    """Path for Executor subclasses that override measure_ncc (the reference's
    test seam, tests/test_exhaustive.py:109-120): host chunks of CHUNK nodes
    through the overridden method, exactly as exhaustive.py:98-109."""
    from .geometry import to_matrix

    center = target.physical_center()
    states = _node_states(g)
    best_value, best_index = -1.0, -1
    for start in range(0, states.shape[0], CHUNK):
        block = states[start: start + CHUNK]
        mats = np.stack([to_matrix(RigidParams.from_array(row), center) for row in block])
        scores, _ = executor.measure_ncc(target, source, mats,
                                         overlap_only=(ncc_region == "overlap"))
        top = int(np.argmax(scores))
        if float(scores[top]) > best_value:
            best_value = float(scores[top])
            best_index = start + top
    return RigidParams.from_array(states[best_index]), MetricValue(best_value, "NCC")
