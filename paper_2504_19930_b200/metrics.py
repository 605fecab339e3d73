"""Similarity and overlap measures on the device (reference metrics.py).

``ncc`` is the two-pass centred squared NCC over the full grid
(metrics.py:49-68) computed by er_warp_ncc_sums; ``dice`` /
``dice_under_transform`` are exact integer voxel counts from
er_warp_dice_counts (metrics.py:71-93), whose fp64 warp reproduces the
reference's samples bit for bit, so the strict '> 0.5' cut and every count
match exactly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import ops
from .errors import DegenerateInput, DimMismatch
from .volume import VARIANCE_EPS, Volume3, require_binary

_RANGE_SLACK = 1e-9


@dataclass(frozen=True)
class MetricValue:
    """A score in [0, 1] tagged with its kind (metrics.py:27-41)."""

    value: float
    kind: str

    def __post_init__(self):
        v = float(self.value)
        if not (-_RANGE_SLACK <= v <= 1.0 + _RANGE_SLACK):
            raise ValueError(f"{self.kind} value {v} outside [0, 1]")
        object.__setattr__(self, "value", min(max(v, 0.0), 1.0))

    def __float__(self) -> float:
        return self.value


def _check_dims(a: Volume3, b: Volume3):
    if a.dims != b.dims:
        raise DimMismatch(f"volume dims differ: {a.dims} vs {b.dims}")


def ncc_from_sums(sst: float, sss: float, sts: float, n: float) -> MetricValue:
    if sst / n < VARIANCE_EPS:
        raise DegenerateInput("target volume is constant; NCC undefined")
    if sss / n < VARIANCE_EPS:
        raise DegenerateInput("source volume is constant; NCC undefined")
    return MetricValue((sts * sts) / (sst * sss), "NCC")


def ncc(t: Volume3, s: Volume3) -> MetricValue:
    """Squared NCC between two same-grid volumes (metrics.py:49-68)."""
    _check_dims(t, s)
    sst, sss, sts, n = (float(x) for x in ops.ncc_sums(t, s, identity=True).cpu().numpy())
    return ncc_from_sums(sst, sss, sts, n)


def ncc_under_transform(t: Volume3, s: Volume3, m: np.ndarray) -> MetricValue:
    """ncc(t, resample(s, t, m)) fused on the device (pipeline.py:126-128)."""
    from .geometry import index_affine

    a, b = index_affine(m, s, t)
    sst, sss, sts, n = (float(x) for x in ops.ncc_sums(t, s, a, b).cpu().numpy())
    return ncc_from_sums(sst, sss, sts, n)


def _dice_from_counts(na: int, nb: int, inter: int) -> MetricValue:
    if na == 0 and nb == 0:
        return MetricValue(1.0, "DSC")
    return MetricValue(2.0 * float(inter) / (float(na) + float(nb)), "DSC")


def dice(a: Volume3, b: Volume3) -> MetricValue:
    """Dice of two binary masks; both empty -> 1.0 (metrics.py:71-85)."""
    _check_dims(a, b)
    require_binary(a, "first mask")
    require_binary(b, "second mask")
    counts = ops.dice_counts(a, b, np.eye(3), np.zeros(3)).cpu().numpy()
    return _dice_from_counts(int(counts[0]), int(counts[1]), int(counts[2]))


def dice_under_transform(a: Volume3, b: Volume3, m: np.ndarray) -> MetricValue:
    """Dice of mask a pulled onto b's grid under m, cut at > 0.5 (metrics.py:88-93)."""
    from .geometry import index_affine

    _check_dims(a, b)
    require_binary(a, "first mask")
    require_binary(b, "second mask")
    A, B = index_affine(m, a, b)
    counts = ops.dice_counts(a, b, A, B).cpu().numpy()
    return _dice_from_counts(int(counts[0]), int(counts[1]), int(counts[2]))
