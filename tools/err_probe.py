"""Per-precision error of the measurement on the C1 golden particles
(iteration 0) against the reference's own likelihoods: max relative and
absolute error, and where it occurs (GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.test_gpu_measure import _c1, _measure, _vol
g, t, s = _c1()
tv, sv = _vol(t, (1, 1, 1), (0, 0, 0)), _vol(s, (1, 1, 1), (0, 0, 0))
ref = g["c1_z"][0]
for prec in ("f32", "f64", "exact"):
    z = _measure(tv, sv, g["c1_a_it0"], g["c1_b_it0"], False, prec)[0]
    rel = np.abs(z - ref) / np.maximum(np.abs(ref), 1e-300)
    i = int(np.argmax(rel))
    print(prec, "max rel", rel.max(), "at z", ref[i], "abs", abs(z[i] - ref[i]),
          "max abs", np.abs(z - ref).max(), "rel for z>1e-3:", rel[ref > 1e-3].max(),
          "n(z<1e-4)", int((ref < 1e-4).sum()))
