"""Exhaustive search on the C2 pair against the reference algorithm
(E/exhaustive.py:71-113): a 5x5x3x5x5x3 = 5,625-node grid (the full 9^6
grid would take ~2.6 h on the host) evaluated by register_exhaustive on the
GPU in every precision, and every node's likelihood by the C oracle (the
bit-exact restatement of _ncc_kernel) on all host threads; the winner is the
first maximum (lowest node index), as in the reference.

    python tools/parity_c4_grid.py      (prints one JSON line)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import kernels as ok  # noqa: E402  (checker)
from paper_2504_19930_b200 import Executor, GridSpec, RigidParams, register_exhaustive  # noqa: E402
from paper_2504_19930_b200.exhaustive import _node_states  # noqa: E402
from paper_2504_19930_b200.geometry import index_affine_batch, to_matrix  # noqa: E402


def main():
    t, s, _ = bench.make_workload()
    g = GridSpec(half_counts=(2, 2, 1, 2, 2, 1))
    states = _node_states(g)
    center = t.physical_center()
    mats = np.stack([to_matrix(RigidParams(*st), center) for st in states])
    a, b = index_affine_batch(mats, s.spacing, s.origin, t.spacing, t.origin)
    ok.build()
    t0 = time.perf_counter()
    z_ref, _ = ok.ncc_measure_batch(t.data, s.data, a, b, False, ok.max_threads())
    cpu_s = time.perf_counter() - t0
    best_ref = int(np.argmax(z_ref))  # first maximum
    out = {"config": "exhaustive 5x5x3x5x5x3 = 5625 nodes on the C2 pair (step 2 deg / 2.5 mm)",
           "cpu_s": cpu_s, "host_threads": ok.max_threads(), "best_node_ref": best_ref,
           "best_ncc_ref": float(z_ref[best_ref])}
    for prec in ("f32", "f64", "exact"):
        ex = Executor(precision=prec)
        t0 = time.perf_counter()
        best, score = register_exhaustive(t, s, g, ex)
        gpu_s = time.perf_counter() - t0
        z = ex.measure_ncc(t, s, mats)[0]
        got = np.asarray(best.to_array())
        out[prec] = {"gpu_s": gpu_s,
                     "best_state_equal": bool(np.array_equal(got, states[best_ref])),
                     "best_ncc": float(score),
                     "node_max_rel_diff": float(np.max(np.abs(z - z_ref) /
                                                       np.maximum(np.abs(z_ref), 1e-300)))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
