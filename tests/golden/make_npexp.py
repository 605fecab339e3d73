"""Known-answer vectors for numpy's float64 exp (the reference's phantom
speckle, E/phantom.py:77), which csrc/npexp.cuh restates.  numpy is the
reference's own dependency (2.3.5 here); on this AVX512_SKX host np.exp runs
the bundled SVML __svml_exp8_ha.  The vectors pin that variant so the test
does not depend on the CPU of the machine that runs it.

    python tests/golden/make_npexp.py
"""
import os

import numpy as np
from numpy._core._multiarray_umath import __cpu_features__

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "npexp.npz")

if __name__ == "__main__":
    assert __cpu_features__.get("AVX512_SKX"), "generate on an AVX512_SKX host"
    g = np.random.Generator(np.random.Philox(key=2504))
    x = np.concatenate([
        0.3 * g.standard_normal(60000),            # the phantom's arguments
        g.uniform(-700.0, 700.0, 4000),            # the whole non-special range
        g.uniform(-1e-6, 1e-6, 500),
        [0.0, -0.0, 5e-324, -5e-324, 1e-300, 1.0, -1.0, np.log(2.0), -np.log(2.0),
         700.0, -700.0, 707.0, -707.0],
    ])
    np.savez_compressed(OUT, x=x, exp=np.exp(x), numpy_version=np.array(np.__version__))
    print(OUT, x.size)
