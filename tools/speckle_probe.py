"""The device speckle of the C2-sized phantom (6.4M normals), three times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_19930_b200.phantom import echo_spec  # noqa: E402
from paper_2504_19930_b200.phantom_device import speckle  # noqa: E402

spec = echo_spec()
for _ in range(3):
    speckle(spec)
torch.cuda.synchronize()
print("ok")
