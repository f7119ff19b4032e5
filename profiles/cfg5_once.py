"""One cfg5 MoE layer forward at G = 1 (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02402_b200 as db  # noqa: E402
from paper_1707_02402_b200.moe_ep import MoeEpLayer  # noqa: E402

db.device_open(0)
layer = MoeEpLayer(1024, 4, 1048576, 2048, 2048, seed=0)
layer.forward(1)
layer.forward(1)
layer.sess.synchronize()
