"""One config-4 step at a small shard (default 64 instances, the 8-GPU shard): for ncu captures.
python tools/cfg4_small_shard.py [instances] [sweeps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402

inst = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
wl = WL.build(T, 4, None, instances=inst)
e = wl["ens"]
e.run(sweeps, swap_every=1)
e.synchronize()
print(e.launch_log(), np.asarray(e.energies()).mean())
