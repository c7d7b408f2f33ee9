"""torch.profiler breakdown of config 2's TAPT rounds (generate_proposals: 60 targets, 5 refinement sweeps)
and of its 100-sweep runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402

stream = torch.cuda.Stream()
w = WL.build(T, 2, stream.cuda_stream)
e = w["ens"]
mb = np.array([WL.yang_m(x) for x in WL.geometric(0.3, 0.6, 64)[:60]])
w["step"]()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for _ in range(5):
        e.run(100, swap_every=1, measure_every=10)
        e.generate_proposals(np.arange(60), mb, refine=5, return_accepted=False)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=14))
