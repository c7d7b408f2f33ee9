"""Config 2: time of the sweep/swap runs vs the TAPT proposal rounds (generate_proposals)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402

stream = torch.cuda.Stream()
w = WL.build(T, 2, stream.cuda_stream)
e = w["ens"]
b = WL.geometric(0.3, 0.6, 64)
mb = np.array([WL.yang_m(x) for x in b[:60]])
w["step"]()
ev = lambda: torch.cuda.Event(enable_timing=True)
tr, tp = 0.0, 0.0
for _ in range(10):
    a0, a1, a2 = ev(), ev(), ev()
    a0.record(stream)
    e.run(100, swap_every=1, measure_every=10)
    a1.record(stream)
    e.generate_proposals(np.arange(60), mb, refine=5, return_accepted=False)
    a2.record(stream)
    torch.cuda.synchronize()
    tr += a0.elapsed_time(a1)
    tp += a1.elapsed_time(a2)
print(f"config 2 per 1000 sweeps: runs {tr:.2f} ms, proposal rounds {tp:.2f} ms ({100 * tp / (tr + tp):.1f} %)")
upd_run = 128 * 64 * 4096 * 1000
upd_prop = 128 * 10 * 60 * 4096 * 5
print(f"run rate {upd_run / tr / 1e6:.3g} G/s, proposal-round rate (refine updates) {upd_prop / tp / 1e6:.3g} G/s")
