"""Share of the per-sweep epilogue (swap pass, measurement) in the fused run: config-1, -3, -4 and
-5 ensembles timed with swap_every = 1 / 0 and measure_every = 0 / 1."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402

stream = torch.cuda.Stream()
for c in (1, 3, 4, 5):
    if c == 5:
        m = T.Model.lattice((32,))
        import numpy as np
        e = T.Ensemble(m, np.linspace(0.2, 3.0, 64), n_instances=296, seed=5)
        e.set_stream(stream.cuda_stream)
        e.generate_ea_disorder(43)
        e.init_random()
    else:
        e = WL.build(T, c, stream.cuda_stream)["ens"]
    for se, me in ((1, 0), (0, 0), (1, 1), (1, 0)):
        e.run(200, swap_every=se, measure_every=me)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        e.run(1000, swap_every=se, measure_every=me)
        b.record(stream)
        torch.cuda.synchronize()
        print(f"config {c} swap_every {se} measure_every {me}: {a.elapsed_time(b):.2f} ms / 1000 sweeps", flush=True)
