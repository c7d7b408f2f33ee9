"""Throughput of the bit-exact reference-order mode (K2 on dependency levels, the unmodified
reference gibbs_sweep's chain) at the config-1 and config-4 sizes, beside the colour-order kernels.
  python tools/reference_order_rate.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402

stream = torch.cuda.Stream()


def rate(e, upd_per_sweep, S=200):
    e.set_stream(stream.cuda_stream)
    e.run(20, swap_every=1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    e.run(S, swap_every=1)
    b.record(stream)
    torch.cuda.synchronize()
    return upd_per_sweep * S / (a.elapsed_time(b) * 1e-3)


m1 = T.Model.lattice((32, 32))
M = T.Multiplier(16)
m4 = M.model()
prods = [T.random_semiprime(4, k, 16) for k in range(512)]
cl = np.stack([M.clamps(p * q) for p, q in prods])
for order in ("colour", "reference"):
    e1 = T.Ensemble(m1, WL.geometric(0.2, 1.0, 32), n_instances=296, seed=1, order=order)
    e1.init_random()
    r1 = rate(e1, 296 * 32 * 1024)
    e4 = T.Ensemble(m4, WL.geometric(0.1, 5.0, 32), n_instances=512, seed=4, order=order)
    e4.set_clamps(cl)
    e4.init_random()
    r4 = rate(e4, 512 * 32 * m4.n_free)
    print(json.dumps({"order": order, "config1_geometry": {"kernel": e1.kernel, "G_updates_per_s": round(r1 / 1e9, 1)},
                      "config4_geometry": {"kernel": e4.kernel, "G_updates_per_s": round(r4 / 1e9, 1)}}), flush=True)
