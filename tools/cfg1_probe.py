"""Config 1 (2D L=32, 32 slots): throughput vs number of seeds, K1 thread count and the
per-sweep measurement/swap epilogue."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402

stream = torch.cuda.Stream()
m = T.Model.lattice((32, 32))
for threads in ("", "128", "512"):
    if threads:
        os.environ["TAPT_K1_THREADS"] = threads
    for I in (16, 148, 296, 592):
        e = T.Ensemble(m, WL.geometric(0.2, 1.0, 32), n_instances=I, seed=1)
        e.set_stream(stream.cuda_stream)
        e.init_random()
        for se, me in ((1, 1), (1, 0), (0, 0)):
            e.run(100, swap_every=se, measure_every=me)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            e.run(2000, swap_every=se, measure_every=me)
            b.record(stream)
            torch.cuda.synchronize()
            r = I * 32 * 1024 * 2000 / (a.elapsed_time(b) * 1e-3)
            print(f"threads={threads or 'auto'} I={I} swap={se} measure={me}: {r / 1e9:.1f} G/s "
                  f"({r / I / 1e9:.2f} G/s per instance)", flush=True)
