"""K3 vs K2 on CSR workloads: config 4 (multiplier: 32 degree-32 sites among degree 6-8) and a
uniform-degree clamped 3D lattice (degree 6, one clamped plane)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402


def timed(e, stream, S=500):
    e.run(50, swap_every=1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    e.run(S, swap_every=1)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e-3


stream = torch.cuda.Stream()
L = 12
ci, cj, w = T.Model.lattice((L,)).couplings()  # the library's LatticeSpec bonds
n = L ** 3
cl = np.zeros(n, np.int8)
cl[: L * L] = 1  # z = 0 plane clamped up
ml = T.Model.graph(n, ci, cj, w, None, cl)
for k3 in ("1", "0"):
    os.environ["TAPT_K3"] = k3
    w4 = WL.build(T, 4, stream.cuda_stream)
    dt = timed(w4["ens"], stream)
    print(f"TAPT_K3={k3} config 4 ({w4['kernel']}): {512 * 32 * 736 * 500 / dt / 1e9:.1f} G updates/s", flush=True)
    e = T.Ensemble(ml, WL.geometric(0.1, 2.0, 32), n_instances=512, seed=3)
    e.set_stream(stream.cuda_stream)
    e.init_random()
    dt = timed(e, stream)
    print(f"TAPT_K3={k3} clamped 3D L={L} ({e.kernel}): {512 * 32 * ml.n_free * 500 / dt / 1e9:.1f} G updates/s",
          flush=True)
