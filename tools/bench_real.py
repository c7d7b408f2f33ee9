#!/usr/bin/env python
"""K5 throughput (real-valued couplings, real.cu) beside the reference CPU path on the same graphs.

Workload: 3D EA lattice L=16 periodic (4096 spins) with Gaussian couplings N(0,1) (SPEC.md:511's
Gaussian option) and Gaussian fields, 64 slots beta linear [0.2, 3.0], colour order and the
reference's index order, swap every sweep.  One JSON line per order.

  python tools/bench_real.py [--instances 256] [--sweeps 200]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=256)
    ap.add_argument("--sweeps", type=int, default=200)
    args = ap.parse_args()
    import torch

    import paper_2509_23043_b200 as T
    from oracle import oracle as O
    L, R, I, S = 16, 64, args.instances, args.sweeps
    n, ci, cj, _ = O.lattice_couplings((L,), 1.0, True)
    rs = np.random.default_rng(5)
    J, h = rs.normal(size=len(ci)), rs.normal(size=n) * 0.3
    m = T.Model.graph(n, ci, cj, J, h)
    betas = np.linspace(0.2, 3.0, R)
    for order in ("colour", "reference"):
        e = T.Ensemble(m, betas, n_instances=I, seed=3, order=order)
        e.init_random()
        e.run(5, swap_every=1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e.run(S, swap_every=1)
        e.synchronize()
        dt = time.perf_counter() - t0
        ties, replays = e.near_ties()
        line = {"what": "K5 real-valued couplings", "order": order, "instances": I, "slots": R, "spins": n,
                "sweeps": S, "updates_per_s": I * R * n * S / dt, "seconds": dt, "near_ties": ties,
                "replays": replays, "kernel": e.launch_log()}
        if order == "reference" and O.have_ref():  # the reference CPU path on the same graph
            g = O.Graph.from_couplings(n, ci, cj, J, h)
            k = min(16, os.cpu_count() or 1)
            hs = [O.ref_graph(g) for _ in range(k)]
            arr = (C.c_void_p * k)(*hs)
            b = np.ascontiguousarray(betas)
            mb = np.zeros(R)
            t0 = time.perf_counter()
            O.ref().ref_pt_run(arr, k, 0, R, b.ctypes.data_as(O._f64p), 3, 20, 1, 0, 0, mb.ctypes.data_as(O._f64p),
                               0, k, None, None, None, None)
            dc = time.perf_counter() - t0
            for hh in hs:
                O.ref().ref_graph_free(hh)
            line["cpu_reference"] = {"updates_per_s": k * R * n * 20 / dc, "threads": k,
                                     "sample": f"{k} instances x 20 sweeps"}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
