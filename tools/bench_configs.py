#!/usr/bin/env python
"""Throughput of every BASELINE.json config on one B200 (secondary measurements; the headline
line is bench.py = config 5).  One JSON line per config.

  python tools/bench_configs.py [--configs 1,2,3,4] [--sweeps N]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def geometric(b0, b1, R):
    return b0 * (b1 / b0) ** (np.arange(R) / (R - 1.0))


def yang_m(beta):
    bc = 0.5 * np.log(1 + np.sqrt(2))
    return 0.0 if beta <= bc else (1.0 - np.sinh(2.0 * beta) ** -4) ** 0.125


def timed(torch, stream, fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--swap-every", type=int, default=1, help="configs 3/4: swap cadence (0: none; diagnostics)")
    ap.add_argument("--sweeps", type=int, default=2000)
    args = ap.parse_args()
    import torch

    import paper_2509_23043_b200 as T
    stream = torch.cuda.Stream()
    S = args.sweeps
    for c in [int(x) for x in args.configs.split(",")]:
        if c == 1:
            m = T.Model.lattice((32, 32))
            R, I, n = 32, 16, 1024
            e = T.Ensemble(m, geometric(0.2, 1.0, R), n_instances=I, seed=1)
            e.set_stream(stream.cuda_stream)
            e.init_random()
            e.run(100, swap_every=1)
            dt = timed(torch, stream, lambda: e.run(S, swap_every=1, measure_every=1, measure_from=0))
            upd = I * R * n * S
            desc = "2D ferro L=32, 32 slots geometric [0.2,1.0], 16 seeds, swap+measure every sweep"
        elif c == 2:
            m = T.Model.lattice((64, 64))
            R, I, n, T_, every = 64, 128, 4096, 60, 100
            b = geometric(0.3, 0.6, R)
            mb = np.array([yang_m(x) for x in b[:T_]])
            e = T.Ensemble(m, b, n_instances=I, seed=2)
            e.set_stream(stream.cuda_stream)
            e.init_random()

            def work():
                for _ in range(S // every):
                    e.run(every, swap_every=1, measure_every=10)
                    e.generate_proposals(np.arange(T_), mb, refine=5)
            work_warm = lambda: (e.run(every, swap_every=1), e.generate_proposals(np.arange(T_), mb, refine=5))
            work_warm()
            dt = timed(torch, stream, work)
            upd = I * (R * n * S + (S // every) * T_ * n * 5)
            desc = "2D ferro L=64, 64 slots geometric [0.3,0.6], 128 chains, TAPT every 100 sweeps into 60 slots"
        elif c == 3:
            m = T.Model.lattice((16,))
            R, I, n = 64, 256, 4096
            e = T.Ensemble(m, np.linspace(0.2, 3.0, R), n_instances=I, seed=3)
            e.set_stream(stream.cuda_stream)
            e.generate_ea_disorder(3)
            e.init_random()
            e.run(100, swap_every=1)
            dt = timed(torch, stream, lambda: e.run(S, swap_every=1))
            upd = I * R * n * S
            desc = "3D EA L=16, 64 slots linear [0.2,3.0], 256 instances, swap every sweep"
        elif c == 4:
            M = T.Multiplier(16)
            m = M.model()
            R, I = 32, 512
            e = T.Ensemble(m, geometric(0.1, 5.0, R), n_instances=I, seed=4)
            e.set_stream(stream.cuda_stream)
            prods = [T.random_semiprime(4, k, 16) for k in range(I)]
            e.set_clamps(np.stack([M.clamps(p * q) for p, q in prods]))
            e.init_random()
            e.run(100, swap_every=1)
            dt = timed(torch, stream, lambda: e.run(S, swap_every=args.swap_every))
            upd = I * R * m.n_free * S
            Sp = e.spins()
            succ = np.mean([M.decode(Sp[k][R - 1], prods[k][0] * prods[k][1])[2] for k in range(I)])
            desc = f"16x16 multiplier (784 spins, 736 free), 32 slots geometric [0.1,5.0], 512 semiprimes " \
                   f"(coldest-slot success after {S + 100} sweeps: {succ:.3f})"
        else:
            continue
        print(json.dumps({"config": c, "workload": desc, "kernel": e.kernel, "sweeps": S, "seconds": dt,
                          "updates": upd, "updates_per_s": upd / dt}), flush=True)


if __name__ == "__main__":
    main()
