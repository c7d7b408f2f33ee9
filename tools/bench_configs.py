#!/usr/bin/env python
"""Throughput of BASELINE.json configs 1-4 on one B200 (GPU only; `bench.py --workload cfgK`
adds the JSON contract fields and the reference CPU path).  One JSON line per config; the
workloads are paper_2509_23043_b200/workloads.py.

  python tools/bench_configs.py [--configs 1,2,3,4] [--steps 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2509_23043_b200 as T
    from paper_2509_23043_b200 import workloads as WL
    stream = torch.cuda.Stream()
    for c in [int(x) for x in args.configs.split(",")]:
        w = WL.build(T, c, stream.cuda_stream)
        w["step"]()  # warm-up
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(args.steps):
            w["step"]()
        b.record(stream)
        torch.cuda.synchronize()
        dt = a.elapsed_time(b) * 1e-3
        upd = w["updates_per_step"] * args.steps
        line = {"config": c, "workload": w["desc"], "kernel": w["kernel"], "seconds": dt, "updates": upd,
                "updates_per_s": upd / dt}
        if c == 4:  # coldest-slot factorisation success after the run (decode_and_check)
            M = T.Multiplier(16)
            S = w["ens"].spins()
            prods = [T.random_semiprime(4, k, 16) for k in range(w["I"])]
            line["coldest_slot_success"] = float(np.mean(
                [M.decode(S[k][w["R"] - 1], p * q)[2] for k, (p, q) in enumerate(prods)]))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
