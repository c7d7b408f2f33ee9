"""K3 lanes per site (TAPT_K3_Q = 1 / 2 / 4, split sites) x instances (config 4 shard sizes and a
few in between): G updates/s of one config-4 step.  python tools/k3_q_shards.py [instances,...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402

stream = torch.cuda.Stream()
counts = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [512, 296, 256, 148, 128, 96, 64, 32]
for inst in counts:
    row = {}
    for q in ("1", "2", "4", "auto"):
        if q == "auto":
            os.environ.pop("TAPT_K3_Q", None)
        else:
            os.environ["TAPT_K3_Q"] = q
        wl = WL.build(T, 4, stream.cuda_stream, instances=inst)
        wl["step"]()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        wl["step"]()
        b.record(stream)
        torch.cuda.synchronize()
        row[q] = {"G": round(wl["updates_per_step"] / (a.elapsed_time(b) * 1e-3) / 1e9, 1),
                  "kernel": wl["ens"].launch_log()}
        del wl
    print(json.dumps({"instances": inst, "by_q": row}), flush=True)
