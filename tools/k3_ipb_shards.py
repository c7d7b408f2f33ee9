"""K3 teams per CTA (TAPT_K3_IPB) x instances (config 4 shard sizes): updates/s.  python tools/k3_ipb_shards.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402

stream = torch.cuda.Stream()
for inst in (512, 256, 128, 64):
    row = {}
    for ipb in ("1", "2", "3", "4", "auto"):
        if ipb == "auto":
            os.environ.pop("TAPT_K3_IPB", None)
        else:
            os.environ["TAPT_K3_IPB"] = ipb
        wl = WL.build(T, 4, stream.cuda_stream, instances=inst)
        wl["step"]()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        wl["step"]()
        b.record(stream)
        torch.cuda.synchronize()
        row[ipb] = round(wl["updates_per_step"] / (a.elapsed_time(b) * 1e-3) / 1e9, 1)
        del wl
    print(json.dumps({"instances": inst, "G_updates_per_s_by_ipb": row}), flush=True)
