"""K1 replica-group width at the 8-GPU shard sizes of configs 2 and 3 (16 chains / 32 instances per
GPU): updates/s with 32-, 16- and 8-replica groups and with the automatic choice.

  python tools/narrow_groups.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402

stream = torch.cuda.Stream()
for cfg, inst in ((3, 32), (2, 16), (3, 64), (3, 256)):
    for w in ("32", "16", "8", "auto"):
        if w == "auto":
            os.environ.pop("TAPT_K1_W", None)
        else:
            os.environ["TAPT_K1_W"] = w
        wl = WL.build(T, cfg, stream.cuda_stream, instances=inst)
        wl["step"]()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        wl["step"]()
        b.record(stream)
        torch.cuda.synchronize()
        dt = a.elapsed_time(b) * 1e-3
        print(json.dumps({"config": cfg, "instances": inst, "W": w, "updates_per_s": wl["updates_per_step"] / dt}),
              flush=True)
        del wl
