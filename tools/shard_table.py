"""Per-GPU throughput of configs 2-4 at their 1/2/4/8-GPU shard sizes (instances split evenly, one
GPU running one shard).  Config 5's table is tools/shard_sizes.sh.

  python tools/shard_table.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402

stream = torch.cuda.Stream()
total = {2: 128, 3: 256, 4: 512}
for cfg in (2, 3, 4):
    row, kern = {}, {}
    for ngpu in (1, 2, 4, 8):
        wl = WL.build(T, cfg, stream.cuda_stream, instances=total[cfg] // ngpu)
        wl["step"]()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        wl["step"]()
        b.record(stream)
        torch.cuda.synchronize()
        row[ngpu] = wl["updates_per_step"] / (a.elapsed_time(b) * 1e-3)
        kern[ngpu] = wl["ens"].launch_log()
        del wl
    print(json.dumps({"config": cfg, "instances_total": total[cfg],
                      "per_gpu_updates_per_s": {k: round(v / 1e9, 1) for k, v in row.items()},
                      "projected_aggregate_G": {k: round(k * v / 1e9, 1) for k, v in row.items()},
                      "per_gpu_efficiency_vs_1gpu": {k: round(v / row[1], 3) for k, v in row.items()},
                      "kernels": kern}), flush=True)
