#!/usr/bin/env python
"""IsingFormer proposal throughput on one B200.  One JSON line per case.

  sample:   tokens/s of ancestral sampling; roofline = K/V-cache bytes read
            (sum_t (t+1) x layers x (K+V) x 64 x 4 B per sequence) / kernel time vs HBM peak.
  log_prob: tokens/s of the causal forward; FLOP/s (dense 2 x 65.5k MAC per token + causal
            attention) vs the fp32 CUDA-core peak (148 SMs x 128 FMA x 2 x f_SM).

  python tools/bench_former.py [--cases mult8,lat16,mult16] [--batch B] [--kv fp32|bf16]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {  # name: (T, prefix, B)
    "mult8": (200, 24, 4096),     # 8x8 multiplier: 3n^2+n spins, product + carry-in bits as prefix
    "lat16": (256, 0, 4096),      # 2D 16x16 lattice, raster order
    "mult16": (784, 48, 4096),    # 16x16 multiplier (config 4 size; a round there proposes 512 x 31)
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="mult8,lat16,mult16")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--kv", default="fp32", choices=["fp32", "bf16"])
    args = ap.parse_args()
    import torch

    import paper_2509_23043_b200 as T
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    bf16_peak = peaks.get("bf16_tflops", peaks.get("bf16_dense_tflops", 2250.0))
    f = T.Former(seed=1, scale=1.0, max_len=1024, kv=args.kv)
    kvb = 2 if args.kv == "bf16" else 4
    L, D = f.config["layers"], f.config["d_model"]
    dense_mac = T.Former.param_count() - 2 * D - 16 * D - D  # every weight once per token (approx.)
    props = torch.cuda.get_device_properties(0)
    for name in args.cases.split(","):
        Tn, npre, B = CASES[name]
        if args.batch:
            B = args.batch
        rs = np.random.default_rng(0)
        betas = rs.uniform(0.2, 3.0, B)
        streams = rs.integers(0, 2 ** 63, B, dtype=np.uint64)
        prefix = rs.integers(0, 2, (B, npre)).astype(np.uint8) if npre else None
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        f.sample(B, Tn, betas, streams, prefix)  # warm-up at full size (grows the K/V cache outside the timing)
        torch.cuda.synchronize()
        ev[0].record()
        tok, lq = f.sample(B, Tn, betas, streams, prefix)
        ev[1].record()
        torch.cuda.synchronize()
        eng = {}
        for tc in (True, False):  # tcgen05 dense products vs the fp32 CUDA-core row engine
            f.set_tensor_cores(tc)
            f.log_prob(tok, betas, npre)
            torch.cuda.synchronize()
            ev[2].record()
            lq2 = f.log_prob(tok, betas, npre)
            ev[3].record()
            torch.cuda.synchronize()
            eng["tc" if tc else "cuda_cores"] = (ev[2].elapsed_time(ev[3]) * 1e-3, lq2)
        f.set_tensor_cores(True)
        ts, tf = ev[0].elapsed_time(ev[1]) * 1e-3, eng["tc"][0]
        lq2 = eng["tc"][1]
        kv = L * 2 * D * kvb * Tn * (Tn + 1) / 2 * B
        attn_flop = L * 2 * 2 * D * Tn * (Tn + 1) / 2 * B
        flop = 2.0 * dense_mac * Tn * B + attn_flop
        f_sm = props.clock_rate * 1e3 if hasattr(props, "clock_rate") else 1.965e9
        fp32_peak = props.multi_processor_count * 128 * 2 * 1.965e9
        print(json.dumps({
            "case": name, "T": Tn, "prefix": npre, "batch": B, "kv": args.kv,
            "sample": {"tokens_per_s": B * Tn / ts, "seconds": ts, "kv_gb": kv / 1e9,
                       "kv_gbs": kv / ts / 1e9, "hbm_frac": kv / ts / 1e9 / hbm},
            "log_prob": {"tokens_per_s": B * Tn / tf, "seconds": tf, "tflops": flop / tf / 1e12,
                         "dense_tflops": 2.0 * dense_mac * Tn * B / tf / 1e12,
                         "dense_bf16_frac": 2.0 * dense_mac * Tn * B / tf / 1e12 / bf16_peak,
                         "cuda_core_engine": {"seconds": eng["cuda_cores"][0],
                                              "tokens_per_s": B * Tn / eng["cuda_cores"][0],
                                              "max_abs_log_q_diff": float(np.max(np.abs(eng["cuda_cores"][1] - lq2)))},
                         "speedup_vs_cuda_cores": eng["cuda_cores"][0] / tf},
            "consistency_max_abs": float(np.max(np.abs(lq - lq2))),
            "peaks": {"hbm_gbs": hbm, "fp32_tflops": fp32_peak / 1e12, "f_sm_assumed": 1.965e9, "f_sm_prop": f_sm},
        }), flush=True)


if __name__ == "__main__":
    main()
