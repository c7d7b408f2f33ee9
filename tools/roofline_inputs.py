#!/usr/bin/env python
"""Derive bench.py's roofline inputs from the ncu --set full summaries of the sweep kernels:

  gpurun_out/k1_summary.txt       config-5 slice (tools/profile_round.sh: 296 instances x 100 sweeps)
  gpurun_out/cfg{1,2,3}_summary.txt  tools/profile_configs.sh (one sweep launch of each config)
  gpurun_out/k3_summary.txt       tools/profile_k3.sh (one 1000-sweep launch of config 4)

-> profiles/k1_traffic.json (DRAM bytes per instance-launch, executed instructions per update and
pipe utilisation of the headline kernel) and profiles/inst_per_update.json (I_exec per config).
I_exec = 32 x smsp__inst_executed.sum / spin updates of the captured launch.

  python tools/roofline_inputs.py [--round 02]
"""
import argparse
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")

# spin updates of the captured launch: instances x slots x free sites x sweeps
UPDATES = {
    "cfg1": 296 * 32 * 1024 * 1000,
    "cfg2": 128 * 64 * 4096 * 100,   # config 2 runs 100 sweeps between TAPT rounds
    "cfg3": 256 * 64 * 4096 * 1000,
    "cfg4": 512 * 32 * 736 * 1000,
    "cfg5": 296 * 64 * 32768 * 100,
}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def parse(path):
    d, kernel = {}, None
    for l in open(path):
        m = re.match(r"kernel:\s*(.*)", l)
        if m and kernel is None:
            kernel = m.group(1).strip()
            continue
        m = re.match(r"\s+(\S+)\s+([0-9.,]+)\s*(\S*)", l)
        if m and m.group(1) not in d:
            d[m.group(1)] = (float(m.group(2).replace(",", "")), m.group(3))
    return kernel, d


def pct(d, k):
    return round(d[k][0] / 100.0, 3) if k in d else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="02")
    a = ap.parse_args()
    r = f"r{a.round}"
    files = {"cfg5": ("k1_summary.txt", f"{r}_k1_ncu_full_summary.txt"),
             "cfg1": ("cfg1_summary.txt", f"{r}_cfg1_k1_ncu_summary.txt"),
             "cfg2": ("cfg2_summary.txt", f"{r}_cfg2_k1_ncu_summary.txt"),
             "cfg3": ("cfg3_summary.txt", f"{r}_cfg3_k1_ncu_summary.txt"),
             "cfg4": ("k3_summary.txt", f"{r}_k3_ncu_full_summary.txt")}
    ipath = os.path.join(P, "inst_per_update.json")
    ipu = json.load(open(ipath))
    for cfg, (src, dst) in files.items():
        p = os.path.join(G, src)
        if not os.path.exists(p):
            print("missing", p)
            continue
        kernel, d = parse(p)
        if "smsp__inst_executed.sum" not in d:
            print("no kernel in", p)
            continue
        ie = 32.0 * d["smsp__inst_executed.sum"][0] / UPDATES[cfg]
        pipes = {"issue_active": pct(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 "alu": pct(d, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                 "fma": pct(d, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                 "fmaheavy": pct(d, "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                 "lsu": pct(d, "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
                 "warps_active": pct(d, "sm__warps_active.avg.pct_of_peak_sustained_active")}
        ipu[cfg] = {"I_exec": round(ie, 3), "kernel": kernel, "source": f"profiles/{dst}",
                    "launch": f"{int(d['launch__grid_size'][0])} CTAs x {int(d['launch__block_size'][0])} threads, "
                              f"{int(d['launch__registers_per_thread'][0])} registers",
                    "pipes": pipes}
        print(cfg, kernel, "I_exec", round(ie, 2), pipes)
        if cfg == "cfg5":
            rd = d["dram__bytes_read.sum"][0] * UNIT[d["dram__bytes_read.sum"][1]]
            wr = d["dram__bytes_write.sum"][0] * UNIT[d["dram__bytes_write.sum"][1]]
            tr = {"dram_bytes_per_instance_launch": round((rd + wr) / 296.0, 1),
                  "source": f"profiles/{dst} (ncu --set full, 296 instances x 100 sweeps, dram__bytes_read.sum + "
                            "dram__bytes_write.sum / instances; per-launch traffic is independent of the sweep "
                            "count: the state is shared-memory resident)",
                  "thread_inst_per_update": round(ie, 3),
                  "inst_source": f"same capture (round {int(a.round)}): 32 x smsp__inst_executed.sum / (296 instances "
                                 "x 64 slots x 32768 sites x 100 sweeps)",
                  "kernel": kernel,
                  "pipes": pipes}
            json.dump(tr, open(os.path.join(P, "k1_traffic.json"), "w"), indent=1)
    json.dump(ipu, open(ipath, "w"), indent=1)


if __name__ == "__main__":
    main()
