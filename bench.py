#!/usr/bin/env python
"""bench.py -- spin updates/s of the TAPT verifier (PT + TAPT sweeps) on 1..8 B200s.

Workload (BASELINE.json configs[4], the scaling run the metric is quoted on): 3D
Edwards-Anderson +-1 spin glass, L=32 periodic (32768 spins), 64 slots with beta linear in
[0.2, 3.0], 4096 disorder instances sharded over the ranks (contiguous blocks of global
instance ids; RNG streams keyed by global id, so results do not depend on N), multi-replica
bit-packed spins.  One step = one TAPT round (synthetic i.i.d. +-1 proposals into the 56
hottest slots + 5 refinement sweeps at the target beta + Metropolis, Eq. 2) followed by 1000
checkerboard sweeps with a swap pass after every sweep and energy/|m| accumulation plus
per-beta energy histograms every 10 sweeps.  Per-beta histograms are reduced with NCCL at the
end of the timed region.

A spin update = one heat-bath decision for one free spin of one replica (refinement sweeps
count, i.i.d. proposal generation does not) -- BASELINE.md.

  python bench.py [--gpus N --steps K --warmup W]              # this framework (one JSON line)
  python bench.py --impl reference [--steps K --warmup W]      # the reference's CPU path
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L, R = 32, 64
N_SPINS = L ** 3
BETA_MIN, BETA_MAX = 0.2, 3.0
N_TARGETS, REFINE = 56, 5
SEED, DISORDER_SEED = 20250923, 43
I_U = 42  # algorithmic integer instructions per update for cfg3/cfg5
METRIC = "spin updates/sec for PT+TAPT sweeps at 1/2/4/8 B200; % of HBM/ALU roofline"
UNIT = "spin updates/s"


def betas():
    return np.linspace(BETA_MIN, BETA_MAX, R)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "real"],
                    help="BASELINE.json config (default cfg5, the headline); cfg1-4 run on one GPU with the "
                         "reference CPU path timed beside them at SURVEY.md 8(d)'s sub-budgets; real: K5 on a "
                         "Gaussian-coupling 3D lattice (no BASELINE config uses real couplings)")
    ap.add_argument("--instances", type=int, default=4096)
    ap.add_argument("--sweeps-per-step", type=int, default=1000)
    ap.add_argument("--measure-every", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-instances", type=int, default=16)
    ap.add_argument("--cpu-sample-sweeps", type=int, default=100)
    return ap.parse_args()


# ----------------------------------------------------------------- clocks ----

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, dev):
        self.dev, self.rows, self.proc = dev, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].strip() == "Active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "power_w_max": max(pw) if pw else None, "samples": len(self.rows)}


# ------------------------------------------------------------ CPU baseline ---

def ea_couplings_numpy(seed, gid, L=L):
    """EA +-1 bonds of DESIGN.md 3.4 (coin per (+x,+y,+z) bond in site order from
    derive(seed, {0x88, gid})), vectorised restatement for building reference graphs."""
    from oracle import oracle as O
    N_SPINS = L ** 3
    s0 = np.uint64(O.derive(seed, [0x88, gid]))
    k = np.arange(1, 3 * N_SPINS + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = s0 + k * np.uint64(O.PHI)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    J = np.where((z >> np.uint64(63)) != 0, 1.0, -1.0)
    i = np.arange(N_SPINS)
    x, y, zz = i % L, (i // L) % L, i // (L * L)
    nb = np.stack([((x + 1) % L) + L * (y + L * zz), x + L * (((y + 1) % L) + L * zz),
                   x + L * (y + L * ((zz + 1) % L))], axis=1)
    ci = np.repeat(i, 3).astype(np.uint32)
    cj = nb.reshape(-1).astype(np.uint32)
    return ci, cj, J


def cpu_reference_rate(n_inst, n_sweeps, threads, prop_every):
    """Reference gibbs_sweep (oracle/_ref, unmodified sources) inside the restated PT/TAPT
    schedule, parallel_for over instances.  Falls back to the oracle C port (1 thread)."""
    import ctypes as C

    from oracle import oracle as O
    b = np.ascontiguousarray(betas())
    mb = np.zeros(R)
    if O.have_ref():
        Rf = O.ref()
        hs = []
        for k in range(n_inst):
            ci, cj, J = ea_couplings_numpy(DISORDER_SEED, k)
            hs.append(Rf.ref_graph_build(N_SPINS, len(ci), ci.ctypes.data_as(O._u32p), cj.ctypes.data_as(O._u32p),
                                         J.ctypes.data_as(O._f64p), None, None))
        arr = (C.c_void_p * n_inst)(*hs)
        t0 = time.perf_counter()
        Rf.ref_pt_run(arr, n_inst, 0, R, b.ctypes.data_as(O._f64p), SEED, n_sweeps, 1, prop_every, N_TARGETS,
                      mb.ctypes.data_as(O._f64p), REFINE, threads, None, None, None, None)
        dt = time.perf_counter() - t0
        for h in hs:
            Rf.ref_graph_free(h)
        kind, cores = "reference", threads
    else:
        g = O.Graph.from_couplings(N_SPINS, *ea_couplings_numpy(DISORDER_SEED, 0))
        t0 = time.perf_counter()
        for k in range(n_inst):
            pt = O.PT(g, b, SEED, k, g.index_order())
            pt.run(n_sweeps, 1, prop_every, N_TARGETS, mb, REFINE)
        dt = time.perf_counter() - t0
        kind, cores = "port", 1
    rounds = n_sweeps // prop_every if prop_every else 0
    updates = n_inst * (R * N_SPINS * n_sweeps + rounds * N_TARGETS * N_SPINS * REFINE)
    return updates / dt, dt, kind, cores, updates


def cpu_workload_rate(k, threads):
    """The reference CPU path (unmodified gibbs_sweep in index order + the restated PT/TAPT driver,
    oracle/_ref, parallel_for over instances) on SURVEY.md 8(d)'s sub-budget of config k:
    cfg1 the full run of one seed, cfg2 16 chains x 10^3 sweeps, cfg3 32 instances x 10^3,
    cfg4 64 instances x 10^3.  Returns (updates/s, seconds, threads used, sample)."""
    import ctypes as C

    import paper_2509_23043_b200 as T
    from paper_2509_23043_b200 import workloads as WL
    from oracle import oracle as O
    Rf = O.ref()
    hs, props = [], (0, 0, None, 0)
    if k == 1:
        hs = [Rf.ref_graph_lattice(2, 32, 32, 0, 1.0, 1)]
        betas_, sweeps, n_free = WL.geometric(0.2, 1.0, 32), 10000, 1024
    elif k == 2:
        hs = [Rf.ref_graph_lattice(2, 64, 64, 0, 1.0, 1) for _ in range(16)]
        betas_, sweeps, n_free = WL.geometric(0.3, 0.6, 64), 1000, 4096
        mb = np.zeros(64)
        mb[:60] = [WL.yang_m(x) for x in betas_[:60]]
        props = (100, 60, mb, 5)
    elif k == 3:
        for g in range(32):
            ci, cj, J = ea_couplings_numpy(3, g, 16)
            hs.append(Rf.ref_graph_build(4096, len(ci), ci.ctypes.data_as(O._u32p), cj.ctypes.data_as(O._u32p),
                                         J.ctypes.data_as(O._f64p), None, None))
        betas_, sweeps, n_free = np.linspace(0.2, 3.0, 64), 1000, 4096
    else:
        M = T.Multiplier(16)
        ci, cj = np.ascontiguousarray(M.ci, np.uint32), np.ascontiguousarray(M.cj, np.uint32)
        J, h = np.ascontiguousarray(M.J, np.float64), np.ascontiguousarray(M.h, np.float64)
        for g in range(64):
            p, q = T.random_semiprime(4, g, 16)
            cl = np.ascontiguousarray(M.clamps(p * q), np.int8)
            hs.append(Rf.ref_graph_build(M.n_spins, len(ci), ci.ctypes.data_as(O._u32p), cj.ctypes.data_as(O._u32p),
                                         J.ctypes.data_as(O._f64p), h.ctypes.data_as(O._f64p),
                                         cl.ctypes.data_as(O._i8p)))
        betas_, sweeps, n_free = WL.geometric(0.1, 5.0, 32), 1000, M.model().n_free
    b = np.ascontiguousarray(betas_, np.float64)
    R_, n_inst = len(b), len(hs)
    every, nt, mb, refine = props
    mbp = np.ascontiguousarray(mb if mb is not None else np.zeros(R_), np.float64)
    arr = (C.c_void_p * n_inst)(*hs)
    t0 = time.perf_counter()
    Rf.ref_pt_run(arr, n_inst, 0, R_, b.ctypes.data_as(O._f64p), SEED, sweeps, 1, every, nt,
                  mbp.ctypes.data_as(O._f64p), refine, threads, None, None, None, None)
    dt = time.perf_counter() - t0
    for hnd in hs:
        Rf.ref_graph_free(hnd)
    rounds = sweeps // every if every else 0
    upd = n_inst * (R_ * n_free * sweeps + rounds * nt * n_free * refine)
    used = min(threads, n_inst)
    sample = f"{n_inst} instance(s) x {sweeps} sweeps of config {k}, {used} thread(s) on '{cpu_model()}'"
    return upd / dt, dt, used, sample


def run_workload(args):
    """bench.py --workload cfg1..cfg4: one GPU, same JSON schema as the headline line."""
    import torch

    import paper_2509_23043_b200 as T
    from paper_2509_23043_b200 import workloads as WL
    k = int(args.workload[3:])
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        raise SystemExit("--workload cfg1..cfg4 runs on one GPU (config 5 is the sharded run)")
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    w = WL.build(T, k, stream.cuda_stream)
    for _ in range(args.warmup):
        w["step"]()
    torch.cuda.synchronize()
    l0 = T.launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with ClockSampler(0) as clk:
        ev[0].record(stream)
        for _ in range(args.steps):
            w["step"]()
        ev[1].record(stream)
        torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    value = w["updates_per_step"] * args.steps / (ms * 1e-3)
    clocks = clk.summary()
    f_sm = (clocks.get("sm_mhz") or 1965.0) * 1e6
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    probe, _ = T.probe_decision_rate(1, 512, 20000)
    ipath = os.path.join(ROOT, "profiles", "inst_per_update.json")
    ie = json.load(open(ipath)).get(f"cfg{k}") if os.path.exists(ipath) else None
    cap = n_sm * 128 * f_sm
    alg = cap / WL.I_U[k]
    roof = {"unit": "Gupdates/s", "achieved": value / 1e9,
            "algorithmic": {"I_u": WL.I_U[k], "peak": alg / 1e9, "frac": value / alg,
                            "what": "SURVEY.md 8(d) estimate of instructions per update (not a bound)"},
            "probe_ceiling": {"value": probe / 1e9, "frac": value / probe}, "traffic": None}
    if ie:
        roof.update({"bound": "issue", "peak": cap / ie["I_exec"] / 1e9, "frac": value * ie["I_exec"] / cap,
                     "peak_source": f"n_SM*128*f_SM/I_exec, I_exec={ie['I_exec']} executed thread-instructions per "
                                    f"update ({ie['source']})"})
    else:
        roof.update({"bound": "alu", "peak": alg / 1e9, "frac": value / alg,
                     "peak_source": f"SURVEY.md 8(d) n_SM*128*f_SM/I_u, I_u={WL.I_U[k]}"})
    out = {
        "metric": f"spin updates/sec, BASELINE config {k}", "value": value, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "replicas only", "vs_baseline": None, "dtype": "u32 multi-spin words / u64 splitmix64",
        "data": "synthetic", "config": {"workload": w["desc"], "kernel": w["kernel"],
                                        "updates_per_step": w["updates_per_step"]},
        "roofline": roof,
        "gpu_launches": T.launch_count() - l0, "clocks": clocks,
    }
    if k == 1:  # BASELINE config 1 itself is ONE instance: its whole 10^4-sweep run, on the device
        e1 = T.Ensemble(T.Model.lattice((32, 32)), WL.geometric(0.2, 1.0, 32), n_instances=1, seed=1)
        e1.set_stream(stream.cuda_stream)
        e1.init_random()
        e1.run(100, swap_every=1, measure_every=1)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e1.run(10000, swap_every=1, measure_every=1, measure_from=5000)
        b.record(stream)
        torch.cuda.synchronize()
        ms1 = a.elapsed_time(b)
        out["single_instance"] = {
            "what": "BASELINE configs[0] as specified: 1 instance x 32 slots x 10^4 sweeps (swap every sweep, "
                    "observables over the last half); the headline line above fills the GPU with 296 "
                    "independent seeds of the same run (replicas only)",
            "seconds": ms1 / 1e3, "value": 32 * 1024 * 10000 / (ms1 * 1e-3), "unit": UNIT,
            "kernel": e1.launch_log()}
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, dt, used, sample = cpu_workload_rate(k, threads)
        out["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": used, "kind": "reference",
                               "sample": f"{sample} ({dt:.1f} s)"}
    print(json.dumps(out), flush=True)


def run_real(args):
    """bench.py --workload real: K5 (real-valued couplings) on a 3D lattice L=16 periodic with Gaussian
    couplings N(0,1) (SPEC.md:511's Gaussian option) and fields N(0, 0.3^2), 64 slots beta linear
    [0.2, 3.0], 256 instances, the reference's index order (bit-exact with its gibbs_sweep), swap every
    sweep; one step = 100 sweeps.  The reference CPU path (oracle/_ref: the unmodified gibbs_sweep in the
    restated PT driver) runs beside it on the same graph."""
    import ctypes as C

    import torch

    import paper_2509_23043_b200 as T
    L, R, I, S = 16, 64, 256, 100
    n = L ** 3
    ci, cj, _ = T.Model.lattice((L,)).couplings()
    rs = np.random.default_rng(5)
    J, h = rs.normal(size=len(ci)), rs.normal(size=n) * 0.3
    m = T.Model.graph(n, ci, cj, J, h)
    b = np.linspace(0.2, 3.0, R)
    torch.cuda.set_device(0)
    e = T.Ensemble(m, b, n_instances=I, seed=3, order="reference")
    e.init_random()
    for _ in range(args.warmup):
        e.run(S // 10, swap_every=1)
    e.synchronize()
    l0 = T.launch_count()
    with ClockSampler(0) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e.run(S, swap_every=1)
        e.synchronize()
        dt = time.perf_counter() - t0
    ties, replays = e.near_ties()
    value = I * R * n * S * args.steps / dt
    out = {"metric": "spin updates/sec, real-valued couplings (K5)", "value": value, "unit": UNIT, "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "replicas only", "vs_baseline": None,
           "dtype": "f64 local fields / u64 splitmix64", "data": "synthetic",
           "config": {"workload": "3D lattice L=16, Gaussian J and h, 64 slots, 256 instances, reference index "
                                  "order, swap every sweep, 100 sweeps per step", "near_ties": ties,
                      "replays": replays, "kernel": e.launch_log()},
           "gpu_launches": T.launch_count() - l0, "clocks": clk.summary()}
    if not args.no_cpu_baseline:
        from oracle import oracle as O  # the reference CPU path (cpu_baseline leg)
        if not O.have_ref():
            raise SystemExit("--workload real: oracle/_ref is not built (run __graft_entry__.build())")
        k = min(16, os.cpu_count() or 1)
        g = O.Graph.from_couplings(n, ci, cj, J, h)
        hs = [O.ref_graph(g) for _ in range(k)]
        arr = (C.c_void_p * k)(*hs)
        bb, mb = np.ascontiguousarray(b), np.zeros(R)
        t0 = time.perf_counter()
        O.ref().ref_pt_run(arr, k, 0, R, bb.ctypes.data_as(O._f64p), 3, 2000, 1, 0, 0, mb.ctypes.data_as(O._f64p), 0,
                           k, None, None, None, None)
        dc = time.perf_counter() - t0
        for hh in hs:
            O.ref().ref_graph_free(hh)
        out["cpu_baseline"] = {"value": k * R * n * 2000 / dc, "unit": UNIT, "cores": k, "kind": "reference",
                               "sample": f"{k} instances x 2000 sweeps of the same graph ({dc:.1f} s, '{cpu_model()}')"}
    print(json.dumps(out), flush=True)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_inst = max(args.cpu_sample_instances, threads)
    sweeps, every = args.cpu_sample_sweeps, args.cpu_sample_sweeps // 2
    for _ in range(args.warmup):
        cpu_reference_rate(n_inst, sweeps, threads, every)
    tot_u, tot_t, kind, cores = 0, 0.0, "reference", threads
    for _ in range(args.steps):
        rate, dt, kind, cores, u = cpu_reference_rate(n_inst, sweeps, threads, every)
        tot_u += u
        tot_t += dt
    v = tot_u / tot_t
    sample = (f"{n_inst} instances x {sweeps} sweeps of the config-5 geometry (EA L=32, 64 slots), TAPT round "
              f"every {every} sweeps, per step; {cores} threads on '{cpu_model()}' (nproc={threads})")
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 RNG / f64 exp (reference CPU)", "data": "synthetic",
        "config": {"workload": "BASELINE configs[4]: 3D EA +-J L=32, 64 slots, beta linear [0.2,3.0], TAPT",
                   "sample": sample},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------- multi-GPU --

def launcher_cmd(argv, gpus, port=None):
    """The torchrun command that re-executes this script with one rank per GPU (used when
    `--gpus N` > 1 is given without a torch.distributed environment)."""
    if port is None:
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


def check_world(args):
    """--gpus N must equal the launcher's world size; without a launcher, N > 1 spawns the ranks."""
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0:
        if args.gpus > 1:
            cmd = launcher_cmd(sys.argv[1:], args.gpus)
            os.execv(cmd[0], cmd)  # does not return
        return 1
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch one rank per GPU)")
    return world


def init_dist(world, local, backend="nccl"):
    import torch
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return dist


def share_unique_id(make_uid, rank):
    """Rank 0 makes the NCCL unique id (128 bytes); every rank receives it (torch.distributed
    broadcast -- the plumbing; the reduction itself is the library's NCCL call)."""
    import torch.distributed as dist
    obj = [make_uid() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def reduce_observables(T, ens, comm):
    """The run's collectives: per-beta energy histograms, per-slot observables and the
    best energy over every rank's instances -- tapt_allreduce_observables, NCCL over NVLink on the
    ensemble's stream (one process per GPU); rank-local at N = 1."""
    if comm is None:
        return {"hist": ens.histogram(), "obs": None, "best": int(ens.best().min())}
    return T.allreduce_observables(ens, comm)


def max_over_ranks(ms, world, device):
    """(max over ranks of a timed-region length, ranks in the communicator)."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        return float(ms), 1
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), dist.get_world_size()


# ---------------------------------------------------------------- roofline --

def issue_roofline(achieved, n_sm, f_sm, probe, n_inst, hbm_bytes, k_ms, g_hbm, path=None):
    """Roofline of the dominant kernel (K1, config 5).  Every spin update is shared-memory resident
    integer work, so the bound is the SMs' instruction issue: n_SM x 128 thread-instructions/clk x
    f_SM divided by the instructions the kernel executes per update (I_exec, from the committed ncu
    --set full capture of the same kernel: smsp__inst_executed x 32 / updates).  frac is therefore
    the share of issue slots the kernel fills (<= 1).  Secondary figures: SURVEY.md 8(d)'s
    algorithmic bound (I_u = 42 estimated instructions per update), the measured decision-probe
    ceiling, the ncu pipe utilisations, and HBM."""
    path = path or os.path.join(ROOT, "profiles", "k1_traffic.json")
    tr = json.load(open(path)) if os.path.exists(path) else {}
    ipu = tr.get("thread_inst_per_update")
    cap = n_sm * 128 * f_sm  # thread-instructions per second
    alg = cap / I_U
    out = {"unit": "Gupdates/s", "achieved": achieved / 1e9,
           "algorithmic": {"I_u": I_U, "peak": alg / 1e9, "frac": achieved / alg,
                           "what": "SURVEY.md 8(d) estimate (splitmix64 draw + threshold compare ~28, stencil ~14); "
                                   "the compiled kernel executes fewer, so this is not a bound"},
           "probe_ceiling": {"value": probe / 1e9, "frac": achieved / probe,
                             "what": "k_decision_probe: the bare per-update work (splitmix64 high word + threshold "
                                     "lookup + compare + bit insert), no stencil or memory traffic, same unroll"},
           "hbm": {"achieved_gbs": hbm_bytes / (k_ms * 1e-3) / 1e9, "peak_gbs": g_hbm,
                   "frac": hbm_bytes / (k_ms * 1e-3) / 1e9 / g_hbm,
                   "note": "spins stay in shared memory for the whole 1000-sweep launch"}}
    if ipu:
        peak = cap / ipu
        out.update({"bound": "issue", "peak": peak / 1e9, "frac": achieved / peak,
                    "peak_source": f"n_SM*128*f_SM/I_exec: n_SM={n_sm}, f_SM = median SM clock sampled during the "
                                   f"timed region ({f_sm / 1e6:.0f} MHz), I_exec={ipu:.2f} executed thread-"
                                   f"instructions per update ({tr.get('inst_source')})",
                    "traffic": tr["dram_bytes_per_instance_launch"] * n_inst,
                    "traffic_detail": {"dram_bytes_per_launch": tr["dram_bytes_per_instance_launch"] * n_inst,
                                       "algorithmic_bytes_per_launch": hbm_bytes, "source": tr["source"]},
                    "pipes": tr.get("pipes")})
    else:  # no committed capture: fall back to the algorithmic estimate
        out.update({"bound": "alu", "peak": alg / 1e9, "frac": achieved / alg, "traffic": None,
                    "peak_source": f"SURVEY.md 8(d) n_SM*128*f_SM/I_u, I_u={I_U} (no committed ncu capture)"})
    return out


# ------------------------------------------------------------------ B200 arm --

def main():
    args = parse()
    world_checked = check_world(args)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.workload == "real":
        run_real(args)
        return
    if args.workload != "cfg5":
        run_workload(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2509_23043_b200 as T

    world = world_checked
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    T.set_device(local)  # the library's own (static) CUDA runtime, explicitly on this rank's GPU
    init_dist(world, local)
    comm = T.NcclComm(share_unique_id(T.NcclComm.unique_id, rank), world, rank) if world > 1 else None
    from paper_2509_23043_b200 import sharding
    off, I = sharding.shard(args.instances, world, rank)  # contiguous global instance ids
    S = args.sweeps_per_step

    model = T.Model.lattice((L,))
    ens = T.Ensemble(model, betas(), n_instances=I, seed=SEED, instance_offset=off)
    stream = torch.cuda.Stream()
    ens.set_stream(stream.cuda_stream)
    ens.generate_ea_disorder(DISORDER_SEED)
    ens.init_random()
    nb = 2 * 3 * N_SPINS // 64
    ens.set_histogram(-3 * N_SPINS, 64, nb)
    targets = np.arange(N_TARGETS, dtype=np.uint32)

    k_ev = []

    def step(timed):
        ens.generate_proposals(targets, None, REFINE, return_accepted=False)
        if timed:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        ens.run(S, swap_every=1, measure_every=args.measure_every)
        if timed:
            b.record(stream)
            k_ev.append((a, b))

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = T.launch_count()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for _ in range(args.steps):
            step(True)
        red = reduce_observables(T, ens, comm)  # inside the timed region
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = T.launch_count() - l0
    ms = t_start.elapsed_time(t_end)
    ms, comm_ranks = max_over_ranks(ms, world, "cuda")
    samples = int(np.asarray(red["hist"]).sum())
    upd_step = args.instances * (R * N_SPINS * S + N_TARGETS * N_SPINS * REFINE)
    value = upd_step * args.steps / (ms * 1e-3)

    # roofline of the dominant kernel (K1, one launch per step, measured on its stream)
    k_ms = float(np.mean([a.elapsed_time(b) for a, b in k_ev]))
    k_upd = I * R * N_SPINS * S
    achieved = k_upd / (k_ms * 1e-3)
    probe, _ = T.probe_decision_rate(1, 512, 20000)
    clocks = clk.summary()
    f_sm = (clocks.get("sm_mhz") or 1965.0) * 1e6
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    g_hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs") if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    hbm_bytes = I * (2 * 4 * N_SPINS * 2 + N_SPINS)  # spins in+out (2 groups) + bond bytes, per launch
    roofline = issue_roofline(achieved, n_sm, f_sm, probe, I, hbm_bytes, k_ms, g_hbm)
    sweep_kernels = [x for x in ens.launch_log() if x.startswith("k1_lattice_pt<3,1,1,")]
    roofline.update({"kernel": sweep_kernels[-1] if sweep_kernels else None, "kernel_ms_per_launch": k_ms,
                     "updates_per_launch": k_upd})
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32 multi-spin words / u64 splitmix64", "data": "synthetic",
        "config": {"workload": "BASELINE configs[4]: 3D EA +-J L=32 periodic, 64 slots beta linear [0.2,3.0], "
                               "4096 instances sharded, TAPT round (56 targets, 5 refine sweeps) + 1000 sweeps "
                               "(swap every sweep, measure every 10) per step",
                   "instances_total": args.instances, "instances_per_gpu": I, "sweeps_per_step": S,
                   "updates_per_step": upd_step, "parallelism": f"instances sharded over {world} GPU(s)",
                   "l2": "state 1 GiB/GPU at N=1 > 126 MB L2; spins are shared-memory resident within a launch",
                   "histogram_samples_reduced": samples},
        "comm": {"backend": "nccl (tapt_allreduce_observables)" if world > 1 else None, "ranks": comm_ranks,
                 "nccl_ranks": comm.size() if comm is not None else 1,
                 "collectives": "all_reduce of the per-beta histograms (u64 [64][3072]), per-slot observables and "
                                "best energy (library NCCL call) + max of the timed region"},
        "roofline": roofline, "gpu_launches": launches,
    }
    if not args.no_e2e:
        out["e2e"] = e2e_leg(args, T, torch, ens, stream, I, S, world, comm)
    out["clocks"] = clocks
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        n_inst = max(args.cpu_sample_instances, threads)
        # about 10-30 s of CPU work: three times the reference arm's per-step sample
        cs = 3 * args.cpu_sample_sweeps
        rate, dt, kind, cores, _ = cpu_reference_rate(n_inst, cs, threads, cs // 2)
        out["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                               "sample": f"{n_inst} instances x {cs} sweeps of the config-5 "
                                         f"geometry with a TAPT round every {cs // 2} sweeps "
                                         f"({dt:.1f} s, '{cpu_model()}')"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_leg(args, T, torch, ens, stream, I, S, world, comm):
    """Same metric and the same step through the public C-ABI calls with HOST buffers: per step the
    externally supplied proposals (the generator's output: bit-packed [I][56][4096 B] in pinned host
    memory) are copied H2D inside the timed region and injected with their 5 refinement sweeps at the
    target beta + Eq. 2 (tapt_inject_proposals_packed_refined), 1000 PT sweeps run with measurement
    every 10 sweeps, and the step's outputs -- the per-beta energy histograms (config 5's output) and
    the per-slot energies -- are read back D2H (histograms all-reduced over the ranks first)."""
    nbytes = (N_SPINS + 7) // 8
    rs = np.random.default_rng(7)
    host = torch.from_numpy(rs.integers(0, 256, size=(I, N_TARGETS, nbytes), dtype=np.uint8)).pin_memory()
    dev = torch.empty_like(host, device="cuda")
    nb = 2 * 3 * N_SPINS // 64
    energies = torch.empty((I, R), dtype=torch.int64).pin_memory()
    targets = np.arange(N_TARGETS, dtype=np.uint32)

    def step():
        with torch.cuda.stream(stream):
            dev.copy_(host, non_blocking=True)
        ens.inject_proposals_packed(None, targets, device_ptr=dev.data_ptr(), refine=REFINE, return_accepted=False)
        ens.run(S, swap_every=1, measure_every=args.measure_every)
        reduce_observables(T, ens, comm)  # per-beta histograms to the host (all-reduced over the ranks)
        energies.copy_(torch.from_numpy(ens.energies()))

    step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    dt, _ = max_over_ranks(dt, world, "cuda")
    upd = args.instances * (R * N_SPINS * S + N_TARGETS * N_SPINS * REFINE) * args.steps
    return {"value": upd / dt, "unit": UNIT, "h2d_bytes_per_step": int(host.numel()),
            "d2h_bytes_per_step": int(R * nb * 8 + I * R * 8 + (R * 5 * 8 + 8 if comm is not None else I * 8)),
            "path": "tapt_inject_proposals_packed_refined (host-supplied proposals, 5 refinement sweeps, Eq. 2) + "
                    "tapt_run + tapt_get_histogram / tapt_allreduce_observables (NCCL at N > 1) + "
                    "tapt_ensemble_get_energies",
            "timer": "host wall clock around K steps, synchronized on both sides, max over ranks"}


if __name__ == "__main__":
    main()
