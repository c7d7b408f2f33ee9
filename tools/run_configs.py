#!/usr/bin/env python
"""Full-length runs of the BASELINE.json configs with each config's own output:

  cfg1  2D ferro L=32, 32 slots, 10^4 sweeps, 16 seeds: per-beta <E>/N and <|m|> over the last half
  cfg2  2D ferro L=64, 64 slots, 2x10^4 sweeps, 128 chains, TAPT every 100 sweeps into 60 slots:
        per-beta <E>/N, <|m|>, proposal acceptance per slot
  cfg3  3D EA L=16, 64 slots, 10^5 sweeps, 256 instances: residual energy vs sweeps
  cfg4  16x16 multiplier, 32 slots, 10^5 sweeps, 512 semiprimes: factorisation success vs sweeps
  cfg5  3D EA L=32, 64 slots, 10^4 sweeps, 4096 instances, TAPT every 1000 sweeps into 56 slots:
        per-beta energy histograms (bin 64 over [-3N, 3N], every 10 sweeps) -> per-beta <E>/N

The whole schedule of each config runs on the device; the wall-clock of the run (CUDA-synchronised,
readouts at the checkpoints included) and the spin updates it performed are reported beside the
output.  Product-side only (no oracle).

  python tools/run_configs.py [--configs 1,2,3,4,5] [--out DIR]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2509_23043_b200 as T  # noqa: E402
from paper_2509_23043_b200 import workloads as WL  # noqa: E402


def checkpoints(total, per_decade=(1, 2, 5)):
    out, d = [], 1
    while d <= total:
        out += [k * d for k in per_decade if k * d <= total]
        d *= 10
    if out[-1] != total:
        out.append(total)
    return out


def per_beta(e, n):
    o = e.observables().astype(np.float64)  # [I][R][count, sumE, sumE2, sum|M|, sumM2]
    cnt = o[:, :, 0]
    mE = o[:, :, 1] / cnt / n          # per instance
    mM = o[:, :, 3] / cnt / n
    S = mE.shape[0]
    return {"E_per_spin": mE.mean(0).tolist(), "E_sd_over_seeds": mE.std(0, ddof=1).tolist() if S > 1 else None,
            "abs_m": mM.mean(0).tolist(), "abs_m_sd_over_seeds": mM.std(0, ddof=1).tolist() if S > 1 else None,
            "samples_per_slot": int(cnt[0, 0])}


def cfg1():
    R, I, n, S = 32, 16, 1024, 10_000
    betas = WL.geometric(0.2, 1.0, R)
    e = T.Ensemble(T.Model.lattice((32, 32)), betas, n_instances=I, seed=1)
    e.init_random()
    e.run(S, swap_every=1, measure_every=1, measure_from=S // 2)
    out = {"betas": betas.tolist(), **per_beta(e, n)}
    # SURVEY.md 8(c) indicative checkerboard values (8 CPU seeds) at slots 0, 9, 15, 21, 30
    out["survey_indicative_checkerboard"] = {"slots": [0, 9, 15, 21, 30],
                                             "E_per_spin": [-0.42823, -0.76793, -1.38623, -1.90475, -1.99566],
                                             "abs_m": [0.04207, 0.07663, 0.58847, 0.97223, 0.99889]}
    return out, I * R * n * S, {"instances": I, "sweeps": S, "note": "16 seeds of the one-instance run"}


def cfg2():
    R, I, n, S, nt, every = 64, 128, 4096, 20_000, 60, 100
    betas = WL.geometric(0.3, 0.6, R)
    mb = np.array([WL.yang_m(b) for b in betas[:nt]])
    e = T.Ensemble(T.Model.lattice((64, 64)), betas, n_instances=I, seed=2)
    e.init_random()
    for _ in range(S // every):
        e.run(every, swap_every=1, measure_every=10, measure_from=S // 2)
        e.generate_proposals(np.arange(nt), mb, refine=5)
    sa, sc, pa, pc = e.acceptance()
    out = {"betas": betas.tolist(), **per_beta(e, n),
           "proposal_acceptance": (pc.sum(0) / np.maximum(pa.sum(0), 1)).tolist(),
           "swap_acceptance": (sc.sum(0) / np.maximum(sa.sum(0), 1)).tolist()}
    upd = I * (R * n * S + (S // every) * nt * n * 5)
    return out, upd, {"instances": I, "sweeps": S, "tapt_rounds": S // every}


def residual(e, n, total, run):
    """best-so-far energy per instance at log-spaced sweeps; residual vs the run's final best."""
    cps, done, best = checkpoints(total), 0, []
    for c in cps:
        run(c - done)
        done = c
        best.append(e.best().astype(np.float64))
    B = np.stack(best)        # [checkpoint][instance]
    # per instance, its lowest energy over the whole run (all slots) stands in for E_gnd
    rho = T.residual_energy(B.T, B[-1], n)
    return cps, B, rho


def cfg3():
    R, I, n, S = 64, 256, 4096, 100_000
    e = T.Ensemble(T.Model.lattice((16,)), np.linspace(0.2, 3.0, R), n_instances=I, seed=3)
    e.generate_ea_disorder(3)
    e.init_random()
    cps, B, rho = residual(e, n, S, lambda k: e.run(k, swap_every=1))
    out = {"sweeps": cps, "residual_energy_per_spin": rho.tolist(),
           "best_E_per_spin_final_mean": float((B[-1] / n).mean()),
           "best_E_per_spin_final_min": float((B[-1] / n).min())}
    return out, I * R * n * S, {"instances": I, "sweeps": S}


def cfg4():
    R, I, S = 32, 512, 100_000
    M = T.Multiplier(16)
    m = M.model()
    e = T.Ensemble(m, WL.geometric(0.1, 5.0, R), n_instances=I, seed=4)
    prods = [T.random_semiprime(4, k, 16) for k in range(I)]
    e.set_clamps(np.stack([M.clamps(p * q) for p, q in prods]))
    e.init_random()
    e_gs = np.array([m.energy(M.forward(p, q)) for p, q in prods])  # energy of the true factorisation
    cps, done, succ, gap = checkpoints(S), 0, [], []
    for c in cps:
        e.run(c - done, swap_every=1)
        done = c
        b = e.best()
        succ.append(float(np.mean(b <= e_gs + 1e-9)))
        gap.append(float(np.mean(b - e_gs)))
    Sp = e.spins()
    cold = float(np.mean([M.decode(Sp[k][R - 1], p * q)[2] for k, (p, q) in enumerate(prods)]))
    # the same pipeline on an 8x8 multiplier (16-bit semiprimes), where plain PT does succeed
    M8 = T.Multiplier(8)
    m8 = M8.model()
    e8 = T.Ensemble(m8, WL.geometric(0.1, 5.0, R), n_instances=64, seed=4)
    pr8 = [T.random_semiprime(4, k, 8) for k in range(64)]
    e8.set_clamps(np.stack([M8.clamps(p * q) for p, q in pr8]))
    e8.init_random()
    g8 = np.array([m8.energy(M8.forward(p, q)) for p, q in pr8])
    c8, d8, s8 = checkpoints(20_000), 0, []
    for c in c8:
        e8.run(c - d8, swap_every=1)
        d8 = c
        s8.append(float(np.mean(e8.best() <= g8 + 1e-9)))
    out = {"sweeps": cps, "success_rate": succ, "mean_best_minus_factorisation_energy": gap,
           "coldest_slot_decodes_at_end": cold,
           "success_definition": "an instance counts from the first sweep after which any slot reached the energy "
                                 "of its true factorisation (in-kernel best-energy tracking after every sweep)",
           "calibration_8x8_multiplier_64_semiprimes": {"sweeps": c8, "success_rate": s8}}
    return out, I * R * m.n_free * S + 64 * R * m8.n_free * 20_000, {"instances": I, "sweeps": S}


def cfg5():
    L, R, I, S, nt, every, refine = 32, 64, 4096, 10_000, 56, 1000, 5
    n = L ** 3
    betas = np.linspace(0.2, 3.0, R)
    e = T.Ensemble(T.Model.lattice((L,)), betas, n_instances=I, seed=20250923)  # bench.py's SEED / DISORDER_SEED
    e.generate_ea_disorder(43)
    e.init_random()
    nb = 2 * 3 * n // 64
    e.set_histogram(-3 * n, 64, nb)
    for _ in range(S // every):
        e.generate_proposals(np.arange(nt), None, refine)
        e.run(every, swap_every=1, measure_every=10)
    h = e.histogram().astype(np.float64)  # [R][nb]
    centres = -3 * n + 64 * (np.arange(nb) + 0.5)
    mean = (h * centres).sum(1) / h.sum(1) / n
    sa, sc, pa, pc = e.acceptance()
    out = {"betas": betas.tolist(), "hist_mean_E_per_spin": mean.tolist(), "hist_samples_per_slot": int(h[0].sum()),
           "hist_nonzero_bins_per_slot": (h > 0).sum(1).tolist(),
           "proposal_acceptance": (pc.sum(0) / np.maximum(pa.sum(0), 1)).tolist()}
    upd = I * (R * n * S + (S // every) * nt * n * refine)
    return out, upd, {"instances": I, "sweeps": S, "tapt_rounds": S // every}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out"))
    args = ap.parse_args()
    if T.device_count() == 0:
        raise SystemExit("run_configs.py needs a GPU")
    import torch
    os.makedirs(args.out, exist_ok=True)
    for c in [int(x) for x in args.configs.split(",")]:
        fn = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4, 5: cfg5}[c]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out, upd, shape = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        rec = {"config": c, "run": shape, "wall_s": dt, "spin_updates": upd, "updates_per_s_wall": upd / dt,
               "output": out}
        json.dump(rec, open(os.path.join(args.out, f"outputs_cfg{c}.json"), "w"))
        summary = {k: (v if not isinstance(v, list) or len(v) <= 12 else f"[{len(v)} values]")
                   for k, v in out.items()}
        print(json.dumps({"config": c, "wall_s": round(dt, 2), "updates_per_s_wall": upd / dt, **summary}),
              flush=True)


if __name__ == "__main__":
    main()
