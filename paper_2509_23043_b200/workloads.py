"""The BASELINE.json workloads (configs 1-4; config 5 is bench.py's default) as device
ensembles with one measured "step" each.  Product-side
construction only -- no oracle, no CPU path.  Used by bench.py --workload and
tools/bench_configs.py.

  step of cfg1: 1000 checkerboard sweeps, swap pass + measurement after every sweep (296 seeds)
  step of cfg2: 10 x (100 sweeps, swap every sweep, measure every 10; then a TAPT round into the
                60 hottest slots: biased i.i.d. proposals, 5 refinement sweeps, Eq. 2)
  step of cfg3: 1000 sweeps, swap every sweep (EA +-1 disorder from derive(3, {0x88, gid}))
  step of cfg4: 1000 colour-class sweeps, swap every sweep (512 semiprime clamps)
"""
import numpy as np

# algorithmic integer instructions per update
I_U = {1: 36, 2: 36, 3: 42, 4: 53, 5: 42}


def geometric(b0, b1, R):
    return b0 * (b1 / b0) ** (np.arange(R) / (R - 1.0))


def yang_m(beta):
    """Spontaneous magnetization of the square-lattice ferromagnet (proposal bias, config 2)."""
    bc = 0.5 * np.log(1 + np.sqrt(2))
    return 0.0 if beta <= bc else (1.0 - np.sinh(2.0 * beta) ** -4) ** 0.125


def build(T, cfg, stream_ptr=None, instances=None):
    """Returns dict(ens, step, updates_per_step, desc, kernel, shape) for BASELINE config cfg."""
    if cfg == 1:
        m = T.Model.lattice((32, 32))
        # BASELINE config 1 is one instance (the CPU-runnable case); its seeds are independent
        # replicas of the whole run (SURVEY asks for >= 16), and 296 of them -- two per SM -- fill
        # the GPU (replicas only)
        R, I, n = 32, instances or 296, 1024
        e = T.Ensemble(m, geometric(0.2, 1.0, R), n_instances=I, seed=1)
        if stream_ptr:
            e.set_stream(stream_ptr)
        e.init_random()

        def step():
            e.run(1000, swap_every=1, measure_every=1, measure_from=0)
        upd = I * R * n * 1000
        desc = f"config 1: 2D ferro L=32 periodic, 32 slots geometric [0.2,1.0], {I} seeds, swap + measure every sweep"
    elif cfg == 2:
        m = T.Model.lattice((64, 64))
        R, I, n, nt, every = 64, instances or 128, 4096, 60, 100
        b = geometric(0.3, 0.6, R)
        mb = np.array([yang_m(x) for x in b[:nt]])
        e = T.Ensemble(m, b, n_instances=I, seed=2)
        if stream_ptr:
            e.set_stream(stream_ptr)
        e.init_random()

        def step():
            for _ in range(1000 // every):
                e.run(every, swap_every=1, measure_every=10)
                e.generate_proposals(np.arange(nt), mb, refine=5, return_accepted=False)
        upd = I * (R * n * 1000 + (1000 // every) * nt * n * 5)
        desc = (f"config 2: 2D ferro L=64, 64 slots geometric [0.3,0.6], {I} chains, TAPT every 100 sweeps into "
                "60 slots (Yang-biased i.i.d. + 5 sweeps + Eq. 2)")
    elif cfg == 3:
        m = T.Model.lattice((16,))
        R, I, n = 64, instances or 256, 4096
        e = T.Ensemble(m, np.linspace(0.2, 3.0, R), n_instances=I, seed=3)
        if stream_ptr:
            e.set_stream(stream_ptr)
        e.generate_ea_disorder(3)
        e.init_random()

        def step():
            e.run(1000, swap_every=1)
        upd = I * R * n * 1000
        desc = f"config 3: 3D EA +-1 L=16 periodic, 64 slots linear [0.2,3.0], {I} instances, swap every sweep"
    elif cfg == 4:
        M = T.Multiplier(16)
        m = M.model()
        R, I = 32, instances or 512
        e = T.Ensemble(m, geometric(0.1, 5.0, R), n_instances=I, seed=4)
        if stream_ptr:
            e.set_stream(stream_ptr)
        prods = [T.random_semiprime(4, k, 16) for k in range(I)]
        e.set_clamps(np.stack([M.clamps(p * q) for p, q in prods]))
        e.init_random()
        n = m.n_free

        def step():
            e.run(1000, swap_every=1)
        upd = I * R * n * 1000
        desc = (f"config 4: 16x16 multiplier (784 spins, 736 free), 32 slots geometric [0.1,5.0], {I} semiprimes, "
                "colour-class sweeps, swap every sweep")
    else:
        raise ValueError("workloads.build covers configs 1-4 (config 5 is bench.py's default)")
    return dict(ens=e, step=step, updates_per_step=upd, desc=desc, kernel=e.kernel, R=R, I=I)
