"""Generate tests/golden/*.npz from the UNMODIFIED reference sources (oracle/_ref).

Run in the build container (where /root/reference exists):
    make -C oracle all && python tests/golden/make_golden.py

Every array here comes out of the reference's own code (RngStream, random_configuration,
gibbs_sweep, energy, LatticeSpec, CouplingGraph::Builder) driven through
oracle/ref_shim.cpp; the PT schedule around it is the restatement in ref_pt_run.
Spin arrays are stored bit-packed (np.packbits of s > 0) to keep fixtures small.
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

R = O.ref


def pack(s):
    return np.packbits(np.asarray(s) > 0)


ref_graph = O.ref_graph


def rng_fixture():
    out = {}
    for name, root, path in (("replica", 2024, [0x22, 7, 3]), ("coord", 99, [0x33, 1]),
                             ("init", 5, [0x11, 0, 31]), ("accept", 42, [0x33, 2, 5]),
                             ("proposal", 42, [0x22, 2, 5, 9]), ("disorder", 7, [0x88, 3])):
        p = np.array(path, np.uint64)
        d = np.zeros(256, np.uint64)
        R().ref_draws(root, O._p(p, O._u64p), len(p), 256, O._p(d, O._u64p))
        out[f"{name}_root"] = np.uint64(root)
        out[f"{name}_path"] = p
        out[f"{name}_draws"] = d
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)


def sweep_fixture(tag, g: O.Graph, betas, seed, n_sweeps):
    """Single-chain gibbs_sweep trajectories: init = random_configuration(derive(seed,{kInit,0,r})),
    dynamics = derive(seed,{kReplica,0,r}); per-sweep dE and final spins per beta."""
    rg = ref_graph(g)
    res = {"betas": np.asarray(betas, np.float64), "seed": np.uint64(seed), "n_sweeps": np.int64(n_sweeps)}
    init, final, dE, E0 = [], [], [], []
    for r, b in enumerate(betas):
        s = np.zeros(g.n, np.int8)
        p = np.array([0x11, 0, r], np.uint64)
        R().ref_random_configuration(rg, seed, O._p(p, O._u64p), 3, O._p(s, O._i8p))
        init.append(pack(s))
        E0.append(R().ref_energy(rg, O._p(s, O._i8p)))
        d = np.zeros(n_sweeps, np.float64)
        p = np.array([0x22, 0, r], np.uint64)
        R().ref_gibbs_sweeps(rg, O._p(s, O._i8p), b, seed, O._p(p, O._u64p), 3, n_sweeps, O._p(d, O._f64p))
        final.append(pack(s))
        dE.append(d)
    R().ref_graph_free(rg)
    res.update(init=np.array(init), final=np.array(final), dE=np.array(dE), E0=np.array(E0))
    np.savez_compressed(os.path.join(HERE, f"sweep_{tag}.npz"), **res)


def pt_fixture(tag, graphs, betas, seed, gid0, n_sweeps, swap_every, prop_every, n_targets, m_bias, refine):
    I, Rr, n = len(graphs), len(betas), graphs[0].n
    hs = [ref_graph(g) for g in graphs]
    arr = (C.c_void_p * I)(*hs)
    spins = np.zeros((I, Rr, n), np.int8)
    E = np.zeros((I, Rr), np.float64)
    sacc = np.zeros((I, max(Rr - 1, 1)), np.uint64)
    pacc = np.zeros((I, Rr), np.uint64)
    b = np.ascontiguousarray(betas, np.float64)
    mb = np.ascontiguousarray(m_bias, np.float64)
    R().ref_pt_run(arr, I, gid0, Rr, O._p(b, O._f64p), seed, n_sweeps, swap_every, prop_every, n_targets,
                   O._p(mb, O._f64p), refine, 4, O._p(spins, O._i8p), O._p(E, O._f64p), O._p(sacc, O._u64p),
                   O._p(pacc, O._u64p))
    for h in hs:
        R().ref_graph_free(h)
    np.savez_compressed(os.path.join(HERE, f"pt_{tag}.npz"), betas=b, seed=np.uint64(seed), gid0=np.uint64(gid0),
                        n_sweeps=np.int64(n_sweeps), swap_every=np.int64(swap_every),
                        prop_every=np.int64(prop_every), n_targets=np.int64(n_targets), m_bias=mb,
                        refine=np.int64(refine), spins=pack(spins.reshape(-1)), shape=np.array(spins.shape),
                        E=E, swap_acc=sacc, prop_acc=pacc)


def corpus_fixture(tag, g: O.Graph, betas, per_beta, mixing, thinning, seed):
    """Reference generate_training_corpus (mcmc.cpp:67-84) records."""
    rg = ref_graph(g)
    b = np.ascontiguousarray(betas, np.float64)
    out = np.zeros((len(b) * per_beta, g.n), np.int8)
    R().ref_generate_corpus(rg, O._p(b, O._f64p), len(b), per_beta, mixing, thinning, seed, O._p(out, O._i8p))
    R().ref_graph_free(rg)
    np.savez_compressed(os.path.join(HERE, f"corpus_{tag}.npz"), betas=b, per_beta=np.int64(per_beta),
                        mixing=np.int64(mixing), thinning=np.int64(thinning), seed=np.uint64(seed),
                        spins=pack(out.reshape(-1)), shape=np.array(out.shape))


def ref_random_graph(n, p, fields, seed):
    """The reference tests' random_graph (proj/tests/test_spin_model.cpp:24-32): Gaussian couplings
    and fields from the reference's RngStream::normal."""
    m = n * (n - 1) // 2
    ci, cj = np.zeros(m, np.uint32), np.zeros(m, np.uint32)
    J, h = np.zeros(m, np.float64), np.zeros(n, np.float64)
    R().ref_random_graph.restype = C.c_uint32
    R().ref_random_graph.argtypes = [C.c_uint32, C.c_double, C.c_int, C.c_uint64, O._u32p, O._u32p, O._f64p,
                                     O._f64p]
    k = R().ref_random_graph(n, p, int(fields), seed, O._p(ci, O._u32p), O._p(cj, O._u32p), O._p(J, O._f64p),
                             O._p(h, O._f64p))
    return ci[:k], cj[:k], J[:k], h


def real_fixtures():
    """Real-valued (Gaussian) couplings and fields: the reference's own random test graphs run
    through the reference gibbs_sweep / gibbs_update and the restated PT/TAPT driver (FP64 energies)."""
    graphs = []
    for k, (n, p, fields, seed) in enumerate(((24, 0.3, True, 101), (40, 0.15, True, 202), (32, 0.25, False, 303))):
        ci, cj, J, h = ref_random_graph(n, p, fields, seed)
        cl = np.zeros(n, np.int8)
        if k == 1:
            cl[[3, 17, 30]] = [1, -1, 1]
        graphs.append(O.Graph.from_couplings(n, ci, cj, J, h, cl))
    out = {}
    for k, g in enumerate(graphs):
        out[f"g{k}_n"] = np.int64(g.n)
        out[f"g{k}_ci"], out[f"g{k}_cj"], out[f"g{k}_J"] = g.ci, g.cj, g.J
        out[f"g{k}_h"], out[f"g{k}_clamp"] = g.h, g.clamp
    # single-chain gibbs_sweep trajectories (drop-in tapt::gibbs_sweep)
    for k, g in enumerate(graphs):
        rg = ref_graph(g)
        s = np.zeros(g.n, np.int8)
        pth = np.array([0x11, 0, k], np.uint64)
        R().ref_random_configuration(rg, 9, O._p(pth, O._u64p), 3, O._p(s, O._i8p))
        out[f"sweep{k}_init"] = s.copy()
        d = np.zeros(25, np.float64)
        pth = np.array([0x22, 0, k], np.uint64)
        R().ref_gibbs_sweeps(rg, O._p(s, O._i8p), 0.7, 9, O._p(pth, O._u64p), 3, 25, O._p(d, O._f64p))
        out[f"sweep{k}_final"], out[f"sweep{k}_dE"] = s, d
        # gibbs_update at every site in turn (ClampedSiteError at clamped sites), stream {kChain, k}
        R().ref_gibbs_update.restype = C.c_uint64
        R().ref_gibbs_update.argtypes = [C.c_void_p, O._i8p, C.c_uint32, C.c_double, C.c_uint64, O._u64p, C.c_int,
                                         C.POINTER(C.c_int)]
        upd, err = np.zeros((g.n, g.n), np.int8), np.zeros(g.n, np.int8)
        for i in range(g.n):
            s2 = out[f"sweep{k}_init"].copy()
            flag = C.c_int(0)
            pth = np.array([0x44, k, i], np.uint64)
            R().ref_gibbs_update(rg, O._p(s2, O._i8p), i, 1.3, 5, O._p(pth, O._u64p), 3, C.byref(flag))
            upd[i], err[i] = s2, flag.value
        out[f"update{k}_spins"], out[f"update{k}_clamped"] = upd, err
        R().ref_graph_free(rg)
    np.savez_compressed(os.path.join(HERE, "real_graphs.npz"), **out)
    # PT + TAPT rounds on them (index order), two instances of graph 0 and one each of graphs 1, 2
    betas = np.linspace(0.1, 2.5, 8)
    pt_fixture("real_g0", [graphs[0], graphs[0]], betas, 41, 3, 60, 1, 20, 4, np.zeros(8), 2)
    pt_fixture("real_g1", [graphs[1]], betas, 42, 0, 60, 1, 30, 6, np.full(8, 0.3), 3)
    pt_fixture("real_g2", [graphs[2]], betas, 43, 0, 80, 2, 0, 0, np.zeros(8), 0)


def main():
    if not O.have_ref():
        raise SystemExit("build oracle/_ref first: make -C oracle all")
    rng_fixture()
    # config-1 geometry: 2D L=32 periodic ferro
    g2 = O.lattice_graph((32, 32))
    sweep_fixture("2d32", g2, [0.2, 0.4407, 1.0], 11, 64)
    # config-3 geometry at L=8: 3D EA +-J
    g3 = O.ea_graph((8,), 7, 0)
    sweep_fixture("ea3d8", g3, [0.3, 1.0, 3.0], 13, 32)
    # clamped 2D open lattice with a field-free top-row clamp (reference graph_clamped semantics)
    cl = np.zeros(36, np.int8)
    cl[:6] = [1, -1, -1, 1, 1, -1]
    g4 = O.lattice_graph((6, 6), 1.0, False, cl)
    sweep_fixture("2d6clamped", g4, [0.5, 2.0], 17, 40)
    # PT with swaps every sweep: config-1 shape, short
    betas1 = 0.2 * 5.0 ** (np.arange(32) / 31.0)
    pt_fixture("cfg1_200", [g2], betas1, 2024, 0, 200, 1, 0, 0, np.zeros(32), 0)
    # PT + synthetic proposals (config-2 style, biased by Yang's m*) at L=16
    g5 = O.lattice_graph((16, 16))
    betas2 = 0.3 * 2.0 ** (np.arange(16) / 15.0)
    mb = np.array([O.yang_m(b) for b in betas2])
    pt_fixture("tapt2d16", [g5, g5], betas2, 77, 5, 120, 1, 20, 12, mb, 5)
    # EA 3D L=6, 2 instances, fair proposals (config-5 style)
    gs = [O.ea_graph((6,), 3, k) for k in range(2)]
    betas3 = np.linspace(0.2, 3.0, 12)
    pt_fixture("ea3d6_tapt", gs, betas3, 31, 0, 90, 1, 30, 8, np.zeros(12), 5)
    # training corpus (run_chain per beta) on a clamped 8x8 open lattice
    cl = np.zeros(64, np.int8)
    cl[:8] = [1, 1, -1, -1, 1, -1, 1, -1]
    corpus_fixture("2d8clamped", O.lattice_graph((8, 8), 1.0, False, cl), [0.2, 0.44, 0.7, 1.5], 3, 20, 5, 99)
    real_fixtures()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
