"""Real-valued couplings and fields on the device (K5, real.h): the reference's own Gaussian random
test graphs (proj/tests/test_spin_model.cpp:24-32) through the reference gibbs_sweep / gibbs_update
and the restated PT/TAPT driver (tests/golden/*real*.npz, from oracle/_ref) must come out of the
device bit for bit -- spins, FP64 energies, swap and proposal decisions.  Marked `gpu`."""
import os

import numpy as np
import pytest

import paper_2509_23043_b200 as T
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if T.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


def load(name):
    return np.load(os.path.join(GOLD, name))


def graphs():
    f = load("real_graphs.npz")
    out = []
    for k in range(3):
        n = int(f[f"g{k}_n"])
        args = (n, f[f"g{k}_ci"], f[f"g{k}_cj"], f[f"g{k}_J"], f[f"g{k}_h"], f[f"g{k}_clamp"])
        out.append((T.Model.graph(*args), O.Graph.from_couplings(*args)))
    return f, out


def unpack(bits, n):
    return np.where(np.unpackbits(bits)[:n] > 0, 1, -1).astype(np.int8)


def _run_schedule(e, f):
    """ref_pt_run's schedule: per global sweep T, sweep; swap if swap_every | T; proposal round if
    prop_every | T (the round comes after the sweep and swap of that T)."""
    S, se, pe = int(f["n_sweeps"]), int(f["swap_every"]), int(f["prop_every"])
    nt, refine, mb = int(f["n_targets"]), int(f["refine"]), np.asarray(f["m_bias"])
    if pe:
        for _ in range(S // pe):
            e.run(pe, swap_every=se)
            e.generate_proposals(np.arange(nt, dtype=np.uint32), mb[:nt], refine=refine)
        if S % pe:
            e.run(S % pe, swap_every=se)
    else:
        e.run(S, swap_every=se)


@pytest.mark.parametrize("tag,which", [("real_g0", [0, 0]), ("real_g1", [1]), ("real_g2", [2])])
def test_real_pt_tapt_matches_reference_golden(tag, which):
    fg, gs = graphs()
    f = load(f"pt_{tag}.npz")
    I, R, n = (int(x) for x in f["shape"])
    m = gs[which[0]][0]
    e = T.Ensemble(m, f["betas"], n_instances=I, seed=int(f["seed"]), instance_offset=int(f["gid0"]),
                   order="reference")
    assert e.kernel == "real" and e.real
    e.init_random()
    _run_schedule(e, f)
    spins = unpack(f["spins"], I * R * n).reshape(I, R, n)
    E = e.energies()
    assert E.dtype == np.float64
    assert np.array_equal(E, f["E"]), np.max(np.abs(E - f["E"]))  # FP64 energies bit for bit
    assert np.array_equal(e.spins(), spins)
    sa, sc, pa, pc = e.acceptance()
    assert np.array_equal(sc, f["swap_acc"][:, : R - 1])
    assert np.array_equal(pc, f["prop_acc"])
    assert f["swap_acc"].sum() > 0
    assert "k5_real_pt" in e.launch_log()


def test_real_colour_order_matches_oracle():
    """Colour-class order with real couplings: the same chain as the oracle restatement (RPT) with
    the engine's greedy colouring, through swaps and synthetic TAPT rounds with refinement."""
    fg, gs = graphs()
    m, g = gs[1]
    betas = np.linspace(0.2, 2.0, 40)  # two replica groups (40 slots > 32)
    e = T.Ensemble(m, betas, n_instances=3, seed=8, instance_offset=2)
    e.init_random()
    for _ in range(3):
        e.run(10, swap_every=1)
        e.generate_proposals(np.arange(12, dtype=np.uint32), None, refine=2)
    e.run(7, swap_every=2)
    colours = m.schedule()[0]
    order = g.colour_order(colours)
    for k in range(3):
        pt = O.RPT(g, betas, 8, 2 + k, order)
        for _ in range(3):
            pt.run(10, 1, 10, 12, None, 2)
        pt.run(7, 2)
        assert np.array_equal(e.energies()[k], pt.E)
        assert np.array_equal(e.spins()[k], pt.spins)
        assert np.array_equal(e.acceptance()[1][k], pt.swap_acc[:39])
        assert np.array_equal(e.acceptance()[3][k], pt.prop_acc)


def test_real_dropin_gibbs_sweep_and_update_match_reference_golden():
    f, gs = graphs()
    for k, (m, g) in enumerate(gs):
        s = f[f"sweep{k}_init"].copy()
        st = O.derive(9, [0x22, 0, k])
        st2, dE = T.gibbs_sweep(m, s, 0.7, st, 25)
        assert np.array_equal(dE, f[f"sweep{k}_dE"])
        assert np.array_equal(s, f[f"sweep{k}_final"])
        assert st2 == (st + 25 * len(g.free) * O.PHI) % 2**64
        for i in range(g.n):
            s2 = f[f"sweep{k}_init"].copy()
            st = O.derive(5, [0x44, k, i])
            if f[f"update{k}_clamped"][i]:
                with pytest.raises(T.ClampedSiteError):
                    T.gibbs_update(m, s2, i, 1.3, st)
                continue
            st2 = T.gibbs_update(m, s2, i, 1.3, st)
            assert np.array_equal(s2, f[f"update{k}_spins"][i])
            assert st2 == (st + O.PHI) % 2**64
        with pytest.raises(T.DimensionError):
            T.gibbs_update(m, np.ones(g.n + 1, np.int8), 0, 1.0, 1)


def test_integer_gibbs_update_matches_reference_rule():
    """gibbs_update on an integer graph (K5 with the exact tables) == mcmc.cpp:24-28 restated."""
    g = O.lattice_graph((6, 6), 1.0, False, np.array([1] + [0] * 35, np.int8))
    m = T.Model.graph(g.n, g.ci, g.cj, g.J, None, g.clamp)
    rs = np.random.default_rng(3)
    for i in range(1, 36):
        s = rs.choice([-1, 1], 36).astype(np.int8)
        s[0] = 1
        want = O.lib().oc_rupdate(g.roc(), s.ctypes.data_as(O._i8p), i, 0.8, 77 + i)
        st = T.gibbs_update(m, s, i, 0.8, 77 + i)
        assert s[i] == want and st == (77 + i + O.PHI) % 2**64
    with pytest.raises(T.ClampedSiteError):
        T.gibbs_update(m, np.ones(36, np.int8), 0, 0.8, 1)


def test_perturbed_device_exp_is_corrected_by_near_tie_replays(monkeypatch):
    """Make the device probabilities wrong by a relative 1e-3 and widen the near-tie band to 1e-2:
    every decision the perturbation could flip is then a near tie, re-evaluated with glibc exp and
    replayed when it differs -- the results must still equal the reference golden bit for bit, and
    replays must actually have happened."""
    monkeypatch.setenv("TAPT_K5_PERTURB", "1e-3")
    monkeypatch.setenv("TAPT_K5_BAND", "1e-2")
    fg, gs = graphs()
    f = load("pt_real_g0.npz")
    I, R, n = (int(x) for x in f["shape"])
    e = T.Ensemble(gs[0][0], f["betas"], n_instances=I, seed=int(f["seed"]), instance_offset=int(f["gid0"]),
                   order="reference")
    e.init_random()
    _run_schedule(e, f)
    assert np.array_equal(e.energies(), f["E"])
    assert np.array_equal(e.spins(), unpack(f["spins"], I * R * n).reshape(I, R, n))
    ties, replays = e.near_ties()
    print("near ties", ties, "replays", replays)
    assert ties > 100 and replays > 0  # the perturbation flipped decisions; the replays undid every one


def test_real_observables_histogram_and_best_are_consistent():
    fg, gs = graphs()
    m, g = gs[0]
    betas = np.linspace(0.3, 2.0, 8)
    e = T.Ensemble(m, betas, n_instances=2, seed=4, order="reference")
    e.init_random()
    e.set_histogram(-60, 2, 64)
    e.run(30, swap_every=1, measure_every=3, measure_from=6)
    obs = e.observables()
    assert obs.dtype == np.float64
    assert np.all(obs[:, :, 0] == 8)  # sweeps 9, 12, ..., 30
    h = e.histogram()
    assert h.sum() == 2 * 8 * 8
    best = e.best()
    assert np.all(best <= e.energies().min(axis=1))
    # exact energies recomputed from the spins (energy() order) equal the tracked ones to rounding
    S = e.spins()
    for k in range(2):
        for r in range(8):
            assert abs(m.energy(S[k, r]) - e.energies()[k, r]) < 1e-9


def test_real_lattice_coupling():
    """LatticeSpec::grid2d with a non-integer J (the reference accepts any double) runs on K5."""
    m = T.Model.lattice((6, 6), J=0.75, periodic=True)
    g = O.lattice_graph((6, 6), 0.75)
    betas = np.linspace(0.2, 1.5, 6)
    e = T.Ensemble(m, betas, n_instances=1, seed=3, order="reference")
    assert e.kernel == "real"
    e.init_random()
    e.run(20, swap_every=1)
    pt = O.RPT(g, betas, 3, 0, g.index_order())
    pt.run(20, 1)
    assert np.array_equal(e.energies()[0], pt.E) and np.array_equal(e.spins()[0], pt.spins)


def test_real_host_proposals_and_mh_correction_match_oracle():
    """Externally supplied proposals on a Gaussian-J graph: plain Eq. 2 and the MH-corrected move
     with arbitrary log q values, against the FP64 oracle."""
    fg, gs = graphs()
    m, g = gs[1]  # clamped Gaussian graph
    betas = np.linspace(0.3, 2.2, 10)
    e = T.Ensemble(m, betas, n_instances=2, seed=12, order="reference")
    e.init_random()
    pts = [O.RPT(g, betas, 12, k, g.index_order()) for k in range(2)]
    rs = np.random.default_rng(8)
    targets = np.array([1, 4, 7, 9], np.uint32)
    for rnd in range(4):
        e.run(6, swap_every=1)
        for pt in pts:
            pt.run(6, 1)
        props = np.where(rs.random((2, len(targets), g.n)) < 0.5, 1, -1).astype(np.int8)
        props[:, :, g.clamp != 0] = g.clamp[g.clamp != 0]
        lqc, lqp = rs.normal(size=(2, len(targets))), rs.normal(size=(2, len(targets)))
        mh = rnd % 2 == 1
        acc = e.inject_proposals(props, targets, lqc if mh else None, lqp if mh else None)
        for k, pt in enumerate(pts):
            mask = np.zeros(pt.R, np.uint8)
            mask[targets] = 1
            full = np.zeros_like(pt.spins)
            Ep = np.zeros(pt.R)
            a, b = np.zeros(pt.R), np.zeros(pt.R)
            for ti, r in enumerate(targets):
                full[r] = props[k, ti]
                Ep[r] = O.lib().oc_renergy(g.roc(), full[r].ctypes.data_as(O._i8p))
                a[r], b[r] = lqc[k, ti], lqp[k, ti]
            dec = pt.inject(mask, full, Ep, a if mh else None, b if mh else None)
            assert np.array_equal(acc[k], (dec[targets] == 1).astype(np.uint8))
    for k, pt in enumerate(pts):
        assert np.array_equal(e.energies()[k], pt.E) and np.array_equal(e.spins()[k], pt.spins)
        assert np.array_equal(e.acceptance()[3][k], pt.prop_acc)


def test_real_clamped_colour_order_ragged_groups():
    """Real couplings with clamps in colour order with R = 40 (a full and a partial 32-lane group) and
    a swap cadence of 3, against the oracle; per-instance clamps are refused (model clamps only)."""
    fg, gs = graphs()
    m, g = gs[1]
    betas = np.linspace(0.1, 3.0, 40)
    e = T.Ensemble(m, betas, n_instances=2, seed=21)
    e.init_random()
    e.run(25, swap_every=3)
    order = g.colour_order(m.schedule()[0])
    for k in range(2):
        pt = O.RPT(g, betas, 21, k, order)
        pt.run(25, 3)
        assert np.array_equal(e.energies()[k], pt.E) and np.array_equal(e.spins()[k], pt.spins)
    with pytest.raises(T.ConfigError):
        e.set_clamps(np.zeros((2, g.n), np.int8))
