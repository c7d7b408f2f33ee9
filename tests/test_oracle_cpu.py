"""CPU tests: pin the oracle restatement (oracle/tapt_oracle.c) against the reference.

Two anchors:
  * tests/golden/*.npz -- produced from the unmodified reference sources (make_golden.py);
  * oracle/_ref/libtapt_ref.so live (skipped where it was not built).
"""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


def unpack(bits, n):
    return np.where(np.unpackbits(bits)[:n] > 0, 1, -1).astype(np.int8)


# ------------------------------------------------------------------ RNG ----

def test_rng_matches_reference_golden():
    f = load("rng.npz")
    for name in ("replica", "coord", "init", "accept", "proposal", "disorder"):
        root = int(f[f"{name}_root"])
        path = [int(x) for x in f[f"{name}_path"]]
        s0 = O.derive(root, path)
        mine = np.array([O.draw(s0, k + 1) for k in range(256)], np.uint64)
        assert np.array_equal(mine, f[f"{name}_draws"]), name


def test_threshold_equivalence():
    """uniform() < p  <=>  (x >> 11) < ceil(p * 2^53)  (rng.hpp:35, mcmc.cpp:13-15)."""
    rs = np.random.default_rng(0)
    for _ in range(20000):
        beta = rs.uniform(0, 5)
        l = float(rs.integers(-64, 65))
        x = int(rs.integers(0, 2**63)) * 2 + int(rs.integers(0, 2))
        p = O.lib().oc_conditional_up(beta, l)
        u = (x >> 11) * 2.0**-53
        assert (u < p) == ((x >> 11) < O.threshold(beta, l))


def test_spec_known_answers():
    cu = O.lib().oc_conditional_up
    assert cu(0.7, 0.0) == 0.5 and cu(0.0, 3.0) == 0.5
    assert abs(cu(1.0, 1.0) - 0.8808) < 1e-4
    assert abs(math.exp(0.1 * -5) - 0.6065) < 1e-4                   # SPEC.md:407 (swap)
    assert abs(math.exp(0.5 * -2) - 0.3679) < 1e-4                   # SPEC.md:416 (proposal)


# --------------------------------------------------------------- energy ----

def and_gate():
    return O.Graph.from_couplings(3, [0, 0, 1], [1, 2, 2], [-1.0, 2.0, 2.0], [1.0, 1.0, -2.0])


def E(g, s):
    gc = g.oc()
    return O.lib().oc_energy(gc, np.ascontiguousarray(s, np.int8).ctypes.data_as(O._i8p))


def test_reference_energy_examples():
    """The assertions of proj/tests/test_spin_model.cpp:36-122 re-expressed."""
    g22 = O.lattice_graph((2, 2), 1.0, periodic=False)
    assert E(g22, np.ones(4)) == -4                                  # :36-40
    g1 = O.Graph.from_couplings(1, [], [], [], [2.0])
    assert E(g1, [1]) == -2                                           # :42-48
    ag = and_gate()
    es = [E(ag, [1 if (m >> k) & 1 else -1 for k in range(3)]) for m in range(8)]
    assert min(es) == -3 and E(ag, [1, 1, 1]) == -3                   # :50-59
    g33 = O.lattice_graph((3, 3), 1.0, periodic=False)
    s = np.ones(9, np.int8)
    assert O.lib().oc_local_field(g33.oc(), s.ctypes.data_as(O._i8p), 4) == 4.0   # :81-84
    e0 = E(g33, s)
    s[4] = -1
    assert E(g33, s) - e0 == 8                                        # :85-88
    for i in range(4):                                                # :106-113
        f = np.ones(4, np.int8)
        f[i] = -1
        assert E(g22, f) - E(g22, np.ones(4)) == 4
    assert E(ag, [1, 1, -1]) - E(ag, [1, 1, 1]) == 4                  # :115-121


def test_lattice_counts_and_indexing():
    """proj/tests/test_spin_model.cpp:244-259."""
    n, ci, _, _ = O.lattice_couplings((4, 5), 1.0, periodic=False)
    assert n == 20 and len(ci) == 4 * 4 + 5 * 3
    n, ci, _, _ = O.lattice_couplings((3,), 1.0, periodic=False)
    assert n == 27 and len(ci) == 3 * 9 * 2


# ------------------------------------------------------- golden sweeps ----

@pytest.mark.parametrize("tag,builder", [
    ("2d32", lambda: O.lattice_graph((32, 32))),
    ("ea3d8", lambda: O.ea_graph((8,), 7, 0)),
    ("2d6clamped", lambda: O.lattice_graph((6, 6), 1.0, False,
                                           np.array([1, -1, -1, 1, 1, -1] + [0] * 30, np.int8))),
])
def test_index_sweeps_match_reference_golden(tag, builder):
    f = load(f"sweep_{tag}.npz")
    g = builder()
    gc = g.oc()
    order = g.index_order()
    seed = int(f["seed"])
    for r, beta in enumerate(f["betas"]):
        s = np.zeros(g.n, np.int8)
        O.lib().oc_random_configuration(gc, O.derive(seed, [0x11, 0, r]), s.ctypes.data_as(O._i8p))
        assert np.array_equal(s, unpack(f["init"][r], g.n))
        assert E(g, s) == f["E0"][r]
        s0 = O.derive(seed, [0x22, 0, r])
        for t in range(int(f["n_sweeps"])):
            d = O.lib().oc_sweep(gc, order.ctypes.data_as(O._u32p), s.ctypes.data_as(O._i8p), float(beta), s0,
                                 t * len(g.free))
            assert d == f["dE"][r][t]
        assert np.array_equal(s, unpack(f["final"][r], g.n))


def _pt_golden(tag, graphs):
    f = load(f"pt_{tag}.npz")
    I, R, n = (int(x) for x in f["shape"])
    spins = unpack(f["spins"], I * R * n).reshape(I, R, n)
    for k, g in enumerate(graphs):
        pt = O.PT(g, f["betas"], int(f["seed"]), int(f["gid0"]) + k, g.index_order())
        pt.run(int(f["n_sweeps"]), int(f["swap_every"]), int(f["prop_every"]), int(f["n_targets"]),
               f["m_bias"], int(f["refine"]))
        assert np.array_equal(pt.spins, spins[k])
        assert np.array_equal(pt.E.astype(np.float64), f["E"][k])
        assert np.array_equal(pt.swap_acc[: R - 1], f["swap_acc"][k][: R - 1])
        assert np.array_equal(pt.prop_acc, f["prop_acc"][k])
    return f


def test_pt_swaps_match_reference_golden():
    f = _pt_golden("cfg1_200", [O.lattice_graph((32, 32))])
    assert f["swap_acc"].sum() > 0


def test_pt_tapt_biased_match_reference_golden():
    g = O.lattice_graph((16, 16))
    f = _pt_golden("tapt2d16", [g, g])
    assert f["prop_acc"].sum() > 0


def test_pt_tapt_ea_match_reference_golden():
    _pt_golden("ea3d6_tapt", [O.ea_graph((6,), 3, k) for k in range(2)])


# --------------------------------------------------- live reference -----

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (no /root/reference here)")


def _ref_graph(g):
    return O.ref_graph(g)


@needs_ref
@pytest.mark.parametrize("dims,periodic", [((5, 7), False), ((4, 4), True), ((6, 3), True), ((3,), True),
                                           ((4,), False), ((2, 2), True)])
def test_lattice_builder_matches_reference(dims, periodic):
    R = O.ref()
    kind = len(dims) + 1 if len(dims) == 2 else 3
    h = R.ref_graph_lattice(2 if len(dims) == 2 else 3, dims[0], dims[-1], dims[0], 1.0, int(periodic))
    m = R.ref_graph_ncoup(h)
    ci, cj, J = np.zeros(m, np.uint32), np.zeros(m, np.uint32), np.zeros(m)
    R.ref_graph_couplings(h, ci.ctypes.data_as(O._u32p), cj.ctypes.data_as(O._u32p), J.ctypes.data_as(O._f64p))
    g = O.lattice_graph(dims, 1.0, periodic)
    assert np.array_equal(ci, g.ci) and np.array_equal(cj, g.cj) and np.array_equal(J, g.J)
    R.ref_graph_free(h)
    del kind


@needs_ref
def test_random_integer_graphs_sweep_like_reference():
    """Integer J in [-3,3], integer h, random clamps: oracle index sweep == reference gibbs_sweep."""
    rs = np.random.default_rng(5)
    R = O.ref()
    for trial in range(12):
        n = int(rs.integers(5, 40))
        m = int(rs.integers(n, 4 * n))
        ci, cj = rs.integers(0, n, m), rs.integers(0, n, m)
        keep = ci != cj
        J = rs.integers(-3, 4, m).astype(float)
        h = rs.integers(-2, 3, n).astype(float) if trial % 2 else None
        cl = np.where(rs.random(n) < 0.15, rs.choice([-1, 1], n), 0).astype(np.int8)
        g = O.Graph.from_couplings(n, ci[keep], cj[keep], J[keep], h, cl)
        rg = _ref_graph(g)
        s = np.zeros(n, np.int8)
        R.ref_random_configuration(rg, 9, np.array([0x11, trial], np.uint64).ctypes.data_as(O._u64p), 2,
                                   s.ctypes.data_as(O._i8p))
        s2 = s.copy()
        assert E(g, s) == R.ref_energy(rg, s.ctypes.data_as(O._i8p))
        beta = float(rs.uniform(0.1, 2.0))
        d = np.zeros(7)
        R.ref_gibbs_sweeps(rg, s.ctypes.data_as(O._i8p), beta, 9, np.array([0x22, trial], np.uint64).ctypes.data_as(
            O._u64p), 2, 7, d.ctypes.data_as(O._f64p))
        s0 = O.derive(9, [0x22, trial])
        gc = g.oc()
        order = g.index_order()
        for t in range(7):
            dd = O.lib().oc_sweep(gc, order.ctypes.data_as(O._u32p), s2.ctypes.data_as(O._i8p), beta, s0,
                                  t * len(g.free))
            assert dd == d[t]
        assert np.array_equal(s, s2)
        R.ref_graph_free(rg)


def test_checkerboard_is_a_different_valid_order():
    """Colour order uses the same per-site draws but is a different chain."""
    g = O.lattice_graph((8, 8))
    pt_a = O.PT(g, [0.5, 1.0], 3, 0, g.index_order())
    pt_b = O.PT(g, [0.5, 1.0], 3, 0, g.colour_order(O.checkerboard_colours((8, 8))))
    assert np.array_equal(pt_a.spins, pt_b.spins)
    for _ in range(5):
        pt_a.sweep()
        pt_b.sweep()
    assert not np.array_equal(pt_a.spins, pt_b.spins)
    for pt in (pt_a, pt_b):
        gc = g.oc()
        for r in range(2):
            assert pt.E[r] == O.lib().oc_energy(gc, pt.spins[r].ctypes.data_as(O._i8p))


# ------------------------------------------- real-valued (Gaussian) couplings --

def real_graphs():
    f = load("real_graphs.npz")
    gs = [O.Graph.from_couplings(int(f[f"g{k}_n"]), f[f"g{k}_ci"], f[f"g{k}_cj"], f[f"g{k}_J"], f[f"g{k}_h"],
                                 f[f"g{k}_clamp"]) for k in range(3)]
    return f, gs


def test_real_graphs_are_not_integer_valued():
    f, gs = real_graphs()
    for g in gs:
        assert np.any(g.J != np.rint(g.J))
    assert np.any(gs[0].h != 0) and np.all(gs[2].h == 0) and np.count_nonzero(gs[1].clamp) == 3


def test_real_sweeps_and_updates_match_reference_golden():
    """oc_rsweep / oc_rupdate (FP64 local fields, libm exp) against the reference's gibbs_sweep and
    gibbs_update on its own Gaussian random graphs (test_spin_model.cpp:24-32)."""
    f, gs = real_graphs()
    for k, g in enumerate(gs):
        gc = g.roc()
        s = f[f"sweep{k}_init"].copy()
        order = g.index_order()
        s0 = O.derive(9, [0x22, 0, k])
        for t in range(25):
            d = O.lib().oc_rsweep(gc, order.ctypes.data_as(O._u32p), s.ctypes.data_as(O._i8p), 0.7, s0,
                                  t * len(g.free))
            assert d == f[f"sweep{k}_dE"][t]
        assert np.array_equal(s, f[f"sweep{k}_final"])
        for i in range(g.n):
            if f[f"update{k}_clamped"][i]:
                assert g.clamp[i] != 0
                continue
            s2 = f[f"sweep{k}_init"].copy()
            s2[i] = O.lib().oc_rupdate(gc, s2.ctypes.data_as(O._i8p), i, 1.3, O.derive(5, [0x44, k, i]))
            assert np.array_equal(s2, f[f"update{k}_spins"][i])


@pytest.mark.parametrize("tag,which", [("real_g0", [0, 0]), ("real_g1", [1]), ("real_g2", [2])])
def test_real_pt_matches_reference_golden(tag, which):
    _, gs = real_graphs()
    f = load(f"pt_{tag}.npz")
    I, R, n = (int(x) for x in f["shape"])
    spins = unpack(f["spins"], I * R * n).reshape(I, R, n)
    for k, w in enumerate(which):
        g = gs[w]
        pt = O.RPT(g, f["betas"], int(f["seed"]), int(f["gid0"]) + k, g.index_order())
        pt.run(int(f["n_sweeps"]), int(f["swap_every"]), int(f["prop_every"]), int(f["n_targets"]),
               f["m_bias"], int(f["refine"]))
        assert np.array_equal(pt.spins, spins[k])
        assert np.array_equal(pt.E, f["E"][k])  # FP64 energies, bit for bit
        assert np.array_equal(pt.swap_acc[: R - 1], f["swap_acc"][k][: R - 1])
        assert np.array_equal(pt.prop_acc, f["prop_acc"][k])
    assert f["swap_acc"].sum() > 0
