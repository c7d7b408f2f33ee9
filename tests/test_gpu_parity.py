"""GPU parity tests: the sm_100a kernels (through the C ABI) against the oracle
restatement and the reference golden vectors -- bit-exact spins, energies, swap and
proposal decisions, observables.  Marked `gpu`."""
import os

import numpy as np
import pytest

import paper_2509_23043_b200 as T
from oracle import oracle as O
import tapt_helpers as H

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def unpack(bits, n):
    return np.where(np.unpackbits(bits)[:n] > 0, 1, -1).astype(np.int8)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if T.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


def compare(ens, pts, check_counts=True):
    S = ens.spins()
    E = ens.energies()
    sa, sc, pa, pc = ens.acceptance()
    for k, pt in enumerate(pts):
        assert np.array_equal(E[k], pt.E), f"energies differ, instance {k}"
        assert np.array_equal(S[k], pt.spins), f"spins differ, instance {k}"
        if check_counts:
            assert np.array_equal(sc[k], pt.swap_acc[: ens.R - 1]), f"swap accepts differ, instance {k}"
            assert np.array_equal(sa[k], pt.swap_att[: ens.R - 1])
            assert np.array_equal(pc[k], pt.prop_acc)


# ------------------------------------------------------------ K1 lattice ----

def test_cfg1_geometry_checkerboard_pt_bit_exact():
    """Config 1 shape: 2D L=32 ferro, 32 slots geometric [0.2, 1.0], swap every sweep."""
    betas = H.geometric(0.2, 1.0, 32)
    m = T.Model.lattice((32, 32))
    e = T.Ensemble(m, betas, n_instances=2, seed=2024)
    assert e.kernel == "lattice"
    e.init_random()
    e.run(300, swap_every=1)
    pts = H.run_oracle([O.lattice_graph((32, 32))] * 2, betas, 2024, 0, H.checkerboard_order((32, 32)), 300)
    compare(e, pts)


@pytest.mark.parametrize("threads", [None, "1024", "128"])
def test_ea3d_cluster_pt_bit_exact(threads, monkeypatch):
    """3D EA +-J, 64 slots (2-CTA cluster per instance), device-generated disorder; also with
    the 1-site/1024-thread and small-CTA launch shapes of K1 (results must not depend on them)."""
    if threads:
        monkeypatch.setenv("TAPT_K1_THREADS", threads)
    L, R = 16 if threads == "1024" else 8, 64
    betas = H.linear(0.2, 3.0, R)
    m = T.Model.lattice((L,))
    e = T.Ensemble(m, betas, n_instances=3, seed=77, instance_offset=5)
    e.generate_ea_disorder(1234)
    graphs = [O.ea_graph((L,), 1234, 5 + k) for k in range(3)]
    n, ci, cj, _ = O.lattice_couplings((L,), 1.0, True)
    signs = e.bond_signs(len(ci))
    for k in range(3):
        assert np.array_equal(signs[k].astype(float), O.ea_signs((L,), 1234, 5 + k))
    e.init_random()
    e.run(120, swap_every=1)
    pts = H.run_oracle(graphs, betas, 77, 5, H.checkerboard_order((L,)), 120)
    compare(e, pts)


def test_2d64_two_groups_and_measurements():
    """2D L=64 (config 2 geometry) with 40 slots (partial second group) and observables."""
    betas = H.geometric(0.3, 0.6, 40)
    m = T.Model.lattice((64, 64))
    e = T.Ensemble(m, betas, n_instances=1, seed=9)
    e.init_random()
    e.run(60, swap_every=1, measure_every=3, measure_from=10)
    pts = H.run_oracle([O.lattice_graph((64, 64))], betas, 9, 0, H.checkerboard_order((64, 64)), 60,
                       measure_every=3, measure_from=10)
    compare(e, pts)
    obs = e.observables()[0]
    mm = pts[0].meas
    for j, key in enumerate(("cnt", "sumE", "sumE2", "sumAbsM", "sumM2")):
        assert np.array_equal(obs[:, j], mm[key]), key


def test_histograms_and_best():
    L, R = 6, 12
    betas = H.linear(0.2, 3.0, R)
    m = T.Model.lattice((8,))
    e = T.Ensemble(m, betas, n_instances=2, seed=3)
    e.generate_ea_disorder(8)
    e.set_histogram(-3 * 512, 64, 48)
    e.init_random()
    e.run(80, swap_every=1, measure_every=10, measure_from=20)
    graphs = [O.ea_graph((8,), 8, k) for k in range(2)]
    pts = H.run_oracle(graphs, betas, 3, 0, H.checkerboard_order((8,)), 80, measure_every=10, measure_from=20,
                       e_lo=-3 * 512, width=64, nbins=48)
    compare(e, pts)
    hist = e.histogram()
    assert np.array_equal(hist.astype(np.int64), pts[0].hist + pts[1].hist)
    assert np.array_equal(e.best(), [pt.best for pt in pts])
    del L


def test_sweep_and_standalone_swap_compose():
    """tapt_sweep + tapt_swap_pass reproduce the fused run."""
    betas = H.geometric(0.2, 1.0, 16)
    m = T.Model.lattice((16, 16))
    a = T.Ensemble(m, betas, seed=1)
    b = T.Ensemble(m, betas, seed=1)
    a.init_random()
    b.init_random()
    a.run(30, swap_every=1)
    for t in range(30):
        b.sweep(1)
        b.swap_pass(t & 1)
    assert np.array_equal(a.spins(), b.spins())
    assert np.array_equal(a.energies(), b.energies())
    assert np.array_equal(a.acceptance()[1], b.acceptance()[1])


# ------------------------------------------------------------ K2 CSR --------

@pytest.mark.parametrize("kernel", ["levels", "csr"])
def test_reference_order_pt_matches_reference_golden(kernel, monkeypatch):
    """Index-order PT on the device == the reference's own gibbs_sweep driven PT (golden), with K4
    (one warp per site word on the dependency levels) and with K2 (TAPT_K4=0)."""
    monkeypatch.setenv("TAPT_K4", "1" if kernel == "levels" else "0")
    f = np.load(os.path.join(GOLD, "pt_cfg1_200.npz"))
    I, R, n = (int(x) for x in f["shape"])
    m = T.Model.lattice((32, 32))
    e = T.Ensemble(m, f["betas"], n_instances=I, seed=int(f["seed"]), instance_offset=int(f["gid0"]),
                   order="reference")
    assert e.kernel == kernel
    e.init_random()
    e.run(int(f["n_sweeps"]), swap_every=int(f["swap_every"]))
    spins = unpack(f["spins"], I * R * n).reshape(I, R, n)
    assert np.array_equal(e.spins(), spins)
    assert np.array_equal(e.energies().astype(np.float64), f["E"])
    assert np.array_equal(e.acceptance()[1], f["swap_acc"][:, : R - 1])


@pytest.mark.parametrize("tag", ["2d32", "ea3d8", "2d6clamped"])
def test_dropin_gibbs_sweep_matches_reference_golden(tag):
    f = np.load(os.path.join(GOLD, f"sweep_{tag}.npz"))
    if tag == "2d32":
        g = O.lattice_graph((32, 32))
        m = T.Model.lattice((32, 32))
    elif tag == "ea3d8":
        g = O.ea_graph((8,), 7, 0)
        m = T.Model.graph(g.n, g.ci, g.cj, g.J)
    else:
        cl = np.array([1, -1, -1, 1, 1, -1] + [0] * 30, np.int8)
        g = O.lattice_graph((6, 6), 1.0, False, cl)
        m = T.Model.graph(g.n, g.ci, g.cj, g.J, None, cl)
    seed = int(f["seed"])
    for r, beta in enumerate(f["betas"]):
        s = unpack(f["init"][r], g.n).copy()
        st = O.derive(seed, [0x22, 0, r])
        st2, dE = T.gibbs_sweep(m, s, float(beta), st, int(f["n_sweeps"]))
        assert np.array_equal(dE, f["dE"][r])
        assert np.array_equal(s, unpack(f["final"][r], g.n))
        assert st2 == (st + int(f["n_sweeps"]) * len(g.free) * O.PHI) % 2**64


def _random_circuit(seed, n=60):
    rs = np.random.default_rng(seed)
    m = 4 * n
    ci, cj = rs.integers(0, n, m), rs.integers(0, n, m)
    keep = ci != cj
    J = rs.choice([-2, -1, 1, 2], m).astype(float)
    h = rs.integers(-3, 4, n).astype(float)
    cl = np.where(rs.random(n) < 0.1, rs.choice([-1, 1], n), 0).astype(np.int8)
    return O.Graph.from_couplings(n, ci[keep], cj[keep], J[keep], h, cl)


def test_k2_colour_order_circuit_like_graph():
    g = _random_circuit(11)
    m = T.Model.graph(g.n, g.ci, g.cj, g.J, g.h, g.clamp)
    colours, _ = m.schedule()
    assert np.array_equal(colours, O.greedy_colours(g))
    betas = H.geometric(0.1, 5.0, 32)
    e = T.Ensemble(m, betas, n_instances=3, seed=5)
    e.init_random()
    e.run(150, swap_every=1)
    pts = H.run_oracle([g] * 3, betas, 5, 0, H.colour_order_for(colours), 150)
    compare(e, pts)


def test_k4_reference_order_circuit_with_clamps_and_fields_equals_k2(monkeypatch):
    """K4 (levels) == K2 in the reference's index order on a clamped circuit with fields (32 slots,
    swaps, measurements, a TAPT round), and both == the oracle."""
    g = _random_circuit(14, n=50)
    m = T.Model.graph(g.n, g.ci, g.cj, g.J, g.h, g.clamp)
    betas = H.geometric(0.2, 3.0, 32)

    def run(k4):
        monkeypatch.setenv("TAPT_K4", "1" if k4 else "0")
        e = T.Ensemble(m, betas, n_instances=5, seed=13, order="reference")
        assert e.kernel == ("levels" if k4 else "csr")
        e.init_random()
        e.set_histogram(-400, 8, 100)
        e.run(60, swap_every=1, measure_every=3)
        e.generate_proposals(np.arange(10), None, refine=2)
        e.run(20, swap_every=1, measure_every=3)
        return e
    a, b = run(True), run(False)
    for x, y in zip((a.spins(), a.energies(), a.permutation(), a.observables(), a.histogram(), a.best()),
                    (b.spins(), b.energies(), b.permutation(), b.observables(), b.histogram(), b.best())):
        assert np.array_equal(x, y)
    for x, y in zip(a.acceptance(), b.acceptance()):
        assert np.array_equal(x, y)
    monkeypatch.setenv("TAPT_K4", "1")
    e = T.Ensemble(m, betas, n_instances=2, seed=13, order="reference")
    e.init_random()
    e.run(40, swap_every=1)
    compare(e, H.run_oracle([g] * 2, betas, 13, 0, H.index_order, 40))


def test_k2_reference_order_with_clamps_and_fields():
    g = _random_circuit(12, n=45)
    m = T.Model.graph(g.n, g.ci, g.cj, g.J, g.h, g.clamp)
    betas = H.linear(0.2, 2.0, 40)  # two groups -> cluster of 2
    e = T.Ensemble(m, betas, n_instances=2, seed=6, order="reference")
    e.init_random()
    e.run(80, swap_every=2)
    pts = H.run_oracle([g] * 2, betas, 6, 0, H.index_order, 80, swap_every=2)
    compare(e, pts)


def test_k1_k2_k3_give_the_same_chain_on_a_lattice(monkeypatch):
    betas = H.geometric(0.2, 1.0, 32)
    a = T.Ensemble(T.Model.lattice((16, 16)), betas, seed=4)
    g = O.lattice_graph((16, 16))
    mg = T.Model.graph(g.n, g.ci, g.cj, g.J)
    monkeypatch.setenv("TAPT_K3", "1")
    b = T.Ensemble(mg, betas, seed=4)
    assert a.kernel == "lattice" and b.kernel == "bitcsr"
    for e in (a, b):
        e.init_random()
        e.run(50, swap_every=1)
    monkeypatch.setenv("TAPT_K3", "0")
    c = T.Ensemble(mg, betas, seed=4)
    assert c.kernel == "csr"
    c.init_random()
    c.run(50, swap_every=1)
    for e in (b, c):
        assert np.array_equal(a.spins(), e.spins())
        assert np.array_equal(a.energies(), e.energies())


@pytest.mark.parametrize("dims,R", [((16,), 64), ((32, 32), 32), ((16, 16), 40)])
def test_k1_group_width_does_not_change_the_chain(monkeypatch, dims, R):
    """Narrow replica groups (16 or 8 replicas per CTA, clusters of up to 8 CTAs; chosen when the
    instances are fewer than the SMs) give the same chain, counters, observables and histograms as
    32-replica groups, and the oracle."""
    betas = H.linear(0.2, 3.0, R)

    def run(w):
        monkeypatch.setenv("TAPT_K1_W", str(w))
        e = T.Ensemble(T.Model.lattice(dims), betas, n_instances=3, seed=21)
        assert e.kernel == "lattice"
        if len(dims) == 1:
            e.generate_ea_disorder(4)
        e.init_random()
        n = e.n
        e.set_histogram(-3 * n, 16, 3 * n // 8)
        e.run(17, swap_every=1, measure_every=3)
        e.generate_proposals(np.arange(min(R, 20)), None, refine=2)
        e.run(13, swap_every=2, measure_every=2)
        return e
    ref = run(32)
    for w in (16, 8):
        e = run(w)
        for x, y in zip((ref.spins(), ref.energies(), ref.permutation(), ref.observables(), ref.histogram(), ref.best()),
                        (e.spins(), e.energies(), e.permutation(), e.observables(), e.histogram(), e.best())):
            assert np.array_equal(x, y)
        for x, y in zip(ref.acceptance(), e.acceptance()):
            assert np.array_equal(x, y)
    monkeypatch.delenv("TAPT_K1_W")


@pytest.mark.parametrize("dims,R,w,packed", [((16,), 64, 16, 2), ((16,), 64, 8, 4), ((4,), 32, 16, 2), ((8,), 16, 8, 4),
                                              ((8, 8), 32, 8, 4), ((64, 4), 32, 16, 2), ((4,), 16, 8, 0),
                                              ((16, 16), 40, 16, 0)])
def test_k1_packed_narrow_groups_match_the_oracle(monkeypatch, dims, R, w, packed):
    """Narrow groups fold the lattice along its slowest dimension and keep 32/W sites per word (the
    launch log's last template argument); seam neighbours, per-field draw counters, bond bytes, energies
    and magnetisations must give the oracle's chain.  Lattices whose fold would hold an odd number of
    planes, and ladders with a partial last group, keep one site per word."""
    monkeypatch.setenv("TAPT_K1_W", str(w))
    betas = H.linear(0.2, 2.5, R)
    I = 2
    e = T.Ensemble(T.Model.lattice(dims), betas, n_instances=I, seed=91, instance_offset=3)
    three_d = len(dims) == 1
    if three_d:
        e.generate_ea_disorder(7)
        graphs = [O.ea_graph(dims, 7, 3 + k) for k in range(I)]
    else:
        graphs = [O.lattice_graph(dims)] * I
    e.init_random()
    e.run(25, swap_every=1, measure_every=5)
    names = [x.split(" ")[0] for x in e.launch_log() if x.startswith("k1_lattice_pt<")]
    if packed:
        assert any(x.count(",") == 8 and x.endswith(f",{packed}>") for x in names), names
    else:
        assert all(x.count(",") == 7 for x in names), names
    pts = H.run_oracle(graphs, betas, 91, 3, H.checkerboard_order(dims), 25, measure_every=5)
    compare(e, pts)
    for k in range(I):
        obs = e.observables()[k]
        for j, key in enumerate(("cnt", "sumE", "sumE2", "sumAbsM", "sumM2")):
            assert np.array_equal(obs[:, j], pts[k].meas[key]), (k, key)


@pytest.mark.parametrize("fuzz_seed", [20251021, 7, 99] + [1000 + k for k in range(int(os.environ.get("TAPT_FUZZ_EXTRA", "0")))])
def test_k1_random_shapes_widths_and_threads_match_the_oracle(monkeypatch, fuzz_seed):
    """Seeded sweep over lattice shapes, ladder lengths, group widths and thread counts (packed and
    unpacked narrow groups, partial groups, clusters, proposal rounds): every run equals the oracle."""
    rs = np.random.default_rng(fuzz_seed)
    shapes = [(4,), (8,), (16,), (4, 4), (8, 8), (16, 8), (8, 32), (32, 32), (64, 16)]
    for case in range(24):
        dims = shapes[rs.integers(len(shapes))]
        R = int(rs.choice([5, 8, 16, 24, 32, 40, 48, 64]))
        w = int(rs.choice([8, 16, 32]))
        if (R + w - 1) // w > 8:
            w = 32
        threads = rs.choice(["", "128", "256", "512"])
        monkeypatch.setenv("TAPT_K1_W", str(w))
        if threads:
            monkeypatch.setenv("TAPT_K1_THREADS", threads)
        else:
            monkeypatch.delenv("TAPT_K1_THREADS", raising=False)
        I, seed, off = int(rs.integers(1, 4)), int(rs.integers(1, 1000)), int(rs.integers(0, 50))
        betas = H.linear(0.15, 2.0, R)
        e = T.Ensemble(T.Model.lattice(dims), betas, n_instances=I, seed=seed, instance_offset=off)
        if len(dims) == 1:
            e.generate_ea_disorder(seed + 1)
            graphs = [O.ea_graph(dims, seed + 1, off + k) for k in range(I)]
        else:
            graphs = [O.lattice_graph(dims)] * I
        e.init_random()
        nt = int(min(R, rs.choice([3, 8, 16, 20])))
        mb = np.full(R, 0.3)
        for _ in range(2):
            e.run(7, swap_every=1, measure_every=2)
            e.generate_proposals(np.arange(nt), mb[:nt], refine=2)
        pts = H.run_oracle(graphs, betas, seed, off, H.checkerboard_order(dims), 14, measure_every=2,
                           props=dict(every=7, targets=nt, m_bias=mb, refine=2))
        try:
            compare(e, pts)
            for k in range(I):
                obs = e.observables()[k]
                for j, key in enumerate(("cnt", "sumE", "sumE2", "sumAbsM", "sumM2")):
                    assert np.array_equal(obs[:, j], pts[k].meas[key]), key
        except AssertionError as err:
            raise AssertionError(f"case {case}: dims={dims} R={R} W={w} threads={threads!r} I={I} nt={nt}: {err}\n"
                                 f"{e.launch_log()}") from err
    monkeypatch.delenv("TAPT_K1_W")


def test_k1_automatic_group_width_for_few_instances(monkeypatch):
    """Few instances (4 x 64 slots on a 16^3 lattice: 8 groups of 32 < SMs) take narrower groups
    automatically; the chain equals the 32-replica one."""
    betas = H.linear(0.2, 3.0, 64)

    def run(w):
        if w is None:
            monkeypatch.delenv("TAPT_K1_W", raising=False)
        else:
            monkeypatch.setenv("TAPT_K1_W", str(w))
        e = T.Ensemble(T.Model.lattice((16,)), betas, n_instances=4, seed=33)
        e.generate_ea_disorder(2)
        e.init_random()
        e.run(30, swap_every=1, measure_every=5)
        return e
    a, b = run(32), run(None)
    for x, y in zip((a.spins(), a.energies(), a.permutation(), a.observables()),
                    (b.spins(), b.energies(), b.permutation(), b.observables())):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("ipb", [1, 2, 3, 4])
def test_k3_teams_per_cta_do_not_change_the_chain(monkeypatch, ipb):
    """1-4 instance teams per CTA (named barriers, shared staged graph) give the same chain."""
    M = T.Multiplier(8)
    m = M.model()
    I, R = 10, 32
    prods = [T.random_semiprime(3, k, 8) for k in range(I)]
    cl = np.stack([M.clamps(p * q) for p, q in prods])

    def run(v):
        monkeypatch.setenv("TAPT_K3_IPB", str(v))
        e = T.Ensemble(m, H.geometric(0.1, 5.0, R), n_instances=I, seed=12)
        assert e.kernel == "bitcsr"
        e.set_clamps(cl)
        e.init_random()
        e.run(35, swap_every=1, measure_every=4)
        return e
    a, b = run(1), run(ipb)
    for x, y in zip((a.spins(), a.energies(), a.permutation(), a.observables(), a.best()),
                    (b.spins(), b.energies(), b.permutation(), b.observables(), b.best())):
        assert np.array_equal(x, y)
    monkeypatch.delenv("TAPT_K3_IPB")


def test_k3_circuit_with_clamps_and_fields_matches_oracle(monkeypatch):
    monkeypatch.setenv("TAPT_K3", "1")
    g = _random_circuit(13)
    m = T.Model.graph(g.n, g.ci, g.cj, g.J, g.h, g.clamp)
    betas = H.geometric(0.1, 5.0, 32)
    e = T.Ensemble(m, betas, n_instances=3, seed=5)
    assert e.kernel == "bitcsr"
    e.init_random()
    e.run(120, swap_every=1)
    compare(e, H.run_oracle([g] * 3, betas, 5, 0, H.colour_order_for(m.schedule()[0]), 120))


def test_k3_equals_k2_on_multiplier_instances(monkeypatch):
    """K3 (bit-sliced, heavy sites, per-instance clamps, swaps, measurements) == K2, bit for bit."""
    M = T.Multiplier(12)
    m = M.model()
    I, R = 64, 32
    prods = [T.random_semiprime(4, k, 12) for k in range(I)]
    cl = np.stack([M.clamps(p * q) for p, q in prods])

    def run(k3):
        monkeypatch.setenv("TAPT_K3", "1" if k3 else "0")
        e = T.Ensemble(m, H.geometric(0.1, 5.0, R), n_instances=I, seed=8)
        e.set_clamps(cl)
        e.init_random()
        e.set_histogram(-2000, 16, 256)
        e.run(150, swap_every=1, measure_every=7)
        return e
    a, b = run(True), run(False)
    assert a.kernel == "bitcsr" and b.kernel == "csr"
    assert np.array_equal(a.spins(), b.spins())
    assert np.array_equal(a.energies(), b.energies())
    for x, y in zip(a.acceptance(), b.acceptance()):
        assert np.array_equal(x, y)
    assert np.array_equal(a.observables(), b.observables())
    assert np.array_equal(a.histogram(), b.histogram())
    assert np.array_equal(a.best(), b.best())


@pytest.mark.parametrize("q", [2, 4])
def test_k3_split_sites_equal_k2_on_multiplier_instances(monkeypatch, q):
    """K3 with Q lanes per site (split sites: shuffled decision words, integer energy deltas) == K2,
    bit for bit: heavy sites, per-instance clamps, swaps, measurements, histograms, best."""
    M = T.Multiplier(12)
    m = M.model()
    I, R = 40, 32
    prods = [T.random_semiprime(4, k, 12) for k in range(I)]
    cl = np.stack([M.clamps(p * q_) for p, q_ in prods])

    def run(k3):
        monkeypatch.setenv("TAPT_K3", "1" if k3 else "0")
        monkeypatch.setenv("TAPT_K3_Q", str(q))
        e = T.Ensemble(m, H.geometric(0.1, 5.0, R), n_instances=I, seed=8)
        e.set_clamps(cl)
        e.init_random()
        e.set_histogram(-2000, 16, 256)
        e.run(150, swap_every=1, measure_every=7)
        return e
    a, b = run(True), run(False)
    assert a.kernel == "bitcsr" and b.kernel == "csr"
    assert any(f"k3_bitcsr_pt<0,1,{q}>" in k for k in a.launch_log())
    assert np.array_equal(a.spins(), b.spins())
    assert np.array_equal(a.energies(), b.energies())
    for x, y in zip(a.acceptance(), b.acceptance()):
        assert np.array_equal(x, y)
    assert np.array_equal(a.observables(), b.observables())
    assert np.array_equal(a.histogram(), b.histogram())
    assert np.array_equal(a.best(), b.best())


@pytest.mark.parametrize("q", [2, 4])
def test_k3_split_sites_circuit_with_partial_group_matches_oracle(monkeypatch, q):
    """Split sites with 20 slots (12 idle lanes of the replica word) on a random circuit with
    clamps and fields, against the oracle."""
    monkeypatch.setenv("TAPT_K3", "1")
    monkeypatch.setenv("TAPT_K3_Q", str(q))
    g = _random_circuit(17)
    m = T.Model.graph(g.n, g.ci, g.cj, g.J, g.h, g.clamp)
    betas = H.geometric(0.1, 5.0, 20)
    e = T.Ensemble(m, betas, n_instances=3, seed=6)
    assert e.kernel == "bitcsr"
    e.init_random()
    e.run(90, swap_every=1)
    compare(e, H.run_oracle([g] * 3, betas, 6, 0, H.colour_order_for(m.schedule()[0]), 90))


def test_k3_split_sites_balanced_schedule(monkeypatch):
    """Q = 4 teams under the balanced persistent schedule (more instances than resident teams,
    jobs split between teams) give the unbalanced chain."""
    M = T.Multiplier(8)
    m = M.model()
    I, R = 230, 32
    prods = [T.random_semiprime(3, k, 8) for k in range(I)]
    cl = np.stack([M.clamps(p * q) for p, q in prods])

    def run(bal):
        monkeypatch.setenv("TAPT_K3_Q", "4")
        monkeypatch.setenv("TAPT_BALANCE", "1" if bal else "0")
        e = T.Ensemble(m, H.geometric(0.1, 5.0, R), n_instances=I, seed=21)
        e.set_clamps(cl)
        e.init_random()
        e.run(60, swap_every=1, measure_every=6)
        return e
    a, b = run(True), run(False)
    assert any("k3_bitcsr_pt<1,1,4>" in k for k in a.launch_log())
    for x, y in zip((a.spins(), a.energies(), a.permutation(), a.observables(), a.best()),
                    (b.spins(), b.energies(), b.permutation(), b.observables(), b.best())):
        assert np.array_equal(x, y)


# ------------------------------------------------------------ proposals -----

def test_synthetic_tapt_rounds_match_oracle_k1():
    """Config 2 style: biased i.i.d. proposals + 5 refinement sweeps + Eq. 2, every 20 sweeps."""
    R = 16
    betas = H.geometric(0.3, 0.6, R)
    mb = np.array([O.yang_m(b) for b in betas])
    targets = np.arange(12)
    m = T.Model.lattice((16, 16))
    e = T.Ensemble(m, betas, n_instances=2, seed=77, instance_offset=5)
    e.init_random()
    for _ in range(6):
        e.run(20, swap_every=1)
        e.generate_proposals(targets, mb[:12], refine=5)
    pts = H.run_oracle([O.lattice_graph((16, 16))] * 2, betas, 77, 5, H.checkerboard_order((16, 16)), 120,
                       props=dict(every=20, targets=12, m_bias=mb, refine=5))
    compare(e, pts)
    assert e.acceptance()[3].sum() > 0


@pytest.mark.parametrize("dims,nt", [((16, 16), 16), ((16, 16), 8), ((8,), 16), ((8,), 8)])
def test_tapt_rounds_with_packed_proposal_groups(dims, nt):
    """16 or 8 targets: the proposal group is a full narrow group, so its energy evaluation and refinement
    sweeps run on the folded lattice (2 / 4 sites per word); the R = 16 main group is packed too."""
    R = 16
    betas = H.geometric(0.3, 0.9, R)
    mb = np.array([O.yang_m(b) for b in betas])
    e = T.Ensemble(T.Model.lattice(dims), betas, n_instances=2, seed=78, instance_offset=2)
    if len(dims) == 1:
        e.generate_ea_disorder(9)
        graphs = [O.ea_graph(dims, 9, 2 + k) for k in range(2)]
    else:
        graphs = [O.lattice_graph(dims)] * 2
    e.init_random()
    for _ in range(4):
        e.run(10, swap_every=1)
        e.generate_proposals(np.arange(nt), mb[:nt], refine=3)
    names = [x.split(" ")[0] for x in e.launch_log() if x.startswith("k1_lattice_pt<")]
    assert any(x.count(",") == 8 and x.endswith(f",{32 // nt}>") for x in names), names  # the proposal groups
    assert any(x.count(",") == 8 and x.endswith(",2>") for x in names), names             # the 16-slot ladder
    pts = H.run_oracle(graphs, betas, 78, 2, H.checkerboard_order(dims), 40,
                       props=dict(every=10, targets=nt, m_bias=mb, refine=3))
    compare(e, pts)


def test_synthetic_tapt_reference_order_matches_reference_golden():
    f = np.load(os.path.join(GOLD, "pt_tapt2d16.npz"))
    I, R, n = (int(x) for x in f["shape"])
    m = T.Model.lattice((16, 16))
    e = T.Ensemble(m, f["betas"], n_instances=I, seed=int(f["seed"]), instance_offset=int(f["gid0"]),
                   order="reference")
    e.init_random()
    every, nt = int(f["prop_every"]), int(f["n_targets"])
    for _ in range(int(f["n_sweeps"]) // every):
        e.run(every, swap_every=1)
        e.generate_proposals(np.arange(nt), f["m_bias"][:nt], refine=int(f["refine"]))
    spins = unpack(f["spins"], I * R * n).reshape(I, R, n)
    assert np.array_equal(e.spins(), spins)
    assert np.array_equal(e.energies().astype(np.float64), f["E"])
    assert np.array_equal(e.acceptance()[3], f["prop_acc"])


def test_ea_fair_proposals_match_reference_golden():
    f = np.load(os.path.join(GOLD, "pt_ea3d6_tapt.npz"))
    I, R, n = (int(x) for x in f["shape"])
    graphs = [O.ea_graph((6,), 3, k) for k in range(I)]
    # per-instance couplings through bond signs on a lattice model (L=6: K2 path)
    m = T.Model.lattice((6,))
    e = T.Ensemble(m, f["betas"], n_instances=I, seed=int(f["seed"]), order="reference")
    e.generate_ea_disorder(3)
    e.init_random()
    every, nt = int(f["prop_every"]), int(f["n_targets"])
    for _ in range(int(f["n_sweeps"]) // every):
        e.run(every, swap_every=1)
        e.generate_proposals(np.arange(nt), None, refine=int(f["refine"]))
    spins = unpack(f["spins"], I * R * n).reshape(I, R, n)
    assert np.array_equal(e.spins(), spins)
    assert np.array_equal(e.energies().astype(np.float64), f["E"])
    del graphs


def test_inject_host_proposals_int8_and_packed():
    R = 8
    betas = H.linear(0.3, 1.5, R)
    g = O.lattice_graph((8, 8))
    m = T.Model.lattice((8, 8))
    rs = np.random.default_rng(0)
    e = T.Ensemble(m, betas, n_instances=2, seed=21)
    e.init_random()
    e.run(10, swap_every=1)
    pts = H.run_oracle([g] * 2, betas, 21, 0, H.checkerboard_order((8, 8)), 10)
    targets = np.array([0, 2, 3, 5])
    props = rs.choice(np.array([-1, 1], np.int8), size=(2, 4, 64))
    acc = e.inject_proposals(props, targets)
    for k, pt in enumerate(pts):
        full = np.zeros((R, 64), np.int8)
        Ep = np.zeros(R, np.int64)
        mask = np.zeros(R, np.uint8)
        for t, r in enumerate(targets):
            full[r] = props[k, t]
            Ep[r] = O.lib().oc_energy(g.oc(), full[r].ctypes.data_as(O._i8p))
            mask[r] = 1
        dec = pt.inject(mask, full, Ep)
        assert np.array_equal(acc[k], (dec[targets] == 1).astype(np.uint8))
    compare(e, pts)
    # packed path, second round
    props2 = rs.choice(np.array([-1, 1], np.int8), size=(2, 4, 64))
    packed = np.packbits(props2 > 0, axis=-1, bitorder="little")
    acc2 = e.inject_proposals_packed(packed, targets)
    for k, pt in enumerate(pts):
        full = np.zeros((R, 64), np.int8)
        Ep = np.zeros(R, np.int64)
        mask = np.zeros(R, np.uint8)
        for t, r in enumerate(targets):
            full[r] = props2[k, t]
            Ep[r] = O.lib().oc_energy(g.oc(), full[r].ctypes.data_as(O._i8p))
            mask[r] = 1
        dec = pt.inject(mask, full, Ep)
        assert np.array_equal(acc2[k], (dec[targets] == 1).astype(np.uint8))
    compare(e, pts)


@pytest.mark.parametrize("host_path", [False, True])
def test_inject_mh_corrected(monkeypatch, host_path):
    """mh_corrected_move: the device decisions (device exp with a 1e-12 tie band) and
    the glibc host decisions (TAPT_MH_HOST forces the tie fallback) both equal the oracle's."""
    if host_path:
        monkeypatch.setenv("TAPT_MH_HOST", "1")
    R = 6
    betas = H.linear(0.5, 2.0, R)
    g = O.lattice_graph((8, 8))
    m = T.Model.lattice((8, 8))
    rs = np.random.default_rng(1)
    e = T.Ensemble(m, betas, n_instances=1, seed=3)
    e.init_random()
    pts = H.run_oracle([g], betas, 3, 0, H.checkerboard_order((8, 8)), 0)
    for _ in range(5):
        targets = np.array([0, 1, 4])
        props = rs.choice(np.array([-1, 1], np.int8), size=(1, 3, 64))
        lqc, lqp = rs.normal(size=(1, 3)) * 3, rs.normal(size=(1, 3)) * 3
        acc = e.inject_proposals(props, targets, lqc, lqp)
        full = np.zeros((R, 64), np.int8)
        Ep = np.zeros(R, np.int64)
        mask = np.zeros(R, np.uint8)
        a = np.zeros(R)
        b = np.zeros(R)
        for t, r in enumerate(targets):
            full[r] = props[0, t]
            Ep[r] = O.lib().oc_energy(g.oc(), full[r].ctypes.data_as(O._i8p))
            mask[r] = 1
            a[r], b[r] = lqc[0, t], lqp[0, t]
        dec = pts[0].inject(mask, full, Ep, a, b)
        assert np.array_equal(acc[0], (dec[targets] == 1).astype(np.uint8))
    compare(e, pts)


# ------------------------------------------------------- full-size properties --

def test_cfg5_full_size_energy_consistency_and_determinism():
    """Config 5 geometry (3D L=32, 64 slots, cluster of 2) on a slice of instances:
    device energies == exact recomputation, permutation valid, run is deterministic and
    chunking-invariant (size-independent properties)."""
    L, R, I = 32, 64, 4
    betas = H.linear(0.2, 3.0, R)
    m = T.Model.lattice((L,))
    a = T.Ensemble(m, betas, n_instances=I, seed=99, instance_offset=1000)
    b = T.Ensemble(m, betas, n_instances=I, seed=99, instance_offset=1000)
    for e in (a, b):
        e.generate_ea_disorder(42)
        e.init_random()
    a.run(40, swap_every=1)
    b.run(15, swap_every=1)
    b.run(25, swap_every=1)
    S, E = a.spins(), a.energies()
    assert np.array_equal(S, b.spins()) and np.array_equal(E, b.energies())
    n, ci, cj, _ = O.lattice_couplings((L,), 1.0, True)
    signs = a.bond_signs(len(ci)).astype(np.int64)
    for k in range(I):
        s = S[k].astype(np.int64)
        Ek = -(signs[k][None, :] * s[:, ci] * s[:, cj]).sum(axis=1)
        assert np.array_equal(Ek, E[k])
        perm = a.permutation()[k]
        assert sorted(perm.tolist()) == list(range(R))
    # instance sharding: the last two instances computed alone give the same result
    c = T.Ensemble(m, betas, n_instances=2, seed=99, instance_offset=1002)
    c.generate_ea_disorder(42)
    c.init_random()
    c.run(40, swap_every=1)
    assert np.array_equal(c.spins(), S[2:])


# ------------------------------------------------------- factorization circuits --

def _mult_graph(M, clamp):
    return O.Graph.from_couplings(M.n_spins, M.ci, M.cj, M.J, M.h, clamp)


def test_multiplier_pt_per_instance_clamps_bit_exact():
    """Config 4 shape at n=8: colour-class K2 sweeps + swaps, each instance its own semiprime."""
    M = T.Multiplier(8)
    m = M.model()
    prods = [T.random_semiprime(5, k, 8) for k in range(3)]
    clamps = np.stack([M.clamps(p * q) for p, q in prods])
    betas = H.geometric(0.1, 5.0, 32)
    e = T.Ensemble(m, betas, n_instances=3, seed=8)
    e.set_clamps(clamps)
    e.init_random()
    e.run(200, swap_every=1)
    colours, _ = m.schedule()
    graphs = [_mult_graph(M, clamps[k]) for k in range(3)]
    pts = H.run_oracle(graphs, betas, 8, 0, H.colour_order_for(colours), 200)
    compare(e, pts)
    S = e.spins()
    for k in range(3):                       # clamped wires hold their values in every slot
        nz = np.nonzero(clamps[k])[0]
        assert np.all(S[k][:, nz] == clamps[k][nz])


def test_multiplier_forward_mode_samples_the_product():
    """SPEC.md:540 forward check: n=4, A=0110, B=0101 clamped -> C reads 30.  (With the
    penalty-derived full adder the gate gap is 2, so plain Gibbs at beta=3 is not enough; PT
    over a 16-slot ladder up to beta=5 is used and the coldest slot must read 30 in >= 90%
    of 64 independent runs.)"""
    M = T.Multiplier(4)
    cl = np.zeros(M.n_spins, np.int8)
    for i in range(4):
        cl[M.A[i]] = 1 if (6 >> i) & 1 else -1
        cl[M.B[i]] = 1 if (5 >> i) & 1 else -1
    cl[M.carry] = -1
    m = T.Model.graph(M.n_spins, M.ci, M.cj, M.J, M.h, cl)
    e = T.Ensemble(m, H.geometric(0.5, 5.0, 16), n_instances=64, seed=123)
    e.init_random()
    e.run(2000, swap_every=1)
    S = e.spins()[:, -1, :]
    prod = ((S[:, M.C] > 0) * (1 << np.arange(8))).sum(axis=1)
    assert (prod == 30).mean() >= 0.90


def test_factorization_finds_factors_4bit():
    """Inverse mode (8-bit products, section 5.2): C = 11*13 = 143 clamped; PT over 32
    slots finds A*B = C in the coldest slots for most of 16 independent seeds.  (The 16-bit
    product 44969 = 193*233 is hard: the paper reports 7% PT success in 1e4 sweeps.)"""
    M = T.Multiplier(4)
    m = M.model()
    C = 11 * 13
    e = T.Ensemble(m, H.geometric(0.1, 5.0, 32), n_instances=16, seed=2)
    e.set_clamps(np.stack([M.clamps(C)] * 16))
    e.init_random()
    found = np.zeros(16, bool)
    for _ in range(10):
        e.run(500, swap_every=1)
        S = e.spins()
        for k in range(16):
            found[k] |= any(M.decode(S[k][r], C)[2] for r in range(26, 32))
    assert found.mean() >= 0.75


# ------------------------------------------------------------- statistical tier --

def _per_slot_means(e, n):
    obs = e.observables().astype(np.float64)          # [I][R][5]
    cnt = obs[:, :, 0]
    return obs[:, :, 1] / cnt / n, obs[:, :, 3] / cnt / n   # <E>/N, <|m|> per instance and slot


def test_checkerboard_vs_reference_order_statistics_cfg1():
    """Config 1: per-beta <E>/N and <|m|> of the checkerboard chain (K1) agree with the
    reference's index-ascending chain (K2 level schedule, bit-exact with the unmodified
    gibbs_sweep) within 4 sigma over S = 16 independent seeds each (SURVEY 8c statistical
    tier; 4 sigma because 64 comparisons are made)."""
    betas = H.geometric(0.2, 1.0, 32)
    m = T.Model.lattice((32, 32))
    out = {}
    for order, off in (("colour", 0), ("reference", 1000)):
        e = T.Ensemble(m, betas, n_instances=16, seed=77, instance_offset=off, order=order)
        e.init_random()
        e.run(10000, swap_every=1, measure_every=1, measure_from=5000)
        out[order] = _per_slot_means(e, 1024)
    for k in range(2):
        a, b = out["colour"][k], out["reference"][k]
        se = np.sqrt(a.var(axis=0, ddof=1) / 16 + b.var(axis=0, ddof=1) / 16) + 1e-6
        z = np.abs(a.mean(axis=0) - b.mean(axis=0)) / se
        assert z.max() < 4.0, (k, z.max(), int(z.argmax()))


def test_pt_stationarity_small_system():
    """3x3 open ferromagnet, 4 replicas beta in [0.1, 1.0]: the coldest replica's
    state distribution matches Boltzmann(beta_max) within TV 0.02 (4096 independent ensembles,
    20 samples each, spaced 50 sweeps apart after 500 sweeps of equilibration)."""
    import itertools
    g = O.lattice_graph((3, 3), 1.0, False)
    m = T.Model.lattice((3, 3), 1.0, periodic=False)
    betas = np.array([0.1, 0.4, 0.7, 1.0])
    e = T.Ensemble(m, betas, n_instances=4096, seed=5)
    e.init_random()
    e.run(500, swap_every=1)
    counts = np.zeros(512)
    w = 1 << np.arange(9)
    for _ in range(20):
        e.run(50, swap_every=1)
        S = e.spins()[:, -1, :]
        np.add.at(counts, ((S > 0) * w).sum(axis=1), 1)
    states = np.array(list(itertools.product([-1, 1], repeat=9)))[:, ::-1]
    idx = ((states > 0) * w).sum(axis=1)
    E = np.array([O.lib().oc_energy(g.oc(), np.ascontiguousarray(s, np.int8).ctypes.data_as(O._i8p))
                  for s in states], np.float64)
    p = np.zeros(512)
    p[idx] = np.exp(-1.0 * (E - E.min()))
    p /= p.sum()
    tv = 0.5 * np.abs(counts / counts.sum() - p).sum()
    assert tv < 0.02, tv


def _circuit_stationarity(model, clamp, betas, slot, k3):
    """TV distance between the empirical distribution of slot `slot` (4096 independent ensembles,
    40 samples each, 25 sweeps apart after 400) and Boltzmann(betas[slot]) over the free spins."""
    import itertools
    import os as _os
    _os.environ["TAPT_K3"] = "1" if k3 else "0"
    try:
        e = T.Ensemble(model, betas, n_instances=4096, seed=8)
        assert e.kernel == ("bitcsr" if k3 else "csr")
        e.init_random()
        e.run(400, swap_every=1)
        free = np.where(clamp == 0)[0]
        w = 1 << np.arange(len(free))
        counts = np.zeros(1 << len(free))
        for _ in range(40):
            e.run(25, swap_every=1)
            S = e.spins()[:, slot, :][:, free]
            np.add.at(counts, ((S > 0) * w).sum(axis=1), 1)
    finally:
        _os.environ.pop("TAPT_K3", None)
    p = np.zeros_like(counts)
    base = clamp.astype(np.int8).copy()
    for bits in itertools.product([-1, 1], repeat=len(free)):
        st = base.copy()
        st[free] = bits
        p[((np.array(bits) > 0) * w).sum()] = -betas[slot] * model.energy(st)
    p = np.exp(p - p.max())
    p /= p.sum()
    return 0.5 * np.abs(counts / counts.sum() - p).sum()


@pytest.mark.parametrize("k3", [True, False])
def test_pt_stationarity_clamped_circuits(k3):
    """Colour-class PT on circuits with fields and clamps is stationary: the 2x2-bit multiplier with
    its product clamped to 6 (8 free spins) and a 10-spin graph whose hub has S' = sum|J| + |h| = 20
    (K3's heavy path), both within TV 0.02 of Boltzmann at two ladder slots.  Measured TV is
    0.003-0.006; sampling the neighbouring slot's beta would give 0.08-0.15, a 5 % beta error ~0.03."""
    M = T.Multiplier(2)
    cl = M.clamps(6)
    mm = T.Model.graph(M.n_spins, M.ci, M.cj, M.J, M.h, cl)
    betas = np.linspace(0.1, 1.0, 8)
    for slot in (4, 7):
        tv = _circuit_stationarity(mm, cl, betas, slot, k3)
        assert tv < 0.02, ("multiplier", slot, tv)
    rs = np.random.default_rng(4)
    n = 10
    ci = [0] * 9 + list(rs.integers(1, n, 8))
    cj = list(range(1, 10)) + list(rs.integers(1, n, 8))
    keep = [i != j for i, j in zip(ci, cj)]
    ci = np.array(ci)[keep]
    cj = np.array(cj)[keep]
    J = np.concatenate([np.where(np.arange(9) % 2 == 0, 2.0, -2.0), rs.choice([-1.0, 1.0], len(ci) - 9)])
    h = rs.integers(-2, 3, n).astype(float)
    h[0] = 2.0
    cl0 = np.zeros(n, np.int8)
    mh = T.Model.graph(n, ci, cj, J, h, cl0)
    betas = np.linspace(0.1, 0.8, 8)
    for slot in (3, 7):
        tv = _circuit_stationarity(mh, cl0, betas, slot, k3)
        assert tv < 0.02, ("hub graph", slot, tv)


# ------------------------------------------------------- annealing --

def test_estimate_ground_energy_ferromagnet_and_small_glass():
    m = T.Model.lattice((16, 16))
    best = T.estimate_ground_energy(m, restarts=8, sweeps=2000, seed=1)
    assert best[0] == -2 * 256                      # ferromagnet: -|edges| J recovered exactly
    # 3x4 open +-J glass: best of 8 restarts equals the brute-force ground energy
    rs = np.random.default_rng(3)
    n, ci, cj, _ = O.lattice_couplings((3, 4), 1.0, False)
    J = rs.choice([-1.0, 1.0], len(ci))
    g = O.Graph.from_couplings(n, ci, cj, J)
    mg = T.Model.graph(n, ci, cj, J)
    states = ((np.arange(2 ** n)[:, None] >> np.arange(n)) & 1) * 2 - 1
    E = -(J[None, :] * states[:, ci] * states[:, cj]).sum(1)
    best = T.estimate_ground_energy(mg, restarts=8, sweeps=1000, seed=2)
    assert best[0] == E.min()
    del g


# ------------------------------------------------------- training corpus (mcmc.cpp:67-84) --

def test_generate_training_corpus_matches_reference_golden():
    f = np.load(os.path.join(GOLD, "corpus_2d8clamped.npz"))
    cl = np.zeros(64, np.int8)
    cl[:8] = [1, 1, -1, -1, 1, -1, 1, -1]
    g = O.lattice_graph((8, 8), 1.0, False, cl)
    m = T.Model.graph(g.n, g.ci, g.cj, g.J, None, cl)
    b, S = T.generate_training_corpus(m, f["betas"], int(f["per_beta"]), int(f["mixing"]), int(f["thinning"]),
                                      int(f["seed"]))
    shape = tuple(int(x) for x in f["shape"])
    assert np.array_equal(S, unpack(f["spins"], shape[0] * shape[1]).reshape(shape))
    assert np.array_equal(b, np.repeat(f["betas"], int(f["per_beta"])))


# ------------------------------------------------- proposal-path stationarity --

def _five_spin():
    ci = [0, 0, 1, 1, 2, 3, 0]
    cj = [1, 2, 2, 3, 4, 4, 4]
    J = [1.0, -1.0, 2.0, 1.0, -1.0, 1.0, 1.0]
    h = [0.0, 1.0, 0.0, -1.0, 0.0]
    return O.Graph.from_couplings(5, ci, cj, J, h), (ci, cj, J, h)


def _boltzmann5(g, beta):
    import itertools
    states = np.array(list(itertools.product([-1, 1], repeat=5)), np.int8)
    E = np.array([O.lib().oc_energy(g.oc(), np.ascontiguousarray(s).ctypes.data_as(O._i8p)) for s in states], float)
    p = np.exp(-beta * (E - E.min()))
    return states, p / p.sum()


def _run_independence_sampler(mh, bias):
    """Per round: one Gibbs sweep (preserves Boltzmann, provides mixing) then three proposal
    rounds into every slot.  With uniform proposals Eq. 2 leaves Boltzmann invariant; with
    biased i.i.d. proposals only the MH-corrected rule does."""
    g, (ci, cj, J, h) = _five_spin()
    m = T.Model.graph(5, ci, cj, J, h)
    betas = np.array([0.5, 1.0, 1.5, 2.0])
    I = 4096
    e = T.Ensemble(m, betas, n_instances=I, seed=31)
    e.init_random()
    rs = np.random.default_rng(7)
    targets = np.arange(4)
    w = 1 << np.arange(5)
    counts = np.zeros((4, 32))
    for rnd in range(80):
        e.sweep(1)
        for _ in range(3):
            props = np.where(rs.random((I, 4, 5)) < bias, 1, -1).astype(np.int8)
            if mh:
                nplus_cur = (e.spins() > 0).sum(axis=2)
                lq_cur = nplus_cur * np.log(bias) + (5 - nplus_cur) * np.log(1 - bias)
                nplus = (props > 0).sum(axis=2)
                lq_prop = nplus * np.log(bias) + (5 - nplus) * np.log(1 - bias)
                e.inject_proposals(props, targets, lq_cur, lq_prop)
            else:
                e.inject_proposals(props, targets)
        if rnd >= 40:
            S = e.spins()
            for r in range(4):
                np.add.at(counts[r], ((S[:, r, :] > 0) * w).sum(axis=1), 1)
    tvs = []
    for r, b in enumerate(betas):
        states, p = _boltzmann5(g, b)
        idx = ((states > 0) * w).sum(axis=1)
        q = np.zeros(32)
        q[idx] = p
        tvs.append(0.5 * np.abs(counts[r] / counts[r].sum() - q).sum())
    return np.array(tvs)


def test_uniform_proposals_keep_boltzmann():
    assert _run_independence_sampler(False, 0.5).max() < 0.02


def test_mh_correction_removes_generator_bias():
    corrected = _run_independence_sampler(True, 0.8)
    biased = _run_independence_sampler(False, 0.8)
    assert corrected.max() < 0.02
    assert biased.max() > 2 * corrected.max() and biased.max() > 0.03   # Eq. 2 alone keeps the bias


@pytest.mark.parametrize("kernel", ["lattice", "csr"])
def test_tapt_rounds_with_two_proposal_groups(kernel):
    """56 targets (two 32-replica proposal groups, as in the config-5 bench) on a 64-slot ladder."""
    R, L = 64, 8
    betas = H.linear(0.2, 3.0, R)
    if kernel == "lattice":
        m = T.Model.lattice((L,))
    else:
        g0 = O.lattice_graph((L,))
        m = T.Model.graph(g0.n, g0.ci, g0.cj, g0.J)
    e = T.Ensemble(m, betas, n_instances=2, seed=12, instance_offset=3)
    assert e.kernel == kernel
    if kernel == "lattice":
        e.generate_ea_disorder(9)
        graphs = [O.ea_graph((L,), 9, 3 + k) for k in range(2)]
    else:
        graphs = [O.lattice_graph((L,))] * 2
    e.init_random()
    for _ in range(3):
        e.run(15, swap_every=1)
        e.generate_proposals(np.arange(56), None, refine=5)
    order = H.checkerboard_order((L,)) if kernel == "lattice" else H.colour_order_for(m.schedule()[0])
    pts = H.run_oracle(graphs, betas, 12, 3, order, 45, props=dict(every=15, targets=56, m_bias=np.zeros(R), refine=5))
    compare(e, pts)


# ---------------------------------------------- the headline kernel, exact --

def mcnaughton_split(I, S, M):
    """Jobs McNaughton's wrap-around rule (engine.cu mcnaughton()) cuts between two clusters."""
    total = I * S
    C = -(-total // M)
    return sorted({(k * C) // S for k in range(1, M) if k * C < total and (k * C) % S})


def _cfg5_oracle(gids, n1, n2, seed=20250923, disorder=43):
    betas = H.linear(0.2, 3.0, 64)
    out = []
    for gid in gids:
        g = O.ea_graph((32,), disorder, gid)
        pt = O.PT(g, betas, seed, gid, H.checkerboard_order((32,))(g))
        pt.run(n1, 1, n1, 56, None, 5)  # n1 sweeps (swap every sweep), then one TAPT round
        pt.run(n2, 1)
        out.append(pt)
    return out


def test_cfg5_headline_kernel_bit_exact_with_oracle():
    """bench.py's exact config-5 path at a size where every one of its code paths engages:
    3D EA L=32 (32768 sites -> cp.async.bulk state loads), 64 slots as a 2-CTA cluster of
    32-replica groups, more instances than co-resident clusters (-> the balanced McNaughton grid
    with split jobs), and a TAPT round (56 fair i.i.d. proposals, 5 refinement sweeps on the
    non-cluster bulk instantiation, Eq. 2).  Spins, energies, swap and proposal counters of the
    first instance, a split instance and the last instance equal the oracle."""
    L, R, I, S1, S2 = 32, 64, 160, 20, 20
    e = T.Ensemble(T.Model.lattice((L,)), H.linear(0.2, 3.0, R), n_instances=I, seed=20250923)
    e.generate_ea_disorder(43)
    e.init_random()
    e.run(S1, swap_every=1)
    e.generate_proposals(np.arange(56, dtype=np.uint32), None, refine=5, return_accepted=False)
    e.run(S2, swap_every=1)
    log = e.launch_log()
    head = [x for x in log if x.startswith("k1_lattice_pt<3,1,1,2,640,1,1,0> balanced M=")]
    assert head, log  # the bench's instantiation (3D, disorder, cluster, bulk) on the balanced grid
    assert any(x.startswith("k1_lattice_pt<3,1,0,2,640,1,1,0>") for x in log), log  # bulk refinement sweeps
    M = int(head[0].split("M=")[1])
    split = mcnaughton_split(I, S1, M)
    assert split, (I, S1, M)
    gids = [0, split[0], I - 1]
    pts = _cfg5_oracle(gids, S1, S2)
    S, E = e.spins(), e.energies()
    sa, sc, pa, pc = e.acceptance()
    for gid, pt in zip(gids, pts):
        assert np.array_equal(E[gid], pt.E), gid
        assert np.array_equal(S[gid], pt.spins), gid
        assert np.array_equal(sc[gid], pt.swap_acc[: R - 1]), gid
        assert np.array_equal(pc[gid], pt.prop_acc), gid


@pytest.mark.parametrize("threads,name", [(None, "k1_lattice_pt<3,1,1,2,640,1,1,0>"),
                                          (512, "k1_lattice_pt<3,1,1,2,512,1,1,0>"),
                                          (768, "k1_lattice_pt<3,1,1,2,768,1,0,1>")])
def test_cfg5_bulk_kernel_with_forced_full_groups(monkeypatch, threads, name):
    """Few instances: the group-width model would narrow the replica groups; TAPT_K1_W=32 forces
    the 32-replica bulk instantiation (plain grid, no balancing) and it must match the oracle.  The
    default launch shape (640 threads), the 512-thread bulk shape and the 768-thread shape all do."""
    monkeypatch.setenv("TAPT_K1_W", "32")
    if threads:
        monkeypatch.setenv("TAPT_K1_THREADS", str(threads))
    L, R, I = 32, 64, 2
    e = T.Ensemble(T.Model.lattice((L,)), H.linear(0.2, 3.0, R), n_instances=I, seed=20250923, instance_offset=7)
    e.generate_ea_disorder(43)
    e.init_random()
    e.run(12, swap_every=1)
    e.generate_proposals(np.arange(56, dtype=np.uint32), None, refine=5, return_accepted=False)
    e.run(12, swap_every=1)
    assert name in e.launch_log(), e.launch_log()
    pts = _cfg5_oracle([7, 8], 12, 12)
    compare(e, pts)


def _fair_proposals_host(seed, gids, targets, rnd, n):
    """The synthetic generator's fair i.i.d. proposals computed on the host (slot r of
    round q draws from derive(seed, {kReplica, gid, r, q+1}); site i: draw i+2, +1 iff the top bit
    is 0), packed LSB-first [I][T][ceil(n/8)]."""
    out = np.zeros((len(gids), len(targets), (n + 7) // 8), np.uint8)
    k = np.arange(2, n + 2, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for a, gid in enumerate(gids):
            for b, r in enumerate(targets):
                z = np.uint64(O.derive(seed, [0x22, gid, int(r), rnd + 1])) + k * np.uint64(O.PHI)
                z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
                z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
                z = z ^ (z >> np.uint64(31))
                up = ((z >> np.uint64(63)) == 0).astype(np.uint8)
                out[a, b] = np.packbits(up, bitorder="little")
    return out


def test_host_supplied_proposals_with_refinement_equal_the_synthetic_round():
    """tapt_inject_proposals_packed_refined (bench.py's e2e path: proposals from host memory, 5
    refinement sweeps at the target beta, Eq. 2) equals the on-device synthetic round when fed the
    same proposals -- spins, energies, acceptance decisions."""
    L, R, I, seed = 16, 64, 3, 5
    betas = H.linear(0.2, 3.0, R)
    targets = np.arange(40, dtype=np.uint32)
    a = T.Ensemble(T.Model.lattice((L,)), betas, n_instances=I, seed=seed, instance_offset=11)
    b = T.Ensemble(T.Model.lattice((L,)), betas, n_instances=I, seed=seed, instance_offset=11)
    for e in (a, b):
        e.generate_ea_disorder(3)
        e.init_random()
        e.run(7, swap_every=1)
    acc_a = a.generate_proposals(targets, None, refine=5)
    host = _fair_proposals_host(seed, [11, 12, 13], targets, 0, L ** 3)
    acc_b = b.inject_proposals_packed(host, targets, refine=5)
    assert np.array_equal(acc_a, acc_b)
    for e in (a, b):
        e.run(5, swap_every=1)
    assert np.array_equal(a.spins(), b.spins()) and np.array_equal(a.energies(), b.energies())
    assert acc_a.sum() > 0
