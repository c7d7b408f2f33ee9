"""The balanced persistent K1 schedule (McNaughton's wrap-around rule):
with more instances than co-resident clusters, split jobs run their first sweeps on one
cluster and their last sweeps on another.  Results must equal the plain one-instance-per-CTA
launch (TAPT_BALANCE=0) bit for bit -- spins, energies, permutations, swap and proposal
counters, observables, histograms, best energies -- and the oracle.  Marked `gpu`."""
import numpy as np
import pytest

import paper_2509_23043_b200 as T
from oracle import oracle as O
import tapt_helpers as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if T.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


def _state(e):
    return (e.spins(), e.energies(), e.permutation(), e.acceptance(), e.observables(), e.histogram(), e.best())


def _run(monkeypatch, balance, model, betas, I, ea=None, sweeps=(23, 41), clamps=None, k3=False):
    monkeypatch.setenv("TAPT_BALANCE", "1" if balance else "0")
    monkeypatch.setenv("TAPT_K3", "1" if k3 else "0")
    e = T.Ensemble(model, betas, n_instances=I, seed=17)
    if ea is not None:
        e.generate_ea_disorder(ea)
    if clamps is not None:
        e.set_clamps(clamps)
    e.init_random()
    e.set_histogram(-4 * model.n_spins, 8, 64)
    e.run(sweeps[0], swap_every=1, measure_every=3)
    e.generate_proposals(np.arange(8), None, refine=2)
    e.run(sweeps[1], swap_every=2, measure_every=5, measure_from=10)
    return e


def _circuit(seed=3, n=60):
    rs = np.random.default_rng(seed)
    ci, cj = rs.integers(0, n, 4 * n), rs.integers(0, n, 4 * n)
    keep = ci != cj
    J = rs.choice([-2.0, -1.0, 1.0, 2.0], 4 * n)[keep]
    h = rs.integers(-3, 4, n).astype(float)
    cl = np.zeros(n, np.int8)
    cl[:6] = 1  # clamped sites whose values vary per instance
    return T.Model.graph(n, ci[keep], cj[keep], J, h, cl), rs


@pytest.mark.parametrize("case", ["2d_no_cluster", "3d_ea_cluster", "k2_circuit_clamps", "k2_odd_ea",
                                  "k3_circuit_clamps"])
def test_balanced_schedule_equals_plain_launch(case, monkeypatch):
    # K1: 4096-site lattices (512-thread CTAs, one per SM); K2: 400 single-instance CTAs on
    # ~296 co-resident; K3: 700 instance teams on 148 x 4 -- I exceeds the co-resident count in
    # every case
    clamps, kern, k3 = None, "lattice", False
    if case == "2d_no_cluster":
        model, betas, I, ea = T.Model.lattice((64, 64)), H.geometric(0.2, 1.0, 32), 200, None
    elif case == "3d_ea_cluster":
        model, betas, I, ea = T.Model.lattice((16,)), H.linear(0.2, 3.0, 64), 100, 5
    elif case == "k2_circuit_clamps":
        model, rs = _circuit()
        betas, I, ea, kern = H.geometric(0.1, 4.0, 32), 400, None, "csr"
        clamps = np.zeros((I, model.n_spins), np.int8)
        clamps[:, :6] = np.where(rs.random((I, 6)) < 0.5, 1, -1)
    elif case == "k3_circuit_clamps":
        model, rs = _circuit()
        betas, I, ea, kern, k3 = H.geometric(0.1, 4.0, 32), 700, None, "bitcsr", True
        clamps = np.zeros((I, model.n_spins), np.int8)
        clamps[:, :6] = np.where(rs.random((I, 6)) < 0.5, 1, -1)
    else:  # odd periodic lattice: not bipartite -> K2, per-instance EA couplings
        model, betas, I, ea, kern = T.Model.lattice((5,)), H.linear(0.2, 3.0, 32), 400, 7, "csr"
    a = _run(monkeypatch, True, model, betas, I, ea, clamps=clamps, k3=k3)
    b = _run(monkeypatch, False, model, betas, I, ea, clamps=clamps, k3=k3)
    assert a.kernel == kern
    for x, y in zip(_state(a), _state(b)):
        if isinstance(x, tuple):
            for u, v in zip(x, y):
                assert np.array_equal(u, v)
        else:
            assert np.array_equal(x, y)
    monkeypatch.delenv("TAPT_BALANCE")
    monkeypatch.delenv("TAPT_K3")


def test_balanced_schedule_matches_oracle_on_a_split_instance():
    dims = (64, 64)
    betas = H.geometric(0.2, 1.0, 32)
    I = 200  # > 148 co-resident CTAs: C = ceil(200*57/148) = 78 > 57, so instance 1 is split
    e = T.Ensemble(T.Model.lattice(dims), betas, n_instances=I, seed=19)
    e.init_random()
    e.run(57, swap_every=1)
    S, E = e.spins(), e.energies()
    g = O.lattice_graph(dims)
    for k in (0, 1, 199):
        pt = O.PT(g, betas, 19, k, g.colour_order(O.checkerboard_colours(dims)))
        pt.run(57, 1)
        assert np.array_equal(S[k], pt.spins) and np.array_equal(E[k], pt.E)


def test_balanced_schedule_with_a_competing_kernel(monkeypatch):
    """Forward progress: the persistent grid numbers McNaughton's timelines in reverse (pt_timeline),
    so every split-job wait is on a lower-numbered, earlier-dispatched unit.  While another stream
    keeps the SMs busy and only part of the grid is resident, the run must still finish (no 2 s
    wait-timeout error) and stay bit-identical to the plain launch."""
    import torch
    dims, betas, I = (64, 64), H.geometric(0.2, 1.0, 32), 200
    ref = _run(monkeypatch, False, T.Model.lattice(dims), betas, I)
    monkeypatch.setenv("TAPT_BALANCE", "1")
    e = T.Ensemble(T.Model.lattice(dims), betas, n_instances=I, seed=17)
    side = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda")
    with torch.cuda.stream(side):
        for _ in range(40):  # ~100 ms of SM work on another stream, racing the sweeps below
            a = torch.tanh(a @ a * 1e-3)
    e.init_random()
    e.set_histogram(-4 * 4096, 8, 64)
    try:
        e.run(23, swap_every=1, measure_every=3)
        e.generate_proposals(np.arange(8), None, refine=2)
        e.run(41, swap_every=2, measure_every=5, measure_from=10)
        st = _state(e)
    finally:
        torch.cuda.synchronize()
    assert any("balanced" in x for x in e.launch_log())
    for x, y in zip(st, _state(ref)):
        if isinstance(x, tuple):
            for u, v in zip(x, y):
                assert np.array_equal(u, v)
        else:
            assert np.array_equal(x, y)
