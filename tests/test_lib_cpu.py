"""CPU tests of the product library (no GPU needed): the C-ABI .so loads and exports
every symbol of include/tapt_gpu.h, host-side model construction matches the reference
(couplings, digest, energy), schedules are valid, errors map to the reference taxonomy,
and every device entry point fails loudly without a GPU (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import paper_2509_23043_b200 as T
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _lib_built():
    if not os.path.exists(T.LIB_PATH):
        import subprocess
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2509_23043_b200", "csrc")], check=True)


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tapt_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tapt_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = T.lib()
    syms = header_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(T.exported_symbols())


def test_version_and_no_gpu_here_is_reported():
    assert b"sm_100a" in T.lib().tapt_version()
    assert T.device_count() >= 0


@pytest.mark.parametrize("dims,periodic", [((32, 32), True), ((5, 7), False), ((8,), True), ((3,), True),
                                           ((4, 6), True), ((2, 2), True)])
def test_lattice_model_matches_reference_builder(dims, periodic):
    m = T.Model.lattice(dims, 1.0, periodic)
    ci, cj, J = m.couplings()
    g = O.lattice_graph(dims, 1.0, periodic)
    assert np.array_equal(ci, g.ci) and np.array_equal(cj, g.cj) and np.array_equal(J, g.J)
    if O.have_ref():
        R = O.ref()
        h = R.ref_graph_lattice(2 if len(dims) == 2 else 3, dims[0], dims[-1], dims[0], 1.0, int(periodic))
        assert m.digest() == R.ref_graph_digest(h)
        R.ref_graph_free(h)


def test_graph_model_digest_energy_and_merging():
    rs = np.random.default_rng(3)
    n = 30
    ci, cj = rs.integers(0, n, 90), rs.integers(0, n, 90)
    keep = ci != cj
    J = rs.integers(-3, 4, 90).astype(float)
    h = rs.integers(-2, 3, n).astype(float)
    cl = np.where(rs.random(n) < 0.2, rs.choice([-1, 1], n), 0).astype(np.int8)
    m = T.Model.graph(n, ci[keep], cj[keep], J[keep], h, cl)
    g = O.Graph.from_couplings(n, ci[keep], cj[keep], J[keep], h, cl)
    a, b, c = m.couplings()
    assert np.array_equal(a, g.ci) and np.array_equal(b, g.cj) and np.array_equal(c, g.J)
    s = rs.choice(np.array([-1, 1], np.int8), n)
    assert m.energy(s) == O.lib().oc_energy(g.oc(), s.ctypes.data_as(O._i8p))
    assert m.n_free == int((cl == 0).sum())
    if O.have_ref():
        rg = O.ref_graph(g)
        assert m.digest() == O.ref().ref_graph_digest(rg)
        O.ref().ref_graph_free(rg)


def test_schedules_are_valid_colourings_and_levels():
    rs = np.random.default_rng(4)
    n = 50
    ci, cj = rs.integers(0, n, 200), rs.integers(0, n, 200)
    keep = ci != cj
    g = O.Graph.from_couplings(n, ci[keep], cj[keep], np.ones(keep.sum()))
    m = T.Model.graph(n, ci[keep], cj[keep], np.ones(keep.sum()))
    col, lev = m.schedule()
    assert np.array_equal(col, O.greedy_colours(g))
    for i in range(n):
        for j in g.col[g.rowptr[i]:g.rowptr[i + 1]]:
            assert col[i] != col[j]
            if j < i:
                assert lev[j] < lev[i]


def test_checkerboard_is_the_greedy_colouring_of_even_periodic_lattices():
    m = T.Model.lattice((16, 16))
    col, _ = m.schedule()
    assert np.array_equal(col, O.checkerboard_colours((16, 16)))
    assert m.n_colours == 2 and m.n_levels == 31


def test_error_taxonomy():
    with pytest.raises(T.ConfigError):
        T.Model.graph(3, [0], [0], [1.0])                     # self-coupling (spin_model.cpp:20)
    with pytest.raises(T.ConfigError):
        T.Model.graph(3, [0], [5], [1.0])                     # out of range (spin_model.cpp:21)
    with pytest.raises(T.ConfigError):
        T.Model.graph(3, [0], [1], [1.0], None, [2, 0, 0])    # clamp value (spin_model.cpp:35)
    half = T.Model.graph(3, [0], [1], [0.5], [0.25, 0.0, -1.5])  # real-valued: accepted (spin_model.cpp:18-24)
    assert half.energy(np.array([1, -1, 1], np.int8)) == 0.5 - 0.25 + 1.5
    m = T.Model.lattice((4, 4))
    with pytest.raises(T.DimensionError):
        m.energy(np.ones(3, np.int8))                         # spin_model.cpp:80-82


@pytest.mark.skipif(T.device_count() > 0, reason="checks the no-GPU behaviour")
def test_device_calls_fail_loudly_without_gpu():
    m = T.Model.lattice((8, 8))
    with pytest.raises(T.CudaError):
        T.Ensemble(m, [0.5, 1.0])
    with pytest.raises(T.CudaError):
        T.gibbs_sweep(m, np.ones(64, np.int8), 0.5, 1)
    with pytest.raises(T.CudaError):
        T.gibbs_update(m, np.ones(64, np.int8), 3, 0.5, 1)
    with pytest.raises(T.CudaError):
        T.NcclComm(bytes(128), 1, 0)  # no communicator without a device
    with pytest.raises(T.ConfigError):
        T.set_device(0)  # no device 0 here
    with pytest.raises(T.ClampedSiteError):  # the reference's error order: dimension, then clamp, then device
        T.gibbs_update(T.Model.graph(2, [0], [1], [1.0], None, [1, 0]), np.ones(2, np.int8), 0, 0.5, 1)


def test_ensemble_argument_validation():
    m = T.Model.lattice((8, 8))
    with pytest.raises(T.ConfigError):
        T.Ensemble(m, [0.5, 0.4])        # ladder must increase
    with pytest.raises(T.ConfigError):
        T.Ensemble(m, [-0.1, 0.4])       # beta >= 0


def test_isingmodel_v1_round_trip_and_errors(tmp_path):
    """CouplingGraph save/load (spin_model.cpp:123-226) through the C ABI, incl. the
    reference's parse errors (test_spin_model.cpp:189-233)."""
    M = T.Multiplier(4)
    m = M.model()
    p = tmp_path / "mult.ising"
    m.save_file(str(p))
    text = p.read_text()
    assert text.startswith("isingmodel v1\nn 52\n")
    m2 = T.Model.load_file(str(p))
    assert m2.digest() == m.digest()
    assert all(np.array_equal(a, b) for a, b in zip(m.couplings(), m2.couplings()))
    bad = tmp_path / "bad.ising"
    for body, err in (("isingmodel v2\nn 2\n", T.FormatError), ("isingmodel v1\nc 0 1 1\n", T.FormatError),
                      ("isingmodel v1\nn 3\nc 0 1 1\nc 1 0 2\n", T.FormatError),
                      ("isingmodel v1\nn 2\nq 1\n", T.FormatError), ("isingmodel v1\nn 2\nc 0 0 1\n", T.ConfigError),
                      ("isingmodel v1\nn 2\nx 0 2\n", T.FormatError)):
        bad.write_text(body)
        with pytest.raises(err):
            T.Model.load_file(str(bad))
    if O.have_ref():
        import ctypes as C
        # the reference loader reads our file to the same graph (digest)
        g = O.Graph.from_couplings(52, M.ci, M.cj, M.J, M.h, M.clamp)
        rg = O.ref_graph(g)
        assert O.ref().ref_graph_digest(rg) == m.digest()
        O.ref().ref_graph_free(rg)
        del C


def test_residual_energy_spec_examples():
    """ground state -> 0; one excited bond on an N = 10 chain (dE = 2J) -> 0.2;
    the mean over runs; best-so-far is non-increasing."""
    eg = -9.0
    assert np.allclose(T.residual_energy([[eg, eg]], eg, 10), 0.0)
    assert np.allclose(T.residual_energy([[eg + 2.0, eg + 2.0]], eg, 10), 0.2)
    assert np.allclose(T.residual_energy([[eg, eg], [eg + 4.0, eg + 4.0]], eg, 10), 0.2)
    r = T.residual_energy([[eg + 6, eg + 2, eg + 4, eg]], eg, 10, best_so_far=True)
    assert np.all(np.diff(r) <= 0) and np.allclose(r, [0.6, 0.2, 0.2, 0.0])
    assert np.allclose(T.residual_energy([[1.0, 0.0], [3.0, 2.0]], [0.0, 2.0], 1), [1.0, 0.0])
    with pytest.raises(T.DimensionError):
        T.residual_energy([], eg, 10)
