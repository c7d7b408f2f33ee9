"""CPU tests of the problem suite: gate Hamiltonians by enumeration,
multiplier size / ground states / clamping / decoding, semiprimes."""
import itertools

import numpy as np
import pytest

import paper_2509_23043_b200 as T


def energy(ci, cj, J, h, s):
    s = np.asarray(s, np.int64)
    return float(-(J * s[ci] * s[cj]).sum() - (h * s).sum())


def gate_table(ci, cj, J, h, n):
    return {st: energy(np.array(ci), np.array(cj), np.array(J, float), np.array(h, float), st)
            for st in itertools.product([-1, 1], repeat=n)}


def test_and_gate_truth_table():
    """ground manifold = AND truth table at E=-3, gap 4."""
    e = gate_table([0, 0, 1], [1, 2, 2], [-1, 2, 2], [1, 1, -2], 3)
    valid = {s for s in e if (s[2] > 0) == (s[0] > 0 and s[1] > 0)}
    assert all(e[s] == -3 for s in valid)
    assert min(e[s] for s in e if s not in valid) == 1
    assert e[(1, 1, 1)] == -3 and e[(1, 1, -1)] == 1


FA_PAIRS = [(0, 1), (0, 2), (1, 2), (0, 3), (1, 3), (2, 3), (0, 4), (1, 4), (2, 4), (3, 4)]
FA_J = [-1, -1, -1, 1, 1, 1, 2, 2, 2, -2]


def _fa_valid(s):
    bit = lambda v: 1 if v > 0 else 0
    return bit(s[0]) + bit(s[1]) + bit(s[2]) == bit(s[3]) + 2 * bit(s[4])


def test_full_adder_truth_table():
    """SPEC.md:525-532 couplings without fields: all 8 valid rows at E=-4, invalid >= -2."""
    e = gate_table([p[0] for p in FA_PAIRS], [p[1] for p in FA_PAIRS], FA_J, [0] * 5, 5)
    valid = {s for s in e if _fa_valid(s)}
    assert len(valid) == 8 and all(e[s] == -4 for s in valid)
    assert min(e[s] for s in e if s not in valid) == -2
    assert e[(-1,) * 5] == -4 and e[(1,) * 5] == -4


def test_spec_full_adder_fields_are_degenerate():
    """The fields h=(1,1,1,-1,-2) of SPEC.md:527 make invalid rows ground states: documented
    deviation."""
    e = gate_table([p[0] for p in FA_PAIRS], [p[1] for p in FA_PAIRS], FA_J, [1, 1, 1, -1, -2], 5)
    assert min(e.values()) == -4
    assert any(e[s] == -4 for s in e if not _fa_valid(s))


@pytest.mark.parametrize("n,spins", [(2, 14), (3, 30), (4, 52), (8, 200), (16, 784)])
def test_multiplier_spin_count(n, spins):
    """3n^2+n spins (52 at n=4, 200 at n=8: PAPER.md section 5.2)."""
    M = T.Multiplier(n)
    assert M.n_spins == spins == 3 * n * n + n
    m = M.model()
    assert m.n_free == spins - 3 * n                 # 2n product bits + n carry-ins clamped
    assert set(m.couplings()[2].tolist()) <= {-2.0, -1.0, 1.0, 2.0}


def test_multiplier_forward_states_are_ground_states_n2():
    """Every consistent assignment has energy n^2*(-3) + n(n-1)*(-4) and is a global minimum
    of the unclamped circuit (enumeration over all 2^14 states at n=2)."""
    M = T.Multiplier(2)
    ci, cj, J, h = M.ci.astype(np.int64), M.cj.astype(np.int64), M.J, M.h
    emin_expect = 4 * -3 + 2 * -4
    for a in range(4):
        for b in range(4):
            assert energy(ci, cj, J, h, M.forward(a, b)) == emin_expect
    N = M.n_spins
    states = ((np.arange(2 ** N)[:, None] >> np.arange(N)) & 1) * 2 - 1
    E = -(J[None, :] * states[:, ci] * states[:, cj]).sum(1) - (h[None, :] * states).sum(1)
    assert E.min() == emin_expect
    # with the carry-ins at logical 0 (their clamp) the minima are exactly the 16 products
    cin0 = np.all(states[:, M.carry] == -1, axis=1)
    assert (E[cin0] == emin_expect).sum() == 16


def test_multiplier_forward_products_and_decode():
    for n in (3, 4, 8):
        M = T.Multiplier(n)
        rs = np.random.default_rng(n)
        for _ in range(20):
            a, b = int(rs.integers(0, 2 ** n)), int(rs.integers(0, 2 ** n))
            s = M.forward(a, b)
            prod = sum(1 << k for k in range(2 * n) if s[M.C[k]] > 0)
            assert prod == a * b
            cl = M.clamps(a * b)
            assert all(s[i] == cl[i] for i in np.nonzero(cl)[0])   # planted state satisfies clamps
            assert M.decode(s, a * b) == (a, b, True)
            E = energy(M.ci.astype(np.int64), M.cj.astype(np.int64), M.J, M.h, s)
            assert E == n * n * -3 + n * (n - 1) * -4


def test_clamp_product_examples():
    """SPEC.md:552-555."""
    M = T.Multiplier(4)
    c = M.clamps(15)
    assert [c[M.C[k]] for k in range(8)] == [1, 1, 1, 1, -1, -1, -1, -1]
    assert all(c[M.carry] == -1)
    assert all(M.clamps(0)[M.C] == -1)
    M8 = T.Multiplier(8)
    c = M8.clamps(44969)
    assert [1 if c[M8.C[k]] > 0 else 0 for k in range(16)] == [(44969 >> k) & 1 for k in range(16)]
    with pytest.raises(T.ConfigError):
        M.clamps(256)


def test_semiprimes():
    """n=4 -> 21 instances, n=2 -> {4, 6, 9}."""
    assert list(T.enumerate_semiprimes(2)) == [4, 6, 9]
    s4 = T.enumerate_semiprimes(4)
    assert len(s4) == 21
    p, q = T.random_semiprime(7, 3, 16)
    assert 2 ** 15 <= p < 2 ** 16 and 2 ** 15 <= q < 2 ** 16
    for v in (p, q):
        assert all(v % d for d in range(2, int(v ** 0.5) + 1))
    assert T.random_semiprime(7, 3, 16) == (p, q)
