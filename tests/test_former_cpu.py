"""IsingFormer host side and fp64 oracle: parameter layout and count,
seeded initialisation, the ISFW1 checkpoint round trip and its error cases (through the C ABI,
no GPU needed), and the SPEC's invariants on the oracle restatement (causality,
normalisation, sample/log_prob consistency, zero head).  CPU only."""
import itertools
import math

import numpy as np
import pytest

import paper_2509_23043_b200 as T
from oracle import isingformer as F

SMALL = dict(d_model=64, heads=2, ffn=128, layers=2, max_len=64, beta_features=16)
CFG = (64, 2, 128, 2, 16)


def test_param_count_matches_spec_default():
    n = T.Former.param_count()
    assert n == sum(int(np.prod(s)) for _, s in F.layout(*CFG))
    assert abs(n - 67_000) <= 0.2 * 67_000  # SPEC: within 20% of 67k (Appendix F)


def test_init_is_seeded_and_structured():
    a = T.Former.init_params(seed=3, **SMALL)
    b = T.Former.init_params(seed=3, **SMALL)
    c = T.Former.init_params(seed=4, **SMALL)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    p = F.unflatten(a, CFG)
    assert np.all(p["ln1_g0"] == 1) and np.all(p["ln1_b0"] == 0) and np.all(p["b_qkv1"] == 0)
    assert abs(p["w_qkv0"].std() - 1 / 8) < 0.01  # N(0, 1/fan_in), fan_in = 64


def test_isfw1_round_trip_and_errors(tmp_path):
    p = T.Former.init_params(seed=5, **SMALL)
    f = T.Former(p, **SMALL)
    path = tmp_path / "m.isfw"
    f.save(path)
    raw = path.read_bytes()
    assert raw[:5] == b"ISFW1" and len(raw) == 5 + 8 * 4 + 4 * len(p)
    g = T.Former.load(path)
    assert g.config == f.config and np.array_equal(g.params(), p)
    bad = tmp_path / "bad.isfw"
    bad.write_bytes(b"ISFWX" + raw[5:])
    with pytest.raises(T.FormatError):
        T.Former.load(bad)
    bad.write_bytes(raw[:-7])
    with pytest.raises(T.FormatError):
        T.Former.load(bad)
    with pytest.raises(T.ConfigError):
        T.Former(None, **dict(SMALL, heads=3))  # d_model not divisible by heads
    with pytest.raises(T.DimensionError):
        T.Former(p[:10], **SMALL)
    with pytest.raises(T.SizeError):  # the device kernels are built for the SPEC default shape
        T.Former(T.Former.init_params(**dict(SMALL, ffn=64)), **dict(SMALL, ffn=64))


def _params(seed=1, scale=2.0):
    return T.Former.init_params(seed=seed, scale=scale, **SMALL)


def test_oracle_causality():
    p = _params()
    rs = np.random.default_rng(0)
    tok = rs.integers(0, 2, 12)
    z = F.forward_logits(p, CFG, tok, 0.7)
    for t in range(11):
        tok2 = tok.copy()
        tok2[t + 1:] = rs.integers(0, 2, 11 - t)
        z2 = F.forward_logits(p, CFG, tok2, 0.7)
        assert np.array_equal(z[:t + 2], z2[:t + 2])  # logit t+1 depends on tokens <= t only


def test_oracle_normalisation_10_spins():
    p = _params(seed=2)
    tot = 0.0
    for bits in itertools.product([0, 1], repeat=10):
        tot += math.exp(F.log_prob(p, CFG, np.array(bits), 1.3))
    assert abs(tot - 1.0) < 1e-8


def test_oracle_sample_log_prob_consistency_and_zero_head():
    p = _params(seed=3)
    tok, lq, _ = F.sample(p, CFG, 0.9, 14, 0x1234, prefix=[1, 0, 1])
    assert list(tok[:3]) == [1, 0, 1]
    assert abs(lq - F.log_prob(p, CFG, tok, 0.9, n_prefix=3)) < 1e-12
    q = F.unflatten(p, CFG)
    z = p.copy()
    off = sum(int(np.prod(s)) for n, s in F.layout(*CFG) if n not in ("head_w", "head_b"))
    z[off:] = 0.0  # head_w, head_b are last
    assert np.allclose(F.forward_logits(z, CFG, tok, 0.9), 0.0)
    assert abs(F.log_prob(z, CFG, tok, 0.9, n_prefix=3) - 11 * math.log(0.5)) < 1e-12
    del q
