"""IsingFormer on the device (csrc/former.cu) against the fp64 oracle restatement
(oracle/isingformer.py): logits and log q within fp32 tolerance, causality, normalisation,
sampling with the same counter-based streams, and the MH-corrected TAPT move (Eq. 2 with
log q) keeping Boltzmann with the Former as the proposal source.  Marked `gpu`."""
import itertools
import math

import numpy as np
import pytest

import paper_2509_23043_b200 as T
from oracle import isingformer as F
from oracle import oracle as O

pytestmark = pytest.mark.gpu

SMALL = dict(d_model=64, heads=2, ffn=128, layers=2, max_len=256, beta_features=16)
CFG = (64, 2, 128, 2, 16)
LOGIT_TOL = 2e-4  # fp32 device vs fp64 oracle, |logit| ~ O(1..10) with scale-2 weights


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if T.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


def model(seed=1, scale=2.0, **kw):
    conf = dict(SMALL, **kw)
    p = T.Former.init_params(seed=seed, scale=scale, **conf)
    return T.Former(p, **conf), p


def test_logits_and_log_prob_match_oracle():
    f, p = model(seed=1)
    rs = np.random.default_rng(0)
    B, Tn = 5, 70  # three 32-row tiles, the last one ragged
    tok = rs.integers(0, 2, (B, Tn)).astype(np.uint8)
    betas = np.array([0.1, 0.5, 1.0, 2.5, 5.0])
    lq, z = f.log_prob(tok, betas, n_prefix=7, return_logits=True)
    for b in range(B):
        zo = F.forward_logits(p, CFG, tok[b], betas[b])
        assert np.max(np.abs(z[b] - zo)) < LOGIT_TOL * max(1.0, np.max(np.abs(zo)))
        assert abs(lq[b] - F.log_prob(p, CFG, tok[b], betas[b], n_prefix=7)) < 1e-3


def test_device_causality_is_exact():
    f, _ = model(seed=2)
    rs = np.random.default_rng(1)
    tok = rs.integers(0, 2, (1, 64)).astype(np.uint8)
    _, z = f.log_prob(tok, 0.8, return_logits=True)
    for t in (0, 5, 31, 32, 50):
        tok2 = tok.copy()
        tok2[0, t + 1:] ^= 1
        _, z2 = f.log_prob(tok2, 0.8, return_logits=True)
        assert np.array_equal(z[0, :t + 2], z2[0, :t + 2])


def test_device_normalisation_10_spins():
    f, _ = model(seed=3)
    toks = np.array(list(itertools.product([0, 1], repeat=10)), np.uint8)
    lq = f.log_prob(toks, 1.1)
    assert abs(np.exp(lq).sum() - 1.0) < 1e-5


def test_zero_head_gives_n_log_half():
    f0, p = model(seed=4)
    off = sum(int(np.prod(s)) for n, s in F.layout(*CFG) if n not in ("head_w", "head_b"))
    p[off:] = 0.0
    f = T.Former(p, **SMALL)
    tok = np.random.default_rng(2).integers(0, 2, (3, 40)).astype(np.uint8)
    assert np.allclose(f.log_prob(tok, 1.0, n_prefix=4), 36 * math.log(0.5), atol=1e-9)
    del f0


def test_sampling_matches_oracle_streams():
    f, p = model(seed=5)
    B, Tn, npre = 40, 24, 4
    betas = np.linspace(0.2, 3.0, B)
    streams = np.array([T.derive_state(77, [0x44, b]) for b in range(B)], np.uint64)
    prefix = np.random.default_rng(3).integers(0, 2, (B, npre)).astype(np.uint8)
    tok, lq = f.sample(B, Tn, betas, streams, prefix)
    assert np.array_equal(tok[:, :npre], prefix)
    # log q of the sample equals the forward log_prob of the sampled tokens (SPEC consistency)
    assert np.allclose(lq, f.log_prob(tok, betas, n_prefix=npre), atol=1e-4)
    same = 0
    for b in range(B):
        to, lo, zo = F.sample(p, CFG, betas[b], Tn, int(streams[b]), prefix=prefix[b])
        if np.array_equal(to, tok[b]):
            same += 1
            assert abs(lo - lq[b]) < 1e-3
        else:  # only a draw within fp32 rounding of the threshold may flip a token
            t = int(np.argmax(to != tok[b]))
            u = (O.draw(int(streams[b]), t + 1) >> 11) * 2.0 ** -53
            assert abs(u - 1 / (1 + math.exp(-zo[t]))) < 1e-4
    assert same >= B - 2


def test_bf16_kv_cache_logits_consistency_and_normalisation():
    """bf16 K/V storage (fp32 math): logits within 3e-2 (relative to max |logit|) of the fp64 oracle,
    sampling and log_prob consistent with each other, and the distribution still normalised."""
    conf = dict(SMALL)
    p = T.Former.init_params(seed=6, scale=2.0, **conf)
    f = T.Former(p, kv="bf16", **conf)
    rs = np.random.default_rng(4)
    B, Tn = 4, 70
    tok = rs.integers(0, 2, (B, Tn)).astype(np.uint8)
    betas = np.array([0.2, 0.9, 1.7, 3.0])
    _, z = f.log_prob(tok, betas, return_logits=True)
    errs = []
    for b in range(B):
        zo = F.forward_logits(p, CFG, tok[b], betas[b])
        errs.append(np.max(np.abs(z[b] - zo)) / max(1.0, np.max(np.abs(zo))))
    assert max(errs) < 3e-2, errs
    assert max(errs) > 0  # the bf16 path really runs (fp32 would be ~1e-5)
    streams = np.array([T.derive_state(91, [0x44, b]) for b in range(32)], np.uint64)
    tok2, lq = f.sample(32, 40, np.linspace(0.2, 3.0, 32), streams)
    assert np.allclose(lq, f.log_prob(tok2, np.linspace(0.2, 3.0, 32)), atol=1e-4)
    toks = np.array(list(itertools.product([0, 1], repeat=10)), np.uint8)
    assert abs(np.exp(f.log_prob(toks, 1.1)).sum() - 1.0) < 1e-5


def test_sample_token_statistics_follow_logits():
    """Many samples of a 3-token sequence: empirical frequencies vs exp(log_prob)."""
    f, _ = model(seed=6, scale=1.0)
    B = 60000
    streams = np.random.default_rng(4).integers(0, 2 ** 63, B, dtype=np.uint64)
    tok, _ = f.sample(B, 3, 0.7, streams)
    idx = tok[:, 0] * 4 + tok[:, 1] * 2 + tok[:, 2]
    freq = np.bincount(idx, minlength=8) / B
    allt = np.array(list(itertools.product([0, 1], repeat=3)), np.uint8)
    prob = np.exp(f.log_prob(allt, 0.7))
    assert 0.5 * np.abs(freq - prob).sum() < 0.01


def _five_spin():
    ci = [0, 1, 2, 3, 0, 1]
    cj = [1, 2, 3, 4, 2, 4]
    J = [1.0, -1.0, 2.0, 1.0, -1.0, 1.0]
    h = [0.0, 1.0, 0.0, -1.0, 0.0]
    return O.Graph.from_couplings(5, ci, cj, J, h), (ci, cj, J, h)


def _boltzmann5(g, beta):
    states = np.array(list(itertools.product([-1, 1], repeat=5)), np.int8)
    E = np.array([O.lib().oc_energy(g.oc(), np.ascontiguousarray(s).ctypes.data_as(O._i8p)) for s in states], float)
    q = np.exp(-beta * (E - E.min()))
    return states, q / q.sum()


def _former_tapt(mh):
    """Per round: one Gibbs sweep, then a Former proposal round into every slot (Eq. 2, with
    log q when mh): proposals sampled at the slot's beta, log q of the current state from a
    forward pass."""
    g, (ci, cj, J, h) = _five_spin()
    m = T.Model.graph(5, ci, cj, J, h)
    betas = np.array([0.5, 1.0, 1.5, 2.0])
    I, R = 4096, 4
    e = T.Ensemble(m, betas, n_instances=I, seed=41)
    e.init_random()
    f, _ = model(seed=9, scale=3.0)  # untrained, far from Boltzmann
    rs = np.random.default_rng(8)
    targets = np.arange(R)
    bseq = np.tile(betas, I)
    w = 1 << np.arange(5)
    counts = np.zeros((R, 32))
    for rnd in range(60):
        e.sweep(1)
        streams = rs.integers(0, 2 ** 63, I * R, dtype=np.uint64)
        tok, lq_prop = f.sample(I * R, 5, bseq, streams)
        props = np.where(tok > 0, 1, -1).astype(np.int8).reshape(I, R, 5)
        if mh:
            cur = (e.spins() > 0).astype(np.uint8).reshape(I * R, 5)
            lq_cur = f.log_prob(cur, bseq)
            e.inject_proposals(props, targets, lq_cur.reshape(I, R), lq_prop.reshape(I, R))
        else:
            e.inject_proposals(props, targets)
        if rnd >= 20:
            S = e.spins()
            for r in range(R):
                np.add.at(counts[r], ((S[:, r, :] > 0) * w).sum(axis=1), 1)
    tvs = []
    for r, b in enumerate(betas):
        states, q = _boltzmann5(g, b)
        ref = np.zeros(32)
        ref[((states > 0) * w).sum(axis=1)] = q
        tvs.append(0.5 * np.abs(counts[r] / counts[r].sum() - ref).sum())
    return np.array(tvs)


def test_former_proposals_with_mh_correction_keep_boltzmann():
    corrected = _former_tapt(True)
    biased = _former_tapt(False)
    assert corrected.max() < 0.02
    assert biased.max() > 2 * corrected.max()


def test_tensor_core_forward_equals_cuda_core_forward():
    """log_prob's tcgen05 path (bf16x3 products, TMEM accumulators) against the fp32 CUDA-core row
    engine on the same inputs: ragged 128-row tiles spanning sequences, 2 layers; and the fp64 oracle."""
    f, p = model(seed=6, max_len=256)
    rs = np.random.default_rng(4)
    B, Tn = 9, 203  # 1827 rows: 15 tiles, the last ragged; sequences straddle tiles
    tok = rs.integers(0, 2, (B, Tn)).astype(np.uint8)
    betas = rs.uniform(0.1, 4.0, B)
    f.set_tensor_cores(True)
    lq_tc, z_tc = f.log_prob(tok, betas, n_prefix=11, return_logits=True)
    f.set_tensor_cores(False)
    lq_cc, z_cc = f.log_prob(tok, betas, n_prefix=11, return_logits=True)
    # bf16x3 products carry ~2^-16 relative error per product (the split residuals): well inside the
    # fp32-vs-fp64 tolerance both engines are held to
    assert np.max(np.abs(z_tc - z_cc)) < 1e-4 * max(1.0, np.max(np.abs(z_cc)))
    assert np.max(np.abs(lq_tc - lq_cc)) < 2e-3
    for b in (0, 4, 8):
        zo = F.forward_logits(p, CFG, tok[b], betas[b])
        assert np.max(np.abs(z_tc[b] - zo)) < LOGIT_TOL * max(1.0, np.max(np.abs(zo)))


@pytest.mark.parametrize("Tn", [1, 31, 32, 33, 127, 128, 129, 200])
def test_tensor_core_forward_ragged_lengths(Tn):
    """Sequence lengths around the 32-key chunk and 128-query block edges (incl. a single position and
    one row in the last block), against the fp64 oracle; n_prefix = T gives log q = 0."""
    f, p = model(seed=7, max_len=256)
    rs = np.random.default_rng(Tn)
    B = 3
    tok = rs.integers(0, 2, (B, Tn)).astype(np.uint8)
    betas = np.array([0.3, 1.0, 4.0])
    lq, z = f.log_prob(tok, betas, return_logits=True)
    for b in range(B):
        zo = F.forward_logits(p, CFG, tok[b], betas[b])
        assert np.max(np.abs(z[b] - zo)) < LOGIT_TOL * max(1.0, np.max(np.abs(zo)))
        assert abs(lq[b] - F.log_prob(p, CFG, tok[b], betas[b])) < 1e-3
    assert np.all(f.log_prob(tok, betas, n_prefix=Tn) == 0.0)
