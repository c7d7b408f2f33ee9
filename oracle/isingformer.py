"""oracle/isingformer.py -- TEST INFRASTRUCTURE ONLY: fp64 numpy restatement of the
IsingFormer proposal model (Appendix F), used to check the device
kernels in paper_2509_23043_b200/csrc/former.cu.  Only tests/, smoke() and tools may import it.

The reference has no implementation (proj/src/generator.cpp:1 is a placeholder), so parity is
UNPINNED against reference code: this file restates the SPEC's model, with the SPEC's
open design choices fixed in DESIGN.md section 10 and repeated here:

  * tokens: 1 <-> spin +1, 0 <-> spin -1.  Position t predicts token t from tokens < t.
  * input  x_t = E[tok_{t-1}] (t > 0; 0 at t = 0) + P_t + e_beta,
           P_t = sinusoidal positional encoding (P[t,2i] = sin(t / 10000^(2i/d)), P[t,2i+1] = cos),
           e_beta = W_beta . phi(beta) + b_beta,  phi(beta) = [sin(w_k beta), cos(w_k beta)]_k,
           w_k = 2^k / 4, k = 0 .. beta_features/2 - 1 (SPEC "fixed sinusoidal features ... followed
           by a learnable linear layer").
  * L pre-LN decoder blocks: x += Wo . Attn(LN1(x)) ; x += W2 . GELU(W1 . LN2(x)), causal
    multi-head attention (scale 1/sqrt(d/H)), GELU tanh form, LayerNorm eps 1e-5.
  * logit_t = head_w . LNf(x_t) + head_b ; P(tok_t = 1) = sigmoid(logit_t) (SPEC: one logit
    per position, Bernoulli).
  * log q = sum over t >= n_prefix of log Bernoulli(tok_t; sigmoid(logit_t)) (prefix = clamped
    tokens, SPEC.md: "log_q = 0 contribution only from free positions").
  * sampling at position t draws u = (x >> 11) * 2^-53 with x = draw t+1 of the sequence's
    stream; tok_t = 1 iff u < sigmoid(logit_t).

Parameter layout (ISFW1 canonical order, little-endian fp32), see `layout()`.
"""
import math

import numpy as np

from oracle import oracle as O


def layout(d, H, f, L, fb):
    """[(name, shape)] in the canonical ISFW1 order (matrices input-major: y = x @ W)."""
    out = [("tok_emb", (2, d)), ("beta_w", (fb, d)), ("beta_b", (d,))]
    for l in range(L):
        out += [(f"ln1_g{l}", (d,)), (f"ln1_b{l}", (d,)), (f"w_qkv{l}", (d, 3 * d)), (f"b_qkv{l}", (3 * d,)),
                (f"w_o{l}", (d, d)), (f"b_o{l}", (d,)), (f"ln2_g{l}", (d,)), (f"ln2_b{l}", (d,)),
                (f"w_1{l}", (d, f)), (f"b_1{l}", (f,)), (f"w_2{l}", (f, d)), (f"b_2{l}", (d,))]
    out += [("lnf_g", (d,)), ("lnf_b", (d,)), ("head_w", (d,)), ("head_b", (1,))]
    return out


def unflatten(flat, cfg):
    d, H, f, L, fb = cfg
    p, o = {}, 0
    for name, shape in layout(d, H, f, L, fb):
        k = int(np.prod(shape))
        p[name] = np.asarray(flat[o:o + k], dtype=np.float64).reshape(shape)
        o += k
    assert o == len(flat), (o, len(flat))
    return p


def layer_norm(x, g, b):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    return (x - mu) / np.sqrt(var + 1e-5) * g + b


def gelu(x):
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def pos_enc(T, d):
    P = np.zeros((T, d))
    t = np.arange(T)[:, None]
    i = np.arange(d // 2)[None, :]
    ang = t / np.power(10000.0, 2.0 * i / d)
    P[:, 0::2] = np.sin(ang)
    P[:, 1::2] = np.cos(ang)
    return P


def beta_features(beta, fb):
    w = np.power(2.0, np.arange(fb // 2)) / 4.0
    return np.concatenate([np.sin(w * beta), np.cos(w * beta)])


def forward_logits(flat, cfg, tokens, beta):
    """Logits [T] of one sequence (tokens [T] in {0,1}); logit t depends on tokens < t."""
    d, H, f, L, fb = cfg
    p = unflatten(flat, cfg)
    T = len(tokens)
    prev = np.zeros((T, d))
    if T > 1:
        prev[1:] = p["tok_emb"][np.asarray(tokens[:-1], dtype=np.int64)]
    x = prev + pos_enc(T, d) + (beta_features(beta, fb) @ p["beta_w"] + p["beta_b"])[None, :]
    dh = d // H
    mask = np.tril(np.ones((T, T), bool))
    for l in range(L):
        a = layer_norm(x, p[f"ln1_g{l}"], p[f"ln1_b{l}"])
        qkv = a @ p[f"w_qkv{l}"] + p[f"b_qkv{l}"]
        q, k, v = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
        o = np.zeros((T, d))
        for h in range(H):
            s = (q[:, h * dh:(h + 1) * dh] @ k[:, h * dh:(h + 1) * dh].T) / math.sqrt(dh)
            s = np.where(mask, s, -np.inf)
            s = s - s.max(1, keepdims=True)
            e = np.exp(s)
            o[:, h * dh:(h + 1) * dh] = (e / e.sum(1, keepdims=True)) @ v[:, h * dh:(h + 1) * dh]
        x = x + o @ p[f"w_o{l}"] + p[f"b_o{l}"]
        a = layer_norm(x, p[f"ln2_g{l}"], p[f"ln2_b{l}"])
        x = x + gelu(a @ p[f"w_1{l}"] + p[f"b_1{l}"]) @ p[f"w_2{l}"] + p[f"b_2{l}"]
    a = layer_norm(x, p["lnf_g"], p["lnf_b"])
    return a @ p["head_w"] + p["head_b"][0]


def log_sigmoid(z):
    return -np.logaddexp(0.0, -z)


def log_prob(flat, cfg, tokens, beta, n_prefix=0):
    z = forward_logits(flat, cfg, tokens, beta)
    t = np.asarray(tokens, dtype=np.float64)
    lp = np.where(t > 0, log_sigmoid(z), log_sigmoid(-z))
    return float(lp[n_prefix:].sum())


def sample(flat, cfg, beta, T, stream_state, prefix=()):
    """Ancestral sampling of one sequence: prefix tokens forced, then tok_t = [u_t < p_t]
    with u_t from draw t+1 of `stream_state`.  Returns (tokens, log_q, logits)."""
    toks = np.zeros(T, np.int64)
    P = len(prefix)
    toks[:P] = prefix
    logits = np.zeros(T)
    for t in range(T):
        z = forward_logits(flat, cfg, toks[:t + 1], beta)[t]  # logit t ignores token t
        logits[t] = z
        if t >= P:
            x = O.draw(stream_state, t + 1)
            u = (x >> 11) * 2.0 ** -53
            toks[t] = 1 if u < 1.0 / (1.0 + math.exp(-z)) else 0
    lp = np.where(toks > 0, log_sigmoid(logits), log_sigmoid(-logits))
    return toks, float(lp[P:].sum()), logits
