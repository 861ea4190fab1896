"""CPU restatement of the reference's float simulator -- TEST INFRASTRUCTURE ONLY (same import
rules as hb_oracle.py: only tests/, smoke() and bench.py's baseline legs may use it).

Restates (reference = ringmpc under /root/reference/pkg/src):
* sim_relu: encode, share_arith split from rng.bytes, drelu_from_shares, keep-or-zero
  ........................................................ simulator.py:47-54 (ring.py:191-213, sharing.py:88-96)
* the float pipeline with a ReLU hook (im2col matmul conv, avgpool as patch means)
  ........................................................ simulator.py:57-82
* exact_relu / plain_forward .............................. simulator.py:85-98
* sim_forward (splits seeded by (seed, layer index)) ...... simulator.py:101-124
* collect_drelu_decisions / collect_activation_ranges ..... simulator.py:127-174

Pinned by tests/test_oracle_golden.py against the sim_* golden cases (produced by running the
reference); the layer list is the oracle's JSON form (hb_oracle_nn).
"""

from __future__ import annotations

import numpy as np

from . import hb_oracle as O
from . import hb_oracle_nn as ON


def sim_relu(x_f, k, m, rng, frac=16, ring_bits=64):
    e = O.encode_fixed(x_f, frac, ring_bits)
    s0, s1 = O.split_additive(e, ring_bits, rng)
    keep = O.drelu_from_shares(s0, s1, ring_bits, k, m)
    return np.asarray(x_f, dtype=np.float64) * keep.astype(np.float64)


def exact_relu(x_f, frac=16, ring_bits=64):
    e = O.encode_fixed(x_f, frac, ring_bits)
    keep = np.uint64(1) - ((e >> np.uint64(ring_bits - 1)) & np.uint64(1))
    return np.asarray(x_f, dtype=np.float64) * keep.astype(np.float64)


def float_forward(layers, weights, x_f, relu_hook):
    cur = np.asarray(x_f, dtype=np.float64)
    for i, L in enumerate(layers):
        kind = L["kind"]
        if kind == "linear":
            w = weights[L["weight"]].astype(np.float64)
            b = weights[L["bias"]].astype(np.float64)
            cur = cur @ w.T + b[None, :]
        elif kind == "conv2d":
            w = weights[L["weight"]].astype(np.float64)
            b = weights[L["bias"]].astype(np.float64)
            patches, oh, ow = ON.im2col(cur, L["kh"], L["kw"], L["stride"], L["pad"])
            out = patches @ w.reshape(L["out_channels"], -1).T + b[None, None, :]
            cur = out.transpose(0, 2, 1).reshape(cur.shape[0], L["out_channels"], oh, ow)
        elif kind == "avgpool":
            bsz, c, h, w_ = cur.shape
            patches, oh, ow = ON.im2col(cur.reshape(bsz * c, 1, h, w_), L["kh"], L["kw"], L["stride"], 0)
            cur = patches.mean(axis=2).reshape(bsz, c, oh, ow)
        elif kind == "relu":
            cur = relu_hook(i, L["group_id"], cur)
        elif kind == "flatten":
            cur = cur.reshape(cur.shape[0], -1)
        else:
            raise ValueError(kind)
    return cur


def plain_forward(layers, weights, x_f):
    return float_forward(layers, weights, x_f, lambda i, g, a: exact_relu(a))


def _rng(seed, i):
    return np.random.default_rng(np.random.SeedSequence([seed, i]))


def sim_forward(layers, weights, x_f, labels, windows, seed):
    def hook(i, g, a):
        w = windows[g]
        return a if w is None else sim_relu(a, w[0], w[1], _rng(seed, i))

    logits = float_forward(layers, weights, x_f, hook)
    acc = float("nan") if labels is None else float(np.mean(np.argmax(logits, axis=1) == np.asarray(labels)))
    return logits, acc


def collect_drelu_decisions(layers, weights, x_f, windows, seed):
    masks = []

    def hook(i, g, a):
        w = windows[g]
        if w is None:
            masks.append(np.ones_like(a, dtype=bool))
            return a
        out = sim_relu(a, w[0], w[1], _rng(seed, i))
        masks.append(out != 0.0)
        return out

    return float_forward(layers, weights, x_f, hook), masks


def collect_activation_ranges(layers, weights, x_f, frac=16, ring_bits=64):
    ext = {}

    def hook(i, g, a):
        e = O.encode_fixed(a, frac, ring_bits).view(np.int64)
        lo, hi = int(e.min()), int(e.max())
        ext[g] = (min(lo, ext[g][0]), max(hi, ext[g][1])) if g in ext else (lo, hi)
        return exact_relu(a, frac, ring_bits)

    float_forward(layers, weights, x_f, hook)

    def bits_for(v):
        return v.bit_length() + 1 if v >= 0 else (-v - 1).bit_length() + 1

    return {g: min(max(2, bits_for(lo), bits_for(hi)), ring_bits) for g, (lo, hi) in ext.items()}
