"""CPU restatement of the reference's linear layers and model-level forward --
TEST INFRASTRUCTURE ONLY (same import rules as hb_oracle.py).

Restates (reference = ringmpc under /root/reference/pkg/src):
* im2col ................................ nn.py:177-195
* local truncation ...................... nn.py:198-211
* linear / conv2d / avgpool forward ..... nn.py:214-259
* model_forward with per-layer meters ... nn.py:271-307
* triple_requirements ................... nn.py:310-325
* run_local_forward (seeded shares + dealer, two party threads) cli.py:33-58,159-180

Pinned by tests/test_oracle_golden.py against tests/golden (nn_* and model_* cases,
produced by running the reference).
"""

from __future__ import annotations

import numpy as np

from . import hb_oracle as O

U64 = np.uint64


def encode(x_f, frac=16, ring_bits=64):
    return O.encode_fixed(x_f, frac, ring_bits)


def im2col(x: np.ndarray, kh: int, kw: int, stride: int, pad: int):
    """[B, C, H, W] -> ([B, oh*ow, C*kh*kw], oh, ow) (nn.py:177-195)."""
    b, c, h, w = x.shape
    if pad:
        xp = np.zeros((b, c, h + 2 * pad, w + 2 * pad), dtype=x.dtype)
        xp[:, :, pad:pad + h, pad:pad + w] = x
    else:
        xp = x
    oh = (h + 2 * pad - kh) // stride + 1
    ow = (w + 2 * pad - kw) // stride + 1
    rows = np.empty((b, oh * ow, c, kh * kw), dtype=x.dtype)
    for i in range(oh):
        for j in range(ow):
            rows[:, i * ow + j] = xp[:, :, i * stride:i * stride + kh, j * stride:j * stride + kw].reshape(b, c, kh * kw)
    return rows.reshape(b, oh * ow, c * kh * kw), oh, ow


def truncate(x: np.ndarray, party: int, frac: int = 16, ring_bits: int = 64) -> np.ndarray:
    """SecureML local truncation (nn.py:198-211)."""
    if party == 0:
        return x >> U64(frac)
    return O.ring_neg(O.ring_neg(x, ring_bits) >> U64(frac), ring_bits)


def linear(x: np.ndarray, party: int, weight, bias, frac=16, ring_bits=64) -> np.ndarray:
    """x @ encode(W)^T mod 2^N, truncate, + encode(b) on party 0 (nn.py:214-224)."""
    w_enc = encode(weight, frac, ring_bits)
    prod = (x @ w_enc.T) & O.wmask(ring_bits)
    out = truncate(prod, party, frac, ring_bits)
    if party == 0:
        out = O.ring_add(out, encode(bias, frac, ring_bits)[None, :], ring_bits)
    return out


def conv2d(x: np.ndarray, party: int, cin, cout, kh, kw, stride, pad, weight, bias, frac=16, ring_bits=64):
    """im2col + linear, back to NCHW (nn.py:227-243)."""
    patches, oh, ow = im2col(x, kh, kw, stride, pad)
    b = x.shape[0]
    out = linear(patches.reshape(b * oh * ow, -1), party, weight.reshape(cout, -1), bias, frac, ring_bits)
    return out.reshape(b, oh * ow, cout).transpose(0, 2, 1).reshape(b, cout, oh, ow)


def avgpool(x: np.ndarray, party: int, kh, kw, stride, frac=16, ring_bits=64) -> np.ndarray:
    """Window sum * encode(1/kk), truncate (nn.py:246-259)."""
    b, c, h, w = x.shape
    patches, oh, ow = im2col(x.reshape(b * c, 1, h, w), kh, kw, stride, 0)
    sums = patches.sum(axis=2, dtype=U64) & O.wmask(ring_bits)
    inv = encode(np.array([1.0 / (kh * kw)]), frac, ring_bits)[0]
    return truncate(O.ring_mul(sums.reshape(b, c, oh, ow), inv, ring_bits), party, frac, ring_bits)


# ------------------------------------------------------------------ model level
def _shape_after(L, cur):
    k = L["kind"]
    if k == "linear":
        return (L["out_features"],)
    if k == "conv2d":
        _, h, w = cur
        return (L["out_channels"], (h + 2 * L["pad"] - L["kh"]) // L["stride"] + 1,
                (w + 2 * L["pad"] - L["kw"]) // L["stride"] + 1)
    if k == "avgpool":
        c, h, w = cur
        return (c, (h - L["kh"]) // L["stride"] + 1, (w - L["kw"]) // L["stride"] + 1)
    if k == "flatten":
        return (int(np.prod(cur)),)
    if k == "residual":
        for B in L["body"]:
            cur = _shape_after(B, cur)
    return cur


def relu_sites(layers, in_shape):
    """(group_id, per-sample elements) of every ReLU in execution order (residual bodies first)."""
    out, cur = [], tuple(in_shape)
    for L in layers:
        if L["kind"] == "relu":
            out.append((L["group_id"], int(np.prod(cur))))
        elif L["kind"] == "residual":
            out += relu_sites(L["body"], cur) + relu_sites(L.get("shortcut", []), cur)
        cur = _shape_after(L, cur)
    return out


def model_forward(party, wire, cur, x, layers, weights, windows, frac=16, ring_bits=64, layer_log=None, prefix=""):
    """Run the layers of one party (nn.py:271-307).  `residual` (out = body(x) + shortcut(x),
    a local share add, sharing.py:118-122) is this repo's extension for ResNets."""
    for i, L in enumerate(layers):
        before = O.tag_totals(wire.trace)
        k = L["kind"]
        if k == "linear":
            x = linear(x, party, weights[L["weight"]], weights[L["bias"]], frac, ring_bits)
        elif k == "conv2d":
            x = conv2d(x, party, L["in_channels"], L["out_channels"], L["kh"], L["kw"], L["stride"], L["pad"],
                       weights[L["weight"]], weights[L["bias"]], frac, ring_bits)
        elif k == "avgpool":
            x = avgpool(x, party, L["kh"], L["kw"], L["stride"], frac, ring_bits)
        elif k == "relu":
            win = windows[L["group_id"]]
            if win is not None:
                x = O.p_relu(party, wire, cur, x, ring_bits, win[0], win[1])
        elif k == "flatten":
            x = x.reshape(x.shape[0], -1)
        elif k == "residual":
            a = model_forward(party, wire, cur, x, L["body"], weights, windows, frac, ring_bits, layer_log,
                              f"{prefix}{i}.body.")
            b = model_forward(party, wire, cur, x, L.get("shortcut", []), weights, windows, frac, ring_bits,
                              layer_log, f"{prefix}{i}.short.")
            x = O.ring_add(a, b, ring_bits)
        if layer_log is not None:
            after = O.tag_totals(wire.trace)
            layer_log.append({"layer": f"{prefix}{i}:{k}", "bytes": sum(after[t][0] - before[t][0] for t in after),
                              "rounds": sum(after[t][1] - before[t][1] for t in after)})
    return x


def triple_requirements(layers, in_shape, windows, batch, ring_bits=64):
    """(kind, width) -> count (nn.py:310-325)."""
    need = {}
    for g, count in relu_sites(layers, in_shape):
        if windows[g] is None:
            continue
        k, m = windows[g]
        for key, num in O.triple_need(count * batch, k - m, ring_bits).items():
            need[key] = need.get(key, 0) + num
    return need


def triple_seed(seed: int, kind: str, width: int) -> int:
    """SeedSequence([seed, 0x7337, kind_code, width]) (cli.py:51-53)."""
    code = 1 if kind == "arith" else 2
    return int(np.random.SeedSequence([seed, 0x7337, code, width]).generate_state(1)[0])


def run_local_forward(layers, in_shape, weights, windows, x_f, seed, frac=16, ring_bits=64):
    """Both parties in process (cli.py:159-180); returns (logits, (trace0, trace1), (log0, log1))."""
    enc = encode(x_f, frac, ring_bits)
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x1289]))
    s0, s1 = O.split_additive(enc, ring_bits, rng)
    need = triple_requirements(layers, in_shape, windows, x_f.shape[0], ring_bits)
    curs = (O.Cursor(0), O.Cursor(1))
    for (kind, width), count in sorted(need.items()):
        t = O.deal(kind, count, width, triple_seed(seed, kind, width))
        for p in (0, 1):
            curs[p].stock(kind, width, t[p])
    w0, w1 = O.wire_pair()
    logs = ([], [])
    y0, y1 = O.run_two(lambda: model_forward(0, w0, curs[0], s0, layers, weights, windows, frac, ring_bits, logs[0]),
                       lambda: model_forward(1, w1, curs[1], s1, layers, weights, windows, frac, ring_bits, logs[1]),
                       (w0, w1))
    rec = O.ring_add(y0, y1, ring_bits)
    sh = U64(64 - ring_bits)
    logits = ((rec << sh).view(np.int64) >> np.int64(64 - ring_bits)).astype(np.float64) / float(1 << frac)
    return logits, (w0.trace, w1.trace), logs
