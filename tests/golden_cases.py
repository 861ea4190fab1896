"""Input recipes for the golden cases -- numpy only, importable everywhere.

``tests/golden/make_golden.py`` feeds these inputs to the reference package;
the CPU tests feed them to the oracle and the GPU tests to the CUDA path.
Each recipe mirrors the reference test it is named after, consuming the numpy
generators in the same order so the shares are bit-identical.
"""

from __future__ import annotations

import functools

import numpy as np

U64 = np.uint64
M64 = U64(2**64 - 1)


def _words(rng, n):
    return np.frombuffer(rng.bytes(8 * n), dtype="<u8").copy()


def _mask(w):
    return U64((1 << w) - 1)


def share_arith(secret, w, rng):
    """Reference sharing.share_arith (sharing.py:88-96): (x + r, -r)."""
    secret = np.asarray(secret).astype(np.int64).view(U64) & _mask(w) if secret.dtype != U64 else secret & _mask(w)
    r = _words(rng, secret.size).reshape(secret.shape) & _mask(w)
    return (secret + r) & _mask(w), (~r + U64(1)) & _mask(w)


def share_binary(secret, w, rng):
    """Reference sharing.share_binary (sharing.py:104-110): (x ^ r, r)."""
    secret = secret & _mask(w)
    r = _words(rng, secret.size).reshape(secret.shape) & _mask(w)
    return secret ^ r, r


def encode(x_f, frac=16):
    """Reference ring.encode_array (ring.py:191-199) at N=64."""
    s = np.asarray(x_f, dtype=np.float64) * float(1 << frac)
    return np.copysign(np.floor(np.abs(s) + 0.5), s).astype(np.int64).view(U64)


def all_splits_u8():
    x, s1 = np.meshgrid(np.arange(256, dtype=U64), np.arange(256, dtype=U64))
    x, s1 = x.ravel(), s1.ravel()
    return x, (x - s1) & U64(255), s1


def all_pairs_u8():
    a, b = np.meshgrid(np.arange(256, dtype=U64), np.arange(256, dtype=U64))
    return a.ravel(), b.ravel()


def baseline_inputs(n, seed=2024):
    """BASELINE.json configs[0] distribution: x_f ~ N(0, 4^2), f=16, N=64."""
    x_f = np.random.default_rng(seed).normal(0.0, 4.0, n)
    return share_arith(encode(x_f), 64, np.random.default_rng(seed + 1))


RELU_CASES = [
    dict(name="fig4_drelu", op="drelu", n_bits=8, k=5, m=2, seed=0, recipe="fig4", keep=True),
    dict(name="fig4_relu", op="relu", n_bits=8, k=5, m=2, seed=0, recipe="fig4", keep=True),
    dict(name="u8_full_drelu", op="drelu", n_bits=8, k=8, m=0, seed=0, recipe="u8_splits"),
    *[dict(name=f"u8_k{k}_drelu", op="drelu", n_bits=8, k=k, m=0, seed=k, recipe="u8_splits") for k in range(2, 9)],
    *[dict(name=f"u8_minus1_k{k}", op="drelu", n_bits=8, k=k, m=0, seed=k, recipe="minus1", keep=True)
      for k in (2, 4, 8)],
    *[dict(name=f"w10_m{m}_relu", op="relu", n_bits=10, k=10, m=m, seed=m, recipe="w10_crit2") for m in (1, 2, 3, 4)],
    dict(name="w10_m3_prune", op="relu", n_bits=10, k=10, m=3, seed=0, recipe="w10_prune"),
    dict(name="w10_zero", op="relu", n_bits=10, k=10, m=3, seed=0, recipe="zero32", keep=True),
    dict(name="sim10k_21_7", op="relu", n_bits=64, k=21, m=7, seed=0, recipe="sim10k", keep=True),
    dict(name="odd37_18_6", op="relu", n_bits=64, k=18, m=6, seed=0, recipe="arange37", keep=True, store_inputs=True),
    dict(name="odd33_12_2", op="relu", n_bits=64, k=12, m=2, seed=1, recipe="fill33", keep=True, store_inputs=True),
    dict(name="odd50_16_0", op="relu", n_bits=64, k=16, m=0, seed=0, recipe="arange50", keep=True, store_inputs=True),
    dict(name="n8_20_4", op="relu", n_bits=64, k=20, m=4, seed=0, recipe="arange8_64", keep=True),
    dict(name="n8_w10_10_3", op="relu", n_bits=10, k=10, m=3, seed=0, recipe="arange8_10", keep=True),
    dict(name="n8_64_0", op="relu", n_bits=64, k=64, m=0, seed=0, recipe="arange8_64b", keep=True),
    *[dict(name=f"base4096_{k}_{m}", op="relu", n_bits=64, k=k, m=m, seed=1, recipe="base4096",
           keep=(k, m) in ((64, 0), (22, 14)))
      for (k, m) in ((64, 0), (32, 0), (22, 6), (22, 14), (22, 16))],
    dict(name="base1001_22_16", op="relu", n_bits=64, k=22, m=16, seed=2, recipe="base1001", keep=True),
    dict(name="base1000_40_3", op="relu", n_bits=64, k=40, m=3, seed=3, recipe="base1000", keep=True),
]


@functools.lru_cache(maxsize=None)
def _recipe(recipe):
    if recipe == "fig4":
        return np.array([47], dtype=U64), np.array([(-38) & 255], dtype=U64)
    if recipe == "u8_splits":
        _, s0, s1 = all_splits_u8()
        return s0, s1
    if recipe == "minus1":
        return share_arith(np.full(16, -1, dtype=np.int64), 8, np.random.default_rng(10))
    if recipe == "w10_crit2":
        raise KeyError  # needs m; handled below
    if recipe == "w10_prune":
        rng = np.random.default_rng(12)
        x = np.arange(1024, dtype=U64)
        s1 = _words(rng, 1024) & U64(1023)
        return (x - s1) & U64(1023), s1
    if recipe == "zero32":
        return share_arith(np.zeros(32, dtype=U64), 10, np.random.default_rng(11))
    if recipe == "sim10k":
        rng = np.random.default_rng(5)
        x_f = rng.uniform(-20, 20, 10_000)
        return share_arith(encode(x_f), 64, rng)
    if recipe == "arange37":
        return share_arith(np.arange(37, dtype=U64), 64, np.random.default_rng(13))
    if recipe == "fill33":
        return share_arith(np.full(33, 2**40, dtype=U64), 64, np.random.default_rng(14))
    if recipe == "arange50":
        return share_arith(np.arange(50, dtype=U64), 64, np.random.default_rng(15))
    if recipe == "arange8_64":
        return share_arith(np.arange(8, dtype=U64), 64, np.random.default_rng(64))
    if recipe == "arange8_10":
        return share_arith(np.arange(8, dtype=U64), 10, np.random.default_rng(10))
    if recipe == "arange8_64b":
        return share_arith(np.arange(8, dtype=U64), 64, np.random.default_rng(65))
    if recipe == "base4096":
        return baseline_inputs(4096)
    if recipe == "base1001":
        return baseline_inputs(1001, seed=7)
    if recipe == "base1000":
        return baseline_inputs(1000, seed=8)
    raise KeyError(recipe)


def make_inputs(case):
    if case["recipe"] == "w10_crit2":
        m = case["m"]
        rng = np.random.default_rng(100 + m)
        x = np.repeat(np.arange(1024, dtype=U64), 64)
        s1 = _words(rng, x.size) & U64(1023)
        return (x - s1) & U64(1023), s1
    x0, x1 = _recipe(case["recipe"])
    return x0.copy(), x1.copy()


STAGE_CASES = [
    dict(name="bmul_w8_exh", op="beaver_mul", w=8, seed=0, recipe="bmul_w8"),
    dict(name="band_w3", op="beaver_and", w=3, seed=0, recipe="band", keep=True),
    dict(name="band_w8", op="beaver_and", w=8, seed=0, recipe="band", keep=True),
    dict(name="band_w64", op="beaver_and", w=64, seed=0, recipe="band", keep=True),
    dict(name="cadd_w8_exh", op="circuit_add", w=8, seed=0, recipe="cadd_w8"),
    dict(name="cadd_w64_zero", op="circuit_add", w=64, seed=0, recipe="cadd_w64", keep=True),
    dict(name="a2b_w8_exh", op="a2b", w=8, seed=0, recipe="a2b_w8"),
    dict(name="a2b_w16", op="a2b", w=16, seed=1, recipe="a2b_w16", keep=True),
    dict(name="b2a_n8", op="b2a", n_bits=8, seed=0, recipe="b2a", keep=True),
    dict(name="b2a_n64", op="b2a", n_bits=64, seed=0, recipe="b2a", keep=True),
]


@functools.lru_cache(maxsize=None)
def _band_all():
    """test_protocol.py:170-181 draws all three widths from one generator."""
    rng = np.random.default_rng(5)
    out = {}
    for width in (3, 8, 64):
        x = _words(rng, 500) & _mask(width)
        y = _words(rng, 500) & _mask(width)
        x0, x1 = share_binary(x, width, rng)
        y0, y1 = share_binary(y, width, rng)
        out[width] = dict(x0=x0, x1=x1, y0=y0, y1=y1, x=x, y=y)
    return out


def make_stage_inputs(case):
    r = case["recipe"]
    if r == "bmul_w8":
        rng = np.random.default_rng(1)
        a, b = all_pairs_u8()
        x0, x1 = share_arith(a, 8, rng)
        y0, y1 = share_arith(b, 8, rng)
        return dict(x0=x0, x1=x1, y0=y0, y1=y1, x=a, y=b)
    if r == "band":
        return {k: v.copy() for k, v in _band_all()[case["w"]].items()}
    if r == "cadd_w8":
        rng = np.random.default_rng(7)
        a, b = all_pairs_u8()
        x0, x1 = share_binary(a, 8, rng)
        y0, y1 = share_binary(b, 8, rng)
        return dict(x0=x0, x1=x1, y0=y0, y1=y1, x=a, y=b)
    if r == "cadd_w64":
        rng = np.random.default_rng(6)
        b = _words(rng, 100)
        x0, x1 = share_binary(np.zeros(100, dtype=U64), 64, rng)
        y0, y1 = share_binary(b, 64, rng)
        return dict(x0=x0, x1=x1, y0=y0, y1=y1, x=np.zeros(100, dtype=U64), y=b)
    if r == "a2b_w8":
        x, s0, s1 = all_splits_u8()
        return dict(x0=s0, x1=s1, x=x)
    if r == "a2b_w16":
        rng = np.random.default_rng(1)
        x = np.arange(100, dtype=U64)
        x0, x1 = share_arith(x, 16, rng)
        return dict(x0=x0, x1=x1, x=x)
    if r == "b2a":
        return dict(x0=np.array([0, 0, 1, 1], dtype=U64), x1=np.array([0, 1, 0, 1], dtype=U64))
    raise KeyError(r)


# ------------------------------------------------------------------ ring linear layers (nn.py:198-259)
NN_CASES = [
    dict(name="nn_linear", op="linear", x_shape=(12, 40), w_shape=(24, 40)),
    dict(name="nn_linear_big", op="linear", x_shape=(33, 300), w_shape=(10, 300), w_scale=3.0),
    dict(name="nn_conv", op="conv", x_shape=(3, 5, 9, 9), w_shape=(7, 5, 3, 3), layer=(5, 7, 3, 3, 2, 1)),
    dict(name="nn_conv_1x1", op="conv", x_shape=(2, 6, 8, 8), w_shape=(4, 6, 1, 1), layer=(6, 4, 1, 1, 2, 0)),
    dict(name="nn_conv_stem", op="conv", x_shape=(2, 3, 8, 8), w_shape=(16, 3, 3, 3), layer=(3, 16, 3, 3, 1, 1)),
    dict(name="nn_avgpool", op="avgpool", x_shape=(3, 7, 8, 8), layer=(2, 2, 2)),
    dict(name="nn_avgpool_4", op="avgpool", x_shape=(2, 5, 8, 8), layer=(4, 4, 4)),
    dict(name="nn_truncate", op="truncate", x_shape=(1000,)),
]


def make_nn_inputs(case):
    """Shares of encoded N(0, 4^2) activations and N(0, 0.2^2) weights (seeded by the case name)."""
    seed = sum(ord(ch) for ch in case["name"])
    rng = np.random.default_rng(seed)
    x_f = rng.normal(0, 4.0, case["x_shape"])
    x0, x1 = share_arith(encode(x_f), 64, rng)
    out = dict(x0=x0, x1=x1)
    if "w_shape" in case:
        out["w"] = (rng.normal(0, 0.2 * case.get("w_scale", 1.0), case["w_shape"])).astype(np.float32)
        out["b"] = rng.normal(0, 0.5, case["w_shape"][0]).astype(np.float32)
    return out


MODEL_CASES = [
    dict(name="model_cnn_full", arch="cnn", windows=[(64, 0), (64, 0)], seed=5, batch=16),
    dict(name="model_cnn_reduced", arch="cnn", windows=[(20, 8), (19, 6)], seed=5, batch=16),
    dict(name="model_cnn_identity", arch="cnn", windows=[None, (22, 14)], seed=7, batch=8),
    dict(name="model_mlp_reduced", arch="mlp", windows=[(21, 13)], seed=3, batch=32),
]


def model_inputs(mc):
    rng = np.random.default_rng(77 + mc["batch"])
    shape = (mc["batch"], 1, 8, 8) if mc["arch"] == "cnn" else (mc["batch"], 64)
    return rng.uniform(0.0, 1.0, shape)


def _conv(cin, cout, k, stride, pad, w, b):
    return dict(kind="conv2d", in_channels=cin, out_channels=cout, kh=k, kw=k, stride=stride, pad=pad, weight=w, bias=b)


# layer lists of the reference desk models (models.py:33-72), as manifest JSON entries (nn.py:440-455)
MODEL_LAYERS = {
    "cnn": ([_conv(1, 8, 3, 1, 1, "conv1.w", "conv1.b"), dict(kind="relu", group_id=0),
             dict(kind="avgpool", kh=2, kw=2, stride=2), _conv(8, 16, 3, 1, 1, "conv2.w", "conv2.b"),
             dict(kind="relu", group_id=1), dict(kind="avgpool", kh=2, kw=2, stride=2), dict(kind="flatten"),
             dict(kind="linear", in_features=64, out_features=10, weight="fc.w", bias="fc.b")], (1, 8, 8)),
    "mlp": ([dict(kind="linear", in_features=64, out_features=32, weight="fc1.w", bias="fc1.b"),
             dict(kind="relu", group_id=0),
             dict(kind="linear", in_features=32, out_features=10, weight="fc2.w", bias="fc2.b")], (64,)),
}


def model_weights(arrays, arch):
    pre = f"model_{arch}/"
    return {k[len(pre):]: v for k, v in arrays.items() if k.startswith(pre)}


# ---------------------------------------------------------------- simulator (simulator.py:33-174)
SIM_RELU_CASES = [
    dict(name="simrelu_22_14", k=22, m=14, n=20000, seed=31, split_seed=[9, 2]),
    dict(name="simrelu_64_0", k=64, m=0, n=5001, seed=32, split_seed=[9, 3]),
    dict(name="simrelu_20_6", k=20, m=6, n=7777, seed=33, split_seed=[4, 1]),
]

SIM_MODEL_CASES = [
    dict(name="sim_cnn_reduced", arch="cnn", windows=[(20, 8), (19, 6)], seed=3, batch=16),
    dict(name="sim_cnn_mixed", arch="cnn", windows=[None, (22, 14)], seed=5, batch=16),
    dict(name="sim_mlp_reduced", arch="mlp", windows=[(21, 13)], seed=7, batch=32),
]


def sim_relu_input(case):
    return np.random.default_rng(case["seed"]).normal(0.0, 4.0, case["n"])


def sim_model_inputs(mc):
    rng = np.random.default_rng(91 + mc["batch"])
    shape = (mc["batch"], 1, 8, 8) if mc["arch"] == "cnn" else (mc["batch"], 64)
    return rng.uniform(0.0, 1.0, shape), rng.integers(0, 10, mc["batch"])


# ---------------------------------------------------------------- window search (search.py:159-334)
SEARCH_CASES = [
    dict(name="search_eco_cnn", kind="eco", seed=4, batch=24),
    dict(name="search_budget_cnn_quarter", kind="budget", budget="1/4", widths=[0, 4, 8, 12, 16], seed=6, batch=24),
    dict(name="search_budget_cnn_eighth", kind="budget", budget="1/8", widths=[0, 2, 4, 6, 8], seed=8, batch=24),
]


def search_inputs(case):
    rng = np.random.default_rng(123 + case["batch"] + case["seed"])
    return rng.uniform(0.0, 1.0, (case["batch"], 1, 8, 8)), rng.integers(0, 10, case["batch"])
