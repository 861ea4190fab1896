"""Pin the CPU oracle against vectors produced by the reference package itself.

Every golden case (tests/golden/golden.json, made by make_golden.py from the
reference ringmpc) is replayed through oracle/hb_oracle.py with the same
inputs and the same dealer seeds; per-party output shares, per-round payload
digests and meter traces must match exactly.  CPU only.
"""

import hashlib

import numpy as np
import pytest

import golden_cases as gc
from oracle import hb_oracle as O


def _sha_bytes(b):
    return hashlib.sha256(b).hexdigest()


@pytest.mark.parametrize("case", gc.RELU_CASES, ids=[c["name"] for c in gc.RELU_CASES])
def test_relu_cases(golden, case):
    meta, arrays = golden
    g = meta[case["name"]]
    x0, x1 = gc.make_inputs(case)
    w = case["k"] - case["m"]
    curs = O.stocked_cursors(x0.size, w, case["n_bits"], case["seed"])
    y0, y1, w0, w1 = O.relu_pair(x0, x1, case["n_bits"], case["k"], case["m"], curs,
                                 keep_payloads=True, op=case["op"])
    assert O.digest(y0) == g["y0_sha"]
    assert O.digest(y1) == g["y1_sha"]
    assert [list(t) for t in w0.trace] == g["trace0"]
    assert [list(t) for t in w1.trace] == g["trace1"]
    assert [_sha_bytes(p) for p in w0.sent] == g["payload0_sha"]
    assert [_sha_bytes(p) for p in w1.sent] == g["payload1_sha"]
    assert w0.trace == O.analytic_trace(x0.size, w, case["n_bits"])[: len(w0.trace)]
    if case.get("keep"):
        assert np.array_equal(y0, arrays[case["name"] + "/y0"])


def test_fig4_values(golden):
    _, arrays = golden
    assert int(arrays["fig4_drelu/recon"][0]) == 1
    assert int(arrays["fig4_relu/recon"][0]) == 9


def test_sim10k_matches_simulator():
    case = next(c for c in gc.RELU_CASES if c["name"] == "sim10k_21_7")
    x0, x1 = gc.make_inputs(case)
    curs = O.stocked_cursors(x0.size, 14, 64, 0)
    y0, y1, _, _ = O.relu_pair(x0, x1, 64, 21, 7, curs)
    keep = O.drelu_from_shares(x0, x1, 64, 21, 7)
    assert np.array_equal(O.ring_add(y0, y1, 64), O.ring_mul(O.ring_add(x0, x1, 64), keep, 64))


def _stage_run(case):
    ins = gc.make_stage_inputs(case)
    op = case["op"]
    cur = (O.Cursor(0), O.Cursor(1))
    n = ins["x0"].size
    if op == "beaver_mul":
        t = O.deal("arith", n, case["w"], 2 * case["seed"] + 2)
        for p in (0, 1):
            cur[p].stock("arith", case["w"], t[p])
        fns = [lambda p=p, wv=None: O.p_mul(p, wv, cur[p], ins[f"x{p}"], ins[f"y{p}"], case["w"]) for p in (0, 1)]
    elif op in ("beaver_and", "circuit_add", "a2b"):
        w = case["w"]
        cnt = n * (1 if op == "beaver_and" else 1 + 2 * O.levels_for(w))
        t = O.deal("bool", cnt, w, 2 * case["seed"] + 1)
        for p in (0, 1):
            cur[p].stock("bool", w, t[p])
        if op == "beaver_and":
            fns = [lambda p=p, wv=None: O.p_and(p, wv, cur[p], ins[f"x{p}"], ins[f"y{p}"], w) for p in (0, 1)]
        elif op == "circuit_add":
            fns = [lambda p=p, wv=None: O.p_adder(p, wv, cur[p], ins[f"x{p}"], ins[f"y{p}"], w) for p in (0, 1)]
        else:
            fns = [lambda p=p, wv=None: O.p_a2b(p, wv, cur[p], ins[f"x{p}"], w) for p in (0, 1)]
    else:
        nb = case["n_bits"]
        t = O.deal("arith", n, nb, 2 * case["seed"] + 2)
        for p in (0, 1):
            cur[p].stock("arith", nb, t[p])
        fns = [lambda p=p, wv=None: O.p_b2a(p, wv, cur[p], ins[f"x{p}"], nb) for p in (0, 1)]
    w0, w1 = O.wire_pair(keep_payloads=True)
    y0, y1 = O.run_two(lambda: fns[0](wv=w0), lambda: fns[1](wv=w1), (w0, w1))
    return y0, y1, w0, w1


@pytest.mark.parametrize("case", gc.STAGE_CASES, ids=[c["name"] for c in gc.STAGE_CASES])
def test_stage_cases(golden, case):
    meta, _ = golden
    g = meta[case["name"]]
    y0, y1, w0, w1 = _stage_run(case)
    assert O.digest(y0) == g["y0_sha"]
    assert O.digest(y1) == g["y1_sha"]
    assert [list(t) for t in w0.trace] == g["trace0"]
    assert [_sha_bytes(p) for p in w0.sent] == g["payload0_sha"]
    assert [_sha_bytes(p) for p in w1.sent] == g["payload1_sha"]


def test_pack_layouts(golden):
    _, arrays = golden
    rng = np.random.default_rng(1)
    blob, offs, counts = arrays["pack/blob"], arrays["pack/offsets"], arrays["pack/counts"]
    for w in range(1, 65):
        n = int(rng.integers(1, 200))
        vals = np.frombuffer(rng.bytes(8 * n), dtype="<u8").copy() & np.uint64((1 << w) - 1)
        assert n == counts[w - 1]
        packed = O.pack_stream(vals, w)
        assert packed == blob[offs[w - 1]:offs[w]].tobytes()
        assert np.array_equal(O.unpack_stream(packed, w, n), vals)


def test_pack_known_layouts():
    vals = np.array([0x0123456789ABCDEF, 0, 2**64 - 1], dtype=np.uint64)
    assert O.pack_stream(vals, 64) == vals.astype("<u8").tobytes()
    assert O.pack_stream(np.ones(64, dtype=np.uint64), 1) == (2**64 - 1).to_bytes(8, "little")
    with pytest.raises(ValueError):
        O.unpack_stream(b"\x00" * 8, 1, 128)


def test_dealer_streams(golden):
    meta, _ = golden
    for key, want in meta["dealer_streams"].items():
        kind, w, seed, cnt = key.split("_")
        t = O.deal(kind, int(cnt), int(w), int(seed))
        assert [O.digest(a) for p in (0, 1) for a in t[p]] == want


def test_analytic_bytes_table():
    """W(w) per element for large n."""
    n = 1 << 16
    for w, want in ((64, 240), (32, 120), (16, 68), (8, 46), (6, 42.5)):
        tot = sum(nb for _, nb in O.analytic_trace(n, w, 64))
        assert tot / n == want


# ------------------------------------------------------------------ ring layers / model level
from oracle import hb_oracle_nn as ON  # noqa: E402


def _nn_oracle(case, ins, party):
    x = ins[f"x{party}"]
    if case["op"] == "linear":
        return ON.linear(x, party, ins["w"], ins["b"])
    if case["op"] == "conv":
        cin, cout, kh, kw, s, p = case["layer"]
        return ON.conv2d(x, party, cin, cout, kh, kw, s, p, ins["w"], ins["b"])
    if case["op"] == "avgpool":
        return ON.avgpool(x, party, *case["layer"])
    return ON.truncate(x, party)


@pytest.mark.parametrize("case", gc.NN_CASES, ids=[c["name"] for c in gc.NN_CASES])
def test_nn_layers(golden, case):
    g = golden[0][case["name"]]
    ins = gc.make_nn_inputs(case)
    for p in (0, 1):
        y = _nn_oracle(case, ins, p)
        assert list(y.shape) == g["shape"]
        assert O.digest(y) == g[f"y{p}_sha"]


@pytest.mark.parametrize("mc", gc.MODEL_CASES, ids=[c["name"] for c in gc.MODEL_CASES])
def test_model_run_local_forward(golden, mc):
    meta, arrays = golden
    g = meta[mc["name"]]
    layers, in_shape = gc.MODEL_LAYERS[mc["arch"]]
    weights = gc.model_weights(arrays, mc["arch"])
    logits, traces, logs = ON.run_local_forward(layers, in_shape, weights, mc["windows"], gc.model_inputs(mc),
                                                mc["seed"])
    assert O.digest(np.ascontiguousarray(logits).view(np.uint64)) == g["logits_sha"]
    assert logs[0] == g["layers0"] and logs[1] == g["layers1"]
    tot = O.tag_totals(traces[0])
    assert {t: {"bytes": tot[t][0], "rounds": tot[t][1]} for t in O.TAGS} == g["meter0"]["tags"]


# ---------------------------------------------------------------- simulator (simulator.py:33-174)
from oracle import hb_oracle_sim as OS  # noqa: E402


@pytest.mark.parametrize("case", gc.SIM_RELU_CASES, ids=[c["name"] for c in gc.SIM_RELU_CASES])
def test_sim_relu_oracle(golden, case):
    meta, arrays = golden
    rng = np.random.default_rng(np.random.SeedSequence(case["split_seed"]))
    out = OS.sim_relu(gc.sim_relu_input(case), case["k"], case["m"], rng)
    assert np.array_equal(out.view(np.uint64), arrays[case["name"] + "/out"].view(np.uint64))


@pytest.mark.parametrize("mc", gc.SIM_MODEL_CASES, ids=[c["name"] for c in gc.SIM_MODEL_CASES])
def test_sim_forward_oracle(golden, mc):
    meta, arrays = golden
    g = meta[mc["name"]]
    layers, _ = gc.MODEL_LAYERS[mc["arch"]]
    weights = gc.model_weights(arrays, mc["arch"])
    x_f, labels = gc.sim_model_inputs(mc)
    logits, acc = OS.sim_forward(layers, weights, x_f, labels, mc["windows"], mc["seed"])
    assert np.array_equal(logits, arrays[mc["name"] + "/logits"]) and acc == g["accuracy"]
    _, masks = OS.collect_drelu_decisions(layers, weights, x_f, mc["windows"], mc["seed"])
    assert len(masks) == g["n_masks"]
    for i, mk in enumerate(masks):
        assert np.array_equal(mk, arrays[mc["name"] + f"/mask{i}"])
    assert np.array_equal(OS.plain_forward(layers, weights, x_f), arrays[mc["name"] + "/plain"])
    assert {str(k): v for k, v in OS.collect_activation_ranges(layers, weights, x_f).items()} == g["ranges"]
