"""GPU parity: the CUDA path against the reference's golden vectors and the oracle.

Bar (integer ring work): bit-exact.  Per-party output shares, per-round
payload bytes (SHA-256) and meter traces must equal what the reference
produced on the same inputs with the same dealer seeds (tests/golden/),
through both the per-party staged driver (run_parties + LocalEndpoint, the
reference's own test harness shape) and the fused 1-GPU pair kernel.
"""

import numpy as np
import pytest
import torch

import golden_cases as gc
from hb_helpers import make_sessions, sha, stocked_sessions_for_relu
from oracle import hb_oracle as O
from paper_2309_04875_b200 import protocol, sharing, transport
from paper_2309_04875_b200.errors import ConfigError, TripleExhaustedError, WindowError
from paper_2309_04875_b200.ring import BitWindow
from paper_2309_04875_b200.sharing import ArithShareTensor, BinShareTensor

pytestmark = pytest.mark.gpu


def _relu_case(case, path, on_device=False):
    x0, x1 = gc.make_inputs(case)
    win = BitWindow(case["k"], case["m"])
    s0, s1, eps = stocked_sessions_for_relu(x0.size, win.width, case["n_bits"], case["seed"], record=True)
    if on_device:
        x0, x1 = torch.from_numpy(x0.view(np.int64)).cuda(), torch.from_numpy(x1.view(np.int64)).cuda()
    t0, t1 = ArithShareTensor(0, case["n_bits"], x0), ArithShareTensor(1, case["n_bits"], x1)
    if path == "pair":
        r0, r1 = protocol.relu_pair((s0, s1), t0, t1, win, drelu_only=case["op"] == "drelu")
        torch.cuda.synchronize()
    else:
        fn = protocol.relu if case["op"] == "relu" else protocol.drelu
        r0, r1 = transport.run_parties(lambda: fn(s0, t0, win), lambda: fn(s1, t1, win), endpoints=eps)
    return r0, r1, eps, (s0, s1)


@pytest.mark.parametrize("path", ["staged", "pair"])
@pytest.mark.parametrize("case", gc.RELU_CASES, ids=[c["name"] for c in gc.RELU_CASES])
def test_relu_golden(golden, case, path):
    meta, arrays = golden
    g = meta[case["name"]]
    r0, r1, eps, sess = _relu_case(case, path)
    assert sha(r0.data) == g["y0_sha"]
    assert sha(r1.data) == g["y1_sha"]
    assert [list(t) for t in eps[0].meter.trace] == g["trace0"]
    assert [list(t) for t in eps[1].meter.trace] == g["trace1"]
    if path == "staged":
        assert eps[0].sent_sha == g["payload0_sha"]
        assert eps[1].sent_sha == g["payload1_sha"]
    w = case["k"] - case["m"]
    cost = protocol.relu_triple_cost(r0.numel, w, case["n_bits"])
    for s in sess:
        assert s.triples.consumed("bool", w) == cost[("bool", w)]
        assert s.triples.consumed("arith", case["n_bits"]) == (cost[("arith", case["n_bits"])]
                                                                // (2 if case["op"] == "drelu" else 1))
    assert eps[0].meter.to_json() == eps[1].meter.to_json()


def test_relu_device_tensors_roundtrip(golden):
    case = next(c for c in gc.RELU_CASES if c["name"] == "base4096_22_14")
    for path in ("staged", "pair"):
        r0, r1, _, _ = _relu_case(case, path, on_device=True)
        assert r0.on_device and r1.on_device
        assert sha(r0.data) == golden[0][case["name"]]["y0_sha"]


def _stage(case):
    ins = gc.make_stage_inputs(case)
    op = case["op"]
    n = ins["x0"].size
    if op == "beaver_mul":
        s0, s1, eps = make_sessions(arith_width=case["w"], arith_count=n, seed=case["seed"], record=True)
        A = [ArithShareTensor(p, case["w"], ins[f"x{p}"]) for p in (0, 1)]
        B = [ArithShareTensor(p, case["w"], ins[f"y{p}"]) for p in (0, 1)]
        fns = [lambda s, a, b: protocol.beaver_mul(s, a, b)] * 2
        args = [(s0, A[0], B[0]), (s1, A[1], B[1])]
    elif op in ("beaver_and", "circuit_add"):
        w = case["w"]
        cnt = n * (1 if op == "beaver_and" else 1 + 2 * protocol.prefix_levels(w))
        s0, s1, eps = make_sessions(bool_width=w, bool_count=cnt, seed=case["seed"], record=True)
        A = [BinShareTensor(p, w, ins[f"x{p}"]) for p in (0, 1)]
        B = [BinShareTensor(p, w, ins[f"y{p}"]) for p in (0, 1)]
        f = protocol.beaver_and if op == "beaver_and" else protocol.circuit_add
        fns = [f, f]
        args = [(s0, A[0], B[0]), (s1, A[1], B[1])]
    elif op == "a2b":
        w = case["w"]
        s0, s1, eps = make_sessions(bool_width=w, bool_count=n * (1 + 2 * protocol.prefix_levels(w)),
                                    seed=case["seed"], record=True)
        fns = [protocol.a2b] * 2
        args = [(s0, ArithShareTensor(0, w, ins["x0"])), (s1, ArithShareTensor(1, w, ins["x1"]))]
    else:
        nb = case["n_bits"]
        s0, s1, eps = make_sessions(arith_width=nb, arith_count=n, seed=case["seed"], record=True)
        fns = [lambda s, b: protocol.b2a_bit(s, b, nb)] * 2
        args = [(s0, BinShareTensor(0, 1, ins["x0"])), (s1, BinShareTensor(1, 1, ins["x1"]))]
    r0, r1 = transport.run_parties(lambda: fns[0](*args[0]), lambda: fns[1](*args[1]), endpoints=eps)
    return r0, r1, eps


@pytest.mark.parametrize("case", gc.STAGE_CASES, ids=[c["name"] for c in gc.STAGE_CASES])
def test_stage_golden(golden, case):
    g = golden[0][case["name"]]
    r0, r1, eps = _stage(case)
    assert sha(r0.data) == g["y0_sha"]
    assert sha(r1.data) == g["y1_sha"]
    assert [list(t) for t in eps[0].meter.trace] == g["trace0"]
    assert eps[0].sent_sha == g["payload0_sha"]
    assert eps[1].sent_sha == g["payload1_sha"]


def test_pack_layouts_gpu(golden):
    _, arrays = golden
    rng = np.random.default_rng(1)
    blob, offs = arrays["pack/blob"], arrays["pack/offsets"]
    for w in range(1, 65):
        n = int(rng.integers(1, 200))
        vals = np.frombuffer(rng.bytes(8 * n), dtype="<u8").copy() & np.uint64((1 << w) - 1)
        packed = transport.pack_words(vals, w)
        assert packed == blob[offs[w - 1]:offs[w]].tobytes()
        assert np.array_equal(transport.unpack_words(packed, w, n), vals)
    assert transport.pack_words(np.empty(0, dtype=np.uint64), 17) == b""
    with pytest.raises(Exception):
        transport.unpack_words(b"\x00" * 8, 1, 128)


# ------------------------------------------------------------------ oracle parity at larger sizes
@pytest.mark.parametrize("k,m", [(64, 0), (32, 0), (22, 6), (22, 14), (22, 16), (13, 0), (40, 3)])
def test_relu_vs_oracle_per_party(k, m):
    """Per-party shares equal the oracle on 2^16 BASELINE-distribution elements."""
    n = 1 << 16
    x0, x1 = gc.baseline_inputs(n, seed=11)
    w = k - m
    curs = O.stocked_cursors(n, w, 64, seed=4)
    y0o, y1o, _, _ = O.relu_pair(x0, x1, 64, k, m, curs)
    s0, s1, eps = stocked_sessions_for_relu(n, w, 64, seed=4)
    t0, t1 = ArithShareTensor(0, 64, x0), ArithShareTensor(1, 64, x1)
    r0, r1 = protocol.relu_pair((s0, s1), t0, t1, BitWindow(k, m))
    assert np.array_equal(r0.data, y0o) and np.array_equal(r1.data, y1o)
    s0, s1, eps = stocked_sessions_for_relu(n, w, 64, seed=4)
    g0, g1 = transport.run_parties(lambda: protocol.relu(s0, t0, BitWindow(k, m)),
                                   lambda: protocol.relu(s1, t1, BitWindow(k, m)), endpoints=eps)
    assert np.array_equal(g0.data, y0o) and np.array_equal(g1.data, y1o)


@pytest.mark.parametrize("logn", [20, 22])
@pytest.mark.parametrize("k,m", [(64, 0), (22, 14), (22, 16)])
def test_relu_large_property(logn, k, m):
    """Size-independent check at large n: reconstruction == x * drelu_from_shares, and
    the staged and fused drivers agree share for share."""
    n = 1 << logn
    x0, x1 = gc.baseline_inputs(n, seed=logn)
    w = k - m
    s0, s1, eps = stocked_sessions_for_relu(n, w, 64, seed=logn)
    t0, t1 = ArithShareTensor(0, 64, x0), ArithShareTensor(1, 64, x1)
    r0, r1 = protocol.relu_pair((s0, s1), t0, t1, BitWindow(k, m))
    want = O.ring_mul(O.ring_add(x0, x1, 64), O.drelu_from_shares(x0, x1, 64, k, m), 64)
    assert np.array_equal(sharing.reconstruct_arith(r0, r1), want)
    s0, s1, eps = stocked_sessions_for_relu(n, w, 64, seed=logn)
    g0, g1 = transport.run_parties(lambda: protocol.relu(s0, t0, BitWindow(k, m)),
                                   lambda: protocol.relu(s1, t1, BitWindow(k, m)), endpoints=eps)
    assert np.array_equal(g0.data, r0.data) and np.array_equal(g1.data, r1.data)


@pytest.mark.parametrize("w", list(range(2, 65)))
def test_all_widths_pair_and_staged(w):
    """Every window width compiles to its own kernel: check each against the oracle
    (n = 1000, not a multiple of 8, exercises partial groups and unaligned segments)."""
    n = 1000 if w % 3 else 1024
    k, m = (w, 0) if w % 2 else (min(64, w + 5), min(64, w + 5) - w)
    x0, x1 = gc.baseline_inputs(n, seed=w)
    curs = O.stocked_cursors(n, w, 64, seed=w)
    y0o, y1o, _, _ = O.relu_pair(x0, x1, 64, k, m, curs)
    s0, s1, _ = stocked_sessions_for_relu(n, w, 64, seed=w)
    t0, t1 = ArithShareTensor(0, 64, x0), ArithShareTensor(1, 64, x1)
    r0, r1 = protocol.relu_pair((s0, s1), t0, t1, BitWindow(k, m))
    assert np.array_equal(r0.data, y0o) and np.array_equal(r1.data, y1o)
    s0, s1, eps = stocked_sessions_for_relu(n, w, 64, seed=w)
    g0, g1 = transport.run_parties(lambda: protocol.relu(s0, t0, BitWindow(k, m)),
                                   lambda: protocol.relu(s1, t1, BitWindow(k, m)), endpoints=eps)
    assert np.array_equal(g0.data, y0o) and np.array_equal(g1.data, y1o)


# ------------------------------------------------------------------ interop: GPU party vs oracle CPU party
def test_gpu_party_against_cpu_oracle_party(golden):
    """Party 0 runs on the GPU (staged driver), party 1 is the CPU oracle; they
    exchange raw wire bytes.  Both outputs must equal the reference's."""
    import queue as _q

    case = next(c for c in gc.RELU_CASES if c["name"] == "base1001_22_16")
    g = golden[0][case["name"]]
    x0, x1 = gc.make_inputs(case)
    win = BitWindow(case["k"], case["m"])
    q01, q10 = _q.Queue(), _q.Queue()

    class BytesLink(transport.Endpoint):
        def _swap(self, payload):
            blob = payload.cpu().numpy().tobytes() if isinstance(payload, torch.Tensor) else payload
            q01.put(blob)
            return q10.get()

    ep0 = BytesLink(0)
    wire1 = O.Wire(1, q01, q10)
    s0, _, _ = stocked_sessions_for_relu(x0.size, win.width, 64, case["seed"])
    s0 = protocol.ProtocolSession(ep0, s0.triples)
    curs = O.stocked_cursors(x0.size, win.width, 64, case["seed"])
    r0, y1 = transport.run_parties(lambda: protocol.relu(s0, ArithShareTensor(0, 64, x0), win),
                                   lambda: O.p_relu(1, wire1, curs[1], x1, 64, win.k, win.m))
    assert sha(r0.data) == g["y0_sha"]
    assert O.digest(y1) == g["y1_sha"]


# ------------------------------------------------------------------ error behaviour
def test_errors():
    s0, s1, eps = stocked_sessions_for_relu(8, 4, 64)
    x = ArithShareTensor(0, 64, np.arange(8, dtype=np.uint64))
    with pytest.raises(WindowError):
        protocol.relu(s0, ArithShareTensor(0, 16, np.arange(8, dtype=np.uint64)), BitWindow(20, 4))
    with pytest.raises(TripleExhaustedError):
        protocol.relu(s0, ArithShareTensor(0, 64, np.arange(16, dtype=np.uint64)), BitWindow(4, 0))
    assert s0.triples.consumed("bool", 4) == 0  # nothing consumed by the failed call
    with pytest.raises(ConfigError):
        protocol.beaver_mul(s0, x, ArithShareTensor(0, 32, np.arange(8, dtype=np.uint64)))
    with pytest.raises(ConfigError):
        ArithShareTensor(0, 64, np.arange(8, dtype=np.int32))
    b0 = BinShareTensor(0, 8, np.array([2], dtype=np.uint64))
    s0, s1, eps = make_sessions(arith_width=8, arith_count=1)
    with pytest.raises(ConfigError):
        protocol.b2a_bit(s0, b0, 8)


def test_beaver_exhaustion_raises():
    rng = np.random.default_rng(3)
    x0, x1 = sharing.share_arith(np.arange(10, dtype=np.uint64), 16, rng)
    s0, s1, eps = make_sessions(arith_width=16, arith_count=5)
    with pytest.raises(TripleExhaustedError):
        transport.run_parties(lambda: protocol.beaver_mul(s0, x0, x0), lambda: protocol.beaver_mul(s1, x1, x1),
                              endpoints=eps)


def test_theorem1_exhaustive_gpu():
    """Reference acceptance criterion 1 on the GPU pair kernel: window (k, 0) equals the
    full window for every in-range 8-bit secret and all 65536 splits, k = 2..8."""
    x, t0v, t1v = gc.all_splits_u8()
    signed = (x.astype(np.int64) ^ 128) - 128
    t0, t1 = ArithShareTensor(0, 8, t0v), ArithShareTensor(1, 8, t1v)

    def run(k):
        s0, s1, _ = stocked_sessions_for_relu(x.size, k, 8, seed=k)
        r0, r1 = protocol.relu_pair((s0, s1), t0, t1, BitWindow(k, 0), drelu_only=True)
        return sharing.reconstruct_arith(r0, r1)

    full = run(8)
    assert np.array_equal(full, (signed >= 0).astype(np.uint64))
    for k in range(2, 8):
        inr = (signed >= -(2 ** (k - 1))) & (signed < 2 ** (k - 1))
        assert np.array_equal(run(k)[inr], full[inr])


# ------------------------------------------------------------------ on-device dealer
@pytest.mark.parametrize("kind,count,width,seed", [("arith", 1000, 16, 1234), ("arith", 777, 64, 9),
                                                    ("bool", 1000, 8, 3), ("bool", 513, 6, 11), ("arith", 100, 10, 5),
                                                    ("bool", 70001, 13, 77)])
def test_device_dealer_bit_exact(kind, count, width, seed):
    from paper_2309_04875_b200 import dealer

    host = (dealer.gen_arith_triples if kind == "arith" else dealer.gen_bool_triples)(count, width, seed)
    dev = dealer.deal_exact_on_device(kind, width, count, seed)
    for p in (0, 1):
        for h, d in zip(host.party_arrays(p), dev[p]):
            assert np.array_equal(h, d.cpu().numpy().view(np.uint64))
    # a sub-range equals the same slice of the full batch (chunked stocking)
    part = dealer.deal_exact_on_device(kind, width, count, seed, first=count // 3, n=count // 2)
    assert np.array_equal(part[0][0].cpu().numpy().view(np.uint64), host.party_arrays(0)[0][count // 3:count // 3 + count // 2])


def test_device_dealer_golden_file_sha(tmp_path, golden):
    from paper_2309_04875_b200 import dealer

    dev = dealer.deal_exact_on_device("arith", 16, 1000, 1234)
    batch = dealer.TripleBatch("arith", 16, 1000, 1234,
                               tuple(tuple(t.cpu().numpy().view(np.uint64) for t in dev[p]) for p in (0, 1)))
    dealer.save_triples(batch, tmp_path / "g.bin")
    import hashlib

    assert hashlib.sha256((tmp_path / "g.bin").read_bytes()).hexdigest() == golden[0]["dealer_hbtrip1_sha"]["sha"]


def test_stock_on_device_matches_reference_stream():
    """Chunked exact stocking == gen_*_triples stocked through add_batch, stream for stream."""
    from paper_2309_04875_b200 import dealer

    a, b = dealer.TripleStore(0), dealer.TripleStore(0)
    dealer.stock_on_device((a,), (0,), "bool", 8, 10_000, 5, chunk=1024)
    b.add_batch(dealer.gen_bool_triples(10_000, 8, 5))
    va, vb = a.draw("bool", 8, 10_000), b.draw("bool", 8, 10_000)
    for x, y in zip(va.unpacked(), vb.unpacked()):
        assert np.array_equal(x, y)


def test_gpu_drelu_from_shares_and_sim_relu():
    """simulator.drelu_from_shares on the GPU == the reference arithmetic (oracle), and the
    protocol agrees with it element for element (test_simulator.py:70-88)."""
    from paper_2309_04875_b200 import ring, simulator
    from paper_2309_04875_b200.ring import FixedPointConfig

    for (k, m) in ((21, 7), (64, 0), (22, 14), (10, 3)):
        x0, x1 = gc.baseline_inputs(1 << 16, seed=k)
        got = simulator.drelu_from_shares(x0, x1, 64, BitWindow(k, m))
        assert np.array_equal(got, O.drelu_from_shares(x0, x1, 64, k, m))
    case = next(c for c in gc.RELU_CASES if c["name"] == "sim10k_21_7")
    x0, x1 = gc.make_inputs(case)
    s0, s1, eps = stocked_sessions_for_relu(x0.size, 14, 64)
    r0, r1 = transport.run_parties(lambda: protocol.relu(s0, ArithShareTensor(0, 64, x0), BitWindow(21, 7)),
                                   lambda: protocol.relu(s1, ArithShareTensor(1, 64, x1), BitWindow(21, 7)),
                                   endpoints=eps)
    keep = simulator.drelu_from_shares(x0, x1, 64, BitWindow(21, 7))
    e = (x0 + x1)
    assert np.array_equal(sharing.reconstruct_arith(r0, r1), ring.mul_mod(e, keep, 64))
    cfg = FixedPointConfig(64, 16)
    xf = np.linspace(-5, 5, 101)
    out = simulator.sim_relu(xf, BitWindow(20, 6), cfg, np.random.default_rng(6))
    e2 = ring.encode_array(xf, cfg)
    t0, t1 = sharing.share_arith(e2, 64, np.random.default_rng(6))
    ref_keep = O.drelu_from_shares(t0.data, t1.data, 64, 20, 6)
    assert np.array_equal(out != 0.0, (ref_keep == 1) & (xf != 0.0))


@pytest.mark.parametrize("n,chunk,layout", [((1 << 22) + 12345, 1 << 20, "separate"), ((1 << 22) + 7, 1 << 19, "separate"),
                                            ((1 << 22) + 99, 1 << 20, "one_buffer_reversed")])
def test_relu_pair_pinned_host_pipeline(n, chunk, layout, monkeypatch):
    """relu_pair on PINNED HOST shares (> 2^22 elements) runs the native pipeline hb_relu_pair_host
    -- H2D / kernel on element ranges / D2H over three streams, ramped chunks, a partial last chunk,
    both shares of a chunk in one two-row copy (also with party 1's share BELOW party 0's in one
    pinned buffer: the reversed row order) -- and returns host shares equal to the device path's on
    the same triples, with the same meters."""
    from paper_2309_04875_b200 import dealer

    monkeypatch.setattr(protocol, "_PIPE_CHUNK", chunk)
    k, m = 22, 14
    w, L = k - m, protocol.prefix_levels(k - m)
    rng = np.random.default_rng(n)
    x = [rng.integers(0, 2**63, n, dtype=np.uint64) for _ in range(2)]
    outs = []
    for pinned in (False, True):
        eps = transport.local_pair()
        stores = (dealer.TripleStore(0), dealer.TripleStore(1))
        dealer.stock_on_device(stores, (0, 1), dealer.BOOL, w, n * (1 + 2 * L), seed=3)
        dealer.stock_on_device(stores, (0, 1), dealer.ARITH, 64, 2 * n, seed=4)
        sess = (protocol.ProtocolSession(eps[0], stores[0]), protocol.ProtocolSession(eps[1], stores[1]))
        ts = [torch.from_numpy(v.view(np.int64)) for v in x]
        if pinned and layout == "one_buffer_reversed":
            buf = torch.cat([ts[1], ts[0]]).pin_memory()
            ts = [buf[n:], buf[:n]]
        else:
            ts = [t.pin_memory() for t in ts] if pinned else [t.cuda() for t in ts]
        r0, r1 = protocol.relu_pair(sess, ArithShareTensor(0, 64, ts[0]), ArithShareTensor(1, 64, ts[1]), BitWindow(k, m))
        if pinned:
            assert not r0.data.is_cuda
        outs.append(([np.asarray(r.data.cpu() if isinstance(r.data, torch.Tensor) else r.data).view(np.uint64)
                      for r in (r0, r1)], eps[0].meter.to_json()))
    assert np.array_equal(outs[0][0][0], outs[1][0][0]) and np.array_equal(outs[0][0][1], outs[1][0][1])
    assert outs[0][1] == outs[1][1]
    want = O.ring_mul(O.ring_add(x[0], x[1], 64), O.drelu_from_shares(x[0], x[1], 64, k, m), 64)
    assert np.array_equal(O.ring_add(outs[1][0][0], outs[1][0][1], 64), want)
