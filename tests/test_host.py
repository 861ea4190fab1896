"""CPU-only checks: the C ABI loads and exports every declared symbol, the
host-side cost model / metering / configuration / dealer logic, and the
endpoints (LocalEndpoint, TCP, torch.distributed gloo with world_size 2)."""

import hashlib
import os
import re
import socket
import threading

import numpy as np
import pytest

from oracle import hb_oracle as O
from paper_2309_04875_b200 import _lib, dealer, protocol, transport
from paper_2309_04875_b200.errors import (ConfigError, DataFormatError, TransportError, TripleExhaustedError,
                                          WindowError)
from paper_2309_04875_b200.ring import BitWindow, FixedPointConfig
from paper_2309_04875_b200.transport import Meter, local_pair, run_parties

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_abi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "hb_relu.h")).read()
    declared = set(re.findall(r"\b(hb_\w+)\s*\(", header))
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTED)


@pytest.mark.parametrize("w", [2, 3, 4, 6, 8, 13, 16, 21, 32, 64])
def test_cost_model_matches_oracle(w):
    lib = _lib.load()
    assert lib.hb_prefix_levels(w) == protocol.prefix_levels(w) == O.levels_for(w)
    for n in (1, 37, 1000, 1 << 20):
        k, m = (w, 0)
        trace = protocol.relu_trace(n, BitWindow(k, m), 64)
        assert trace == O.analytic_trace(n, w, 64)
        assert trace[:-1] == protocol.relu_trace(n, BitWindow(k, m), 64, drelu_only=True)
        assert lib.hb_payload_bytes(n, w) == O.stream_nbytes(n, w)


def test_abi_rejects_bad_configs_before_any_kernel():
    lib = _lib.load()
    t = _lib.Triples(0, 0, 0, 0, 0, 8)
    for ring_bits, k, m in ((64, 5, 4), (64, 65, 0), (16, 20, 4), (0, 8, 0)):
        rc = lib.hb_relu_pair(ring_bits, k, m, 8, None, None, None, None, t, t, t, t, 0, None)
        assert rc == _lib.HB_ERR_CONFIG
    rc = lib.hb_relu_pair(64, 8, 0, 8, None, None, None, None, t, t, _lib.Triples(0, 0, 0, 0, 0, 64),
                          _lib.Triples(0, 0, 0, 0, 0, 64), 0, None)
    assert rc == _lib.HB_ERR_TRIPLES
    with pytest.raises(TripleExhaustedError):
        _lib.check(rc)
    assert b"needs" in lib.hb_last_error()


def test_window_validation():
    for k, m in ((5, 4), (65, 0), (3, 3), (2, -1)):
        with pytest.raises(WindowError):
            BitWindow(k, m)
    with pytest.raises(WindowError):
        BitWindow(20, 4).check_fits(16)
    assert BitWindow(22, 14).width == 8
    assert BitWindow.from_json(BitWindow(9, 2).to_json()) == BitWindow(9, 2)
    with pytest.raises(ConfigError):
        FixedPointConfig(64, 0)


def test_meter_semantics():
    m = Meter()
    m.record(10)
    assert m.bytes_sent["Other"] == 10 and m.rounds["Other"] == 1
    m = Meter()
    with m.tag("Circuit"):
        m.record(1)
        with m.tag("B2A"):
            m.record(2)
        m.record(4)
    m.record(8)
    assert m.bytes_sent == {"Circuit": 5, "Mult": 0, "B2A": 2, "Other": 8}
    assert m.trace == [("Circuit", 1), ("B2A", 2), ("Circuit", 4), ("Other", 8)]
    with pytest.raises(ConfigError):
        with m.tag("Bogus"):
            pass


def test_dealer_golden_sha(tmp_path, golden):
    meta, _ = golden
    p = tmp_path / "g.bin"
    dealer.save_triples(dealer.gen_arith_triples(1000, 16, seed=1234), p)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == meta["dealer_hbtrip1_sha"]["sha"]
    assert hashlib.sha256(p.read_bytes()).hexdigest() == "4df0822d744dc28807cbc8b47e94711a0baac20e57a38722342f76599396ac3f"
    for key, want in meta["dealer_streams"].items():
        kind, w, seed, cnt = key.split("_")
        gen = dealer.gen_arith_triples if kind == "arith" else dealer.gen_bool_triples
        b = gen(int(cnt), int(w), int(seed))
        assert [O.digest(a) for p_ in (0, 1) for a in b.party_arrays(p_)] == want


def test_triple_file_roundtrip_and_errors(tmp_path):
    for batch in (dealer.gen_arith_triples(257, 24, seed=9), dealer.gen_bool_triples(31, 5, seed=10)):
        path = tmp_path / f"{batch.kind}.bin"
        dealer.save_triples(batch, path)
        got = dealer.load_triples(path)
        assert (got.kind, got.width, got.count, got.seed) == (batch.kind, batch.width, batch.count, batch.seed)
        for p in (0, 1):
            for x, y in zip(got.party_arrays(p), batch.party_arrays(p)):
                assert np.array_equal(x, y)
    blob = (tmp_path / "arith.bin").read_bytes()
    for bad in (blob[:-8], b"NOTMAGIC" + blob[8:], blob[:10]):
        (tmp_path / "bad.bin").write_bytes(bad)
        with pytest.raises(DataFormatError):
            dealer.load_triples(tmp_path / "bad.bin")


def test_local_pair_bytes_and_close():
    ep0, ep1 = local_pair()
    r0, r1 = run_parties(lambda: ep0.exchange(b"from0"), lambda: ep1.exchange(b"from1"))
    assert r0 == b"from1" and r1 == b"from0"
    assert ep0.meter.total_bytes() == 5 and ep0.meter.total_rounds() == 1
    ep0, ep1 = local_pair()
    ep1.close()
    with pytest.raises(TransportError):
        ep0.exchange(b"hello")
    ep0, ep1 = local_pair()

    def bad():
        raise ValueError("boom")

    with pytest.raises(ValueError, match="boom"):
        run_parties(bad, lambda: ep1.exchange(b"x"), endpoints=(ep0, ep1))


def test_length_mismatch_is_transport_error():
    ep0, ep1 = local_pair()
    with pytest.raises(TransportError):
        run_parties(lambda: ep0.exchange(b"abcd"), lambda: ep1.exchange(b"ab"), endpoints=(ep0, ep1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_tcp_loopback_exchange():
    port = _free_port()
    out = {}

    def serve():
        ep = transport.tcp_listen("127.0.0.1", port)
        out[0] = ep.exchange(b"a" * 100_000)
        ep.close()

    def dial():
        ep = transport.tcp_connect("127.0.0.1", port)
        out[1] = ep.exchange(b"b" * 100_000)
        ep.close()

    ts = [threading.Thread(target=serve), threading.Thread(target=dial)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(30)
    assert out[0] == b"b" * 100_000 and out[1] == b"a" * 100_000


def _dist_worker(rank, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    ep = transport.DistEndpoint(rank % 2, rank ^ 1)
    got = []
    with ep.tag("Circuit"):
        for i in range(3):
            got.append(ep.exchange(bytes([rank]) * (8 * (i + 1))))
    # no CUDA here: the NVLink party path cannot map the peer, both ranks agree to stay staged
    p2p = ep.enable_p2p(timeout_s=1.0)
    got.append(p2p is None and ep.p2p is None)
    q.put((rank, got, ep.meter.to_json()))
    dist.destroy_process_group()


def test_dist_endpoint_gloo_world2():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_dist_worker, args=(r, port, q)) for r in (0, 1)]
    for p in ps:
        p.start()
    res = dict((r, (g, m)) for r, g, m in (q.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(60)
    assert res[0][0] == [bytes([1]) * 8, bytes([1]) * 16, bytes([1]) * 24, True]
    assert res[1][0] == [bytes([0]) * 8, bytes([0]) * 16, bytes([0]) * 24, True]
    assert res[0][1]["tags"]["Circuit"] == {"bytes": 48, "rounds": 3}


class _WireOverEndpoint:
    """Oracle party logic (Wire.swap + tag) on top of one of this package's endpoints."""

    def __init__(self, ep):
        self.ep, self.tag, self.trace = ep, "Other", []

    def swap(self, payload: bytes) -> bytes:
        with self.ep.tag(self.tag):
            got = self.ep.exchange(payload)
        self.trace.append((self.tag, len(payload)))
        return got


def _dist_relu_worker(rank, port, q):
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import golden_cases as gc
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    case = next(c for c in gc.RELU_CASES if c["name"] == "base1001_22_16")
    xs = gc.make_inputs(case)
    w = case["k"] - case["m"]
    curs = O.stocked_cursors(xs[0].size, w, 64, case["seed"])
    ep = transport.DistEndpoint(rank, rank ^ 1)
    y = O.p_relu(rank, _WireOverEndpoint(ep), curs[rank], xs[rank], 64, case["k"], case["m"])
    q.put((rank, O.digest(y), [list(t) for t in ep.meter.trace]))
    dist.destroy_process_group()


def test_dist_relu_rounds_gloo_world2(golden):
    """The N>1 transport path: two processes, one party each, every ReLU round a
    torch.distributed send/recv (gloo here, NCCL on GPUs).  Shares and meter traces
    equal the reference's."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_dist_relu_worker, args=(r, port, q)) for r in (0, 1)]
    for p in ps:
        p.start()
    res = {r: (d, t) for r, d, t in (q.get(timeout=180) for _ in ps)}
    for p in ps:
        p.join(60)
    g = golden[0]["base1001_22_16"]
    assert res[0][0] == g["y0_sha"] and res[1][0] == g["y1_sha"]
    assert res[0][1] == g["trace0"] and res[1][1] == g["trace1"]


def test_bench_self_launches_n_ranks():
    """`bench.py --gpus N` without torchrun re-launches itself as N ranks (the driver's SCALE run form);
    rank 0's JSON line reports n_gpus = N and the pair/party map of ranks 2i / 2i+1."""
    import json
    import subprocess
    import sys

    import bench

    cmd = bench.spawn_cmd(["--gpus", "4"], 4, 29999)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo",
                          "--spawn-selftest"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["rank_sum"] == 3 and rec["party_of_rank"] == [0, 1]


def test_tma_geometry_mirror_matches_the_c_checks():
    """nn._tma_box_ok accepts exactly the output geometries hb_conv_limbs_tma accepts, so a conv the
    C side would reject falls back to the gather kernel instead of raising (advisor, round 1)."""
    from paper_2309_04875_b200 import nn

    assert nn._tma_box_ok(32, 32) and nn._tma_box_ok(4, 4, 2) and nn._tma_box_ok(1, 128)
    assert not nn._tma_box_ok(1, 384)          # OW > 256
    assert not nn._tma_box_ok(64, 128, 3)      # box width 128 x stride 3 > 256
    assert not nn._tma_box_ok(8, 64, 5)        # 64 x 5 > 256
    assert not nn._tma_box_ok(7, 7)            # 49 pixels do not tile 128
    assert not nn._tma_box_ok(16, 16, 9)       # traversal stride > 8


