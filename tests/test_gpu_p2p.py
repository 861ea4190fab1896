"""GPU parity of the one-launch NVLink party kernel (hb_relu_p2p, protocol.relu_p2p).

The kernel is written for one party per GPU with the peer's receive buffer mapped over NVLink.
This run has one GPU, so both parties' party kernels run in one launch on the same device (CTAs
split between the parties, protocol.relu_p2p_pair), each pointing at the other's buffers
(transport.local_p2p_pair) -- the same per-party code, flags and fences; only the "remote" stores
land in local HBM.  A second test runs the two parties as two
processes on the one GPU with the buffers exchanged as CUDA IPC handles (the multi-GPU plumbing).
Bar: bit-exact per-party shares against the oracle and the fused pair kernel.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import golden_cases as gc
from hb_helpers import stocked_sessions_for_relu
from oracle import hb_oracle as O
from paper_2309_04875_b200 import protocol, sharing, transport
from paper_2309_04875_b200.errors import TransportError
from paper_2309_04875_b200.ring import BitWindow
from paper_2309_04875_b200.sharing import ArithShareTensor

pytestmark = pytest.mark.gpu


def _p2p_pair(s0, s1, t0, t1, win, links, drelu_only=False):
    links[0].timeout_s = 20.0
    out = protocol.relu_p2p_pair((s0, s1), t0, t1, win, links, drelu_only=drelu_only)
    links[0].check(sync=True)
    return out


@pytest.mark.parametrize("k,m", [(64, 0), (32, 0), (22, 6), (22, 14), (22, 16), (13, 0), (40, 3)])
def test_p2p_vs_oracle_per_party(k, m):
    n = (1 << 16) + 37  # a partial last tile
    x0, x1 = gc.baseline_inputs(n, seed=5)
    w = k - m
    curs = O.stocked_cursors(n, w, 64, seed=6)
    y0o, y1o, _, _ = O.relu_pair(x0, x1, 64, k, m, curs)
    s0, s1, eps = stocked_sessions_for_relu(n, w, 64, seed=6)
    t0, t1 = ArithShareTensor(0, 64, torch.from_numpy(x0.view(np.int64)).cuda()), \
        ArithShareTensor(1, 64, torch.from_numpy(x1.view(np.int64)).cuda())
    r0, r1 = _p2p_pair(s0, s1, t0, t1, BitWindow(k, m), transport.local_p2p_pair())
    assert np.array_equal(r0.data.cpu().numpy().view(np.uint64), y0o)
    assert np.array_equal(r1.data.cpu().numpy().view(np.uint64), y1o)
    # the reference meter trace, per party
    for ep in eps:
        assert ep.meter.trace == protocol.relu_trace(n, BitWindow(k, m), 64)


@pytest.mark.parametrize("w", [2, 3, 5, 6, 7, 8, 9, 12, 16, 17, 24, 31, 33, 48, 63, 64])
def test_p2p_widths_and_drelu(w):
    n = 3000
    k, m = (w, 0) if w % 2 else (min(64, w + 5), min(64, w + 5) - w)
    x0, x1 = gc.baseline_inputs(n, seed=w + 100)
    curs = O.stocked_cursors(n, w, 64, seed=w)
    y0o, y1o, _, _ = O.relu_pair(x0, x1, 64, k, m, curs)
    s0, s1, _ = stocked_sessions_for_relu(n, w, 64, seed=w)
    t0, t1 = ArithShareTensor(0, 64, x0), ArithShareTensor(1, 64, x1)
    r0, r1 = _p2p_pair(s0, s1, t0, t1, BitWindow(k, m), transport.local_p2p_pair())
    assert np.array_equal(r0.data, y0o) and np.array_equal(r1.data, y1o)
    # DReLU through the same kernel reconstructs to the windowed sign
    s0, s1, _ = stocked_sessions_for_relu(n, w, 64, seed=w + 1)
    d0, d1 = _p2p_pair(s0, s1, t0, t1, BitWindow(k, m), transport.local_p2p_pair(), drelu_only=True)
    assert np.array_equal(sharing.reconstruct_arith(d0, d1), O.drelu_from_shares(x0, x1, 64, k, m))


def test_p2p_sequence_growth_and_large():
    """Several layers in a row on the same links (monotonic flags, buffer growth), then 2^22."""
    links = transport.local_p2p_pair()
    for i, logn in enumerate((12, 18, 14, 22)):
        n = (1 << logn) + i
        k, m = (22, 14) if i % 2 == 0 else (64, 0)
        x0, x1 = gc.baseline_inputs(n, seed=logn)
        s0, s1, _ = stocked_sessions_for_relu(n, k - m, 64, seed=logn)
        t0 = ArithShareTensor(0, 64, torch.from_numpy(x0.view(np.int64)).cuda())
        t1 = ArithShareTensor(1, 64, torch.from_numpy(x1.view(np.int64)).cuda())
        r0, r1 = _p2p_pair(s0, s1, t0, t1, BitWindow(k, m), links)
        s0, s1, _ = stocked_sessions_for_relu(n, k - m, 64, seed=logn)
        q0, q1 = protocol.relu_pair((s0, s1), t0, t1, BitWindow(k, m))
        assert torch.equal(r0.data, q0.data) and torch.equal(r1.data, q1.data)


def test_p2p_parties_with_different_grids():
    """The parties' grids need not match (tile = cta, cta + grid, ...): party 0 with 37 CTAs and party
    1 with 101 complete bit-exact (no cross-wait, no timeout); and the agreed grid of a PeerLink pair is
    the smaller request."""
    n, k, m = (1 << 18) + 5, 22, 14
    x0, x1 = gc.baseline_inputs(n, seed=21)
    curs = O.stocked_cursors(n, k - m, 64, seed=21)
    y0o, y1o, _, _ = O.relu_pair(x0, x1, 64, k, m, curs)
    s0, s1, _ = stocked_sessions_for_relu(n, k - m, 64, seed=21)
    t0 = ArithShareTensor(0, 64, torch.from_numpy(x0.view(np.int64)).cuda())
    t1 = ArithShareTensor(1, 64, torch.from_numpy(x1.view(np.int64)).cuda())
    r0, r1 = _p2p_pair(s0, s1, t0, t1, BitWindow(k, m), transport.local_p2p_pair((37, 101)))
    assert np.array_equal(r0.data.cpu().numpy().view(np.uint64), y0o)
    assert np.array_equal(r1.data.cpu().numpy().view(np.uint64), y1o)


@pytest.mark.parametrize("sys_scope", [False, True], ids=["gpu_scope", "sys_scope"])
def test_p2p_scopes_agree(sys_scope):
    """The same-device harness (gpu-scope flags) and the cross-GPU protocol (system scope) give the
    same shares."""
    n, k, m = 50000, 22, 16
    x0, x1 = gc.baseline_inputs(n, seed=31)
    curs = O.stocked_cursors(n, k - m, 64, seed=31)
    y0o, y1o, _, _ = O.relu_pair(x0, x1, 64, k, m, curs)
    s0, s1, _ = stocked_sessions_for_relu(n, k - m, 64, seed=31)
    links = transport.local_p2p_pair()
    links[0].timeout_s = 20.0
    r0, r1 = protocol.relu_p2p_pair((s0, s1), ArithShareTensor(0, 64, x0), ArithShareTensor(1, 64, x1),
                                    BitWindow(k, m), links, sys_scope=sys_scope)
    links[0].check(sync=True)
    assert np.array_equal(r0.data, y0o) and np.array_equal(r1.data, y1o)


@pytest.mark.parametrize("k,m", [(22, 17), (22, 16), (22, 0), (22, 14), (64, 0), (40, 7)],
                         ids=["w5", "w6", "w22", "w8", "w64", "w33"])
def test_p2p_wire_bytes_are_the_reference_payload(k, m):
    """What crosses NVLink = the reference payload (transport.py:33-49, protocol.py:62-72): the kernel
    counts every byte it stores into the peer's buffer; per launch that equals hb_relu_p2p_wire_bytes,
    which is the reference trace less only the zero padding of each round's last 64-bit word."""
    from paper_2309_04875_b200 import _lib

    lib = _lib.load()
    for n in (3000, (1 << 16) + 37):
        w = k - m
        x0, x1 = gc.baseline_inputs(n, seed=w)
        s0, s1, _ = stocked_sessions_for_relu(n, w, 64, seed=w)
        links = transport.local_p2p_pair()
        counter = links[0].count_wire()
        _p2p_pair(s0, s1, ArithShareTensor(0, 64, x0), ArithShareTensor(1, 64, x1), BitWindow(k, m), links)
        ours = int(lib.hb_relu_p2p_wire_bytes(k, m, n, 0))
        assert int(counter.item()) == 2 * ours  # both parties of the one-launch harness count into it
        trace = protocol.relu_trace(n, BitWindow(k, m), 64)
        ref = sum(b for _, b in trace)
        assert 0 <= ref - ours < 8 * len(trace), (ref, ours)
        if (n * w) % 64 == 0:
            assert ours == ref


def test_p2p_parties_on_two_streams_layer_sequence():
    """Each party's kernel is its own launch on its own stream (as on two GPUs), so a party can start
    the next layer while its peer still reads the previous layer's last round.  Layers whose receive
    layouts overlap (a narrow large layer, then a wide larger one; a small layer, then a large one)
    stay bit-exact: consecutive launches alternate between the two receive regions."""
    links = transport.local_p2p_pair(max_ctas=64)
    links[0].timeout_s = links[1].timeout_s = 30.0
    st = [torch.cuda.Stream(), torch.cuda.Stream()]
    layers = [((1 << 20), (22, 20)), ((1 << 21), (64, 0)), (25088, (22, 14)), (802816, (22, 14)),
              ((1 << 20) + 3, (22, 20)), ((1 << 21), (64, 0))]
    sess = [stocked_sessions_for_relu(n, k - m, 64, seed=40 + i)[:2] for i, (n, (k, m)) in enumerate(layers)]
    ins = [gc.baseline_inputs(n, seed=50 + i) for i, (n, _) in enumerate(layers)]
    dev_in = [(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda()) for a, b in ins]
    # grow the buffers to the largest layer first (a growth synchronises the device)
    sizes = [_lib_bytes(n, km) for n, km in layers]
    links[0].ensure(max(b for b, _ in sizes), max(t for _, t in sizes))
    torch.cuda.synchronize()
    # outputs allocated up front: an allocation between the two parties' launches can make the caching
    # allocator synchronise the device (cudaFree), which would wait on the first party's spinning kernel
    ybuf = [[torch.empty(n, dtype=torch.int64, device="cuda") for _ in (0, 1)] for n, _ in layers]
    torch.cuda.synchronize()
    outs = []
    for i, (n, (k, m)) in enumerate(layers):
        ys = []
        for p in (0, 1):
            with torch.cuda.stream(st[p]):
                ys.append(protocol.relu_p2p(sess[i][p], ArithShareTensor(p, 64, dev_in[i][p]), BitWindow(k, m),
                                            links[p], stream=st[p], out=ybuf[i][p]))
        outs.append(ys)
    for lk in links:
        lk.check(sync=True)
    # each party's kernels advanced its own device link state by every launch's rounds
    want_seq = sum(protocol.prefix_levels(k - m) + 3 for _, (k, m) in layers)
    for lk in links:
        assert lk.state.tolist() == [want_seq, len(layers), 0]
    for i, (n, (k, m)) in enumerate(layers):
        q0, q1 = stocked_sessions_for_relu(n, k - m, 64, seed=40 + i)[:2]
        w0, w1 = protocol.relu_pair((q0, q1), ArithShareTensor(0, 64, dev_in[i][0]), ArithShareTensor(1, 64, dev_in[i][1]),
                                    BitWindow(k, m))
        assert torch.equal(outs[i][0].data, w0.data) and torch.equal(outs[i][1].data, w1.data), i


def _lib_bytes(n, km):
    import ctypes

    from paper_2309_04875_b200 import _lib

    nt = ctypes.c_int64(0)
    return _lib.load().hb_relu_p2p_bytes(km[0], km[1], n, 0, ctypes.byref(nt)), nt.value


def test_p2p_missing_peer_times_out():
    """Only party 0 runs (relu_p2p, one party): its kernel gives up after the timeout and the
    link raises instead of hanging."""
    links = transport.local_p2p_pair()
    links[0].timeout_s = 0.05
    n = 4096
    x0, _ = gc.baseline_inputs(n, seed=1)
    s0, _, _ = stocked_sessions_for_relu(n, 8, 64, seed=1)
    protocol.relu_p2p(s0, ArithShareTensor(0, 64, x0), BitWindow(22, 14), links[0])
    with pytest.raises(TransportError):
        links[0].check(sync=True)


_CHILD = r"""
import os, sys
sys.path.insert(0, os.environ["HB_ROOT"]); sys.path.insert(0, os.path.join(os.environ["HB_ROOT"], "tests"))
import numpy as np, torch, torch.distributed as dist
import golden_cases as gc
from hb_helpers import stocked_sessions_for_relu
from paper_2309_04875_b200 import protocol, transport
from paper_2309_04875_b200.protocol import ProtocolSession
from paper_2309_04875_b200.ring import BitWindow
from paper_2309_04875_b200.sharing import ArithShareTensor
rank = int(os.environ["RANK"])
dist.init_process_group("gloo", rank=rank, world_size=2)
n, k, m = 20000, 22, 14
x0, x1 = gc.baseline_inputs(n, seed=3)
s0, s1, _ = stocked_sessions_for_relu(n, k - m, 64, seed=3)
sess = (s0, s1)[rank]
ep = transport.DistEndpoint(rank, 1 - rank)
ep.enable_p2p(timeout_s=60.0)
session = ProtocolSession(ep, sess.triples)
x = ArithShareTensor(rank, 64, torch.from_numpy((x0, x1)[rank].view(np.int64)).cuda())
y = protocol.relu(session, x, BitWindow(k, m))
ep.p2p.check(sync=True)
np.save(os.environ["HB_OUT"] + f"/y{rank}.npy", y.data.cpu().numpy())
dist.barrier()
ep.p2p.close()
dist.destroy_process_group()
"""


def test_p2p_two_processes_ipc(tmp_path):
    """Two party processes on the one GPU, receive buffers exchanged as CUDA IPC handles over a
    gloo group (the multi-GPU plumbing; kernels of two processes time-slice on one device)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   HB_ROOT=root, HB_OUT=str(tmp_path))
        procs.append(subprocess.Popen([sys.executable, "-c", _CHILD], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT))
    outs = [p.communicate(timeout=300)[0].decode(errors="replace") for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    y0, y1 = np.load(tmp_path / "y0.npy"), np.load(tmp_path / "y1.npy")
    x0, x1 = gc.baseline_inputs(20000, seed=3)
    s0, s1, _ = stocked_sessions_for_relu(20000, 8, 64, seed=3)
    q0, q1 = protocol.relu_pair((s0, s1), ArithShareTensor(0, 64, x0), ArithShareTensor(1, 64, x1), BitWindow(22, 14))
    assert np.array_equal(y0.view(np.uint64), np.asarray(q0.data).view(np.uint64))
    assert np.array_equal(y1.view(np.uint64), np.asarray(q1.data).view(np.uint64))


def test_p2p_layers_replayed_as_cuda_graph():
    """A sequence of layers through the NVLink party kernels captured in ONE CUDA graph and replayed
    twice: the flag sequence and the receive-region parity live on the device (PeerLink.state, the
    kernel's last CTA advances them), so the launch arguments never change and every replay is a
    fresh, correctly sequenced run -- shares equal the eager launches' on the same triples."""
    links = transport.local_p2p_pair()
    links[0].timeout_s = 20.0
    layers = [((1 << 16) + 5, (22, 14)), ((1 << 18), (64, 0)), (40000, (20, 6))]
    sess, ins = [], []
    for i, (n, (k, m)) in enumerate(layers):
        x0, x1 = gc.baseline_inputs(n, seed=50 + i)
        s0, s1, _ = stocked_sessions_for_relu(n, k - m, 64, seed=60 + i)
        sess.append((s0, s1))
        ins.append((ArithShareTensor(0, 64, torch.from_numpy(x0.view(np.int64)).cuda()),
                    ArithShareTensor(1, 64, torch.from_numpy(x1.view(np.int64)).cuda())))

    def forward():
        return [protocol.relu_p2p_pair(s, a, b, BitWindow(*km), links) for s, (a, b), (_, km) in zip(sess, ins, layers)]

    def rewind():
        for (s0, s1), (_, (k, m)) in zip(sess, layers):
            for s in (s0, s1):
                s.triples.rewind("bool", k - m)
                s.triples.rewind("arith", 64)

    want = [(a.data.clone(), b.data.clone()) for a, b in forward()]  # eager (also sizes the buffers)
    links[0].check(sync=True)
    launches0, seq0 = int(links[0].state[1]), int(links[0].state[0])
    rewind()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        outs = forward()
    for _ in range(2):
        g.replay()
        links[0].check(sync=True)
        for (a, b), (wa, wb) in zip(outs, want):
            assert torch.equal(a.data, wa) and torch.equal(b.data, wb)
    # every replayed launch advanced both parties' device sequences identically, by its rounds, and
    # the last CTA reset the done counter
    assert torch.equal(links[0].state[:2], links[1].state[:2])
    assert int(links[0].state[1]) == launches0 + 2 * len(layers)
    assert int(links[0].state[2]) == 0 and int(links[1].state[2]) == 0
    seq_per_pass = sum(protocol.prefix_levels(k - m) + 3 for _, (k, m) in layers)
    assert int(links[0].state[0]) == seq0 + 2 * seq_per_pass
