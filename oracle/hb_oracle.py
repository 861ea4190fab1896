"""CPU restatement of the reduced-ring secure ReLU path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker* for the CUDA path, never part of it.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference`` arm) may import it.  The product package
``paper_2309_04875_b200`` does not import it and fails loudly without its CUDA
library.

What it restates (reference = ``ringmpc`` under /root/reference/pkg/src):

* ring arithmetic on Z/2^w with explicit masks ........ ring.py:24-77
* LSB-first w-bit packing into 64-bit LE words ......... transport.py:33-71
* one-round exchange + tagged meter trace .............. transport.py:74-133
* Beaver multiply / Beaver AND ......................... protocol.py:62-105
* Kogge-Stone adder, A2B, single-bit B2A ............... protocol.py:108-176
* windowed DReLU and ReLU .............................. protocol.py:179-199
* triple cost model .................................... protocol.py:202-213
* trusted-dealer triples (PCG64 stream layout) ......... dealer.py:50-83
* plaintext windowed sign oracle ....................... simulator.py:33-44

Parity is pinned: ``tests/golden/`` holds vectors produced by running the
reference package itself (``tests/golden/make_golden.py``), and
``tests/test_oracle_golden.py`` checks this module against every one of them
(per-party output shares, per-round payload digests, meter traces, packing
layouts, the dealer's golden SHA-256).

The two parties run on two threads that meet only in ``Wire.swap`` -- the same
execution model as the reference's ``run_parties``/``LocalEndpoint`` -- so
this module doubles as the timed CPU baseline ("kind": "port").  Its codec
deliberately keeps the reference's byte-per-bit ``unpackbits``/``packbits``
formulation so the CPU timing reflects the reference algorithm.
"""

from __future__ import annotations

import hashlib
import math
import queue
import threading
from dataclasses import dataclass, field

import numpy as np

U64 = np.uint64
TAGS = ("Circuit", "Mult", "B2A", "Other")


# ---------------------------------------------------------------- ring (ring.py:24-77)
def wmask(w: int) -> np.uint64:
    """All-ones residue mask of a w-bit ring (ring.py:24-28)."""
    assert 1 <= w <= 64
    return U64((1 << w) - 1)


def ring_add(a, b, w):
    return (a + b) & wmask(w)


def ring_sub(a, b, w):
    return (a - b) & wmask(w)


def ring_neg(a, w):
    return (~a + U64(1)) & wmask(w)


def ring_mul(a, b, w):
    return (a * b) & wmask(w)


def window_slice(v: np.ndarray, k: int, m: int) -> np.ndarray:
    """Bits m..k-1 of each residue on the (k-m)-bit ring (ring.py:69-72)."""
    return (v >> U64(m)) & wmask(k - m)


def top_bit(v: np.ndarray, w: int) -> np.ndarray:
    """Bit w-1 as 0/1 (ring.py:75-77)."""
    return (v >> U64(w - 1)) & U64(1)


def check_window(k: int, m: int, ring_bits: int) -> None:
    """BitWindow validation + check_fits (ring.py:116-128)."""
    if not (0 <= m < k <= 64) or k - m < 2:
        raise ValueError(f"bad window (k={k}, m={m})")
    if k > ring_bits:
        raise ValueError(f"window (k={k}, m={m}) exceeds ring width {ring_bits}")


def encode_fixed(x_f: np.ndarray, frac_bits: int = 16, ring_bits: int = 64) -> np.ndarray:
    """Round-half-away-from-zero fixed-point encode (ring.py:191-199)."""
    x = np.asarray(x_f, dtype=np.float64) * float(1 << frac_bits)
    r = np.copysign(np.floor(np.abs(x) + 0.5), x)
    return r.astype(np.int64).view(U64) & wmask(ring_bits)


def split_additive(secret: np.ndarray, w: int, rng: np.random.Generator):
    """(x + r, -r) split with r drawn as rng.bytes words (sharing.py:88-96, ring.py:207-213)."""
    r = np.frombuffer(rng.bytes(8 * secret.size), dtype="<u8").copy().reshape(secret.shape) & wmask(w)
    return ring_add(secret & wmask(w), r, w), ring_neg(r, w)


def split_xor(secret: np.ndarray, w: int, rng: np.random.Generator):
    """(x ^ r, r) split (sharing.py:104-110)."""
    r = np.frombuffer(rng.bytes(8 * secret.size), dtype="<u8").copy().reshape(secret.shape) & wmask(w)
    return (secret & wmask(w)) ^ r, r


# ------------------------------------------------------------- codec (transport.py:33-71)
def stream_nbytes(count: int, w: int) -> int:
    """Bytes of a packed stream: whole 64-bit words (transport.py:70-71)."""
    return 8 * ((count * w + 63) // 64)


def pack_stream(vals: np.ndarray, w: int) -> bytes:
    """Low w bits of each value, LSB-first, 64-bit LE words, zero-padded tail.

    Byte-per-bit formulation, like the reference (transport.py:33-49)."""
    vals = np.ascontiguousarray(vals, dtype=U64).reshape(-1)
    n = vals.size
    if n == 0:
        return b""
    if w == 64:
        return vals.astype("<u8").tobytes()
    bitmat = np.unpackbits(vals.astype("<u8").view(np.uint8).reshape(n, 8), axis=1, bitorder="little")
    flat = np.zeros(stream_nbytes(n, w) * 8, dtype=np.uint8)
    flat[: n * w] = bitmat[:, :w].reshape(-1)
    return np.packbits(flat, bitorder="little").tobytes()


def unpack_stream(blob: bytes, w: int, count: int) -> np.ndarray:
    """Inverse of pack_stream; length mismatch is a transport error (transport.py:52-67)."""
    if len(blob) != stream_nbytes(count, w):
        raise ValueError(f"payload is {len(blob)} bytes, expected {stream_nbytes(count, w)}")
    if count == 0:
        return np.empty(0, dtype=U64)
    if w == 64:
        return np.frombuffer(blob, dtype="<u8").copy()
    bits = np.unpackbits(np.frombuffer(blob, dtype=np.uint8), bitorder="little")[: count * w]
    full = np.zeros((count, 64), dtype=np.uint8)
    full[:, :w] = bits.reshape(count, w)
    return np.packbits(full, axis=1, bitorder="little").view("<u8").reshape(count).copy()


# ------------------------------------------------------ link + meter (transport.py:74-183)
class Wire:
    """One party's end of an in-process duplex link with a tagged trace.

    ``swap`` is one round: hand over a payload, receive the peer's
    (transport.py:129-133).  The trace records (tag, nbytes) like Meter.record
    (transport.py:87-91); ``sent`` keeps the payloads for byte-level parity.
    """

    def __init__(self, party: int, inbox: queue.Queue, outbox: queue.Queue, keep_payloads: bool = False):
        self.party = party
        self._in, self._out = inbox, outbox
        self.trace: list[tuple[str, int]] = []
        self.sent: list[bytes] = []
        self.keep = keep_payloads
        self.tag = "Other"

    def swap(self, payload: bytes) -> bytes:
        self._out.put(payload)
        got = self._in.get()
        if got is None:
            raise RuntimeError("peer closed")
        self.trace.append((self.tag, len(payload)))
        if self.keep:
            self.sent.append(payload)
        return got

    def close(self):
        self._out.put(None)


def wire_pair(keep_payloads: bool = False) -> tuple[Wire, Wire]:
    a, b = queue.Queue(), queue.Queue()
    return Wire(0, b, a, keep_payloads), Wire(1, a, b, keep_payloads)


def tag_totals(trace) -> dict[str, tuple[int, int]]:
    """Per-tag (bytes, rounds) from a trace, as Meter.snapshot (transport.py:115-116)."""
    out = {t: [0, 0] for t in TAGS}
    for tag, nb in trace:
        out[tag][0] += nb
        out[tag][1] += 1
    return {t: (v[0], v[1]) for t, v in out.items()}


def run_two(fn0, fn1, wires=None):
    """Run both party callables on threads (transport.py:271-302)."""
    res, err = [None, None], [None, None]

    def go(i, fn):
        try:
            res[i] = fn()
        except BaseException as exc:  # noqa: BLE001
            err[i] = exc
            if wires is not None:
                for wv in wires:
                    wv.close()

    ts = [threading.Thread(target=go, args=(i, f)) for i, f in enumerate((fn0, fn1))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return res[0], res[1]


# ---------------------------------------------------------- triples (dealer.py:50-83,130-171)
def _raw(rng: np.random.Generator, count: int, w: int) -> np.ndarray:
    if count == 0:
        return np.empty(0, dtype=U64)
    return np.frombuffer(rng.bytes(8 * count), dtype="<u8").copy() & wmask(w)


def deal(kind: str, count: int, w: int, seed: int):
    """Both parties' shares of `count` triples: ((a0,b0,c0),(a1,b1,c1)).

    Stream layout a, b, r_a, r_b, r_c over one PCG64 generator seeded with
    SeedSequence(seed) (dealer.py:50-83)."""
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    a, b = _raw(rng, count, w), _raw(rng, count, w)
    if kind == "arith":
        c = ring_mul(a, b, w)
        ra, rb, rc = _raw(rng, count, w), _raw(rng, count, w), _raw(rng, count, w)
        return ((ring_add(a, ra, w), ring_add(b, rb, w), ring_add(c, rc, w)),
                (ring_neg(ra, w), ring_neg(rb, w), ring_neg(rc, w)))
    c = a & b
    ra, rb, rc = _raw(rng, count, w), _raw(rng, count, w), _raw(rng, count, w)
    return (a ^ ra, b ^ rb, c ^ rc), (ra, rb, rc)


@dataclass
class Cursor:
    """Forward-only per-(kind, width) triple cursor (dealer.py:152-163)."""

    party: int
    streams: dict = field(default_factory=dict)
    pos: dict = field(default_factory=dict)

    def stock(self, kind: str, w: int, arrays) -> None:
        key = (kind, w)
        if key in self.streams:
            self.streams[key] = tuple(np.concatenate([o, n]) for o, n in zip(self.streams[key], arrays))
        else:
            self.streams[key] = tuple(np.array(a, dtype=U64) for a in arrays)
            self.pos[key] = 0

    def take(self, kind: str, w: int, count: int):
        key = (kind, w)
        if key not in self.streams or self.pos[key] + count > self.streams[key][0].size:
            raise LookupError(f"party {self.party}: {kind}/{w} triples exhausted")
        lo = self.pos[key]
        self.pos[key] = lo + count
        return tuple(s[lo:lo + count] for s in self.streams[key])


def levels_for(w: int) -> int:
    """Kogge-Stone prefix depth max(1, ceil(log2 w)) (protocol.py:108-110)."""
    return max(1, math.ceil(math.log2(w)))


def triple_need(count: int, w: int, ring_bits: int) -> dict:
    """Triples one ReLU consumes (protocol.py:202-213)."""
    return {("bool", w): count * (1 + 2 * levels_for(w)), ("arith", ring_bits): 2 * count}


# ----------------------------------------------------- per-party protocol (protocol.py:62-199)
def _open(wire: Wire, lhs: np.ndarray, rhs: np.ndarray, w: int, xor: bool):
    """Reveal two masked tensors in one packed round (protocol.py:62-72)."""
    mine = np.concatenate([lhs.reshape(-1), rhs.reshape(-1)])
    theirs = unpack_stream(wire.swap(pack_stream(mine, w)), w, mine.size)
    both = (mine ^ theirs) if xor else ring_add(mine, theirs, w)
    k = lhs.size
    return both[:k].reshape(lhs.shape), both[k:].reshape(rhs.shape)


def p_mul(party: int, wire: Wire, cur: Cursor, x: np.ndarray, y: np.ndarray, w: int) -> np.ndarray:
    """Beaver multiply (protocol.py:75-89)."""
    a, b, c = (t.reshape(x.shape) for t in cur.take("arith", w, x.size))
    e, f = _open(wire, ring_sub(x, a, w), ring_sub(y, b, w), w, xor=False)
    z = ring_add(c, ring_add(ring_mul(e, b, w), ring_mul(f, a, w), w), w)
    return ring_add(z, ring_mul(e, f, w), w) if party == 0 else z


def p_and(party: int, wire: Wire, cur: Cursor, x: np.ndarray, y: np.ndarray, w: int) -> np.ndarray:
    """Beaver AND on w-bit words (protocol.py:92-105)."""
    a, b, c = (t.reshape(x.shape) for t in cur.take("bool", w, x.size))
    e, f = _open(wire, x ^ a, y ^ b, w, xor=True)
    z = c ^ (e & b) ^ (f & a)
    return z ^ (e & f) if party == 0 else z


def p_adder(party: int, wire: Wire, cur: Cursor, u: np.ndarray, v: np.ndarray, w: int) -> np.ndarray:
    """Kogge-Stone adder on XOR shares (protocol.py:113-143)."""
    mk = wmask(w)
    p0 = u ^ v
    wire.tag = "Other"
    g = p_and(party, wire, cur, u, v, w)
    p = p0
    wire.tag = "Circuit"
    for lvl in range(levels_for(w)):
        sh = U64(1 << lvl)
        low = U64((1 << (1 << lvl)) - 1) & mk
        g_up = (g << sh) & mk
        p_up = (p << sh) & mk
        if party == 0:
            p_up = p_up ^ low
        res = p_and(party, wire, cur, np.stack([p, p]), np.stack([g_up, p_up]), w)
        g = g ^ res[0]
        p = res[1]
    wire.tag = "Other"
    return p0 ^ ((g << U64(1)) & mk)


def p_a2b(party: int, wire: Wire, cur: Cursor, s: np.ndarray, w: int) -> np.ndarray:
    """A2B: own share as one XOR operand, zeros as the other (protocol.py:146-157)."""
    z = np.zeros_like(s)
    return p_adder(party, wire, cur, s if party == 0 else z, z if party == 0 else s, w)


def p_b2a(party: int, wire: Wire, cur: Cursor, bit: np.ndarray, n_bits: int) -> np.ndarray:
    """Lift an XOR-shared bit to Z/2^N: u + v - 2uv (protocol.py:160-176)."""
    if np.any(bit > 1):
        raise ValueError("b2a expects 0/1 words")
    z = np.zeros_like(bit)
    u, v = (bit, z) if party == 0 else (z, bit)
    wire.tag = "B2A"
    t = p_mul(party, wire, cur, u, v, n_bits)
    wire.tag = "Other"
    return ring_sub(ring_add(u, v, n_bits), ring_add(t, t, n_bits), n_bits)


def p_drelu(party: int, wire: Wire, cur: Cursor, x: np.ndarray, ring_bits: int, k: int, m: int) -> np.ndarray:
    """Windowed DReLU (protocol.py:179-192)."""
    check_window(k, m, ring_bits)
    w = k - m
    bits = p_a2b(party, wire, cur, window_slice(x, k, m), w)
    lifted = p_b2a(party, wire, cur, top_bit(bits, w), ring_bits)
    d = ring_neg(lifted, ring_bits)
    return ring_add(d, U64(1), ring_bits) if party == 0 else d


def p_relu(party: int, wire: Wire, cur: Cursor, x: np.ndarray, ring_bits: int, k: int, m: int) -> np.ndarray:
    """x * DReLU(x[k:m]) with the multiply metered as Mult (protocol.py:195-199)."""
    d = p_drelu(party, wire, cur, x, ring_bits, k, m)
    wire.tag = "Mult"
    y = p_mul(party, wire, cur, x, d, ring_bits)
    wire.tag = "Other"
    return y


# ------------------------------------------------------------------ pair drivers
def relu_pair(x0, x1, ring_bits, k, m, cursors, keep_payloads=False, op="relu"):
    """Run both parties of one windowed (D)ReLU; returns (y0, y1, wire0, wire1)."""
    fn = p_relu if op == "relu" else p_drelu
    w0, w1 = wire_pair(keep_payloads)
    y0, y1 = run_two(lambda: fn(0, w0, cursors[0], x0, ring_bits, k, m),
                     lambda: fn(1, w1, cursors[1], x1, ring_bits, k, m), (w0, w1))
    return y0, y1, w0, w1


def stocked_cursors(count: int, w: int, ring_bits: int, seed: int = 0):
    """Cursors holding exactly one ReLU's triples with the reference test seeds
    (bool seed 2*seed+1, arith seed 2*seed+2; reference tests/conftest.py:26-61)."""
    need = triple_need(count, w, ring_bits)
    curs = (Cursor(0), Cursor(1))
    bt = deal("bool", need[("bool", w)], w, 2 * seed + 1)
    at = deal("arith", need[("arith", ring_bits)], ring_bits, 2 * seed + 2)
    for p in (0, 1):
        curs[p].stock("bool", w, bt[p])
        curs[p].stock("arith", ring_bits, at[p])
    return curs


def drelu_from_shares(s0, s1, ring_bits, k, m) -> np.ndarray:
    """Plaintext windowed sign decision from an explicit split (simulator.py:33-44)."""
    check_window(k, m, ring_bits)
    t = ring_add(window_slice(s0, k, m), window_slice(s1, k, m), k - m)
    return U64(1) - top_bit(t, k - m)


def analytic_trace(count: int, w: int, ring_bits: int) -> list[tuple[str, int]]:
    """Per-round (tag, bytes) of one ReLU (protocol.py:8-13 cost model)."""
    return ([("Other", stream_nbytes(2 * count, w))]
            + [("Circuit", stream_nbytes(4 * count, w))] * levels_for(w)
            + [("B2A", stream_nbytes(2 * count, ring_bits)), ("Mult", stream_nbytes(2 * count, ring_bits))])


def digest(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<u8").tobytes()).hexdigest()
