"""Trusted-dealer triples and the device-resident per-party triple store.

Generation (offline, host): the same PCG64 stream layout as the reference
dealer (dealer.py:50-83) -- a, b, r_a, r_b, r_c drawn as ``rng.bytes`` words
from ``default_rng(SeedSequence(seed))`` -- so a store stocked here holds
bit-identical shares to the reference's for the same seed.  The HBTRIP1 file
format (dealer.py:9-11, 86-119) is read and written unchanged.

Store (online, device): ``TripleStore.add_batch`` uploads one party's shares
to HBM once.  Boolean triples are re-laid as packed w-bit streams (the wire
layout, built by the CUDA packer) so the ReLU kernels read exactly w bits per
triple word; arithmetic triples stay one uint64 per element.  ``draw`` keeps
the reference's forward-only cursor semantics (dealer.py:152-171) and hands
out cursor-addressed views instead of array slices.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _dev, _lib, ring
from .errors import ConfigError, DataFormatError, TripleExhaustedError

MAGIC = b"HBTRIP1"
KIND_ARITH = 0
KIND_BOOL = 1
_HEADER = struct.Struct("<7sBBQQ")

ARITH = "arith"
BOOL = "bool"
_CODES = {ARITH: KIND_ARITH, BOOL: KIND_BOOL}
_NAMES = {v: k for k, v in _CODES.items()}


@dataclass
class TripleBatch:
    """Both parties' shares of `count` triples on one ring (dealer.py:36-47)."""

    kind: str
    width: int
    count: int
    seed: int
    shares: tuple

    def party_arrays(self, party: int):
        return self.shares[party]


def _stream(seed: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(seed))


def gen_arith_triples(count: int, width: int, seed: int) -> TripleBatch:
    """Additive (a, b, ab mod 2^width) triples (dealer.py:54-67)."""
    if count < 0:
        raise ConfigError("count must be >= 0")
    g = _stream(seed)
    a, b = ring.random_residues(g, count, width), ring.random_residues(g, count, width)
    c = ring.mul_mod(a, b, width)
    ra, rb, rc = (ring.random_residues(g, count, width) for _ in range(3))
    p0 = tuple(ring.add_mod(v, r, width) for v, r in ((a, ra), (b, rb), (c, rc)))
    p1 = tuple(ring.neg_mod(r, width) for r in (ra, rb, rc))
    return TripleBatch(ARITH, width, count, seed, (p0, p1))


def gen_bool_triples(count: int, word_width: int, seed: int) -> TripleBatch:
    """XOR-shared (a, b, a & b) word triples (dealer.py:70-83)."""
    if count < 0:
        raise ConfigError("count must be >= 0")
    g = _stream(seed)
    a, b = ring.random_residues(g, count, word_width), ring.random_residues(g, count, word_width)
    ra, rb, rc = (ring.random_residues(g, count, word_width) for _ in range(3))
    return TripleBatch(BOOL, word_width, count, seed, ((a ^ ra, b ^ rb, (a & b) ^ rc), (ra, rb, rc)))


def save_triples(batch: TripleBatch, path) -> None:
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, _CODES[batch.kind], batch.width, batch.count, batch.seed))
        for party in (0, 1):
            for arr in batch.party_arrays(party):
                fh.write(np.asarray(arr, dtype="<u8").tobytes())


def load_triples(path) -> TripleBatch:
    try:
        blob = Path(path).read_bytes()
    except OSError as exc:
        raise DataFormatError(f"{path}: cannot read triple file: {exc}") from exc
    if len(blob) < _HEADER.size:
        raise DataFormatError(f"{path}: too short for a triple file header")
    magic, code, width, count, seed = _HEADER.unpack_from(blob, 0)
    if magic != MAGIC:
        raise DataFormatError(f"{path}: bad magic {magic!r}")
    if code not in _NAMES:
        raise DataFormatError(f"{path}: unknown triple kind {code}")
    if not 1 <= width <= ring.MAX_WIDTH:
        raise DataFormatError(f"{path}: invalid width {width}")
    if len(blob) != _HEADER.size + 48 * count:
        raise DataFormatError(f"{path}: expected {_HEADER.size + 48 * count} bytes, found {len(blob)}")
    arrs = np.frombuffer(blob, dtype="<u8", offset=_HEADER.size, count=6 * count).reshape(6, count).copy()
    return TripleBatch(_NAMES[code], width, count, seed, ((arrs[0], arrs[1], arrs[2]), (arrs[3], arrs[4], arrs[5])))


def deal_on_device(kind: str, width: int, count: int, seed: int, device=None):
    """Dealer for large benchmark stocks: valid Beaver triples generated in HBM.

    Same algebra as gen_*_triples (c = ab mod 2^w or a & b, shares (v + r, -r)
    or (v ^ r, r)) but drawn from torch's CUDA generator instead of the
    reference's PCG64 stream, so it stocks gigabytes in milliseconds.  Returns
    ((a0, b0, c0), (a1, b1, c1)) as CUDA int64 tensors.  Offline phase only."""
    dev = device or _dev.device()
    g = torch.Generator(device=dev)
    g.manual_seed(seed)

    def rnd():
        hi = torch.empty(count, dtype=torch.int64, device=dev).random_(0, 1 << 32, generator=g)
        lo = torch.empty(count, dtype=torch.int64, device=dev).random_(0, 1 << 32, generator=g)
        v = torch.bitwise_or(torch.bitwise_left_shift(hi, 32), lo)
        return v if width == 64 else torch.bitwise_and(v, (1 << width) - 1)

    def fit(v):
        return v if width == 64 else torch.bitwise_and(v, (1 << width) - 1)

    a, b = rnd(), rnd()
    ra, rb, rc = rnd(), rnd(), rnd()
    if kind == ARITH:
        c = fit(a * b)
        return (fit(a + ra), fit(b + rb), fit(c + rc)), (fit(-ra), fit(-rb), fit(-rc))
    c = torch.bitwise_and(a, b)
    return (a ^ ra, b ^ rb, c ^ rc), (ra, rb, rc)


def pcg64_seed_state(seed: int) -> tuple:
    """(state, inc) of default_rng(SeedSequence(seed)) before any draw -- the stream the
    reference dealer reads (dealer.py:50-51)."""
    st = np.random.default_rng(np.random.SeedSequence(seed)).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


def deal_exact_on_device(kind: str, width: int, count: int, seed: int, first: int = 0, n: int | None = None,
                         device=None):
    """Triples [first, first + n) of gen_arith_triples / gen_bool_triples(count, width, seed),
    computed in HBM by hb_deal_triples (PCG64 jump-ahead) -- bit-identical to the host
    generator.  Returns ((a0, b0, c0), (a1, b1, c1)) CUDA int64 tensors."""
    if count < 0:
        raise ConfigError("count must be >= 0")
    n = count - first if n is None else n
    dev = device or _dev.device()
    s, inc = pcg64_seed_state(seed)
    out = [torch.empty(max(n, 1), dtype=torch.int64, device=dev) for _ in range(6)]
    m64 = (1 << 64) - 1
    _lib.call("hb_deal_triples", s & m64, s >> 64, inc & m64, inc >> 64, _CODES[kind], width, count, first, n,
              *(t.data_ptr() for t in out), _dev.stream_handle())
    out = [t[:n] for t in out]
    return (out[0], out[1], out[2]), (out[3], out[4], out[5])


def stock_on_device(stores, parties, kind: str, width: int, count: int, seed: int, chunk: int = 1 << 25,
                    exact: bool = True) -> None:
    """Stock `count` triples of one (kind, width) into each store (store i holds party
    parties[i]'s share), generated chunk by chunk in HBM and packed straight into the final
    stream -- peak scratch is one chunk, not the whole stock.  exact=True deals exactly
    gen_*_triples(count, width, seed) (the reference dealer's stream); exact=False uses
    torch's generator.  Ranks that each hold one party call this with the same seed."""
    dev = _dev.device()
    chunk = max(64, (chunk // 64) * 64)  # whole 64-bit words per chunk for any width
    if kind == BOOL:
        words = (count * width + 63) // 64
        outs = [[torch.zeros(max(words, 1), dtype=torch.int64, device=dev) for _ in range(3)] for _ in stores]
    else:
        outs = [[torch.empty(max(count, 1), dtype=torch.int64, device=dev) for _ in range(3)] for _ in stores]
    for i, lo in enumerate(range(0, count, chunk)):
        c = min(chunk, count - lo)
        shares = (deal_exact_on_device(kind, width, count, seed, lo, c, dev) if exact
                  else deal_on_device(kind, width, c, seed * 100003 + i, dev))
        for out, p in zip(outs, parties):
            for dst, src in zip(out, shares[p]):
                if kind == BOOL:
                    w0 = lo * width // 64
                    nw = (c * width + 63) // 64
                    _lib.call("hb_pack", src.data_ptr(), c, width, dst[w0:w0 + nw].data_ptr(), _dev.stream_handle())
                else:
                    dst[lo:lo + c].copy_(src)
        del shares
    for st, out in zip(stores, outs):
        if (kind, width) in st._streams:
            raise ConfigError("stream already stocked")
        st._streams[(kind, width)] = _DevStream(kind, width, count, *out)


# ------------------------------------------------------------------ device store
@dataclass
class TripleView:
    """Cursor-addressed slice [cursor, cursor+count) of one device stream."""

    kind: str
    width: int
    a: torch.Tensor
    b: torch.Tensor
    c: torch.Tensor
    cursor: int
    count: int
    capacity: int

    def abi(self) -> _lib.Triples:
        return _lib.Triples(self.a.data_ptr(), self.b.data_ptr(), self.c.data_ptr(), self.cursor, self.capacity,
                            self.width)

    def unpacked(self):
        """(a, b, c) as uint64 numpy arrays (test / debug helper)."""
        out = []
        for t in (self.a, self.b, self.c):
            if self.kind == BOOL:
                v = _unpack_dev(t, self.cursor + self.count, self.width)[self.cursor:]
            else:
                v = t[self.cursor:self.cursor + self.count]
            out.append(v.cpu().numpy().view(np.uint64))
        return tuple(out)


@dataclass
class _DevStream:
    kind: str
    width: int
    count: int
    a: torch.Tensor
    b: torch.Tensor
    c: torch.Tensor
    cursor: int = 0


def _upload(arr: np.ndarray) -> torch.Tensor:
    return _dev.to_device(np.ascontiguousarray(arr, dtype=np.uint64))


def _pack_dev(vals: torch.Tensor, count: int, width: int) -> torch.Tensor:
    out = torch.zeros(max((count * width + 63) // 64, 1), dtype=torch.int64, device=vals.device)
    _lib.call("hb_pack", vals.data_ptr(), count, width, out.data_ptr(), _dev.stream_handle())
    return out


def _unpack_dev(packed: torch.Tensor, count: int, width: int) -> torch.Tensor:
    out = torch.empty(max(count, 1), dtype=torch.int64, device=packed.device)
    _lib.call("hb_unpack", packed.data_ptr(), count, width, out.data_ptr(), _dev.stream_handle())
    return out[:count]


@dataclass
class TripleStore:
    """One party's dealt triples in HBM, consumed front to back (dealer.py:130-171)."""

    party: int
    _streams: dict = field(default_factory=dict)

    def add_batch(self, batch: TripleBatch) -> None:
        key = (batch.kind, batch.width)
        arrs = [_upload(a) for a in batch.party_arrays(self.party)]
        if batch.kind == BOOL:
            old = self._streams.get(key)
            if old is not None:
                arrs = [torch.cat([_unpack_dev(o, old.count, batch.width), n])
                        for o, n in zip((old.a, old.b, old.c), arrs)]
            total = (old.count if old else 0) + batch.count
            packed = [_pack_dev(a, total, batch.width) for a in arrs]
            self._streams[key] = _DevStream(BOOL, batch.width, total, *packed, cursor=old.cursor if old else 0)
        else:
            old = self._streams.get(key)
            if old is not None:
                arrs = [torch.cat([o[:old.count], n]) for o, n in zip((old.a, old.b, old.c), arrs)]
            total = (old.count if old else 0) + batch.count
            self._streams[key] = _DevStream(ARITH, batch.width, total, *arrs, cursor=old.cursor if old else 0)

    def add_device(self, kind: str, width: int, arrays) -> None:
        """Install one party's device-resident (a, b, c) (e.g. from deal_on_device)."""
        a, b, c = (t.reshape(-1) for t in arrays)
        count = a.numel()
        if (kind, width) in self._streams:
            raise ConfigError("add_device replaces nothing: stream already stocked")
        if kind == BOOL:
            a, b, c = (_pack_dev(t, count, width) for t in (a, b, c))
        self._streams[(kind, width)] = _DevStream(kind, width, count, a, b, c)

    def rewind(self, kind: str, width: int, cursor: int = 0) -> None:
        """Move a stream's cursor back (benchmarks cycling over stocked sets only)."""
        self._streams[(kind, width)].cursor = cursor

    def _get(self, kind: str, width: int, count: int) -> _DevStream:
        s = self._streams.get((kind, width))
        if s is None or s.cursor + count > s.count:
            have = 0 if s is None else s.count - s.cursor
            raise TripleExhaustedError(f"party {self.party} needs {count} {kind} triples of width {width}, "
                                       f"{have} left")
        return s

    def check(self, needs: dict) -> None:
        """Raise before anything is consumed if any (kind, width) -> count is short."""
        for (kind, width), count in needs.items():
            self._get(kind, width, count)

    def draw(self, kind: str, width: int, count: int) -> TripleView:
        """Next `count` unused triples as a device view; advances the cursor."""
        s = self._get(kind, width, count)
        v = TripleView(kind, width, s.a, s.b, s.c, s.cursor, count, s.count)
        s.cursor += count
        return v

    def consumed(self, kind: str, width: int) -> int:
        s = self._streams.get((kind, width))
        return 0 if s is None else s.cursor

    def remaining(self, kind: str, width: int) -> int:
        s = self._streams.get((kind, width))
        return 0 if s is None else s.count - s.cursor
