// hb_common.cuh -- bit-level building blocks for the reduced-ring ReLU kernels (sm_100a).
//
// Layout vocabulary used by every kernel in this library:
//
//   element   one share of one activation (uint64 residue on Z/2^N), or one
//             w-bit word of a boolean share.
//   stream    the reference wire / triple layout: the low w bits of each
//             element, LSB-first, concatenated into 64-bit little-endian words
//             (ringmpc transport.py:33-49).  Element e sits at bits [e*w, e*w+w).
//   group     GS consecutive elements handled by one thread.  GS is chosen so
//             that GS*w is a multiple of 8: a group's packed bits are whole
//             bytes, so threads write disjoint bytes of a stream (no atomics)
//             whenever the stream segment starts on a group boundary.
//   container SWAR register form of a group: element j occupies a C-bit lane
//             (C = next power of two >= w, >= 8) of NW uint64 words.  XOR/AND
//             act on all lanes at once; the Kogge-Stone shift is one shift plus
//             one lane mask per word (bits that cross a lane are exactly the
//             bits the reference drops with `& mask`, protocol.py:132-133).
//
// For w in {8,16,32,64} the container form is bit-identical to the stream, so
// packing is free; other widths convert with compile-time unrolled shifts.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define HB_DEV __device__ __forceinline__

namespace hb {

typedef uint64_t u64;

HB_DEV void atom_or(u64* p, u64 v) {
  atomicOr(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
}

// Lane bits and elements per group as functions of the width, shared by the
// kernels (Geo<W>) and the host-side launch / workspace arithmetic.
//   lane bits C: next power of two >= w, at least 8.
//   group size : the fewest elements whose packed bits are whole bytes, raised so
//                a group spans at least 32 packed bits for narrow lanes.  Small
//                groups keep every load of a tile in registers at once (more bytes
//                in flight per SM).
__host__ __device__ constexpr int lane_bits_for(int w) { return w <= 8 ? 8 : w <= 16 ? 16 : w <= 32 ? 32 : 64; }
__host__ __device__ constexpr int group_size_for(int w) {
  const int by = w % 8 == 0 ? 1 : (w % 4 == 0 ? 2 : (w % 2 == 0 ? 4 : 8));
  const int c = lane_bits_for(w);
  return c == 64 ? by : (c == 32 ? (by < 2 ? 2 : by) : (by < 4 ? 4 : by));
}
__host__ __device__ constexpr int group_words_for(int w) {
  return (group_size_for(w) + (64 / lane_bits_for(w)) - 1) / (64 / lane_bits_for(w));
}

template <int W>
struct Geo {
  static_assert(W >= 1 && W <= 64, "width must be in 1..64");
  static constexpr int C = lane_bits_for(W);
  static constexpr int GS = group_size_for(W);
  static constexpr int PER = 64 / C;                    // lanes per word
  static constexpr int NW = (GS + PER - 1) / PER;       // container words per group
  static constexpr int PB = GS * W;                     // packed bits per group (multiple of 8)
  static constexpr int PW = (PB + 63) / 64;             // words holding the packed bits
  static constexpr u64 FM = W == 64 ? ~0ull : ((1ull << W) - 1);
  static_assert(PB % 8 == 0, "group must pack to whole bytes");

  // Replicate a C-bit lane pattern across a 64-bit word.
  HB_DEV static constexpr u64 rep(u64 f) {
    u64 r = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) r |= (C == 64 ? f : (f & ((1ull << C) - 1))) << (i * C);
    return r;
  }
};

template <int W>
struct Cg {  // container group
  u64 v[Geo<W>::NW];
};

template <int W>
struct Pk {  // packed group (stream bits of GS elements)
  u64 v[Geo<W>::PW];
};

template <int W>
HB_DEV Cg<W> cg_zero() {
  Cg<W> r;
#pragma unroll
  for (int k = 0; k < Geo<W>::NW; ++k) r.v[k] = 0;
  return r;
}

template <int W>
HB_DEV Cg<W> operator^(const Cg<W>& a, const Cg<W>& b) {
  Cg<W> r;
#pragma unroll
  for (int k = 0; k < Geo<W>::NW; ++k) r.v[k] = a.v[k] ^ b.v[k];
  return r;
}

template <int W>
HB_DEV Cg<W> operator&(const Cg<W>& a, const Cg<W>& b) {
  Cg<W> r;
#pragma unroll
  for (int k = 0; k < Geo<W>::NW; ++k) r.v[k] = a.v[k] & b.v[k];
  return r;
}

// XOR a replicated public word (only ever applied by party 0).
template <int W>
HB_DEV Cg<W> xor_rep(const Cg<W>& a, u64 repword) {
  Cg<W> r;
#pragma unroll
  for (int k = 0; k < Geo<W>::NW; ++k) r.v[k] = a.v[k] ^ repword;
  return r;
}

// (lane << sh) & keep, for every lane; keep = rep(FM & ~((1<<sh)-1)).
template <int W>
HB_DEV Cg<W> shl_keep(const Cg<W>& a, int sh, u64 keep) {
  Cg<W> r;
#pragma unroll
  for (int k = 0; k < Geo<W>::NW; ++k) r.v[k] = (a.v[k] << sh) & keep;
  return r;
}

template <int W>
HB_DEV u64 lane_get(const Cg<W>& a, int j) {  // j must be a compile-time constant after unrolling
  using G = Geo<W>;
  if constexpr (G::C == 64) return a.v[j];
  else return (a.v[j / G::PER] >> ((j % G::PER) * G::C)) & ((1ull << G::C) - 1);
}

template <int W>
HB_DEV void lane_or(Cg<W>& a, int j, u64 val) {  // val < 2^C
  using G = Geo<W>;
  if constexpr (G::C == 64) a.v[j] |= val;
  else a.v[j / G::PER] |= val << ((j % G::PER) * G::C);
}

// ---------------------------------------------------------------- container <-> packed
template <int W>
HB_DEV Pk<W> to_packed(const Cg<W>& c) {
  using G = Geo<W>;
  Pk<W> p;
  if constexpr (W == G::C) {
    static_assert(G::PW == G::NW, "identity layout");
#pragma unroll
    for (int k = 0; k < G::PW; ++k) p.v[k] = c.v[k];
  } else {
#pragma unroll
    for (int k = 0; k < G::PW; ++k) p.v[k] = 0;
#pragma unroll
    for (int j = 0; j < G::GS; ++j) {
      const u64 f = lane_get<W>(c, j) & G::FM;
      const int pos = j * W, k = pos >> 6, o = pos & 63;
      p.v[k] |= f << o;
      if (o + W > 64) p.v[k + 1] |= f >> (64 - o);
    }
  }
  return p;
}

template <int W>
HB_DEV Cg<W> from_packed(const Pk<W>& p) {
  using G = Geo<W>;
  Cg<W> c;
  if constexpr (W == G::C) {
#pragma unroll
    for (int k = 0; k < G::NW; ++k) c.v[k] = p.v[k];
  } else {
    c = cg_zero<W>();
#pragma unroll
    for (int j = 0; j < G::GS; ++j) {
      const int pos = j * W, k = pos >> 6, o = pos & 63;
      u64 f = p.v[k] >> o;
      if (o + W > 64) f |= p.v[k + 1] << (64 - o);
      lane_or<W>(c, j, f & G::FM);
    }
  }
  return c;
}

// ---------------------------------------------------------------- global stream access
HB_DEV u64 ldg64(const u64* p) { return (u64)__ldg(reinterpret_cast<const unsigned long long*>(p)); }

// Read the packed bits of the group whose first element is stream element `e`
// (any bit alignment).  Words at or beyond `nwords` read as zero.
HB_DEV uint32_t ldg32(const uint32_t* p) { return __ldg(p); }

// Read the packed bits of the group whose first element is stream element `e`
// (any bit alignment).  Words at or beyond `nwords` read as zero.  Groups of at
// most 32 bits use 32-bit loads (one load when the group does not straddle).
template <int W>
HB_DEV Pk<W> load_pk(const u64* __restrict__ s, u64 e, u64 nwords) {
  using G = Geo<W>;
  const u64 B = e * (u64)W;
  Pk<W> p;
  if constexpr (G::PB <= 32) {
    const uint32_t* s32 = reinterpret_cast<const uint32_t*>(s);
    const u64 n32 = 2 * nwords, w0 = B >> 5;
    const int sh = (int)(B & 31);
    u64 v = (w0 < n32) ? (u64)ldg32(s32 + w0) : 0ull;
    if (sh + G::PB > 32 && w0 + 1 < n32) v |= (u64)ldg32(s32 + w0 + 1) << 32;
    p.v[0] = (v >> sh) & ((1ull << G::PB) - 1);
    return p;
  } else {
    const u64 w0 = B >> 6;
    const int sh = (int)(B & 63);
    if (sh == 0) {
#pragma unroll
      for (int k = 0; k < G::PW; ++k) p.v[k] = (w0 + k < nwords) ? ldg64(s + w0 + k) : 0ull;
    } else {
      u64 prev = (w0 < nwords) ? ldg64(s + w0) : 0ull;
#pragma unroll
      for (int k = 0; k < G::PW; ++k) {
        const bool need = (sh + G::PB - 64 * k) > 64;  // bits continue into the next word
        const u64 nxt = (need && w0 + k + 1 < nwords) ? ldg64(s + w0 + k + 1) : 0ull;
        p.v[k] = (prev >> sh) | (nxt << (64 - sh));
        prev = nxt;
      }
    }
    if constexpr (G::PB % 64 != 0) p.v[G::PW - 1] &= (1ull << (G::PB % 64)) - 1;
    return p;
  }
}

// GS consecutive uint64 elements starting at p (128-bit loads when aligned).
template <int GS>
HB_DEV void load_u64s(const u64* __restrict__ p, int valid, u64 (&out)[GS]) {
  if (valid == GS && GS % 2 == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
    for (int j = 0; j < GS; j += 2) {
      const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p + j));
      out[j] = v.x;
      out[j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < GS; ++j) out[j] = (j < valid) ? ldg64(p + j) : 0ull;
  }
}

template <int GS>
HB_DEV void store_u64s(u64* __restrict__ p, int valid, const u64 (&v)[GS]) {
  if (valid == GS && GS % 2 == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
    for (int j = 0; j < GS; j += 2) *reinterpret_cast<ulonglong2*>(p + j) = make_ulonglong2(v[j], v[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < GS; ++j)
      if (j < valid) p[j] = v[j];
  }
}

template <int W>
HB_DEV Cg<W> load_cg(const u64* __restrict__ s, u64 e, u64 nwords) {
  return from_packed<W>(load_pk<W>(s, e, nwords));
}

// Keep only the first `valid` elements' bits of a packed group.
template <int W>
HB_DEV void pk_trim(Pk<W>& p, int valid) {
  using G = Geo<W>;
  const int nb = valid * W;
#pragma unroll
  for (int k = 0; k < G::PW; ++k) {
    const int lo = 64 * k;
    if (nb <= lo) p.v[k] = 0;
    else if (nb < lo + 64) p.v[k] &= (1ull << (nb - lo)) - 1;
  }
}

// Write the packed bits of a group whose first element is stream element `e`.
// exclusive=true: the caller guarantees the group starts on a byte boundary
// and no other thread touches these bytes (plain stores).  Otherwise the bits
// are OR-ed into a zero-initialised stream with 64-bit atomics.
template <int W>
HB_DEV void store_pk(u64* __restrict__ s, u64 e, Pk<W> p, int valid, bool exclusive) {
  using G = Geo<W>;
  const u64 B = e * (u64)W;
  if (exclusive && valid == G::GS) {
    if ((B & 63) == 0 && G::PB % 64 == 0) {
#pragma unroll
      for (int k = 0; k < G::PW; ++k) s[(B >> 6) + k] = p.v[k];
      return;
    }
    unsigned char* d = reinterpret_cast<unsigned char*>(s) + (B >> 3);
    constexpr int NB = G::PB / 8;
    const uintptr_t a = reinterpret_cast<uintptr_t>(d);
    if (NB % 4 == 0 && (a & 3) == 0) {
#pragma unroll
      for (int i = 0; i < NB / 4; ++i)
        reinterpret_cast<uint32_t*>(d)[i] = (uint32_t)(p.v[(4 * i) / 8] >> (8 * ((4 * i) % 8)));
    } else if (NB % 2 == 0 && (a & 1) == 0) {
#pragma unroll
      for (int i = 0; i < NB / 2; ++i)
        reinterpret_cast<uint16_t*>(d)[i] = (uint16_t)(p.v[(2 * i) / 8] >> (8 * ((2 * i) % 8)));
    } else {
#pragma unroll
      for (int i = 0; i < NB; ++i) d[i] = (unsigned char)(p.v[i / 8] >> (8 * (i % 8)));
    }
    return;
  }
  pk_trim<W>(p, valid);
  const u64 w0 = B >> 6;
  const int sh = (int)(B & 63);
#pragma unroll
  for (int k = 0; k < G::PW; ++k) {
    if (p.v[k] == 0) continue;
    atom_or(s + w0 + k, p.v[k] << sh);
    if (sh) {
      const u64 hi = p.v[k] >> (64 - sh);
      if (hi) atom_or(s + w0 + k + 1, hi);
    }
  }
}

// ---------------------------------------------------------------- misc
HB_DEV u64 nmask(int nbits) { return nbits >= 64 ? ~0ull : ((1ull << nbits) - 1); }

HB_DEV int prefix_levels_dev(int w) {  // max(1, ceil(log2 w)), protocol.py:108-110
  int l = 0;
  while ((1 << l) < w) ++l;
  return l < 1 ? 1 : l;
}

}  // namespace hb
