// hb_relu_impl.cuh -- the windowed secure ReLU, one template per window width W = k - m.
//
// Reference control flow (ringmpc protocol.py:113-199), per party p:
//
//   s = (x >> m) & (2^W - 1)                         slice          ring.py:69-72
//   round 0 "Other":   G = AND(u, v),  u/v = s or 0  generate bits  protocol.py:123-125
//   round 1+l "Circuit" (l < L): [X;Y] = AND([P;P], [G<<2^l ; P<<2^l ^ ones])
//                      G ^= X, P = Y                 Kogge-Stone    protocol.py:128-141
//   sign = msb(s ^ (G << 1))                                        protocol.py:142,190
//   round L+1 "B2A":   t = MUL(u, v) on Z/2^N, d = [p0] - (u + v - 2t)  protocol.py:160-176,192
//   round L+2 "Mult":  y = MUL(x, d)                                 protocol.py:195-199
//
// Every AND/MUL is a Beaver opening: mask with the triple (a, b), swap the
// masked pair with the peer (one round), then z = c ^ (E&b) ^ (F&a) ^ [p0](E&F)
// (or the ring analogue).  Triples are consumed in the reference cursor order:
// bool stream [Other n][level0: g n, p n][level1 ...], arith stream [B2A n][Mult n]
// (protocol.py:97,137-139,173,199; dealer.py:152-163).
//
// Two drivers share the per-group round math below:
//
//   k_relu_pair   -- 1-GPU time-sliced party pair.  A CTA holds both parties:
//                    threads [0,TP) are party 0 and [TP,2TP) party 1, each thread
//                    one group of the same elements.  A party thread only ever
//                    touches its own share, its own triples and the peer's packed
//                    opening, which it reads from the shared-memory wire after a
//                    barrier (the "exchange").  Nothing but x, the triples and y
//                    touches HBM.
//
//   k_stage_*     -- one party, one round per launch.  State (S, G, P, sign, d)
//                    lives in a workspace between launches and the openings go
//                    through global wire buffers in the exact reference layout,
//                    so the host can move them with NCCL / TCP / a local swap.
#pragma once
#include "hb_common.cuh"

namespace hb {

// ------------------------------------------------------------------ argument blocks
struct PartyIO {
  const u64* x;   // n input shares
  u64* y;         // n output shares (relu) or DReLU shares (drelu_only)
  const u64 *ba, *bb, *bc;  // bool triple streams (packed, width W)
  u64 bcur, bnw;            // cursor (elements), stream length (words)
  const u64 *aa, *ab, *ac;  // arith triple arrays (uint64 per element)
  u64 acur;                 // cursor (elements)
};

struct PairArgs {
  PartyIO io[2];
  u64 n;      // layer size: stride between the triple segments
  u64 first;  // this launch covers elements [first, first + count)
  u64 count;
  int N;      // ring bits
  int m;      // window low bit
  int drelu_only;
};

constexpr int constexpr_levels(int w) {
  int l = 0;
  while ((1 << l) < w) ++l;
  return l < 1 ? 1 : l;
}

template <int W>
struct Kit {
  using G = Geo<W>;
  static constexpr int GS = G::GS;
  static constexpr int L = constexpr_levels(W);

  static HB_DEV Cg<W> slice(const u64 (&x)[GS], int m) {
    Cg<W> s = cg_zero<W>();
#pragma unroll
    for (int j = 0; j < GS; ++j) lane_or<W>(s, j, (x[j] >> m) & G::FM);
    return s;
  }

  // Beaver AND result from the opened masks (protocol.py:102-104).
  static HB_DEV Cg<W> and_z(bool p0, const Cg<W>& E, const Cg<W>& F, const Cg<W>& a, const Cg<W>& b,
                            const Cg<W>& c) {
    Cg<W> z = c ^ (E & b) ^ (F & a);
    if (p0) z = z ^ (E & F);
    return z;
  }

  static HB_DEV u64 keep_mask(int sh) { return G::rep(G::FM & ~((1ull << sh) - 1)); }
  static HB_DEV u64 low_mask(int sh) { return G::rep(((1ull << sh) - 1) & G::FM); }

  // Level-l masked openings [P^ag, P^ap, gS^bg, pS^bp] (protocol.py:130-139, 101).
  static HB_DEV void level_open(bool p0, int l, const Cg<W>& Gc, const Cg<W>& P, const Cg<W>& ag,
                                const Cg<W>& bg, const Cg<W>& ap, const Cg<W>& bp, Cg<W> (&o)[4]) {
    const int sh = 1 << l;
    const u64 keep = keep_mask(sh);
    const Cg<W> gS = shl_keep<W>(Gc, sh, keep);
    Cg<W> pS = shl_keep<W>(P, sh, keep);
    if (p0) pS = xor_rep<W>(pS, low_mask(sh));
    o[0] = P ^ ag;
    o[1] = P ^ ap;
    o[2] = gS ^ bg;
    o[3] = pS ^ bp;
  }

  // Sign bits of s + carries: msb(s ^ ((G << 1) & mask)) (protocol.py:142-143,190).
  static HB_DEV unsigned sign_bits(const Cg<W>& S, const Cg<W>& Gc) {
    const Cg<W> bits = S ^ shl_keep<W>(Gc, 1, keep_mask(1));
    unsigned sg = 0;
#pragma unroll
    for (int j = 0; j < GS; ++j) sg |= (unsigned)((lane_get<W>(bits, j) >> (W - 1)) & 1ull) << j;
    return sg;
  }
};

// Beaver multiply result on Z/2^N (protocol.py:86-88).
HB_DEV u64 mul_z(bool p0, u64 E, u64 F, u64 a, u64 b, u64 c, u64 MN) {
  u64 z = c + E * b + F * a;
  if (p0) z += E * F;
  return z & MN;
}

// ------------------------------------------------------------------ fused pair kernel
template <int W>
struct PairGeo {
  static constexpr int GS = Geo<W>::GS, PW = Geo<W>::PW;
  static constexpr int SEGW = (4 * PW > 2 * GS) ? 4 * PW : 2 * GS;  // words per thread per wire buffer
};

// Resident CTAs per SM the pair kernel's register budget is set for (__launch_bounds__ min blocks).
// The kernel issues every load of a group up front, so more resident warps = more bytes in flight:
// widths 2/4/6/8 compile to 96-112 registers unconstrained (8 CTAs of 64 threads per SM) and fit 96
// without spills -> 10 CTAs per SM: w = 8 at 2^24 3.59e10 -> 4.03e10 elements/s (same-box A/B,
// tools/gpu_ab_lib.sh); forcing 12 (80 registers) spills and is slower (3.39e10).  Odd and wider
// widths need more registers and keep the compiler's choice.  HB_PAIR_MINB overrides (experiments).
template <int W>
constexpr int pair_minb() {
#ifdef HB_PAIR_MINB
  return HB_PAIR_MINB;
#else
  return (W <= 8 && W % 2 == 0) ? 10 : 1;
#endif
}
// One group of both parties' elements through every round: thread t of party `party` owns the GS
// elements starting at layer element e0 (`valid` of them in the layer); the peer thread (t of the
// other half of the CTA) owns the same elements.  Returns the output share (or the DReLU share when
// drelu_only) in `out`; every thread of the CTA must call it (it holds the exchange barriers).
template <int W, int TP, bool RING64>
HB_DEV void pair_group(const PairArgs& A, const int party, const int t, const u64 e0, const int valid,
                       u64* __restrict__ wire, u64 (&out)[Geo<W>::GS]) {
  using G = Geo<W>;
  using K = Kit<W>;
  constexpr int GS = G::GS, PW = G::PW, SEGW = PairGeo<W>::SEGW, L = K::L, NSEG = 1 + 2 * L;
  const bool p0 = party == 0;
  const u64 n = A.n;
  const PartyIO& io = A.io[party];
  const u64 MN = RING64 ? ~0ull : nmask(A.N);  // Z/2^64: masks fold away at compile time
  const bool mult = !A.drelu_only;

  auto slot = [&](int buf, int who, int k) -> u64& { return wire[((buf * 2 + who) * SEGW + k) * TP + t]; };
  auto put_pk = [&](int buf, int k0, const Cg<W>& v) {
    const Pk<W> p = to_packed<W>(v);
#pragma unroll
    for (int q = 0; q < PW; ++q) slot(buf, party, k0 + q) = p.v[q];
  };
  auto get_pk = [&](int buf, int k0) -> Cg<W> {
    Pk<W> p;
#pragma unroll
    for (int q = 0; q < PW; ++q) p.v[q] = slot(buf, party ^ 1, k0 + q);
    return from_packed<W>(p);
  };

  // ---- every load of this tile is issued up front (memory-level parallelism):
  //      the share, all 1+2L bool triple segments, both arith triple segments.
  //      Bool segment s: 0 = Other, 1+2l = level l g-part, 2+2l = level l p-part.
  u64 x[GS];
  load_u64s<GS>(io.x + e0, valid, x);
  Cg<W> ta[NSEG], tbv[NSEG], tc[NSEG];
#pragma unroll
  for (int sgi = 0; sgi < NSEG; ++sgi) {
    const u64 e = io.bcur + (u64)sgi * n + e0;
    ta[sgi] = load_cg<W>(io.ba, e, io.bnw);
    tbv[sgi] = load_cg<W>(io.bb, e, io.bnw);
    tc[sgi] = load_cg<W>(io.bc, e, io.bnw);
  }
  u64 a1[GS], b1[GS], c1[GS], a2[GS], b2[GS], c2[GS];
  const u64 ta0 = io.acur + e0;
  load_u64s<GS>(io.aa + ta0, valid, a1);
  load_u64s<GS>(io.ab + ta0, valid, b1);
  load_u64s<GS>(io.ac + ta0, valid, c1);
  if (mult) {
    load_u64s<GS>(io.aa + ta0 + n, valid, a2);
    load_u64s<GS>(io.ab + ta0 + n, valid, b2);
    load_u64s<GS>(io.ac + ta0 + n, valid, c2);
  }

  // ---- slice (local)
  const Cg<W> S = K::slice(x, A.m);

  // ---- round 0: generate bits G = AND(u, v)
  Cg<W> Gc, P = S;
  {
    const Cg<W> z0 = cg_zero<W>();
    const Cg<W> e = (p0 ? S : z0) ^ ta[0];
    const Cg<W> f = (p0 ? z0 : S) ^ tbv[0];
    put_pk(0, 0, e);
    put_pk(0, PW, f);
    __syncthreads();
    Gc = K::and_z(p0, e ^ get_pk(0, 0), f ^ get_pk(0, PW), ta[0], tbv[0], tc[0]);
  }

  // ---- rounds 1..L: Kogge-Stone levels
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const int buf = (l + 1) & 1, sg = 1 + 2 * l, sp = 2 + 2 * l;
    Cg<W> o[4];
    K::level_open(p0, l, Gc, P, ta[sg], tbv[sg], ta[sp], tbv[sp], o);
#pragma unroll
    for (int q = 0; q < 4; ++q) put_pk(buf, q * PW, o[q]);
    __syncthreads();
    const Cg<W> zg = K::and_z(p0, o[0] ^ get_pk(buf, 0), o[2] ^ get_pk(buf, 2 * PW), ta[sg], tbv[sg], tc[sg]);
    const Cg<W> zp = K::and_z(p0, o[1] ^ get_pk(buf, PW), o[3] ^ get_pk(buf, 3 * PW), ta[sp], tbv[sp], tc[sp]);
    Gc = Gc ^ zg;
    P = zp;
  }

  // ---- round L+1: B2A of the sign bit on Z/2^N
  const unsigned sgn = K::sign_bits(S, Gc);
  u64 d[GS];
  {
    const int buf = (L + 1) & 1;
    u64 e1[GS], f1[GS];
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const u64 bit = (sgn >> j) & 1u;
      e1[j] = ((p0 ? bit : 0ull) - a1[j]) & MN;
      f1[j] = ((p0 ? 0ull : bit) - b1[j]) & MN;
      slot(buf, party, j) = e1[j];
      slot(buf, party, GS + j) = f1[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const u64 E = (e1[j] + slot(buf, party ^ 1, j)) & MN;
      const u64 F = (f1[j] + slot(buf, party ^ 1, GS + j)) & MN;
      const u64 tt = mul_z(p0, E, F, a1[j], b1[j], c1[j], MN);
      const u64 bit = (sgn >> j) & 1u;
      d[j] = ((p0 ? 1ull : 0ull) - ((bit - 2 * tt) & MN)) & MN;  // u + v = bit on one party
    }
  }
  if (!mult) {
#pragma unroll
    for (int j = 0; j < GS; ++j) out[j] = d[j];
    return;
  }

  // ---- round L+2: y = MUL(x, d)
  {
    const int buf = L & 1;
    u64 e2[GS], f2[GS];
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      e2[j] = (x[j] - a2[j]) & MN;
      f2[j] = (d[j] - b2[j]) & MN;
      slot(buf, party, j) = e2[j];
      slot(buf, party, GS + j) = f2[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const u64 E = (e2[j] + slot(buf, party ^ 1, j)) & MN;
      const u64 F = (f2[j] + slot(buf, party ^ 1, GS + j)) & MN;
      out[j] = mul_z(p0, E, F, a2[j], b2[j], c2[j], MN);
    }
  }
}

template <int W, int TP, bool RING64>
__global__ void __launch_bounds__(2 * TP, pair_minb<W>()) k_relu_pair(const PairArgs A) {
  constexpr int GS = Geo<W>::GS;
  extern __shared__ u64 wire[];  // [buf 2][party 2][SEGW][TP]
  const int party = threadIdx.x >= TP ? 1 : 0;
  const int t = threadIdx.x - party * TP;
  const u64 end = A.first + A.count;
  const u64 e0 = A.first + ((u64)blockIdx.x * TP + t) * GS;
  const int valid = e0 >= end ? 0 : (int)min((u64)GS, end - e0);
  u64 yv[GS];
  pair_group<W, TP, RING64>(A, party, t, e0, valid, wire, yv);
  store_u64s<GS>(A.io[party].y + e0, valid, yv);
}

// ------------------------------------------------------------------ staged (one party per launch)
// Workspace (per party, planar so that thread g's words are coalesced):
//   S, Gs, Ps : NW words per group, [NW][ngroups]
//   sign      : one uint32 per group
//   d         : n words
struct StageArgs {
  PartyIO io;
  u64 n, ngroups;
  int N, m, party, round, drelu_only;
  int bool_excl, arith_excl;  // exclusive (plain-store) wire writes allowed
  u64 *S, *Gs, *Ps, *d;
  unsigned* sign;
  const u64* peer;  // peer's payload of the previous round
  u64 peer_nw;      // its length in words
  u64* own;         // this round's payload
};

template <int W>
HB_DEV Cg<W> ws_load(const u64* base, u64 g, u64 ng) {
  Cg<W> r;
#pragma unroll
  for (int k = 0; k < Geo<W>::NW; ++k) r.v[k] = base[k * ng + g];
  return r;
}

template <int W>
HB_DEV void ws_store(u64* base, u64 g, u64 ng, const Cg<W>& v) {
#pragma unroll
  for (int k = 0; k < Geo<W>::NW; ++k) base[k * ng + g] = v.v[k];
}

// Arithmetic openings are N-bit streams; N = 64 is the identity layout (plain
// stores), smaller rings (used by the reference's small-width tests) OR bits
// into a zero-initialised payload.
HB_DEV void put_arith(u64* own, u64 idx, u64 v, int N) {
  if (N == 64) {
    own[idx] = v;
    return;
  }
  const u64 b = idx * (u64)N;
  const int sh = (int)(b & 63);
  if (v == 0) return;
  atom_or(own + (b >> 6), v << sh);
  if (sh + N > 64) atom_or(own + (b >> 6) + 1, v >> (64 - sh));
}

HB_DEV u64 get_arith(const u64* s, u64 idx, int N) {
  if (N == 64) return s[idx];
  const u64 b = idx * (u64)N;
  const int sh = (int)(b & 63);
  u64 v = s[b >> 6] >> sh;
  if (sh + N > 64) v |= s[(b >> 6) + 1] << (64 - sh);
  return v & nmask(N);
}

// A group's two arithmetic openings [e | f] at stream positions e0.. and n+e0..
template <int GS>
HB_DEV void put_arith_group(u64* own, u64 e0, u64 n, int valid, const u64 (&e)[GS], const u64 (&f)[GS], int N) {
  if (N == 64) {
    store_u64s<GS>(own + e0, valid, e);
    store_u64s<GS>(own + n + e0, valid, f);
    return;
  }
#pragma unroll
  for (int j = 0; j < GS; ++j)
    if (j < valid) {
      put_arith(own, e0 + j, e[j], N);
      put_arith(own, n + e0 + j, f[j], N);
    }
}

template <int GS>
HB_DEV void get_arith_group(const u64* peer, u64 e0, u64 n, int valid, u64 (&e)[GS], u64 (&f)[GS], int N) {
  if (N == 64) {
    load_u64s<GS>(peer + e0, valid, e);
    load_u64s<GS>(peer + n + e0, valid, f);
    return;
  }
#pragma unroll
  for (int j = 0; j < GS; ++j) {
    e[j] = (j < valid) ? get_arith(peer, e0 + j, N) : 0ull;
    f[j] = (j < valid) ? get_arith(peer, n + e0 + j, N) : 0ull;
  }
}

// round kinds of the staged driver (round index r):
//   RK_OTHER  r = 0        slice, open the generate-AND masks
//   RK_LEVEL  r = 1..L     combine round r-1, open level r-1
//   RK_B2A    r = L+1      combine level L-1, sign, open the B2A multiply
//   RK_MULT   r = L+2      combine B2A -> d; open x*d (or write d for drelu)
//   RK_FINAL  r = L+3      combine x*d -> y
enum { RK_OTHER = 0, RK_LEVEL = 1, RK_B2A = 2, RK_MULT = 3, RK_FINAL = 4 };

// Combine the bool round r-1 (Other when r == 1, level r-2 otherwise).
template <int W>
HB_DEV void stage_combine_bool(const StageArgs& A, u64 g, u64 e0, bool p0, Cg<W>& Gc, Cg<W>& P) {
  using K = Kit<W>;
  const PartyIO& io = A.io;
  const u64 n = A.n, ng = A.ngroups, tb = io.bcur;
  const int prev = A.round - 1;
  if (prev == 0) {
    const Cg<W> S = ws_load<W>(A.S, g, ng);
    const Cg<W> a = load_cg<W>(io.ba, tb + e0, io.bnw), b = load_cg<W>(io.bb, tb + e0, io.bnw);
    const Cg<W> c = load_cg<W>(io.bc, tb + e0, io.bnw);
    const Cg<W> z0 = cg_zero<W>();
    const Cg<W> e = (p0 ? S : z0) ^ a, f = (p0 ? z0 : S) ^ b;
    Gc = K::and_z(p0, e ^ load_cg<W>(A.peer, e0, A.peer_nw), f ^ load_cg<W>(A.peer, n + e0, A.peer_nw), a, b, c);
    P = S;
    return;
  }
  const int l = prev - 1;
  Gc = ws_load<W>(A.Gs, g, ng);
  P = ws_load<W>(A.Ps, g, ng);
  const u64 base = tb + n + 2 * n * (u64)l + e0;
  const Cg<W> ag = load_cg<W>(io.ba, base, io.bnw), bg = load_cg<W>(io.bb, base, io.bnw);
  const Cg<W> ap = load_cg<W>(io.ba, base + n, io.bnw), bp = load_cg<W>(io.bb, base + n, io.bnw);
  const Cg<W> cg = load_cg<W>(io.bc, base, io.bnw), cp = load_cg<W>(io.bc, base + n, io.bnw);
  Cg<W> o[4];
  K::level_open(p0, l, Gc, P, ag, bg, ap, bp, o);
  const Cg<W> zg =
      K::and_z(p0, o[0] ^ load_cg<W>(A.peer, e0, A.peer_nw), o[2] ^ load_cg<W>(A.peer, 2 * n + e0, A.peer_nw), ag, bg, cg);
  const Cg<W> zp =
      K::and_z(p0, o[1] ^ load_cg<W>(A.peer, n + e0, A.peer_nw), o[3] ^ load_cg<W>(A.peer, 3 * n + e0, A.peer_nw), ap, bp, cp);
  Gc = Gc ^ zg;
  P = zp;
}

template <int W, int KIND>
__global__ void __launch_bounds__(256) k_stage(const StageArgs A) {
  using G = Geo<W>;
  using K = Kit<W>;
  constexpr int GS = G::GS;
  const u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= A.ngroups) return;
  const u64 n = A.n, ng = A.ngroups, e0 = g * GS;
  const int valid = (int)min((u64)GS, n - e0);
  const bool p0 = A.party == 0;
  const PartyIO& io = A.io;
  const u64 tb = io.bcur, ta = io.acur + e0;
  const u64 MN = nmask(A.N);
  const bool bx = A.bool_excl != 0;

  if constexpr (KIND == RK_OTHER) {
    u64 x[GS];
#pragma unroll
    for (int j = 0; j < GS; ++j) x[j] = (j < valid) ? io.x[e0 + j] : 0ull;
    const Cg<W> S = K::slice(x, A.m);
    ws_store<W>(A.S, g, ng, S);
    const Cg<W> a = load_cg<W>(io.ba, tb + e0, io.bnw), b = load_cg<W>(io.bb, tb + e0, io.bnw);
    const Cg<W> z0 = cg_zero<W>();
    store_pk<W>(A.own, e0, to_packed<W>((p0 ? S : z0) ^ a), valid, bx);
    store_pk<W>(A.own, n + e0, to_packed<W>((p0 ? z0 : S) ^ b), valid, bx);
  } else if constexpr (KIND == RK_LEVEL) {
    Cg<W> Gc, P;
    stage_combine_bool<W>(A, g, e0, p0, Gc, P);
    const int l = A.round - 1;
    const u64 base = tb + n + 2 * n * (u64)l + e0;
    const Cg<W> ag = load_cg<W>(io.ba, base, io.bnw), bg = load_cg<W>(io.bb, base, io.bnw);
    const Cg<W> ap = load_cg<W>(io.ba, base + n, io.bnw), bp = load_cg<W>(io.bb, base + n, io.bnw);
    Cg<W> o[4];
    K::level_open(p0, l, Gc, P, ag, bg, ap, bp, o);
#pragma unroll
    for (int s = 0; s < 4; ++s) store_pk<W>(A.own, (u64)s * n + e0, to_packed<W>(o[s]), valid, bx);
    ws_store<W>(A.Gs, g, ng, Gc);
    ws_store<W>(A.Ps, g, ng, P);
  } else if constexpr (KIND == RK_B2A) {
    Cg<W> Gc, P;
    stage_combine_bool<W>(A, g, e0, p0, Gc, P);
    const unsigned sg = K::sign_bits(ws_load<W>(A.S, g, ng), Gc);
    A.sign[g] = sg;
    u64 a[GS], b[GS], e[GS], f[GS];
    load_u64s<GS>(io.aa + ta, valid, a);
    load_u64s<GS>(io.ab + ta, valid, b);
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const u64 bit = (sg >> j) & 1u;
      e[j] = ((p0 ? bit : 0ull) - a[j]) & MN;
      f[j] = ((p0 ? 0ull : bit) - b[j]) & MN;
    }
    put_arith_group<GS>(A.own, e0, n, valid, e, f, A.N);
  } else if constexpr (KIND == RK_MULT) {
    const unsigned sg = A.sign[g];
    u64 a[GS], b[GS], c[GS], pe[GS], pf[GS], d[GS];
    load_u64s<GS>(io.aa + ta, valid, a);
    load_u64s<GS>(io.ab + ta, valid, b);
    load_u64s<GS>(io.ac + ta, valid, c);
    get_arith_group<GS>(A.peer, e0, n, valid, pe, pf, A.N);
    u64 x[GS], a2[GS], b2[GS];
    if (!A.drelu_only) {
      load_u64s<GS>(io.x + e0, valid, x);
      load_u64s<GS>(io.aa + ta + n, valid, a2);
      load_u64s<GS>(io.ab + ta + n, valid, b2);
    }
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const u64 bit = (sg >> j) & 1u;
      const u64 E = (((p0 ? bit : 0ull) - a[j]) + pe[j]) & MN;
      const u64 F = (((p0 ? 0ull : bit) - b[j]) + pf[j]) & MN;
      const u64 tt = mul_z(p0, E, F, a[j], b[j], c[j], MN);
      d[j] = ((p0 ? 1ull : 0ull) - ((bit - 2 * tt) & MN)) & MN;
    }
    if (A.drelu_only) {
      store_u64s<GS>(io.y + e0, valid, d);
    } else {
      store_u64s<GS>(A.d + e0, valid, d);
      u64 e2[GS], f2[GS];
#pragma unroll
      for (int j = 0; j < GS; ++j) {
        e2[j] = (x[j] - a2[j]) & MN;
        f2[j] = (d[j] - b2[j]) & MN;
      }
      put_arith_group<GS>(A.own, e0, n, valid, e2, f2, A.N);
    }
  } else {  // RK_FINAL
    u64 a[GS], b[GS], c[GS], x[GS], d[GS], pe[GS], pf[GS], y[GS];
    load_u64s<GS>(io.aa + ta + n, valid, a);
    load_u64s<GS>(io.ab + ta + n, valid, b);
    load_u64s<GS>(io.ac + ta + n, valid, c);
    load_u64s<GS>(io.x + e0, valid, x);
    load_u64s<GS>(A.d + e0, valid, d);
    get_arith_group<GS>(A.peer, e0, n, valid, pe, pf, A.N);
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const u64 E = ((x[j] - a[j]) + pe[j]) & MN, F = ((d[j] - b[j]) + pf[j]) & MN;
      y[j] = mul_z(p0, E, F, a[j], b[j], c[j], MN);
    }
    store_u64s<GS>(io.y + e0, valid, y);
  }
}

}  // namespace hb
