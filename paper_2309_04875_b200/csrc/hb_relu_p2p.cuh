// hb_relu_p2p.cuh -- one party's whole windowed ReLU in ONE persistent launch, the openings of every
// round exchanged tile by tile through the peer GPU's memory (NVLink P2P stores + flags).
//
// This is the N > 1 counterpart of k_relu_pair: party p runs on its own GPU, both parties run this
// kernel on the same element tiles in the same order.  For tile t and round r a CTA
//   1. computes its masked openings (same Kit<W> round math as k_relu_pair / k_stage),
//   2. stores them straight into the PEER's receive buffer (remote HBM, over NVLink),
//   3. __syncthreads; one thread releases the peer's flag[t] = seq(r) at system scope,
//   4. polls its own flag[t] (relaxed) until >= seq(r), then one acquire load of it -- the peer's
//      openings of round r are in its local receive buffer -- and combines them with its own.
// The combine of round r and the openings of round r+1 are one pass over the tile's groups, so the
// loads of both (the peer's openings, this round's c segment, the next round's a / b segments) are
// in flight together.  The transfer of tile t overlaps the math of the other resident tiles: no
// per-round launches, no host round trips, no NCCL on the data path.
//
// Wire format = the reference payload, exactly.  A bool round's packet for tile t holds its
// segments ([e | f] for Other, [P^ag | P^ap | gS^bg | pS^bp] for a level -- the order of
// protocol.py:62-72 / 130-139), each segment the LSB-first w-bit stream (transport.py:33-49) of the
// tile's elements: the tile is a whole number of bytes per segment, so the segments of all tiles
// concatenate to the reference stream and the bytes that cross NVLink per round are
// nseg * ceil(n w / 8), i.e. the reference's 8 ceil(nseg n w / 64) less its zero padding of the last
// word.  Groups whose packed bits are whole 32-bit words are stored directly (coalesced); other
// widths (w = 5, 6, 22, ...) and the partial last tile are packed byte-exactly into shared memory
// and copied to the peer in 16-byte units.  The arithmetic rounds (B2A, Mult) send 8 bytes per
// element and segment.  The meter records the reference sizes (relu_trace).
//
// Receive regions: round r of a launch owns region r; a party can be at most one round ahead of its
// peer on a tile, so a region is never rewritten while being read within a launch.  ACROSS launches
// the caller alternates two halves of the receive buffer (transport.PeerLink, by launch parity):
// a peer that finished launch k and started k+1 writes the other half while this party may still be
// reading launch k's last round, and it cannot reach launch k+2 before this party finished k.
//
// Deadlock freedom: the launch is cooperative (all CTAs co-resident or the launch fails), and every
// CTA walks its tiles in increasing order (tile = cta, cta + grid, ...), so the smallest unfinished
// tile always has both parties' CTAs at it -- progress does not depend on the two parties' grids
// being equal (transport.PeerLink still agrees them).  A bounded spin (globaltimer, timeout_ns)
// turns a missing peer into an error word instead of a hang.
#pragma once
#include <cstdio>
#include <cstdlib>

#include "hb_relu_impl.cuh"


namespace hb {


// Memory-model scope of the flag protocol (P2PArgs::sys_scope, a uniform branch in the one thread
// that handles the flags): system scope for parties on different GPUs (the peer is only in system
// scope), gpu scope when both parties run on the same device (the single-device harness; the
// narrowest scope containing both parties -- measured ~0.4 us per release vs ~4 us at system scope).
#ifndef HB_P2P_C
#define HB_P2P_C 4
#endif
constexpr int P2P_C = HB_P2P_C;  // groups per thread per tile
constexpr int P2P_MAXR = 10;     // rounds per ReLU <= L + 3 with L <= 6

struct P2PArgs {
  PartyIO io;
  u64 n, ntiles;
  int N, m, party, drelu_only;
  unsigned grid;                  // this party's CTAs (the tile stride)
  int sys_scope;                  // 1: system-scope flags (peer on another GPU); 0: gpu scope (same device)
  u64 seq0;                       // flag value before this launch's round 0 (rounds of earlier launches)
  uint8_t* recv;                  // this party's receive buffer (written by the peer)
  const unsigned long long* my_flag;  // [ntiles], written by the peer
  uint8_t* peer_recv;             // the peer's receive buffer (mapped)
  unsigned long long* peer_flag;  // the peer's flags (mapped)
  u64 round_off[P2P_MAXR];        // byte offset of each round's region (identical on both sides)
  u64 timeout_ns;
  int* err;                       // set to 1 on a spin timeout
  unsigned long long* wire_bytes; // optional [P2P_MAXR] counters of the bytes stored to the peer
  unsigned long long* stamps;     // optional phase timestamps (tools/micro/p2p_bench), else null
  // Device-resident link state (optional, this party only): [0] flag sequence, [1] launches, [2]
  // CTAs done.  When set, seq0 and the receive region (launch parity x region_bytes past recv /
  // peer_recv) come from the device and the party's last CTA advances them -- the launch arguments
  // are then the same every call, so a sequence of layers can be captured in a CUDA graph.
  unsigned long long* state;
  u64 region_bytes;               // offset of the second receive region (odd launches)
};

template <int W>
struct P2PGeo {
  static constexpr int GS = Geo<W>::GS, PB = Geo<W>::PB, NB = PB / 8;
  static constexpr int L = constexpr_levels(W);
  // threads per CTA (= per tile): one flag release per tile and round, so bigger tiles move more
  // per release -- which pays most at system scope (two GPUs), where a release costs ~4 us.
  // Measured (tools/micro_run8.sh, gpu / system scope, fraction of H): w = 64: 128 threads x 7 CTAs
  // 1.0 / 0.73, 512 x 2: 1.0 / 0.82; w = 32: 0.70 / 0.49 -> 0.73 / 0.63 (512 x 2); w = 16: 0.69 /
  // 0.57 -> 0.68 / 0.63 (256 x 4); w = 6: 0.54 / 0.44 -> 0.54 / 0.49 (256 x 4); w = 8 keeps 128 x 5
  // (0.77 / 0.56; 256 x 3: 0.76 / 0.60).  Bigger tiles only while the byte-exact staging of the
  // resident CTAs fits in shared memory.
#ifdef HB_P2P_TP
  static constexpr int TP = HB_P2P_TP;
#else
  static constexpr int TP = (W >= 32 && 4 * P2P_C * 512 * NB <= 96 * 1024)
                                ? 512
                                : ((W != 8 && 4 * P2P_C * 256 * NB <= 56 * 1024) ? 256 : 128);
#endif
  static constexpr bool DIRECT = NB % 4 == 0;               // a group is whole 32-bit words
  static constexpr u64 TE = (u64)P2P_C * TP * GS;           // elements per tile
  static constexpr u64 SB = (u64)P2P_C * TP * NB;           // bytes of a bool segment per tile
  static constexpr u64 SA = TE * 8;                         // bytes of an arith segment per tile
  static constexpr __host__ __device__ int nseg(int r) { return r == 0 ? 2 : (r <= L ? 4 : 2); }
  static constexpr __host__ __device__ u64 packet(int r) { return nseg(r) * (r <= L ? SB : SA); }
  static_assert(SB % 16 == 0 && SA % 16 == 0, "segments stay 16-byte aligned");
  // resident CTAs per SM the register budget is set for, and whether the exchange warms L2 with
  // the next round's inputs (helps the wide rounds only).  Measured on B200 with tools/micro/p2p_bench
  // (both parties on one GPU, 2^24; tools/micro_run2.sh / run4.sh): the kernel is latency-bound per
  // round, so more resident tiles win until registers spill -- w = 6: 6 CTAs (1.09e10 elem/s), w = 8:
  // 5 (1.44e10; 6-8 are slower), w = 16 / 32: 7 (9.1e9 / 5.2e9, vs 8.5e9 / 4.3e9 at 5 / 4), w = 64: 7 +
  // prefetch (1.0 of H; 4 CTAs: 0.98).  With system-scope flags (two GPUs; tools/micro_run7.sh) more
  // tiles in flight matter more: w = 64 0.52 -> 0.73 of H going from 4 to 7 CTAs.  Loading the next
  // level's inputs into registers before each exchange (instead of after it) was slower at every width.
#ifdef HB_P2P_MINB
  static constexpr int MINB = HB_P2P_MINB;
#else
  static constexpr int MINB = TP == 512 ? 2 : (TP == 256 ? 4 : (W == 8 ? 5 : (W < 8 ? 6 : 7)));
#endif
#ifdef HB_P2P_PF
  static constexpr bool PF = HB_P2P_PF;
#else
  static constexpr bool PF = W > 32;
#endif
};

// Warm L2 with [p, p + bytes) (TMA prefetch, no registers held).
HB_DEV void prefetch_l2(const void* p, u64 bytes) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  while (a < e) {
    const unsigned chunk = (e - a) > (1u << 20) ? (1u << 20) : (unsigned)(e - a);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(chunk) : "memory");
    a += chunk;
  }
}

HB_DEV void flag_release(bool sys, unsigned long long* p, unsigned long long v) {
  if (sys) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
HB_DEV unsigned long long flag_relaxed(bool sys, const unsigned long long* p) {
  unsigned long long v;
  if (sys) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
HB_DEV unsigned long long flag_acquire(bool sys, const unsigned long long* p) {
  unsigned long long v;
  if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

HB_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The packed bits of the group starting at stream element e of a segment the PEER wrote during
// this launch: L2 loads (ld.global.cg), never the non-coherent read-only path.
template <int W>
HB_DEV Pk<W> load_pk_cg(const u64* s, u64 e, u64 nwords) {
  using G = Geo<W>;
  const u64 B = e * (u64)W;
  Pk<W> p;
  if constexpr (G::PB <= 32) {
    const unsigned* s32 = reinterpret_cast<const unsigned*>(s);
    const u64 n32 = 2 * nwords, w0 = B >> 5;
    const int sh = (int)(B & 31);
    u64 v = (w0 < n32) ? (u64)__ldcg(s32 + w0) : 0ull;
    if (sh + G::PB > 32 && w0 + 1 < n32) v |= (u64)__ldcg(s32 + w0 + 1) << 32;
    p.v[0] = (v >> sh) & ((1ull << G::PB) - 1);
  } else {
    const unsigned long long* s64 = reinterpret_cast<const unsigned long long*>(s);
    const u64 w0 = B >> 6;
    const int sh = (int)(B & 63);
    if (sh == 0) {
#pragma unroll
      for (int k = 0; k < G::PW; ++k) p.v[k] = (w0 + k < nwords) ? (u64)__ldcg(s64 + w0 + k) : 0ull;
    } else {
      u64 prev = (w0 < nwords) ? (u64)__ldcg(s64 + w0) : 0ull;
#pragma unroll
      for (int k = 0; k < G::PW; ++k) {
        const bool need = (sh + G::PB - 64 * k) > 64;
        const u64 nxt = (need && w0 + k + 1 < nwords) ? (u64)__ldcg(s64 + w0 + k + 1) : 0ull;
        p.v[k] = (prev >> sh) | (nxt << (64 - sh));
        prev = nxt;
      }
    }
    if constexpr (G::PB % 64 != 0) p.v[G::PW - 1] &= (1ull << (G::PB % 64)) - 1;
  }
  return p;
}

template <int GS>
HB_DEV void load_u64s_cg(const u64* p, int valid, u64 (&out)[GS]) {
  const unsigned long long* q = reinterpret_cast<const unsigned long long*>(p);
  if (valid == GS && GS % 2 == 0) {
#pragma unroll
    for (int j = 0; j < GS; j += 2) {
      const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(q + j));
      out[j] = v.x;
      out[j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < GS; ++j) out[j] = (j < valid) ? (u64)__ldcg(q + j) : 0ull;
  }
}

// NB bytes of a packed group to `d` (global or shared), widest aligned units.
template <int W>
HB_DEV void put_bytes(uint8_t* d, const Pk<W>& p) {
  constexpr int NB = Geo<W>::PB / 8;
  if constexpr (NB % 16 == 0) {
#pragma unroll
    for (int i = 0; i < NB / 16; ++i)
      reinterpret_cast<ulonglong2*>(d)[i] = make_ulonglong2(p.v[2 * i], p.v[2 * i + 1]);
  } else if constexpr (NB % 8 == 0) {
#pragma unroll
    for (int i = 0; i < NB / 8; ++i) reinterpret_cast<u64*>(d)[i] = p.v[i];
  } else if constexpr (NB % 4 == 0) {
#pragma unroll
    for (int i = 0; i < NB / 4; ++i) reinterpret_cast<uint32_t*>(d)[i] = (uint32_t)(p.v[i / 2] >> (32 * (i % 2)));
  } else if constexpr (NB % 2 == 0) {
#pragma unroll
    for (int i = 0; i < NB / 2; ++i) reinterpret_cast<uint16_t*>(d)[i] = (uint16_t)(p.v[i / 4] >> (16 * (i % 4)));
  } else {
#pragma unroll
    for (int i = 0; i < NB; ++i) d[i] = (uint8_t)(p.v[i / 8] >> (8 * (i % 8)));
  }
}

// Stores into the PEER's receive buffer: plain C++ stores, so the compiler keeps hoisting the
// (read-only, ld.global.nc) triple loads of later groups above them; the exchange's barrier +
// release store orders them for the peer.
template <int W>
HB_DEV void put_peer(uint8_t* d, const Pk<W>& p) {
  put_bytes<W>(d, p);
}


// GS consecutive u64 of a group: FAST = the whole group is valid and 16-byte aligned (no runtime
// checks, so the compiler schedules these loads freely), else the checked load / store.
template <int GS, bool FAST>
HB_DEV void ld_grp(const u64* p, int valid, u64 (&o)[GS]) {
  if constexpr (FAST && GS % 2 == 0) {
#pragma unroll
    for (int j = 0; j < GS; j += 2) {
      const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p + j));
      o[j] = v.x;
      o[j + 1] = v.y;
    }
  } else if constexpr (FAST) {
#pragma unroll
    for (int j = 0; j < GS; ++j) o[j] = ldg64(p + j);
  } else {
    load_u64s<GS>(p, valid, o);
  }
}
template <int GS, bool FAST>
HB_DEV void ld_grp_cg(const u64* p, int valid, u64 (&o)[GS]) {
  const unsigned long long* q = reinterpret_cast<const unsigned long long*>(p);
  if constexpr (FAST && GS % 2 == 0) {
#pragma unroll
    for (int j = 0; j < GS; j += 2) {
      const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(q + j));
      o[j] = v.x;
      o[j + 1] = v.y;
    }
  } else if constexpr (FAST) {
#pragma unroll
    for (int j = 0; j < GS; ++j) o[j] = (u64)__ldcg(q + j);
  } else {
    load_u64s_cg<GS>(p, valid, o);
  }
}
template <int GS, bool FAST>
HB_DEV void st_grp(u64* p, int valid, const u64 (&v)[GS]) {
  if constexpr (FAST && GS % 2 == 0) {
#pragma unroll
    for (int j = 0; j < GS; j += 2) *reinterpret_cast<ulonglong2*>(p + j) = make_ulonglong2(v[j], v[j + 1]);
  } else if constexpr (FAST) {
#pragma unroll
    for (int j = 0; j < GS; ++j) p[j] = v[j];
  } else {
    store_u64s<GS>(p, valid, v);
  }
}

// Per-CTA launch constants of the party kernel: [0] flag sequence base (read by the flag thread
// each round, so no register holds it across the tile), [1] receive-region offset.
__shared__ u64 p2p_link_s[2];

// One tile of one party: all rounds.  FULL = every element of the tile is in the layer (the
// direct-store fast path); the partial last tile stages every bool round byte-exactly.
// Returns false when the peer timed out.  `wbytes` accumulates the bytes stored to the peer.
template <int W, bool FULL>
__device__ __forceinline__ bool p2p_tile(const P2PArgs& A, const unsigned cta, const u64 tile, const u64 it,
                                         uint8_t* __restrict__ stage, int& abort_s, u64& wbytes, const u64 roff) {
  using G = Geo<W>;
  using K = Kit<W>;
  using PG = P2PGeo<W>;
  constexpr int GS = G::GS, L = K::L, C = P2P_C, TP = PG::TP, NB = PG::NB;
  constexpr u64 TE = PG::TE, SB = PG::SB, SA = PG::SA;
  const int t = threadIdx.x % TP;
  const bool p0 = A.party == 0;
  const u64 n = A.n;
  const PartyIO& io = A.io;
  constexpr u64 MN = ~0ull;  // Z/2^64 (other rings take the staged path)
  const bool mult = !A.drelu_only;
  (void)it;
  (void)cta;
  const u64 first = tile * TE;
  const u64 cnt = min(TE, n - first);
  constexpr bool full = FULL;
  u64 e0[C];
  int valid[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    e0[c] = first + (u64)(c * TP + t) * GS;
    valid[c] = FULL ? GS : (e0[c] >= n ? 0 : (int)min((u64)GS, n - e0[c]));
  }
  unsigned long long* stamp = nullptr;
#ifdef HB_P2P_STAMPS
  if (A.stamps && t == 0 && cta < 4 && it < 32) stamp = A.stamps + ((A.party * 4 + cta) * 32 + it) * (P2P_MAXR * 5);
#endif
  // this launch's receive region: the kernel-parameter base plus the launch's region offset (0 or
  // region_bytes by launch parity, from the device link state; read once per party)
  auto pkt = [&](bool peer, int r) -> uint8_t* {
    uint8_t* base = (peer ? A.peer_recv : A.recv) + roff;
    return base + A.round_off[r] + tile * PG::packet(r);
  };

  // ---- bool openings: direct coalesced stores into the peer's packet, or byte-exact staging
  auto put_bool = [&](int r, int sg, int c, const Cg<W>& v) {
    Pk<W> p = to_packed<W>(v);
    if constexpr (PG::DIRECT && full) {
      put_peer<W>(pkt(true, r) + sg * SB + (u64)(c * TP + t) * NB, p);
      wbytes += NB;
    } else {
      pk_trim<W>(p, valid[c]);
      put_bytes<W>(stage + sg * SB + (u64)(c * TP + t) * NB, p);
    }
  };
  // staged packets: the valid bytes of each segment to the peer, 16-byte units + byte tail
  auto flush_bool = [&](int r) {
    if constexpr (PG::DIRECT && full) return;
    __syncthreads();
    const unsigned vb = (unsigned)((cnt * W + 7) / 8);  // <= SB
    const unsigned ns = PG::nseg(r);
    uint8_t* dst = pkt(true, r);
    const unsigned nv = vb / 16;
    for (unsigned sg = 0; sg < ns; ++sg)
      for (unsigned k = t; k < nv; k += TP)
        *reinterpret_cast<uint4*>(dst + sg * SB + 16 * k) = *reinterpret_cast<const uint4*>(stage + sg * SB + 16 * k);
    const unsigned tail = vb - 16 * nv;
    if ((unsigned)t < tail)
      for (unsigned sg = 0; sg < ns; ++sg) dst[sg * SB + 16 * nv + t] = stage[sg * SB + 16 * nv + t];
    if (t == 0) wbytes += (u64)vb * ns;
  };
  auto get_bool = [&](int r, int sg, int c) -> Cg<W> {
    const u64* s = reinterpret_cast<const u64*>(pkt(false, r) + sg * SB);
    return from_packed<W>(load_pk_cg<W>(s, (u64)(c * TP + t) * GS, SB / 8));
  };
  auto put_arith = [&](int r, int sg, int c, const u64 (&v)[GS]) {
    u64* d = reinterpret_cast<u64*>(pkt(true, r) + sg * SA) + (u64)(c * TP + t) * GS;
    st_grp<GS, FULL>(d, valid[c], v);
    wbytes += 8 * (u64)valid[c];
  };
  auto get_arith = [&](int r, int sg, int c, u64 (&v)[GS]) {
    ld_grp_cg<GS, FULL>(reinterpret_cast<const u64*>(pkt(false, r) + sg * SA) + (u64)(c * TP + t) * GS, valid[c], v);
  };
  auto bseg = [&](const u64* arr, int sgi, int c) { return load_cg<W>(arr, io.bcur + (u64)sgi * n + e0[c], io.bnw); };

  // lane i < 7 of warp 1 warms L2 with one input range of round q of tile tl while the exchange of
  // the current round is in flight (x, the bool segments of the round, or its arith triples)
  auto prefetch_round = [&](u64 tl, int q) {
    const int lane = t - 32;
    if (lane < 0 || lane >= 7 || tl >= A.ntiles) return;
    const u64 f0 = tl * TE, cn = min(TE, n - f0);
    const int R = L + (mult ? 3 : 2);
    if (lane == 6) {
      if (q == 0 || (mult && q == R - 1)) prefetch_l2(io.x + f0, 8 * cn);
      return;
    }
    if (q <= L) {
      const int nsg = q == 0 ? 1 : 2;
      if (lane >= 3 * nsg) return;
      const int sgi = q == 0 ? 0 : 2 * q - 1 + lane / 3;
      const u64* arr = lane % 3 == 0 ? io.ba : (lane % 3 == 1 ? io.bb : io.bc);
      const u64 b0 = ((io.bcur + (u64)sgi * n + f0) * W) >> 3;
      const u64 b1 = ((io.bcur + (u64)sgi * n + f0 + cn) * W + 7) >> 3;
      const u64 lim = io.bnw * 8;
      if (b0 < lim) prefetch_l2(reinterpret_cast<const uint8_t*>(arr) + b0, min(b1, lim) - b0);
    } else if (lane < 3) {
      const u64* arr = lane == 0 ? io.aa : (lane == 1 ? io.ab : io.ac);
      prefetch_l2(arr + io.acur + (q == L + 1 ? 0 : n) + f0, 8 * cn);
    }
  };
  auto exchange = [&](int r) -> bool {  // release round r of this tile, acquire the peer's
    if (stamp) stamp[r * 5 + 0] = globaltimer();
    __syncthreads();
    if (stamp) stamp[r * 5 + 1] = globaltimer();
    if constexpr (PG::PF) {
      const int R = L + (mult ? 3 : 2);
      if (r + 1 < R) prefetch_round(tile, r + 1);
      else prefetch_round(tile + A.grid, 0);
    }
    if (t == 0) {
      // the CTA's stores to the peer are ordered before this thread by the barrier; the release
      // store is cumulative over them at system scope
      const unsigned long long seq = *reinterpret_cast<volatile u64*>(&p2p_link_s[0]) + (u64)r + 1;
      flag_release(A.sys_scope, A.peer_flag + tile, seq);
      if (stamp) stamp[r * 5 + 2] = globaltimer();
      if (flag_relaxed(A.sys_scope, A.my_flag + tile) < seq) {
        const unsigned long long t0 = globaltimer();
        while (flag_relaxed(A.sys_scope, A.my_flag + tile) < seq) {
          if (globaltimer() - t0 > A.timeout_ns) {
            atomicExch(A.err, 1);
            abort_s = 1;
            break;
          }
        }
      }
      (void)flag_acquire(A.sys_scope, A.my_flag + tile);  // the peer's stores are visible before the barrier
      if (stamp) stamp[r * 5 + 3] = globaltimer();
    }
    __syncthreads();
    if (stamp) stamp[r * 5 + 4] = globaltimer();
    return abort_s == 0;
  };

  // Live across an exchange: only the protocol state S, G, P (and later sign, d).  A round's own
  // openings are recomputed after the exchange from the state and the triple segments the combine
  // reloads anyway (a, b), instead of being held in registers.
  Cg<W> S[C], Gc[C], P[C];
  // ---- round 0: slice, open the generate-bit AND: e = u ^ a, f = v ^ b
#pragma unroll
  for (int c = 0; c < C; ++c) {
    u64 x[GS];
    ld_grp<GS, FULL>(io.x + e0[c], valid[c], x);
    S[c] = K::slice(x, A.m);
    P[c] = S[c];
    const Cg<W> z0 = cg_zero<W>();
    put_bool(0, 0, c, (p0 ? S[c] : z0) ^ bseg(io.ba, 0, c));
    put_bool(0, 1, c, (p0 ? z0 : S[c]) ^ bseg(io.bb, 0, c));
  }
  flush_bool(0);
  if (!exchange(0)) return false;

  // combine of level lv (round 1 + lv): G ^= AND(P, gS), P = AND(P, pS) from the peer's openings
  auto combine_level = [&](int lv, int c, bool need_p) {
    const int qg = 1 + 2 * lv, qp = 2 + 2 * lv, r = 1 + lv;
    const Cg<W> ag = bseg(io.ba, qg, c), bg = bseg(io.bb, qg, c), ap = bseg(io.ba, qp, c), bp = bseg(io.bb, qp, c);
    Cg<W> o[4];
    K::level_open(p0, lv, Gc[c], P[c], ag, bg, ap, bp, o);
    const Cg<W> zg = K::and_z(p0, o[0] ^ get_bool(r, 0, c), o[2] ^ get_bool(r, 2, c), ag, bg, bseg(io.bc, qg, c));
    if (need_p)
      P[c] = K::and_z(p0, o[1] ^ get_bool(r, 1, c), o[3] ^ get_bool(r, 3, c), ap, bp, bseg(io.bc, qp, c));
    Gc[c] = Gc[c] ^ zg;
  };

  // ---- rounds 1..L: combine the previous bool round, open Kogge-Stone level l
#pragma unroll 1
  for (int l = 0; l < L; ++l) {
    const int r = 1 + l, sg = 1 + 2 * l, sp = 2 + 2 * l;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (l == 0) {
        const Cg<W> a0 = bseg(io.ba, 0, c), b0 = bseg(io.bb, 0, c), z0 = cg_zero<W>();
        Gc[c] = K::and_z(p0, ((p0 ? S[c] : z0) ^ a0) ^ get_bool(0, 0, c), ((p0 ? z0 : S[c]) ^ b0) ^ get_bool(0, 1, c),
                         a0, b0, bseg(io.bc, 0, c));
      } else {
        combine_level(l - 1, c, true);
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      Cg<W> o[4];
      K::level_open(p0, l, Gc[c], P[c], bseg(io.ba, sg, c), bseg(io.bb, sg, c), bseg(io.ba, sp, c),
                    bseg(io.bb, sp, c), o);
#pragma unroll
      for (int q = 0; q < 4; ++q) put_bool(r, q, c, o[q]);
    }
    flush_bool(r);
    if (!exchange(r)) return false;
  }

  // ---- combine level L-1, open B2A of the sign bit on Z/2^N (round L+1)
  unsigned sgn[C];
  {
    const int r = L + 1;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      combine_level(L - 1, c, false);
      sgn[c] = K::sign_bits(S[c], Gc[c]);
      u64 e[GS], f[GS];
      ld_grp<GS, FULL>(io.aa + io.acur + e0[c], valid[c], e);
      ld_grp<GS, FULL>(io.ab + io.acur + e0[c], valid[c], f);
#pragma unroll
      for (int j = 0; j < GS; ++j) {
        const u64 bit = (sgn[c] >> j) & 1u;
        e[j] = ((p0 ? bit : 0ull) - e[j]) & MN;
        f[j] = ((p0 ? 0ull : bit) - f[j]) & MN;
      }
      put_arith(r, 0, c, e);
      put_arith(r, 1, c, f);
    }
    if (!exchange(r)) return false;
  }

  // ---- combine B2A -> d = DReLU share (parked in y); open the Mult round y = x * d (round L+2)
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int r = L + 1;
    u64 a1[GS], b1[GS], c1[GS], pe[GS], pf[GS], d[GS];
    ld_grp<GS, FULL>(io.aa + io.acur + e0[c], valid[c], a1);
    ld_grp<GS, FULL>(io.ab + io.acur + e0[c], valid[c], b1);
    ld_grp<GS, FULL>(io.ac + io.acur + e0[c], valid[c], c1);
    get_arith(r, 0, c, pe);
    get_arith(r, 1, c, pf);
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const u64 bit = (sgn[c] >> j) & 1u;
      const u64 E = (((p0 ? bit : 0ull) - a1[j]) + pe[j]) & MN;
      const u64 F = (((p0 ? 0ull : bit) - b1[j]) + pf[j]) & MN;
      const u64 tt = mul_z(p0, E, F, a1[j], b1[j], c1[j], MN);
      d[j] = ((p0 ? 1ull : 0ull) - ((bit - 2 * tt) & MN)) & MN;
    }
    st_grp<GS, FULL>(io.y + e0[c], valid[c], d);
    if (mult) {
      u64 x[GS], a2[GS], b2[GS];
      ld_grp<GS, FULL>(io.x + e0[c], valid[c], x);
      ld_grp<GS, FULL>(io.aa + io.acur + n + e0[c], valid[c], a2);
      ld_grp<GS, FULL>(io.ab + io.acur + n + e0[c], valid[c], b2);
#pragma unroll
      for (int j = 0; j < GS; ++j) {
        x[j] = (x[j] - a2[j]) & MN;  // e
        d[j] = (d[j] - b2[j]) & MN;  // f
      }
      put_arith(r + 1, 0, c, x);
      put_arith(r + 1, 1, c, d);
    }
  }
  if (!mult) return true;
  if (!exchange(L + 2)) return false;

  // ---- combine Mult: y = x * d
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int r = L + 2;
    u64 x[GS], a2[GS], b2[GS], c2[GS], d[GS], pe[GS], pf[GS];
    ld_grp<GS, FULL>(io.x + e0[c], valid[c], x);
    ld_grp<GS, FULL>(io.aa + io.acur + n + e0[c], valid[c], a2);
    ld_grp<GS, FULL>(io.ab + io.acur + n + e0[c], valid[c], b2);
    ld_grp<GS, FULL>(io.ac + io.acur + n + e0[c], valid[c], c2);
    ld_grp_cg<GS, FULL>(io.y + e0[c], valid[c], d);  // this thread's own store of d (program order)
    get_arith(r, 0, c, pe);
    get_arith(r, 1, c, pf);
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const u64 E = (((x[j] - a2[j]) & MN) + pe[j]) & MN;
      const u64 F = (((d[j] - b2[j]) & MN) + pf[j]) & MN;
      x[j] = mul_z(p0, E, F, a2[j], b2[j], c2[j], MN);
    }
    st_grp<GS, FULL>(io.y + e0[c], valid[c], x);
  }
  return true;
}

template <int W>
__device__ __forceinline__ void p2p_party(const P2PArgs& A, const unsigned cta, const unsigned ncta,
                                          uint8_t* __restrict__ stage) {
  constexpr u64 TE = P2PGeo<W>::TE;
  __shared__ int abort_s;
  if (threadIdx.x % P2PGeo<W>::TP == 0) abort_s = 0;
  // the FULL fast path loads / stores whole groups with 16-byte vectors: every per-element array
  // (x, y, the arith triple segments at the cursor and at +n) must be 16-byte aligned
  const PartyIO& io = A.io;
  const uintptr_t al = reinterpret_cast<uintptr_t>(io.x) | reinterpret_cast<uintptr_t>(io.y) |
                       reinterpret_cast<uintptr_t>(io.aa + io.acur) | reinterpret_cast<uintptr_t>(io.ab + io.acur) |
                       reinterpret_cast<uintptr_t>(io.ac + io.acur) | (uintptr_t)(8 * A.n);
  const bool aligned = Geo<W>::GS % 2 == 1 ? (al & 7) == 0 : (al & 15) == 0;
  if (threadIdx.x % P2PGeo<W>::TP == 0) {
    // this launch's flag sequence base and receive-region offset: the host's, or the device link
    // state written by this party's previous launch (stream order)
    p2p_link_s[0] = A.state ? __ldcg(A.state) : A.seq0;
    p2p_link_s[1] = A.state ? (__ldcg(A.state + 1) & 1ull) * A.region_bytes : 0ull;
  }
  __syncthreads();
  const u64 roff = p2p_link_s[1];
  u64 wbytes = 0, it = 0;
  for (u64 tile = cta; tile < A.ntiles; tile += ncta, ++it) {
    const bool ok = aligned && (tile + 1) * TE <= A.n
                        ? p2p_tile<W, true>(A, cta, tile, it, stage, abort_s, wbytes, roff)
                        : p2p_tile<W, false>(A, cta, tile, it, stage, abort_s, wbytes, roff);
    if (!ok) return;  // timed out: the error word is set and the link is dead (state left as is)
  }
  if (A.wire_bytes && wbytes) atomicAdd(A.wire_bytes, (unsigned long long)wbytes);
  if (A.state) {
    // the party's last CTA to finish (every CTA read the state before it got here) advances the
    // sequence by this launch's rounds and flips the region parity for the next launch
    __syncthreads();
    if (threadIdx.x % P2PGeo<W>::TP == 0) {
      __threadfence();
      if (atomicAdd(A.state + 2, 1ull) == ncta - 1) {
        A.state[0] = p2p_link_s[0] + (u64)(Kit<W>::L + (A.drelu_only ? 2 : 3));
        A.state[1] += 1;
        A.state[2] = 0;
        __threadfence();
      }
    }
  }
}

template <int W>
constexpr size_t p2p_smem_bytes() {
  return 4 * P2PGeo<W>::SB;  // the byte-exact staging of one bool round (at most 4 segments)
}

// ONE kernel per width for both uses: CTAs [0, A0.grid) run party A0, CTAs [A0.grid, A0.grid +
// A1.grid) run party A1.  One party on its own GPU (the peer over NVLink): A1.grid = 0.  Both
// parties in one grid on one device (the single-GPU harness; the "remote" buffers are the other
// party's): A1.grid > 0.
template <int W>
__global__ void __launch_bounds__(P2PGeo<W>::TP, P2PGeo<W>::MINB) k_relu_p2p(const P2PArgs A0, const P2PArgs A1) {
  extern __shared__ __align__(16) uint8_t p2p_stage[];
  if (blockIdx.x < A0.grid)
    p2p_party<W>(A0, blockIdx.x, A0.grid, p2p_stage);
  else
    p2p_party<W>(A1, blockIdx.x - A0.grid, A1.grid, p2p_stage);
}

// Receive-buffer layout of ONE launch, identical on both sides: per round, ntiles packets.
template <int W>
u64 p2p_layout(u64 n, int drelu_only, u64 (&off)[P2P_MAXR], u64* ntiles_out) {
  using PG = P2PGeo<W>;
  const u64 ntiles = (n + PG::TE - 1) / PG::TE;
  const int R = PG::L + (drelu_only ? 2 : 3);
  u64 o = 0;
  for (int r = 0; r < P2P_MAXR; ++r) {
    off[r] = o;
    if (r < R) o += ntiles * PG::packet(r);
    o = (o + 255) & ~255ull;
  }
  *ntiles_out = ntiles;
  return o;
}

// Bytes a party stores into its peer's buffer in round r (what crosses NVLink): the exact w-bit
// segments of bool rounds, 8 bytes per element and segment of arithmetic rounds.
template <int W>
u64 p2p_wire_bytes(u64 n, int r) {
  using PG = P2PGeo<W>;
  return r <= PG::L ? (u64)PG::nseg(r) * ((n * W + 7) / 8) : 2 * 8 * n;
}

template <int W>
cudaError_t launch_p2p(P2PArgs A, const P2PArgs* B, int max_ctas, int max_ctas1, int dual_sys, cudaStream_t s) {
  // B == nullptr: one party (A) on this device; otherwise both parties A (party 0), *B (party 1)
  u64 ntiles;
  (void)p2p_layout<W>(A.n, A.drelu_only, A.round_off, &ntiles);
  A.ntiles = ntiles;
  P2PArgs A1 = {};
  if (B) {
    A1 = *B;
    (void)p2p_layout<W>(A1.n, A1.drelu_only, A1.round_off, &ntiles);
    A1.ntiles = ntiles;
  }
  if (ntiles == 0) return cudaSuccess;
  // Z/2^64 only (the configs' ring; masks fold away): other rings take the staged path
  if (A.N != 64) return cudaErrorNotSupported;
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = p2p_smem_bytes<W>();
  const void* fn = (const void*)k_relu_p2p<W>;
  // once per width and device: the shared-memory limit (odd widths stage a bool round byte-exactly:
  // up to 126 KB at w = 63) and the co-resident CTAs per SM -- a per-launch query costs more host
  // time than a small layer's kernel
  static int occ_cache[16] = {};  // per device, 0 = not yet known
  if (dev < 0 || dev >= 16 || occ_cache[dev] == 0) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, P2PGeo<W>::TP, smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 16) occ_cache[dev] = occ;
  } else {
    occ = occ_cache[dev];
  }
  // persistent cooperative grid: every CTA of the launch co-resident (the launch fails otherwise)
  const long long full = (long long)occ * sms;
  auto clamp = [&](long long g, int mx) {
    if (mx > 0 && g > mx) g = mx;
    if ((u64)g > ntiles) g = (long long)ntiles;
    return g < 1 ? 1ll : g;
  };
  const long long g0 = clamp(B ? full / 2 : full, max_ctas);
  const long long g1 = B ? clamp(full / 2, max_ctas1 > 0 ? max_ctas1 : max_ctas) : 0;
  A.grid = (unsigned)g0;
  A1.grid = (unsigned)g1;
  if (getenv("HB_P2P_DEBUG"))
    fprintf(stderr, "[hb_relu_p2p] W=%d %s occ=%d/SM sms=%d grid=%lld+%lld tiles=%llu smem=%zu\n", W,
            B ? (dual_sys ? "both parties (sys scope)" : "both parties (gpu scope)") : "one party", occ, sms, g0, g1,
            (unsigned long long)ntiles, smem);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.gridDim = dim3((unsigned)(g0 + g1));
  cfg.blockDim = dim3(P2PGeo<W>::TP);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  A.sys_scope = B ? (dual_sys ? 1 : 0) : 1;
  A1.sys_scope = A.sys_scope;
  return cudaLaunchKernelEx(&cfg, k_relu_p2p<W>, A, A1);
}

}  // namespace hb
