// hb_relu_p2p.cuh -- one party's whole windowed ReLU in ONE persistent launch, the openings of every
// round exchanged tile by tile through the peer GPU's memory (NVLink P2P stores + flags).
//
// This is the N > 1 counterpart of k_relu_pair: party p runs on its own GPU, both parties run this
// kernel on the same element tiles in the same order.  For tile t and round r a CTA
//   1. computes its masked opening (same Kit<W> round math as k_relu_pair / k_stage),
//   2. stores it straight into the PEER's receive buffer (remote HBM, over NVLink),
//   3. __syncthreads; one thread fences at system scope and releases the peer's flag[t] = seq(r),
//   4. polls its own flag[t] (relaxed) until >= seq(r), then one acquire load of it -- the peer's
//      opening of round r is in its local receive buffer -- and combines.
// The transfer of tile t overlaps the math of the other resident tiles: no per-round launches, no
// host round trips, no NCCL.  Flags are monotonic (seq = epoch * rounds + r + 1) so nothing is
// reset between launches; each round owns a region of the receive buffer, and a party can only be
// one round ahead of its peer on a tile, so regions are never overwritten while still being read.
//
// Wire units: a bool round sends each thread's packed opening words (32-bit units when a group
// packs into <= 32 bits -- w = 8: exactly the reference's bytes; wider groups in 64-bit words);
// the arithmetic rounds send uint64 per element.  The reference meter records the reference
// payload sizes (relu_trace); the wire carries the same bytes for w in {8, 16, 32, 64}.
//
// Deadlock freedom: the grid is persistent and co-resident with margin (3/4 of the occupancy; both
// parties in one grid at 1/2 each when they share a device, k_relu_p2p_dual, party 0 dispatched
// first), so CTA c of either party always reaches tile t.  A bounded spin (globaltimer, ~timeout_ms) turns a missing peer into an
// error flag instead of a hang.
#pragma once
#include <cstdio>
#include <cstdlib>

#include "hb_relu_impl.cuh"

namespace hb {

constexpr int P2P_TP = 128;      // threads per CTA
constexpr int P2P_C = 4;         // groups per thread per chunk (the unit of synchronisation)
constexpr int P2P_MAXR = 10;     // rounds per ReLU <= L + 3 with L <= 6

struct P2PArgs {
  PartyIO io;
  u64 n, ntiles;
  int N, m, party, drelu_only;
  u64 seq0;                       // epoch * rounds: flag value before this launch's round 0
  uint8_t* recv;                  // this party's receive buffer (written by the peer)
  const unsigned long long* my_flag;  // [ntiles], written by the peer
  uint8_t* peer_recv;             // the peer's receive buffer (mapped)
  unsigned long long* peer_flag;  // the peer's flags (mapped)
  u64 round_off[P2P_MAXR];        // byte offset of each round's region (identical on both sides)
  u64 timeout_ns;
  int* err;                       // set to 1 on a spin timeout
};

template <int W>
struct P2PGeo {
  static constexpr int GS = Geo<W>::GS, PW = Geo<W>::PW, PB = Geo<W>::PB;
  static constexpr int UB = PB <= 32 ? 4 : 8;          // wire unit bytes of one packed group
  static constexpr int NU = PB <= 32 ? 1 : PW;         // units per packed group
  static constexpr int L = constexpr_levels(W);
  // bytes per thread of round r: Other 2 groups, level 4 groups, B2A / Mult 2 GS words
  static constexpr __host__ __device__ int round_bytes(int r) {
    return r == 0 ? 2 * NU * UB : (r <= L ? 4 * NU * UB : 2 * GS * 8);
  }
  static constexpr __host__ __device__ int round_unit(int r) { return r <= L ? UB : 8; }
};

HB_DEV void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
HB_DEV unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
HB_DEV unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
HB_DEV void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
HB_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Round-major chunks: a CTA's unit of synchronisation is a chunk of P2P_C x P2P_TP groups (thread t
// owns groups t, t + TP, ..: coalesced), so one flag round trip is amortised over 4x more elements
// than a one-group-per-thread tile.  Between rounds each thread keeps only the protocol state of its
// groups in registers (S, G, P, sign, d); each round's triple segment is loaded in that round (every
// segment is used by exactly one round) and x is re-read for the final multiply.
template <int W, bool RING64>
__device__ __forceinline__ void p2p_party(const P2PArgs& A, const unsigned cta, const unsigned ncta) {
  using G = Geo<W>;
  using K = Kit<W>;
  using PG = P2PGeo<W>;
  constexpr int GS = G::GS, PW = G::PW, L = K::L, UB = PG::UB, NU = PG::NU, C = P2P_C;
  constexpr int TP = P2P_TP;
  __shared__ int abort_s;
  const int t = threadIdx.x;
  const bool p0 = A.party == 0;
  const u64 n = A.n;
  const PartyIO& io = A.io;
  const u64 MN = RING64 ? ~0ull : nmask(A.N);
  const bool mult = !A.drelu_only;
  if (t == 0) abort_s = 0;

  for (u64 tile = cta; tile < A.ntiles; tile += ncta) {
    u64 e0[C];
    int valid[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      e0[c] = ((tile * C + c) * TP + t) * GS;
      valid[c] = e0[c] >= n ? 0 : (int)min((u64)GS, n - e0[c]);
    }
    // unit k of group c of this thread in round r: [round][tile][k][c][t]
    auto wire = [&](uint8_t* base, int r, int k, int c) -> uint8_t* {
      const int ru = PG::round_unit(r);
      return base + A.round_off[r] + (((tile * (PG::round_bytes(r) / ru) + k) * C + c) * TP + t) * ru;
    };
    auto put_group = [&](int r, int k0, int c, const Cg<W>& v) {
      const Pk<W> p = to_packed<W>(v);
      if constexpr (UB == 4) {
        *reinterpret_cast<uint32_t*>(wire(A.peer_recv, r, k0, c)) = (uint32_t)p.v[0];
      } else {
#pragma unroll
        for (int q = 0; q < PW; ++q) *reinterpret_cast<u64*>(wire(A.peer_recv, r, k0 + q, c)) = p.v[q];
      }
    };
    auto get_group = [&](int r, int k0, int c) -> Cg<W> {
      Pk<W> p;
      if constexpr (UB == 4) {
        p.v[0] = (u64)__ldcg(reinterpret_cast<const unsigned int*>(wire(A.recv, r, k0, c)));
#pragma unroll
        for (int q = 1; q < PW; ++q) p.v[q] = 0;
      } else {
#pragma unroll
        for (int q = 0; q < PW; ++q)
          p.v[q] = (u64)__ldcg(reinterpret_cast<const unsigned long long*>(wire(A.recv, r, k0 + q, c)));
      }
      return from_packed<W>(p);
    };
    auto put_word = [&](int r, int k, int c, u64 v) { *reinterpret_cast<u64*>(wire(A.peer_recv, r, k, c)) = v; };
    auto get_word = [&](int r, int k, int c) -> u64 {
      return (u64)__ldcg(reinterpret_cast<const unsigned long long*>(wire(A.recv, r, k, c)));
    };
    auto exchange = [&](int r) -> bool {  // release round r of this chunk, acquire the peer's
      __syncthreads();
      if (t == 0) {
        // the CTA's stores to the peer are ordered before this thread by the barrier; the release
        // store is cumulative over them at system scope
        const unsigned long long seq = A.seq0 + (u64)r + 1;
        st_release_sys(A.peer_flag + tile, seq);
        if (ld_relaxed_sys(A.my_flag + tile) < seq) {
          const unsigned long long t0 = globaltimer();
          while (ld_relaxed_sys(A.my_flag + tile) < seq) {
            if (globaltimer() - t0 > A.timeout_ns) {
              atomicExch(A.err, 1);
              abort_s = 1;
              break;
            }
          }
        }
        (void)ld_acquire_sys(A.my_flag + tile);  // acquire: the peer's stores are visible before the barrier
      }
      __syncthreads();
      return abort_s == 0;
    };
    auto bseg = [&](const u64* arr, int sgi, int c) { return load_cg<W>(arr, io.bcur + (u64)sgi * n + e0[c], io.bnw); };

    Cg<W> S[C], Gc[C], P[C];
    // ---- round 0: slice, generate-bit AND
    {
      Cg<W> e[C], f[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        u64 x[GS];
        load_u64s<GS>(io.x + e0[c], valid[c], x);
        S[c] = K::slice(x, A.m);
        P[c] = S[c];
        const Cg<W> z0 = cg_zero<W>();
        e[c] = (p0 ? S[c] : z0) ^ bseg(io.ba, 0, c);
        f[c] = (p0 ? z0 : S[c]) ^ bseg(io.bb, 0, c);
        put_group(0, 0, c, e[c]);
        put_group(0, NU, c, f[c]);
      }
      if (!exchange(0)) return;
#pragma unroll
      for (int c = 0; c < C; ++c)
        Gc[c] = K::and_z(p0, e[c] ^ get_group(0, 0, c), f[c] ^ get_group(0, NU, c), bseg(io.ba, 0, c),
                         bseg(io.bb, 0, c), bseg(io.bc, 0, c));
    }
    // ---- rounds 1..L: Kogge-Stone levels
#pragma unroll 1
    for (int l = 0; l < L; ++l) {
      const int r = 1 + l, sg = 1 + 2 * l, sp = 2 + 2 * l;
      Cg<W> o[C][4];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        K::level_open(p0, l, Gc[c], P[c], bseg(io.ba, sg, c), bseg(io.bb, sg, c), bseg(io.ba, sp, c),
                      bseg(io.bb, sp, c), o[c]);
#pragma unroll
        for (int q = 0; q < 4; ++q) put_group(r, q * NU, c, o[c][q]);
      }
      if (!exchange(r)) return;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const Cg<W> zg = K::and_z(p0, o[c][0] ^ get_group(r, 0, c), o[c][2] ^ get_group(r, 2 * NU, c),
                                  bseg(io.ba, sg, c), bseg(io.bb, sg, c), bseg(io.bc, sg, c));
        const Cg<W> zp = K::and_z(p0, o[c][1] ^ get_group(r, NU, c), o[c][3] ^ get_group(r, 3 * NU, c),
                                  bseg(io.ba, sp, c), bseg(io.bb, sp, c), bseg(io.bc, sp, c));
        Gc[c] = Gc[c] ^ zg;
        P[c] = zp;
      }
    }
    // ---- round L+1: B2A of the sign bit
    u64 d[C][GS];
    {
      const int r = L + 1;
      unsigned sgn[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        sgn[c] = K::sign_bits(S[c], Gc[c]);
        u64 a1[GS], b1[GS];
        load_u64s<GS>(io.aa + io.acur + e0[c], valid[c], a1);
        load_u64s<GS>(io.ab + io.acur + e0[c], valid[c], b1);
#pragma unroll
        for (int j = 0; j < GS; ++j) {
          const u64 bit = (sgn[c] >> j) & 1u;
          put_word(r, j, c, ((p0 ? bit : 0ull) - a1[j]) & MN);
          put_word(r, GS + j, c, ((p0 ? 0ull : bit) - b1[j]) & MN);
        }
      }
      if (!exchange(r)) return;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        u64 a1[GS], b1[GS], c1[GS];
        load_u64s<GS>(io.aa + io.acur + e0[c], valid[c], a1);
        load_u64s<GS>(io.ab + io.acur + e0[c], valid[c], b1);
        load_u64s<GS>(io.ac + io.acur + e0[c], valid[c], c1);
#pragma unroll
        for (int j = 0; j < GS; ++j) {
          const u64 bit = (sgn[c] >> j) & 1u;
          const u64 e1 = ((p0 ? bit : 0ull) - a1[j]) & MN, f1 = ((p0 ? 0ull : bit) - b1[j]) & MN;
          const u64 E = (e1 + get_word(r, j, c)) & MN;
          const u64 F = (f1 + get_word(r, GS + j, c)) & MN;
          const u64 tt = mul_z(p0, E, F, a1[j], b1[j], c1[j], MN);
          d[c][j] = ((p0 ? 1ull : 0ull) - ((bit - 2 * tt) & MN)) & MN;
        }
      }
    }
    if (!mult) {
#pragma unroll
      for (int c = 0; c < C; ++c) store_u64s<GS>(io.y + e0[c], valid[c], d[c]);
      continue;
    }
    // ---- round L+2: y = MUL(x, d)
    {
      const int r = L + 2;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        u64 x[GS], a2[GS], b2[GS];
        load_u64s<GS>(io.x + e0[c], valid[c], x);
        load_u64s<GS>(io.aa + io.acur + n + e0[c], valid[c], a2);
        load_u64s<GS>(io.ab + io.acur + n + e0[c], valid[c], b2);
#pragma unroll
        for (int j = 0; j < GS; ++j) {
          put_word(r, j, c, (x[j] - a2[j]) & MN);
          put_word(r, GS + j, c, (d[c][j] - b2[j]) & MN);
        }
      }
      if (!exchange(r)) return;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        u64 x[GS], a2[GS], b2[GS], c2[GS], yv[GS];
        load_u64s<GS>(io.x + e0[c], valid[c], x);
        load_u64s<GS>(io.aa + io.acur + n + e0[c], valid[c], a2);
        load_u64s<GS>(io.ab + io.acur + n + e0[c], valid[c], b2);
        load_u64s<GS>(io.ac + io.acur + n + e0[c], valid[c], c2);
#pragma unroll
        for (int j = 0; j < GS; ++j) {
          const u64 E = (((x[j] - a2[j]) & MN) + get_word(r, j, c)) & MN;
          const u64 F = (((d[c][j] - b2[j]) & MN) + get_word(r, GS + j, c)) & MN;
          yv[j] = mul_z(p0, E, F, a2[j], b2[j], c2[j], MN);
        }
        store_u64s<GS>(io.y + e0[c], valid[c], yv);
      }
    }
  }
}

template <int W, bool RING64>
__global__ void __launch_bounds__(P2P_TP) k_relu_p2p(const P2PArgs A) {
  p2p_party<W, RING64>(A, blockIdx.x, gridDim.x);
}

// Both parties in ONE grid on one device (CTAs [0, G) party 0, [G, 2G) party 1): the single-GPU
// harness of the party kernel -- no dependence on two streams actually running concurrently.
template <int W, bool RING64>
__global__ void __launch_bounds__(P2P_TP) k_relu_p2p_dual(const P2PArgs A0, const P2PArgs A1) {
  const unsigned g = gridDim.x / 2;
  if (blockIdx.x < g)
    p2p_party<W, RING64>(A0, blockIdx.x, g);
  else
    p2p_party<W, RING64>(A1, blockIdx.x - g, g);
}

// receive-buffer layout shared by both parties: per round, ntiles x round_bytes(r) x TP bytes
template <int W>
u64 p2p_layout(u64 n, int drelu_only, u64 (&off)[P2P_MAXR], u64* ntiles_out) {
  using PG = P2PGeo<W>;
  const u64 chunk = (u64)P2P_TP * P2P_C * PG::GS;  // elements per chunk
  const u64 ntiles = (n + chunk - 1) / chunk;
  const int R = PG::L + (drelu_only ? 2 : 3);
  u64 o = 0;
  for (int r = 0; r < P2P_MAXR; ++r) {
    off[r] = o;
    if (r < R) o += ntiles * (u64)PG::round_bytes(r) * P2P_TP * P2P_C;
    o = (o + 255) & ~255ull;
  }
  *ntiles_out = ntiles;
  return o;
}

template <int W>
cudaError_t launch_p2p(P2PArgs A, const P2PArgs* B, int max_ctas, cudaStream_t s) {
  // B == nullptr: one party (A) on this device; otherwise both parties A (party 0), *B (party 1)
  u64 ntiles;
  (void)p2p_layout<W>(A.n, A.drelu_only, A.round_off, &ntiles);
  A.ntiles = ntiles;
  P2PArgs A1;
  if (B) {
    A1 = *B;
    (void)p2p_layout<W>(A1.n, A1.drelu_only, A1.round_off, &ntiles);
    A1.ntiles = ntiles;
  }
  if (ntiles == 0) return cudaSuccess;
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Z/2^64 only (the configs' ring; masks fold away): other rings take the staged path
  if (A.N != 64) return cudaErrorNotSupported;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_relu_p2p<W, true>, P2P_TP, 0);
  if (e != cudaSuccess) return e;
  // persistent grid: 3/4 of the co-resident CTAs for one party on its own GPU (residency margin: a
  // deadlock needs BOTH parties partially resident); half each for the single-grid two-party harness,
  // whose party-0 CTAs are dispatched first and so are always all resident
  const long long full = (long long)occ * sms;
  long long grid = B ? full / 2 : (3 * full) / 4;
  if (grid < 1) grid = 1;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if ((u64)grid > ntiles) grid = (long long)ntiles;
  if (getenv("HB_P2P_DEBUG"))
    fprintf(stderr, "[hb_relu_p2p] W=%d %s occ=%d/SM sms=%d grid=%lld per party, tiles=%llu\n", W,
            B ? "both parties" : "one party", occ, sms, grid, (unsigned long long)ntiles);
  if (B)
    k_relu_p2p_dual<W, true><<<(unsigned)(2 * grid), P2P_TP, 0, s>>>(A, A1);
  else
    k_relu_p2p<W, true><<<(unsigned)grid, P2P_TP, 0, s>>>(A);
  return cudaGetLastError();
}

}  // namespace hb
