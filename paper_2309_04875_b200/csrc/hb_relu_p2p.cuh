// hb_relu_p2p.cuh -- one party's whole windowed ReLU in ONE persistent launch, the openings of every
// round exchanged tile by tile through the peer GPU's memory (NVLink P2P stores + flags).
//
// This is the N > 1 counterpart of k_relu_pair: party p runs on its own GPU, both parties run this
// kernel on the same element tiles in the same order.  For tile t and round r a CTA
//   1. computes its masked opening (same Kit<W> round math as k_relu_pair / k_stage),
//   2. stores it straight into the PEER's receive buffer (remote HBM, over NVLink),
//   3. __syncthreads; one thread fences at system scope and releases the peer's flag[t] = seq(r),
//   4. waits (acquire) until its own flag[t] >= seq(r) -- the peer's opening of round r is in its
//      local receive buffer -- and combines.
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
// Deadlock freedom: the grid is persistent and co-resident with margin (3/4 of the occupancy, 1/4
// when both parties share one device), so CTA c of either party always reaches tile t.  A bounded spin (globaltimer, ~timeout_ms) turns a missing peer into an
// error flag instead of a hang.
#pragma once
#include <cstdio>
#include <cstdlib>

#include "hb_relu_impl.cuh"

namespace hb {

constexpr int P2P_TP = 128;      // threads (groups) per CTA = one tile
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
HB_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int W, bool RING64>
__global__ void __launch_bounds__(P2P_TP) k_relu_p2p(const P2PArgs A) {
  using G = Geo<W>;
  using K = Kit<W>;
  using PG = P2PGeo<W>;
  constexpr int GS = G::GS, PW = G::PW, L = K::L, NSEG = 1 + 2 * L, UB = PG::UB, NU = PG::NU;
  constexpr int TP = P2P_TP;
  __shared__ int abort_s;
  const int t = threadIdx.x;
  const bool p0 = A.party == 0;
  const u64 n = A.n;
  const PartyIO& io = A.io;
  const u64 MN = RING64 ? ~0ull : nmask(A.N);
  const bool mult = !A.drelu_only;
  if (t == 0) abort_s = 0;

  for (u64 tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    const u64 e0 = (tile * TP + t) * GS;
    const int valid = e0 >= n ? 0 : (int)min((u64)GS, n - e0);

    // round r: my words k of this tile -> peer, then wait for the peer's and read them locally
    auto wire = [&](uint8_t* base, int r, int k) -> uint8_t* {  // unit k of this thread in round r
      const int ru = PG::round_unit(r);
      return base + A.round_off[r] + ((tile * (PG::round_bytes(r) / ru) + k) * TP + t) * ru;
    };
    auto put_group = [&](int r, int k0, const Cg<W>& v) {
      const Pk<W> p = to_packed<W>(v);
      if constexpr (UB == 4) {
        *reinterpret_cast<uint32_t*>(wire(A.peer_recv, r, k0)) = (uint32_t)p.v[0];
      } else {
#pragma unroll
        for (int q = 0; q < PW; ++q) *reinterpret_cast<u64*>(wire(A.peer_recv, r, k0 + q)) = p.v[q];
      }
    };
    auto get_group = [&](int r, int k0) -> Cg<W> {
      Pk<W> p;
      if constexpr (UB == 4) {
        p.v[0] = (u64)__ldcg(reinterpret_cast<const unsigned int*>(wire(A.recv, r, k0)));
#pragma unroll
        for (int q = 1; q < PW; ++q) p.v[q] = 0;
      } else {
#pragma unroll
        for (int q = 0; q < PW; ++q)
          p.v[q] = (u64)__ldcg(reinterpret_cast<const unsigned long long*>(wire(A.recv, r, k0 + q)));
      }
      return from_packed<W>(p);
    };
    auto put_word = [&](int r, int k, u64 v) { *reinterpret_cast<u64*>(wire(A.peer_recv, r, k)) = v; };
    auto get_word = [&](int r, int k) -> u64 {
      return (u64)__ldcg(reinterpret_cast<const unsigned long long*>(wire(A.recv, r, k)));
    };
    // release round r of this tile to the peer, then acquire the peer's round r
    auto exchange = [&](int r) -> bool {
      __syncthreads();
      if (t == 0) {
        const unsigned long long seq = A.seq0 + (u64)r + 1;
        __threadfence_system();
        st_release_sys(A.peer_flag + tile, seq);
        const unsigned long long t0 = globaltimer();
        while (ld_acquire_sys(A.my_flag + tile) < seq) {
          if (globaltimer() - t0 > A.timeout_ns) {
            atomicExch(A.err, 1);
            abort_s = 1;
            break;
          }
        }
      }
      __syncthreads();
      return abort_s == 0;
    };

    // ---- loads up front, as in k_relu_pair
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

    const Cg<W> S = K::slice(x, A.m);

    // ---- round 0: generate bits
    Cg<W> Gc, P = S;
    {
      const Cg<W> z0 = cg_zero<W>();
      const Cg<W> e = (p0 ? S : z0) ^ ta[0];
      const Cg<W> f = (p0 ? z0 : S) ^ tbv[0];
      put_group(0, 0, e);
      put_group(0, NU, f);
      if (!exchange(0)) return;
      Gc = K::and_z(p0, e ^ get_group(0, 0), f ^ get_group(0, NU), ta[0], tbv[0], tc[0]);
    }
    // ---- rounds 1..L: Kogge-Stone levels
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const int r = 1 + l, sg = 1 + 2 * l, sp = 2 + 2 * l;
      Cg<W> o[4];
      K::level_open(p0, l, Gc, P, ta[sg], tbv[sg], ta[sp], tbv[sp], o);
#pragma unroll
      for (int q = 0; q < 4; ++q) put_group(r, q * NU, o[q]);
      if (!exchange(r)) return;
      const Cg<W> zg = K::and_z(p0, o[0] ^ get_group(r, 0), o[2] ^ get_group(r, 2 * NU), ta[sg], tbv[sg], tc[sg]);
      const Cg<W> zp = K::and_z(p0, o[1] ^ get_group(r, NU), o[3] ^ get_group(r, 3 * NU), ta[sp], tbv[sp], tc[sp]);
      Gc = Gc ^ zg;
      P = zp;
    }
    // ---- round L+1: B2A of the sign bit
    const unsigned sgn = K::sign_bits(S, Gc);
    u64 d[GS];
    {
      const int r = L + 1;
      u64 e1[GS], f1[GS];
#pragma unroll
      for (int j = 0; j < GS; ++j) {
        const u64 bit = (sgn >> j) & 1u;
        e1[j] = ((p0 ? bit : 0ull) - a1[j]) & MN;
        f1[j] = ((p0 ? 0ull : bit) - b1[j]) & MN;
        put_word(r, j, e1[j]);
        put_word(r, GS + j, f1[j]);
      }
      if (!exchange(r)) return;
#pragma unroll
      for (int j = 0; j < GS; ++j) {
        const u64 E = (e1[j] + get_word(r, j)) & MN;
        const u64 F = (f1[j] + get_word(r, GS + j)) & MN;
        const u64 tt = mul_z(p0, E, F, a1[j], b1[j], c1[j], MN);
        const u64 bit = (sgn >> j) & 1u;
        d[j] = ((p0 ? 1ull : 0ull) - ((bit - 2 * tt) & MN)) & MN;
      }
    }
    if (!mult) {
      store_u64s<GS>(io.y + e0, valid, d);
      continue;
    }
    // ---- round L+2: y = MUL(x, d)
    {
      const int r = L + 2;
      u64 e2[GS], f2[GS], yv[GS];
#pragma unroll
      for (int j = 0; j < GS; ++j) {
        e2[j] = (x[j] - a2[j]) & MN;
        f2[j] = (d[j] - b2[j]) & MN;
        put_word(r, j, e2[j]);
        put_word(r, GS + j, f2[j]);
      }
      if (!exchange(r)) return;
#pragma unroll
      for (int j = 0; j < GS; ++j) {
        const u64 E = (e2[j] + get_word(r, j)) & MN;
        const u64 F = (f2[j] + get_word(r, GS + j)) & MN;
        yv[j] = mul_z(p0, E, F, a2[j], b2[j], c2[j], MN);
      }
      store_u64s<GS>(io.y + e0, valid, yv);
    }
  }
}

// receive-buffer layout shared by both parties: per round, ntiles x round_bytes(r) x TP bytes
template <int W>
u64 p2p_layout(u64 n, int drelu_only, u64 (&off)[P2P_MAXR], u64* ntiles_out) {
  using PG = P2PGeo<W>;
  const u64 ntiles = (n + (u64)P2P_TP * PG::GS - 1) / ((u64)P2P_TP * PG::GS);
  const int R = PG::L + (drelu_only ? 2 : 3);
  u64 o = 0;
  for (int r = 0; r < P2P_MAXR; ++r) {
    off[r] = o;
    if (r < R) o += ntiles * (u64)PG::round_bytes(r) * P2P_TP;
    o = (o + 255) & ~255ull;
  }
  *ntiles_out = ntiles;
  return o;
}

template <int W>
cudaError_t launch_p2p(P2PArgs A, int max_ctas, cudaStream_t s) {
  u64 ntiles;
  (void)p2p_layout<W>(A.n, A.drelu_only, A.round_off, &ntiles);
  A.ntiles = ntiles;
  if (ntiles == 0) return cudaSuccess;
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = A.N == 64 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_relu_p2p<W, true>, P2P_TP, 0)
                            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_relu_p2p<W, false>, P2P_TP, 0);
  if (e != cudaSuccess) return e;
  // persistent grid with residency margin: 3/4 of the co-resident CTAs when this party has the GPU
  // to itself, 1/4 when both parties' kernels share one device (max_ctas < 0) -- a deadlock needs
  // BOTH parties partially resident, which the margin keeps away from
  const long long full = (long long)occ * sms;
  long long grid = max_ctas < 0 ? full / 4 : (3 * full) / 4;
  if (grid < 1) grid = 1;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if ((u64)grid > ntiles) grid = (long long)ntiles;
  if (getenv("HB_P2P_DEBUG"))
    fprintf(stderr, "[hb_relu_p2p] W=%d party=%d occ=%d/SM sms=%d grid=%lld tiles=%llu\n", W, A.party, occ, sms, grid,
            (unsigned long long)ntiles);
  if (A.N == 64)
    k_relu_p2p<W, true><<<(unsigned)grid, P2P_TP, 0, s>>>(A);
  else
    k_relu_p2p<W, false><<<(unsigned)grid, P2P_TP, 0, s>>>(A);
  return cudaGetLastError();
}

}  // namespace hb
