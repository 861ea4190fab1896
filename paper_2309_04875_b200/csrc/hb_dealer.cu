// hb_dealer.cu -- trusted-dealer Beaver triples generated in HBM, bit-exact with the
// reference dealer (ringmpc dealer.py:50-83) -- SURVEY 8(f)-3.
//
// The reference draws every array with rng.bytes(8*count) from
// numpy.random.default_rng(SeedSequence(seed)), i.e. consecutive 64-bit outputs of
// PCG64: state <- state * M + inc (128-bit LCG), output = XSL-RR of the NEW state
// (rotr64(hi ^ lo, hi >> 58)).  A batch of `count` triples consumes raw outputs
//     a = raw[0, c)  b = raw[c, 2c)  r_a = raw[2c, 3c)  r_b = raw[3c, 4c)  r_c = raw[4c, 5c)
// (each masked to the width), and party shares are (v + r, -r) or (v ^ r, r).
//
// Each thread owns a run of RUN consecutive triples: it jumps its five stream
// positions ahead in O(log n) 128-bit multiplies (the PCG advance recurrence), then
// steps sequentially -- ~2 128-bit multiply-adds per output.
#include <cstdint>
#include <cuda_runtime.h>

namespace hb {
namespace dealer {

typedef unsigned __int128 u128;

constexpr int RUN = 32;

__device__ __forceinline__ u128 mk(uint64_t lo, uint64_t hi) { return ((u128)hi << 64) | lo; }

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64 - rot) & 63));
}

// state after `delta` LCG steps (pcg_advance_lcg_128)
__device__ u128 advance(u128 state, u128 mult, u128 inc, unsigned long long delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = mult, cur_plus = inc;
  while (delta) {
    if (delta & 1ull) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// kind 0 = arith (c = ab mod 2^w, shares (v + r, -r)), kind 1 = bool (c = a & b, shares (v ^ r, r))
__global__ void k_deal(uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi, int kind, int width,
                       unsigned long long count, unsigned long long first, unsigned long long n, uint64_t* __restrict__ a0,
                       uint64_t* __restrict__ b0, uint64_t* __restrict__ c0, uint64_t* __restrict__ a1,
                       uint64_t* __restrict__ b1, uint64_t* __restrict__ c1) {
  const unsigned long long run = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long e0 = run * RUN;  // offset within [first, first + n)
  if (e0 >= n) return;
  const u128 M = mk(0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull);
  const u128 s0 = mk(s_lo, s_hi), inc = mk(i_lo, i_hi);
  const uint64_t mask = width >= 64 ? ~0ull : ((1ull << width) - 1);
  // stream q (0..4) element e lives at raw position q*count + e; output k uses the state after k+1 steps
  u128 st[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) st[q] = advance(s0, M, inc, (unsigned long long)q * count + first + e0);
  const unsigned long long end = (e0 + RUN < n) ? e0 + RUN : n;
  for (unsigned long long e = e0; e < end; ++e) {
    uint64_t v[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      st[q] = st[q] * M + inc;
      v[q] = xsl_rr(st[q]) & mask;
    }
    const uint64_t a = v[0], b = v[1], ra = v[2], rb = v[3], rc = v[4];
    if (kind == 0) {
      const uint64_t c = (a * b) & mask;
      a0[e] = (a + ra) & mask;
      b0[e] = (b + rb) & mask;
      c0[e] = (c + rc) & mask;
      a1[e] = (0ull - ra) & mask;
      b1[e] = (0ull - rb) & mask;
      c1[e] = (0ull - rc) & mask;
    } else {
      a0[e] = a ^ ra;
      b0[e] = b ^ rb;
      c0[e] = (a & b) ^ rc;
      a1[e] = ra;
      b1[e] = rb;
      c1[e] = rc;
    }
  }
}

// Simulator ReLU (ringmpc simulator.py:47-54 sim_relu): encode x * 2^f round-half-away-from-zero
// onto Z/2^N (ring.py:191-199), split with r = raw PCG64 outputs of the caller's generator
// (rng.bytes, ring.py:207-213; share_arith sharing.py:88-96), decide on the window [m, k)
// (drelu_from_shares simulator.py:33-44) and keep-or-zero in float64 -- x * 1.0 / x * 0.0, the
// reference's arithmetic, so the output is bit-identical.
__global__ void k_sim_relu(const double* __restrict__ x, unsigned long long n, double scale, int ring_bits, int k,
                           int m, uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi, double* __restrict__ out,
                           int* __restrict__ err) {
  const unsigned long long e0 = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) * RUN;
  if (e0 >= n) return;
  const u128 M = mk(0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull);
  const u128 inc = mk(i_lo, i_hi);
  u128 st = advance(mk(s_lo, s_hi), M, inc, e0);
  const uint64_t mask = ring_bits >= 64 ? ~0ull : ((1ull << ring_bits) - 1);
  const int w = k - m;
  const uint64_t wmask = w >= 64 ? ~0ull : ((1ull << w) - 1);
  const double half = ldexp(1.0, ring_bits - 1);
  const unsigned long long end = e0 + RUN < n ? e0 + RUN : n;
  for (unsigned long long i = e0; i < end; ++i) {
    st = st * M + inc;
    const uint64_t r = xsl_rr(st) & mask;
    const double v = x[i], sc = v * scale;
    const double rd = copysign(floor(fabs(sc) + 0.5), sc);
    if (fabs(rd) >= half) atomicExch(err, 1);  // EncodeRangeError
    const uint64_t enc = (uint64_t)(long long)rd & mask;
    const uint64_t s0 = (enc + r) & mask, s1 = (0ull - r) & mask;
    const uint64_t t = (((s0 >> m) & wmask) + ((s1 >> m) & wmask)) & wmask;
    const double keep = (double)(1ull - ((t >> (w - 1)) & 1ull));
    out[i] = v * keep;
  }
}

}  // namespace dealer
}  // namespace hb

cudaError_t hb_sim_relu_launch(const double* x, unsigned long long n, double scale, int ring_bits, int k, int m,
                               uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi, double* out, int* err,
                               cudaStream_t s) {
  const unsigned long long runs = (n + hb::dealer::RUN - 1) / hb::dealer::RUN;
  if (runs)
    hb::dealer::k_sim_relu<<<(unsigned)((runs + 127) / 128), 128, 0, s>>>(x, n, scale, ring_bits, k, m, s_lo, s_hi,
                                                                          i_lo, i_hi, out, err);
  return cudaGetLastError();
}

cudaError_t hb_dealer_launch(uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi, int kind, int width,
                             unsigned long long count, unsigned long long first, unsigned long long n, uint64_t* a0,
                             uint64_t* b0, uint64_t* c0, uint64_t* a1, uint64_t* b1, uint64_t* c1, cudaStream_t s) {
  const unsigned long long runs = (n + hb::dealer::RUN - 1) / hb::dealer::RUN;
  if (runs)
    hb::dealer::k_deal<<<(unsigned)((runs + 127) / 128), 128, 0, s>>>(s_lo, s_hi, i_lo, i_hi, kind, width, count,
                                                                       first, n, a0, b0, c0, a1, b1, c1);
  return cudaGetLastError();
}
