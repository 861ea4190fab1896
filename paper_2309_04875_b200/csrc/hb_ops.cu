// hb_ops.cu -- stage-level kernels behind the per-operation API (beaver_and,
// beaver_mul, circuit_add, a2b, b2a_bit) and the standalone wire codec.
//
// These are element-per-thread kernels on uint64 words: they exist so each
// protocol stage can be checked against the oracle on its own
// (reference tests/test_protocol.py:110-271).  The fused ReLU path does not
// use them.
#include <cstdint>
#include <cuda_runtime.h>

#include "hb_common.cuh"

namespace hb {

constexpr int OPS_TPB = 256;

inline unsigned blocks_for(u64 n) { return (unsigned)((n + OPS_TPB - 1) / OPS_TPB); }

// ---------------------------------------------------------------- codec (transport.py:33-67)
// One thread per output word: OR together the (at most 64/w + 2) element
// fields that overlap bits [64k, 64k + 64) of the stream.
__global__ void k_pack(const u64* __restrict__ v, u64 count, int w, u64* __restrict__ out, u64 nwords) {
  const u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nwords) return;
  const u64 mk = nmask(w);
  const u64 lo_bit = 64 * k, hi_bit = lo_bit + 64;
  u64 e = lo_bit / (u64)w;
  u64 word = 0;
  for (; e < count && e * (u64)w < hi_bit; ++e) {
    const u64 f = v[e] & mk;
    const long long pos = (long long)(e * (u64)w) - (long long)lo_bit;
    word |= pos >= 0 ? (f << pos) : (f >> (-pos));
  }
  out[k] = word;
}

__global__ void k_unpack(const u64* __restrict__ in, u64 count, int w, u64* __restrict__ v) {
  const u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  const u64 b = e * (u64)w;
  const int sh = (int)(b & 63);
  u64 f = in[b >> 6] >> sh;
  if (sh + w > 64) f |= in[(b >> 6) + 1] << (64 - sh);
  v[e] = f & nmask(w);
}

HB_DEV u64 stream_get(const u64* s, u64 e, int w) {
  const u64 b = e * (u64)w;
  const int sh = (int)(b & 63);
  u64 f = s[b >> 6] >> sh;
  if (sh + w > 64) f |= s[(b >> 6) + 1] << (64 - sh);
  return f & nmask(w);
}

// ---------------------------------------------------------------- Beaver openings
// kind 0 = bool (XOR, AND), kind 1 = arith (mod 2^w, MUL); triples are packed
// w-bit streams (bool) or uint64 arrays (arith) at element offset `cur`.
struct Trip {
  const u64 *a, *b, *c;
  u64 cur;
};

HB_DEV u64 trip_get(const u64* s, u64 e, int w, int kind) { return kind == 0 ? stream_get(s, e, w) : s[e]; }

// masked operands [x - a ; y - b] (arith) or [x ^ a ; y ^ b] (bool), unpacked, 2n words
__global__ void k_open_mask(int kind, int w, u64 n, const u64* __restrict__ x, const u64* __restrict__ y, Trip T,
                            u64* __restrict__ out) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 mk = nmask(w);
  const u64 a = trip_get(T.a, T.cur + i, w, kind), b = trip_get(T.b, T.cur + i, w, kind);
  if (kind == 0) {
    out[i] = (x[i] ^ a) & mk;
    out[n + i] = (y[i] ^ b) & mk;
  } else {
    out[i] = (x[i] - a) & mk;
    out[n + i] = (y[i] - b) & mk;
  }
}

// z from own operands + peer's packed payload (protocol.py:85-88, 101-104)
__global__ void k_open_close(int kind, int party, int w, u64 n, const u64* __restrict__ x, const u64* __restrict__ y,
                             Trip T, const u64* __restrict__ peer, u64* __restrict__ z) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 mk = nmask(w);
  const u64 a = trip_get(T.a, T.cur + i, w, kind), b = trip_get(T.b, T.cur + i, w, kind);
  const u64 c = trip_get(T.c, T.cur + i, w, kind);
  const u64 pe = stream_get(peer, i, w), pf = stream_get(peer, n + i, w);
  if (kind == 0) {
    const u64 E = ((x[i] ^ a) ^ pe) & mk, F = ((y[i] ^ b) ^ pf) & mk;
    u64 r = c ^ (E & b) ^ (F & a);
    if (party == 0) r ^= E & F;
    z[i] = r & mk;
  } else {
    const u64 E = ((x[i] - a) + pe) & mk, F = ((y[i] - b) + pf) & mk;
    u64 r = c + E * b + F * a;
    if (party == 0) r += E * F;
    z[i] = r & mk;
  }
}

// ---------------------------------------------------------------- elementwise helpers
enum EwOp {
  EW_SLICE = 0,      // out = (a >> p) & mask(w)                         ring.py:69-72
  EW_MSB = 1,        // out = (a >> (w-1)) & 1                           ring.py:75-77
  EW_XOR = 2,        // out = (a ^ b) & mask(w)
  EW_KS_RHS = 3,     // out[0:n] = (G<<s)&mk ; out[n:2n] = (P<<s)&mk ^ [p0]ones, s = 2^p   protocol.py:130-138
  EW_KS_UPDATE = 4,  // a = G, b = z[2n]: out = G ^ z[0:n] ; out2 = z[n:2n]                   protocol.py:140-141
  EW_KS_FINISH = 5,  // out = a ^ ((b << 1) & mk)                        protocol.py:142-143
  EW_B2A_LIFT = 6,   // a = bit, b = t: out = (bit - 2t) & mk             protocol.py:174-175
  EW_DRELU_OUT = 7,  // out = [p0]1 - a                                  protocol.py:192
  EW_OWNER = 8,      // out = a if party == p else 0  (a2b / b2a operand split)  protocol.py:153-156
  EW_STACK2 = 9,     // out = [a ; a]
  EW_MASKW = 10,     // out = a & mask(w)
  EW_DRELU_SHARES = 11,  // out = 1 - msb((a>>p & mk) + (b>>p & mk)), the plaintext sign oracle  simulator.py:33-44
};

__global__ void k_ewise(int op, int party, int w, u64 n, int p, const u64* __restrict__ a, const u64* __restrict__ b,
                        u64* __restrict__ out, u64* __restrict__ out2) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 mk = nmask(w);
  switch (op) {
    case EW_SLICE: out[i] = (a[i] >> p) & mk; break;
    case EW_MSB: out[i] = (a[i] >> (w - 1)) & 1ull; break;
    case EW_XOR: out[i] = (a[i] ^ b[i]) & mk; break;
    case EW_KS_RHS: {
      const int s = 1 << p;
      const u64 ones = ((s >= 64) ? ~0ull : ((1ull << s) - 1)) & mk;
      out[i] = (a[i] << s) & mk;
      u64 ps = (b[i] << s) & mk;
      if (party == 0) ps ^= ones;
      out[n + i] = ps;
      break;
    }
    case EW_KS_UPDATE:
      out[i] = (a[i] ^ b[i]) & mk;
      out2[i] = b[n + i] & mk;
      break;
    case EW_KS_FINISH: out[i] = (a[i] ^ (b[i] << 1)) & mk; break;
    case EW_B2A_LIFT: out[i] = (a[i] - 2 * b[i]) & mk; break;
    case EW_DRELU_OUT: out[i] = ((party == 0 ? 1ull : 0ull) - a[i]) & mk; break;
    case EW_OWNER: out[i] = (party == p) ? (a[i] & mk) : 0ull; break;
    case EW_STACK2: out[i] = a[i]; out[n + i] = a[i]; break;
    case EW_MASKW: out[i] = a[i] & mk; break;
    case EW_DRELU_SHARES: out[i] = 1ull - (((((a[i] >> p) & mk) + ((b[i] >> p) & mk)) & mk) >> (w - 1)); break;
  }
}

// any word > 1 -> flag (b2a_bit's precondition, protocol.py:166-167)
__global__ void k_any_gt1(const u64* __restrict__ a, u64 n, int* __restrict__ flag) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && a[i] > 1) atomicOr(flag, 1);
}

}  // namespace hb

// ---------------------------------------------------------------- launch wrappers (C++ linkage, used by hb_api.cu)
cudaError_t hb_ops_pack(const hb::u64* v, hb::u64 count, int w, hb::u64* out, cudaStream_t s) {
  const hb::u64 nwords = (count * (hb::u64)w + 63) / 64;
  if (nwords) hb::k_pack<<<hb::blocks_for(nwords), hb::OPS_TPB, 0, s>>>(v, count, w, out, nwords);
  return cudaGetLastError();
}

cudaError_t hb_ops_unpack(const hb::u64* in, hb::u64 count, int w, hb::u64* v, cudaStream_t s) {
  if (count) hb::k_unpack<<<hb::blocks_for(count), hb::OPS_TPB, 0, s>>>(in, count, w, v);
  return cudaGetLastError();
}

cudaError_t hb_ops_open_mask(int kind, int w, hb::u64 n, const hb::u64* x, const hb::u64* y, const hb::u64* ta,
                             const hb::u64* tb, hb::u64 cur, hb::u64* tmp, hb::u64* payload, cudaStream_t s) {
  if (!n) return cudaSuccess;
  hb::Trip T{ta, tb, nullptr, cur};
  hb::k_open_mask<<<hb::blocks_for(n), hb::OPS_TPB, 0, s>>>(kind, w, n, x, y, T, tmp);
  return hb_ops_pack(tmp, 2 * n, w, payload, s);
}

cudaError_t hb_ops_open_close(int kind, int party, int w, hb::u64 n, const hb::u64* x, const hb::u64* y,
                              const hb::u64* ta, const hb::u64* tb, const hb::u64* tc, hb::u64 cur,
                              const hb::u64* peer, hb::u64* z, cudaStream_t s) {
  if (!n) return cudaSuccess;
  hb::Trip T{ta, tb, tc, cur};
  hb::k_open_close<<<hb::blocks_for(n), hb::OPS_TPB, 0, s>>>(kind, party, w, n, x, y, T, peer, z);
  return cudaGetLastError();
}

cudaError_t hb_ops_ewise(int op, int party, int w, hb::u64 n, int p, const hb::u64* a, const hb::u64* b, hb::u64* out,
                         hb::u64* out2, cudaStream_t s) {
  if (!n) return cudaSuccess;
  hb::k_ewise<<<hb::blocks_for(n), hb::OPS_TPB, 0, s>>>(op, party, w, n, p, a, b, out, out2);
  return cudaGetLastError();
}

cudaError_t hb_ops_any_gt1(const hb::u64* a, hb::u64 n, int* flag_dev, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(flag_dev, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  if (n) hb::k_any_gt1<<<hb::blocks_for(n), hb::OPS_TPB, 0, s>>>(a, n, flag_dev);
  return cudaGetLastError();
}
