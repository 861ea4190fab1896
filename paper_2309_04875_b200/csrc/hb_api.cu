// hb_api.cu -- extern "C" entry points of libhbrelu.so (declared in include/hb_relu.h).
//
// Host-side validation mirrors the reference's error behaviour: bad windows /
// widths / shapes are ConfigError (ring.py:116-128, protocol.py:78-79,95-96),
// short triple streams are TripleExhaustedError (dealer.py:152-163), and all of
// it is decided before the first kernel or exchange so both parties fail alike.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hb_relu.h"
#include "hb_relu_impl.cuh"
#include "hb_relu_p2p.cuh"
#include "hb_ring_tc.cuh"
#include "hb_conv_tma.cuh"

cudaError_t hb_sim_relu_launch(const double* x, unsigned long long n, double scale, int ring_bits, int k, int m,
                               uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi, double* out, int* err,
                               cudaStream_t s);

using hb::u64;

// ---- per-range dispatchers (hb_relu_w*.cu)
#define HB_RANGE(lo, hi)                                                                            \
  cudaError_t hb_pair_dispatch_##lo##_##hi(int W, const hb::PairArgs& A, cudaStream_t s);          \
  cudaError_t hb_stage_dispatch_##lo##_##hi(int W, const hb::StageArgs& A, int L, cudaStream_t s); \
  cudaError_t hb_p2p_dispatch_##lo##_##hi(int W, const hb::P2PArgs& A, const hb::P2PArgs* B, int max_ctas, \
                                          int max_ctas1, int dual_sys, cudaStream_t s);                \
  unsigned long long hb_p2p_layout_##lo##_##hi(int W, unsigned long long n, int drelu_only,        \
                                               unsigned long long* ntiles);                        \
  size_t hb_pair_smem_##lo##_##hi(int W);
HB_RANGE(2, 8)
HB_RANGE(9, 16)
HB_RANGE(17, 24)
HB_RANGE(25, 32)
HB_RANGE(33, 40)
HB_RANGE(41, 48)
HB_RANGE(49, 56)
HB_RANGE(57, 64)
#undef HB_RANGE

// ---- stage-op wrappers (hb_ops.cu)
cudaError_t hb_ops_pack(const u64* v, u64 count, int w, u64* out, cudaStream_t s);
cudaError_t hb_ops_unpack(const u64* in, u64 count, int w, u64* v, cudaStream_t s);
cudaError_t hb_ops_open_mask(int kind, int w, u64 n, const u64* x, const u64* y, const u64* ta, const u64* tb, u64 cur,
                             u64* tmp, u64* payload, cudaStream_t s);
cudaError_t hb_ops_open_close(int kind, int party, int w, u64 n, const u64* x, const u64* y, const u64* ta,
                              const u64* tb, const u64* tc, u64 cur, const u64* peer, u64* z, cudaStream_t s);
cudaError_t hb_ops_ewise(int op, int party, int w, u64 n, int p, const u64* a, const u64* b, u64* out, u64* out2,
                         cudaStream_t s);
cudaError_t hb_ops_any_gt1(const u64* a, u64 n, int* flag_dev, cudaStream_t s);
cudaError_t hb_dealer_launch(uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi, int kind, int width,
                             unsigned long long count, unsigned long long first, unsigned long long n, uint64_t* a0,
                             uint64_t* b0, uint64_t* c0, uint64_t* a1, uint64_t* b1, uint64_t* c1, cudaStream_t s);

// ---- ring linear-layer kernels (hb_ring.cu)
cudaError_t hb_ring_limbs_im2col(const u64* x, int B, int C, int H, int W, int kh, int kw, int stride, int pad,
                                 long long Kp, int8_t* A, cudaStream_t s);
cudaError_t hb_ring_combine(const int32_t* P, long long M, long long N, long long Np, int J, const int32_t* colsum,
                            int party, int frac, const u64* bias, int layout, long long S, u64* out, cudaStream_t s);
cudaError_t hb_ring_avgpool(const u64* x, long long BC, int H, int W, int kh, int kw, int stride, u64 inv, int party,
                            int frac, u64* out, cudaStream_t s);
cudaError_t hb_ring_add(const u64* a, const u64* b, long long n, u64* out, cudaStream_t s);
cudaError_t hb_ring_avgpool_nhwc(const u64* x, long long B, int H, int W, int C, int kh, int kw, int stride, u64 inv,
                                 int party, int frac, u64* out, cudaStream_t s);

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return HB_OK;
  (void)cudaGetLastError();  // a failed launch must not surface again in the next call's status
  return fail(HB_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int levels(int w) {
  int l = 0;
  while ((1 << l) < w) ++l;
  return l < 1 ? 1 : l;
}

int group_size(int w) { return hb::group_size_for(w); }
int group_words(int w) { return hb::group_words_for(w); }

int64_t nbytes(int64_t count, int w) { return 8 * ((count * (int64_t)w + 63) / 64); }

int check_window(int ring_bits, int k, int m) {
  if (ring_bits < 1 || ring_bits > 64) return fail(HB_ERR_CONFIG, "ring width must be in 1..64, got %d", ring_bits);
  if (!(0 <= m && m < k && k <= 64)) return fail(HB_ERR_CONFIG, "need 0 <= m < k <= 64, got (k=%d, m=%d)", k, m);
  if (k - m < 2) return fail(HB_ERR_CONFIG, "window width must be >= 2, got (k=%d, m=%d)", k, m);
  if (k > ring_bits) return fail(HB_ERR_CONFIG, "window (k=%d, m=%d) exceeds ring width %d", k, m, ring_bits);
  return HB_OK;
}

int check_triples(const hb_triples_t& t, const char* kind, int width, int64_t need, int party) {
  if (t.width != width)
    return fail(HB_ERR_TRIPLES, "party %d needs %s triples of width %d, stream has width %d", party, kind, width,
                t.width);
  if (t.cursor < 0 || t.cursor + need > t.capacity)
    return fail(HB_ERR_TRIPLES, "party %d needs %lld %s triples of width %d, %lld left", party, (long long)need, kind,
                width, (long long)(t.capacity - t.cursor));
  if (need > 0 && (!t.a || !t.b || !t.c)) return fail(HB_ERR_CONFIG, "null triple pointer");
  return HB_OK;
}

cudaError_t pair_dispatch(int W, const hb::PairArgs& A, cudaStream_t s) {
  if (W <= 8) return hb_pair_dispatch_2_8(W, A, s);
  if (W <= 16) return hb_pair_dispatch_9_16(W, A, s);
  if (W <= 24) return hb_pair_dispatch_17_24(W, A, s);
  if (W <= 32) return hb_pair_dispatch_25_32(W, A, s);
  if (W <= 40) return hb_pair_dispatch_33_40(W, A, s);
  if (W <= 48) return hb_pair_dispatch_41_48(W, A, s);
  if (W <= 56) return hb_pair_dispatch_49_56(W, A, s);
  return hb_pair_dispatch_57_64(W, A, s);
}

cudaError_t stage_dispatch(int W, const hb::StageArgs& A, int L, cudaStream_t s) {
  if (W <= 8) return hb_stage_dispatch_2_8(W, A, L, s);
  if (W <= 16) return hb_stage_dispatch_9_16(W, A, L, s);
  if (W <= 24) return hb_stage_dispatch_17_24(W, A, L, s);
  if (W <= 32) return hb_stage_dispatch_25_32(W, A, L, s);
  if (W <= 40) return hb_stage_dispatch_33_40(W, A, L, s);
  if (W <= 48) return hb_stage_dispatch_41_48(W, A, L, s);
  if (W <= 56) return hb_stage_dispatch_49_56(W, A, L, s);
  return hb_stage_dispatch_57_64(W, A, L, s);
}

#define HB_RANGE_CALL(fn, W, ...)                              \
  ((W) <= 8    ? fn##_2_8(W, __VA_ARGS__)                       \
   : (W) <= 16 ? fn##_9_16(W, __VA_ARGS__)                      \
   : (W) <= 24 ? fn##_17_24(W, __VA_ARGS__)                     \
   : (W) <= 32 ? fn##_25_32(W, __VA_ARGS__)                     \
   : (W) <= 40 ? fn##_33_40(W, __VA_ARGS__)                     \
   : (W) <= 48 ? fn##_41_48(W, __VA_ARGS__)                     \
   : (W) <= 56 ? fn##_49_56(W, __VA_ARGS__)                     \
               : fn##_57_64(W, __VA_ARGS__))

hb::PartyIO make_io(const uint64_t* x, uint64_t* y, const hb_triples_t& bw, const hb_triples_t& ar, int w) {
  hb::PartyIO io;
  io.x = x;
  io.y = y;
  io.ba = bw.a;
  io.bb = bw.b;
  io.bc = bw.c;
  io.bcur = (u64)bw.cursor;
  io.bnw = (u64)((bw.capacity * (int64_t)w + 63) / 64);
  io.aa = ar.a;
  io.ab = ar.b;
  io.ac = ar.c;
  io.acur = (u64)ar.cursor;
  return io;
}

// workspace carve-up for the staged driver
struct WsLayout {
  size_t S, G, P, d, sign, total;
};

size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

WsLayout ws_layout(int w, int64_t n) {
  const int gs = group_size(w), nw = group_words(w);
  const size_t ng = (size_t)((n + gs - 1) / gs);
  WsLayout L{};
  size_t off = 0;
  L.S = off;
  off += align256(8 * nw * ng);
  L.G = off;
  off += align256(8 * nw * ng);
  L.P = off;
  off += align256(8 * nw * ng);
  L.d = off;
  off += align256(8 * (size_t)n);
  L.sign = off;
  off += align256(4 * ng);
  L.total = off;
  return L;
}

}  // namespace

extern "C" {

const char* hb_last_error(void) { return g_err.c_str(); }
int hb_version(void) { return 1; }

int hb_prefix_levels(int w) { return levels(w); }
int64_t hb_payload_bytes(int64_t count, int w) { return nbytes(count, w); }

int hb_relu_rounds(int k, int m, int drelu_only) { return levels(k - m) + (drelu_only ? 2 : 3); }

int64_t hb_relu_round_bytes(int ring_bits, int k, int m, int64_t n, int round) {
  const int w = k - m, L = levels(w);
  if (round == 0) return nbytes(2 * n, w);
  if (round <= L) return nbytes(4 * n, w);
  return nbytes(2 * n, ring_bits);
}

int hb_relu_round_tag(int k, int m, int round) {
  const int L = levels(k - m);
  if (round == 0) return HB_TAG_OTHER;
  if (round <= L) return HB_TAG_CIRCUIT;
  if (round == L + 1) return HB_TAG_B2A;
  return HB_TAG_MULT;
}

int hb_relu_pair(int ring_bits, int k, int m, int64_t n, const uint64_t* x0, const uint64_t* x1, uint64_t* y0,
                 uint64_t* y1, hb_triples_t bool0, hb_triples_t bool1, hb_triples_t arith0, hb_triples_t arith1,
                 int drelu_only, void* stream) {
  return hb_relu_pair_range(ring_bits, k, m, n, 0, n, x0, x1, y0, y1, bool0, bool1, arith0, arith1, drelu_only,
                            stream);
}

int hb_relu_pair_range(int ring_bits, int k, int m, int64_t n, int64_t first, int64_t count, const uint64_t* x0,
                       const uint64_t* x1, uint64_t* y0, uint64_t* y1, hb_triples_t bool0, hb_triples_t bool1,
                       hb_triples_t arith0, hb_triples_t arith1, int drelu_only, void* stream) {
  if (first < 0 || count < 0 || first + count > n) return fail(HB_ERR_CONFIG, "element range outside the layer");
  int rc = check_window(ring_bits, k, m);
  if (rc) return rc;
  if (n < 0) return fail(HB_ERR_CONFIG, "negative element count");
  const int w = k - m, L = levels(w);
  const int64_t nb = n * (1 + 2 * (int64_t)L), na = (drelu_only ? 1 : 2) * n;
  if ((rc = check_triples(bool0, "bool", w, nb, 0)) || (rc = check_triples(bool1, "bool", w, nb, 1)) ||
      (rc = check_triples(arith0, "arith", ring_bits, na, 0)) || (rc = check_triples(arith1, "arith", ring_bits, na, 1)))
    return rc;
  if (count == 0) return HB_OK;
  hb::PairArgs A;
  A.io[0] = make_io(x0, y0, bool0, arith0, w);
  A.io[1] = make_io(x1, y1, bool1, arith1, w);
  A.n = (u64)n;
  A.first = (u64)first;
  A.count = (u64)count;
  A.N = ring_bits;
  A.m = m;
  A.drelu_only = drelu_only ? 1 : 0;
  return cuda_status(pair_dispatch(w, A, S(stream)), "hb_relu_pair");
}

// Per-device streams and events of the pinned-host pipeline (created once, reused by every call).
struct HostPipe {
  cudaStream_t in = nullptr, k = nullptr, out = nullptr;
  std::vector<cudaEvent_t> ev;
  std::mutex busy;  // one pipelined call at a time per device (the events are reused)
};
static HostPipe& host_pipe(int dev) {
  static std::mutex mu;
  static std::map<int, HostPipe> pipes;
  std::lock_guard<std::mutex> g(mu);
  HostPipe& p = pipes[dev];  // std::map: references stay valid as devices are added
  if (!p.in) {
    cudaStreamCreateWithFlags(&p.in, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&p.k, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&p.out, cudaStreamNonBlocking);
  }
  return p;
}

int hb_relu_pair_host(int ring_bits, int k, int m, int64_t n, const uint64_t* hx0, const uint64_t* hx1, uint64_t* hy0,
                      uint64_t* hy1, hb_triples_t bool0, hb_triples_t bool1, hb_triples_t arith0, hb_triples_t arith1,
                      int drelu_only, int64_t chunk, uint64_t* scratch, void* stream) {
  if (n < 0 || chunk <= 0) return fail(HB_ERR_CONFIG, "bad element count or chunk");
  if (n == 0)
    return hb_relu_pair_range(ring_bits, k, m, n, 0, 0, nullptr, nullptr, nullptr, nullptr, bool0, bool1, arith0,
                              arith1, drelu_only, stream);
  if (!hx0 || !hx1 || !hy0 || !hy1 || !scratch) return fail(HB_ERR_CONFIG, "missing host buffer or scratch");
  // chunk schedule: `chunk` elements in the middle, ramping from chunk/8 at both ends (shorter
  // pipeline fill and drain)
  std::vector<std::pair<int64_t, int64_t>> ch;  // (first, count)
  {
    int64_t left = n;
    std::vector<int64_t> head, mid, tail;
    for (int s = 3; s >= 1 && left > 0; --s) {
      const int64_t c = std::min<int64_t>(std::max<int64_t>(chunk >> s, 1), left);
      head.push_back(c);
      left -= c;
    }
    for (int s = 3; s >= 1 && left > chunk; --s) {
      const int64_t c = std::max<int64_t>(chunk >> s, 1);
      tail.push_back(c);
      left -= c;
    }
    while (left > 0) {
      mid.push_back(std::min(chunk, left));
      left -= mid.back();
    }
    int64_t lo = 0;
    for (int64_t c : head) ch.push_back({lo, c}), lo += c;
    for (int64_t c : mid) ch.push_back({lo, c}), lo += c;
    for (auto it = tail.rbegin(); it != tail.rend(); ++it) ch.push_back({lo, *it}), lo += *it;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  HostPipe& P = host_pipe(dev);
  std::lock_guard<std::mutex> hold(P.busy);
  while (P.ev.size() < 2 * ch.size() + 2) {  // only the holder of `busy` touches the events
    cudaEvent_t ev;
    const cudaError_t ce = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (ce != cudaSuccess) return cuda_status(ce, "hb_relu_pair_host events");
    P.ev.push_back(ev);
  }
  // Both parties' shares of a chunk move in ONE two-row copy when the host buffers allow it (each
  // copy costs ~20 us of fixed overhead on these boxes, comparable to a 1 MB transfer): the device
  // rows are laid out in the host buffers' address order so both row pitches are positive.
  const bool in_fwd = hx0 < hx1, out_fwd = hy0 < hy1;
  uint64_t *d0 = scratch + (in_fwd ? 0 : n), *d1 = scratch + (in_fwd ? n : 0);
  uint64_t *e0 = scratch + (out_fwd ? 2 * n : 3 * n), *e1 = scratch + (out_fwd ? 3 * n : 2 * n);
  const size_t pin = (size_t)(in_fwd ? (const char*)hx1 - (const char*)hx0 : (const char*)hx0 - (const char*)hx1);
  const size_t pout = (size_t)(out_fwd ? (const char*)hy1 - (const char*)hy0 : (const char*)hy0 - (const char*)hy1);
  static const bool no2d = getenv("HB_PIPE_2D") && getenv("HB_PIPE_2D")[0] == '0';
  int max_pitch = 0;
  cudaDeviceGetAttribute(&max_pitch, cudaDevAttrMaxPitch, dev);
  const bool pitch_ok = (size_t)8 * n <= (size_t)max_pitch;
  // a two-row copy is only valid when both rows lie in ONE host allocation (e.g. a pinned [2, n]
  // buffer); the runtime rejects it otherwise (cudaErrorInvalidValue, synchronous, not sticky) and
  // that direction falls back to one copy per share
  bool row_in = !no2d && pitch_ok && pin >= (size_t)8 * n && pin <= (size_t)max_pitch;
  bool row_out = !no2d && pitch_ok && pout >= (size_t)8 * n && pout <= (size_t)max_pitch;
  auto h2d = [&](int64_t lo, int64_t c) {
    if (row_in) {
      const cudaError_t r = cudaMemcpy2DAsync(in_fwd ? d0 + lo : d1 + lo, 8 * (size_t)n, in_fwd ? hx0 + lo : hx1 + lo,
                                              pin, 8 * c, 2, cudaMemcpyHostToDevice, P.in);
      if (r != cudaErrorInvalidValue) return r;
      (void)cudaGetLastError();
      row_in = false;
    }
    cudaError_t r = cudaMemcpyAsync(d0 + lo, hx0 + lo, 8 * c, cudaMemcpyHostToDevice, P.in);
    return r == cudaSuccess ? cudaMemcpyAsync(d1 + lo, hx1 + lo, 8 * c, cudaMemcpyHostToDevice, P.in) : r;
  };
  auto d2h = [&](int64_t lo, int64_t c) {
    if (row_out) {
      const cudaError_t r = cudaMemcpy2DAsync(out_fwd ? hy0 + lo : hy1 + lo, pout, out_fwd ? e0 + lo : e1 + lo,
                                              8 * (size_t)n, 8 * c, 2, cudaMemcpyDeviceToHost, P.out);
      if (r != cudaErrorInvalidValue) return r;
      (void)cudaGetLastError();
      row_out = false;
    }
    cudaError_t r = cudaMemcpyAsync(hy0 + lo, e0 + lo, 8 * c, cudaMemcpyDeviceToHost, P.out);
    return r == cudaSuccess ? cudaMemcpyAsync(hy1 + lo, e1 + lo, 8 * c, cudaMemcpyDeviceToHost, P.out) : r;
  };
  cudaEvent_t start = P.ev[2 * ch.size()], done = P.ev[2 * ch.size() + 1];
  // the scratch and the triples are ordered on the caller's stream
  cudaError_t e = cudaEventRecord(start, S(stream));
  for (cudaStream_t st : {P.in, P.k, P.out})
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, start, 0);
  if (e != cudaSuccess) return cuda_status(e, "hb_relu_pair_host");
  // on a failure after work was queued, drain the internal streams before returning: the caller
  // frees the scratch and host buffers the queued copies / kernels still reference
  auto drain = [&](int rc) {
    for (cudaStream_t st : {P.in, P.k, P.out}) (void)cudaStreamSynchronize(st);
    return rc;
  };
  // Three issue phases -- every H2D chunk, then every kernel range, then every D2H chunk -- so no
  // D2H that waits on an event is queued between two H2D copies (with torch-level streams the
  // interleaved order measured 7.9 ms per 2^24 step vs 6.3-6.5 ordered; natively both orders land
  // at 6.2-7.0 ms, box to box -- tools/diag_zerocopy.py, tools/gpu_e2e_chunk_sweep.sh)
  for (size_t i = 0; i < ch.size(); ++i) {
    const int64_t lo = ch[i].first, c = ch[i].second;
    e = h2d(lo, c);
    if (e == cudaSuccess) e = cudaEventRecord(P.ev[2 * i], P.in);
    if (e != cudaSuccess) return drain(cuda_status(e, "hb_relu_pair_host H2D"));
  }
  for (size_t i = 0; i < ch.size(); ++i) {
    const int64_t lo = ch[i].first, c = ch[i].second;
    e = cudaStreamWaitEvent(P.k, P.ev[2 * i], 0);
    if (e != cudaSuccess) return drain(cuda_status(e, "hb_relu_pair_host"));
    const int rc = hb_relu_pair_range(ring_bits, k, m, n, lo, c, d0, d1, e0, e1, bool0, bool1, arith0, arith1,
                                      drelu_only, P.k);
    if (rc) return drain(rc);
    e = cudaEventRecord(P.ev[2 * i + 1], P.k);
    if (e != cudaSuccess) return drain(cuda_status(e, "hb_relu_pair_host"));
  }
  for (size_t i = 0; i < ch.size(); ++i) {
    const int64_t lo = ch[i].first, c = ch[i].second;
    e = cudaStreamWaitEvent(P.out, P.ev[2 * i + 1], 0);
    if (e == cudaSuccess) e = d2h(lo, c);
    if (e != cudaSuccess) return drain(cuda_status(e, "hb_relu_pair_host D2H"));
  }
  e = cudaEventRecord(done, P.out);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(S(stream), done, 0);
  if (e == cudaSuccess) e = cudaEventSynchronize(done);  // the host outputs are complete on return
  return cuda_status(e, "hb_relu_pair_host");
}

uint64_t hb_relu_p2p_bytes(int k, int m, int64_t n, int drelu_only, int64_t* ntiles) {
  if (k - m < 2 || k - m > 64 || n < 0) return 0;
  unsigned long long nt = 0;
  const uint64_t b = HB_RANGE_CALL(hb_p2p_layout, k - m, (unsigned long long)n, drelu_only, &nt);
  if (ntiles) *ntiles = (int64_t)nt;
  return b;
}

uint64_t hb_relu_p2p_wire_bytes(int k, int m, int64_t n, int drelu_only) {
  // what hb_relu_p2p stores into the peer's buffer per launch: every bool round's segments as exact
  // w-bit streams (ceil(n w / 8) bytes each), 8 bytes per element and segment of the arith rounds
  const int w = k - m;
  if (w < 2 || w > 64 || n < 0) return 0;
  const int L = levels(w), R = L + (drelu_only ? 2 : 3);
  const uint64_t seg = ((uint64_t)n * (uint64_t)w + 7) / 8;
  uint64_t b = 0;
  for (int r = 0; r < R; ++r) b += r == 0 ? 2 * seg : (r <= L ? 4 * seg : 16 * (uint64_t)n);
  return b;
}

namespace {
int p2p_args(int party, int ring_bits, int k, int m, int64_t n, const uint64_t* x, uint64_t* y,
             const hb_triples_t& boolw, const hb_triples_t& arith, void* recv, const uint64_t* my_flags,
             void* peer_recv, uint64_t* peer_flags, uint64_t seq0, double timeout_s, int* err_dev, int drelu_only,
             uint64_t* wire_bytes, hb::P2PArgs& A) {
  int rc = check_window(ring_bits, k, m);
  if (rc) return rc;
  if (ring_bits != 64) return fail(HB_ERR_CONFIG, "the P2P party kernel runs on Z/2^64 shares (ring_bits %d)", ring_bits);
  if (party != 0 && party != 1) return fail(HB_ERR_CONFIG, "party must be 0 or 1, got %d", party);
  if (n < 0) return fail(HB_ERR_CONFIG, "negative element count");
  if (n > 0 && (!recv || !my_flags || !peer_recv || !peer_flags || !err_dev))
    return fail(HB_ERR_CONFIG, "null p2p buffer");
  if ((reinterpret_cast<uintptr_t>(recv) | reinterpret_cast<uintptr_t>(peer_recv)) & 255)
    return fail(HB_ERR_CONFIG, "p2p receive buffers must be 256-byte aligned");
  const int w = k - m, L = levels(w);
  const int64_t nb = n * (1 + 2 * (int64_t)L), na = (drelu_only ? 1 : 2) * n;
  if ((rc = check_triples(boolw, "bool", w, nb, party)) || (rc = check_triples(arith, "arith", ring_bits, na, party)))
    return rc;
  A.io = make_io(x, y, boolw, arith, w);
  A.n = (u64)n;
  A.N = ring_bits;
  A.m = m;
  A.party = party;
  A.drelu_only = drelu_only ? 1 : 0;
  A.seq0 = seq0;
  A.recv = static_cast<uint8_t*>(recv);
  A.my_flag = reinterpret_cast<const unsigned long long*>(my_flags);
  A.peer_recv = static_cast<uint8_t*>(peer_recv);
  A.peer_flag = reinterpret_cast<unsigned long long*>(peer_flags);
  A.timeout_ns = (u64)(timeout_s * 1e9);
  A.err = err_dev;
  A.wire_bytes = reinterpret_cast<unsigned long long*>(wire_bytes);
  A.stamps = nullptr;
  A.state = nullptr;
  A.region_bytes = 0;
  return HB_OK;
}
}  // namespace

int hb_relu_p2p(int party, int ring_bits, int k, int m, int64_t n, const uint64_t* x, uint64_t* y,
                hb_triples_t boolw, hb_triples_t arith, void* recv, const uint64_t* my_flags, void* peer_recv,
                uint64_t* peer_flags, uint64_t seq0, int max_ctas, double timeout_s, int* err_dev, int drelu_only,
                uint64_t* wire_bytes_dev, void* stream) {
  hb::P2PArgs A;
  const int rc = p2p_args(party, ring_bits, k, m, n, x, y, boolw, arith, recv, my_flags, peer_recv, peer_flags, seq0,
                          timeout_s, err_dev, drelu_only, wire_bytes_dev, A);
  if (rc || n == 0) return rc;
  return cuda_status(
      HB_RANGE_CALL(hb_p2p_dispatch, k - m, A, (const hb::P2PArgs*)nullptr, max_ctas, 0, 0, S(stream)),
      "hb_relu_p2p");
}

int hb_relu_p2p_pair(int ring_bits, int k, int m, int64_t n, const uint64_t* x0, const uint64_t* x1, uint64_t* y0,
                     uint64_t* y1, hb_triples_t bool0, hb_triples_t bool1, hb_triples_t arith0, hb_triples_t arith1,
                     void* recv0, void* recv1, uint64_t* flags0, uint64_t* flags1, uint64_t seq0, int max_ctas0,
                     int max_ctas1, int sys_scope, double timeout_s, int* err_dev, int drelu_only,
                     uint64_t* wire_bytes_dev, void* stream) {
  hb::P2PArgs A0, A1;
  int rc = p2p_args(0, ring_bits, k, m, n, x0, y0, bool0, arith0, recv0, flags0, recv1, flags1, seq0, timeout_s,
                    err_dev, drelu_only, wire_bytes_dev, A0);
  if (rc) return rc;
  rc = p2p_args(1, ring_bits, k, m, n, x1, y1, bool1, arith1, recv1, flags1, recv0, flags0, seq0, timeout_s, err_dev,
                drelu_only, wire_bytes_dev, A1);
  if (rc || n == 0) return rc;
  return cuda_status(HB_RANGE_CALL(hb_p2p_dispatch, k - m, A0, &A1, max_ctas0, max_ctas1, sys_scope, S(stream)),
                     "hb_relu_p2p_pair");
}

int hb_relu_p2p_dev(int party, int ring_bits, int k, int m, int64_t n, const uint64_t* x, uint64_t* y,
                    hb_triples_t boolw, hb_triples_t arith, void* recv, const uint64_t* my_flags, void* peer_recv,
                    uint64_t* peer_flags, uint64_t* state_dev, uint64_t region_bytes, int max_ctas, double timeout_s,
                    int* err_dev, int drelu_only, uint64_t* wire_bytes_dev, void* stream) {
  if (!state_dev || (region_bytes & 255)) return fail(HB_ERR_CONFIG, "device link state and a 256-byte region needed");
  hb::P2PArgs A;
  const int rc = p2p_args(party, ring_bits, k, m, n, x, y, boolw, arith, recv, my_flags, peer_recv, peer_flags, 0,
                          timeout_s, err_dev, drelu_only, wire_bytes_dev, A);
  if (rc || n == 0) return rc;
  A.state = reinterpret_cast<unsigned long long*>(state_dev);
  A.region_bytes = region_bytes;
  return cuda_status(
      HB_RANGE_CALL(hb_p2p_dispatch, k - m, A, (const hb::P2PArgs*)nullptr, max_ctas, 0, 0, S(stream)),
      "hb_relu_p2p_dev");
}

int hb_relu_p2p_pair_dev(int ring_bits, int k, int m, int64_t n, const uint64_t* x0, const uint64_t* x1, uint64_t* y0,
                         uint64_t* y1, hb_triples_t bool0, hb_triples_t bool1, hb_triples_t arith0,
                         hb_triples_t arith1, void* recv0, void* recv1, uint64_t* flags0, uint64_t* flags1,
                         uint64_t* state0, uint64_t* state1, uint64_t region_bytes, int max_ctas0, int max_ctas1,
                         int sys_scope, double timeout_s, int* err_dev, int drelu_only, uint64_t* wire_bytes_dev,
                         void* stream) {
  if (!state0 || !state1 || (region_bytes & 255))
    return fail(HB_ERR_CONFIG, "device link states and a 256-byte region needed");
  hb::P2PArgs A0, A1;
  int rc = p2p_args(0, ring_bits, k, m, n, x0, y0, bool0, arith0, recv0, flags0, recv1, flags1, 0, timeout_s, err_dev,
                    drelu_only, wire_bytes_dev, A0);
  if (rc) return rc;
  rc = p2p_args(1, ring_bits, k, m, n, x1, y1, bool1, arith1, recv1, flags1, recv0, flags0, 0, timeout_s, err_dev,
                drelu_only, wire_bytes_dev, A1);
  if (rc || n == 0) return rc;
  A0.state = reinterpret_cast<unsigned long long*>(state0);
  A1.state = reinterpret_cast<unsigned long long*>(state1);
  A0.region_bytes = A1.region_bytes = region_bytes;
  return cuda_status(HB_RANGE_CALL(hb_p2p_dispatch, k - m, A0, &A1, max_ctas0, max_ctas1, sys_scope, S(stream)),
                     "hb_relu_p2p_pair_dev");
}

int hb_set_device(int device) {
  // this library links its own (static) CUDA runtime: bind the calling thread to the caller's device
  // explicitly instead of relying on the driver context another runtime made current
  return cuda_status(cudaSetDevice(device), "hb_set_device");
}

int hb_dev_alloc(uint64_t bytes, void** dev_ptr) {
  // a whole allocation of its own (CUDA IPC maps allocations, not sub-ranges of a caching
  // allocator's segment), zero-filled
  cudaError_t e = cudaMalloc(dev_ptr, bytes ? bytes : 1);
  if (e == cudaSuccess) e = cudaMemset(*dev_ptr, 0, bytes ? bytes : 1);
  // the zero fill must land before the buffer is exported or a kernel on any stream (or the peer's
  // kernel, through IPC) stores into it: cudaMemset is asynchronous to the host
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return cuda_status(e, "hb_dev_alloc");
}

int hb_dev_free(void* dev_ptr) { return cuda_status(cudaFree(dev_ptr), "hb_dev_free"); }

int hb_ipc_export(void* dev_ptr, uint8_t* handle64) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
  if (e != cudaSuccess) return cuda_status(e, "hb_ipc_export");
  memcpy(handle64, &h, sizeof(h));
  return HB_OK;
}

int hb_ipc_open(const uint8_t* handle64, void** dev_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "hb_ipc_open");
}

int hb_ipc_close(void* dev_ptr) { return cuda_status(cudaIpcCloseMemHandle(dev_ptr), "hb_ipc_close"); }

size_t hb_relu_workspace_bytes(int k, int m, int64_t n) {
  if (k - m < 2 || k - m > 64 || n < 0) return 0;
  return ws_layout(k - m, n).total;
}

int hb_relu_round(int party, int ring_bits, int k, int m, int64_t n, int round, const uint64_t* x, uint64_t* y,
                  hb_triples_t boolw, hb_triples_t arith, void* workspace, const uint64_t* peer, uint64_t* own,
                  int drelu_only, void* stream) {
  int rc = check_window(ring_bits, k, m);
  if (rc) return rc;
  if (party != 0 && party != 1) return fail(HB_ERR_CONFIG, "party must be 0 or 1, got %d", party);
  if (n < 0) return fail(HB_ERR_CONFIG, "negative element count");
  const int w = k - m, L = levels(w);
  const int last = hb_relu_rounds(k, m, drelu_only);
  if (round < 0 || round > last) return fail(HB_ERR_CONFIG, "round %d outside 0..%d", round, last);
  const int64_t nb = n * (1 + 2 * (int64_t)L), na = (drelu_only ? 1 : 2) * n;
  if ((rc = check_triples(boolw, "bool", w, nb, party)) || (rc = check_triples(arith, "arith", ring_bits, na, party)))
    return rc;
  if (n == 0) return HB_OK;
  if (round > 0 && !peer) return fail(HB_ERR_TRANSPORT, "round %d needs the peer payload", round);
  const bool writes_payload = round < last;
  if (writes_payload && !own) return fail(HB_ERR_CONFIG, "round %d needs an output payload buffer", round);

  const WsLayout Lw = ws_layout(w, n);
  char* ws = static_cast<char*>(workspace);
  hb::StageArgs A;
  A.io = make_io(x, y, boolw, arith, w);
  A.n = (u64)n;
  A.ngroups = (u64)((n + group_size(w) - 1) / group_size(w));
  A.N = ring_bits;
  A.m = m;
  A.party = party;
  A.round = round;
  A.drelu_only = drelu_only ? 1 : 0;
  A.bool_excl = (n % group_size(w)) == 0;
  A.arith_excl = ring_bits == 64;
  A.S = reinterpret_cast<u64*>(ws + Lw.S);
  A.Gs = reinterpret_cast<u64*>(ws + Lw.G);
  A.Ps = reinterpret_cast<u64*>(ws + Lw.P);
  A.d = reinterpret_cast<u64*>(ws + Lw.d);
  A.sign = reinterpret_cast<unsigned*>(ws + Lw.sign);
  A.peer = peer;
  const int64_t peer_segs = round == 1 ? 2 : 4;
  A.peer_nw = (u64)((peer_segs * n * (int64_t)w + 63) / 64);
  A.own = own;

  if (writes_payload) {
    const bool bool_round = round <= L;
    const bool needs_zero = bool_round ? !A.bool_excl : !A.arith_excl;
    const size_t bytes = (size_t)hb_relu_round_bytes(ring_bits, k, m, n, round);
    if (needs_zero) {
      cudaError_t e = cudaMemsetAsync(own, 0, bytes, S(stream));
      if (e != cudaSuccess) return cuda_status(e, "hb_relu_round memset");
    } else {
      // the stream's last word is zero-padded past count*w bits (transport.py:39-49);
      // the kernel's byte-exact stores never touch the padding, so clear that word first
      const int64_t segs = round == 0 ? 2 : (bool_round ? 4 : 2);
      const int64_t bits = segs * n * (int64_t)(bool_round ? w : ring_bits);
      if (bits % 64) {
        cudaError_t e = cudaMemsetAsync(reinterpret_cast<char*>(own) + bytes - 8, 0, 8, S(stream));
        if (e != cudaSuccess) return cuda_status(e, "hb_relu_round pad");
      }
    }
  }
  return cuda_status(stage_dispatch(w, A, L, S(stream)), "hb_relu_round");
}

size_t hb_relu_callback_workspace_bytes(int ring_bits, int k, int m, int64_t n) {
  if (k - m < 2 || n < 0) return 0;
  const int w = k - m;
  size_t pay = (size_t)nbytes(4 * n, w);
  const size_t ar = (size_t)nbytes(2 * n, ring_bits);
  if (ar > pay) pay = ar;
  return hb_relu_workspace_bytes(k, m, n) + 2 * align256(pay);
}

int hb_relu(int party, int ring_bits, int k, int m, int64_t n, const uint64_t* x, uint64_t* y, hb_triples_t boolw,
            hb_triples_t arith, void* workspace, int drelu_only, hb_exchange_fn exchange, void* user, void* stream) {
  int rc = check_window(ring_bits, k, m);
  if (rc) return rc;
  if (!exchange) return fail(HB_ERR_CONFIG, "null exchange callback");
  const int last = hb_relu_rounds(k, m, drelu_only);
  const int w = k - m, L = levels(w);
  const int64_t nb = n * (1 + 2 * (int64_t)L), na = (drelu_only ? 1 : 2) * n;
  if ((rc = check_triples(boolw, "bool", w, nb, party)) || (rc = check_triples(arith, "arith", ring_bits, na, party)))
    return rc;
  char* ws = static_cast<char*>(workspace);
  const size_t base = hb_relu_workspace_bytes(k, m, n);
  size_t pay = (size_t)nbytes(4 * n, w);
  const size_t ar = (size_t)nbytes(2 * n, ring_bits);
  if (ar > pay) pay = ar;
  uint64_t* own = reinterpret_cast<uint64_t*>(ws + base);
  uint64_t* peer = reinterpret_cast<uint64_t*>(ws + base + align256(pay));
  for (int r = 0; r <= last; ++r) {
    rc = hb_relu_round(party, ring_bits, k, m, n, r, x, y, boolw, arith, workspace, r ? peer : nullptr,
                       r < last ? own : nullptr, drelu_only, stream);
    if (rc) return rc;
    if (r < last) {
      const int64_t bytes = hb_relu_round_bytes(ring_bits, k, m, n, r);
      // the callback may read `own` / write `peer` with any copy engine or stream: finish the round first
      if ((rc = cuda_status(cudaStreamSynchronize(S(stream)), "hb_relu"))) return rc;
      if (exchange(user, hb_relu_round_tag(k, m, r), own, peer, bytes, stream) != 0)
        return fail(HB_ERR_TRANSPORT, "exchange failed in round %d", r);
    }
  }
  return HB_OK;
}

int hb_pack(const uint64_t* values, int64_t count, int w, uint64_t* out, void* stream) {
  if (w < 1 || w > 64) return fail(HB_ERR_CONFIG, "pack width must be in 1..64, got %d", w);
  if (count < 0) return fail(HB_ERR_CONFIG, "negative count");
  return cuda_status(hb_ops_pack(values, (u64)count, w, out, S(stream)), "hb_pack");
}

int hb_unpack(const uint64_t* packed, int64_t count, int w, uint64_t* values, void* stream) {
  if (w < 1 || w > 64) return fail(HB_ERR_CONFIG, "pack width must be in 1..64, got %d", w);
  if (count < 0) return fail(HB_ERR_CONFIG, "negative count");
  return cuda_status(hb_ops_unpack(packed, (u64)count, w, values, S(stream)), "hb_unpack");
}

int hb_beaver_open(int kind, int w, int64_t count, const uint64_t* x, const uint64_t* y, hb_triples_t t, uint64_t* tmp,
                   uint64_t* payload, void* stream) {
  if (w < 1 || w > 64) return fail(HB_ERR_CONFIG, "width must be in 1..64, got %d", w);
  if (kind != 0 && kind != 1) return fail(HB_ERR_CONFIG, "kind must be 0 (bool) or 1 (arith)");
  int rc = check_triples(t, kind ? "arith" : "bool", w, count, -1);
  if (rc) return rc;
  return cuda_status(hb_ops_open_mask(kind, w, (u64)count, x, y, t.a, t.b, (u64)t.cursor, tmp, payload, S(stream)),
                     "hb_beaver_open");
}

int hb_beaver_close(int kind, int party, int w, int64_t count, const uint64_t* x, const uint64_t* y, hb_triples_t t,
                    const uint64_t* peer_payload, uint64_t* z, void* stream) {
  if (w < 1 || w > 64) return fail(HB_ERR_CONFIG, "width must be in 1..64, got %d", w);
  if (party != 0 && party != 1) return fail(HB_ERR_CONFIG, "party must be 0 or 1, got %d", party);
  int rc = check_triples(t, kind ? "arith" : "bool", w, count, party);
  if (rc) return rc;
  return cuda_status(hb_ops_open_close(kind, party, w, (u64)count, x, y, t.a, t.b, t.c, (u64)t.cursor, peer_payload, z,
                                       S(stream)),
                     "hb_beaver_close");
}

int hb_ewise(int op, int party, int w, int64_t count, int p, const uint64_t* a, const uint64_t* b, uint64_t* out,
             uint64_t* out2, void* stream) {
  if (w < 1 || w > 64) return fail(HB_ERR_CONFIG, "width must be in 1..64, got %d", w);
  if (op < HB_EW_SLICE || op > HB_EW_DRELU_SHARES) return fail(HB_ERR_CONFIG, "unknown elementwise op %d", op);
  return cuda_status(hb_ops_ewise(op, party, w, (u64)count, p, a, b, out, out2, S(stream)), "hb_ewise");
}

int hb_any_above_one(const uint64_t* a, int64_t count, int* result, void* stream) {
  int* flag = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int), S(stream));
  if (e != cudaSuccess) return cuda_status(e, "hb_any_above_one alloc");
  e = hb_ops_any_gt1(a, (u64)count, flag, S(stream));
  int host = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&host, flag, sizeof(int), cudaMemcpyDeviceToHost, S(stream));
  cudaFreeAsync(flag, S(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
  if (e != cudaSuccess) return cuda_status(e, "hb_any_above_one");
  *result = host;
  return HB_OK;
}

int hb_im2col_limbs(const uint64_t* x, int batch, int channels, int height, int width, int kh, int kw, int stride,
                    int pad, int64_t k_padded, int8_t* out, void* stream) {
  if (batch < 0 || channels <= 0 || height <= 0 || width <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0)
    return fail(HB_ERR_CONFIG, "bad conv geometry");
  if (k_padded < (int64_t)channels * kh * kw) return fail(HB_ERR_CONFIG, "k_padded smaller than C*kh*kw");
  if (height + 2 * pad < kh || width + 2 * pad < kw) return fail(HB_ERR_CONFIG, "kernel larger than padded input");
  return cuda_status(hb_ring_limbs_im2col(x, batch, channels, height, width, kh, kw, stride, pad, k_padded, out,
                                          S(stream)),
                     "hb_im2col_limbs");
}

int hb_limb_combine(const int32_t* products, int64_t m, int64_t n, int64_t n_padded, int j_limbs,
                    const int32_t* colsum, int party, int frac_bits, const uint64_t* bias, int layout, int64_t spatial,
                    uint64_t* out, void* stream) {
  if (n_padded < n) return fail(HB_ERR_CONFIG, "n_padded < n");
  if (j_limbs < 1 || j_limbs > 8) return fail(HB_ERR_CONFIG, "weight limbs must be in 1..8");
  if (party != 0 && party != 1) return fail(HB_ERR_CONFIG, "party must be 0 or 1, got %d", party);
  if (frac_bits < 0 || frac_bits >= 64) return fail(HB_ERR_CONFIG, "frac_bits must be in 0..63");
  if (layout == 1 && (spatial <= 0 || m % spatial)) return fail(HB_ERR_CONFIG, "spatial must divide m");
  return cuda_status(hb_ring_combine(products, m, n, n_padded, j_limbs, colsum, party, frac_bits, bias, layout,
                                     spatial, out, S(stream)),
                     "hb_limb_combine");
}

int hb_avgpool(const uint64_t* x, int64_t batch_channels, int height, int width, int kh, int kw, int stride,
               uint64_t inv, int party, int frac_bits, uint64_t* out, void* stream) {
  if (kh <= 0 || kw <= 0 || stride <= 0 || kh > height || kw > width) return fail(HB_ERR_CONFIG, "bad pool geometry");
  return cuda_status(hb_ring_avgpool(x, batch_channels, height, width, kh, kw, stride, inv, party, frac_bits, out,
                                     S(stream)),
                     "hb_avgpool");
}

int hb_conv_limbs_tc(const uint64_t* x, int batch, int channels, int height, int width, int kh, int kw, int stride,
                     int pad, const int8_t* wlimbs, int n_out, int j_limbs, int64_t k_padded, int n_tile, int party,
                     int frac_bits, const uint64_t* bias, uint64_t* y, void* stream) {
  if (batch < 0 || channels <= 0 || height <= 0 || width <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0)
    return fail(HB_ERR_CONFIG, "bad conv geometry");
  if (height + 2 * pad < kh || width + 2 * pad < kw) return fail(HB_ERR_CONFIG, "kernel larger than padded input");
  const int64_t K = (int64_t)channels * kh * kw;
  if (k_padded % 64 || k_padded < K) return fail(HB_ERR_CONFIG, "k_padded must be a multiple of 64 >= C*kh*kw");
  if (K > 21900) return fail(HB_ERR_CONFIG, "K = %lld too large for exact int32 shift accumulators", (long long)K);
  if (j_limbs < 1 || j_limbs > 3) return fail(HB_ERR_CONFIG, "tensor-core path supports 1..3 weight limbs");
  if (n_tile != 16 && n_tile != 32 && n_tile != 64) return fail(HB_ERR_CONFIG, "n_tile must be 16, 32 or 64");
  if (party != 0 && party != 1) return fail(HB_ERR_CONFIG, "party must be 0 or 1, got %d", party);
  hb::tc::ConvArgs A;
  A.x = x;
  A.B = batch;
  A.C = channels;
  A.H = height;
  A.W = width;
  A.kh = kh;
  A.kw = kw;
  A.stride = stride;
  A.pad = pad;
  A.OH = (height + 2 * pad - kh) / stride + 1;
  A.OW = (width + 2 * pad - kw) / stride + 1;
  A.M = (long long)batch * A.OH * A.OW;
  A.K = K;
  A.Kp = (int)k_padded;
  A.N = n_out;
  A.J = j_limbs;
  A.wl = wlimbs;
  A.party = party;
  A.frac = frac_bits;
  A.bias = bias;
  A.y = y;
  if (A.M == 0) return HB_OK;
  return cuda_status(hb_tc_conv(A, n_tile, S(stream)), "hb_conv_limbs_tc");
}

int hb_sim_relu(const double* x, int64_t n, int frac_bits, int ring_bits, int k, int m, uint64_t state_lo,
                uint64_t state_hi, uint64_t inc_lo, uint64_t inc_hi, double* out, int* err_dev, void* stream) {
  int rc = check_window(ring_bits, k, m);
  if (rc) return rc;
  if (n < 0 || frac_bits < 0 || frac_bits >= ring_bits) return fail(HB_ERR_CONFIG, "bad sim_relu arguments");
  return cuda_status(hb_sim_relu_launch(x, (unsigned long long)n, ldexp(1.0, frac_bits), ring_bits, k, m, state_lo,
                                        state_hi, inc_lo, inc_hi, out, err_dev, S(stream)),
                     "hb_sim_relu");
}

int hb_limbs_nhwc(const uint64_t* x, int batch, int channels, int height, int width, uint8_t* planes, void* stream) {
  if (batch < 0 || channels <= 0 || height <= 0 || width <= 0) return fail(HB_ERR_CONFIG, "bad tensor geometry");
  if (channels % 64) return fail(HB_ERR_CONFIG, "limb planes need channels %% 64 == 0, got %d", channels);
  return cuda_status(hb_limbs_nhwc_launch(x, batch, channels, (long long)height * width, planes, S(stream)),
                     "hb_limbs_nhwc");
}

int hb_im2col_planes(const uint64_t* x, int batch, int channels, int height, int width, int kh, int kw, int stride,
                     int pad, uint8_t* planes, void* stream) {
  if (batch < 0 || channels <= 0 || height <= 0 || width <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0)
    return fail(HB_ERR_CONFIG, "bad conv geometry");
  if (channels * kh * kw > 64) return fail(HB_ERR_CONFIG, "im2col planes need C*kh*kw <= 64");
  if (height + 2 * pad < kh || width + 2 * pad < kw) return fail(HB_ERR_CONFIG, "kernel larger than padded input");
  return cuda_status(hb_im2col_planes_launch(x, batch, channels, height, width, kh, kw, stride, pad, planes, S(stream)),
                     "hb_im2col_planes");
}

static int hb_conv_check_tma(int batch, int channels, int height, int width, int kh, int kw, int stride, int pad,
                             int j_limbs, int n_tile) {
  if (batch < 0 || channels <= 0 || height <= 0 || width <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0)
    return fail(HB_ERR_CONFIG, "bad conv geometry");
  if (height + 2 * pad < kh || width + 2 * pad < kw) return fail(HB_ERR_CONFIG, "kernel larger than padded input");
  if (channels % 64) return fail(HB_ERR_CONFIG, "TMA conv needs channels %% 64 == 0, got %d", channels);
  if (stride > 8 || (width + 2 * pad - kw) / stride + 1 > 256) return fail(HB_ERR_CONFIG, "stride / width out of range");
  const int64_t K = (int64_t)channels * kh * kw;
  if (K > 21900) return fail(HB_ERR_CONFIG, "K = %lld too large for exact int32 shift accumulators", (long long)K);
  if (j_limbs < 1 || j_limbs > 3) return fail(HB_ERR_CONFIG, "tensor-core path supports 1..3 weight limbs");
  if (n_tile != 16 && n_tile != 32 && n_tile != 64 && n_tile != 128)
    return fail(HB_ERR_CONFIG, "n_tile must be 16, 32, 64 or 128");
  int bb, bh, bw;
  const int oh = (height + 2 * pad - kh) / stride + 1, ow = (width + 2 * pad - kw) / stride + 1;
  if (hb_tma_conv_box(batch, oh, ow, &bb, &bh, &bw))
    return fail(HB_ERR_CONFIG, "output %dx%d does not tile into 128-pixel boxes", oh, ow);
  return HB_OK;
}

int hb_conv_limbs_tma(const uint8_t* planes, int batch, int channels, int height, int width, int kh, int kw,
                      int stride, int pad, const int8_t* wlimbs, int n_out, int j_limbs, int n_tile, int party,
                      int frac_bits, const uint64_t* bias, const uint64_t* residual, uint64_t* y, void* stream) {
  int rc = hb_conv_check_tma(batch, channels, height, width, kh, kw, stride, pad, j_limbs, n_tile);
  if (rc) return rc;
  if (party != 0 && party != 1) return fail(HB_ERR_CONFIG, "party must be 0 or 1, got %d", party);
  const uint8_t* pl[1] = {planes};
  const uint64_t* rs[1] = {residual};
  uint64_t* ys[1] = {y};
  return cuda_status(hb_tma_conv(1, pl, batch, channels, height, width, kh, kw, stride, pad, wlimbs, n_out, j_limbs,
                                 n_tile, &party, frac_bits, bias, rs, ys, S(stream)),
                     "hb_conv_limbs_tma");
}

int hb_conv_limbs_tma_pair(const uint8_t* planes0, const uint8_t* planes1, int batch, int channels, int height,
                           int width, int kh, int kw, int stride, int pad, const int8_t* wlimbs, int n_out, int j_limbs,
                           int n_tile, int frac_bits, const uint64_t* bias, const uint64_t* residual0,
                           const uint64_t* residual1, uint64_t* y0, uint64_t* y1, void* stream) {
  if ((residual0 == nullptr) != (residual1 == nullptr))
    return fail(HB_ERR_CONFIG, "residual0 / residual1 must both be given or both be NULL");
  // the single-party entry point validates the geometry; run its checks once for party 0
  int rc = hb_conv_check_tma(batch, channels, height, width, kh, kw, stride, pad, j_limbs, n_tile);
  if (rc) return rc;
  const uint8_t* pl[2] = {planes0, planes1};
  const uint64_t* rs[2] = {residual0, residual1};
  uint64_t* ys[2] = {y0, y1};
  const int parties[2] = {0, 1};
  return cuda_status(hb_tma_conv(2, pl, batch, channels, height, width, kh, kw, stride, pad, wlimbs, n_out, j_limbs,
                                 n_tile, parties, frac_bits, bias, rs, ys, S(stream)),
                     "hb_conv_limbs_tma_pair");
}

int hb_deal_triples(uint64_t state_lo, uint64_t state_hi, uint64_t inc_lo, uint64_t inc_hi, int kind, int width,
                    int64_t count, int64_t first, int64_t n, uint64_t* a0, uint64_t* b0, uint64_t* c0, uint64_t* a1,
                    uint64_t* b1, uint64_t* c1, void* stream) {
  if (kind != 0 && kind != 1) return fail(HB_ERR_CONFIG, "kind must be 0 (arith) or 1 (bool)");
  if (width < 1 || width > 64) return fail(HB_ERR_CONFIG, "width must be in 1..64, got %d", width);
  if (count < 0 || first < 0 || n < 0 || first + n > count) return fail(HB_ERR_CONFIG, "bad triple range");
  return cuda_status(hb_dealer_launch(state_lo, state_hi, inc_lo, inc_hi, kind, width, (unsigned long long)count,
                                      (unsigned long long)first, (unsigned long long)n, a0, b0, c0, a1, b1, c1,
                                      S(stream)),
                     "hb_deal_triples");
}

int hb_avgpool_nhwc(const uint64_t* x, int64_t batch, int height, int width, int channels, int kh, int kw, int stride,
                    uint64_t inv, int party, int frac_bits, uint64_t* out, void* stream) {
  if (kh <= 0 || kw <= 0 || stride <= 0 || kh > height || kw > width || channels <= 0)
    return fail(HB_ERR_CONFIG, "bad pool geometry");
  return cuda_status(hb_ring_avgpool_nhwc(x, batch, height, width, channels, kh, kw, stride, inv, party, frac_bits, out,
                                          S(stream)),
                     "hb_avgpool_nhwc");
}

int hb_add_shares(const uint64_t* a, const uint64_t* b, int64_t n, uint64_t* out, void* stream) {
  return cuda_status(hb_ring_add(a, b, n, out, S(stream)), "hb_add_shares");
}

}  // extern "C"
