/* hb_relu.h -- C ABI of libhbrelu.so, the B200 (sm_100a) reduced-ring secure ReLU.
 *
 * Drop-in boundary for the ringmpc hot path (reference: /root/reference/pkg/src/ringmpc).
 * Every entry point takes plain device pointers, sizes and a cudaStream_t passed as
 * `void *stream` (NULL = legacy default stream); no torch types cross this boundary.
 *
 * Status codes mirror ringmpc/errors.py exit codes (errors.py:8-47):
 *   HB_OK 0, HB_ERR_CUDA 1 (RingMpcError base), HB_ERR_CONFIG 2 (ConfigError/WindowError),
 *   HB_ERR_TRANSPORT 3 (TransportError), HB_ERR_DATA 4 (DataFormatError),
 *   HB_ERR_TRIPLES 5 (TripleExhaustedError).
 * Every check that can fail runs on the host BEFORE any kernel or exchange, so both
 * parties fail symmetrically (failure detection).
 * hb_last_error() returns a thread-local message for the last failure.
 *
 * Data layouts (all little-endian, device memory):
 *   arithmetic shares      uint64 residues on Z/2^N, one per element
 *   bool triple stream     a, b, c each packed LSB-first at w bits per element into
 *                          64-bit words (the wire layout, transport.py:33-49)
 *   arith triple stream    a, b, c each one uint64 residue per element
 *   payload (opening)      packed stream of 64-bit words, 8*ceil(count*w/64) bytes
 */
#ifndef HB_RELU_H
#define HB_RELU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_OK 0
#define HB_ERR_CUDA 1
#define HB_ERR_CONFIG 2
#define HB_ERR_TRANSPORT 3
#define HB_ERR_DATA 4
#define HB_ERR_TRIPLES 5

#define HB_TAG_CIRCUIT 0 /* meter tags, transport.py:26-30 */
#define HB_TAG_MULT 1
#define HB_TAG_B2A 2
#define HB_TAG_OTHER 3

/* One party's view of a (kind, width) triple stream, cursor-addressed like
 * TripleStore.draw (dealer.py:152-163): the op consumes elements
 * [cursor, cursor + need) and the caller advances its cursor afterwards. */
typedef struct {
  const uint64_t* a;
  const uint64_t* b;
  const uint64_t* c;
  int64_t cursor;   /* first unused element */
  int64_t capacity; /* elements in the stream */
  int32_t width;    /* ring / word width of the stream */
} hb_triples_t;

const char* hb_last_error(void);
int hb_version(void);

/* ---- cost model (protocol.py:108-110, 202-213; transport.py:70-71) ---- */
int hb_prefix_levels(int w);
int64_t hb_payload_bytes(int64_t count, int w);
/* rounds of one ReLU (drelu_only=0: L+3) or DReLU (drelu_only=1: L+2) */
int hb_relu_rounds(int k, int m, int drelu_only);
/* payload bytes of round r and its meter tag */
int64_t hb_relu_round_bytes(int ring_bits, int k, int m, int64_t n, int round);
int hb_relu_round_tag(int k, int m, int round);

/* ---- 1-GPU time-sliced party pair: the whole windowed ReLU of both parties
 * in one launch.  Replaces the two-thread run_parties(relu, relu) of
 * protocol.py:195-199 / transport.py:271-302 when both parties share a device.
 * y_p receives party p's output share (relu) or DReLU share (drelu_only). */
int hb_relu_pair(int ring_bits, int k, int m, int64_t n,
                 const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1,
                 hb_triples_t bool0, hb_triples_t bool1, hb_triples_t arith0, hb_triples_t arith1,
                 int drelu_only, void* stream);
/* Same, for the elements [first, first + count) of an n-element layer (triple segments still
 * n apart): lets a host pipeline H2D / compute / D2H chunks of one layer across streams. */
int hb_relu_pair_range(int ring_bits, int k, int m, int64_t n, int64_t first, int64_t count,
                       const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1,
                       hb_triples_t bool0, hb_triples_t bool1, hb_triples_t arith0, hb_triples_t arith1,
                       int drelu_only, void* stream);

/* Same ReLU with the shares in (pinned) HOST memory: x_p are read from and y_p written to host
 * buffers, pipelined over three internal streams -- host-to-device copies, the fused kernel on
 * element ranges, device-to-host copies -- in chunks of `chunk` elements (ramped at both ends), so
 * both PCIe directions and the kernel overlap.  scratch: 4n uint64 of device memory.  Returns when
 * y0 / y1 are complete.  Same shares, triples and rounds as hb_relu_pair. */
int hb_relu_pair_host(int ring_bits, int k, int m, int64_t n, const uint64_t* hx0, const uint64_t* hx1,
                      uint64_t* hy0, uint64_t* hy1, hb_triples_t bool0, hb_triples_t bool1,
                      hb_triples_t arith0, hb_triples_t arith1, int drelu_only, int64_t chunk,
                      uint64_t* scratch, void* stream);

/* Bind the calling host thread to CUDA device `device` (the library links its own CUDA runtime;
 * the Python package calls this with torch's current device before any other entry point). */
int hb_set_device(int device);

/* ---- one party, staged: protocol.relu / protocol.drelu (protocol.py:179-199)
 * split at its exchanges.  Call round r = 0 .. hb_relu_rounds(): round r writes
 * this party's payload of round r into `own` (hb_relu_round_bytes bytes, except
 * the last call, which writes y) after consuming the peer's payload of round
 * r-1 from `peer` (NULL for r = 0).  The caller exchanges own/peer between calls
 * (Endpoint.exchange, transport.py:129-133) under tag hb_relu_round_tag(r). */
size_t hb_relu_workspace_bytes(int k, int m, int64_t n);

/* ---- one party per GPU, openings through the peer's memory (NVLink P2P), one launch per ReLU.
 * Replaces the per-round Endpoint.exchange loop of protocol.relu / drelu (protocol.py:179-199,
 * transport.py:129-133) for two parties on two GPUs of one node: the party kernel stores each
 * round's masked opening of a tile straight into the peer's receive buffer -- the reference payload
 * bytes exactly, w-bit packed (transport.py:33-49) -- and releases a per-tile flag at system scope;
 * the peer's kernel acquires it.  Same outputs / triple consumption as hb_relu_round.
 * Z/2^64 shares (ring_bits = 64) only.
 * hb_relu_p2p_bytes: receive-buffer bytes of ONE launch (identical layout on both sides) and the
 * flag count (uint64 each, zero-initialised once).  Consecutive launches must alternate between two
 * such regions (transport.PeerLink: launch parity), since a peer may start launch k+1 while this
 * party still reads launch k's last round.  seq0 = rounds of all earlier launches on these flags
 * (hb_relu_rounds each; flags are monotonic).  The launch is cooperative: max_ctas 0 = every
 * co-resident CTA, > 0 = at most that many.  A peer that does not answer within timeout_s sets
 * *err_dev = 1 (no hang).  wire_bytes_dev (optional, one uint64 accumulated by the kernel) counts
 * the bytes stored into the peer's buffer = hb_relu_p2p_wire_bytes. */
uint64_t hb_relu_p2p_bytes(int k, int m, int64_t n, int drelu_only, int64_t* ntiles);
uint64_t hb_relu_p2p_wire_bytes(int k, int m, int64_t n, int drelu_only);
int hb_relu_p2p(int party, int ring_bits, int k, int m, int64_t n, const uint64_t* x, uint64_t* y,
                hb_triples_t bool_w, hb_triples_t arith_n, void* recv, const uint64_t* my_flags, void* peer_recv,
                uint64_t* peer_flags, uint64_t seq0, int max_ctas, double timeout_s, int* err_dev, int drelu_only,
                uint64_t* wire_bytes_dev, void* stream);
/* Both parties' party kernels in ONE launch on one device (max_ctas0 / max_ctas1 CTAs per party, 0 =
 * half the co-resident CTAs each), the openings going through each other's receive buffers exactly
 * as across two GPUs: the single-GPU harness of hb_relu_p2p (recv1 / flags1 play the peer's mapped
 * buffers for party 0 and vice versa).  sys_scope = 0: gpu-scope flags (the scope both parties
 * share on one device); 1: the system-scope protocol of hb_relu_p2p, for measurement. */
int hb_relu_p2p_pair(int ring_bits, int k, int m, int64_t n, const uint64_t* x0, const uint64_t* x1, uint64_t* y0,
                     uint64_t* y1, hb_triples_t bool0, hb_triples_t bool1, hb_triples_t arith0, hb_triples_t arith1,
                     void* recv0, void* recv1, uint64_t* flags0, uint64_t* flags1, uint64_t seq0, int max_ctas0,
                     int max_ctas1, int sys_scope, double timeout_s, int* err_dev, int drelu_only,
                     uint64_t* wire_bytes_dev, void* stream);
/* The same two launches with the link state on the DEVICE (graph-capturable): state_dev = three
 * zero-initialised uint64 per party [flag sequence, launches, CTAs done], recv / peer_recv = the base
 * of the two receive regions of region_bytes each (256-byte multiple).  The kernel reads seq0 and the
 * region parity from the state and the party's last CTA advances them, so the arguments do not change
 * from call to call and a sequence of layers can be replayed as one CUDA graph.  Replaces the same
 * reference interface as hb_relu_p2p (protocol.py:195-199 over Endpoint.exchange, transport.py:129-133). */
int hb_relu_p2p_dev(int party, int ring_bits, int k, int m, int64_t n, const uint64_t* x, uint64_t* y,
                    hb_triples_t bool_w, hb_triples_t arith_n, void* recv, const uint64_t* my_flags, void* peer_recv,
                    uint64_t* peer_flags, uint64_t* state_dev, uint64_t region_bytes, int max_ctas, double timeout_s,
                    int* err_dev, int drelu_only, uint64_t* wire_bytes_dev, void* stream);
int hb_relu_p2p_pair_dev(int ring_bits, int k, int m, int64_t n, const uint64_t* x0, const uint64_t* x1, uint64_t* y0,
                         uint64_t* y1, hb_triples_t bool0, hb_triples_t bool1, hb_triples_t arith0,
                         hb_triples_t arith1, void* recv0, void* recv1, uint64_t* flags0, uint64_t* flags1,
                         uint64_t* state0, uint64_t* state1, uint64_t region_bytes, int max_ctas0, int max_ctas1,
                         int sys_scope, double timeout_s, int* err_dev, int drelu_only, uint64_t* wire_bytes_dev,
                         void* stream);
/* CUDA IPC for the receive buffers / flags of a party on another GPU (64-byte handles); the buffers
 * are whole allocations (hb_dev_alloc, zero-filled) so a handle maps exactly them. */
int hb_dev_alloc(uint64_t bytes, void** dev_ptr);
int hb_dev_free(void* dev_ptr);
int hb_ipc_export(void* dev_ptr, uint8_t* handle64);
int hb_ipc_open(const uint8_t* handle64, void** dev_ptr);
int hb_ipc_close(void* dev_ptr);
int hb_relu_round(int party, int ring_bits, int k, int m, int64_t n, int round,
                  const uint64_t* x, uint64_t* y, hb_triples_t boolw, hb_triples_t arith,
                  void* workspace, const uint64_t* peer, uint64_t* own, int drelu_only, void* stream);

/* Same, driving the exchanges itself through a callback (the shape of
 * protocol.relu with an Endpoint): the callback must deliver the peer's payload
 * of `nbytes` bytes into `recv` (device memory) and return 0, or nonzero for a
 * transport failure.  Scratch comes from `workspace` (hb_relu_callback_workspace_bytes). */
typedef int (*hb_exchange_fn)(void* user, int tag, const uint64_t* send, uint64_t* recv, int64_t nbytes,
                              void* stream);
size_t hb_relu_callback_workspace_bytes(int ring_bits, int k, int m, int64_t n);
int hb_relu(int party, int ring_bits, int k, int m, int64_t n, const uint64_t* x, uint64_t* y,
            hb_triples_t boolw, hb_triples_t arith, void* workspace, int drelu_only,
            hb_exchange_fn exchange, void* user, void* stream);

/* ---- wire codec (transport.py:33-67) ---- */
int hb_pack(const uint64_t* values, int64_t count, int w, uint64_t* out, void* stream);
int hb_unpack(const uint64_t* packed, int64_t count, int w, uint64_t* values, void* stream);

/* ---- stage operations, one party (protocol.py:75-105): open = mask + pack the
 * payload (tmp: 2*count words of scratch); close = combine with the peer's payload.
 * kind 0 = bool (beaver_and, width-w words), kind 1 = arith (beaver_mul, Z/2^w). */
int hb_beaver_open(int kind, int w, int64_t count, const uint64_t* x, const uint64_t* y, hb_triples_t t,
                   uint64_t* tmp, uint64_t* payload, void* stream);
int hb_beaver_close(int kind, int party, int w, int64_t count, const uint64_t* x, const uint64_t* y, hb_triples_t t,
                    const uint64_t* peer_payload, uint64_t* z, void* stream);

/* elementwise helpers used to compose circuit_add / a2b / b2a_bit / drelu stage by stage */
#define HB_EW_SLICE 0     /* out = (a >> p) & mask(w)                 ring.py:69-72 */
#define HB_EW_MSB 1       /* out = (a >> (w-1)) & 1                   ring.py:75-77 */
#define HB_EW_XOR 2       /* out = (a ^ b) & mask(w) */
#define HB_EW_KS_RHS 3    /* out = [(G<<2^p)&m ; (P<<2^p)&m ^ [p0]ones]  protocol.py:130-138 */
#define HB_EW_KS_UPDATE 4 /* out = G ^ z[0:n], out2 = z[n:2n]          protocol.py:140-141 */
#define HB_EW_KS_FINISH 5 /* out = a ^ ((b << 1) & m)                 protocol.py:142-143 */
#define HB_EW_B2A_LIFT 6  /* out = (bit - 2 t) & m                    protocol.py:174-175 */
#define HB_EW_DRELU_OUT 7 /* out = [p0]1 - a                          protocol.py:192 */
#define HB_EW_OWNER 8     /* out = party == p ? a : 0                 protocol.py:153-156 */
#define HB_EW_STACK2 9    /* out = [a ; a] */
#define HB_EW_MASKW 10    /* out = a & mask(w) */
#define HB_EW_DRELU_SHARES 11 /* out = 1 - msb(((a>>p)&m) + ((b>>p)&m)), w = k - m, p = m  simulator.py:33-44 */
int hb_ewise(int op, int party, int w, int64_t count, int p, const uint64_t* a, const uint64_t* b, uint64_t* out,
             uint64_t* out2, void* stream);
/* 1 if any word > 1 (b2a_bit precondition, protocol.py:166-167); synchronises `stream` */
int hb_any_above_one(const uint64_t* a, int64_t count, int* result, void* stream);

/* ---- ring-exact linear layers on Z/2^64 shares (nn.py:198-259), SURVEY 8(f)-1 ----
 * (X W^T) mod 2^64 = sum_{i+j<=7} 256^(i+j) x_i w_j^T with x_i the 8 byte limbs of the
 * share and w_j the J balanced signed byte limbs of the encoded weight; every x_i w_j^T
 * is an exact int8 x int8 -> int32 tensor-core GEMM over A = [x_i - 128] stacked along M.
 *
 * hb_im2col_limbs: share NCHW [batch, channels, height, width] (or [batch, K] with
 *   1x1 geometry) -> out int8 [8][M][k_padded], M = batch*OH*OW, column k = c*kh*kw +
 *   ki*kw + kj (the reference im2col order, nn.py:177-195), value = limb_i - 128.
 * hb_limb_combine: products int32 [8*m][j_limbs*n_padded] (row i*m + mm, column
 *   j*n_padded + nn; colsum [j_limbs][n_padded]) -> out uint64 = local truncation by
 *   frac_bits (nn.py:198-211) of sum_{i+j<=7} (P + 128 colsum[j][nn]) << 8(i+j), plus bias[nn] on party 0
 *   (nn.py:224).  layout 0: out[mm*n + nn]; layout 1 (conv): out[(b*n + nn)*spatial + s]
 *   with mm = b*spatial + s (nn.py:242-243).
 * hb_avgpool: window sum, times `inv` = encode(1/(kh*kw)), truncation (nn.py:246-259).
 * hb_add_shares: out = a + b mod 2^64 (residual add, sharing.py:118-122). */
int hb_im2col_limbs(const uint64_t* x, int batch, int channels, int height, int width, int kh, int kw, int stride,
                    int pad, int64_t k_padded, int8_t* out, void* stream);
int hb_limb_combine(const int32_t* products, int64_t m, int64_t n, int64_t n_padded, int j_limbs,
                    const int32_t* colsum, int party, int frac_bits, const uint64_t* bias, int layout, int64_t spatial,
                    uint64_t* out, void* stream);
int hb_avgpool(const uint64_t* x, int64_t batch_channels, int height, int width, int kh, int kw, int stride,
               uint64_t inv, int party, int frac_bits, uint64_t* out, void* stream);
int hb_add_shares(const uint64_t* a, const uint64_t* b, int64_t n, uint64_t* out, void* stream);
/* hb_avgpool on NHWC shares: x [batch][height][width][channels] -> out [batch][OH][OW][channels] */
int hb_avgpool_nhwc(const uint64_t* x, int64_t batch, int height, int width, int channels, int kh, int kw, int stride,
                    uint64_t inv, int party, int frac_bits, uint64_t* out, void* stream);

/* ---- trusted dealer in HBM (dealer.py:50-83), bit-exact with gen_arith_triples /
 * gen_bool_triples: (state, inc) = the 128-bit PCG64 state of default_rng(SeedSequence(seed)) before
 * any draw (numpy bit_generator.state).  Writes triples [first, first + n) of a batch of `count`
 * (both parties' a, b, c as uint64 residues of `width` bits).  kind 0 = arith, 1 = bool. */
int hb_deal_triples(uint64_t state_lo, uint64_t state_hi, uint64_t inc_lo, uint64_t inc_hi, int kind, int width,
                    int64_t count, int64_t first, int64_t n, uint64_t* a0, uint64_t* b0, uint64_t* c0, uint64_t* a1,
                    uint64_t* b1, uint64_t* c1, void* stream);

/* Fused ring conv/linear on tcgen05 tensor cores (hand-written, sm_100a): im2col gather, byte-limb
 * split, u8 x s8 -> s32 MMAs with the 8 byte-shift accumulators in TMEM, fold mod 2^64, local
 * truncation, party-0 bias, NCHW store -- one kernel, no int32 intermediates in HBM.
 * x NCHW [batch][channels][height][width] (a linear layer is the 1x1 case [batch][K]), y NCHW
 * [batch][n_out][OH][OW]; patch index k = c*kh*kw + ki*kw + kj (nn.py:177-195).
 * wlimbs: int8 [ceil(n_out/n_tile)][k_padded/64][j_limbs][n_tile x 64 UMMA canonical K-major tile];
 * k_padded % 64 == 0, C*kh*kw <= 21900, j_limbs <= 3, n_tile in {16, 32, 64}. */
int hb_conv_limbs_tc(const uint64_t* x, int batch, int channels, int height, int width, int kh, int kw, int stride,
                     int pad, const int8_t* wlimbs, int n_out, int j_limbs, int64_t k_padded, int n_tile, int party,
                     int frac_bits, const uint64_t* bias, uint64_t* y, void* stream);

/* Simulator ReLU in the clear (simulator.py:47-54 sim_relu, the window search's inner loop):
 * encode x * 2^frac_bits (ring.py:191-199), split with r = the raw PCG64 stream whose 128-bit
 * (state, inc) the caller's numpy generator holds before the draw (share_arith, sharing.py:88-96),
 * keep x iff drelu_from_shares (simulator.py:33-44) on [m, k) says so; out = x * keep in float64,
 * bit-identical to the reference.  *err_dev = 1 if an input leaves the signed ring (EncodeRangeError). */
int hb_sim_relu(const double* x, int64_t n, int frac_bits, int ring_bits, int k, int m, uint64_t state_lo,
                uint64_t state_hi, uint64_t inc_lo, uint64_t inc_hi, double* out, int* err_dev, void* stream);

/* Byte-limb planes of an NCHW share for the TMA conv, channel-blocked NHWC:
 * planes[i][c/64][b][h][w][c%64] = byte i of x[b][c][h][w] (uint8; channels % 64 == 0;
 * 8 planes of batch*height*width*channels bytes).
 * Replaces the limb split inside the reference's uint64 matmul (nn.py:222). */
int hb_limbs_nhwc(const uint64_t* x, int batch, int channels, int height, int width, uint8_t* planes, void* stream);

/* Small-K convs (channels*kh*kw <= 64, e.g. a 3-channel stem): the byte-limb planes of the im2col
 * patches, [limb][1][batch][OH][OW][64] with patch index c*kh*kw + ki*kw + kj (nn.py:177-195) zero-
 * padded to 64 -- the conv then runs through hb_conv_limbs_tma as a 1x1 conv over 64 channels. */
int hb_im2col_planes(const uint64_t* x, int batch, int channels, int height, int width, int kh, int kw, int stride,
                     int pad, uint8_t* planes, void* stream);

/* Ring conv/linear (nn.py:214-243 conv2d_forward / linear_forward + truncate_local nn.py:198-211) as a
 * TMA-fed tcgen05 implicit GEMM over the limb planes of hb_limbs_nhwc: same result as
 * hb_conv_limbs_tc.  wlimbs: int8 [ceil(n_out/n_tile)][kh*kw*channels/64][j_limbs][n_tile x 64
 * SWIZZLE_64B K-major tile], K order (ki, kj, c), n_tile in {16, 32, 64, 128} (128: two shift
 * passes).  channels % 64 == 0; the output (OH, OW) must tile
 * into 128-pixel (batch, oh, ow) boxes (OW a divisor or multiple of 128, ...).  residual: optional NCHW
 * share of y's shape added after truncation and bias (a ResNet block's add_shares, sharing.py:118-122). */
int hb_conv_limbs_tma(const uint8_t* planes, int batch, int channels, int height, int width, int kh, int kw,
                      int stride, int pad, const int8_t* wlimbs, int n_out, int j_limbs, int n_tile, int party,
                      int frac_bits, const uint64_t* bias, const uint64_t* residual, uint64_t* y, void* stream);

/* Both parties' convs of one layer in ONE launch (same geometry and weights; the pair of a 1-GPU
 * time-sliced forward): party 0 on planes0 -> y0 (+ bias), party 1 on planes1 -> y1, each with its
 * own truncation and optional residual.  Same results as two hb_conv_limbs_tma calls. */
int hb_conv_limbs_tma_pair(const uint8_t* planes0, const uint8_t* planes1, int batch, int channels, int height,
                           int width, int kh, int kw, int stride, int pad, const int8_t* wlimbs, int n_out,
                           int j_limbs, int n_tile, int frac_bits, const uint64_t* bias, const uint64_t* residual0,
                           const uint64_t* residual1, uint64_t* y0, uint64_t* y1, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HB_RELU_H */
