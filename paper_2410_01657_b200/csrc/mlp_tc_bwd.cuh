// Tensor-core processor-MLP backward (sm_100a, tcgen05 kind::tf32, H = 64).
//
// Same math as mlp_backward_kernel (mlp_simt.cuh) / mlp_backward_rows
// (nn.cpp:204-285): recompute the forward pass of a 128-row tile, then walk the
// linears in reverse computing the input adjoints (dX = d W^T) and the weight
// gradients (dW += h^T d), all products as 3xTF32 on the tensor cores.
//
// Per CTA (persistent, one per SM), two 128-row tile slots ping-pong as in
// the forward kernel. TMEM (512 columns):
//   slot s: [A_hi 64 | A_lo 64 | D 64]  (s = 0, 1)      cols [192 s, 192 s + 192)
//   dW accumulator 128 x 128                               cols [384, 512)
// Per 8-row K-step the dW product is one SS MMA (kDwN128):
//   [h_hi^T ; h_lo^T] (128 x 8) x [d_hi | d_lo] (8 x 128),
// so lanes 0-63 collect hh | hl and lanes 64-127 lh | ll in the two column
// halves (the tiny ll term is kept: free and slightly more accurate). Both operands are staged per warp
// (32 rows) in shared memory as MN-major SWIZZLE_128B_BASE32B tiles (the layout
// tf32 MN-major operands require), through a ring of NSTAGE buffers consumed
// in a fixed warp order (deterministic accumulation) by a dW issuer warp that
// runs separately from the dX issuer. With two accumulators, job j drains
// while job j + 1 accumulates: the epilogue warps drain job j - 2 before
// staging job j, each warp its TMEM lane quarter and one column half, adding
// hh + hl into a per-CTA fp32 partial and lh + ll into a second one (one
// owning thread per element: deterministic); bias gradients come from
// fixed-order per-warp column sums.
// Forward-recompute intermediates of the reverse pass (normed t_j, inv_std_j)
// go to a per-CTA global scratch; the residual stream is rebuilt backwards as
// h_{j-1} = h_j - ELU(t_j). The residual term of d_prev = d_u W^T + d_h is
// folded into the MMA by pre-loading D with d_h.
// Warp roles: 0-7 epilogue (slot = warp / 4), 8 dX issuer, 9 dW issuer,
// 10 weight loader, 11 idle.
#pragma once

#include "mlp_tc.cuh"

namespace hgnn_b200 {

struct TcBwdCfg {
  static constexpr int H = 64;
  static constexpr int CHUNK_FLOATS = 2 * H * H;
  static constexpr int CHUNK_BYTES = CHUNK_FLOATS * 4;  // 32 KB
  static constexpr uint32_t LBO = (2 * H / 8) * 128;   // K-major weight chunks
  static constexpr uint32_t SBO = 128;
  static constexpr uint32_t LO_OFF = (H / 8) * 128;
#ifndef HGNN_BWD_WSTAGES
#define HGNN_BWD_WSTAGES 2
#endif
  static constexpr int WSTAGES = HGNN_BWD_WSTAGES;
#ifndef HGNN_BWD_NSTAGE
#define HGNN_BWD_NSTAGE 4
#endif
  static constexpr int NSTAGE = HGNN_BWD_NSTAGE;       // dW staging buffers
  static constexpr int STAGE_BYTES = 32 * 1024;        // A (16 KB) + B (16 KB), 32 rows
  // MN-major SWIZZLE_128B_BASE32B staging: atoms of 4 K-rows x 128 B of MN,
  // 32-byte granule g of atom row r stored at granule g ^ r.
  static constexpr uint32_t ST_LBO = 512;              // MN-atom stride (32 tf32 of MN)
  static constexpr uint32_t ST_SBO = 2048;             // K-atom stride (4 rows): 128 MN = 4 atoms
  static constexpr int SLOT_COLS = 3 * H;
  static constexpr int DW_COL = 2 * SLOT_COLS;         // 384: two 64-column dW accumulators (job parity)
  static constexpr int THREADS = 384;  // 2 epilogue warpgroups + 1 control warpgroup
  static constexpr size_t OFF_STAGE = (size_t)WSTAGES * CHUNK_BYTES;
  static constexpr size_t OFF_BARS = OFF_STAGE + (size_t)NSTAGE * STAGE_BYTES;
  static constexpr size_t OFF_DBP = OFF_BARS + 256;               // db partials [4][8][64]
  static constexpr size_t OFF_BIAS = OFF_DBP + 4 * 8 * 64 * 4;    // biases (k+2) x 64
  static constexpr size_t SMEM = OFF_BIAS + 18 * 64 * 4 + 1024;
};

constexpr bool kDiscardScratch = true;  // see the backward walk
// dW as ONE N = 128 MMA per 8-row K-step: [h_hi ; h_lo] (M = 128) x [d_hi | d_lo]
// (N = 128) into a single 128-column accumulator (hh hl / lh ll quadrants),
// instead of two N = 64 MMAs into two double-buffered 64-column ones: the A
// operand is read from shared memory once instead of twice (the SS dW MMAs are
// shared-memory-bandwidth bound), half the MMA issues. The accumulator of job j
// is drained when the warps start staging job j + 1.
#ifndef HGNN_DW_N128
#define HGNN_DW_N128 1
#endif
constexpr bool kDwN128 = HGNN_DW_N128;
// Packed fp32 (f32x2) variants of the backward epilogue pieces. Measured at C3
// (edge backward per layer, 3 runs): all scalar 67.5 ms, all packed 69.3 ms,
// single pieces 67.7-72.9 ms: the backward epilogue is not FP-issue bound,
// so the scalar code (shorter, fewer register pair moves) is the default.
#ifndef HGNN_PARK_AUX
#define HGNN_PARK_AUX 0  // 1: loader / dW-issuer waits park (measured neutral at C3: 67.3 vs 66.8 ms)
#endif
#ifndef HGNN_PK_LNB
#define HGNN_PK_LNB 0
#endif
#ifndef HGNN_PK_STAGE
#define HGNN_PK_STAGE 0
#endif
#ifndef HGNN_PK_TMEM
#define HGNN_PK_TMEM 0
#endif
#ifndef HGNN_GATHER_HINT
#define HGNN_GATHER_HINT 1  // edge modes: recompute gathers evict_last, the dW0 re-gathers evict_first (C3 edge bwd 53.2 -> 52.35 ms)
#endif
#ifndef HGNN_SCRATCH_KEEP
#define HGNN_SCRATCH_KEEP 1  // recompute scratch stored evict_last (C3: step 336 -> 332.5 ms; round 1 measured it neutral)
#endif
#ifndef HGNN_LNB_KEEP_T
#define HGNN_LNB_KEEP_T 0  // 1: the LayerNorm-adjoint's second pass reads t_l from registers, not L1 (A/B knob)
#endif
#ifndef HGNN_BWD_PREFETCH
#define HGNN_BWD_PREFETCH 0  // 1: input-segment gathers one step ahead (behind the MMA / dX wait): measured neutral at C3 (edge 67.4 ms, node 9.85 vs 9.5 ms)
#endif
#ifndef HGNN_EXP
#define HGNN_EXP 0  // timing experiments only (scripts/build_exp.py): bits drop work, results are wrong
#endif
constexpr int kExp = HGNN_EXP;

struct TcBwdArgs {
  int64_t n_rows;
  const int32_t* src;
  const int32_t* dst;
  const float* x;
  const float* e_in;
  const float* a;
  // output adjoint
  const float* d_out;    // node mode: dx rows
  const float* inv_deg;  // edge mode
  const float* d_a;      // edge mode
  const float* de_in;    // edge mode: adjoint of the edge output (nullptr: zero, the last layer)
  float* de_io;          // edge mode: adjoint of the edge input out (may alias de_in or e_in row by row)
  float* d_src;          // edge mode outputs
  float* d_dst;
  float* d_a_out;        // node mode outputs
  float* d_x_out;
  const float* proj;     // kEdgeFact: rows x 2H node projections [P_s | P_d] (recompute input)
  float* dy_out;         // kEdgeFact: adjoint of the input linear's output (N_e x H), for the node-level sums
  const float* chunks;   // 2 nseg + 2k + 1 chunks in MMA order
  const float* params;   // fp32 for_each layout (biases)
  float* grad_partial;   // [gridDim.x][2][n_par]: (hh + hl, db) and lh partials
  float* scratch;        // [gridDim.x][2][k][16][128] float4 + [gridDim.x][2][k][128] inv_std
  int k;
  unsigned long long* prof;  // optional: wait-cycle counters (see kProf*)
  // kEncoder: in_dim input features (<= 8, zero-padded to one segment; the
  // padded rows of dW0 are not written, no input adjoint is stored), d_out =
  // adjoint of the pre-LayerNorm output (enc_out_backward_kernel), n_par =
  // stride of the gradient partials (the encoder's full parameter count)
  int in_dim;
  int64_t n_par;
  // kDecoder: x = decoder input rows (H wide), d_out = n_rows x out_dim output
  // adjoint (zero-padded to H), d_x_out = the MLP part of the input adjoint;
  // W_{k+1} is H x out_dim in the gradient layout
  int out_dim;
};

// Optional instrumentation of the MMA issuer (cycles, summed over CTAs).
enum { kProfTotal = 0, kProfW = 1, kProfA = 2, kProfSt = 3, kProfDwE = 4, kProfFwd = 5, kProfDw = 6, kProfMma = 7,
       kProfEpiTotal = 8, kProfEpiRecompute = 9, kProfEpiFlush = 10, kProfEpiStage = 11, kProfEpiDb = 12,
       kProfEpiWaitDx = 13, kProfEpiLnBwd = 14, kProfEpiInput = 15, kProfCount = 16 };

// HL-wide row (HL = 32: the zero-padded H = 32 instance) into v[0, 64)
template <int HL>
__device__ __forceinline__ void bwd_row(const float* p, float (&v)[64]) {
#pragma unroll
  for (int q = 0; q < HL / 8; ++q) ptx::ldg256(p + 8 * q, v + 8 * q);
#pragma unroll
  for (int j = HL; j < 64; ++j) v[j] = 0.f;
}

template <int MODE, int HL = 64>
__device__ __forceinline__ void bwd_gather(const TcBwdArgs& a, int64_t row, bool valid, int c, float (&v)[64],
                                           uint64_t pol = 0) {
  if (HGNN_EXP & 16) valid = false;
  if (HL != 64) {  // kEdgeInput / kNodeInput rows of width HL, zero-padded
    if (!valid) {
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = 0.f;
      return;
    }
    const float* seg;
    if (MODE == kEdgeInput)
      seg = c == 0 ? a.x + (int64_t)__ldg(a.src + row) * HL
                   : (c == 1 ? a.x + (int64_t)__ldg(a.dst + row) * HL : a.e_in + row * HL);
    else
      seg = c == 0 ? a.a + row * HL : a.x + row * HL;
    bwd_row<HL>(seg, v);
    return;
  }
  TcFwdArgs f{};
  f.src = a.src;
  f.dst = a.dst;
  f.x = a.x;
  f.e_in = a.e_in;
  f.a = a.a;
  f.in_dim = a.in_dim;
  f.out_dim = a.out_dim;
  // edge modes: the rows are gathered twice (recompute, dW0 operand); node rows are contiguous streams
  constexpr bool hint = HGNN_GATHER_HINT && (MODE == kEdgeInput || MODE == kEdgeFact);
  tc_gather<64, MODE>(f, row, valid, c, v, hint ? pol : 0);
}
__device__ __forceinline__ void bwd_gather_proj(const TcBwdArgs& a, int64_t row, bool valid, float (&v)[64]) {
  TcFwdArgs f{};
  f.src = a.src;
  f.dst = a.dst;
  f.proj = a.proj;
  tc_gather_proj<64>(f, row, valid, v);
}

// A <- [hi | lo] split of v, 16 columns at a time (low register pressure).
__device__ __forceinline__ void bwd_store_a(uint32_t t_hi, uint32_t t_lo, const float (&v)[64]) {
#pragma unroll
  for (int c = 0; c < 64; c += 16) {
    float hi[16], lo[16];
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      hi[j] = ptx::tf32_hi(v[c + j]);
      hi[j + 1] = ptx::tf32_hi(v[c + j + 1]);
      if (HGNN_PK_TMEM) {
        f2_put(lo + j, f2_add(f2_pair(v + c + j), make_float2(-hi[j], -hi[j + 1])));
      } else {
        lo[j] = v[c + j] - hi[j];
        lo[j + 1] = v[c + j + 1] - hi[j + 1];
      }
    }
    ptx::tmem_st16(t_hi + c, hi);
    ptx::tmem_st16(t_lo + c, lo);
  }
}

// y = D (+ b): four 16-column TMEM loads in flight, one wait.
__device__ __forceinline__ void bwd_load_d(uint32_t t_d, const float* b, float (&y)[64]) {
#pragma unroll
  for (int c = 0; c < 64; c += 16) ptx::tmem_ld16(t_d + c, *reinterpret_cast<float(*)[16]>(y + c));
  ptx::tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < 64; c += 16) {
    float p[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) p[j] = y[c + j];
    if (b && HGNN_PK_TMEM) {
#pragma unroll
      for (int j = 0; j < 16; j += 2) f2_put(y + c + j, f2_add(f2_pair(p + j), f2_pair(b + c + j)));
    } else if (b) {
#pragma unroll
      for (int j = 0; j < 16; ++j) y[c + j] = p[j] + b[c + j];
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) y[c + j] = p[j];
    }
  }
}

__device__ __forceinline__ void bwd_store_raw(uint32_t t_d, const float (&y)[64]) {
#pragma unroll
  for (int c = 0; c < 64; c += 16) {
    float p[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) p[j] = y[c + j];
    ptx::tmem_st16(t_d + c, p);
  }
}

// Producer side of the staging ring: use m = gi / NSTAGE of buffer gi % NSTAGE
// waits until use m-1 was consumed. Completions of even / odd uses land on two
// barrier sets, so the parity wait cannot alias even if use m-2 is still queued.
__device__ __forceinline__ void stage_acquire(uint64_t* st_empty, int64_t gi) {
  const int64_t m = gi / TcBwdCfg::NSTAGE;
  if (m == 0) return;
  const int buf = (int)(gi % TcBwdCfg::NSTAGE);
  const int64_t prev = m - 1;
  ptx::mbar_wait(&st_empty[(prev & 1) * TcBwdCfg::NSTAGE + buf], (uint32_t)((prev >> 1) & 1));
}

// Byte offset of the 16-byte group (mn = 4 mn4 .. 4 mn4 + 3, row) inside a
// 16 KB MN-major SWIZZLE_128B_BASE32B staging operand (128 MN x 32 rows).
// (MN-major tf32 operands must use this swizzle; SWIZZLE_NONE reads zeros.)
__device__ __forceinline__ uint32_t st_off(int mn4, int row) {
  const int mn = 4 * mn4, a = mn / 32, g = (mn % 32) / 8, h = (mn % 8) / 4, r = row % 4;
  return (uint32_t)(row / 4) * TcBwdCfg::ST_SBO + (uint32_t)a * TcBwdCfg::ST_LBO + (uint32_t)r * 128 +
         (uint32_t)((g ^ r) * 32) + (uint32_t)h * 16;
}

// Writes [v_hi | v_lo] (128 MN entries) of this lane's row into a staging operand.
// Bank-conflict-free: a 16-byte store is served per quarter warp (8 lanes);
// lanes r and r + 4 share r % 4, i.e. the same swizzled 32-byte granule, so
// lanes with bit 2 of the row set store the two 16-byte halves of each
// granule in the opposite order (chunk pair (2p, 2p+1) swapped).
__device__ __forceinline__ void stage_row(uint8_t* base, int row, const float (&v)[64]) {
  const bool sw = (row >> 2) & 1;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int qa = 2 * p + k, qb = 2 * p + (k ^ 1);
      float4 x;
      x.x = sw ? v[4 * qb] : v[4 * qa];
      x.y = sw ? v[4 * qb + 1] : v[4 * qa + 1];
      x.z = sw ? v[4 * qb + 2] : v[4 * qa + 2];
      x.w = sw ? v[4 * qb + 3] : v[4 * qa + 3];
      const int q = sw ? qb : qa;
      float4 hi, lo;
      hi.x = ptx::tf32_hi_stage(x.x);
      hi.y = ptx::tf32_hi_stage(x.y);
      hi.z = ptx::tf32_hi_stage(x.z);
      hi.w = ptx::tf32_hi_stage(x.w);
      if (HGNN_PK_STAGE) {
        const float2 l0 = f2_add(make_float2(x.x, x.y), make_float2(-hi.x, -hi.y));
        const float2 l1 = f2_add(make_float2(x.z, x.w), make_float2(-hi.z, -hi.w));
        lo = make_float4(l0.x, l0.y, l1.x, l1.y);
      } else {
        lo = make_float4(x.x - hi.x, x.y - hi.y, x.z - hi.z, x.w - hi.w);
      }
      *reinterpret_cast<float4*>(base + st_off(q, row)) = hi;
      *reinterpret_cast<float4*>(base + st_off(16 + q, row)) = lo;
    }
  }
}

// Column sums of a warp's 32 x 64 tile (one row per lane), transpose-reduce:
// lane L ends with the sums of columns 2L and 2L+1, fixed order.
__device__ __forceinline__ float2 warp_colsum64(const float (&v)[64]) {
  const int lane = threadIdx.x & 31;
  float a[32];
  {
    const bool up = lane & 16;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float send = up ? v[j] : v[32 + j];
      const float keep = up ? v[32 + j] : v[j];
      a[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
#pragma unroll
  for (int w = 32, bit = 8; w >= 4; w /= 2, bit /= 2) {
    const bool up = lane & bit;
#pragma unroll
    for (int j = 0; j < w / 2; ++j) {
      const float send = up ? a[j] : a[w / 2 + j];
      const float keep = up ? a[w / 2 + j] : a[j];
      a[j] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
    }
  }
  // lane bits (16,8,4,2,1) selected halves 32,16,8,4,2 -> columns colsum_base(lane) + {0, 1}
  return make_float2(a[0], a[1]);
}

// Parameter-free LayerNorm over the first HL of 64 values (kernels.cpp:81-94);
// the padding columns [HL, 64) become 0. Returns inv_std.
template <int HL>
__device__ __forceinline__ float ln0_pad(float (&v)[64]) {
  if (HL == 64) return ln0_tree<64>(v);
  float m[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < HL; ++j) m[j % 4] += v[j];
  const float mean = ((m[0] + m[1]) + (m[2] + m[3])) * (1.0f / HL);
  float q[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < HL; ++j) {
    const float d = v[j] - mean;
    q[j % 4] = fmaf(d, d, q[j % 4]);
  }
  const float inv_std = ptx::rsqrt_fast(((q[0] + q[1]) + (q[2] + q[3])) * (1.0f / HL) + 1e-12f);
#pragma unroll
  for (int j = 0; j < 64; ++j) v[j] = j < HL ? (v[j] - mean) * inv_std : 0.f;
  return inv_std;
}

__device__ __forceinline__ int colsum_base(int lane) {
  return 32 * ((lane >> 4) & 1) + 16 * ((lane >> 3) & 1) + 8 * ((lane >> 2) & 1) + 4 * ((lane >> 1) & 1) +
         2 * (lane & 1);
}

// HL: logical hidden width. 64, or 32 for the H = 32 processor MLPs
// (kEdgeInput / kNodeInput) run zero-padded to 64: padded weight chunks,
// rows of width HL in HBM, LayerNorms over the first HL columns, padding
// columns forced to 0, gradients written in the HL-wide parameter layout.
template <int MODE, bool PROF, int HL = 64>
__global__ void __launch_bounds__(TcBwdCfg::THREADS, 1) mlp_tc_backward_kernel(TcBwdArgs a) {
  using Cfg = TcBwdCfg;
  constexpr int H = Cfg::H;
  static_assert(HL == 64 || (HL == 32 && (MODE == kEdgeInput || MODE == kNodeInput)), "padded width: 3-segment MLPs");
  constexpr bool FACT = MODE == kEdgeFact;
  constexpr bool ENC = MODE == kEncoder;
  constexpr bool DEC = MODE == kDecoder;
  constexpr bool EDGE = MODE != kNodeInput && !ENC && !DEC;
  constexpr int nseg = MODE == kEdgeInput ? 3 : (MODE == kNodeInput ? 2 : 1);
  const int in_dim = ENC ? a.in_dim : (DEC ? H : (MODE == kNodeInput ? 2 : 3) * HL);  // parameter layout
  constexpr int seg0 = FACT ? 2 : 0;                         // W0 row block of the first input segment
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* wring = reinterpret_cast<float*>(smem);
  uint8_t* stage = smem + Cfg::OFF_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BARS);
  uint64_t* w_full = bars;                        // [WSTAGES]
  uint64_t* w_empty = w_full + Cfg::WSTAGES;      // [WSTAGES]
  uint64_t* a_full = w_empty + Cfg::WSTAGES;      // [2]
  uint64_t* a_empty = a_full + 2;                 // [2]
  uint64_t* d_full = a_empty + 2;                 // [2]
  uint64_t* st_full = d_full + 2;                 // [NSTAGE]
  uint64_t* st_empty = st_full + Cfg::NSTAGE;     // [2][NSTAGE]: split by use parity so a producer
                                                  // running a whole job ahead cannot alias a phase
  uint64_t* dw_full = st_empty + 2 * Cfg::NSTAGE; // [2] per accumulator
  uint64_t* dw_empty = dw_full + 2;               // [2], count 8 (epilogue warps)
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(dw_empty + 2);
  float* dbp = reinterpret_cast<float*>(smem + Cfg::OFF_DBP);
  float* sbias = reinterpret_cast<float*>(smem + Cfg::OFF_BIAS);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int K = a.k;
  const int n_w = 2 * nseg + 2 * K + 1;     // weight chunks per pair
  const int n_dw = K + 1 + nseg;            // dW jobs per pair
  const int64_t n_tiles = (a.n_rows + 127) / 128;
  const int64_t n_pairs = (n_tiles + 1) / 2;
  const int64_t n_par = (ENC || DEC) ? a.n_par : mlp_param_count(in_dim, HL, K);

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::WSTAGES; ++s) {
      ptx::mbar_init(&w_full[s], 1);
      ptx::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&a_full[s], 4);
      ptx::mbar_init(&a_empty[s], 1);
      ptx::mbar_init(&d_full[s], 1);
    }
    for (int s = 0; s < Cfg::NSTAGE; ++s) {
      ptx::mbar_init(&st_full[s], 1);
      ptx::mbar_init(&st_empty[s], 1);
      ptx::mbar_init(&st_empty[Cfg::NSTAGE + s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&dw_full[s], 1);
      ptx::mbar_init(&dw_empty[s], 8);
    }
    ptx::fence_mbarrier_init();
  }
  // biases of the recomputed linears 0..K (the output bias has no backward use)
  for (int i = threadIdx.x; i < (K + 1) * H; i += blockDim.x)
    sbias[i] = i % H < HL ? __ldg(a.params + mlp_b_offset(i / H, in_dim, HL) + (i % H)) : 0.f;
  if (warp == 8) ptx::tmem_alloc<512>(tmem_base_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_base_slot;

  // Register budget per warpgroup: the CTA pool is fixed at launch (384 x 168);
  // setmaxnreg moves registers from the control warpgroup to the epilogue.
  static_assert(256 * 224 + 128 * 56 <= Cfg::THREADS * 168, "setmaxnreg exceeds the CTA register pool");
  if (warp < 8) ptx::regs_inc<224>();
  else ptx::regs_dec<56>();

  if (warp < 8) {
    // ================================================================ epilogue
    const int g = warp / 4;
    const int wq = warp % 4;
    const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
    const uint32_t t_ahi = tmem + g * Cfg::SLOT_COLS + lane_off;
    const uint32_t t_alo = t_ahi + H;
    const uint32_t t_d = t_ahi + 2 * H;
    const uint32_t t_dw = tmem + Cfg::DW_COL + lane_off;
    float4* scr = reinterpret_cast<float4*>(a.scratch) + ((int64_t)blockIdx.x * 2 + g) * K * 16 * 128;
    float* scr_inv = a.scratch + (int64_t)gridDim.x * 2 * K * 16 * 128 * 4 + ((int64_t)blockIdx.x * 2 + g) * K * 128;
    float* gpart0 = a.grad_partial + (int64_t)blockIdx.x * 2 * n_par;  // hh + hl, db
    float* gpart1 = gpart0 + n_par;                                    // lh
    const int trow = 32 * wq + lane;  // row inside the tile
    const uint64_t keep = ptx::policy_evict_last();   // scratch, gradient partials
    const uint64_t once = ptx::policy_evict_first();  // single-use streams
    uint32_t pe = 0, pd = 0;
    int64_t job = 0;                  // global dW job counter (all pairs)
    unsigned long long pf[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // epilogue cycle counters (PROF)
    const long long pf_t0 = PROF ? clock64() : 0;

    // Drain dW job jf from accumulator jf & 1 (two 64-column accumulators in
    // TMEM, so job jf + 1 accumulates while jf drains): this warp reads its
    // lane quarter, output columns [32 g, 32 g + 32). Lanes < 64 hold
    // (h_hi row i) x (d_hi + d_lo) = hh + hl; lanes >= 64 hold
    // (h_lo row i - 64) x (d_hi + d_lo) = lh + ll.
    auto flush = [&](int64_t jf) {
      const long long tf0 = PROF ? clock64() : 0;
      const int jj = (int)(jf % n_dw);
      const int lin = jj <= K ? K + 1 - jj : 0;
      const int rowbase = jj <= K ? 0 : (jj - K - 1 + seg0) * HL;
      const bool with_db = jj <= K + 1;
      const int acc = kDwN128 ? 0 : (int)(jf & 1);
      ptx::mbar_wait(&dw_full[acc], kDwN128 ? (uint32_t)(jf & 1) : (uint32_t)((jf >> 1) & 1));
      ptx::tc_fence_after();
      const int c0 = 32 * g;
      float* gw = wq < 2 ? gpart0 + mlp_w_offset(lin, in_dim, HL) + (int64_t)(rowbase + trow) * HL + c0
                         : gpart1 + mlp_w_offset(lin, in_dim, HL) + (int64_t)(rowbase + trow - 64) * HL + c0;
      // kEncoder: rows >= in_dim of dW0 belong to the zero padding; kDecoder:
      // dW_{k+1} is H x out_dim (columns >= out_dim are padding)
      const bool w_ok = (!ENC || lin > 0 || (wq < 2 ? trow : trow - 64) < in_dim) && !(DEC && lin == K + 1) &&
                        (HL == 64 || ((wq < 2 ? trow : trow - 64) < HL && c0 < HL));
      float p0[16], p1[16];
      if (kDwN128) {  // columns c and 64 + c: (row block) x d_hi and x d_lo
        float q0[16], q1[16];
        ptx::tmem_ld16(t_dw + c0, p0);
        ptx::tmem_ld16(t_dw + c0 + 16, p1);
        ptx::tmem_ld16(t_dw + 64 + c0, q0);
        ptx::tmem_ld16(t_dw + 64 + c0 + 16, q1);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          p0[j] += q0[j];
          p1[j] += q1[j];
        }
      } else {
        ptx::tmem_ld16(t_dw + 64 * acc + c0, p0);
        ptx::tmem_ld16(t_dw + 64 * acc + c0 + 16, p1);
      }
      float dbs = 0.f;
      if (with_db && warp < 2) {  // bias gradient: fixed-order sum of the 8 warp partials
        const float* db = dbp + (jf % 4) * 8 * 64 + trow;
#pragma unroll
        for (int w = 0; w < 8; ++w) dbs += db[w * 64];
      }
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&dw_empty[acc]);  // this warp's part is read (and its db partials)
      // Fire-and-forget vector reductions into this CTA's partial: every
      // element has a single owning thread, so the adds land in program order
      // (deterministic) and no load latency is exposed.
      if (w_ok) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          ptx::red_add4_hint(gw + 4 * j, p0[4 * j], p0[4 * j + 1], p0[4 * j + 2], p0[4 * j + 3], keep);
          ptx::red_add4_hint(gw + 16 + 4 * j, p1[4 * j], p1[4 * j + 1], p1[4 * j + 2], p1[4 * j + 3], keep);
        }
      }
      if (DEC && lin == K + 1) {
        const int64_t wk = mlp_w_offset(K + 1, H, H);
        float* gd = (wq < 2 ? gpart0 + wk + (int64_t)trow * a.out_dim : gpart1 + wk + (int64_t)(trow - 64) * a.out_dim);
        if (g == 0) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < a.out_dim) asm volatile("red.global.add.f32 [%0], %1;" ::"l"(gd + j), "f"(p0[j]) : "memory");
        }
        if (warp == 0 && trow < a.out_dim)
          asm volatile("red.global.add.f32 [%0], %1;" ::"l"(gpart0 + wk + H * a.out_dim + trow), "f"(dbs) : "memory");
      } else if (with_db && warp < 2 && trow < HL) {
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(gpart0 + mlp_b_offset(lin, in_dim, HL) + trow), "f"(dbs)
                     : "memory");
      }
      if (PROF) pf[2] += (unsigned long long)(clock64() - tf0);
    };
    // Job j - 2 shares this job's accumulator and must be drained before the
    // dW MMAs of job j (which release this job's staging ring slots) can run.
    auto stage_chunk = [&](const float (&hin)[H], const float (&d)[H]) {
      if (kExp & 1) return;
      if (kDwN128 ? job >= 1 : job >= 2) flush(kDwN128 ? job - 1 : job - 2);
      const long long ts0 = PROF ? clock64() : 0;
      const int64_t gi = job * 8 + warp;  // staging chunk counter
      stage_acquire(st_empty, gi);
      uint8_t* sb = stage + (size_t)(gi % Cfg::NSTAGE) * Cfg::STAGE_BYTES;
      stage_row(sb, lane, hin);
      stage_row(sb + 16384, lane, d);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&st_full[gi % Cfg::NSTAGE]);
      if (PROF) pf[3] += (unsigned long long)(clock64() - ts0);
    };
    auto write_db = [&](const float (&d)[H]) {
      if (kExp & 4) return;
      const long long t0 = PROF ? clock64() : 0;
      const float2 cs = warp_colsum64(d);
      float* dst = dbp + ((job % 4) * 8 + warp) * 64 + colsum_base(lane);
      dst[0] = cs.x;
      dst[1] = cs.y;
      if (PROF) pf[4] += (unsigned long long)(clock64() - t0);
    };
    auto wait_dx = [&]() {
      const long long t0 = PROF ? clock64() : 0;
      ptx::mbar_wait(&d_full[g], pd);
      pd ^= 1;
      ptx::tc_fence_after();
      if (PROF) pf[5] += (unsigned long long)(clock64() - t0);
    };

    float h[H];
    bool h_ready = false;  // h holds this tile's input segment 0 (gathered during the previous tile)
    for (int64_t pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
      const int64_t row = (2 * pair + g) * 128 + trow;
      const bool valid = row < a.n_rows;
      const long long tr0 = PROF ? clock64() : 0;
      // ---------------------------------------------- forward recompute
      // (segment c + 1 is gathered while the MMA of segment c runs)
      if (!HGNN_BWD_PREFETCH || !h_ready) bwd_gather<MODE, HL>(a, row, valid, 0, h, keep);
#pragma unroll 1
      for (int c = 0; c < nseg; ++c) {
        if (c > 0) {
          ptx::mbar_wait(&a_empty[g], pe);
          pe ^= 1;
          ptx::tc_fence_after();
          if (!HGNN_BWD_PREFETCH) bwd_gather<MODE, HL>(a, row, valid, c, h, keep);
        }
        bwd_store_a(t_ahi, t_alo, h);
        tc_signal(&a_full[g]);
        if (HGNN_BWD_PREFETCH && c + 1 < nseg) bwd_gather<MODE, HL>(a, row, valid, c + 1, h);
      }
      if (FACT) bwd_gather_proj(a, row, valid, h);  // P_s[src] + P_d[dst], during the e W0_e MMA
      ptx::mbar_wait(&d_full[g], pd);
      pd ^= 1;
      ptx::tc_fence_after();
      if (FACT) {
        float u[H];
        bwd_load_d(t_d, sbias, u);
#pragma unroll
        for (int j = 0; j < H; ++j) h[j] += u[j];  // (D + b0) + proj, the forward's order
      } else {
        bwd_load_d(t_d, sbias, h);
      }
      for (int l = 1; l <= K; ++l) {
        bwd_store_a(t_ahi, t_alo, h);
        tc_signal(&a_full[g]);
        ptx::mbar_wait(&d_full[g], pd);
        pd ^= 1;
        ptx::tc_fence_after();
        float u[H];
        bwd_load_d(t_d, sbias + l * H, u);
        const float inv_std = (kExp & 8) ? 1.0f : ln0_pad<HL>(u);
        float4* st = scr + (int64_t)(l - 1) * 16 * 128 + trow;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float4 tq = make_float4(u[4 * q], u[4 * q + 1], u[4 * q + 2], u[4 * q + 3]);
          if (HGNN_SCRATCH_KEEP) ptx::st_hint(st + q * 128, tq, keep);  // A/B knob: evict_last scratch lines
          else st[q * 128] = tq;
        }
        scr_inv[(l - 1) * 128 + trow] = inv_std;
        add_elu<H>(h, u);
      }
      if (PROF) pf[1] += (unsigned long long)(clock64() - tr0);
      // ---------------------------------------------- backward
      float dh[H];
      if (valid) {
        if (EDGE) {  // d_y = de + inv_d * d_a[dst] (model.cpp:354-360)
          const float s = __ldg(a.inv_deg + row);
          const float* da = a.d_a + (int64_t)__ldg(a.dst + row) * HL;
          const float4* de = a.de_in ? reinterpret_cast<const float4*>(a.de_in + row * HL) : nullptr;
#pragma unroll
          for (int q = 0; q < HL / 8; ++q) {  // de: read, later rewritten in place: coherent path
            float x1[8];
            ptx::ldg256(da + 8 * q, x1);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const float4 x2 = de ? ptx::ld_hint(de + 2 * q + u, once) : make_float4(0.f, 0.f, 0.f, 0.f);
              dh[8 * q + 4 * u] = fmaf(s, x1[4 * u], x2.x);
              dh[8 * q + 4 * u + 1] = fmaf(s, x1[4 * u + 1], x2.y);
              dh[8 * q + 4 * u + 2] = fmaf(s, x1[4 * u + 2], x2.z);
              dh[8 * q + 4 * u + 3] = fmaf(s, x1[4 * u + 3], x2.w);
            }
          }
#pragma unroll
          for (int j = HL; j < H; ++j) dh[j] = 0.f;
        } else if (DEC) {
#pragma unroll
          for (int j = 0; j < H; ++j) dh[j] = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < a.out_dim) dh[j] = __ldg(a.d_out + row * a.out_dim + j);
        } else {
          bwd_row<HL>(a.d_out + row * HL, dh);
        }
      } else {
#pragma unroll
        for (int j = 0; j < H; ++j) dh[j] = 0.f;
      }
      // One loop over the tile's backward linears (a single inlined copy of the
      // staging / drain / column-sum code keeps the kernel's instruction
      // footprint small): jb = 0 output linear (nn.cpp:241-245), jb = 1..K
      // residual blocks in reverse (nn.cpp:259-274), jb = K+1.. input segments
      // (nn.cpp:277-281). Every job: dX = d W^T on the tensor cores, dW += h^T d.
      long long ti0 = 0;
#pragma unroll 1
      for (int jb = 0; jb < K + 1 + nseg; ++jb) {
        const int c = jb - (K + 1);  // input segment (>= 0 in the input phase)
        if (jb >= 1 && jb <= K) {
          const int l = K + 1 - jb;
          const float4* st = scr + (int64_t)(l - 1) * 16 * 128 + trow;
          const float inv_std = (kExp & 2) ? 1.0f : scr_inv[(l - 1) * 128 + trow];
          const long long tl0 = PROF ? clock64() : 0;
          bwd_store_raw(t_d, dh);  // residual d_h pre-loaded into the accumulator
          static_assert(!HGNN_PK_LNB || HL == 64, "packed LN adjoint: H = 64 only");
          if constexpr (HGNN_PK_LNB) {
          // ELU adjoint (kernels.cpp:68-71), residual rebuild h_{l-1} = h_l - ELU(t_l),
          // LN adjoint (kernels.cpp:99-126), on packed pairs
          float2 p1[4], p2[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) p1[i] = p2[i] = make_float2(0.f, 0.f);
          const float2 l2e = make_float2(1.4426950408889634f, 1.4426950408889634f);
          const float2 m1 = make_float2(-1.f, -1.f);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float4 t4 = (kExp & 2) ? make_float4(0.5f, -0.5f, 0.25f, -0.25f) : ptx::ld_hint(st + q * 128, keep);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int jx = 4 * q + 2 * u;
              const float2 tt = u == 0 ? make_float2(t4.x, t4.y) : make_float2(t4.z, t4.w);
              const float2 z = f2_mul(tt, l2e);
              float2 ex;
              asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex.x) : "f"(z.x));
              asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex.y) : "f"(z.y));
              const float2 em1 = f2_add(ex, m1);
              const float2 el = make_float2(tt.x > 0.f ? tt.x : em1.x, tt.y > 0.f ? tt.y : em1.y);
              const float2 dp = make_float2(tt.x > 0.f ? 1.0f : ex.x, tt.y > 0.f ? 1.0f : ex.y);
              f2_put(h + jx, f2_fma(el, m1, f2_pair(h + jx)));  // h_{l-1}
              const float2 dd = f2_mul(f2_pair(dh + jx), dp);
              f2_put(dh + jx, dd);
              p1[(jx / 2) % 4] = f2_add(p1[(jx / 2) % 4], dd);
              p2[(jx / 2) % 4] = f2_fma(dd, tt, p2[(jx / 2) % 4]);
            }
          }
          const float2 s1 = f2_add(f2_add(p1[0], p1[1]), f2_add(p1[2], p1[3]));
          const float2 s2 = f2_add(f2_add(p2[0], p2[1]), f2_add(p2[2], p2[3]));
          const float g_mean = (s1.x + s1.y) * (1.0f / HL);
          const float gx_mean = (s2.x + s2.y) * (1.0f / HL);
          const float2 ngx = make_float2(-gx_mean, -gx_mean), ngm = make_float2(-g_mean, -g_mean);
          const float2 is2 = make_float2(inv_std, inv_std);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float4 t4 = (kExp & 2) ? make_float4(0.5f, -0.5f, 0.25f, -0.25f) : ptx::ld_hint(st + q * 128, keep);
            const float2 w0 = f2_add(f2_fma(make_float2(t4.x, t4.y), ngx, f2_pair(dh + 4 * q)), ngm);
            const float2 w1 = f2_add(f2_fma(make_float2(t4.z, t4.w), ngx, f2_pair(dh + 4 * q + 2)), ngm);
            f2_put(dh + 4 * q, f2_mul(w0, is2));
            f2_put(dh + 4 * q + 2, f2_mul(w1, is2));
          }
          } else {
          float p1[8], p2[8];
          float tk[HGNN_LNB_KEEP_T ? 64 : 1];  // HGNN_LNB_KEEP_T: t_l kept in registers for pass 2
#pragma unroll
          for (int i = 0; i < 8; ++i) p1[i] = p2[i] = 0.f;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float4 t4 = (kExp & 2) ? make_float4(0.5f, -0.5f, 0.25f, -0.25f) : ptx::ld_hint(st + q * 128, keep);
            const float tv[4] = {t4.x, t4.y, t4.z, t4.w};
            if (HGNN_LNB_KEEP_T) {
#pragma unroll
              for (int u = 0; u < 4; ++u) tk[(4 * q + u) % (HGNN_LNB_KEEP_T ? 64 : 1)] = tv[u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int jx = 4 * q + u;
              const float t = tv[u];
              const float ex = ptx::exp_fast(t);
              const float elu = t > 0.f ? t : ex - 1.0f;
              const float dd = dh[jx] * (t > 0.f ? 1.0f : ex);  // elu', kernels.cpp:68-71
              h[jx] -= elu;                                      // h_{l-1}
              dh[jx] = dd;
              p1[jx % 8] += dd;
              p2[jx % 8] = fmaf(dd, t, p2[jx % 8]);
            }
          }
          const float g_mean =
              (((p1[0] + p1[1]) + (p1[2] + p1[3])) + ((p1[4] + p1[5]) + (p1[6] + p1[7]))) * (1.0f / HL);
          const float gx_mean =
              (((p2[0] + p2[1]) + (p2[2] + p2[3])) + ((p2[4] + p2[5]) + (p2[6] + p2[7]))) * (1.0f / HL);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float4 t4 = HGNN_LNB_KEEP_T ? make_float4(tk[(4 * q) % (HGNN_LNB_KEEP_T ? 64 : 1)],
                                                            tk[(4 * q + 1) % (HGNN_LNB_KEEP_T ? 64 : 1)],
                                                            tk[(4 * q + 2) % (HGNN_LNB_KEEP_T ? 64 : 1)],
                                                            tk[(4 * q + 3) % (HGNN_LNB_KEEP_T ? 64 : 1)])
                              : (kExp & 2) ? make_float4(0.5f, -0.5f, 0.25f, -0.25f) : ptx::ld_hint(st + q * 128, keep);
            if (4 * q >= HL) {  // zero padding
              dh[4 * q] = dh[4 * q + 1] = dh[4 * q + 2] = dh[4 * q + 3] = 0.f;
              continue;
            }
            dh[4 * q] = (dh[4 * q] - g_mean - t4.x * gx_mean) * inv_std;  // kernels.cpp:99-126
            dh[4 * q + 1] = (dh[4 * q + 1] - g_mean - t4.y * gx_mean) * inv_std;
            dh[4 * q + 2] = (dh[4 * q + 2] - g_mean - t4.z * gx_mean) * inv_std;
            dh[4 * q + 3] = (dh[4 * q + 3] - g_mean - t4.w * gx_mean) * inv_std;
          }
          }
          if (kDiscardScratch) {
            // t_l and inv_std of this tile are dead: drop their L2 lines instead
            // of letting them be written back (8 rows of one q per 128-B line)
            __syncwarp();
            if ((trow & 7) == 0) {
#pragma unroll 4
              for (int q = 0; q < 16; ++q) ptx::discard_l2_line(st + q * 128);
            }
            if ((trow & 31) == 0) ptx::discard_l2_line(scr_inv + (l - 1) * 128 + trow);
          }
          if (PROF) pf[6] += (unsigned long long)(clock64() - tl0);
        }
        if (c == 0 && PROF) ti0 = clock64();
        if (c <= 0) {  // new A operand (split d) for this linear; the input segments share one
          bwd_store_a(t_ahi, t_alo, dh);
          tc_signal(&a_full[g]);
          write_db(dh);
        }
        if (FACT && c == 0 && valid) {  // dY: the input linear's output adjoint, for the node-level sums
#pragma unroll
          for (int q = 0; q < 8; ++q) ptx::stg256_hint(a.dy_out + row * H + 8 * q, dh + 8 * q, once);
        }
        if (c >= 0 && !HGNN_BWD_PREFETCH) bwd_gather<MODE, HL>(a, row, valid, c, h, once);  // dW0 segment operand
        stage_chunk(h, dh);
        if (HGNN_BWD_PREFETCH && jb >= K) {  // h is dead: fetch the next dW0 segment operand, or the next
          if (c + 1 < nseg) {                // tile's first input segment, behind the dX wait
            bwd_gather<MODE, HL>(a, row, valid, c + 1, h);
          } else {
            const int64_t nrow = (2 * (pair + gridDim.x) + g) * 128 + trow;
            h_ready = pair + gridDim.x < n_pairs;
            if (h_ready) bwd_gather<MODE, HL>(a, nrow, nrow < a.n_rows, 0, h);
          }
        }
        wait_dx();
        ++job;
        if (c < 0) {
          bwd_load_d(t_d, nullptr, dh);  // d_prev = d_u W^T + d_h
        } else {
          float* outp;
          if (FACT) outp = a.de_io;
          else if (MODE == kEdgeInput) outp = c == 0 ? a.d_src : (c == 1 ? a.d_dst : a.de_io);
          else if (DEC) outp = a.d_x_out;
          else outp = c == 0 ? a.d_a_out : a.d_x_out;
#pragma unroll
          for (int cc = 0; cc < (ENC ? 0 : HL); cc += 16) {  // kEncoder: the feature adjoint is not needed
            float p[16];
            ptx::tmem_ld16(t_d + cc, p);
            ptx::tmem_wait_ld();
            if (valid) {
              ptx::stg256_hint(outp + row * HL + cc, p, once);
              ptx::stg256_hint(outp + row * HL + cc + 8, p + 8, once);
            }
          }
          if (c + 1 < nseg) tc_signal(&a_full[g]);  // D consumed; A (= split d_h) stays
        }
      }
      if (PROF) pf[7] += (unsigned long long)(clock64() - ti0);
    }
    if (!kDwN128 && !(kExp & 1) && job >= 2) flush(job - 2);  // last dW job(s) of this CTA
    if (!(kExp & 1) && job >= 1) flush(job - 1);
    if (PROF && warp == 0 && lane == 0) {
      pf[0] = (unsigned long long)(clock64() - pf_t0);
#pragma unroll
      for (int i = 0; i < 8; ++i) atomicAdd(a.prof + kProfEpiTotal + i, pf[i]);
    }
  } else if (warp == 8) {
    // ================================================================ MMA issuer
    // warp-uniform TMEM base; all 32 lanes run the schedule, mma/commit elect one lane
    const uint32_t tm = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile uint32_t*>(tmem_base_slot), 0);
    {
      constexpr uint32_t idesc = ptx::idesc_tf32(128, H);
      int ws = 0;
      uint32_t wph = 0, pa[2] = {0, 0};
      auto mma3 = [&](int s, uint32_t bbase, bool first_zero) {
        const uint32_t slot = ptx::opaque(tm + s * Cfg::SLOT_COLS);
        // descriptor start addresses advance in 16-byte units: bump the encoded
        // base instead of re-encoding (keeps the issuer's register use small)
        const uint64_t d0 = ptx::opaque64(ptx::smem_desc(bbase, Cfg::LBO, Cfg::SBO));
#pragma unroll
        for (int ks = 0; ks < H / 8; ++ks) {
          const uint64_t b_hi = d0 + (uint64_t)((ks * 2 * Cfg::LBO) >> 4);
          const uint64_t b_lo = b_hi + (uint64_t)(Cfg::LO_OFF >> 4);
          ptx::mma_tf32_ts_w(slot + 2 * H, slot + 8 * ks, b_hi, idesc, (!first_zero || ks > 0) ? 1u : 0u);
          ptx::mma_tf32_ts_w(slot + 2 * H, slot + 8 * ks, b_lo, idesc, 1u);
          ptx::mma_tf32_ts_w(slot + 2 * H, slot + H + 8 * ks, b_hi, idesc, 1u);
        }
      };
      unsigned long long pc_w = 0, pc_a = 0;  // wait cycles (profiling only)
      const long long t_start = clock64();
      auto timed_wait = [&](uint64_t* bar, uint32_t par, unsigned long long& acc) {
        if (!PROF) {
          ptx::mbar_wait(bar, par);
          return;
        }
        const long long t0 = clock64();
        ptx::mbar_wait(bar, par);
        acc += (unsigned long long)(clock64() - t0);
      };
      auto next_w = [&]() -> uint32_t {
        timed_wait(&w_full[ws], wph, pc_w);
        ptx::tc_fence_after();
        return ptx::smem_u32(wring + (size_t)ws * Cfg::CHUNK_FLOATS);
      };
      auto release_w = [&]() {
        ptx::mma_commit_w(&w_empty[ws]);
        if (++ws == Cfg::WSTAGES) {
          ws = 0;
          wph ^= 1;
        }
      };
      unsigned long long pc_fwd = 0, pc_mma = 0;  // phase cycles (profiling only)
      // One loop over the linears of a tile (single inlined copy of the MMA
      // sequence keeps the issuer's code small): forward recompute (input
      // segments, hidden blocks), backward output linear and hidden blocks in
      // reverse (D pre-loaded with the residual d_h except for the output
      // linear), backward input segments. dW MMAs run on the dW issuer.
      for (int64_t pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
        const long long t_p0 = PROF ? clock64() : 0;
#pragma unroll 1
        for (int st = 0; st < n_w; ++st) {
          const bool first_zero = st == 0 || (st >= nseg && st < nseg + K) || st >= nseg + 2 * K + 1 ||
                                  st == nseg + K;  // recompute input c = 0, recompute hidden, input dX, output dX
          const bool to_a_empty = st + 1 < nseg;   // recompute input segments before the last
          if (PROF && st == nseg + K) pc_fwd += (unsigned long long)(clock64() - t_p0);
          const uint32_t bb = next_w();
#pragma unroll 1
          for (int s = 0; s < 2; ++s) {
            timed_wait(&a_full[s], pa[s], pc_a);
            pa[s] ^= 1;
            ptx::tc_fence_after();
            const long long t_m0 = PROF ? clock64() : 0;
            mma3(s, bb, first_zero);
            ptx::mma_commit_w(to_a_empty ? &a_empty[s] : &d_full[s]);
            if (PROF) pc_mma += (unsigned long long)(clock64() - t_m0);
          }
          release_w();
        }
      }
      if (PROF && lane == 0) {
        atomicAdd(a.prof + kProfTotal, (unsigned long long)(clock64() - t_start));
        atomicAdd(a.prof + kProfW, pc_w);
        atomicAdd(a.prof + kProfA, pc_a);
        atomicAdd(a.prof + kProfFwd, pc_fwd);
        atomicAdd(a.prof + kProfMma, pc_mma);
      }
    }
  } else if (warp == 9) {
    // ================================================================ dW issuer
    // Separate instruction stream from the dX issuer, so the dX MMAs of one
    // slot never wait behind the other slot's staging of the current job.
    const uint32_t tm = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile uint32_t*>(tmem_base_slot), 0);
    constexpr uint32_t idesc_dw =
        ptx::idesc_tf32(128, kDwN128 ? 2 * H : H) | (1u << 15) | (1u << 16);  // A, B MN-major, N = 128 / 64
    int64_t gi = 0;  // staging chunk counter
    unsigned long long pc_st = 0, pc_dw = 0, pc_dwt = 0;
    const long long t_start = PROF ? clock64() : 0;
    const int64_t n_jobs = (kExp & 1) ? 0 : ((n_pairs - blockIdx.x + gridDim.x - 1) / gridDim.x) * n_dw;
    for (int64_t jd = 0; jd < n_jobs; ++jd) {
      const int acc = kDwN128 ? 0 : (int)(jd & 1);
      const long long t0 = PROF ? clock64() : 0;
      // the accumulator's previous job (jd - 1, or jd - 2 when double-buffered) drained
      const uint32_t dwe_par = kDwN128 ? (uint32_t)((jd & 1) ^ 1) : (uint32_t)(((jd >> 1) & 1) ^ 1);
      if (HGNN_PARK_AUX) ptx::mbar_wait_parked(&dw_empty[acc], dwe_par);
      else ptx::mbar_wait(&dw_empty[acc], dwe_par);
      ptx::tc_fence_after();
      if (PROF) pc_dw += (unsigned long long)(clock64() - t0);
      const uint32_t t_dw = ptx::opaque(tm + Cfg::DW_COL + 64 * acc);
      for (int b = 0; b < 8; ++b, ++gi) {
        const int buf = (int)(gi % Cfg::NSTAGE);
        const uint32_t par = (uint32_t)((gi / Cfg::NSTAGE) & 1);
        const long long t1 = PROF ? clock64() : 0;
        if (HGNN_PARK_AUX) ptx::mbar_wait_parked(&st_full[buf], par);
        else ptx::mbar_wait(&st_full[buf], par);
        ptx::tc_fence_after();
        if (PROF) pc_st += (unsigned long long)(clock64() - t1);
        const uint32_t sa = ptx::smem_u32(stage + (size_t)buf * Cfg::STAGE_BYTES);
        constexpr uint64_t swz = (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
        const uint64_t a0 = ptx::opaque64(ptx::smem_desc(sa, Cfg::ST_LBO, Cfg::ST_SBO) | swz);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          // [h_hi ; h_lo] (M = 128) x d_hi and x d_lo (N = 64 each, MN atoms 0-1 / 2-3)
          const uint64_t ad = a0 + (uint64_t)((ks * 2 * Cfg::ST_SBO) >> 4);
          const uint64_t bd_hi = ad + (uint64_t)(16384 >> 4);
          const uint64_t bd_lo = bd_hi + (uint64_t)((2 * Cfg::ST_LBO) >> 4);
          ptx::mma_tf32_ss_w(t_dw, ad, bd_hi, idesc_dw, (b > 0 || ks > 0) ? 1u : 0u);
          if (!kDwN128) ptx::mma_tf32_ss_w(t_dw, ad, bd_lo, idesc_dw, 1u);
        }
        ptx::mma_commit_w(&st_empty[((gi / Cfg::NSTAGE) & 1) * Cfg::NSTAGE + buf]);
      }
      ptx::mma_commit_w(&dw_full[acc]);
      if (PROF) pc_dwt += (unsigned long long)(clock64() - t0);
    }
    if (PROF && lane == 0) {
      (void)t_start;
      atomicAdd(a.prof + kProfSt, pc_st);
      atomicAdd(a.prof + kProfDwE, pc_dw);
      atomicAdd(a.prof + kProfDw, pc_dwt);
    }
  } else {
    // ================================================================ loader (warp 10; 11 idle)
    if (warp == 10 && lane == 0) {
      int ws = 0;
      uint32_t wph = 0;
      for (int64_t pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
        for (int j = 0; j < n_w; ++j) {
          if (HGNN_PARK_AUX) ptx::mbar_wait_parked(&w_empty[ws], wph ^ 1);
          else ptx::mbar_wait(&w_empty[ws], wph ^ 1);
          ptx::mbar_arrive_expect_tx(&w_full[ws], Cfg::CHUNK_BYTES);
          ptx::bulk_g2s(wring + (size_t)ws * Cfg::CHUNK_FLOATS, a.chunks + (size_t)j * Cfg::CHUNK_FLOATS,
                        Cfg::CHUNK_BYTES, &w_full[ws]);
          if (++ws == Cfg::WSTAGES) {
            ws = 0;
            wph ^= 1;
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

}  // namespace hgnn_b200
