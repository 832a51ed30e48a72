// Tensor-core processor-MLP forward (sm_100a, tcgen05 kind::tf32).
//
// Same math as mlp_forward_kernel (mlp_simt.cuh), at fp32-level accuracy
// through a 3xTF32 split: for every linear y = a W,
//   y = a_hi W_hi + a_hi W_lo + a_lo W_hi        (a_lo W_lo ~ 2^-22 dropped)
// issued as three M=128, N=H MMAs per K-step into one fp32 accumulator.
//
// Data placement (per CTA, persistent, one CTA per SM):
//   TMEM  2 tile slots x [A_hi (H cols) | A_lo (H cols) | D (H cols)], 128
//         lanes; lane = row of the 128-row tile.
//   SMEM  ring of weight chunks: each chunk = K = H rows of one linear as the
//         B operand [W_hi | W_lo]^T (2H x H, K-major, SWIZZLE_NONE core
//         matrices), laid out on the host so one cp.async.bulk moves it.
// Warp roles: warps 0-3 epilogue of slot 0, warps 4-7 of slot 1 (thread =
// TMEM lane = row: bias, LN0, ELU, residual, hi/lo split, all row-local),
// warp 8 lane 0 issues MMAs, warp 9 lane 0 streams weight chunks.
// The two slots ping-pong: the MMA of one tile runs while the other tile's
// epilogue works. Input rows (x[src], x[dst], e / a*, x) are gathered one
// segment ahead so their latency hides behind the MMA of the previous one.
//
// kEdgeFused / kEdgeFact (the edge update of the MP layer, model.cpp:233-240,
// as ONE kernel): tiles are runs of whole receiver segments (<= 128 slots,
// from a table built at graph upload); kEdgeFused gathers [x_src | x_dst | e]
// as kEdgeInput, kEdgeFact computes the input linear as one K = H segment
// (e W0_e) plus the gathered node projections P_s[src] + P_d[dst]; the output
// rows go through a swizzled shared-memory tile to a reducer warp per slot
// (warps 10 / 11) that streams e' to HBM with coalesced row stores and forms
// the degree-scaled aggregate a[i] = sum inv_d e' over each receiver segment
// in slot order (= scatter_rows_csr's in-CSR order, kernels.cpp:355-368), so
// e' is never re-read and no atomics are used.
#pragma once

#include <cuda.h>  // CUtensorMap

#include "mlp_simt.cuh"
#include "tc_ptx.cuh"

namespace hgnn_b200 {

template <int H>
struct TcCfg {
  static constexpr int NB = 2 * H;                      // rows of a chunk: [W_hi | W_lo]^T
  static constexpr int CHUNK_FLOATS = NB * H;           // one K = H chunk
  static constexpr int CHUNK_BYTES = CHUNK_FLOATS * 4;  // 32 KB at H = 64
  static constexpr uint32_t LBO = (NB / 8) * 128;       // K-adjacent core matrices
  static constexpr uint32_t SBO = 128;                  // N-adjacent core matrices
  static constexpr uint32_t LO_OFF = (H / 8) * 128;     // start of the W_lo half
  static constexpr int SLOT_COLS = 3 * H;
  static constexpr int TMEM_COLS = H == 64 ? 512 : 256;  // power of two >= 2 slots
  static constexpr int STAGES = H == 64 ? 4 : 8;
  static constexpr int THREADS = 384;  // 2 epilogue warpgroups + 1 control warpgroup
  static constexpr size_t OFF_BARS = (size_t)STAGES * CHUNK_BYTES;
  static constexpr size_t OFF_BIAS = OFF_BARS + 256;
  static constexpr size_t OFF_Y = OFF_BIAS + 18 * H * 4;              // kEdgeFact: 2 output tiles (128 x H)
  static constexpr size_t SMEM = OFF_Y + 1024;                         // + biases (k <= 16)
  static constexpr size_t SMEM_FACT = OFF_Y + 2 * 128 * H * 4 + 1024;
  static constexpr size_t SMEM_ENC = OFF_Y + 10 * H * 4 + 1024;       // kEncoder: skip W (<= 8 x H), LN gamma, beta
  // fused edge kernel with TMA-gathered input rows (mlp_tc_forward_tma_kernel):
  // 2 weight stages, output tiles, one 128-row gather buffer per slot
  static constexpr int T_STAGES = 2;
  static constexpr size_t T_OFF_BARS = (size_t)T_STAGES * CHUNK_BYTES;
  static constexpr size_t T_OFF_BIAS = T_OFF_BARS + 256;
  static constexpr size_t T_OFF_Y = (T_OFF_BIAS + 18 * H * 4 + 1023) / 1024 * 1024;
  static constexpr size_t T_OFF_GX = T_OFF_Y + 2 * 128 * H * 4;
  static constexpr size_t SMEM_TMA = T_OFF_GX + 2 * 128 * H * 4 + 1024;
};

// Index (in floats) of B element (n, k) inside a chunk (K-major core matrices).
__host__ __device__ inline int64_t tc_chunk_index(int n, int k, int H) {
  const int nb = 2 * H;
  return (int64_t)(k / 4) * (nb / 8) * 32 + (n / 8) * 32 + (n % 8) * 4 + (k % 4);
}

struct TcFwdArgs {
  int64_t n_rows;
  const int32_t* src;
  const int32_t* dst;
  const float* x;
  const float* e_in;
  const float* a;
  float* out;
  const float* chunks;  // (nseg + k + 1) chunks in MMA order
  const float* params;  // fp32 for_each layout (biases)
  int k;
  unsigned long long* prof;  // optional cycle counters (kFwdProf*), PROF instantiation only
  // kEdgeFact
  int64_t n_tiles;
  const int32_t* tiles;  // [n_tiles + 1] slot offsets; tile t = slots [tiles[t], tiles[t+1])
  const float* proj;     // rows x 2H: [P_s | P_d] = x [W0_s | W0_d]
  const float* inv;      // per slot 1/d
  float* agg;            // rows x H aggregate (rows with an empty segment are not written)
  // kEncoder (encoder MLP, model.cpp:70-80): e_in = n_rows x in_dim features
  // (in_dim <= 8, zero-padded to one K = H segment); params in the encoder's
  // for_each layout (GenLayout, mlp_generic.cuh); out = LN(y) * gamma + beta
  // with y = MLP(x) + x W_skip, or y itself (enc_ln = 0: the backward's
  // pre-LayerNorm recompute)
  int in_dim;
  int enc_ln;
  // kDecoder (decoder MLP, model.cpp:92-101): x rows (H wide) in, out =
  // n_rows x out_dim (<= 8): y = MLP(x) + x W_skip, the output linear's
  // columns >= out_dim zero-padded in the chunks
  int out_dim;
};

// Optional instrumentation of the forward kernel (cycles summed over CTAs;
// epilogue figures from warp 0 lane 0).
enum { kFwdProfIssTotal = 0, kFwdProfIssA = 1, kFwdProfIssW = 2, kFwdProfIssMma = 3, kFwdProfEpiTotal = 4,
       kFwdProfEpiD = 5, kFwdProfEpiAE = 6, kFwdProfEpiSig = 7, kFwdProfEpiLd = 8, kFwdProfEpiMath = 9,
       kFwdProfEpiStA = 10, kFwdProfEpiGather = 11 /* whole input phase */, kFwdProfEpiOut = 12 };

__device__ __forceinline__ float elu_fast(float z) { return z > 0.f ? z : ptx::exp_fast(z) - 1.0f; }

// Packed fp32 (FFMA2 / FADD2 / FMUL2, sm_100): two lanes of a row per
// instruction in the epilogue math — half the FP issue slots of the scalar code.
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 f2_pair(const float* v) { return make_float2(v[0], v[1]); }
__device__ __forceinline__ void f2_put(float* v, float2 p) {
  v[0] = p.x;
  v[1] = p.y;
}

// Sum of H values with 8 independent partial sums (4 packed pairs, short chains).
template <int H>
__device__ __forceinline__ float tree_sum(const float (&v)[H]) {
  float2 p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = f2_pair(v + 2 * i);
#pragma unroll
  for (int j = 4; j < H / 2; ++j) p[j % 4] = f2_add(p[j % 4], f2_pair(v + 2 * j));
  const float2 q = f2_add(f2_add(p[0], p[1]), f2_add(p[2], p[3]));
  return q.x + q.y;
}

// Parameter-free LayerNorm (kernels.cpp:81-94) with tree reductions; returns inv_std.
template <int H>
__device__ __forceinline__ float ln0_tree(float (&v)[H]) {
  const float mean = tree_sum<H>(v) * (1.0f / H);
  const float2 nm = make_float2(-mean, -mean);
  float2 p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < H / 2; ++j) {
    const float2 d = f2_add(f2_pair(v + 2 * j), nm);
    p[j % 4] = f2_fma(d, d, p[j % 4]);
  }
  const float2 q = f2_add(f2_add(p[0], p[1]), f2_add(p[2], p[3]));
  const float var = (q.x + q.y) * (1.0f / H);
  const float inv_std = ptx::rsqrt_fast(var + 1e-12f);
  const float2 is = make_float2(inv_std, inv_std);
#pragma unroll
  for (int j = 0; j < H / 2; ++j) f2_put(v + 2 * j, f2_mul(f2_add(f2_pair(v + 2 * j), nm), is));
  return inv_std;
}

// h += ELU(t) (kernels.cpp:263-266) on packed pairs: one FMUL2 for the
// exponent scaling, two ex2.approx, one FADD2 for e^t - 1, selects, one FADD2.
template <int H>
__device__ __forceinline__ void add_elu(float (&h)[H], const float (&t)[H]) {
  const float2 l2e = make_float2(1.4426950408889634f, 1.4426950408889634f), m1 = make_float2(-1.f, -1.f);
#pragma unroll
  for (int j = 0; j < H / 2; ++j) {
    const float2 tt = f2_pair(t + 2 * j);
    const float2 z = f2_mul(tt, l2e);
    float2 e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(z.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(z.y));
    e = f2_add(e, m1);
    const float2 el = make_float2(tt.x > 0.f ? tt.x : e.x, tt.y > 0.f ? tt.y : e.y);
    f2_put(h + 2 * j, f2_add(f2_pair(h + 2 * j), el));
  }
}

template <int H>
__device__ __forceinline__ void tc_store_a(uint32_t t_hi, uint32_t t_lo, const float (&v)[H]) {
#pragma unroll
  for (int c = 0; c < H; c += 32) {
    float hi[32], lo[32];
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      hi[j] = ptx::tf32_hi(v[c + j]);
      hi[j + 1] = ptx::tf32_hi(v[c + j + 1]);
      f2_put(lo + j, f2_add(f2_pair(v + c + j), make_float2(-hi[j], -hi[j + 1])));
    }
    ptx::tmem_st32(t_hi + c, hi);
    ptx::tmem_st32(t_lo + c, lo);
  }
}

// y[j] = D[:, j] + b[j]; all TMEM loads in flight before the one wait
template <int H>
__device__ __forceinline__ void tc_load_d(uint32_t t_d, const float* __restrict__ b, float (&y)[H]) {
#pragma unroll
  for (int c = 0; c < H; c += 32) ptx::tmem_ld32(t_d + c, *reinterpret_cast<float(*)[32]>(y + c));
  ptx::tmem_wait_ld();
#pragma unroll
  for (int j = 0; j < H; j += 2) f2_put(y + j, f2_add(f2_pair(y + j), f2_pair(b + j)));
}

__device__ __forceinline__ void tc_signal(uint64_t* bar) {
  ptx::tmem_wait_st();
  ptx::tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(bar);
}

#ifndef HGNN_FWD_STREAM_HINT
#define HGNN_FWD_STREAM_HINT 0
#endif
#ifndef HGNN_EXP
#define HGNN_EXP 0  // timing experiments only (scripts/build_exp.py); bits 32: input gathers dropped, 64: no e' stores, 128: no reducer work
#endif

// pol != 0: L2 cache-hint policy of the row loads (the backward keeps rows it
// gathers twice, evict_last, and streams the second read, evict_first)
template <int H, int MODE>
__device__ __forceinline__ void tc_gather(const TcFwdArgs& a, int64_t row, bool valid, int c, float (&v)[H],
                                          uint64_t pol = 0) {
  if (HGNN_EXP & 32) valid = false;
  if (MODE == kEncoder) {  // in_dim (<= 8) features, zero-padded to H
#pragma unroll
    for (int j = 0; j < H; ++j) v[j] = 0.f;
    if (valid) {
      const float* f = a.e_in + row * a.in_dim;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < a.in_dim) v[j] = __ldg(f + j);
    }
    return;
  }
  if (valid) {
    const float* seg;
    if (MODE == kEdgeFact)
      seg = a.e_in + row * H;
    else if (MODE == kDecoder)
      seg = a.x + row * H;
    else if (MODE == kEdgeInput || MODE == kEdgeFused)
      seg = c == 0 ? a.x + (int64_t)__ldg(a.src + row) * H
                   : (c == 1 ? a.x + (int64_t)__ldg(a.dst + row) * H : a.e_in + row * H);
    else
      seg = c == 0 ? a.a + row * H : a.x + row * H;
#ifndef HGNN_LDG256
#define HGNN_LDG256 1
#endif
    if (HGNN_LDG256) {
      if (pol) {
#pragma unroll
        for (int j = 0; j < H / 8; ++j) ptx::ldg256_hint(seg + 8 * j, v + 8 * j, pol);
      } else {
#pragma unroll
        for (int j = 0; j < H / 8; ++j) ptx::ldg256(seg + 8 * j, v + 8 * j);
      }
    } else {
#pragma unroll
      for (int j = 0; j < H / 4; ++j) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(seg) + j);
        v[4 * j] = t.x;
        v[4 * j + 1] = t.y;
        v[4 * j + 2] = t.z;
        v[4 * j + 3] = t.w;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < H; ++j) v[j] = 0.f;
  }
}

// v = P_s[src[row]] + P_d[dst[row]] (kEdgeFact input projection of the node ends)
template <int H>
__device__ __forceinline__ void tc_gather_proj(const TcFwdArgs& a, int64_t row, bool valid, float (&v)[H]) {
  if (!valid) {
#pragma unroll
    for (int j = 0; j < H; ++j) v[j] = 0.f;
    return;
  }
  const float* ps = a.proj + (int64_t)__ldg(a.src + row) * (2 * H);
  const float* pd = a.proj + (int64_t)__ldg(a.dst + row) * (2 * H) + H;
#pragma unroll
  for (int j = 0; j < H / 8; ++j) {
    float s[8], d[8];
    ptx::ldg256(ps + 8 * j, s);
    ptx::ldg256(pd + 8 * j, d);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[8 * j + i] = s[i] + d[i];
  }
}

// Byte offset of 16-byte chunk c of row r in a 128 x H fp32 tile (chunk index
// XOR row % 8: conflict-free row writes by row-per-thread warps and
// conflict-free row reads by column-per-lane warps).
template <int H>
__device__ __forceinline__ uint32_t ytile_off(int r, int c) {
  return (uint32_t)(r * H * 4 + ((c ^ (r & 7)) << 4));
}

#ifndef HGNN_PRODUCER_SLEEP_NS
#define HGNN_PRODUCER_SLEEP_NS 100
#endif
// TMA tile::gather4: rows i0..i3 of a 2-D tensor map (box 32 floats x 1 row,
// 128-byte swizzle), columns [col, col + 32), into 4 consecutive 128-byte
// smem rows, completing on bar.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int col, int i0, int i1, int i2, int i3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(i0), "r"(i1), "r"(i2), "r"(i3), "r"(ptx::smem_u32(bar))
      : "memory");
}

// TMAG (fused edge modes, H = 64): the input segments of each tile are
// gathered by TMA (tile::gather4 over the receiver-sorted slots' src / dst
// indices, or the slots' own e rows) into a per-slot 128-row SMEM buffer
// (two 16 KB halves, 128-byte swizzle), issued by warp 9 between its weight
// chunk loads, and the epilogue reads its row from SMEM right before the
// operand store — coalesced 128-byte TMA requests instead of per-thread row
// loads through L1, and segment 0 of the next tile lands during the current
// tile's hidden layers.
template <int H, int MODE, bool PROF, bool TMAG>
__device__ __forceinline__ void mlp_tc_forward_body(const TcFwdArgs& a, const CUtensorMap* tmx, const CUtensorMap* tme) {
  using Cfg = TcCfg<H>;
  constexpr bool FACT = MODE == kEdgeFact;
  constexpr bool FUSED = MODE == kEdgeFact || MODE == kEdgeFused;  // segment tiles + in-kernel aggregate
  constexpr bool ENC = MODE == kEncoder;
  constexpr bool DEC = MODE == kDecoder;
  constexpr int nseg = (MODE == kEdgeFact || ENC || DEC) ? 1 : (MODE == kNodeInput ? 2 : 3);
  // parameter layout (kEdgeFact: the 3H-input MLP; kEncoder: F input features)
  const int in_dim = ENC ? a.in_dim : (DEC ? H : (MODE == kNodeInput ? 2 : 3) * H);
  static_assert(!TMAG || (FUSED && H == 64), "TMA gathers: fused edge modes at H = 64");
  constexpr int STAGES = TMAG ? Cfg::T_STAGES : Cfg::STAGES;
  constexpr size_t OFF_BARS = TMAG ? Cfg::T_OFF_BARS : Cfg::OFF_BARS;
  constexpr size_t OFF_BIAS = TMAG ? Cfg::T_OFF_BIAS : Cfg::OFF_BIAS;
  constexpr size_t OFF_Y = TMAG ? Cfg::T_OFF_Y : Cfg::OFF_Y;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* wring = reinterpret_cast<float*>(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BARS);
  uint64_t* w_full = bars;                    // [STAGES]
  uint64_t* w_empty = bars + STAGES;          // [STAGES]
  uint64_t* a_full = bars + 2 * STAGES;       // [2]
  uint64_t* a_empty = a_full + 2;             // [2]
  uint64_t* d_full = a_empty + 2;             // [2]
  uint64_t* y_full = d_full + 2;              // [2] kEdgeFact: output tile written (4 epilogue warps)
  uint64_t* y_empty = y_full + 2;             // [2] kEdgeFact: output tile consumed (reducer warp)
  uint64_t* gx_full = y_empty + 2;            // [2] TMAG: gather buffer landed (TMA transaction bytes)
  uint64_t* gx_empty = gx_full + 2;           // [2] TMAG: gather buffer read (4 epilogue warps)
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(gx_empty + 2);
  float* sbias = reinterpret_cast<float*>(smem + OFF_BIAS);  // (k+2) x H
  uint8_t* ytile = smem + OFF_Y;                             // kEdgeFact: [2][128][H] swizzled
  float* senc = reinterpret_cast<float*>(smem + OFF_Y);       // kEncoder: W_skip [8][H], gamma, beta
  uint8_t* gx = smem + Cfg::T_OFF_GX;                         // TMAG: [2][2 halves][128][32] swizzled

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n_chunks = nseg + a.k + 1;
  const int64_t n_tiles = FUSED ? a.n_tiles : (a.n_rows + 127) / 128;
  const int64_t n_pairs = (n_tiles + 1) / 2;
  // rows of tile t: [t_beg, t_end) (kEdgeFact: a run of whole receiver segments)
  auto tile_rows = [&](int64_t t, int64_t& beg, int64_t& end) {
    if (FUSED) {
      beg = t < n_tiles ? (int64_t)__ldg(a.tiles + t) : 0;
      end = t < n_tiles ? (int64_t)__ldg(a.tiles + t + 1) : 0;
    } else {
      beg = t * 128;
      end = beg + 128 < a.n_rows ? beg + 128 : a.n_rows;
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&w_full[s], 1);
      ptx::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&a_full[s], 4);
      ptx::mbar_init(&a_empty[s], 1);
      ptx::mbar_init(&d_full[s], 1);
      ptx::mbar_init(&y_full[s], 4);
      ptx::mbar_init(&y_empty[s], 1);
      ptx::mbar_init(&gx_full[s], 1);
      ptx::mbar_init(&gx_empty[s], 4);
    }
    ptx::fence_mbarrier_init();
  }
  for (int i = threadIdx.x; i < (a.k + 2) * H; i += blockDim.x) {
    const int l = i / H, j = i % H;
    if (DEC && l == a.k + 1)  // decoder output bias: out_dim entries after W_{k+1} (H x out_dim)
      sbias[i] = j < a.out_dim ? __ldg(a.params + mlp_w_offset(l, H, H) + H * a.out_dim + j) : 0.f;
    else
      sbias[i] = __ldg(a.params + mlp_b_offset(l, in_dim, H) + j);
  }
  if (DEC) {  // W_skip (H x out_dim) as [H][8]
    const int64_t skip = mlp_w_offset(a.k + 1, H, H) + (H + 1) * a.out_dim;
    for (int i = threadIdx.x; i < 8 * H; i += blockDim.x) {
      const int r = i / 8, o = i % 8;
      senc[i] = o < a.out_dim ? __ldg(a.params + skip + r * a.out_dim + o) : 0.f;
    }
  }
  if (ENC) {  // GenLayout{in_dim, H, k, H}: skip at b(k+1) + H, then gamma, beta
    const int64_t skip = mlp_b_offset(a.k + 1, in_dim, H) + H;
    for (int i = threadIdx.x; i < 10 * H; i += blockDim.x) {
      const int r = i / H;
      float w = 0.f;
      if (r < in_dim) w = __ldg(a.params + skip + i);
      else if (r >= 8) w = __ldg(a.params + skip + (int64_t)in_dim * H + (r - 8) * H + (i % H));
      senc[i] = w;
    }
  }
  if (warp == 8) ptx::tmem_alloc<Cfg::TMEM_COLS>(tmem_base_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_base_slot;

#ifndef HGNN_FWD_EPI_REGS
#define HGNN_FWD_EPI_REGS 224
#endif
  // the CTA's pool is fixed at launch (384 threads x 168): what the control
  // warpgroup releases is all the epilogue can take
  constexpr int EPI_REGS = HGNN_FWD_EPI_REGS, CTL_REGS = (384 * 168 - 256 * EPI_REGS) / 128 / 8 * 8;
  static_assert(256 * EPI_REGS + 128 * CTL_REGS <= 384 * 168 && CTL_REGS >= 24, "setmaxnreg exceeds the CTA pool");
  // HGNN_FWD_STREAM_HINT: the slots' own e rows (read once) and e' (read by the
  // next layer only) go through L2 evict_first, keeping it for the reused
  // node rows / projections
  const uint64_t stream_pol = HGNN_FWD_STREAM_HINT ? ptx::policy_evict_first() : 0;
  auto fwd_e_pol = [&](int c) -> uint64_t {
    return (HGNN_FWD_STREAM_HINT && (FACT || (MODE == kEdgeFused && c == 2))) ? stream_pol : 0;
  };
  if (warp < 8) ptx::regs_inc<EPI_REGS>();
  else ptx::regs_dec<CTL_REGS>();

  if (warp < 8) {
    // ------------------------------------------------------------ epilogue
    uint32_t pgx = 0;  // TMAG: gx_full phase of this slot
    const int g = warp / 4;   // tile slot
    const int wq = warp % 4;  // TMEM lane quarter
    const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
    const uint32_t t_ahi = tmem + g * Cfg::SLOT_COLS + lane_off;
    const uint32_t t_alo = t_ahi + H;
    const uint32_t t_d = t_ahi + 2 * H;
    uint32_t pe = 0, pd = 0;
    unsigned long long e_d = 0, e_ae = 0, e_sig = 0, e_ld = 0, e_math = 0, e_sta = 0, e_in = 0, e_out = 0;
    const long long e_t0 = PROF ? clock64() : 0;
    auto wait_d = [&]() {
      const long long t0 = PROF ? clock64() : 0;
      ptx::mbar_wait(&d_full[g], pd);
      pd ^= 1;
      ptx::tc_fence_after();
      if (PROF) e_d += (unsigned long long)(clock64() - t0);
    };
    auto signal_a = [&]() {
      const long long t0 = PROF ? clock64() : 0;
      tc_signal(&a_full[g]);
      if (PROF) e_sig += (unsigned long long)(clock64() - t0);
    };
    float v[H];
    const int trow = 32 * wq + lane;  // row inside the tile
    uint32_t py = 0;                  // y_empty phase (kEdgeFact)
    // TMAG: this thread's row of the slot's gather buffer (128-byte swizzle:
    // 16-byte chunk j of row r at r * 128 + ((j ^ r % 8) << 4)); conflict-free
    auto read_seg = [&](bool valid_row) {
      ptx::mbar_wait(&gx_full[g], pgx);
      pgx ^= 1;
      const uint8_t* rb = gx + (size_t)g * (128 * H * 4) + trow * 128;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 t = *reinterpret_cast<const float4*>(rb + hf * (128 * 128) + ((j ^ (trow & 7)) << 4));
          v[32 * hf + 4 * j] = valid_row ? t.x : 0.f;
          v[32 * hf + 4 * j + 1] = valid_row ? t.y : 0.f;
          v[32 * hf + 4 * j + 2] = valid_row ? t.z : 0.f;
          v[32 * hf + 4 * j + 3] = valid_row ? t.w : 0.f;
        }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&gx_empty[g]);
    };
    int64_t pair = blockIdx.x;
    if (!TMAG && pair < n_pairs) {
      int64_t b0, e0;
      tile_rows(2 * pair + g, b0, e0);
      tc_gather<H, MODE>(a, b0 + trow, b0 + trow < e0, 0, v, fwd_e_pol(0));
    }
    for (; pair < n_pairs; pair += gridDim.x) {
      int64_t tb, te;
      tile_rows(2 * pair + g, tb, te);
      const int64_t row = tb + trow;
      const bool valid = row < te;
      float h[H];
      const long long t_in0 = PROF ? clock64() : 0;
      // input projection: nseg K-chunks streamed through A, next one prefetched
#pragma unroll 1
      for (int c = 0; c < nseg; ++c) {
        if (c > 0) {
          const long long t0 = PROF ? clock64() : 0;
          ptx::mbar_wait(&a_empty[g], pe);
          pe ^= 1;
          ptx::tc_fence_after();
          if (PROF) e_ae += (unsigned long long)(clock64() - t0);
        }
        if (TMAG) read_seg(valid);
        tc_store_a<H>(t_ahi, t_alo, v);
        signal_a();
        if (!TMAG && c + 1 < nseg) tc_gather<H, MODE>(a, row, valid, c + 1, v, fwd_e_pol(c + 1));
      }
      if (FACT) tc_gather_proj<H>(a, row, valid, v);  // node-end projections, during the e W0_e MMA
      wait_d();
      tc_load_d<H>(t_d, sbias, h);
      if (FACT) {
#pragma unroll
        for (int j = 0; j < H; ++j) h[j] += v[j];
      }
      if (PROF) e_in += (unsigned long long)(clock64() - t_in0);
      // residual blocks
      for (int l = 1; l <= a.k; ++l) {
        long long t0 = PROF ? clock64() : 0;
        tc_store_a<H>(t_ahi, t_alo, h);
        if (PROF) {
          const long long t1 = clock64();
          e_sta += (unsigned long long)(t1 - t0);
        }
        signal_a();
        wait_d();
        if (PROF) t0 = clock64();
        float u[H];
        tc_load_d<H>(t_d, sbias + l * H, u);
        if (PROF) {
          const long long t1 = clock64();
          e_ld += (unsigned long long)(t1 - t0);
          t0 = t1;
        }
        ln0_tree<H>(u);
        add_elu<H>(h, u);
        if (PROF) {
          __syncwarp();
          e_math += (unsigned long long)(clock64() - t0);
        }
      }
      // output projection; the next tile's first segment is gathered meanwhile
      tc_store_a<H>(t_ahi, t_alo, h);
      signal_a();
      const int64_t next = pair + gridDim.x;
      if (!TMAG && next < n_pairs) {
        int64_t nb, ne_;
        tile_rows(2 * next + g, nb, ne_);
        tc_gather<H, MODE>(a, nb + trow, nb + trow < ne_, 0, v, fwd_e_pol(0));
      }
      wait_d();
      const long long t_out0 = PROF ? clock64() : 0;
      if (FUSED) {  // y = D + b into this slot's output tile, for the reducer warp
        const float* bo = sbias + (a.k + 1) * H;
        ptx::mbar_wait(&y_empty[g], py ^ 1);  // previous tile of this slot consumed
        py ^= 1;
        uint8_t* yt = ytile + (size_t)g * 128 * H * 4;
        tc_load_d<H>(t_d, bo, h);  // h is dead after the output projection's A store
#pragma unroll
        for (int j = 0; j < H / 4; ++j)
          *reinterpret_cast<float4*>(yt + ytile_off<H>(trow, j)) =
              make_float4(h[4 * j], h[4 * j + 1], h[4 * j + 2], h[4 * j + 3]);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&y_full[g]);
      } else if (DEC) {  // y = D + b + x W_skip on the first out_dim columns
        float p[16];
        ptx::tmem_ld16(t_d, p);
        ptx::tmem_wait_ld();
        float y[8];
#pragma unroll
        for (int o = 0; o < 8; ++o) y[o] = p[o] + sbias[(a.k + 1) * H + o];
        if (valid) {
          const float4* xr = reinterpret_cast<const float4*>(a.x + row * H);
#pragma unroll 4
          for (int q = 0; q < H / 4; ++q) {
            const float4 xv = __ldg(xr + q);
            const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int o = 0; o < 8; ++o) y[o] = fmaf(xs[u], senc[(4 * q + u) * 8 + o], y[o]);
          }
#pragma unroll
          for (int o = 0; o < 8; ++o)
            if (o < a.out_dim) a.out[row * a.out_dim + o] = y[o];
        }
      } else if (ENC) {  // y = D + b + x W_skip, output LayerNorm (mlp_generic.cuh forward)
        float xf[8];
        {
          const float* f = a.e_in + row * a.in_dim;
#pragma unroll
          for (int i = 0; i < 8; ++i) xf[i] = (valid && i < a.in_dim) ? __ldg(f + i) : 0.f;
        }
        tc_load_d<H>(t_d, sbias + (a.k + 1) * H, h);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < a.in_dim) {
#pragma unroll
            for (int j = 0; j < H; j += 2)
              f2_put(h + j, f2_fma(make_float2(xf[i], xf[i]), f2_pair(senc + i * H + j), f2_pair(h + j)));
          }
        }
        if (a.enc_ln) {
          ln0_tree<H>(h);
#pragma unroll
          for (int j = 0; j < H; j += 2)
            f2_put(h + j, f2_fma(f2_pair(h + j), f2_pair(senc + 8 * H + j), f2_pair(senc + 9 * H + j)));
        }
        if (valid) {
#pragma unroll
          for (int j = 0; j < H / 8; ++j) ptx::stg256(a.out + row * H + 8 * j, h + 8 * j);
        }
      } else {  // stream y = D + b straight to global, 32 columns at a time
        const float* bo = sbias + (a.k + 1) * H;
#pragma unroll
        for (int c = 0; c < H; c += 32) {
          float p[32];
          ptx::tmem_ld32(t_d + c, p);
          ptx::tmem_wait_ld();
          if (valid) {
#pragma unroll
            for (int j = 0; j < 32; ++j) p[j] += bo[c + j];
#pragma unroll
            for (int j = 0; j < 4; ++j) ptx::stg256(a.out + row * H + c + 8 * j, p + 8 * j);
          }
        }
      }
      if (PROF) e_out += (unsigned long long)(clock64() - t_out0);
    }
    if (PROF && warp == 0 && lane == 0) {
      atomicAdd(a.prof + kFwdProfEpiTotal, (unsigned long long)(clock64() - e_t0));
      atomicAdd(a.prof + kFwdProfEpiD, e_d);
      atomicAdd(a.prof + kFwdProfEpiAE, e_ae);
      atomicAdd(a.prof + kFwdProfEpiSig, e_sig);
      atomicAdd(a.prof + kFwdProfEpiLd, e_ld);
      atomicAdd(a.prof + kFwdProfEpiMath, e_math);
      atomicAdd(a.prof + kFwdProfEpiStA, e_sta);
      atomicAdd(a.prof + kFwdProfEpiGather, e_in);
      atomicAdd(a.prof + kFwdProfEpiOut, e_out);
    }
  } else if (warp == 8) {
    // ------------------------------------------------------------ MMA issuer
    // warp-uniform TMEM base (uniform registers; no per-MMA waterfall loop)
    const uint32_t tm = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile uint32_t*>(tmem_base_slot), 0);
    {  // all 32 lanes run the schedule; mma/commit elect one lane
      constexpr uint32_t idesc = ptx::idesc_tf32(128, H);
      int ws = 0;
      uint32_t wph = 0, pa[2] = {0, 0};
      unsigned long long i_a = 0, i_w = 0, i_m = 0;
      const long long i_t0 = PROF ? clock64() : 0;
      for (int64_t pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
        for (int j = 0; j < n_chunks; ++j) {
          const int l = j < nseg ? 0 : j - nseg + 1;
          const int c = j < nseg ? j : 0;
          const bool last_chunk = (l > 0) || (c == nseg - 1);
          long long t0 = PROF ? clock64() : 0;
          ptx::mbar_wait(&w_full[ws], wph);
          ptx::tc_fence_after();
          if (PROF) i_w += (unsigned long long)(clock64() - t0);
          const uint32_t bbase = ptx::smem_u32(wring + (size_t)ws * Cfg::CHUNK_FLOATS);
          for (int s = 0; s < 2; ++s) {
            if (PROF) t0 = clock64();
            ptx::mbar_wait(&a_full[s], pa[s]);
            pa[s] ^= 1;
            ptx::tc_fence_after();
            if (PROF) {
              const long long t1 = clock64();
              i_a += (unsigned long long)(t1 - t0);
              t0 = t1;
            }
            const uint32_t slot = ptx::opaque(tm + s * Cfg::SLOT_COLS);
            const uint64_t d0 = ptx::opaque64(ptx::smem_desc(bbase, Cfg::LBO, Cfg::SBO));
#pragma unroll
            for (int ks = 0; ks < H / 8; ++ks) {
              const uint64_t b_hi = d0 + (uint64_t)((ks * 2 * Cfg::LBO) >> 4);
              const uint64_t b_lo = b_hi + (uint64_t)(Cfg::LO_OFF >> 4);
              ptx::mma_tf32_ts_w(slot + 2 * H, slot + 8 * ks, b_hi, idesc, (c > 0 || ks > 0) ? 1u : 0u);
              ptx::mma_tf32_ts_w(slot + 2 * H, slot + 8 * ks, b_lo, idesc, 1u);
              ptx::mma_tf32_ts_w(slot + 2 * H, slot + H + 8 * ks, b_hi, idesc, 1u);
            }
            ptx::mma_commit_w(last_chunk ? &d_full[s] : &a_empty[s]);
            if (PROF) i_m += (unsigned long long)(clock64() - t0);
          }
          ptx::mma_commit_w(&w_empty[ws]);
          if (++ws == STAGES) {
            ws = 0;
            wph ^= 1;
          }
        }
      }
      if (PROF && lane == 0) {
        atomicAdd(a.prof + kFwdProfIssTotal, (unsigned long long)(clock64() - i_t0));
        atomicAdd(a.prof + kFwdProfIssA, i_a);
        atomicAdd(a.prof + kFwdProfIssW, i_w);
        atomicAdd(a.prof + kFwdProfIssMma, i_m);
      }
    }
  } else if (FUSED && warp >= 10) {
    // ------------------------------------------------------------ reducer of slot g (warps 10, 11)
    // e' rows to HBM (coalesced: the lanes cover one row) and the segment sums
    // a[i] = sum_p inv[p] e'[p] in slot order (fmaf chain from 0, as
    // aggregate_kernel): each receiver segment lies inside one tile.
    const int g = warp - 10;
    constexpr int CPL = H / 32;  // columns per lane
    const uint8_t* yt = ytile + (size_t)g * 128 * H * 4;
    uint32_t pf = 0;
    for (int64_t pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
      int64_t tb, te;
      tile_rows(2 * pair + g, tb, te);
      const int n = (HGNN_EXP & 128) ? 0 : (int)(te - tb);
      ptx::mbar_wait(&y_full[g], pf);
      pf ^= 1;
      float acc[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) acc[q] = 0.f;
      for (int r0 = 0; r0 < n; r0 += 32) {
        const int rr = r0 + lane;
        const int32_t d_l = rr < n ? __ldg(a.dst + tb + rr) : -1;
        const int32_t dn_l = rr + 1 < n ? __ldg(a.dst + tb + rr + 1) : -1;
        const float w_l = rr < n ? __ldg(a.inv + tb + rr) : 0.f;
        const int cnt = n - r0 < 32 ? n - r0 : 32;
        for (int i = 0; i < cnt; ++i) {
          const int r = r0 + i;
          const int32_t d = __shfl_sync(0xffffffffu, d_l, i);
          const int32_t dn = __shfl_sync(0xffffffffu, dn_l, i);
          const float w = __shfl_sync(0xffffffffu, w_l, i);
          float* eo = (a.out && !(HGNN_EXP & 64)) ? a.out + (tb + r) * H + CPL * lane : nullptr;  // nullptr: e' not stored (dead)
          if (CPL == 2) {
            const float2 y = *reinterpret_cast<const float2*>(yt + ytile_off<H>(r, lane / 2) + 8 * (lane & 1));
            if (eo) {
              if (HGNN_FWD_STREAM_HINT)
                asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(eo), "f"(y.x), "f"(y.y),
                             "l"(stream_pol)
                             : "memory");
              else
                *reinterpret_cast<float2*>(eo) = y;
            }
            acc[0] = fmaf(w, y.x, acc[0]);
            acc[CPL - 1] = fmaf(w, y.y, acc[CPL - 1]);
          } else {
            const float y = *reinterpret_cast<const float*>(yt + ytile_off<H>(r, lane / 4) + 4 * (lane & 3));
            if (eo) *eo = y;
            acc[0] = fmaf(w, y, acc[0]);
          }
          if (dn != d) {  // last slot of receiver d's segment
            float* ag = a.agg + (int64_t)d * H + CPL * lane;
            if (CPL == 2) *reinterpret_cast<float2*>(ag) = make_float2(acc[0], acc[CPL - 1]);
            else *ag = acc[0];
#pragma unroll
            for (int q = 0; q < CPL; ++q) acc[q] = 0.f;
          }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&y_empty[g]);
    }
  } else {
    // ------------------------------------------------------------ weight loader (warp 9; 10-11 idle)
    if (TMAG && warp == 9) {
      // Weight chunks (lane 0) and the input-row gathers (all lanes), polled
      // in turn: a gather of segment c for slot g is issued once the slot's
      // buffer is read (per slot in its epilogue's consumption order: per
      // pair, per segment); lane L gathers rows 4L .. 4L + 3 of the
      // tile (indices clamped to its last row) as two tile::gather4 (columns
      // 0-31 / 32-63), and expect_tx covers the groups issued.
      int ws = 0, wj = 0, gc[2] = {0, 0};
      uint32_t wph = 0, pge[2] = {0, 0};
      int64_t wp = blockIdx.x, gp[2] = {blockIdx.x, blockIdx.x};
      // prepared next gather per slot: row groups, this lane's 4 row indices, e rows?
      int ngr[2] = {0, 0}, nix[2][4];
      bool nes[2] = {false, false};
      auto prep = [&](int gg) {
        if (gp[gg] >= n_pairs) return;
        int64_t tb, te;
        tile_rows(2 * gp[gg] + gg, tb, te);
        const int n = (int)(te - tb);
        ngr[gg] = (n + 3) / 4;
        nes[gg] = FACT || gc[gg] == 2;  // the slots' own e rows
        const int32_t* ix = gc[gg] == 0 ? a.src : a.dst;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = 4 * lane + i < n ? 4 * lane + i : n - 1;
          nix[gg][i] = (nes[gg] || lane >= ngr[gg]) ? (int)(tb + r) : __ldg(ix + tb + r);
        }
      };
      prep(0);
      prep(1);
      const long long t0 = clock64();
      while (wp < n_pairs || gp[0] < n_pairs || gp[1] < n_pairs) {
        bool idle = true;  // nothing issued this round: back off (the warp shares its issue slots with an epilogue warp)
        if (wp < n_pairs) {
          const bool ok = __shfl_sync(0xffffffffu, lane == 0 ? (int)ptx::mbar_test_wait(&w_empty[ws], wph ^ 1) : 0, 0);
          if (ok) {
            idle = false;
            if (lane == 0) {
              ptx::mbar_arrive_expect_tx(&w_full[ws], Cfg::CHUNK_BYTES);
              ptx::bulk_g2s(wring + (size_t)ws * Cfg::CHUNK_FLOATS, a.chunks + (size_t)wj * Cfg::CHUNK_FLOATS,
                            Cfg::CHUNK_BYTES, &w_full[ws]);
            }
            if (++ws == STAGES) {
              ws = 0;
              wph ^= 1;
            }
            if (++wj == n_chunks) {
              wj = 0;
              wp += gridDim.x;
            }
          }
        }
#pragma unroll
        for (int gg = 0; gg < 2; ++gg) {  // per slot: its own cursor (pair gp[gg], segment gc[gg])
          if (gp[gg] >= n_pairs) continue;
          const bool ok =
              __shfl_sync(0xffffffffu, lane == 0 ? (int)ptx::mbar_test_wait(&gx_empty[gg], pge[gg] ^ 1) : 0, 0);
          if (!ok) continue;
          idle = false;
          pge[gg] ^= 1;
          if (lane == 0) ptx::mbar_arrive_expect_tx(&gx_full[gg], (uint32_t)ngr[gg] * 2 * 512);
          __syncwarp();
          if (lane < ngr[gg]) {
            uint8_t* dst = gx + (size_t)gg * (128 * H * 4) + lane * 512;
            const CUtensorMap* map = nes[gg] ? tme : tmx;
            tma_gather4(dst, map, 0, nix[gg][0], nix[gg][1], nix[gg][2], nix[gg][3], &gx_full[gg]);
            tma_gather4(dst + 128 * 128, map, 32, nix[gg][0], nix[gg][1], nix[gg][2], nix[gg][3], &gx_full[gg]);
          }
          if (++gc[gg] == nseg) {
            gc[gg] = 0;
            gp[gg] += gridDim.x;
          }
          prep(gg);  // the slot's next gather: its indices load while the buffer is in use
        }
        if (idle) __nanosleep(HGNN_PRODUCER_SLEEP_NS);
        if (clock64() - t0 > 40000000000ll) {  // watchdog, as mbar_wait
          if (lane == 0) printf("hgnn_b200: gather producer timeout (block %d)\n", (int)blockIdx.x);
          __trap();
        }
      }
    } else if (!TMAG && warp == 9 && lane == 0) {
      int ws = 0;
      uint32_t wph = 0;
      for (int64_t pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
        for (int j = 0; j < n_chunks; ++j) {
          ptx::mbar_wait(&w_empty[ws], wph ^ 1);
          ptx::mbar_arrive_expect_tx(&w_full[ws], Cfg::CHUNK_BYTES);
          ptx::bulk_g2s(wring + (size_t)ws * Cfg::CHUNK_FLOATS, a.chunks + (size_t)j * Cfg::CHUNK_FLOATS,
                        Cfg::CHUNK_BYTES, &w_full[ws]);
          if (++ws == STAGES) {
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
    ptx::tmem_dealloc<Cfg::TMEM_COLS>(tmem);
  }
}

template <int H, int MODE, bool PROF>
__global__ void __launch_bounds__(TcCfg<H>::THREADS, 1) mlp_tc_forward_kernel(TcFwdArgs a) {
  mlp_tc_forward_body<H, MODE, PROF, false>(a, nullptr, nullptr);
}
// fused edge modes with TMA-gathered input rows; tmx over x (rows x H),
// tme over e (N_e x H): 2-D fp32, box 32 x 1, 128-byte swizzle
template <int H, int MODE>
__global__ void __launch_bounds__(TcCfg<H>::THREADS, 1)
    mlp_tc_forward_tma_kernel(TcFwdArgs a, const __grid_constant__ CUtensorMap tmx,
                              const __grid_constant__ CUtensorMap tme) {
  mlp_tc_forward_body<H, MODE, false, true>(a, &tmx, &tme);
}

}  // namespace hgnn_b200
