// Tensor-core processor-MLP backward, split-row epilogue (sm_100a, H = 64).
//
// Same algorithm, tensor-core schedule and results as mlp_tc_backward_kernel
// (mlp_tc_bwd.cuh): per 128-row tile, recompute the forward (3xTF32 tcgen05,
// A operands and accumulators in TMEM), then walk the linears in reverse with
// dX = d W^T on the tensor cores and dW += h^T d as one N = 128 SS MMA per
// 8-row K-step, staged in SMEM. What changes is the epilogue: 16 epilogue warps
// instead of 8, reading / writing TMEM with the 16x256b shape, so a thread owns
// two rows x 16 columns (4 threads per row) instead of one full row:
//   * twice the warps per SM sub-partition to hide the LDTM / MMA / load
//     latencies of the serial per-linear chain (the 1-row-per-thread kernel is
//     latency-bound: tensor pipe ~24 %, issue ~30 %);
//   * half the per-thread work and code per linear (the row sums of LayerNorm
//     close with two shuffles inside the row's thread quad);
//   * two independent rows per thread (instruction-level parallelism).
// Thread layout (measured, tc_ptx.cuh tmem_ld16x256_x8): warp w, slot
// g = w / 8, quarter q = w % 4 (its TMEM lane quarter), half hb = (w / 4) % 2;
// the warp covers tile rows r0 = 32 q + 16 hb .. r0 + 15; thread t holds rows
// r0 + t/4 and r0 + t/4 + 8, columns 8 j + 2 (t % 4) + {0, 1}, j = 0..7, as
// v[4 j + 0..1] (row a) and v[4 j + 2..3] (row b).
// Warps 16 (dX MMA issuer), 17 (dW MMA issuer), 18 (weight loader), 19 idle.
#pragma once

#include "mlp_tc_bwd.cuh"

namespace hgnn_b200 {

struct TcBwdCsCfg {
  static constexpr int H = 64;
  static constexpr int THREADS = 640;  // 4 epilogue warpgroups + 1 control warpgroup
  static constexpr int EPI_WARPS = 16;
  static constexpr size_t OFF_STAGE = TcBwdCfg::OFF_STAGE;
  static constexpr size_t OFF_BARS = TcBwdCfg::OFF_BARS;
  static constexpr size_t OFF_DBP = OFF_BARS + 256;                     // db partials [4][16][64]
  static constexpr size_t OFF_BIAS = OFF_DBP + 4 * EPI_WARPS * 64 * 4;  // biases (k+2) x 64
  static constexpr size_t SMEM = OFF_BIAS + 18 * 64 * 4 + 1024;
};

// Rows a / b of this thread from a row-major H = 64 matrix: 8 float2 each.
__device__ __forceinline__ void cs_load_rows(const float* pa, const float* pb, int cp, float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 x = pa ? __ldg(reinterpret_cast<const float2*>(pa + 8 * j + 2 * cp)) : make_float2(0.f, 0.f);
    const float2 y = pb ? __ldg(reinterpret_cast<const float2*>(pb + 8 * j + 2 * cp)) : make_float2(0.f, 0.f);
    v[4 * j] = x.x;
    v[4 * j + 1] = x.y;
    v[4 * j + 2] = y.x;
    v[4 * j + 3] = y.y;
  }
}

// A <- [hi | lo] split of v (16x256b layout), 32 columns per store (register footprint).
__device__ __forceinline__ void cs_store_a(uint32_t t_hi, uint32_t t_lo, const float (&v)[32]) {
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    float hi[16], lo[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      hi[i] = ptx::tf32_hi(v[16 * hf + i]);
      lo[i] = v[16 * hf + i] - hi[i];
    }
    ptx::tmem_st16x256_x4(t_hi + 32 * hf, hi);
    ptx::tmem_st16x256_x4(t_lo + 32 * hf, lo);
  }
}

// Row sums of rows a / b over the 4 threads of each row (fixed order; the
// butterfly gives all four threads the same bits: fp addition commutes).
__device__ __forceinline__ void cs_row_sums(float& sa, float& sb) {
  sa += __shfl_xor_sync(0xffffffffu, sa, 1);
  sb += __shfl_xor_sync(0xffffffffu, sb, 1);
  sa += __shfl_xor_sync(0xffffffffu, sa, 2);
  sb += __shfl_xor_sync(0xffffffffu, sb, 2);
}

// Parameter-free LayerNorm of rows a / b in place (kernels.cpp:81-94); inverse std out.
__device__ __forceinline__ void cs_ln0(float (&u)[32], float& inv_a, float& inv_b) {
  float sa0 = 0.f, sa1 = 0.f, sb0 = 0.f, sb1 = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sa0 += u[4 * j];
    sa1 += u[4 * j + 1];
    sb0 += u[4 * j + 2];
    sb1 += u[4 * j + 3];
  }
  float sa = sa0 + sa1, sb = sb0 + sb1;
  cs_row_sums(sa, sb);
  const float ma = sa * (1.0f / 64), mb = sb * (1.0f / 64);
  float qa0 = 0.f, qa1 = 0.f, qb0 = 0.f, qb1 = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float d0 = u[4 * j] - ma, d1 = u[4 * j + 1] - ma, d2 = u[4 * j + 2] - mb, d3 = u[4 * j + 3] - mb;
    qa0 = fmaf(d0, d0, qa0);
    qa1 = fmaf(d1, d1, qa1);
    qb0 = fmaf(d2, d2, qb0);
    qb1 = fmaf(d3, d3, qb1);
  }
  float qa = qa0 + qa1, qb = qb0 + qb1;
  cs_row_sums(qa, qb);
  inv_a = ptx::rsqrt_fast(qa * (1.0f / 64) + 1e-12f);
  inv_b = ptx::rsqrt_fast(qb * (1.0f / 64) + 1e-12f);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    u[4 * j] = (u[4 * j] - ma) * inv_a;
    u[4 * j + 1] = (u[4 * j + 1] - ma) * inv_a;
    u[4 * j + 2] = (u[4 * j + 2] - mb) * inv_b;
    u[4 * j + 3] = (u[4 * j + 3] - mb) * inv_b;
  }
}

// Byte offset of the 8-byte piece (columns mn, mn + 1) of staging row `row`
// in a 16 KB MN-major SWIZZLE_128B_BASE32B operand (st_off in mlp_tc_bwd.cuh).
__device__ __forceinline__ uint32_t cs_st_off(int mn, int row) {
  return st_off(mn >> 2, row) + (uint32_t)((mn & 2) << 2);
}

// This thread's two rows of [v_hi | v_lo] (128 MN entries each) into a staging operand.
__device__ __forceinline__ void cs_stage_rows(uint8_t* base, int row_a, int cp, const float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int mn = 8 * j + 2 * cp;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float x0 = v[4 * j + 2 * r], x1 = v[4 * j + 2 * r + 1];
      const float h0 = ptx::tf32_hi_stage(x0), h1 = ptx::tf32_hi_stage(x1);
      const int row = row_a + 8 * r;
      *reinterpret_cast<float2*>(base + cs_st_off(mn, row)) = make_float2(h0, h1);
      *reinterpret_cast<float2*>(base + cs_st_off(64 + mn, row)) = make_float2(x0 - h0, x1 - h1);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(TcBwdCsCfg::THREADS, 1) mlp_tc_backward_cs_kernel(TcBwdArgs a) {
  using Cfg = TcBwdCfg;
  using Cs = TcBwdCsCfg;
  constexpr int H = Cfg::H;
  constexpr bool FACT = MODE == kEdgeFact;
  constexpr bool EDGE = MODE != kNodeInput;
  constexpr int nseg = MODE == kEdgeInput ? 3 : (MODE == kNodeInput ? 2 : 1);
  constexpr int in_dim = (MODE == kNodeInput ? 2 : 3) * H;
  constexpr int seg0 = FACT ? 2 : 0;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* wring = reinterpret_cast<float*>(smem);
  uint8_t* stage = smem + Cs::OFF_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cs::OFF_BARS);
  uint64_t* w_full = bars;
  uint64_t* w_empty = w_full + Cfg::WSTAGES;
  uint64_t* a_full = w_empty + Cfg::WSTAGES;  // [2], 8 epilogue warps per slot
  uint64_t* a_empty = a_full + 2;
  uint64_t* d_full = a_empty + 2;
  uint64_t* st_full = d_full + 2;             // [NSTAGE], 2 warps per staging buffer
  uint64_t* st_empty = st_full + Cfg::NSTAGE;  // [2][NSTAGE]
  uint64_t* dw_full = st_empty + 2 * Cfg::NSTAGE;
  uint64_t* dw_empty = dw_full + 2;            // 16 epilogue warps
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(dw_empty + 2);
  float* dbp = reinterpret_cast<float*>(smem + Cs::OFF_DBP);
  float* sbias = reinterpret_cast<float*>(smem + Cs::OFF_BIAS);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int K = a.k;
  const int n_w = 2 * nseg + 2 * K + 1;
  const int n_dw = K + 1 + nseg;
  const int64_t n_tiles = (a.n_rows + 127) / 128;
  const int64_t n_pairs = (n_tiles + 1) / 2;
  const int64_t n_par = mlp_param_count(in_dim, H, K);

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::WSTAGES; ++s) {
      ptx::mbar_init(&w_full[s], 1);
      ptx::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&a_full[s], 8);
      ptx::mbar_init(&a_empty[s], 1);
      ptx::mbar_init(&d_full[s], 1);
    }
    for (int s = 0; s < Cfg::NSTAGE; ++s) {
      ptx::mbar_init(&st_full[s], 2);
      ptx::mbar_init(&st_empty[s], 1);
      ptx::mbar_init(&st_empty[Cfg::NSTAGE + s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&dw_full[s], 1);
      ptx::mbar_init(&dw_empty[s], Cs::EPI_WARPS);
    }
    ptx::fence_mbarrier_init();
  }
  for (int i = threadIdx.x; i < (K + 2) * H; i += blockDim.x)
    sbias[i] = __ldg(a.params + mlp_b_offset(i / H, in_dim, H) + (i % H));
  if (warp == 16) ptx::tmem_alloc<512>(tmem_base_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_base_slot;

  static_assert(512 * 112 + 128 * 32 <= Cs::THREADS * 96, "setmaxnreg exceeds the CTA register pool");
  if (warp < 16) ptx::regs_inc<112>();
  else ptx::regs_dec<32>();

  if (warp < 16) {
    // ================================================================ epilogue
    const int g = warp / 8, q = warp % 4, hb = (warp / 4) % 2;
    const int r0 = 32 * q + 16 * hb;
    const int cp = lane % 4, rg = lane / 4;
    const int ra = r0 + rg;  // tile rows of this thread: ra, ra + 8
    const uint32_t t_ahi = tmem + g * Cfg::SLOT_COLS + ((uint32_t)r0 << 16);
    const uint32_t t_alo = t_ahi + H;
    const uint32_t t_d = t_ahi + 2 * H;
    const uint32_t t_dw = tmem + Cfg::DW_COL + ((uint32_t)(32 * q) << 16);  // 32x32b drain (lane quarter)
    // per-CTA scratch of this slot: t_l as [l][j][row][t % 4] float2, inv_std as [l][row]
    // (recomputed from the kernel parameters at each use: keeps them out of the
    // epilogue's register budget)
    auto scr_t = [&](int l) -> float2* {
      return reinterpret_cast<float2*>(a.scratch) + (((int64_t)blockIdx.x * 2 + g) * K + (l - 1)) * 8 * 128 * 4;
    };
    auto scr_inv = [&](int l) -> float* {
      return a.scratch + (int64_t)gridDim.x * 2 * K * 16 * 128 * 4 + (((int64_t)blockIdx.x * 2 + g) * K + (l - 1)) * 128;
    };
    const int sbuf = 4 * g + q;  // staging buffer of (slot, quarter) inside a job
    uint32_t pe = 0, pd = 0;
    int job = 0;

    auto wait_d = [&]() {
      ptx::mbar_wait(&d_full[g], pd);
      pd ^= 1;
      ptx::tc_fence_after();
    };
    auto signal_a = [&]() {
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&a_full[g]);
    };
    // D (+ bias of linear l, or none) of rows a / b
    auto load_d = [&](int l, float (&y)[32]) {
      ptx::tmem_ld16x256_x8(t_d, y);
      ptx::tmem_wait_ld();
      if (l >= 0) {
        const float* b = sbias + l * H + 2 * cp;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          y[4 * j] += b[8 * j];
          y[4 * j + 1] += b[8 * j + 1];
          y[4 * j + 2] += b[8 * j];
          y[4 * j + 3] += b[8 * j + 1];
        }
      }
    };
    // Drain dW job jf (single 128-column accumulator): this warp's lane
    // quarter, output columns [16 k, 16 k + 16), k = warp / 4; lanes < 64 hold
    // h_hi x (d_hi | d_lo) = hh | hl, lanes >= 64 h_lo x (d_hi | d_lo) = lh | ll.
    auto flush = [&](int jf) {
      const int jj = (int)(jf % n_dw);
      const int lin = jj <= K ? K + 1 - jj : 0;
      const int rowbase = jj <= K ? 0 : (jj - K - 1 + seg0) * H;
      const bool with_db = jj <= K + 1;
      ptx::mbar_wait(&dw_full[0], (uint32_t)(jf & 1));
      ptx::tc_fence_after();
      const int c0 = 16 * (warp / 4);
      const int feat = 32 * (q & 1) + lane;
      float* gpart0 = a.grad_partial + (int64_t)blockIdx.x * 2 * n_par;  // hh + hl, db
      float* gw = gpart0 + (q < 2 ? 0 : n_par) + mlp_w_offset(lin, in_dim, H) + (int64_t)(rowbase + feat) * H + c0;
      const uint64_t keep = ptx::policy_evict_last();
      float p0[16], p1[16];
      ptx::tmem_ld16(t_dw + c0, p0);
      ptx::tmem_ld16(t_dw + 64 + c0, p1);
      float dbs = 0.f;
      if (with_db && warp < 2) {  // bias gradient: fixed-order sum of the 16 warp partials
        const float* db = dbp + (jf % 4) * Cs::EPI_WARPS * 64 + 32 * warp + lane;
#pragma unroll
        for (int w = 0; w < Cs::EPI_WARPS; ++w) dbs += db[w * 64];
      }
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&dw_empty[0]);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        ptx::red_add4_hint(gw + 4 * j, p0[4 * j] + p1[4 * j], p0[4 * j + 1] + p1[4 * j + 1],
                           p0[4 * j + 2] + p1[4 * j + 2], p0[4 * j + 3] + p1[4 * j + 3], keep);
      if (with_db && warp < 2)
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(gpart0 + mlp_b_offset(lin, in_dim, H) + 32 * warp + lane),
                     "f"(dbs)
                     : "memory");
    };
    // Stage this thread's rows of (h, d) for the dW MMAs of job `job`; the
    // accumulator's previous job is drained first.
    auto stage_chunk = [&](const float (&hin)[32], const float (&d)[32]) {
      if (job >= 1) flush(job - 1);
      const int64_t gi = (int64_t)job * 8 + sbuf;
      stage_acquire(st_empty, gi);
      uint8_t* sb = stage + (size_t)(gi % Cfg::NSTAGE) * Cfg::STAGE_BYTES;
      cs_stage_rows(sb, 16 * hb + rg, cp, hin);
      cs_stage_rows(sb + 16384, 16 * hb + rg, cp, d);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&st_full[gi % Cfg::NSTAGE]);
    };
    // Column sums of d over this warp's 16 rows: rows a + b, then a
    // transpose-reduce over the row-group bits of the lane (fixed order); lane
    // ends with columns 8 rg + 2 cp + {0, 1}.
    auto write_db = [&](const float (&d)[32]) {
      float x[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        x[2 * j] = d[4 * j] + d[4 * j + 2];
        x[2 * j + 1] = d[4 * j + 1] + d[4 * j + 3];
      }
#pragma unroll
      for (int w = 16, bit = 16; w >= 4; w /= 2, bit /= 2) {  // lane bits 16, 8, 4 = j bits 2, 1, 0
        const bool up = lane & bit;
#pragma unroll
        for (int i = 0; i < w / 2; ++i) {
          const float send = up ? x[i] : x[w / 2 + i];
          const float kept = up ? x[w / 2 + i] : x[i];
          x[i] = kept + __shfl_xor_sync(0xffffffffu, send, bit);
        }
      }
      float* dst = dbp + ((job % 4) * Cs::EPI_WARPS + warp) * 64 + 8 * rg + 2 * cp;
      dst[0] = x[0];
      dst[1] = x[1];
    };
    // input segment c of rows a / b (global row indices ga, gb)
    auto gather = [&](int64_t ga, int64_t gb, bool va, bool vb, int c, float (&v)[32]) {
      const float* pa = nullptr;
      const float* pb = nullptr;
      if (kExp & 16) va = vb = false;
      if (FACT) {
        pa = va ? a.e_in + ga * H : nullptr;
        pb = vb ? a.e_in + gb * H : nullptr;
      } else if (EDGE) {
        if (c == 0) {
          pa = va ? a.x + (int64_t)__ldg(a.src + ga) * H : nullptr;
          pb = vb ? a.x + (int64_t)__ldg(a.src + gb) * H : nullptr;
        } else if (c == 1) {
          pa = va ? a.x + (int64_t)__ldg(a.dst + ga) * H : nullptr;
          pb = vb ? a.x + (int64_t)__ldg(a.dst + gb) * H : nullptr;
        } else {
          pa = va ? a.e_in + ga * H : nullptr;
          pb = vb ? a.e_in + gb * H : nullptr;
        }
      } else {
        const float* base = c == 0 ? a.a : a.x;
        pa = va ? base + ga * H : nullptr;
        pb = vb ? base + gb * H : nullptr;
      }
      cs_load_rows(pa, pb, cp, v);
    };

    for (int64_t pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
      const int64_t tile0 = (2 * pair + g) * 128;
      const int64_t ga = tile0 + ra, gb = ga + 8;
      const bool va = ga < a.n_rows, vb = gb < a.n_rows;
      float h[32];
      // ---------------------------------------------- forward recompute
#pragma unroll 1
      for (int c = 0; c < nseg; ++c) {
        if (c > 0) {
          ptx::mbar_wait(&a_empty[g], pe);
          pe ^= 1;
          ptx::tc_fence_after();
        }
        gather(ga, gb, va, vb, c, h);
        cs_store_a(t_ahi, t_alo, h);
        signal_a();
      }
      if (FACT) {  // h = P_s[src] + P_d[dst]
        const float* psa = va ? a.proj + (int64_t)__ldg(a.src + ga) * 2 * H : nullptr;
        const float* psb = vb ? a.proj + (int64_t)__ldg(a.src + gb) * 2 * H : nullptr;
        const float* pda = va ? a.proj + (int64_t)__ldg(a.dst + ga) * 2 * H + H : nullptr;
        const float* pdb = vb ? a.proj + (int64_t)__ldg(a.dst + gb) * 2 * H + H : nullptr;
        float w2[32];
        cs_load_rows(psa, psb, cp, h);
        cs_load_rows(pda, pdb, cp, w2);
#pragma unroll
        for (int i = 0; i < 32; ++i) h[i] += w2[i];
      }
      wait_d();
      if (FACT) {
        float u[32];
        load_d(0, u);
#pragma unroll
        for (int i = 0; i < 32; ++i) h[i] = u[i] + h[i];  // (D + b0) + proj
      } else {
        load_d(0, h);
      }
      for (int l = 1; l <= K; ++l) {
        cs_store_a(t_ahi, t_alo, h);
        signal_a();
        wait_d();
        float u[32];
        load_d(l, u);
        float inv_a, inv_b;
        cs_ln0(u, inv_a, inv_b);
        float2* st = scr_t(l);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          st[(j * 128 + ra) * 4 + cp] = make_float2(u[4 * j], u[4 * j + 1]);
          st[(j * 128 + ra + 8) * 4 + cp] = make_float2(u[4 * j + 2], u[4 * j + 3]);
        }
        if (cp == 0) {
          scr_inv(l)[ra] = inv_a;
          scr_inv(l)[ra + 8] = inv_b;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) h[i] += elu_fast(u[i]);
      }
      // ---------------------------------------------- backward
      float dh[32];
      if (EDGE) {  // d_y = de + inv_d * d_a[dst] (model.cpp:354-360)
        const float sa = va ? __ldg(a.inv_deg + ga) : 0.f, sb = vb ? __ldg(a.inv_deg + gb) : 0.f;
        float da[32], de[32];
        cs_load_rows(va ? a.d_a + (int64_t)__ldg(a.dst + ga) * H : nullptr,
                     vb ? a.d_a + (int64_t)__ldg(a.dst + gb) * H : nullptr, cp, da);
        cs_load_rows((va && a.de_in) ? a.de_in + ga * H : nullptr, (vb && a.de_in) ? a.de_in + gb * H : nullptr, cp,
                     de);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          dh[4 * j] = fmaf(sa, da[4 * j], de[4 * j]);
          dh[4 * j + 1] = fmaf(sa, da[4 * j + 1], de[4 * j + 1]);
          dh[4 * j + 2] = fmaf(sb, da[4 * j + 2], de[4 * j + 2]);
          dh[4 * j + 3] = fmaf(sb, da[4 * j + 3], de[4 * j + 3]);
        }
      } else {
        cs_load_rows(va ? a.d_out + ga * H : nullptr, vb ? a.d_out + gb * H : nullptr, cp, dh);
      }
#pragma unroll 1
      for (int jb = 0; jb < K + 1 + nseg; ++jb) {
        const int c = jb - (K + 1);
        if (jb >= 1 && jb <= K) {
          const int l = K + 1 - jb;
          const float2* st = scr_t(l);
          const float inv_a = scr_inv(l)[ra], inv_b = scr_inv(l)[ra + 8];
          ptx::tmem_st16x256_x8(t_d, dh);  // residual d_h pre-loaded into the accumulator
          // pass 1: ELU adjoint, residual rebuild, LayerNorm-adjoint sums
          // (t_l is read twice, the second time from L1: keeps the register
          // footprint of the 104-register epilogue)
          float s_a0 = 0.f, s_a1 = 0.f, s_b0 = 0.f, s_b1 = 0.f, x_a0 = 0.f, x_a1 = 0.f, x_b0 = 0.f, x_b1 = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float2 ta = st[(j * 128 + ra) * 4 + cp];
            const float2 tb = st[(j * 128 + ra + 8) * 4 + cp];
            const float tv[4] = {ta.x, ta.y, tb.x, tb.y};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = 4 * j + e;
              const float ex = ptx::exp_fast(tv[e]);
              h[i] -= tv[e] > 0.f ? tv[e] : ex - 1.0f;          // h_{l-1}
              dh[i] = dh[i] * (tv[e] > 0.f ? 1.0f : ex);         // elu', kernels.cpp:68-71
            }
            s_a0 += dh[4 * j];
            s_a1 += dh[4 * j + 1];
            s_b0 += dh[4 * j + 2];
            s_b1 += dh[4 * j + 3];
            x_a0 = fmaf(dh[4 * j], tv[0], x_a0);
            x_a1 = fmaf(dh[4 * j + 1], tv[1], x_a1);
            x_b0 = fmaf(dh[4 * j + 2], tv[2], x_b0);
            x_b1 = fmaf(dh[4 * j + 3], tv[3], x_b1);
          }
          float s_a = s_a0 + s_a1, s_b = s_b0 + s_b1, x_a = x_a0 + x_a1, x_b = x_b0 + x_b1;
          cs_row_sums(s_a, s_b);
          cs_row_sums(x_a, x_b);
          const float gm_a = s_a * (1.0f / 64), gm_b = s_b * (1.0f / 64);
          const float gx_a = x_a * (1.0f / 64), gx_b = x_b * (1.0f / 64);
#pragma unroll
          for (int j = 0; j < 8; ++j) {  // pass 2: LayerNorm adjoint, kernels.cpp:99-126
            const float2 ta = st[(j * 128 + ra) * 4 + cp];
            const float2 tb = st[(j * 128 + ra + 8) * 4 + cp];
            dh[4 * j] = (dh[4 * j] - gm_a - ta.x * gx_a) * inv_a;
            dh[4 * j + 1] = (dh[4 * j + 1] - gm_a - ta.y * gx_a) * inv_a;
            dh[4 * j + 2] = (dh[4 * j + 2] - gm_b - tb.x * gx_b) * inv_b;
            dh[4 * j + 3] = (dh[4 * j + 3] - gm_b - tb.y * gx_b) * inv_b;
          }
          if (kDiscardScratch) {  // t_l of this tile is dead: drop its lines (4 rows x 4 threads per line)
            __syncwarp();
            if (cp == 0 && (rg & 3) == 0) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                ptx::discard_l2_line(st + (j * 128 + ra) * 4);
                ptx::discard_l2_line(st + (j * 128 + ra + 8) * 4);
              }
            }
          }
        }
        if (c <= 0) {  // new A operand (split d) for this linear; the input segments share one
          cs_store_a(t_ahi, t_alo, dh);
          signal_a();
          write_db(dh);
        }
        if (FACT && c == 0) {  // dY for the node-level sums
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (va) *reinterpret_cast<float2*>(a.dy_out + ga * H + 8 * j + 2 * cp) = make_float2(dh[4 * j], dh[4 * j + 1]);
            if (vb)
              *reinterpret_cast<float2*>(a.dy_out + gb * H + 8 * j + 2 * cp) =
                  make_float2(dh[4 * j + 2], dh[4 * j + 3]);
          }
        }
        if (c >= 0) gather(ga, gb, va, vb, c, h);  // dW0 segment operand
        stage_chunk(h, dh);
        wait_d();
        ++job;
        if (c < 0) {
          load_d(-1, dh);  // d_prev = d_u W^T + d_h
        } else {
          float* outp;
          if (FACT) outp = a.de_io;
          else if (MODE == kEdgeInput) outp = c == 0 ? a.d_src : (c == 1 ? a.d_dst : a.de_io);
          else outp = c == 0 ? a.d_a_out : a.d_x_out;
          float o[32];
          load_d(-1, o);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (va) *reinterpret_cast<float2*>(outp + ga * H + 8 * j + 2 * cp) = make_float2(o[4 * j], o[4 * j + 1]);
            if (vb)
              *reinterpret_cast<float2*>(outp + gb * H + 8 * j + 2 * cp) = make_float2(o[4 * j + 2], o[4 * j + 3]);
          }
          if (c + 1 < nseg) signal_a();  // D consumed; A (= split d_h) stays
        }
      }
    }
    if (job >= 1) flush(job - 1);
  } else if (warp == 16) {
    // ================================================================ dX MMA issuer (as mlp_tc_bwd.cuh)
    const uint32_t tm = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile uint32_t*>(tmem_base_slot), 0);
    constexpr uint32_t idesc = ptx::idesc_tf32(128, H);
    int ws = 0;
    uint32_t wph = 0, pa[2] = {0, 0};
    for (int64_t pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
#pragma unroll 1
      for (int st = 0; st < n_w; ++st) {
        const bool first_zero = st == 0 || (st >= nseg && st < nseg + K) || st >= nseg + 2 * K + 1 || st == nseg + K;
        const bool to_a_empty = st + 1 < nseg;
        ptx::mbar_wait(&w_full[ws], wph);
        ptx::tc_fence_after();
        const uint32_t bb = ptx::smem_u32(wring + (size_t)ws * Cfg::CHUNK_FLOATS);
#pragma unroll 1
        for (int s = 0; s < 2; ++s) {
          ptx::mbar_wait(&a_full[s], pa[s]);
          pa[s] ^= 1;
          ptx::tc_fence_after();
          const uint32_t slot = ptx::opaque(tm + s * Cfg::SLOT_COLS);
          const uint64_t d0 = ptx::opaque64(ptx::smem_desc(bb, Cfg::LBO, Cfg::SBO));
#pragma unroll
          for (int ks = 0; ks < H / 8; ++ks) {
            const uint64_t b_hi = d0 + (uint64_t)((ks * 2 * Cfg::LBO) >> 4);
            const uint64_t b_lo = b_hi + (uint64_t)(Cfg::LO_OFF >> 4);
            ptx::mma_tf32_ts_w(slot + 2 * H, slot + 8 * ks, b_hi, idesc, (!first_zero || ks > 0) ? 1u : 0u);
            ptx::mma_tf32_ts_w(slot + 2 * H, slot + 8 * ks, b_lo, idesc, 1u);
            ptx::mma_tf32_ts_w(slot + 2 * H, slot + H + 8 * ks, b_hi, idesc, 1u);
          }
          ptx::mma_commit_w(to_a_empty ? &a_empty[s] : &d_full[s]);
        }
        ptx::mma_commit_w(&w_empty[ws]);
        if (++ws == Cfg::WSTAGES) {
          ws = 0;
          wph ^= 1;
        }
      }
    }
  } else if (warp == 17) {
    // ================================================================ dW MMA issuer (N = 128, one accumulator)
    const uint32_t tm = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile uint32_t*>(tmem_base_slot), 0);
    constexpr uint32_t idesc_dw = ptx::idesc_tf32(128, 2 * H) | (1u << 15) | (1u << 16);  // A, B MN-major
    int64_t gi = 0;
    const int64_t n_jobs = ((n_pairs - blockIdx.x + gridDim.x - 1) / gridDim.x) * n_dw;
    const uint32_t t_dw = ptx::opaque(tm + Cfg::DW_COL);
    for (int64_t jd = 0; jd < n_jobs; ++jd) {
      ptx::mbar_wait(&dw_empty[0], (uint32_t)((jd & 1) ^ 1));  // job jd - 1 drained
      ptx::tc_fence_after();
      for (int b = 0; b < 8; ++b, ++gi) {
        const int buf = (int)(gi % Cfg::NSTAGE);
        ptx::mbar_wait(&st_full[buf], (uint32_t)((gi / Cfg::NSTAGE) & 1));
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(stage + (size_t)buf * Cfg::STAGE_BYTES);
        constexpr uint64_t swz = (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
        const uint64_t a0 = ptx::opaque64(ptx::smem_desc(sa, Cfg::ST_LBO, Cfg::ST_SBO) | swz);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t ad = a0 + (uint64_t)((ks * 2 * Cfg::ST_SBO) >> 4);
          const uint64_t bd = ad + (uint64_t)(16384 >> 4);
          ptx::mma_tf32_ss_w(t_dw, ad, bd, idesc_dw, (b > 0 || ks > 0) ? 1u : 0u);
        }
        ptx::mma_commit_w(&st_empty[((gi / Cfg::NSTAGE) & 1) * Cfg::NSTAGE + buf]);
      }
      ptx::mma_commit_w(&dw_full[0]);
    }
  } else if (warp == 18 && lane == 0) {
    // ================================================================ weight loader
    int ws = 0;
    uint32_t wph = 0;
    for (int64_t pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
      for (int j = 0; j < n_w; ++j) {
        ptx::mbar_wait(&w_empty[ws], wph ^ 1);
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
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 16) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

}  // namespace hgnn_b200
