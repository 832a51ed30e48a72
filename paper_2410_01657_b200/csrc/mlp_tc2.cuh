// Tensor-core processor-MLP forward, column-split epilogue (sm_100a, H = 64).
//
// Same math and MMA schedule as mlp_tc_forward_kernel (mlp_tc.cuh): 3xTF32,
// two ping-pong 128-row tile slots, TMEM per slot [A_hi | A_lo | D], weight
// chunks streamed by cp.async.bulk, one elected MMA-issuing warp.
//
// Difference: TWO epilogue threads per row. The epilogue was latency-bound
// with one thread per row (two epilogue warps per SM sub-partition, ~40 %
// issue use); here 16 epilogue warps own (slot, TMEM lane quarter, column
// half): warp w -> slot w / 8, quarter w % 4 (a warp may only touch the TMEM
// lanes of its sub-partition, w % 4), half (w / 4) % 2. Row reductions
// (LayerNorm mean / variance, kernels.cpp:81-94) combine the two halves through
// shared memory under a 64-thread named barrier per (slot, quarter); both
// halves read the two partial sums in the same fixed order, so the statistics
// are bitwise identical on both sides and deterministic.
//
// Warp roles: 0-15 epilogue, 16 MMA issuer, 17 weight loader, 18-19 idle.
#pragma once

#include "mlp_tc.cuh"

namespace hgnn_b200 {

struct Tc2Cfg {
  static constexpr int H = 64;
  static constexpr int HALF = 32;
  static constexpr int EPI_WARPS = 16;
  static constexpr int THREADS = 640;  // 4 epilogue warpgroups + 1 control warpgroup
  static constexpr int STAGES = 4;
  static constexpr size_t OFF_BARS = (size_t)STAGES * TcCfg<64>::CHUNK_BYTES;
  static constexpr size_t OFF_XCH = OFF_BARS + 256;                 // [2 buf][2 slot][4 q][2 half][32] floats
  static constexpr size_t OFF_BIAS = OFF_XCH + 2 * 2 * 4 * 2 * 32 * 4;
  static constexpr size_t SMEM = OFF_BIAS + 18 * 64 * 4 + 1024;
};

// Sum of 32 values, 8 independent chains.
__device__ __forceinline__ float sum32(const float (&v)[32]) {
  float p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = v[i];
#pragma unroll
  for (int j = 8; j < 32; ++j) p[j % 8] += v[j];
  return ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Half-row gather: this thread's 32 columns of input segment c.
template <int MODE>
__device__ __forceinline__ void tc2_gather(const TcFwdArgs& a, int64_t row, bool valid, int c, int col0,
                                           float (&v)[32]) {
  if (valid) {
    const float* seg;
    if (MODE == kEdgeInput)
      seg = c == 0 ? a.x + (int64_t)__ldg(a.src + row) * 64
                   : (c == 1 ? a.x + (int64_t)__ldg(a.dst + row) * 64 : a.e_in + row * 64);
    else
      seg = c == 0 ? a.a + row * 64 : a.x + row * 64;
    const float4* s4 = reinterpret_cast<const float4*>(seg + col0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 t = __ldg(s4 + j);
      v[4 * j] = t.x;
      v[4 * j + 1] = t.y;
      v[4 * j + 2] = t.z;
      v[4 * j + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = 0.f;
  }
}

__device__ __forceinline__ void tc2_store_a(uint32_t t_hi, uint32_t t_lo, const float (&v)[32]) {
  float hi[32], lo[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    hi[j] = ptx::tf32_trunc(v[j]);
    lo[j] = v[j] - hi[j];
  }
  ptx::tmem_st32(t_hi, hi);
  ptx::tmem_st32(t_lo, lo);
}

template <int MODE, bool PROF>
__global__ void __launch_bounds__(Tc2Cfg::THREADS, 1) mlp_tc_forward2_kernel(TcFwdArgs a) {
  using Cfg = TcCfg<64>;
  using C2 = Tc2Cfg;
  constexpr int H = 64;
  constexpr int nseg = MODE == kEdgeInput ? 3 : 2;
  constexpr int in_dim = nseg * H;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* wring = reinterpret_cast<float*>(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C2::OFF_BARS);
  uint64_t* w_full = bars;                    // [STAGES]
  uint64_t* w_empty = bars + C2::STAGES;      // [STAGES]
  uint64_t* a_full = bars + 2 * C2::STAGES;   // [2]
  uint64_t* a_empty = a_full + 2;             // [2]
  uint64_t* d_full = a_empty + 2;             // [2]
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(d_full + 2);
  float* xch = reinterpret_cast<float*>(smem + C2::OFF_XCH);
  float* sbias = reinterpret_cast<float*>(smem + C2::OFF_BIAS);  // (k+2) x H

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n_chunks = nseg + a.k + 1;
  const int64_t n_tiles = (a.n_rows + 127) / 128;
  const int64_t n_pairs = (n_tiles + 1) / 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C2::STAGES; ++s) {
      ptx::mbar_init(&w_full[s], 1);
      ptx::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&a_full[s], 8);  // 8 epilogue warps per slot
      ptx::mbar_init(&a_empty[s], 1);
      ptx::mbar_init(&d_full[s], 1);
    }
    ptx::fence_mbarrier_init();
  }
  for (int i = threadIdx.x; i < (a.k + 2) * H; i += blockDim.x)
    sbias[i] = __ldg(a.params + mlp_b_offset(i / H, in_dim, H) + (i % H));
  if (warp == C2::EPI_WARPS) ptx::tmem_alloc<512>(tmem_base_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_base_slot;

  // CTA register pool = 640 x 96; epilogue warpgroups 104, control 56.
  static_assert(512 * 104 + 128 * 56 <= C2::THREADS * 96, "setmaxnreg exceeds the CTA register pool");
  if (warp < C2::EPI_WARPS) ptx::regs_inc<104>();
  else ptx::regs_dec<56>();

  if (warp < C2::EPI_WARPS) {
    // ------------------------------------------------------------ epilogue
    const int g = warp / 8;         // tile slot
    const int wq = warp % 4;        // TMEM lane quarter (= SM sub-partition)
    const int ch = (warp / 4) % 2;  // column half
    const int col0 = ch * C2::HALF;
    const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
    const uint32_t t_ahi = tmem + g * Cfg::SLOT_COLS + lane_off + col0;
    const uint32_t t_alo = t_ahi + H;
    const uint32_t t_d = t_ahi + 2 * H;
    const int bar_id = 1 + g * 4 + wq;  // 64-thread pair (two column halves)
    // exchange slots: [buf][g][wq][half][lane]
    float* xbase = xch + ((g * 4 + wq) * 2) * 32 + lane;
    auto row_sum = [&](float part, int buf) -> float {
      float* xb = xbase + buf * (2 * 4 * 2 * 32);
      xb[ch * 32] = part;
      named_bar(bar_id, 64);
      return xb[0] + xb[32];  // fixed order: half 0 + half 1
    };
    uint32_t pe = 0, pd = 0;
    unsigned long long e_d = 0, e_ae = 0, e_sig = 0;
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
    float v[32];
    int64_t pair = blockIdx.x;
    if (pair < n_pairs) {
      const int64_t row0 = (2 * pair + g) * 128 + 32 * wq + lane;
      tc2_gather<MODE>(a, row0, row0 < a.n_rows, 0, col0, v);
    }
    for (; pair < n_pairs; pair += gridDim.x) {
      const int64_t row = (2 * pair + g) * 128 + 32 * wq + lane;
      const bool valid = row < a.n_rows;
      float h[32];
      for (int c = 0; c < nseg; ++c) {
        if (c > 0) {
          const long long t0 = PROF ? clock64() : 0;
          ptx::mbar_wait(&a_empty[g], pe);
          pe ^= 1;
          ptx::tc_fence_after();
          if (PROF) e_ae += (unsigned long long)(clock64() - t0);
        }
        tc2_store_a(t_ahi, t_alo, v);
        signal_a();
        if (c + 1 < nseg) tc2_gather<MODE>(a, row, valid, c + 1, col0, v);
      }
      wait_d();
      {
        ptx::tmem_ld32(t_d, h);
        ptx::tmem_wait_ld();
        const float* b = sbias + col0;
#pragma unroll
        for (int j = 0; j < 32; ++j) h[j] += b[j];
      }
      for (int l = 1; l <= a.k; ++l) {
        tc2_store_a(t_ahi, t_alo, h);
        signal_a();
        wait_d();
        float u[32];
        ptx::tmem_ld32(t_d, u);
        ptx::tmem_wait_ld();
        const float* b = sbias + l * H + col0;
#pragma unroll
        for (int j = 0; j < 32; ++j) u[j] += b[j];
        // LayerNorm without affine (kernels.cpp:81-94), two-pass, row split in halves
        const float mean = row_sum(sum32(u), 0) * (1.0f / H);
        float p[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) p[i] = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          u[j] -= mean;
          p[j % 8] = fmaf(u[j], u[j], p[j % 8]);
        }
        const float var =
            row_sum(((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7])), 1) * (1.0f / H);
        const float inv_std = ptx::rsqrt_fast(var + 1e-12f);
#pragma unroll
        for (int j = 0; j < 32; ++j) h[j] += elu_fast(u[j] * inv_std);
      }
      tc2_store_a(t_ahi, t_alo, h);
      signal_a();
      const int64_t next = pair + gridDim.x;
      if (next < n_pairs) {
        const int64_t nrow = (2 * next + g) * 128 + 32 * wq + lane;
        tc2_gather<MODE>(a, nrow, nrow < a.n_rows, 0, col0, v);
      }
      wait_d();
      {
        const float* bo = sbias + (a.k + 1) * H + col0;
        float p[32];
        ptx::tmem_ld32(t_d, p);
        ptx::tmem_wait_ld();
        if (valid) {
          float4* o = reinterpret_cast<float4*>(a.out + row * H + col0);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            o[j] = make_float4(p[4 * j] + bo[4 * j], p[4 * j + 1] + bo[4 * j + 1], p[4 * j + 2] + bo[4 * j + 2],
                               p[4 * j + 3] + bo[4 * j + 3]);
        }
      }
    }
    if (PROF && warp == 0 && lane == 0) {
      atomicAdd(a.prof + kFwdProfEpiTotal, (unsigned long long)(clock64() - e_t0));
      atomicAdd(a.prof + kFwdProfEpiD, e_d);
      atomicAdd(a.prof + kFwdProfEpiAE, e_ae);
      atomicAdd(a.prof + kFwdProfEpiSig, e_sig);
    }
  } else if (warp == C2::EPI_WARPS) {
    // ------------------------------------------------------------ MMA issuer (all lanes; one elected issues)
    const uint32_t tm = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile uint32_t*>(tmem_base_slot), 0);
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
        if (++ws == C2::STAGES) {
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
  } else if (warp == C2::EPI_WARPS + 1) {
    // ------------------------------------------------------------ weight loader
    if (lane == 0) {
      int ws = 0;
      uint32_t wph = 0;
      for (int64_t pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
        for (int j = 0; j < n_chunks; ++j) {
          ptx::mbar_wait(&w_empty[ws], wph ^ 1);
          ptx::mbar_arrive_expect_tx(&w_full[ws], Cfg::CHUNK_BYTES);
          ptx::bulk_g2s(wring + (size_t)ws * Cfg::CHUNK_FLOATS, a.chunks + (size_t)j * Cfg::CHUNK_FLOATS,
                        Cfg::CHUNK_BYTES, &w_full[ws]);
          if (++ws == C2::STAGES) {
            ws = 0;
            wph ^= 1;
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == C2::EPI_WARPS) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

}  // namespace hgnn_b200
