// Encoder / decoder MLPs (SIMT fp32, sm_100a): the row-wise MLPs on either
// side of the message-passing stack.
//
// Spec (nn.hpp:27-58, model.cpp:70-101), H = 32 or 64 hidden width, k hidden blocks:
//   h = x W0 + b0;  h += ELU(LN0(h Wj + bj)), j = 1..k;
//   y = h W_{k+1} + b_{k+1} (+ x W_skip);  y = LN(y) * gamma + beta (encoders)
// encoder: IN = F_x or F_e, OUT = H, skip + output LayerNorm (model.cpp:70-80)
// decoder: IN = H, OUT = F_y, skip, no LayerNorm (model.cpp:92-101)
// Parameters in MlpParams::for_each order (nn.cpp:38-46): w0, b0, ..., w_{k+1},
// b_{k+1}, skip, [ln_g, ln_b]; fp32 copies, staged whole in shared memory.
//
// One thread owns one row. The backward recomputes the forward per row and
// keeps the per-row intermediates (hidden states, normed values, inverse
// standard deviations, pre-LayerNorm output) in a per-CTA global scratch
// ([slot][row] layout: coalesced). Weight gradients are reduced over a tile
// of kGenThreads rows through shared memory — every (i, j) element summed
// by one owning thread in row order — and added to a per-CTA partial owned
// by that thread, so the result is deterministic run to run.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

namespace hgnn_b200 {

constexpr int kGenThreads = 128;
constexpr int kGenRow = 68;  // staged row stride (floats): 16-byte aligned, conflict-free float4 row writes

__host__ __device__ inline int64_t gen_param_count(int in_dim, int out_dim, int k, bool skip, bool out_ln, int H) {
  return (int64_t)in_dim * H + H + (int64_t)k * (H * H + H) + (int64_t)H * out_dim + out_dim +
         (skip ? (int64_t)in_dim * out_dim : 0) + (out_ln ? 2 * out_dim : 0);
}

// Offsets (floats) inside one MLP's for_each block.
struct GenLayout {
  int in_dim, out_dim, k, H;
  __host__ __device__ int64_t w(int l) const {  // l = 0 .. k+1
    return l == 0 ? 0 : (int64_t)in_dim * H + H + (int64_t)(l - 1) * (H * H + H);
  }
  __host__ __device__ int64_t b(int l) const {
    return w(l) + (l == 0 ? (int64_t)in_dim * H : (l <= k ? (int64_t)H * H : (int64_t)H * out_dim));
  }
  __host__ __device__ int64_t skip() const { return b(k + 1) + out_dim; }
  __host__ __device__ int64_t ln_g() const { return skip() + (int64_t)in_dim * out_dim; }
  __host__ __device__ int64_t ln_b() const { return ln_g() + out_dim; }
};

struct GenArgs {
  int64_t n_rows;
  const float* in;        // n_rows x IN
  float* out;             // n_rows x OUT (forward)
  const float* d_out;     // n_rows x OUT (backward)
  float* d_in;            // n_rows x IN input adjoint (backward, decoder only)
  const float* params;    // fp32, for_each layout
  float* grad_partial;    // [gridDim.x][n_par] fp32 (backward)
  float* scratch;         // [gridDim.x][slots][kGenThreads] (backward)
  int k;
  int64_t n_par;
};

__device__ __forceinline__ float gen_elu(float z) { return z > 0.f ? z : ptx::exp_fast(z) - 1.0f; }

// Sum of N values with 4 independent chains.
template <int N>
__device__ __forceinline__ float gen_sum(const float (&v)[N]) {
  float p[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < N; ++j) p[j % 4] += v[j];
  return (p[0] + p[1]) + (p[2] + p[3]);
}

// Two-pass LayerNorm statistics of N values (kernels.cpp:81-94).
template <int N>
__device__ __forceinline__ void gen_ln_stats(const float (&v)[N], float& mean, float& inv_std) {
  mean = gen_sum<N>(v) * (1.0f / N);
  float q[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const float d = v[j] - mean;
    q[j % 4] = fmaf(d, d, q[j % 4]);
  }
  inv_std = ptx::rsqrt_fast(((q[0] + q[1]) + (q[2] + q[3])) * (1.0f / N) + 1e-12f);
}

// acc[j] += sum_t v[t] W[t*NO + j] (W row-major, shared memory, warp-uniform
// reads). Long inputs (NI >= 16) go through this thread's shared-memory
// column (stride kGenThreads, conflict-free) so the t loop can stay rolled:
// a fully unrolled 64 x 64 product is ~5K instructions and the kernels were
// instruction-fetch bound.
template <int NI, int NO>
__device__ __forceinline__ void gen_gemv(float (&acc)[NO], const float (&v)[NI], const float* __restrict__ W,
                                         float* col) {
  if (NI >= 16) {
#pragma unroll
    for (int t = 0; t < NI; ++t) col[t * kGenThreads] = v[t];
#pragma unroll 2
    for (int t = 0; t < NI; ++t) {
      const float vt = col[t * kGenThreads];
      if (NO % 4 == 0) {
        const float4* w4 = reinterpret_cast<const float4*>(W + t * NO);
#pragma unroll
        for (int j = 0; j < NO / 4; ++j) {
          const float4 w = w4[j];
          acc[4 * j] = fmaf(vt, w.x, acc[4 * j]);
          acc[4 * j + 1] = fmaf(vt, w.y, acc[4 * j + 1]);
          acc[4 * j + 2] = fmaf(vt, w.z, acc[4 * j + 2]);
          acc[4 * j + 3] = fmaf(vt, w.w, acc[4 * j + 3]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < NO; ++j) acc[j] = fmaf(vt, W[t * NO + j], acc[j]);
      }
    }
    return;
  }
#pragma unroll
  for (int t = 0; t < NI; ++t) {
    const float vt = v[t];
    if (NO % 4 == 0) {
      const float4* w4 = reinterpret_cast<const float4*>(W + t * NO);
#pragma unroll
      for (int j = 0; j < NO / 4; ++j) {
        const float4 w = w4[j];
        acc[4 * j] = fmaf(vt, w.x, acc[4 * j]);
        acc[4 * j + 1] = fmaf(vt, w.y, acc[4 * j + 1]);
        acc[4 * j + 2] = fmaf(vt, w.z, acc[4 * j + 2]);
        acc[4 * j + 3] = fmaf(vt, w.w, acc[4 * j + 3]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < NO; ++j) acc[j] = fmaf(vt, W[t * NO + j], acc[j]);
    }
  }
}

// acc[t] += sum_j d[j] W[t*NO + j]  (adjoint product d W^T): a rolled loop
// over t writing this thread's shared-memory column, then one unrolled pass
// adding the column into acc.
template <int NI, int NO>
__device__ __forceinline__ void gen_gemv_t(float (&acc)[NI], const float (&d)[NO], const float* __restrict__ W,
                                           float* col) {
#pragma unroll 2
  for (int t = 0; t < NI; ++t) {
    float p[4] = {0.f, 0.f, 0.f, 0.f};
    if (NO % 4 == 0) {
      const float4* w4 = reinterpret_cast<const float4*>(W + t * NO);
#pragma unroll
      for (int j = 0; j < NO / 4; ++j) {
        const float4 w = w4[j];
        p[0] = fmaf(d[4 * j], w.x, p[0]);
        p[1] = fmaf(d[4 * j + 1], w.y, p[1]);
        p[2] = fmaf(d[4 * j + 2], w.z, p[2]);
        p[3] = fmaf(d[4 * j + 3], w.w, p[3]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < NO; ++j) p[j % 4] = fmaf(d[j], W[t * NO + j], p[j % 4]);
    }
    col[t * kGenThreads] = (p[0] + p[1]) + (p[2] + p[3]);
  }
#pragma unroll
  for (int t = 0; t < NI; ++t) acc[t] += col[t * kGenThreads];
}

template <int N>
__device__ __forceinline__ void gen_load_row(float (&v)[N], const float* __restrict__ src, bool valid) {
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = valid ? __ldg(src + j) : 0.f;
}

__device__ __forceinline__ void gen_stage_params(float* dst, const float* __restrict__ src, int64_t n) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldg(src + i);
}

// ------------------------------------------------------------------ forward
template <int IN, int OUT, bool SKIP, bool OUT_LN, int H>
__global__ void __launch_bounds__(kGenThreads) gen_mlp_forward_kernel(GenArgs a) {
  extern __shared__ __align__(16) float gsm[];
  const GenLayout L{IN, OUT, a.k, H};
  float* col = gsm + ((a.n_par + 3) / 4) * 4 + threadIdx.x;  // this thread's column (H x kGenThreads)
  gen_stage_params(gsm, a.params, a.n_par);
  __syncthreads();
  for (int64_t row = (int64_t)blockIdx.x * kGenThreads + threadIdx.x; row - threadIdx.x < a.n_rows;
       row += (int64_t)gridDim.x * kGenThreads) {
    const bool valid = row < a.n_rows;
    float h[H];
    {
      float x[IN];
      gen_load_row<IN>(x, a.in + row * IN, valid);
#pragma unroll
      for (int j = 0; j < H; ++j) h[j] = gsm[L.b(0) + j];
      gen_gemv<IN, H>(h, x, gsm + L.w(0), col);
    }
    for (int l = 1; l <= a.k; ++l) {
      float u[H];
#pragma unroll
      for (int j = 0; j < H; ++j) u[j] = gsm[L.b(l) + j];
      gen_gemv<H, H>(u, h, gsm + L.w(l), col);
      float mean, inv_std;
      gen_ln_stats<H>(u, mean, inv_std);
#pragma unroll
      for (int j = 0; j < H; ++j) h[j] += gen_elu((u[j] - mean) * inv_std);
    }
    float y[OUT];
#pragma unroll
    for (int j = 0; j < OUT; ++j) y[j] = gsm[L.b(a.k + 1) + j];
    gen_gemv<H, OUT>(y, h, gsm + L.w(a.k + 1), col);
    if (SKIP) {
      float x[IN];
      gen_load_row<IN>(x, a.in + row * IN, valid);
      gen_gemv<IN, OUT>(y, x, gsm + L.skip(), col);
    }
    if (OUT_LN) {
      float mean, inv_std;
      gen_ln_stats<OUT>(y, mean, inv_std);
#pragma unroll
      for (int j = 0; j < OUT; ++j) y[j] = gsm[L.ln_g() + j] * ((y[j] - mean) * inv_std) + gsm[L.ln_b() + j];
    }
    if (valid) {
#pragma unroll
      for (int j = 0; j < OUT; ++j) a.out[row * OUT + j] = y[j];
    }
  }
}

// ------------------------------------------------------------------ backward
// Scratch slots per row: hidden states h_0..h_k (k+1) x H, normed t_1..t_k
// k x H, inv_std k, pre-LayerNorm output OUT (+ mean / inv_std 2).
// Dynamic shared memory of gen_mlp_backward_kernel<IN, OUT, ...>.
__host__ __device__ inline size_t gen_backward_smem(int in_dim, int out_dim, int H) {
  const int wblk = (H * H + H) > (in_dim * H + H) ? (H * H + H) : (in_dim * H + H);
  return (size_t)(((wblk + 3) / 4) * 4 + ((in_dim * out_dim + 3) / 4) * 4 + ((out_dim + 3) / 4) * 4 +
                  2 * kGenThreads * kGenRow) * 4;
}

__host__ __device__ inline int64_t gen_scratch_slots(int k, int out_dim, int H) {
  return (int64_t)(2 * k + 1) * H + k + out_dim + 2;
}

// Tile reduction of dW += sum_rows A[r][i] D[r][j] for NI x NO, A / D staged
// in shared memory as [i][row] / [j][row]; thread t owns elements t, t + T, ...
// Tile reduction dW[i][j] += sum_rows A[r][i] D[r][j] (NI x NO), A / D staged
// row-major ([row][kGenRow]). Each thread owns a 4 x BJ register block of dW
// (i, j ascending, rows summed in order: deterministic) and reads it with
// 16-byte shared loads: 3 loads per 32 FMAs.
template <int NI, int NO>
__device__ __forceinline__ void gen_dw_tile(float* __restrict__ gp, const float* __restrict__ sa,
                                            const float* __restrict__ sd) {
  constexpr int BJ = NO >= 8 ? 8 : 4;
  constexpr int NBI = (NI + 3) / 4, NBJ = (NO + BJ - 1) / BJ;
  for (int b = threadIdx.x; b < NBI * NBJ; b += kGenThreads) {
    const int i0 = 4 * (b / NBJ), j0 = BJ * (b % NBJ);
    float acc[4][BJ];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jj = 0; jj < BJ; ++jj) acc[ii][jj] = 0.f;
#pragma unroll 4
    for (int r = 0; r < kGenThreads; ++r) {
      const float4 av = *reinterpret_cast<const float4*>(sa + r * kGenRow + i0);
      float dv[BJ];
#pragma unroll
      for (int q = 0; q < BJ / 4; ++q) {
        const float4 t = *reinterpret_cast<const float4*>(sd + r * kGenRow + j0 + 4 * q);
        dv[4 * q] = t.x;
        dv[4 * q + 1] = t.y;
        dv[4 * q + 2] = t.z;
        dv[4 * q + 3] = t.w;
      }
      const float a4[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) acc[ii][jj] = fmaf(a4[ii], dv[jj], acc[ii][jj]);
    }
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jj = 0; jj < BJ; ++jj)
        if (i0 + ii < NI && j0 + jj < NO) gp[(i0 + ii) * NO + j0 + jj] += acc[ii][jj];
  }
}
template <int NO>
__device__ __forceinline__ void gen_db_tile(float* __restrict__ gp, const float* __restrict__ sd) {
  for (int j = threadIdx.x; j < NO; j += kGenThreads) {
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
    for (int r = 0; r < kGenThreads; r += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] += sd[(r + u) * kGenRow + j];
    }
    gp[j] += (s[0] + s[1]) + (s[2] + s[3]);
  }
}
// This thread's row v[0..N) into the row-major staging buffer.
template <int N>
__device__ __forceinline__ void gen_stage_col(float* s, const float (&v)[N]) {
  float* d = s + threadIdx.x * kGenRow;
  if (N % 4 == 0) {
#pragma unroll
    for (int j = 0; j < N; j += 4) *reinterpret_cast<float4*>(d + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) d[j] = v[j];
  }
}

// smem: one streamed layer block (W, b) | skip weights | LN gamma | A stage | D stage.
// Weights are streamed layer by layer (the CTA walks the layers of its tile in
// lock-step), so two CTAs fit per SM.
template <int IN, int OUT, bool SKIP, bool OUT_LN, bool DIN, int H>
__global__ void __launch_bounds__(kGenThreads) gen_mlp_backward_kernel(GenArgs a) {
  extern __shared__ __align__(16) float gsm[];
  const GenLayout L{IN, OUT, a.k, H};
  const int K = a.k;
  constexpr int WBLK = ((H * H + H) > (IN * H + H) ? (H * H + H) : (IN * H + H));
  constexpr int SW_N = ((WBLK + 3) / 4) * 4, SK_N = ((IN * OUT + 3) / 4) * 4, LN_N = ((OUT + 3) / 4) * 4;
  float* sW = gsm;
  float* sSkip = sW + SW_N;
  float* sG = sSkip + SK_N;
  float* sA = sG + LN_N;
  float* sD = sA + kGenThreads * kGenRow;
  // this thread's gemv column (H x kGenThreads floats) aliases the A
  // staging buffer: every use is separated from the dW tiles by the CTA
  // barriers of load_linear / the staging
  float* col = sA + threadIdx.x;
  if (SKIP)
    for (int i = threadIdx.x; i < IN * OUT; i += kGenThreads) sSkip[i] = __ldg(a.params + L.skip() + i);
  if (OUT_LN)
    for (int i = threadIdx.x; i < OUT; i += kGenThreads) sG[i] = __ldg(a.params + L.ln_g() + i);
  // (W, b) of linear l into sW; all threads of the CTA call it together
  auto load_linear = [&](int l) -> const float* {
    const int rows = l == 0 ? IN : H, cols = l == K + 1 ? OUT : H;
    __syncthreads();
    gen_stage_params(sW, a.params + L.w(l), (int64_t)rows * cols + cols);
    __syncthreads();
    return sW;
  };
  float* gp = a.grad_partial + (int64_t)blockIdx.x * a.n_par;
  const int64_t slots = gen_scratch_slots(K, OUT, H);
  float* scr = a.scratch + (int64_t)blockIdx.x * slots * kGenThreads + threadIdx.x;
  auto S = [&](int64_t slot) -> float& { return scr[slot * kGenThreads]; };
  const int64_t s_h = 0, s_t = (int64_t)(K + 1) * H, s_inv = s_t + (int64_t)K * H, s_y = s_inv + K,
                s_yst = s_y + OUT;
  __syncthreads();
  for (int64_t row0 = (int64_t)blockIdx.x * kGenThreads; row0 < a.n_rows; row0 += (int64_t)gridDim.x * kGenThreads) {
    const int64_t row = row0 + threadIdx.x;
    const bool valid = row < a.n_rows;
    // ---- forward recompute, keeping the intermediates
    {
      float h[H];
      {
        float x[IN];
        gen_load_row<IN>(x, a.in + row * IN, valid);
        const float* W = load_linear(0);
#pragma unroll
        for (int j = 0; j < H; ++j) h[j] = W[IN * H + j];
        gen_gemv<IN, H>(h, x, W, col);
      }
#pragma unroll
      for (int j = 0; j < H; ++j) S(s_h + j) = h[j];
      for (int l = 1; l <= K; ++l) {
        float u[H];
        const float* W = load_linear(l);
#pragma unroll
        for (int j = 0; j < H; ++j) u[j] = W[H * H + j];
        gen_gemv<H, H>(u, h, W, col);
        float mean, inv_std;
        gen_ln_stats<H>(u, mean, inv_std);
#pragma unroll
        for (int j = 0; j < H; ++j) {
          const float t = (u[j] - mean) * inv_std;
          S(s_t + (int64_t)(l - 1) * H + j) = t;
          h[j] += gen_elu(t);
          S(s_h + (int64_t)l * H + j) = h[j];
        }
        S(s_inv + l - 1) = inv_std;
      }
      float y[OUT];
      const float* W = load_linear(K + 1);
#pragma unroll
      for (int j = 0; j < OUT; ++j) y[j] = W[H * OUT + j];
      gen_gemv<H, OUT>(y, h, W, col);
      if (SKIP) {
        float x[IN];
        gen_load_row<IN>(x, a.in + row * IN, valid);
        gen_gemv<IN, OUT>(y, x, sSkip, col);
      }
      if (OUT_LN) {
        float mean, inv_std;
        gen_ln_stats<OUT>(y, mean, inv_std);
#pragma unroll
        for (int j = 0; j < OUT; ++j) S(s_y + j) = (y[j] - mean) * inv_std;  // xhat
        S(s_yst) = inv_std;
      }
    }
    // ---- output adjoint, output LayerNorm (kernels.cpp:99-126 with gamma)
    float dy[OUT];
    gen_load_row<OUT>(dy, a.d_out + row * OUT, valid);
    if (OUT_LN) {
      float xh[OUT];
#pragma unroll
      for (int j = 0; j < OUT; ++j) xh[j] = S(s_y + j);
      // d gamma += dy * xhat, d beta += dy (tile-reduced below)
      float gdy[OUT], gm = 0.f, gxm = 0.f;
#pragma unroll
      for (int j = 0; j < OUT; ++j) {
        gdy[j] = sG[j] * dy[j];
        gm += gdy[j];
        gxm = fmaf(gdy[j], xh[j], gxm);
      }
      gm *= 1.0f / OUT;
      gxm *= 1.0f / OUT;
      const float inv_std = S(s_yst);
      __syncthreads();
      {
        float prod[OUT];
#pragma unroll
        for (int j = 0; j < OUT; ++j) prod[j] = dy[j] * xh[j];
        gen_stage_col<OUT>(sA, prod);
        gen_stage_col<OUT>(sD, dy);
      }
      __syncthreads();
      gen_db_tile<OUT>(gp + L.ln_g(), sA);
      gen_db_tile<OUT>(gp + L.ln_b(), sD);
#pragma unroll
      for (int j = 0; j < OUT; ++j) dy[j] = (gdy[j] - gm - xh[j] * gxm) * inv_std;
    }
    // ---- output projection (nn.cpp:241-245) and skip (nn.cpp:247-254)
    float dh[H];
    {
      float hk[H];
#pragma unroll
      for (int j = 0; j < H; ++j) hk[j] = S(s_h + (int64_t)K * H + j);
      __syncthreads();
      gen_stage_col<H>(sA, hk);
      gen_stage_col<OUT>(sD, dy);
      __syncthreads();
      gen_dw_tile<H, OUT>(gp + L.w(K + 1), sA, sD);
      gen_db_tile<OUT>(gp + L.b(K + 1), sD);
      if (SKIP) {
        float x[IN];
        gen_load_row<IN>(x, a.in + row * IN, valid);
        __syncthreads();
        gen_stage_col<IN>(sA, x);
        __syncthreads();
        gen_dw_tile<IN, OUT>(gp + L.skip(), sA, sD);
      }
#pragma unroll
      for (int j = 0; j < H; ++j) dh[j] = 0.f;
      gen_gemv_t<H, OUT>(dh, dy, load_linear(K + 1), col);
    }

    // ---- hidden blocks in reverse (nn.cpp:259-274)
    for (int l = K; l >= 1; --l) {
      float du[H];
      float pm[4] = {0.f, 0.f, 0.f, 0.f}, px[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < H; ++j) {
        const float t = S(s_t + (int64_t)(l - 1) * H + j);
        du[j] = dh[j] * (t > 0.f ? 1.0f : ptx::exp_fast(t));  // elu', kernels.cpp:68-71
        pm[j % 4] += du[j];
        px[j % 4] = fmaf(du[j], t, px[j % 4]);
      }
      const float gm = ((pm[0] + pm[1]) + (pm[2] + pm[3])) * (1.0f / H);
      const float gxm = ((px[0] + px[1]) + (px[2] + px[3])) * (1.0f / H);
      const float inv_std = S(s_inv + l - 1);
#pragma unroll
      for (int j = 0; j < H; ++j) du[j] = (du[j] - gm - S(s_t + (int64_t)(l - 1) * H + j) * gxm) * inv_std;
      {
        float hp[H];
#pragma unroll
        for (int j = 0; j < H; ++j) hp[j] = S(s_h + (int64_t)(l - 1) * H + j);
        __syncthreads();
        gen_stage_col<H>(sA, hp);
        gen_stage_col<H>(sD, du);
        __syncthreads();
      }
      gen_dw_tile<H, H>(gp + L.w(l), sA, sD);
      gen_db_tile<H>(gp + L.b(l), sD);
      gen_gemv_t<H, H>(dh, du, load_linear(l), col);  // d_prev = d_u W^T + d_h
    }
    // ---- input projection (nn.cpp:277-281)
    if (DIN) {  // d_in = d_h W0^T (+ d_y W_skip^T), 16 input columns at a time
      const float* W0 = load_linear(0);
#pragma unroll
      for (int c = 0; c < IN; c += 16) {
        float din[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          float s = 0.f;
          if (c + t < IN) {
            const float* w0 = W0 + (int64_t)(c + t) * H;
#pragma unroll
            for (int j = 0; j < H; ++j) s = fmaf(dh[j], w0[j], s);
            if (SKIP) {
              const float* ws = sSkip + (int64_t)(c + t) * OUT;
#pragma unroll
              for (int j = 0; j < OUT; ++j) s = fmaf(dy[j], ws[j], s);
            }
          }
          din[t] = s;
        }
        if (valid) {
#pragma unroll
          for (int t = 0; t < 16; ++t)
            if (c + t < IN) a.d_in[row * IN + c + t] = din[t];
        }
      }
    }
    {
      float x[IN];
      gen_load_row<IN>(x, a.in + row * IN, valid);
      __syncthreads();
      gen_stage_col<IN>(sA, x);
      gen_stage_col<H>(sD, dh);
      __syncthreads();
      gen_dw_tile<IN, H>(gp + L.w(0), sA, sD);
      gen_db_tile<H>(gp + L.b(0), sD);
    }
  }
}

}  // namespace hgnn_b200
