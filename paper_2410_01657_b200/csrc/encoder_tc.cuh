// Encoders and decoder on the tensor cores (sm_100a, H = 64; SURVEY §8f row 1,
// model.cpp:70-101). The node / edge encoder MLP
//   h = x W0 + b0;  h += ELU(LN0(h Wj + bj)), j = 1..k;
//   y = h W_{k+1} + b_{k+1} + x W_skip;  out = LN(y) * gamma + beta
// runs through the processor-MLP tcgen05 kernels in mode kEncoder: the F
// (<= 8) input features are one zero-padded K = H segment, the forward
// epilogue adds the skip product and the output LayerNorm (mlp_tc.cuh). The
// backward is three launches:
//   1. the forward kernel recomputes y (pre-LayerNorm, enc_ln = 0) into a dead
//      N x H buffer,
//   2. enc_out_backward_kernel (below) turns it in place into dy, the adjoint
//      of y, and forms the gamma / beta / W_skip gradient partials,
//   3. the tcgen05 backward kernel (mlp_tc_bwd.cuh, kEncoder) walks the MLP
//      with d_out = dy: dW_{k+1} .. dW0 (padded rows dropped), the biases.
// The decoder (y = MLP(x_M) + x_M W_skip, F_y <= 8 outputs, no LayerNorm) is
// mode kDecoder: the output linear's columns >= F_y are zero padding, the
// forward epilogue adds the skip product; its backward is the tcgen05 kernel
// (input adjoint of the MLP) plus dec_skip_backward_kernel (skip adjoint, W_skip).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

namespace hgnn_b200 {

constexpr int kEncLnThreads = 256;  // 8 warps, one row per warp at a time
constexpr int kEncLnBlocks = 296;   // fixed grid: the partial layout and summation order do not depend on the device

__device__ __forceinline__ float enc_warp_sum(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o /= 2) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y (n x 64, in: pre-LayerNorm output, out: its adjoint dy), d (n x 64):
// adjoint of the encoder output, x (n x F): features, gamma (64). Output LN
// adjoint (kernels.cpp:99-126 with the affine scale, the same statistics as
// the forward: two-pass mean / variance, eps 1e-12):
//   n = (y - mean) inv,  dn = d * gamma,
//   dy = inv (dn - mean(dn) - n mean(dn n))
// part[block][(F + 2) x 64]: dW_skip (F x 64, = sum x^T dy), dgamma (= sum d n),
// dbeta (= sum d): each warp owns a fixed strided set of rows, lane L columns
// 2L, 2L + 1; warps are summed in order (deterministic).
__global__ void __launch_bounds__(kEncLnThreads) enc_out_backward_kernel(float* __restrict__ y,
                                                                         const float* __restrict__ d,
                                                                         const float* __restrict__ x, int F,
                                                                         const float* __restrict__ gamma, int64_t n,
                                                                         float* __restrict__ part) {
  constexpr int H = 64;
  __shared__ float red[kEncLnThreads / 32][10 * H];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int c0 = 2 * lane;
  const float g0 = __ldg(gamma + c0), g1 = __ldg(gamma + c0 + 1);
  float ws[8][2], dg[2] = {0.f, 0.f}, db[2] = {0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 8; ++i) ws[i][0] = ws[i][1] = 0.f;
  const int64_t n_warps = (int64_t)gridDim.x * (kEncLnThreads / 32);
  for (int64_t row = (int64_t)blockIdx.x * (kEncLnThreads / 32) + warp; row < n; row += n_warps) {
    float2* yr = reinterpret_cast<float2*>(y + row * H) + lane;
    const float2 yv = *yr;
    const float2 dv = __ldg(reinterpret_cast<const float2*>(d + row * H) + lane);
    const float xv = lane < F ? __ldg(x + row * F + lane) : 0.f;
    const float mean = enc_warp_sum(yv.x + yv.y) * (1.0f / H);
    const float e0 = yv.x - mean, e1 = yv.y - mean;
    const float inv = ptx::rsqrt_fast(enc_warp_sum(fmaf(e0, e0, e1 * e1)) * (1.0f / H) + 1e-12f);
    const float n0 = e0 * inv, n1 = e1 * inv;
    dg[0] = fmaf(dv.x, n0, dg[0]);
    dg[1] = fmaf(dv.y, n1, dg[1]);
    db[0] += dv.x;
    db[1] += dv.y;
    const float dn0 = dv.x * g0, dn1 = dv.y * g1;
    const float m1 = enc_warp_sum(dn0 + dn1) * (1.0f / H);
    const float m2 = enc_warp_sum(fmaf(dn0, n0, dn1 * n1)) * (1.0f / H);
    const float dy0 = (dn0 - m1 - n0 * m2) * inv, dy1 = (dn1 - m1 - n1 * m2) * inv;
    *yr = make_float2(dy0, dy1);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < F) {
        const float xi = __shfl_sync(0xffffffffu, xv, i);
        ws[i][0] = fmaf(xi, dy0, ws[i][0]);
        ws[i][1] = fmaf(xi, dy1, ws[i][1]);
      }
    }
  }
  float* r = red[warp];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i < F) {
      r[i * H + c0] = ws[i][0];
      r[i * H + c0 + 1] = ws[i][1];
    }
  }
  r[F * H + c0] = dg[0];
  r[F * H + c0 + 1] = dg[1];
  r[(F + 1) * H + c0] = db[0];
  r[(F + 1) * H + c0 + 1] = db[1];
  __syncthreads();
  const int n_out = (F + 2) * H;
  for (int j = threadIdx.x; j < n_out; j += kEncLnThreads) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kEncLnThreads / 32; ++w) s += red[w][j];
    part[(int64_t)blockIdx.x * n_out + j] = s;
  }
}

// Decoder skip term (model.cpp:92-101) around the tcgen05 decoder MLP
// (kDecoder): dx += dy W_skip^T on the MLP's input adjoint, and the W_skip
// gradient partials part[block][H x F] (= sum x^T dy; fixed warp / row
// assignment and warp order: deterministic). x, dx: n x 64, dy: n x F (<= 8),
// wskip: 64 x F.
__global__ void __launch_bounds__(kEncLnThreads) dec_skip_backward_kernel(const float* __restrict__ x,
                                                                          const float* __restrict__ dy,
                                                                          const float* __restrict__ wskip, int F,
                                                                          int64_t n, float* __restrict__ dx,
                                                                          float* __restrict__ part) {
  constexpr int H = 64;
  __shared__ float red[kEncLnThreads / 32][8 * H];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int c0 = 2 * lane;
  float w0[8], w1[8], acc0[8], acc1[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    w0[o] = o < F ? __ldg(wskip + c0 * F + o) : 0.f;
    w1[o] = o < F ? __ldg(wskip + (c0 + 1) * F + o) : 0.f;
    acc0[o] = acc1[o] = 0.f;
  }
  const int64_t n_warps = (int64_t)gridDim.x * (kEncLnThreads / 32);
  for (int64_t row = (int64_t)blockIdx.x * (kEncLnThreads / 32) + warp; row < n; row += n_warps) {
    const float dl = lane < F ? __ldg(dy + row * F + lane) : 0.f;
    const float2 xv = __ldg(reinterpret_cast<const float2*>(x + row * H) + lane);
    float2* dr = reinterpret_cast<float2*>(dx + row * H) + lane;
    float2 dv = *dr;
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      if (o < F) {
        const float d = __shfl_sync(0xffffffffu, dl, o);
        dv.x = fmaf(d, w0[o], dv.x);
        dv.y = fmaf(d, w1[o], dv.y);
        acc0[o] = fmaf(xv.x, d, acc0[o]);
        acc1[o] = fmaf(xv.y, d, acc1[o]);
      }
    }
    *dr = dv;
  }
  float* r = red[warp];
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    if (o < F) {
      r[c0 * F + o] = acc0[o];
      r[(c0 + 1) * F + o] = acc1[o];
    }
  }
  __syncthreads();
  const int n_out = H * F;
  for (int j = threadIdx.x; j < n_out; j += kEncLnThreads) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kEncLnThreads / 32; ++w) s += red[w][j];
    part[(int64_t)blockIdx.x * n_out + j] = s;
  }
}

}  // namespace hgnn_b200
