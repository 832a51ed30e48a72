// Model-level element-wise kernels (sm_100a): consistent loss and its
// adjoint, gradient averaging, Adam, and the on-device refresh of the fp32 /
// tf32-split parameter images after an optimizer step.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hgnn_b200 {

constexpr int kLossThreads = 256;
constexpr int kLossBlocks = 296;  // fixed grid: the fp64 reduction order does not depend on the device

// Per-block partial sums of the consistent loss (model.cpp:455-480):
//   s = sum_i inv_d_i sum_j (y_ij - t_ij)^2,   n = sum_i inv_d_i   (fp64)
__global__ void loss_partial_kernel(const float* __restrict__ y, const float* __restrict__ t,
                                    const double* __restrict__ inv_d, int64_t n_rows, int cols,
                                    double* __restrict__ part) {
  __shared__ double ss[kLossThreads], sn[kLossThreads];
  double s = 0.0, n = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kLossThreads + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * kLossThreads) {
    double row = 0.0;
    for (int j = 0; j < cols; ++j) {
      const double d = (double)y[i * cols + j] - (double)t[i * cols + j];
      row += d * d;
    }
    s += inv_d[i] * row;
    n += inv_d[i];
  }
  ss[threadIdx.x] = s;
  sn[threadIdx.x] = n;
  __syncthreads();
  for (int w = kLossThreads / 2; w > 0; w /= 2) {
    if (threadIdx.x < w) {
      ss[threadIdx.x] += ss[threadIdx.x + w];
      sn[threadIdx.x] += sn[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = ss[0];
    part[2 * blockIdx.x + 1] = sn[0];
  }
}
// out[0..1] = fixed-order sums of the block partials
__global__ void loss_final_kernel(const double* __restrict__ part, int nblocks, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double s = 0.0, n = 0.0;
    for (int b = 0; b < nblocks; ++b) {
      s += part[2 * b];
      n += part[2 * b + 1];
    }
    out[0] = s;
    out[1] = n;
  }
}

// d_y = 2 seed inv_d_i (y - t)   (model.cpp:482-500); seed on the device
__global__ void loss_backward_kernel(const float* __restrict__ y, const float* __restrict__ t,
                                     const double* __restrict__ inv_d, const double* __restrict__ seed,
                                     int64_t n_rows, int cols, float* __restrict__ dy) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows * cols) return;
  const int64_t r = i / cols;
  dy[i] = (float)(2.0 * seed[0] * inv_d[r] * ((double)y[i] - (double)t[i]));
}

// seed = R / (n_eff * cols): the reference all-reduces the same local seed
// 1 / (n_eff cols) over R ranks (model.cpp:487-489).
__global__ void loss_seed_kernel(double* __restrict__ st, int cols, int nranks) {
  if (threadIdx.x == 0) st[2] = (double)nranks / (st[1] * (double)cols);
}

__global__ void scale_f64_kernel(double* __restrict__ v, int64_t n, double s) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] *= s;
}

// fp32 partials [blocks][stride] -> dst[n] (fp64, n <= stride), fixed block order
__global__ void reduce_partials_kernel(const float* __restrict__ part, int64_t blocks, int64_t n,
                                       double* __restrict__ dst, int64_t stride) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t b = 0; b < blocks; ++b) s += (double)part[b * stride + i];
  dst[i] = s;
}

// Bias-corrected Adam (nn.cpp:331-360), fp64 master parameters; flags any
// non-finite gradient (OptimizerError in the reference).
// Pass 1 of adam_step (nn.cpp:331-360): flag any non-finite gradient. The
// reference throws before touching a parameter, so the update runs only when
// this pass found none (all state stays consistent on failure).
__global__ void nonfinite_kernel(const double* __restrict__ g, int64_t n, int* __restrict__ nonfinite) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !isfinite(g[i])) atomicExch(nonfinite, 1);
}

__global__ void adam_kernel(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                            double* __restrict__ v, int64_t n, double lr, double b1, double b2, double eps,
                            double bc1, double bc2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double gi = g[i];
  const double mi = b1 * m[i] + (1.0 - b1) * gi;
  const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  p[i] -= lr * (mi / bc1) / (sqrt(vi / bc2) + eps);
}

__global__ void f64_to_f32_kernel(const double* __restrict__ src, int64_t n, float* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (float)src[i];
}

// dst[i] = (float) src[map[i]]   (transposed weight copies)
__global__ void gather_f64_to_f32_kernel(const double* __restrict__ src, const int32_t* __restrict__ map, int64_t n,
                                         float* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (float)src[map[i]];
}

// Round to nearest tf32, ties away (same bits as the host chunk builder).
__device__ __forceinline__ float tf32_rna_bits(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
// chunk[i] = hi or lo tf32 part of (float) src[map[i] & 0x7fffffff]; bit 31 = lo
__global__ void chunk_refresh_kernel(const double* __restrict__ src, const uint32_t* __restrict__ map, int64_t n,
                                     float* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t m = map[i];
  if (m == 0x7fffffffu) {  // zero padding (the encoders' F-feature input segment)
    dst[i] = 0.f;
    return;
  }
  const float w = (float)src[m & 0x7fffffffu];
  const float hi = tf32_rna_bits(w);
  dst[i] = (m >> 31) ? tf32_rna_bits(w - hi) : hi;
}

}  // namespace hgnn_b200
