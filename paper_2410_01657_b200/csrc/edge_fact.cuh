// Node-level halves of the factorised edge-MLP input linear (kEdgeFact).
//
// The edge MLP's first linear acts on [x_src | x_dst | e] (edge_concat_filler,
// model.cpp:184-195): h0 = x_src W0_s + x_dst W0_d + e W0_e + b0, W0_s / W0_d /
// W0_e the three H-row blocks of W0 (nn.cpp:139-147). The x terms depend on
// nodes only, so they are computed once per node instead of once per edge:
//   forward   P[i] = [x_i W0_s | x_i W0_d]                 (edge_proj_kernel)
//   backward  with dY_e = dL/dh0_e from the edge kernel,
//             S_src(i) = sum over out-edges of dY = sum_{p in seg(i)} dY[twin p]
//             S_dst(i) = sum over in-edges  of dY = sum_{p in seg(i)} dY[p]
//             dx_i  = dx_node_i + S_src W0_s^T + S_dst W0_d^T   (model.cpp:362-386)
//             dW0_s = sum_i x_i^T S_src(i),  dW0_d = sum_i x_i^T S_dst(i)
// (edge_input_adjoint_kernel): the same sums as the reference's per-edge
// products (nn.cpp:241-281 for the input linear, then the two CSR scatters of
// model.cpp:362-378), regrouped through the nodes — 2/3 of the input linear's
// flops and all per-edge x gathers leave the edge kernels.
// fp32 SIMT; weights staged in shared memory; per-block weight-gradient
// partials (fixed ownership, no atomics) reduced in block order.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "mlp_simt.cuh"

namespace hgnn_b200 {

constexpr int kFactThreads = 256;

// P[i] = x_i [W0_s | W0_d] for local rows i < n. W0 rows 0..2H-1 (in x H,
// row-major) are exactly [W0_s; W0_d].
template <int H>
__global__ void __launch_bounds__(kFactThreads) edge_proj_kernel(const float* __restrict__ x,
                                                                 const float* __restrict__ w0, int64_t n,
                                                                 float* __restrict__ P) {
  constexpr int TPN = 2 * H / 8;                // threads per node (8 outputs each)
  constexpr int NPB = kFactThreads / TPN;       // nodes per block iteration
  __shared__ __align__(16) float ws[2 * H * H];  // [k'][j], k' < 2H: W0_s rows then W0_d rows
  __shared__ __align__(16) float xs[NPB][H];
  for (int i = threadIdx.x; i < 2 * H * H / 4; i += blockDim.x)
    reinterpret_cast<float4*>(ws)[i] = __ldg(reinterpret_cast<const float4*>(w0) + i);
  const int nl = threadIdx.x / TPN, o = threadIdx.x % TPN;
  const int half = (8 * o) / H, j0 = (8 * o) % H;  // output block: P_s or P_d, columns j0..j0+7
  for (int64_t base = (int64_t)blockIdx.x * NPB; base < n; base += (int64_t)gridDim.x * NPB) {
    __syncthreads();
    for (int t = threadIdx.x; t < NPB * H / 4; t += blockDim.x) {
      const int r = t / (H / 4), c = t % (H / 4);
      const int64_t i = base + r;
      reinterpret_cast<float4*>(&xs[r][0])[c] =
          i < n ? __ldg(reinterpret_cast<const float4*>(x + i * H) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
#pragma unroll 4
    for (int k = 0; k < H; ++k) {
      const float xv = xs[nl][k];
      const float4 wa = *reinterpret_cast<const float4*>(&ws[(half * H + k) * H + j0]);
      const float4 wb = *reinterpret_cast<const float4*>(&ws[(half * H + k) * H + j0 + 4]);
      acc[0] = fmaf(xv, wa.x, acc[0]);
      acc[1] = fmaf(xv, wa.y, acc[1]);
      acc[2] = fmaf(xv, wa.z, acc[2]);
      acc[3] = fmaf(xv, wa.w, acc[3]);
      acc[4] = fmaf(xv, wb.x, acc[4]);
      acc[5] = fmaf(xv, wb.y, acc[5]);
      acc[6] = fmaf(xv, wb.z, acc[6]);
      acc[7] = fmaf(xv, wb.w, acc[7]);
    }
    const int64_t i = base + nl;
    if (i < n) {
      float4* out = reinterpret_cast<float4*>(P + i * 2 * H + half * H + j0);
      out[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      out[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
  }
}

// Backward of the node-level input projection, rows [0, rows):
//   dx_i = (i < n_local ? dx_node_i : 0) + S_src W0_s^T + S_dst W0_d^T
// and per-block partials of dW0_s / dW0_d: part[block][0 .. H*H) = dW0_s,
// [H*H .. 2*H*H) = dW0_d (row-major k x j, the layout of W0's row blocks).
template <int H>
__global__ void __launch_bounds__(kFactThreads) edge_input_adjoint_kernel(
    const float* __restrict__ dy, const float* __restrict__ x, const float* __restrict__ dx_node,
    const float* __restrict__ w0, const int32_t* __restrict__ beg, const int32_t* __restrict__ end,
    const int32_t* __restrict__ twin, int64_t rows, int64_t n_local, float* __restrict__ dx,
    float* __restrict__ part) {
  constexpr int NC = kFactThreads / (H / 4);  // nodes per chunk (one float4 column group per thread)
  constexpr int OUT4 = H / 4;                 // dx: threads per node in the product phase = H / 4 (4 outputs each)
  constexpr int NW = 2 * H * H / kFactThreads;  // dW elements per thread (split between s and d)
  __shared__ __align__(16) float wt[2][H][H];   // wt[s][j][k] = W0_s[k][j] (s = 0) / W0_d[k][j] (s = 1)
  __shared__ __align__(16) float ss[2][NC][H];  // S_src, S_dst of the chunk's nodes
  __shared__ __align__(16) float xs[NC][H];
  for (int t = threadIdx.x; t < 2 * H * H; t += blockDim.x) {
    const int s = t / (H * H), k = (t / H) % H, j = t % H;  // coalesced read of W0 row block s
    wt[s][j][k] = __ldg(w0 + t);
  }
  // dW ownership: thread owns (s, k, j0 .. j0 + NW/2) of both blocks? -> element e = threadIdx.x * NW / 2 + q of
  // each block (row-major k x j): NW / 2 consecutive elements per block.
  constexpr int PER = NW / 2;
  const int e0 = threadIdx.x * PER;
  const int wk = e0 / H, wj0 = e0 % H;
  float acc_s[PER], acc_d[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) acc_s[q] = acc_d[q] = 0.f;
  const int nd = threadIdx.x / OUT4, oc = threadIdx.x % OUT4;  // gather / product phase mapping
  for (int64_t base = (int64_t)blockIdx.x * NC; base < rows; base += (int64_t)gridDim.x * NC) {
    __syncthreads();
    {  // segment sums, one float4 column group per thread
      const int64_t i = base + nd;
      float4 s1 = make_float4(0.f, 0.f, 0.f, 0.f), s2 = s1, xv = s1;
      if (i < rows) {
        const int32_t p1 = __ldg(end + i);
        for (int32_t p = __ldg(beg + i); p < p1; ++p) {
          const float4 a = __ldg(reinterpret_cast<const float4*>(dy + (int64_t)__ldg(twin + p) * H) + oc);
          const float4 b = __ldg(reinterpret_cast<const float4*>(dy + (int64_t)p * H) + oc);
          s1 = make_float4(s1.x + a.x, s1.y + a.y, s1.z + a.z, s1.w + a.w);
          s2 = make_float4(s2.x + b.x, s2.y + b.y, s2.z + b.z, s2.w + b.w);
        }
        if (i < n_local) xv = __ldg(reinterpret_cast<const float4*>(x + i * H) + oc);
      }
      reinterpret_cast<float4*>(&ss[0][nd][0])[oc] = s1;
      reinterpret_cast<float4*>(&ss[1][nd][0])[oc] = s2;
      reinterpret_cast<float4*>(&xs[nd][0])[oc] = xv;
    }
    __syncthreads();
    {  // dx = dx_node + S_src W0_s^T + S_dst W0_d^T, 4 outputs per thread
      const int64_t i = base + nd;
      float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
      for (int j = 0; j < H; ++j) {
        const float a = ss[0][nd][j], b = ss[1][nd][j];
        const float4 u = *reinterpret_cast<const float4*>(&wt[0][j][4 * oc]);
        const float4 v = *reinterpret_cast<const float4*>(&wt[1][j][4 * oc]);
        o.x = fmaf(a, u.x, fmaf(b, v.x, o.x));
        o.y = fmaf(a, u.y, fmaf(b, v.y, o.y));
        o.z = fmaf(a, u.z, fmaf(b, v.z, o.z));
        o.w = fmaf(a, u.w, fmaf(b, v.w, o.w));
      }
      if (i < rows) {
        if (i < n_local) {
          const float4 d = __ldg(reinterpret_cast<const float4*>(dx_node + i * H) + oc);
          o = make_float4(o.x + d.x, o.y + d.y, o.z + d.z, o.w + d.w);
        }
        reinterpret_cast<float4*>(dx + i * H)[oc] = o;
      }
    }
    // dW0_s[k][j] += x[k] S_src[j], dW0_d[k][j] += x[k] S_dst[j], nodes in order
#pragma unroll 2
    for (int n = 0; n < NC; ++n) {
      const float xk = xs[n][wk];
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        acc_s[q] = fmaf(xk, ss[0][n][wj0 + q], acc_s[q]);
        acc_d[q] = fmaf(xk, ss[1][n][wj0 + q], acc_d[q]);
      }
    }
  }
  float* ps = part + (int64_t)blockIdx.x * 2 * H * H;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    ps[e0 + q] = acc_s[q];
    ps[H * H + e0 + q] = acc_d[q];
  }
}

// out[i] += sum_b part[b][i] in block order (fp64): the node-level W0_s / W0_d
// gradient blocks on top of the edge kernel's reduction (deterministic).
__global__ void grad_reduce_add_kernel(const float* __restrict__ partial, int64_t n_blocks, int64_t n,
                                       double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t b = 0; b < n_blocks; ++b) s += (double)__ldg(partial + b * n + i);
  out[i] += s;
}

// Zero the rows of a that the fused edge kernel never writes (empty receiver
// segments: halo rows and isolated nodes; scatter_rows_csr writes 0 there).
__global__ void zero_rows_kernel(const int32_t* __restrict__ rows_idx, int64_t n, int H, float* __restrict__ a) {
  const int q = H / 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * q) return;
  reinterpret_cast<float4*>(a + (int64_t)__ldg(rows_idx + tid / q) * H)[tid % q] = make_float4(0.f, 0.f, 0.f, 0.f);
}

}  // namespace hgnn_b200
