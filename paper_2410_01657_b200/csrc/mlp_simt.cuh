// Row-parallel processor-MLP kernels (SIMT fp32, sm_100a), forward and
// backward-with-recompute, for the edge update (input [x_src | x_dst | e]) and
// the node update (input [a* | x]).
//
// MLP (nn.hpp:14-26, processor spec model.cpp:82-90):
//   h = A W0 + b0;  h += ELU(LN0(h Wj + bj)) for j = 1..k;  y = h W_{k+1} + b_{k+1}
// One thread owns one row. Its residual stream lives in a private column of
// shared memory ([feature][row] layout: conflict-free, no register spills);
// the accumulator of the current linear lives in registers; weights are read
// as warp-uniform broadcasts (shared memory when they fit, else L1).
// Weight gradients are reduced per tile through two column-staged shared
// buffers and accumulated into a per-CTA partial (fixed thread ownership, no
// atomics), so results are deterministic run to run.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hgnn_b200 {

constexpr int kMlpThreads = 128;
constexpr int kColPad = 4;  // column stride kMlpThreads + 4: conflict-free LDS.128 (see dw_accumulate)
constexpr int kColStride = kMlpThreads + kColPad;

// kEdgeFact: the edge MLP with its input linear factorised through the nodes,
// [x_src | x_dst | e] W0 = P_s[src] + P_d[dst] + e W0_e with P = x [W0_s | W0_d]
// computed once per node (tensor-core kernels only; same parameters).
// kEdgeFused: kEdgeInput's 3-segment input with the aggregate formed in the
// same kernel (tensor-core forward only).
enum MlpInput : int { kEdgeInput = 0, kNodeInput = 1, kEdgeFact = 2, kEdgeFused = 3, kEncoder = 4, kDecoder = 5 };

// Flattened processor-MLP parameters (for_each order, fp32): W0 (in x H), b0,
// W1, b1, ..., W_{k+1}, b_{k+1}. wt points at the same list with every W
// transposed (out x in), used by the adjoint products.
struct MlpParamsDev {
  const float* p;
  const float* wt;
  int k;
  int in_dim;
};

__host__ __device__ inline int64_t mlp_param_count(int in_dim, int H, int k) {
  return (int64_t)in_dim * H + H + (int64_t)k * (H * H + H) + (int64_t)H * H + H;
}
__host__ __device__ inline int64_t mlp_w_offset(int l, int in_dim, int H) {
  return l == 0 ? 0 : (int64_t)in_dim * H + H + (int64_t)(l - 1) * (H * H + H);
}
__host__ __device__ inline int64_t mlp_b_offset(int l, int in_dim, int H) {
  return mlp_w_offset(l, in_dim, H) + (l == 0 ? (int64_t)in_dim * H : (int64_t)H * H);
}

// Arguments shared by the forward and backward kernels.
struct MlpRowArgs {
  int64_t n_rows;
  // edge input: rows are receiver-sorted edge slots p
  const int32_t* src;
  const int32_t* dst;
  const float* x;      // node features (rows x H)
  const float* e_in;   // edge features (n_rows x H), edge mode
  const float* a;      // synchronized aggregate (node mode)
  // forward output
  float* out;
  // backward
  const float* d_out;     // node mode: dx (rows x H)
  const float* inv_deg;   // edge mode: 1/d per slot
  const float* d_a;       // edge mode: aggregate adjoint (rows x H)
  float* de_io;           // edge mode: in: de, out: de_next (in place)
  float* d_src;           // edge mode: adjoint of x_src (n_rows x H)
  float* d_dst;           // edge mode: adjoint of x_dst (n_rows x H)
  float* d_a_out;         // node mode: adjoint of a* (rows x H)
  float* d_x_out;         // node mode: adjoint of x (n_rows x H)
  float* grad_partial;    // [gridDim.x][param_count] fp32
  float* scratch;         // [gridDim.x][slots][kMlpThreads]
  int64_t n_slots;        // scratch slots per row
};

// acc[j] = sum_t col[t*kColStride] * W[t*H + j]   (one row, t ascending)
template <int H>
__device__ __forceinline__ void gemm_row(float (&acc)[H], const float* __restrict__ col, const float* __restrict__ W,
                                         int K) {
#pragma unroll 2
  for (int t = 0; t < K; ++t) {
    const float hv = col[t * kColStride];
    const float4* w4 = reinterpret_cast<const float4*>(W + (int64_t)t * H);
#pragma unroll
    for (int j = 0; j < H / 4; ++j) {
      const float4 w = w4[j];
      acc[4 * j + 0] = fmaf(hv, w.x, acc[4 * j + 0]);
      acc[4 * j + 1] = fmaf(hv, w.y, acc[4 * j + 1]);
      acc[4 * j + 2] = fmaf(hv, w.z, acc[4 * j + 2]);
      acc[4 * j + 3] = fmaf(hv, w.w, acc[4 * j + 3]);
    }
  }
}

// Same product with the input row streamed from global memory (first linear).
template <int H>
__device__ __forceinline__ void gemm_row_global(float (&acc)[H], const float* __restrict__ in,
                                                const float* __restrict__ W) {
#pragma unroll 1
  for (int t4 = 0; t4 < H / 4; ++t4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(in) + t4);
    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4* w4 = reinterpret_cast<const float4*>(W + (int64_t)(4 * t4 + u) * H);
#pragma unroll
      for (int j = 0; j < H / 4; ++j) {
        const float4 w = w4[j];
        acc[4 * j + 0] = fmaf(vv[u], w.x, acc[4 * j + 0]);
        acc[4 * j + 1] = fmaf(vv[u], w.y, acc[4 * j + 1]);
        acc[4 * j + 2] = fmaf(vv[u], w.z, acc[4 * j + 2]);
        acc[4 * j + 3] = fmaf(vv[u], w.w, acc[4 * j + 3]);
      }
    }
  }
}

// Parameter-free LayerNorm (kernels.cpp:81-94, eps nn.hpp:65) in place;
// returns inv_std. Two-pass mean / variance as in the reference.
template <int H>
__device__ __forceinline__ float ln0_inplace(float (&v)[H]) {
  float mean = 0.f;
#pragma unroll
  for (int j = 0; j < H; ++j) mean += v[j];
  mean /= (float)H;
  float var = 0.f;
#pragma unroll
  for (int j = 0; j < H; ++j) {
    const float d = v[j] - mean;
    var = fmaf(d, d, var);
  }
  var /= (float)H;
  const float inv_std = 1.0f / sqrtf(var + 1e-12f);
#pragma unroll
  for (int j = 0; j < H; ++j) v[j] = (v[j] - mean) * inv_std;
  return inv_std;
}

__device__ __forceinline__ float elu1(float z) { return z > 0.f ? z : expm1f(z); }

// Pointer to the first-linear input segment `seg` of row `r`.
template <int H, int MODE>
__device__ __forceinline__ const float* input_segment(const MlpRowArgs& a, int64_t r, int seg) {
  if (MODE == kEdgeInput) {
    if (seg == 0) return a.x + (int64_t)__ldg(a.src + r) * H;
    if (seg == 1) return a.x + (int64_t)__ldg(a.dst + r) * H;
    return a.e_in + r * H;
  }
  return seg == 0 ? a.a + r * H : a.x + r * H;
}

// Copies all weights+biases into shared memory (when they fit).
__device__ __forceinline__ void stage_params(float* dst, const float* __restrict__ src, int64_t n) {
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int64_t i = threadIdx.x; i < n / 4; i += blockDim.x) d4[i] = __ldg(s4 + i);
  for (int64_t i = (n / 4) * 4 + threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldg(src + i);
}

// --------------------------------------------------------------------------
// forward
// --------------------------------------------------------------------------
// smem: [params if W_SMEM][H x kColStride private residual columns]
template <int H, int MODE, bool W_SMEM>
__global__ void __launch_bounds__(kMlpThreads) mlp_forward_kernel(MlpRowArgs a, MlpParamsDev prm) {
  extern __shared__ __align__(16) float smem[];
  const int nseg = MODE == kEdgeInput ? 3 : 2;
  const int in_dim = nseg * H;
  const int64_t n_par = mlp_param_count(in_dim, H, prm.k);
  const float* P = prm.p;
  float* col_base = smem;
  if (W_SMEM) {
    stage_params(smem, prm.p, n_par);
    P = smem;
    col_base = smem + ((n_par + 3) / 4) * 4;
    __syncthreads();
  }
  float* col = col_base + threadIdx.x;  // this thread's residual column
  const int64_t n_tiles = (a.n_rows + kMlpThreads - 1) / kMlpThreads;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t r = tile * kMlpThreads + threadIdx.x;
    if (r >= a.n_rows) continue;
    float acc[H];
    // input projection
#pragma unroll
    for (int j = 0; j < H; ++j) acc[j] = 0.f;
    for (int seg = 0; seg < nseg; ++seg)
      gemm_row_global<H>(acc, input_segment<H, MODE>(a, r, seg), P + (int64_t)seg * H * H);
    {
      const float* b0 = P + mlp_b_offset(0, in_dim, H);
#pragma unroll
      for (int j = 0; j < H; ++j) col[j * kColStride] = acc[j] + b0[j];
    }
    // residual blocks
    for (int l = 1; l <= prm.k; ++l) {
#pragma unroll
      for (int j = 0; j < H; ++j) acc[j] = 0.f;
      gemm_row<H>(acc, col, P + mlp_w_offset(l, in_dim, H), H);
      const float* b = P + mlp_b_offset(l, in_dim, H);
#pragma unroll
      for (int j = 0; j < H; ++j) acc[j] += b[j];
      ln0_inplace<H>(acc);
#pragma unroll
      for (int j = 0; j < H; ++j) col[j * kColStride] = elu1(acc[j]) + col[j * kColStride];
    }
    // output projection
#pragma unroll
    for (int j = 0; j < H; ++j) acc[j] = 0.f;
    gemm_row<H>(acc, col, P + mlp_w_offset(prm.k + 1, in_dim, H), H);
    const float* bo = P + mlp_b_offset(prm.k + 1, in_dim, H);
    float4* o4 = reinterpret_cast<float4*>(a.out + r * H);
#pragma unroll
    for (int j = 0; j < H / 4; ++j)
      o4[j] = make_float4(acc[4 * j] + bo[4 * j], acc[4 * j + 1] + bo[4 * j + 1], acc[4 * j + 2] + bo[4 * j + 2],
                          acc[4 * j + 3] + bo[4 * j + 3]);
  }
}

// --------------------------------------------------------------------------
// backward
// --------------------------------------------------------------------------

// gW[i][j] += sum_r hcol[i][r] * dcol[j][r]  over the tile's rows,
// gb[j] += sum_r dcol[j][r]. Thread t owns i in {t/8 + 16u}, j in {t%8 + 8v}.
template <int H>
__device__ __forceinline__ void dw_accumulate(const float* hcol, const float* dcol, int rows4, float* gW,
                                              float* gb) {
  static_assert(H % 8 == 0 && H <= 128, "hidden width must be a multiple of 8");
  constexpr int IU = H >= 16 ? H / 16 : 1;  // i values per thread
  constexpr int JV = H / 8;                 // j values per thread
  const int t = threadIdx.x;
  const int i0 = t / 8, j0 = t % 8;
  if (H >= 16 || i0 < H) {
    float acc[IU][JV];
#pragma unroll
    for (int u = 0; u < IU; ++u)
#pragma unroll
      for (int v = 0; v < JV; ++v) acc[u][v] = 0.f;
    for (int r = 0; r < rows4; r += 4) {
      float4 hv[IU], dv[JV];
#pragma unroll
      for (int u = 0; u < IU; ++u) hv[u] = *reinterpret_cast<const float4*>(hcol + (i0 + 16 * u) * kColStride + r);
#pragma unroll
      for (int v = 0; v < JV; ++v) dv[v] = *reinterpret_cast<const float4*>(dcol + (j0 + 8 * v) * kColStride + r);
#pragma unroll
      for (int u = 0; u < IU; ++u)
#pragma unroll
        for (int v = 0; v < JV; ++v) {
          acc[u][v] = fmaf(hv[u].x, dv[v].x, acc[u][v]);
          acc[u][v] = fmaf(hv[u].y, dv[v].y, acc[u][v]);
          acc[u][v] = fmaf(hv[u].z, dv[v].z, acc[u][v]);
          acc[u][v] = fmaf(hv[u].w, dv[v].w, acc[u][v]);
        }
    }
#pragma unroll
    for (int u = 0; u < IU; ++u)
#pragma unroll
      for (int v = 0; v < JV; ++v) gW[(int64_t)(i0 + 16 * u) * H + (j0 + 8 * v)] += acc[u][v];
  }
  if (gb && t < H) {
    float s = 0.f;
    for (int r = 0; r < rows4; ++r) s += dcol[t * kColStride + r];
    gb[t] += s;
  }
}

// smem: [params if W_SMEM][hcol H x kColStride][dcol H x kColStride]
// scratch slots per row: hidden[0..k] (H each), normed[1..k] (H each), inv_std[1..k]
template <int H, int MODE, bool W_SMEM>
__global__ void __launch_bounds__(kMlpThreads) mlp_backward_kernel(MlpRowArgs a, MlpParamsDev prm) {
  extern __shared__ __align__(16) float smem[];
  const int nseg = MODE == kEdgeInput ? 3 : 2;
  const int in_dim = nseg * H;
  const int k = prm.k;
  const int64_t n_par = mlp_param_count(in_dim, H, k);
  const float* P = prm.p;
  const float* PT = prm.wt;
  float* base = smem;
  if (W_SMEM) {
    stage_params(smem, prm.p, n_par);
    P = smem;
    base = smem + ((n_par + 3) / 4) * 4;
  }
  float* hcol_all = base;
  float* dcol_all = base + H * kColStride;
  // zero unused tail columns once so partial tiles reduce exact zeros
  for (int i = threadIdx.x; i < 2 * H * kColStride; i += blockDim.x) base[i] = 0.f;
  __syncthreads();
  float* hcol = hcol_all + threadIdx.x;
  float* dcol = dcol_all + threadIdx.x;
  float* gpart = a.grad_partial + (int64_t)blockIdx.x * n_par;
  float* scr = a.scratch + (int64_t)blockIdx.x * a.n_slots * kMlpThreads + threadIdx.x;
  const int64_t n_tiles = (a.n_rows + kMlpThreads - 1) / kMlpThreads;

  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t r = tile * kMlpThreads + threadIdx.x;
    const bool live = r < a.n_rows;
    const int64_t left = a.n_rows - tile * kMlpThreads;
    const int rows_in_tile = left < kMlpThreads ? (int)left : kMlpThreads;
    const int rows4 = (rows_in_tile + 3) & ~3;
    float acc[H];
    // ---- recompute the forward pass (nn.cpp:226-227), saving the stream
    if (live) {
#pragma unroll
      for (int j = 0; j < H; ++j) acc[j] = 0.f;
      for (int seg = 0; seg < nseg; ++seg)
        gemm_row_global<H>(acc, input_segment<H, MODE>(a, r, seg), P + (int64_t)seg * H * H);
      const float* b0 = P + mlp_b_offset(0, in_dim, H);
#pragma unroll
      for (int j = 0; j < H; ++j) {
        const float h = acc[j] + b0[j];
        hcol[j * kColStride] = h;
        scr[(int64_t)j * kMlpThreads] = h;
      }
      for (int l = 1; l <= k; ++l) {
#pragma unroll
        for (int j = 0; j < H; ++j) acc[j] = 0.f;
        gemm_row<H>(acc, hcol, P + mlp_w_offset(l, in_dim, H), H);
        const float* b = P + mlp_b_offset(l, in_dim, H);
#pragma unroll
        for (int j = 0; j < H; ++j) acc[j] += b[j];
        const float inv_std = ln0_inplace<H>(acc);
        float* s_t = scr + ((int64_t)(k + 1) * H + (int64_t)(l - 1) * H) * kMlpThreads;
        scr[((int64_t)(k + 1) * H + (int64_t)k * H + (l - 1)) * kMlpThreads] = inv_std;
#pragma unroll
        for (int j = 0; j < H; ++j) {
          s_t[(int64_t)j * kMlpThreads] = acc[j];
          const float h = elu1(acc[j]) + hcol[j * kColStride];
          hcol[j * kColStride] = h;
          scr[((int64_t)l * H + j) * kMlpThreads] = h;
        }
      }
      // ---- output adjoint d_y
      if (MODE == kEdgeInput) {
        const float s = __ldg(a.inv_deg + r);
        const float* da = a.d_a + (int64_t)__ldg(a.dst + r) * H;
        const float* de = a.de_io + r * H;
#pragma unroll
        for (int j = 0; j < H; ++j) acc[j] = fmaf(s, da[j], de[j]);  // model.cpp:354-360
      } else {
        const float* dy = a.d_out + r * H;
#pragma unroll
        for (int j = 0; j < H; ++j) acc[j] = dy[j];
      }
#pragma unroll
      for (int j = 0; j < H; ++j) dcol[j * kColStride] = acc[j];
    } else {
#pragma unroll
      for (int j = 0; j < H; ++j) {
        hcol[j * kColStride] = 0.f;
        dcol[j * kColStride] = 0.f;
      }
    }
    __syncthreads();
    // ---- output projection (nn.cpp:241-245)
    dw_accumulate<H>(hcol_all, dcol_all, rows4, gpart + mlp_w_offset(k + 1, in_dim, H),
                     gpart + mlp_b_offset(k + 1, in_dim, H));
    __syncthreads();
    if (live) {
#pragma unroll
      for (int j = 0; j < H; ++j) acc[j] = 0.f;
      gemm_row<H>(acc, dcol, PT + mlp_w_offset(k + 1, in_dim, H), H);  // d_h = d_y W^T
    }
    // ---- residual blocks in reverse (nn.cpp:259-274)
    for (int l = k; l >= 1; --l) {
      if (live) {
        const float* s_t = scr + ((int64_t)(k + 1) * H + (int64_t)(l - 1) * H) * kMlpThreads;
        const float inv_std = scr[((int64_t)(k + 1) * H + (int64_t)k * H + (l - 1)) * kMlpThreads];
        float g_mean = 0.f, gx_mean = 0.f;
        float dt[H];
#pragma unroll
        for (int j = 0; j < H; ++j) {
          const float tj = s_t[(int64_t)j * kMlpThreads];
          dt[j] = acc[j] * (tj > 0.f ? 1.f : expf(tj));  // elu', kernels.cpp:68-71
          g_mean += dt[j];
          gx_mean = fmaf(dt[j], tj, gx_mean);
        }
        g_mean /= (float)H;
        gx_mean /= (float)H;
#pragma unroll
        for (int j = 0; j < H; ++j) {
          const float tj = s_t[(int64_t)j * kMlpThreads];
          dcol[j * kColStride] = (dt[j] - g_mean - tj * gx_mean) * inv_std;  // kernels.cpp:99-126
          hcol[j * kColStride] = scr[((int64_t)(l - 1) * H + j) * kMlpThreads];
        }
      }
      __syncthreads();
      dw_accumulate<H>(hcol_all, dcol_all, rows4, gpart + mlp_w_offset(l, in_dim, H),
                       gpart + mlp_b_offset(l, in_dim, H));
      __syncthreads();
      if (live) gemm_row<H>(acc, dcol, PT + mlp_w_offset(l, in_dim, H), H);  // d_h += d_u W^T
    }
    // ---- input projection (nn.cpp:277-281)
    if (live) {
#pragma unroll
      for (int j = 0; j < H; ++j) dcol[j * kColStride] = acc[j];
    }
    for (int seg = 0; seg < nseg; ++seg) {
      if (live) {
        const float* in = input_segment<H, MODE>(a, r, seg);
#pragma unroll
        for (int j = 0; j < H; ++j) hcol[j * kColStride] = __ldg(in + j);
      }
      __syncthreads();
      dw_accumulate<H>(hcol_all, dcol_all, rows4, gpart + (int64_t)seg * H * H,
                       seg == 0 ? gpart + mlp_b_offset(0, in_dim, H) : nullptr);
      __syncthreads();
    }
    if (live) {
      // d_in = d_h W0^T, written segment by segment
      for (int seg = 0; seg < nseg; ++seg) {
        float o[H];
#pragma unroll
        for (int j = 0; j < H; ++j) o[j] = 0.f;
        // W0^T is (H x in_dim): row t holds W0[:, t]; segment columns [seg*H, seg*H+H)
#pragma unroll 2
        for (int t = 0; t < H; ++t) {
          const float dv = dcol[t * kColStride];
          const float4* w4 = reinterpret_cast<const float4*>(PT + (int64_t)t * in_dim + seg * H);
#pragma unroll
          for (int j = 0; j < H / 4; ++j) {
            const float4 w = w4[j];
            o[4 * j + 0] = fmaf(dv, w.x, o[4 * j + 0]);
            o[4 * j + 1] = fmaf(dv, w.y, o[4 * j + 1]);
            o[4 * j + 2] = fmaf(dv, w.z, o[4 * j + 2]);
            o[4 * j + 3] = fmaf(dv, w.w, o[4 * j + 3]);
          }
        }
        float* dst;
        if (MODE == kEdgeInput) dst = seg == 0 ? a.d_src + r * H : (seg == 1 ? a.d_dst + r * H : a.de_io + r * H);
        else dst = seg == 0 ? a.d_a_out + r * H : a.d_x_out + r * H;
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int j = 0; j < H / 4; ++j) d4[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
      }
    }
    __syncthreads();
  }
}

}  // namespace hgnn_b200
