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
constexpr int kFactRows = 64;  // nodes per block iteration

// P[i] = x_i [W0_s | W0_d] for local rows i < n. W0 rows 0..2H-1 (in x H,
// row-major) are exactly [W0_s; W0_d]: P = X W with W = [W0_s | W0_d] (H x 2H).
// Register-blocked: warp w owns nodes 8 w .. 8 w + 7 of the 64-node tile, lane
// l outputs 4 l .. 4 l + 3; per k one broadcast pair of 16-byte loads (8 x
// values, from the transposed tile) and one 16-byte weight load feed 32 FMAs.
template <int H>
__global__ void __launch_bounds__(kFactThreads) edge_proj_kernel(const float* __restrict__ x,
                                                                 const float* __restrict__ w0, int64_t n,
                                                                 float* __restrict__ P) {
  static_assert(H == 64, "the factorised edge path is built for H = 64");
  constexpr int NO = 2 * H;              // outputs per node (= 4 x 32 lanes)
  constexpr int XS = kFactRows + 4;      // transposed tile row stride
  extern __shared__ __align__(16) float fsm[];
  float* ws = fsm;                       // [k][NO]: W[k][o] = (o < H ? W0_s[k][o] : W0_d[k][o - H])
  float* xt = fsm + H * NO;              // [k][XS]: x transposed
  for (int t = threadIdx.x; t < H * NO; t += blockDim.x) {
    const int k = t / NO, o = t % NO;
    ws[t] = __ldg(w0 + (int64_t)((o < H ? 0 : H) + k) * H + (o % H));
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int64_t base = (int64_t)blockIdx.x * kFactRows; base < n; base += (int64_t)gridDim.x * kFactRows) {
    __syncthreads();
    // lanes walk rows (conflict-free transposed stores); the other column
    // pieces of each row are read by the neighbouring warps from L1
    for (int t = threadIdx.x; t < kFactRows * H / 4; t += blockDim.x) {
      const int r = t % kFactRows, c = t / kFactRows;
      const float4 v = base + r < n ? __ldg(reinterpret_cast<const float4*>(x + (base + r) * H) + c)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      xt[(4 * c) * XS + r] = v.x;
      xt[(4 * c + 1) * XS + r] = v.y;
      xt[(4 * c + 2) * XS + r] = v.z;
      xt[(4 * c + 3) * XS + r] = v.w;
    }
    __syncthreads();
    float acc[8][4];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[a][q] = 0.f;
#pragma unroll 4
    for (int k = 0; k < H; ++k) {
      const float4 x0 = *reinterpret_cast<const float4*>(xt + k * XS + 8 * warp);
      const float4 x1 = *reinterpret_cast<const float4*>(xt + k * XS + 8 * warp + 4);
      const float xa[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      const float4 wv = *reinterpret_cast<const float4*>(ws + k * NO + 4 * lane);
      const float w[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[a][q] = fmaf(xa[a], w[q], acc[a][q]);
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int64_t i = base + 8 * warp + a;
      if (i < n)
        *reinterpret_cast<float4*>(P + i * NO + 4 * lane) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
    }
  }
}
template <int H>
constexpr size_t edge_proj_smem() { return (size_t)(H * 2 * H + H * (kFactRows + 4)) * 4; }

// Backward of the node-level input projection, rows [0, rows), 64 per block
// iteration:
//   S = [S_src | S_dst] (segment sums of dY through the twin / slot index)
//   dx_i = (i < n_local ? dx_node_i : 0) + S_i [W0_s^T ; W0_d^T]
//   dW[k][j] += sum_i x_i[k] S_i[j]  (j < H: dW0_s, j >= H: dW0_d)
// per-block partials part[block][k * 2H + j] (fixed ownership, nodes in
// order): reduced in block order by grad_reduce_add_kernel after a reorder
// into W0's row layout (k x H blocks).
// PRE_S: the segment sums come precomputed (seg_sum_kernel, rows x 2H in
// `pre_s`) and are read as coalesced rows instead of gathered here.
template <int H, bool PRE_S = false>
__global__ void __launch_bounds__(kFactThreads) edge_input_adjoint_kernel(
    const float* __restrict__ dy, const float* __restrict__ x, const float* __restrict__ dx_node,
    const float* __restrict__ w0, const int32_t* __restrict__ beg, const int32_t* __restrict__ end,
    const int32_t* __restrict__ twin, int64_t rows, int64_t n_local, float* __restrict__ dx,
    float* __restrict__ part, const float* __restrict__ pre_s = nullptr) {
  static_assert(H == 64, "the factorised edge path is built for H = 64");
  constexpr int NS = 2 * H;  // S width
  constexpr int WK = 4;      // dW: thread owns 4 k-rows x 8 j-columns (16 x 16 thread grid)
  constexpr int WJ = 8;
  extern __shared__ __align__(16) float fsm[];
  float* wt = fsm;                  // [j][o] (j < 2H, o < H): W0_s[o][j] (j < H), W0_d[o][j - H]
  float* sr = wt + NS * H;          // [r][NS]: S rows
  float* xr = sr + kFactRows * NS;  // [r][H]: x rows
  for (int t = threadIdx.x; t < NS * H; t += blockDim.x) {
    const int j = t / H, o = t % H;
    wt[t] = __ldg(w0 + (int64_t)((j < H ? 0 : H) + o) * H + (j % H));
  }
  const int g16 = threadIdx.x / 16, l16 = threadIdx.x % 16;
  float accw[WK][WJ];
#pragma unroll
  for (int a = 0; a < WK; ++a)
#pragma unroll
    for (int b = 0; b < WJ; ++b) accw[a][b] = 0.f;
  for (int64_t base = (int64_t)blockIdx.x * kFactRows; base < rows; base += (int64_t)gridDim.x * kFactRows) {
    __syncthreads();
    if (PRE_S) {
      for (int t = threadIdx.x; t < kFactRows * NS / 4; t += blockDim.x) {
        const int r = t / (NS / 4), c4 = t % (NS / 4);
        const int64_t i = base + r;
        *reinterpret_cast<float4*>(sr + r * NS + 4 * c4) =
            i < rows ? __ldg(reinterpret_cast<const float4*>(pre_s + i * NS) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else
    // segment sums, item (r, c4): lanes 0-15 of a warp read the twin row
    // (S_src), lanes 16-31 the slot row (S_dst): 256-byte coalesced pieces.
    // A thread owns column piece c4 of rows r0, r0 + 8, ..., r0 + 56 and walks
    // their 8 segments together, slot offset u at a time: 8 independent
    // twin-index -> dY-row load pairs in flight (each row still summed in slot
    // order; slots past a segment's end add +0, which leaves the sum bitwise
    // unchanged since it starts at +0 and never becomes -0).
    {
      static_assert(kFactThreads == 256 && kFactRows == 64 && NS / 4 == 32, "item layout: 8 rows per thread");
      const int c4 = threadIdx.x % (NS / 4), r0 = threadIdx.x / (NS / 4);
      const bool src_half = c4 < H / 4;
      const int cc = src_half ? c4 : c4 - H / 4;
      int32_t pb[8], pe[8];
      float4 s[8];
      int maxd = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t i = base + r0 + 8 * j;
        pb[j] = i < rows ? __ldg(beg + i) : 0;
        pe[j] = i < rows ? __ldg(end + i) : 0;
        s[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        maxd = max(maxd, pe[j] - pb[j]);
      }
      // the twin indices of slot offset u + 1 load while the dY rows of u do
      int32_t tw[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) tw[j] = (src_half && pb[j] < pe[j]) ? __ldg(twin + pb[j]) : 0;
      for (int u = 0; u < maxd; ++u) {
        int64_t e[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          e[j] = pb[j] + u < pe[j] ? (src_half ? (int64_t)tw[j] : (int64_t)(pb[j] + u)) : (int64_t)-1;
          tw[j] = (src_half && pb[j] + u + 1 < pe[j]) ? __ldg(twin + pb[j] + u + 1) : 0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v =
              e[j] >= 0 ? __ldg(reinterpret_cast<const float4*>(dy + e[j] * H) + cc) : make_float4(0.f, 0.f, 0.f, 0.f);
          s[j] = make_float4(s[j].x + v.x, s[j].y + v.y, s[j].z + v.z, s[j].w + v.w);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) *reinterpret_cast<float4*>(sr + (r0 + 8 * j) * NS + 4 * c4) = s[j];
    }
    for (int t = threadIdx.x; t < kFactRows * H / 4; t += blockDim.x) {
      const int r = t / (H / 4), c = t % (H / 4);
      const int64_t i = base + r;
      *reinterpret_cast<float4*>(xr + r * H + 4 * c) =
          i < n_local ? __ldg(reinterpret_cast<const float4*>(x + i * H) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    {  // dx: thread = nodes 4 g16 .. +3 x outputs 4 l16 .. +3
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[a][q] = 0.f;
#pragma unroll 4
      for (int j = 0; j < NS; ++j) {
        float sa[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) sa[a] = sr[(4 * g16 + a) * NS + j];
        const float4 wv = *reinterpret_cast<const float4*>(wt + j * H + 4 * l16);
        const float w[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[a][q] = fmaf(sa[a], w[q], acc[a][q]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int64_t i = base + 4 * g16 + a;
        if (i < rows) {
          float4 o = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
          if (i < n_local) {
            const float4 d = __ldg(reinterpret_cast<const float4*>(dx_node + i * H) + l16);
            o = make_float4(o.x + d.x, o.y + d.y, o.z + d.z, o.w + d.w);
          }
          reinterpret_cast<float4*>(dx + i * H)[l16] = o;
        }
      }
    }
    // dW: thread owns k in [4 g16, +4), j in [8 l16, +8); nodes in order
#pragma unroll 2
    for (int r = 0; r < kFactRows; ++r) {
      const float4 xv = *reinterpret_cast<const float4*>(xr + r * H + WK * g16);
      const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
      const float4 s0 = *reinterpret_cast<const float4*>(sr + r * NS + WJ * l16);
      const float4 s1 = *reinterpret_cast<const float4*>(sr + r * NS + WJ * l16 + 4);
      const float sb[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
      for (int a = 0; a < WK; ++a)
#pragma unroll
        for (int b = 0; b < WJ; ++b) accw[a][b] = fmaf(xa[a], sb[b], accw[a][b]);
    }
  }
  // partial in W0's layout: rows 0..H-1 = W0_s (j < H), rows H..2H-1 = W0_d
  float* ps = part + (int64_t)blockIdx.x * 2 * H * H;
#pragma unroll
  for (int a = 0; a < WK; ++a)
#pragma unroll
    for (int b = 0; b < WJ; ++b) {
      const int k = WK * g16 + a, j = WJ * l16 + b;
      ps[(j < H ? 0 : H * H) + k * H + (j % H)] = accw[a][b];
    }
}
// S = [S_src | S_dst] for every row, one thread per (row, 16-byte piece):
// the same sums in the same slot order as the in-kernel gather (bitwise), at
// full occupancy (the adjoint kernel's own gather runs at 2 blocks per SM).
template <int H>
__global__ void seg_sum_kernel(const float* __restrict__ dy, const int32_t* __restrict__ beg,
                               const int32_t* __restrict__ end, const int32_t* __restrict__ twin, int64_t rows,
                               float* __restrict__ S) {
  constexpr int Q = 2 * H / 4;  // 16-byte pieces per S row
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= rows * Q) return;
  const int64_t i = tid / Q;
  const int c4 = (int)(tid % Q);
  const bool src_half = c4 < H / 4;
  const int cc = src_half ? c4 : c4 - H / 4;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  const int32_t p1 = __ldg(end + i);
  for (int32_t p = __ldg(beg + i); p < p1; p += 4) {  // 4 slots in flight; +0 padding is bitwise neutral
    int64_t e[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      e[u] = p + u < p1 ? (src_half ? (int64_t)__ldg(twin + p + u) : (int64_t)(p + u)) : (int64_t)-1;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 v =
          e[u] >= 0 ? __ldg(reinterpret_cast<const float4*>(dy + e[u] * H) + cc) : make_float4(0.f, 0.f, 0.f, 0.f);
      s = make_float4(s.x + v.x, s.y + v.y, s.z + v.z, s.w + v.w);
    }
  }
  reinterpret_cast<float4*>(S + i * 2 * H)[c4] = s;
}

template <int H>
constexpr size_t edge_input_adjoint_smem() {
  return (size_t)(2 * H * H + kFactRows * 2 * H + kFactRows * H) * 4;
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
