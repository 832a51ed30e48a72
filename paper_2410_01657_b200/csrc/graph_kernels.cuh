// HBM-bound graph kernels of the consistent NMP layer (sm_100a):
// degree-scaled segmented aggregation, halo pack/unpack, synchronisation,
// exchange-adjoint accumulation, input-node adjoint gather, boundary format
// conversions and the deterministic gradient reduction.
//
// Edges live on the device in receiver-sorted order (slot p = the reference's
// in-CSR position, graph.cpp:122-136), so every per-node sum is a contiguous
// segment read in the reference's summation order. All kernels are 128-bit
// vectorised along the feature axis (thread = (row, 4 features)).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.hpp"

namespace hgnn_b200 {

__device__ __forceinline__ float4 f4_fma(float s, float4 v, float4 acc) {
  return make_float4(fmaf(s, v.x, acc.x), fmaf(s, v.y, acc.y), fmaf(s, v.z, acc.z), fmaf(s, v.w, acc.w));
}
__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// a[i] = sum_{p in [off[i], off[i+1])} inv[p] * e[p]   (scatter_rows_csr,
// kernels.cpp:174-186, applied at model.cpp:238-240). Halo rows: empty -> 0.
// Rows row_list[0..n) (all rows when row_list is null); row i's in-edges are
// slots [beg[i], end[i]) in in-CSR order.
__global__ void aggregate_kernel(const float* __restrict__ e, const float* __restrict__ inv,
                                 const int32_t* __restrict__ beg, const int32_t* __restrict__ end,
                                 const int32_t* __restrict__ row_list, int64_t n, int H, float* __restrict__ a) {
  const int q = H / 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * q) return;
  const int64_t t = tid / q;
  const int64_t i = row_list ? (int64_t)__ldg(row_list + t) : t;
  const int c = (int)(tid % q);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  const int32_t p1 = __ldg(end + i);
  for (int32_t p = __ldg(beg + i); p < p1; ++p)
    s = f4_fma(__ldg(inv + p), __ldg(reinterpret_cast<const float4*>(e + (int64_t)p * H) + c), s);
  reinterpret_cast<float4*>(a + i * H)[c] = s;
}

// dst[t] = src[rows[t]]  (halo_exchange pack, comm.cpp:287-296)
__global__ void gather_rows_kernel(const float* __restrict__ src, const int32_t* __restrict__ rows_idx,
                                   const int64_t* __restrict__ dst_pos, int64_t n, int H, float* __restrict__ dst) {
  const int q = H / 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * q) return;
  const int64_t t = tid / q;
  const int c = (int)(tid % q);
  const int64_t d = dst_pos ? __ldg(dst_pos + t) : t;
  reinterpret_cast<float4*>(dst + d * H)[c] =
      __ldg(reinterpret_cast<const float4*>(src + (int64_t)__ldg(rows_idx + t) * H) + c);
}

// dst[rows[t]] = src[src_pos[t]]  (halo_exchange unpack, comm.cpp:302-314)
__global__ void scatter_rows_kernel(const float* __restrict__ src, const int64_t* __restrict__ src_pos,
                                    const int32_t* __restrict__ rows_idx, int64_t n, int H, float* __restrict__ dst) {
  const int q = H / 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * q) return;
  const int64_t t = tid / q;
  const int c = (int)(tid % q);
  reinterpret_cast<float4*>(dst + (int64_t)__ldg(rows_idx + t) * H)[c] =
      __ldg(reinterpret_cast<const float4*>(src + __ldg(src_pos + t) * H) + c);
}

// a*[local] = sum over slots in ascending owner rank (model.cpp:247-254), in
// place: slot -1 reads this thread's own pre-sync element before it is written.
__global__ void sync_kernel(float* __restrict__ a, const int32_t* __restrict__ g_local,
                            const int32_t* __restrict__ g_off, const int32_t* __restrict__ g_slots, int64_t n_groups,
                            int H) {
  const int q = H / 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n_groups * q) return;
  const int64_t g = tid / q;
  const int c = (int)(tid % q);
  const int64_t li = __ldg(g_local + g);
  float4* out = reinterpret_cast<float4*>(a + li * H) + c;
  const float4 own = *out;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int32_t t = __ldg(g_off + g); t < __ldg(g_off + g + 1); ++t) {
    const int32_t slot = __ldg(g_slots + t);
    s = f4_add(s, slot < 0 ? own : reinterpret_cast<const float4*>(a + (int64_t)slot * H)[c]);
  }
  *out = s;
}

// Sync adjoint (model.cpp:345-349): every halo slot of a group receives the
// local adjoint.
__global__ void sync_adjoint_kernel(float* __restrict__ d_a, const int32_t* __restrict__ g_local,
                                    const int32_t* __restrict__ g_off, const int32_t* __restrict__ g_slots,
                                    int64_t n_groups, int H) {
  const int q = H / 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n_groups * q) return;
  const int64_t g = tid / q;
  const int c = (int)(tid % q);
  const float4 v = reinterpret_cast<const float4*>(d_a + (int64_t)__ldg(g_local + g) * H)[c];
  for (int32_t t = __ldg(g_off + g); t < __ldg(g_off + g + 1); ++t) {
    const int32_t slot = __ldg(g_slots + t);
    if (slot >= 0) reinterpret_cast<float4*>(d_a + (int64_t)slot * H)[c] = v;
  }
}

// Exchange-adjoint accumulation (comm.cpp:344-356): for each local row that
// appears in any send mask, add the returned halo adjoints in ascending
// neighbour order. acc_pos lists buffer positions per row in that order.
__global__ void adjoint_accumulate_kernel(float* __restrict__ d_a, const float* __restrict__ recv,
                                          const int32_t* __restrict__ acc_rows, const int32_t* __restrict__ acc_off,
                                          const int64_t* __restrict__ acc_pos, int64_t n_rows, int H) {
  const int q = H / 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n_rows * q) return;
  const int64_t t = tid / q;
  const int c = (int)(tid % q);
  float4* dst = reinterpret_cast<float4*>(d_a + (int64_t)__ldg(acc_rows + t) * H) + c;
  float4 v = *dst;
  for (int32_t u = __ldg(acc_off + t); u < __ldg(acc_off + t + 1); ++u)
    v = f4_add(v, __ldg(reinterpret_cast<const float4*>(recv + __ldg(acc_pos + u) * H) + c));
  *dst = v;
}

// Input-node adjoint (model.cpp:378-386): out-CSR sum of d_x_src (read through
// the twin index: the out-edges of i are the twins of its in-edges, in the
// same ascending order), plus the in-CSR sum of d_x_dst, plus the node-update
// adjoint on local rows.
__global__ void dx_gather_kernel(const float* __restrict__ d_src, const float* __restrict__ d_dst,
                                 const float* __restrict__ dx_node, const int32_t* __restrict__ beg,
                                 const int32_t* __restrict__ end, const int32_t* __restrict__ twin, int64_t rows, int64_t n_local, int H,
                                 float* __restrict__ dx) {
  const int q = H / 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= rows * q) return;
  const int64_t i = tid / q;
  const int c = (int)(tid % q);
  float4 s1 = make_float4(0.f, 0.f, 0.f, 0.f), s2 = s1;
  const int32_t p1 = __ldg(end + i);
  for (int32_t p = __ldg(beg + i); p < p1; ++p) {
    s1 = f4_add(s1, __ldg(reinterpret_cast<const float4*>(d_src + (int64_t)__ldg(twin + p) * H) + c));
    s2 = f4_add(s2, __ldg(reinterpret_cast<const float4*>(d_dst + (int64_t)p * H) + c));
  }
  float4 o = f4_add(s1, s2);
  if (i < n_local) o = f4_add(o, __ldg(reinterpret_cast<const float4*>(dx_node + i * H) + c));
  reinterpret_cast<float4*>(dx + i * H)[c] = o;
}

// grads[i] = sum_b partial[b][i] in block order (fp64): deterministic.
__global__ void grad_reduce_kernel(const float* __restrict__ partial, int64_t n_blocks, int64_t n,
                                   double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t b = 0; b < n_blocks; ++b) s += (double)__ldg(partial + b * n + i);
  out[i] = s;
}

// Boundary conversions. Edge tensors are permuted between the reference's
// edge-id order (host) and receiver-sorted slots (device): slot_of[e] = p.
__global__ void rows_f64_to_f32_kernel(const double* __restrict__ src, int64_t n, float* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (float)src[i];
}
__global__ void rows_f32_to_f64_kernel(const float* __restrict__ src, int64_t n, double* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (double)src[i];
}
// edge ids [e0, e0+n): dev[slot_of[e]] = (float) stage[e - e0]
__global__ void edges_in_kernel(const double* __restrict__ stage, const int32_t* __restrict__ slot_of, int64_t e0,
                                int64_t n, int H, float* __restrict__ dev) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * H) return;
  const int64_t e = tid / H;
  const int c = (int)(tid % H);
  dev[(int64_t)__ldg(slot_of + e0 + e) * H + c] = (float)stage[tid];
}
__global__ void edges_out_kernel(const float* __restrict__ dev, const int32_t* __restrict__ slot_of, int64_t e0,
                                 int64_t n, int H, double* __restrict__ stage) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * H) return;
  const int64_t e = tid / H;
  const int c = (int)(tid % H);
  stage[tid] = (double)__ldg(dev + (int64_t)__ldg(slot_of + e0 + e) * H + c);
}

// Seeded values depending only on (key, column, seed): identical on every rank
// for coincident nodes / duplicated edges.
__device__ __forceinline__ float hash_uniform(uint64_t key, uint64_t c, uint64_t seed) {
  uint64_t z = key * 0x9E3779B97F4A7C15ull ^ (c + 0x632BE59BD9B4E019ull) * 0xBF58476D1CE4E5B9ull ^ seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (float)((double)(z >> 11) * 0x1.0p-53 * 2.0 - 1.0);
}
__global__ void synth_rows_kernel(const int64_t* __restrict__ gid, int64_t rows, int64_t live_rows, int H,
                                  uint64_t seed, float scale, float* __restrict__ out) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= rows * H) return;
  const int64_t i = tid / H;
  const int c = (int)(tid % H);
  out[tid] = i < live_rows ? scale * hash_uniform((uint64_t)__ldg(gid + i), (uint64_t)c, seed) : 0.f;
}
__global__ void synth_edges_kernel(const int64_t* __restrict__ gid, const int32_t* __restrict__ src,
                                   const int32_t* __restrict__ dst, int64_t ne, int H, uint64_t seed,
                                   float* __restrict__ out) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= ne * H) return;
  const int64_t p = tid / H;
  const int c = (int)(tid % H);
  const uint64_t key = (uint64_t)__ldg(gid + __ldg(src + p)) * 0x100000001B3ull ^ (uint64_t)__ldg(gid + __ldg(dst + p));
  out[tid] = hash_uniform(key, (uint64_t)c, seed);
}

}  // namespace hgnn_b200
