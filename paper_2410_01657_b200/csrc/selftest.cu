// Hardware self-tests of the tcgen05 building blocks used by the MLP kernels:
// one 128-row MMA (K = 32) in each operand configuration, on caller data.
//   mode 0: A in TMEM (TS), B K-major in SMEM          (forward / dX path)
//   mode 1: A, B both MN-major in SMEM (SS), N = 128   (dW path)
//   mode 2: A, B both K-major in SMEM (SS), N = 128
//   modes 6-8: MN-major SWIZZLE_128B_BASE32B operands (dW path)
//   modes 9/10: M = N = 64, both MN-major swizzled, D addressed at TMEM lane 0 / 16
//               (D read back for all 128 lanes: where M = 64 rows land)
// A: 128 x 32 (row-major m, k), B: 32 x N (row-major k, n), D = A B (fp32 out).
#include <cstring>
#include <vector>

#include "../../include/hgnn_b200_debug.h"
#include "common.hpp"
#include "tc_ptx.cuh"

using namespace hgnn_b200;

namespace {

constexpr int TM = 128, TK = 32, TN = 128;

// K-major core-matrix offset (bytes) of element (mn, k): 8 MN rows x 16 B of K
__device__ uint32_t kmaj(int mn, int k, int n_mn) {
  const uint32_t lbo = (uint32_t)(n_mn / 8) * 128;  // K-chunk stride
  return (uint32_t)(k / 4) * lbo + (uint32_t)(mn / 8) * 128 + (uint32_t)(mn % 8) * 16 + (uint32_t)(k % 4) * 4;
}
// MN-major SWIZZLE_128B_BASE32B: atoms of 4 K-rows x 128 B of MN (32 tf32);
// 32-byte granule g of row r stored at granule g ^ r. Atoms: MN stride lbo,
// K stride sbo.
__device__ uint32_t mn_sw(int mn, int k, uint32_t lbo, uint32_t sbo) {
  const int a = mn / 32, w = mn % 32, g = w / 8, e = w % 8, r = k % 4;
  return (uint32_t)(k / 4) * sbo + (uint32_t)a * lbo + (uint32_t)r * 128 + (uint32_t)((g ^ r) * 32) + (uint32_t)e * 4;
}
// MN-major core-matrix offset (bytes): 8 K rows x 16 B of MN
__device__ uint32_t mnmaj(int mn, int k, int n_k) {
  const uint32_t sbo = (uint32_t)(n_k / 8) * 128;  // MN-chunk stride
  return (uint32_t)(mn / 4) * sbo + (uint32_t)(k / 8) * 128 + (uint32_t)(k % 8) * 16 + (uint32_t)(mn % 4) * 4;
}

__global__ void __launch_bounds__(128) selftest_kernel(int mode, const float* A, const float* B, float* D) {
  __shared__ __align__(1024) uint8_t sa[TM * TK * 4];
  __shared__ __align__(1024) uint8_t sb[TK * TN * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  const int warp = t / 32;
  // stage operands
  const bool sw = mode >= 6;
  const bool m64 = mode >= 9;  // M = N = 64, D at lane 0 (mode 9) or lane 64 (mode 10)
  const bool a_mn = mode == 1 || mode == 3 || mode == 5 || mode == 6 || mode == 7 || m64;
  const bool b_mn = mode == 1 || mode == 4 || mode == 5 || mode == 6 || mode == 8 || m64;
  // swizzled MN-major: MN atoms (128 B) at lbo = 512, K atoms (4 rows) at sbo = (MN/32) * 512
  const uint32_t sw_lbo = 512, sw_sbo_a = ((m64 ? 64 : TM) / 32) * 512, sw_sbo_b = ((m64 ? 64 : TN) / 32) * 512;
  for (int i = t; i < TM * TK; i += 128) {
    const int m = i / TK, k = i % TK;
    if (m64 && m >= 64) continue;
    const uint32_t off = (sw && a_mn) ? mn_sw(m, k, sw_lbo, sw_sbo_a) : (a_mn ? mnmaj(m, k, TK) : kmaj(m, k, TM));
    *reinterpret_cast<float*>(sa + off) = A[i];
  }
  for (int i = t; i < TK * TN; i += 128) {
    const int k = i / TN, n = i % TN;
    if (m64 && n >= 64) continue;
    const uint32_t off = (sw && b_mn) ? mn_sw(n, k, sw_lbo, sw_sbo_b) : (b_mn ? mnmaj(n, k, TK) : kmaj(n, k, TN));
    *reinterpret_cast<float*>(sb + off) = B[i];
  }
  if (t == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbarrier_init();
  }
  if (warp == 0) ptx::tmem_alloc<256>(&tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
  if (m64) {  // zero D region (all lanes, columns [0, 128)) so untouched lanes read back as 0
    float z[32];
    for (int j = 0; j < 32; ++j) z[j] = 0.f;
    for (int c = 0; c < 128; c += 32) ptx::tmem_st32(tmem + lane_off + c, z);
    ptx::tmem_wait_st();
  }
  if (mode == 0) {  // A into TMEM columns [128, 160): thread = row
    float v[32];
    for (int k = 0; k < 32; ++k) v[k] = A[t * TK + k];
    ptx::tmem_st32(tmem + 128 + lane_off, v);
    ptx::tmem_wait_st();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (t == 0) {
    const uint32_t a_s = ptx::smem_u32(sa), b_s = ptx::smem_u32(sb);
    for (int ks = 0; ks < TK / 8; ++ks) {
      if (mode == 0) {
        const uint32_t lbo = (TN / 8) * 128;  // N = 128 K-major
        const uint64_t bd = ptx::smem_desc(b_s + ks * 2 * lbo, lbo, 128);
        ptx::mma_tf32_ts(tmem, tmem + 128 + 8 * ks, bd, ptx::idesc_tf32(128, TN), ks > 0);
      } else {
        uint64_t ad, bd;
        uint32_t idesc = m64 ? ptx::idesc_tf32(64, 64) : ptx::idesc_tf32(128, TN);
        const uint32_t lbo_a = (TM / 8) * 128, lbo_b = (TN / 8) * 128;
        const uint32_t mn_lbo = mode == 5 ? (TK / 8) * 128 : 128, mn_sbo = mode == 5 ? 128 : (TK / 8) * 128;
        ad = a_mn ? ptx::smem_desc(a_s + ks * 128, mn_lbo, mn_sbo) : ptx::smem_desc(a_s + ks * 2 * lbo_a, lbo_a, 128);
        bd = b_mn ? ptx::smem_desc(b_s + ks * 128, mn_lbo, mn_sbo) : ptx::smem_desc(b_s + ks * 2 * lbo_b, lbo_b, 128);
        if (sw) {
          const uint64_t swz = (uint64_t)1 << 61;  // layout type 1 = SWIZZLE_128B_BASE32B
          if (a_mn) ad = ptx::smem_desc(a_s + ks * 2 * sw_sbo_a, sw_lbo, sw_sbo_a) | swz;
          if (b_mn) bd = ptx::smem_desc(b_s + ks * 2 * sw_sbo_b, sw_lbo, sw_sbo_b) | swz;
        }
        if (a_mn) idesc |= (1u << 15);
        if (b_mn) idesc |= (1u << 16);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (mode == 10 ? (16u << 16) : 0u)),
            "l"(ad), "l"(bd), "r"(idesc), "r"(ks > 0 ? 1u : 0u)
            : "memory");
      }
    }
    ptx::mma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  for (int c = 0; c < TN; c += 32) {
    float v[32];
    ptx::tmem_ld32(tmem + lane_off + c, v);
    ptx::tmem_wait_ld();
    for (int j = 0; j < 32; ++j) D[t * TN + c + j] = v[j];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(tmem);
  }
}

}  // namespace

extern "C" int hgnn_selftest_mma(int mode, const float* A, const float* B, float* D) {
  return guarded([&] {
    float *dA, *dB, *dD;
    if (cudaMalloc(&dA, TM * TK * 4) || cudaMalloc(&dB, TK * TN * 4) || cudaMalloc(&dD, TM * TN * 4))
      fail(HGNN_ERR_CUDA, "selftest alloc");
    cudaMemcpy(dA, A, TM * TK * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, TK * TN * 4, cudaMemcpyHostToDevice);
    selftest_kernel<<<1, 128>>>(mode, dA, dB, dD);
    const cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D, dD, TM * TN * 4, cudaMemcpyDeviceToHost);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    if (e != cudaSuccess) fail(HGNN_ERR_CUDA, cudaGetErrorString(e));
  });
}

// ---- MMA issue-rate microbenchmark (debug aid) ------------------------------
// One CTA per SM issues `iters` x 24 tcgen05.mma (kind::tf32, M = 128, K = 8)
// back to back from an elected lane of warp 0 with warp-uniform operands,
// N = n, A from TMEM (ts) or shared memory, B from shared memory, into nd
// round-robin accumulators. Operands are uninitialised (timing only).
// cycles[blockIdx] = clock64 span from first issue to commit arrival.
namespace {
template <int N, bool TS, int ND>
__global__ void __launch_bounds__(128) mma_rate_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbarrier_init();
  }
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, tslot, 0);
  if (warp == 0) {
    constexpr uint32_t idesc = ptx::idesc_tf32(128, N);
    const uint32_t base = ptx::smem_u32(sm);
    const uint64_t bd = ptx::smem_desc(base, (uint32_t)(N / 8) * 128, 128);
    const uint64_t ad = ptx::smem_desc(base + 65536, 16 * 128, 128);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 24; ++j) {
        const uint32_t dcol = tmem + 256 + (uint32_t)((j % ND) * (256 / ND));
        if (TS) ptx::mma_tf32_ts_w(dcol, tmem + 8 * (j % 16), bd + (uint64_t)(j % 8) * 16, idesc, 1u);
        else ptx::mma_tf32_ss_w(dcol, ad + (uint64_t)(j % 8) * 16, bd + (uint64_t)(j % 8) * 16, idesc, 1u);
      }
    }
    ptx::mma_commit_w(&bar);
    ptx::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <int N, bool TS, int ND>
void run_rate(int iters, int blocks, unsigned long long* d) {
  cudaFuncSetAttribute(mma_rate_kernel<N, TS, ND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  mma_rate_kernel<N, TS, ND><<<blocks, 128, 160 * 1024>>>(iters, d);
}
}  // namespace

extern "C" int hgnn_bench_mma(int iters, int n, int ts, int nd, int blocks, uint64_t* cycles_out) {
  return guarded([&] {
    unsigned long long* d;
    if (cudaMalloc(&d, sizeof(unsigned long long) * (size_t)blocks)) fail(HGNN_ERR_CUDA, "bench alloc");
    const int key = n * 100 + (ts ? 10 : 0) + nd;
    switch (key) {
      case 6411: run_rate<64, true, 1>(iters, blocks, d); break;
      case 6412: run_rate<64, true, 2>(iters, blocks, d); break;
      case 12811: run_rate<128, true, 1>(iters, blocks, d); break;
      case 12812: run_rate<128, true, 2>(iters, blocks, d); break;
      case 25611: run_rate<256, true, 1>(iters, blocks, d); break;
      case 6401: run_rate<64, false, 1>(iters, blocks, d); break;
      case 12801: run_rate<128, false, 1>(iters, blocks, d); break;
      case 25601: run_rate<256, false, 1>(iters, blocks, d); break;
      default: fail(HGNN_ERR_CONFIG, "hgnn_bench_mma: unsupported (n, ts, nd)");
    }
    const cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(cycles_out, d, sizeof(unsigned long long) * (size_t)blocks, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) fail(HGNN_ERR_CUDA, cudaGetErrorString(e));
  });
}

// ---- SFU / FMA throughput microbenchmark (debug aid) -------------------------
// Each of `threads` threads runs 8 independent chains of `iters` operations:
// kind 0: ex2.approx.ftz.f32, kind 1: fma.rn.f32, kind 2: rsqrt.approx.
// cycles[b] = clock64 span of thread 0 of block b; sink keeps the results live.
namespace {
__global__ void alu_rate_kernel(int kind, int iters, unsigned long long* cycles, float* sink) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  const long long t0 = clock64();
  if (kind == 0) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
    }
  } else if (kind == 1) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A83126F;" : "+f"(v[i]));
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345.f) sink[threadIdx.x] = s;
}
}  // namespace

extern "C" int hgnn_bench_alu(int kind, int iters, int threads, int blocks, uint64_t* cycles_out) {
  return guarded([&] {
    unsigned long long* d;
    float* sink;
    if (cudaMalloc(&d, sizeof(unsigned long long) * (size_t)blocks) || cudaMalloc(&sink, 4096 * 4))
      fail(HGNN_ERR_CUDA, "bench alloc");
    alu_rate_kernel<<<blocks, threads>>>(kind, iters, d, sink);
    const cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(cycles_out, d, sizeof(unsigned long long) * (size_t)blocks, cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(sink);
    if (e != cudaSuccess) fail(HGNN_ERR_CUDA, cudaGetErrorString(e));
  });
}
