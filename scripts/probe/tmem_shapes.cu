// Probe (debug only): thread <-> (TMEM lane, column) mapping of the
// tcgen05.ld .16x256b / .16x128b / .16x64b shapes on this B200, by storing
// value (lane * 1000 + column) with the .32x32b shape (thread = lane) and
// reading back with the other shapes from warp 0 (lanes 0..31).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void k(int* out) {
  __shared__ uint32_t taddr;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = taddr + ((uint32_t)(32 * warp) << 16);
  // each of the 4 warps writes its 32 lanes, 8 columns: value lane*1000 + col
  uint32_t v[8];
  for (int c = 0; c < 8; ++c) v[c] = (32 * warp + lane) * 1000 + c;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(t));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 4; ++i) out[lane * 4 + i] = r[i];
    uint32_t q[2];
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(q[0]), "=r"(q[1]) : "r"(t));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 2; ++i) out[128 + lane * 2 + i] = q[i];
    uint32_t s;
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(s) : "r"(t));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[192 + lane] = s;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(taddr));
}
int main() {
  int* d; cudaMalloc(&d, 256 * 4); cudaMemset(d, 0xff, 256 * 4);
  k<<<1, 128>>>(d);
  int h[256]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  printf("16x256b.x1 (thread: 4 values = lane*1000+col)\n");
  for (int t = 0; t < 32; ++t) printf("t%02d: %d %d %d %d\n", t, h[t*4], h[t*4+1], h[t*4+2], h[t*4+3]);
  printf("16x128b.x1\n");
  for (int t = 0; t < 32; ++t) printf("t%02d: %d %d\n", t, h[128+t*2], h[128+t*2+1]);
  printf("16x64b.x1\n");
  for (int t = 0; t < 32; ++t) printf("t%02d: %d\n", t, h[192+t]);
}
