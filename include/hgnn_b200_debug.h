/* include/hgnn_b200_debug.h — debugging aids, NOT part of the product ABI.
 *
 * Built into lib/libhgnn_b200_debug.so (csrc/selftest.cu), which links the
 * product library; used only by scripts/dbg_*.py to check tcgen05 operand
 * layouts and to measure MMA / SFU issue rates on the box.
 */
#ifndef HGNN_B200_DEBUG_H
#define HGNN_B200_DEBUG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- hardware self-test ----------------------------------------------------- */
/* One 128 x 128 x 32 tcgen05 kind::tf32 MMA on caller data (A 128x32, B 32x128,
 * row-major fp32; D 128x128). mode 0: A in TMEM + B K-major (forward / dX path),
 * 1: A and B MN-major in shared memory (dW path), 2: both K-major in shared memory. */
int hgnn_selftest_mma(int mode, const float* A, const float* B, float* D);
/* MMA issue-rate microbenchmark (debug aid): `blocks` CTAs each issue iters x 24
 * kind::tf32 M=128 K=8 MMAs with N = n (A from TMEM if ts, else SMEM) into nd
 * round-robin accumulators (nd * n <= 256 columns); cycles_out[b] = clock64
 * cycles of CTA b from first issue to completion. */
int hgnn_bench_mma(int iters, int n, int ts, int nd, int blocks, uint64_t* cycles_out);
/* SFU / FMA throughput microbenchmark (debug aid): kind 0 ex2.approx, 1 fma,
 * 2 rsqrt.approx; threads x 8 independent chains x iters operations per block. */
int hgnn_bench_alu(int kind, int iters, int threads, int blocks, uint64_t* cycles_out);

#ifdef __cplusplus
}
#endif
#endif /* HGNN_B200_DEBUG_H */
