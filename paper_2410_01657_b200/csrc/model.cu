// Model level on the device: encoders + MP stack +
// decoder, consistent loss, rank-averaged gradients, Adam (model.cpp:289-307,
// 390-424, 455-579; nn.cpp:331-360) and their C-ABI (include/hgnn_b200.h).
#include <cmath>

#include "encoder_tc.cuh"
#include "engine_ctx.hpp"
#include "mlp_generic.cuh"
#include "mlp_tc_bwd.cuh"
#include "model_kernels.cuh"

using namespace hgnn_b200;
using namespace hgnn_b200::engine;

namespace {

bool gen_supported(int64_t fx, int64_t fe, int64_t fy) { return fx == 3 && fe == 7 && fy == 3; }

template <int IN, int OUT, bool SKIP, bool LN, int H>
void gen_forward(hgnn_ctx* c, int64_t n_rows, const float* in, float* out, int64_t par_off, int64_t n_par) {
  if (n_rows == 0) return;
  GenArgs a{};
  a.n_rows = n_rows;
  a.in = in;
  a.out = out;
  a.params = c->gen_par.p + par_off;
  a.k = (int)c->K;
  a.n_par = n_par;
  auto k = gen_mlp_forward_kernel<IN, OUT, SKIP, LN, H>;
  const size_t smem = (size_t)((n_par + 3) / 4) * 16 + (size_t)H * kGenThreads * 4;  // params + gemv columns
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t tiles = (n_rows + kGenThreads - 1) / kGenThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 2 * (int64_t)c->num_sms));
  k<<<grid, kGenThreads, smem, c->stream>>>(a);
  check_launch(c);
}

// Backward of one encoder / decoder MLP; parameter gradients (rank-local)
// land in mgrads[par_off, par_off + n_par).
template <int IN, int OUT, bool SKIP, bool LN, bool DIN, int H>
void gen_backward(hgnn_ctx* c, int64_t n_rows, const float* in, const float* d_out, float* d_in, int64_t par_off,
                  int64_t n_par) {
  if (n_rows == 0) {
    CUDA_OK(cudaMemsetAsync(c->mgrads.p + par_off, 0, sizeof(double) * (size_t)n_par, c->stream));
    return;
  }
  const int64_t tiles = (n_rows + kGenThreads - 1) / kGenThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 2 * (int64_t)c->num_sms));  // 2 CTAs / SM
  const int64_t slots = gen_scratch_slots((int)c->K, OUT, H);
  c->gen_part.alloc(std::max<int64_t>(c->gen_part.n, (int64_t)grid * n_par));
  c->gen_scratch.alloc(std::max<int64_t>(c->gen_scratch.n, (int64_t)grid * slots * kGenThreads));
  CUDA_OK(cudaMemsetAsync(c->gen_part.p, 0, sizeof(float) * (size_t)(grid * n_par), c->stream));
  GenArgs a{};
  a.n_rows = n_rows;
  a.in = in;
  a.d_out = d_out;
  a.d_in = d_in;
  a.params = c->gen_par.p + par_off;
  a.grad_partial = c->gen_part.p;
  a.scratch = c->gen_scratch.p;
  a.k = (int)c->K;
  a.n_par = n_par;
  auto k = gen_mlp_backward_kernel<IN, OUT, SKIP, LN, DIN, H>;
  const size_t smem = gen_backward_smem(IN, OUT, H);
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<grid, kGenThreads, smem, c->stream>>>(a);
  check_launch(c);
  reduce_partials_kernel<<<blocks_for(n_par), kEwThreads, 0, c->stream>>>(c->gen_part.p, grid, n_par,
                                                                          c->mgrads.p + par_off, n_par);
  check_launch(c);
}

// ---- tcgen05 encoders (encoder_tc.cuh) ------------------------------------
bool enc_tc(const hgnn_ctx* c) { return c->enc_impl == 1 && c->H == 64 && c->fwd_impl == 1 && c->bwd_impl == 1; }

// which: 0 node encoder, 1 edge encoder. enc_ln = 0: pre-LayerNorm y (backward recompute).
void enc_forward_tc(hgnn_ctx* c, int which, int64_t n, int F, const float* feat, float* out, int64_t par_off,
                    int enc_ln) {
  if (n == 0) return;
  using Cfg = TcCfg<64>;
  TcFwdArgs a{};
  a.n_rows = n;
  a.e_in = feat;
  a.out = out;
  a.chunks = c->enc_ch.p + c->enc_off[which];
  a.params = c->gen_par.p + par_off;
  a.k = (int)c->K;
  a.in_dim = F;
  a.enc_ln = enc_ln;
  auto k = mlp_tc_forward_kernel<64, kEncoder, false>;
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM_ENC));
  const int64_t pairs = ((n + 127) / 128 + 1) / 2;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(pairs, c->num_sms));
  k<<<grid, Cfg::THREADS, Cfg::SMEM_ENC, c->stream>>>(a);
  check_launch(c);
}

// A device buffer of >= n floats that is dead while the encoder backward runs:
// d_x_src (or x_M under the memory-lean plan), else a dedicated one.
float* enc_scratch(hgnn_ctx* c, int64_t n) {
  if (c->dsrc.n >= n) return c->dsrc.p;
  if (c->enc_tmp.n < n) c->enc_tmp.alloc(n);
  return c->enc_tmp.p;
}

// Parameter gradients of one encoder into mgrads[par_off, par_off + n_par)
// (rank-local); d_out = adjoint of the encoder output (N x 64).
void enc_backward_tc(hgnn_ctx* c, int which, int64_t n, int F, const float* feat, const float* d_out,
                     int64_t par_off, int64_t n_par) {
  if (n == 0) {
    CUDA_OK(cudaMemsetAsync(c->mgrads.p + par_off, 0, sizeof(double) * (size_t)n_par, c->stream));
    return;
  }
  constexpr int H = 64;
  const int K = (int)c->K;
  const GenLayout L{F, H, K, H};
  float* y = enc_scratch(c, n * H);
  enc_forward_tc(c, which, n, F, feat, y, par_off, 0);  // 1. pre-LayerNorm y
  const int n_ln = (F + 2) * H;                          // 2. LN adjoint in place, W_skip / gamma / beta partials
  if (c->enc_part.n < (int64_t)kEncLnBlocks * n_ln) c->enc_part.alloc((int64_t)kEncLnBlocks * n_ln);
  enc_out_backward_kernel<<<kEncLnBlocks, kEncLnThreads, 0, c->stream>>>(y, d_out, feat, F,
                                                                        c->gen_par.p + par_off + L.ln_g(), n,
                                                                        c->enc_part.p);
  check_launch(c);
  // 3. the MLP backward on the tensor cores, d_out = dy
  const int64_t pairs = ((n + 127) / 128 + 1) / 2;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(pairs, c->num_sms));
  const int64_t stride = (n_par + 3) & ~int64_t(3);  // 16-byte aligned partial rows (vector reductions)
  if (c->grad_part.n < 2 * (int64_t)grid * stride) c->grad_part.alloc(2 * (int64_t)grid * stride);
  CUDA_OK(cudaMemsetAsync(c->grad_part.p, 0, sizeof(float) * (size_t)(2 * grid * stride), c->stream));
  TcBwdArgs a{};
  a.n_rows = n;
  a.e_in = feat;
  a.d_out = y;
  a.chunks = c->enc_ch.p + c->enc_off[3 + which];
  a.params = c->gen_par.p + par_off;
  a.grad_partial = c->grad_part.p;
  a.scratch = c->tc_scratch.p;
  a.k = K;
  a.in_dim = F;
  a.n_par = stride;
  auto k = mlp_tc_backward_kernel<kEncoder, false>;
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TcBwdCfg::SMEM));
  k<<<grid, TcBwdCfg::THREADS, TcBwdCfg::SMEM, c->stream>>>(a);
  check_launch(c);
  // W, b partials (the skip / LayerNorm entries of these partials stay zero) ...
  reduce_partials_kernel<<<blocks_for(n_par), kEwThreads, 0, c->stream>>>(c->grad_part.p, 2 * grid, n_par,
                                                                          c->mgrads.p + par_off, stride);
  check_launch(c);
  // ... then W_skip, gamma, beta (contiguous in the for_each layout)
  reduce_partials_kernel<<<blocks_for(n_ln), kEwThreads, 0, c->stream>>>(c->enc_part.p, kEncLnBlocks, n_ln,
                                                                         c->mgrads.p + par_off + L.skip(), n_ln);
  check_launch(c);
}

// Chunk sequences of the node encoder, edge encoder and decoder (fwd at
// enc_off[0..2], bwd at enc_off[3..5]) as a refresh map over the full fp64
// parameter vector.
void build_enc_map(hgnn_ctx* c) {
  const int H = (int)c->H, K = (int)c->K;
  if (H != 64) {
    c->enc_map.release();
    c->enc_ch.release();
    return;
  }
  const int Fs[3] = {(int)c->fx, (int)c->fe, H};   // input widths
  const int Os[3] = {H, H, (int)c->fy};             // output widths
  const int64_t offs[3] = {c->off_ne, c->off_ee, c->off_dec};
  int64_t total = 0;
  for (int d = 0; d < 2; ++d)
    for (int w = 0; w < 3; ++w) {
      c->enc_off[3 * d + w] = total;
      total += d == 0 ? chunk_floats_fwd(Fs[w], H, K, 1) : chunk_floats_bwd(Fs[w], H, K, 1);
    }
  std::vector<uint32_t> map((size_t)total);
  for (int d = 0; d < 2; ++d)
    for (int w = 0; w < 3; ++w) {
      auto emit = [&](int64_t pos, int64_t src, bool lo) {
        map[(size_t)pos] = src < 0 ? 0x7fffffffu : ((uint32_t)(offs[w] + src) | (lo ? 0x80000000u : 0u));
      };
      if (d == 0) chunk_layout_fwd(Fs[w], H, K, c->enc_off[3 * d + w], emit, 0, 1, Os[w]);
      else chunk_layout_bwd(Fs[w], H, K, c->enc_off[3 * d + w], emit, 0, 1, Os[w]);
    }
  c->enc_map.upload(map.data(), total, c->stream);
  c->enc_ch.alloc(total);
}

void refresh_enc_chunks(hgnn_ctx* c) {
  if (c->enc_map.n == 0) return;
  chunk_refresh_kernel<<<blocks_for(c->enc_map.n), kEwThreads, 0, c->stream>>>(c->mparams.p, c->enc_map.p,
                                                                              c->enc_map.n, c->enc_ch.p);
  check_launch(c);
}

// Encoders / decoder of width H (model.cpp:70-101): node encoder F_x = 3,
// edge encoder F_e = 7, decoder F_y = 3.
template <int H>
void encode(hgnn_ctx* c) {
  if (H == 64 && enc_tc(c)) {
    enc_forward_tc(c, 0, c->rows, (int)c->fx, c->node_feat.p, c->xs[0]->p, c->off_ne, 1);
    enc_forward_tc(c, 1, c->ne, (int)c->fe, c->edge_feat.p, c->es[0]->p, c->off_ee, 1);
    return;
  }
  gen_forward<3, H, true, true, H>(c, c->rows, c->node_feat.p, c->xs[0]->p, c->off_ne, c->n_ne);
  gen_forward<7, H, true, true, H>(c, c->ne, c->edge_feat.p, c->es[0]->p, c->off_ee, c->n_ee);
}
// decoder (kDecoder): y = MLP(x_M) + x_M W_skip on the local rows
void dec_forward_tc(hgnn_ctx* c) {
  if (c->nl == 0) return;
  using Cfg = TcCfg<64>;
  TcFwdArgs a{};
  a.n_rows = c->nl;
  a.x = x_buf(c, c->M);
  a.out = c->y.p;
  a.chunks = c->enc_ch.p + c->enc_off[2];
  a.params = c->gen_par.p + c->off_dec;
  a.k = (int)c->K;
  a.in_dim = (int)c->H;
  a.out_dim = (int)c->fy;
  auto k = mlp_tc_forward_kernel<64, kDecoder, false>;
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM_ENC));
  const int64_t pairs = ((c->nl + 127) / 128 + 1) / 2;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(pairs, c->num_sms));
  k<<<grid, Cfg::THREADS, Cfg::SMEM_ENC, c->stream>>>(a);
  check_launch(c);
}

// decoder backward: dx (zeroed by the caller) = the input adjoint on the local
// rows, gradients into mgrads[off_dec, off_dec + n_dec)
void dec_backward_tc(hgnn_ctx* c) {
  const int64_t n = c->nl, n_par = c->n_dec;
  if (n == 0) {
    CUDA_OK(cudaMemsetAsync(c->mgrads.p + c->off_dec, 0, sizeof(double) * (size_t)n_par, c->stream));
    return;
  }
  constexpr int H = 64;
  const int K = (int)c->K, F = (int)c->fy;
  const GenLayout L{H, F, K, H};
  const int64_t pairs = ((n + 127) / 128 + 1) / 2;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(pairs, c->num_sms));
  const int64_t stride = (n_par + 3) & ~int64_t(3);  // 16-byte aligned partial rows (vector reductions)
  if (c->grad_part.n < 2 * (int64_t)grid * stride) c->grad_part.alloc(2 * (int64_t)grid * stride);
  CUDA_OK(cudaMemsetAsync(c->grad_part.p, 0, sizeof(float) * (size_t)(2 * grid * stride), c->stream));
  const float* x = x_buf(c, c->M);
  TcBwdArgs a{};
  a.n_rows = n;
  a.x = x;
  a.d_out = c->dy.p;
  a.d_x_out = c->dx.p;
  a.chunks = c->enc_ch.p + c->enc_off[5];
  a.params = c->gen_par.p + c->off_dec;
  a.grad_partial = c->grad_part.p;
  a.scratch = c->tc_scratch.p;
  a.k = K;
  a.in_dim = H;
  a.out_dim = F;
  a.n_par = stride;
  auto k = mlp_tc_backward_kernel<kDecoder, false>;
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TcBwdCfg::SMEM));
  k<<<grid, TcBwdCfg::THREADS, TcBwdCfg::SMEM, c->stream>>>(a);
  check_launch(c);
  reduce_partials_kernel<<<blocks_for(n_par), kEwThreads, 0, c->stream>>>(c->grad_part.p, 2 * grid, n_par,
                                                                          c->mgrads.p + c->off_dec, stride);
  check_launch(c);
  const int n_sk = H * F;
  if (c->enc_part.n < (int64_t)kEncLnBlocks * n_sk) c->enc_part.alloc((int64_t)kEncLnBlocks * n_sk);
  dec_skip_backward_kernel<<<kEncLnBlocks, kEncLnThreads, 0, c->stream>>>(
      x, c->dy.p, c->gen_par.p + c->off_dec + L.skip(), F, n, c->dx.p, c->enc_part.p);
  check_launch(c);
  reduce_partials_kernel<<<blocks_for(n_sk), kEwThreads, 0, c->stream>>>(c->enc_part.p, kEncLnBlocks, n_sk,
                                                                         c->mgrads.p + c->off_dec + L.skip(), n_sk);
  check_launch(c);
}

template <int H>
void decode(hgnn_ctx* c) {
  if (H == 64 && enc_tc(c)) {
    dec_forward_tc(c);
    return;
  }
  gen_forward<H, 3, true, false, H>(c, c->nl, x_buf(c, c->M), c->y.p, c->off_dec, c->n_dec);
}
template <int H>
void decode_backward(hgnn_ctx* c) {
  if (H == 64 && enc_tc(c)) {
    dec_backward_tc(c);
    return;
  }
  gen_backward<H, 3, true, false, true, H>(c, c->nl, x_buf(c, c->M), c->dy.p, c->dx.p, c->off_dec, c->n_dec);
}
template <int H>
void encode_backward(hgnn_ctx* c) {
  if (H == 64 && enc_tc(c)) {
    enc_backward_tc(c, 0, c->rows, (int)c->fx, c->node_feat.p, c->dx.p, c->off_ne, c->n_ne);
    enc_backward_tc(c, 1, c->ne, (int)c->fe, c->edge_feat.p, de_out_buf(c, 0), c->off_ee, c->n_ee);
    return;
  }
  gen_backward<3, H, true, true, false, H>(c, c->rows, c->node_feat.p, c->dx.p, nullptr, c->off_ne, c->n_ne);
  gen_backward<7, H, true, true, false, H>(c, c->ne, c->edge_feat.p, de_out_buf(c, 0), nullptr, c->off_ee, c->n_ee);
}

void require_model(hgnn_ctx* c) {
  require_ready(c);
  if (!c->model_configured) fail(HGNN_ERR_UNINITIALIZED, "hgnn_model_configure has not been called");
  if (!c->model_params_ready) fail(HGNN_ERR_UNINITIALIZED, "hgnn_model_params_upload has not been called");
  if (!c->model_data_ready) fail(HGNN_ERR_UNINITIALIZED, "hgnn_model_set_data has not been called");
}

// compute_gradients (model.cpp:556-567) on the device; rank-averaged
// gradients in mgrads, loss in c->last_loss.
void model_compute_gradients(hgnn_ctx* c) {
  const int64_t H = c->H, nl = c->nl;
  ensure_buffers(c);
  {  // encoders (model.cpp:289-294), every row / edge
    Timed t(c, HGNN_K_ENCODE);
    if (H == 64) encode<64>(c);
    else encode<32>(c);
  }
  // message passing (model.cpp:295-300)
  run_forward(c);
  // decoder on local rows (model.cpp:303-306)
  c->y.alloc(std::max<int64_t>(nl * c->fy, 1));
  c->dy.alloc(std::max<int64_t>(nl * c->fy, 1));
  {
    Timed t(c, HGNN_K_DECODE);
    if (H == 64) decode<64>(c);
    else decode<32>(c);
  }
  Timed t_loss(c, HGNN_K_LOSS_ADAM);
  // consistent loss (model.cpp:455-480) and its adjoint (model.cpp:482-500)
  c->loss_part.alloc(2 * kLossBlocks);
  c->loss_st.alloc(3);
  loss_partial_kernel<<<kLossBlocks, kLossThreads, 0, c->stream>>>(c->y.p, c->target.p, c->node_inv.p, nl,
                                                                   (int)c->fy, c->loss_part.p);
  check_launch(c);
  loss_final_kernel<<<1, 32, 0, c->stream>>>(c->loss_part.p, kLossBlocks, c->loss_st.p);
  check_launch(c);
  if (c->nranks > 1) allreduce_sum_f64(c, c->loss_st.p, 2);
  loss_seed_kernel<<<1, 32, 0, c->stream>>>(c->loss_st.p, (int)c->fy, c->nranks);
  check_launch(c);
  loss_backward_kernel<<<blocks_for(nl * c->fy), kEwThreads, 0, c->stream>>>(
      c->y.p, c->target.p, c->node_inv.p, c->loss_st.p + 2, nl, (int)c->fy, c->dy.p);
  check_launch(c);
  t_loss.stop();
  {  // decoder backward (model.cpp:402-409): adjoint of x_M on local rows, halo rows 0
    Timed t(c, HGNN_K_DECODE);
    CUDA_OK(cudaMemsetAsync(c->dx.p, 0, sizeof(float) * (size_t)(c->rows * H), c->stream));
    if (H == 64) decode_backward<64>(c);
    else decode_backward<32>(c);
  }
  // message-passing backward (model.cpp:411-415), de_M = 0 (model.cpp:412)
  if (!c->lean) CUDA_OK(cudaMemsetAsync(c->de.p, 0, sizeof(float) * (size_t)(c->ne * H), c->stream));
  run_backward(c);
  CUDA_OK(cudaMemcpyAsync(c->mgrads.p + c->off_mp, c->grads.p, sizeof(double) * (size_t)c->n_mp_par,
                          cudaMemcpyDeviceToDevice, c->stream));
  {  // encoder backward (model.cpp:417-423)
    Timed t(c, HGNN_K_ENCODE);
    if (H == 64) encode_backward<64>(c);
    else encode_backward<32>(c);
  }
  // average over ranks (model.cpp:516-531)
  if (c->nranks > 1) {
    allreduce_sum_f64(c, c->mgrads.p, c->n_full);
    scale_f64_kernel<<<blocks_for(c->n_full), kEwThreads, 0, c->stream>>>(c->mgrads.p, c->n_full,
                                                                           1.0 / (double)c->nranks);
    check_launch(c);
  }
  double st[2];
  CUDA_OK(cudaMemcpyAsync(st, c->loss_st.p, sizeof(double) * 2, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaStreamSynchronize(c->stream));
  c->last_loss = st[0] / (st[1] * (double)c->fy);
}

// fp32 / tf32 images of the parameters from the fp64 master copy.
void model_refresh_params(hgnn_ctx* c) {
  f64_to_f32_kernel<<<blocks_for(c->n_full), kEwThreads, 0, c->stream>>>(c->mparams.p, c->n_full, c->gen_par.p);
  check_launch(c);
  const double* mp = c->mparams.p + c->off_mp;
  f64_to_f32_kernel<<<blocks_for(c->n_mp_par), kEwThreads, 0, c->stream>>>(mp, c->n_mp_par, c->par.p);
  check_launch(c);
  gather_f64_to_f32_kernel<<<blocks_for(c->n_mp_par), kEwThreads, 0, c->stream>>>(mp, c->pt_src.p, c->n_mp_par,
                                                                                  c->par_t.p);
  check_launch(c);
  if (c->ch_map.n > 0) {
    chunk_refresh_kernel<<<blocks_for(c->ch_map.n), kEwThreads, 0, c->stream>>>(mp, c->ch_map.p, c->ch_map.n,
                                                                              c->chunks.p);
    check_launch(c);
  }
  if (c->bch_map.n > 0) {
    chunk_refresh_kernel<<<blocks_for(c->bch_map.n), kEwThreads, 0, c->stream>>>(mp, c->bch_map.p, c->bch_map.n,
                                                                                c->bchunks.p);
    check_launch(c);
  }
  refresh_enc_chunks(c);
}

// Device-refresh maps of the MP block (same element placement as the host
// builders in hgnn_params_upload).
void build_refresh_maps(hgnn_ctx* c) {
  const int H = (int)c->H, K = (int)c->K;
  std::vector<int32_t> pt((size_t)c->n_mp_par);
  std::vector<uint32_t> ch, bch;
  int64_t off = 0;
  for (int64_t m = 0; m < c->M; ++m)
    for (int which = 0; which < 2; ++which) {
      const int in_dim = (which == 0 ? 3 : 2) * H;
      for (int l = 0; l < K + 2; ++l) {
        const int rin = l == 0 ? in_dim : H;
        const int64_t wo = off + mlp_w_offset(l, in_dim, H), bo = off + mlp_b_offset(l, in_dim, H);
        for (int i = 0; i < rin; ++i)
          for (int j = 0; j < H; ++j) pt[(size_t)(wo + (int64_t)j * rin + i)] = (int32_t)(wo + (int64_t)i * H + j);
        for (int j = 0; j < H; ++j) pt[(size_t)(bo + j)] = (int32_t)(bo + j);
      }
      off += mlp_param_count(in_dim, H, K);
    }
  if (tc_eligible(c)) {
    std::vector<int64_t> fo, bo;
    int64_t nf = 0, nb = 0;
    mp_chunk_plan(H, K, c->M, true, [](bool, int64_t, int64_t, bool) {}, fo, bo, nf, nb);
    ch.resize((size_t)nf);
    bch.resize((size_t)nb);
    mp_chunk_plan(
        H, K, c->M, true,
        [&](bool fwd, int64_t pos, int64_t src, bool lo) {
          (fwd ? ch : bch)[(size_t)pos] = src < 0 ? 0x7fffffffu : ((uint32_t)src | (lo ? 0x80000000u : 0u));
        },
        fo, bo, nf, nb);
  }
  c->pt_src.upload(pt.data(), (int64_t)pt.size(), c->stream);
  c->ch_map.upload(ch.data(), (int64_t)ch.size(), c->stream);
  c->bch_map.upload(bch.data(), (int64_t)bch.size(), c->stream);
  build_enc_map(c);
  refresh_enc_chunks(c);
}


}  // namespace

extern "C" {

// ---- model level ----------------------------------------
int hgnn_model_configure(hgnn_ctx* c, int64_t in_node_dim, int64_t in_edge_dim, int64_t out_dim) {
  return guarded([&] {
    bind(c);
    if (!c->configured) fail(HGNN_ERR_UNINITIALIZED, "hgnn_configure has not been called");
    if (c->H != 64 && c->H != 32) fail(HGNN_ERR_CONFIG, "model level: hidden width 32 or 64");
    if (!gen_supported(in_node_dim, in_edge_dim, out_dim))
      fail(HGNN_ERR_CONFIG, "model level: feature widths (F_x, F_e, F_y) = (3, 7, 3) supported");
    c->fx = in_node_dim;
    c->fe = in_edge_dim;
    c->fy = out_dim;
    const int K = (int)c->K;
    const int H = (int)c->H;
    c->n_ne = gen_param_count((int)c->fx, H, K, true, true, H);
    c->n_ee = gen_param_count((int)c->fe, H, K, true, true, H);
    c->n_dec = gen_param_count(H, (int)c->fy, K, true, false, H);
    c->off_ne = 0;
    c->off_ee = c->n_ne;
    c->off_mp = c->off_ee + c->n_ee;
    c->off_dec = c->off_mp + c->n_mp_par;
    c->n_full = c->off_dec + c->n_dec;
    c->model_configured = true;
    c->model_params_ready = c->model_data_ready = false;
  });
}

int64_t hgnn_model_param_count(hgnn_ctx* c) { return c && c->model_configured ? c->n_full : -1; }

int hgnn_model_params_upload(hgnn_ctx* c, const double* params, int64_t count) {
  return guarded([&] {
    bind(c);
    if (!c->model_configured) fail(HGNN_ERR_UNINITIALIZED, "hgnn_model_configure has not been called");
    if (count != c->n_full)
      fail(HGNN_ERR_SHAPE, "hgnn_model_params_upload: expected " + std::to_string(c->n_full) + " values");
    const int rc = hgnn_params_upload(c, params + c->off_mp, c->n_mp_par);
    if (rc != HGNN_OK) fail(rc, hgnn_last_error());
    c->mparams.upload(params, count, c->stream);
    c->mgrads.alloc(count);
    c->adam_m.alloc(count);
    c->adam_v.alloc(count);
    CUDA_OK(cudaMemsetAsync(c->adam_m.p, 0, sizeof(double) * (size_t)count, c->stream));
    CUDA_OK(cudaMemsetAsync(c->adam_v.p, 0, sizeof(double) * (size_t)count, c->stream));
    c->adam_step = 0;
    c->gen_par.alloc(count);
    f64_to_f32_kernel<<<blocks_for(count), kEwThreads, 0, c->stream>>>(c->mparams.p, count, c->gen_par.p);
    check_launch(c);
    build_refresh_maps(c);
    c->nonfinite.alloc(1);
    CUDA_OK(cudaStreamSynchronize(c->stream));
    c->model_params_ready = true;
  });
}

int hgnn_model_params_download(hgnn_ctx* c, double* params) {
  return guarded([&] {
    bind(c);
    if (!c->model_params_ready) fail(HGNN_ERR_UNINITIALIZED, "hgnn_model_params_upload has not been called");
    CUDA_OK(cudaMemcpy(params, c->mparams.p, sizeof(double) * (size_t)c->n_full, cudaMemcpyDeviceToHost));
  });
}

int hgnn_model_set_data(hgnn_ctx* c, const double* node_features, const double* edge_features,
                        const double* target) {
  return guarded([&] {
    bind(c);
    require_ready(c);
    if (!c->model_configured) fail(HGNN_ERR_UNINITIALIZED, "hgnn_model_configure has not been called");
    if (!node_features || !edge_features) fail(HGNN_ERR_SHAPE, "hgnn_model_set_data: null features");
    if (!c->node_inv.p && c->nl > 0)
      fail(HGNN_ERR_UNINITIALIZED, "hgnn_model_set_data: the graph was uploaded without node_inv_degree");
    ensure_buffers(c);
    c->node_feat.alloc(std::max<int64_t>(c->rows * c->fx, 1));
    rows_to_device(c, node_features, c->rows * c->fx, c->node_feat.p);
    c->edge_feat.alloc(std::max<int64_t>(c->ne * c->fe, 1));
    edges_cols_to_device(c, edge_features, (int)c->fe, c->edge_feat.p);  // edge-id order -> slots
    c->target.alloc(std::max<int64_t>(c->nl * c->fy, 1));
    if (target) {
      rows_to_device(c, target, c->nl * c->fy, c->target.p);
    } else {  // autoencoding (model.cpp:605-607): target = local rows of the node features
      if (c->fy != c->fx) fail(HGNN_ERR_SHAPE, "autoencoding target needs out_dim == in_node_dim");
      CUDA_OK(cudaMemcpyAsync(c->target.p, c->node_feat.p, sizeof(float) * (size_t)(c->nl * c->fy),
                              cudaMemcpyDeviceToDevice, c->stream));
    }
    CUDA_OK(cudaStreamSynchronize(c->stream));
    c->model_data_ready = true;
  });
}

int hgnn_compute_gradients(hgnn_ctx* c, double* loss, double* grads, double* y) {
  return guarded([&] {
    bind(c);
    require_model(c);
    model_compute_gradients(c);
    if (loss) *loss = c->last_loss;
    if (grads) CUDA_OK(cudaMemcpy(grads, c->mgrads.p, sizeof(double) * (size_t)c->n_full, cudaMemcpyDeviceToHost));
    if (y) rows_to_host(c, c->y.p, c->nl * c->fy, y);
  });
}

int hgnn_train_step(hgnn_ctx* c, double lr, double beta1, double beta2, double eps, double* loss) {
  return guarded([&] {
    bind(c);
    require_model(c);
    model_compute_gradients(c);
    Timed t(c, HGNN_K_LOSS_ADAM);
    CUDA_OK(cudaMemsetAsync(c->nonfinite.p, 0, sizeof(int), c->stream));
    nonfinite_kernel<<<blocks_for(c->n_full), kEwThreads, 0, c->stream>>>(c->mgrads.p, c->n_full, c->nonfinite.p);
    check_launch(c);
    int bad = 0;
    CUDA_OK(cudaMemcpyAsync(&bad, c->nonfinite.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    // same error as nn.cpp:352; unlike the reference (which has updated the
    // elements before the bad one) no state changes, so the fp64 master and
    // its fp32 / tf32 working copies stay consistent
    if (bad) fail(HGNN_ERR_OPTIMIZER, "adam_step: non-finite gradient");
    c->adam_step += 1;
    const double bc1 = 1.0 - std::pow(beta1, (double)c->adam_step);
    const double bc2 = 1.0 - std::pow(beta2, (double)c->adam_step);
    adam_kernel<<<blocks_for(c->n_full), kEwThreads, 0, c->stream>>>(c->mparams.p, c->mgrads.p, c->adam_m.p,
                                                                     c->adam_v.p, c->n_full, lr, beta1, beta2, eps,
                                                                     bc1, bc2);
    check_launch(c);
    model_refresh_params(c);
    t.stop();
    CUDA_OK(cudaStreamSynchronize(c->stream));
    if (loss) *loss = c->last_loss;
  });
}

}  // extern "C"
