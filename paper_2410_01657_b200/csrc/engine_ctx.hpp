// Internal state of the device engine shared by engine.cu (message-passing
// stack, C-ABI) and model.cu (encoders, decoder, loss, Adam): the per-rank
// context, device buffers, error macros and the engine helpers model.cu uses.
#pragma once

#include <nccl.h>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "local_group.hpp"
#include "mlp_simt.cuh"
#include "mlp_tc.cuh"

#define CUDA_OK(expr)                                                                                  \
  do {                                                                                                 \
    cudaError_t _e = (expr);                                                                           \
    if (_e != cudaSuccess) fail(HGNN_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));    \
  } while (0)
#define NCCL_OK(expr)                                                                                  \
  do {                                                                                                 \
    ncclResult_t _r = (expr);                                                                          \
    if (_r != ncclSuccess) fail(HGNN_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));    \
  } while (0)

namespace hgnn_b200 {


template <class T>
struct DevBuf {
  T* p = nullptr;
  int64_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(int64_t count) {
    if (count == n && p) return;
    release();
    if (count <= 0) return;
    CUDA_OK(cudaMalloc(&p, sizeof(T) * (size_t)count));
    n = count;
  }
  void upload(const T* h, int64_t count, cudaStream_t s) {
    alloc(count);
    if (count > 0) CUDA_OK(cudaMemcpyAsync(p, h, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice, s));
  }
};

struct EventPair {
  cudaEvent_t a, b;
};


}  // namespace hgnn_b200

struct hgnn_ctx {
  int device = 0;
  int32_t rank = 0, nranks = 1;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  // debug collective-sequence guard for the NCCL path (option "collective_check",
  // the reference poisons mismatched sequences, comm.cpp:168-208)
  int coll_check = 0;
  int64_t coll_timeout_ms = 120000;
  int64_t coll_seq = 0;
  bool comm_aborted = false;
  hgnn_b200::DevBuf<int32_t> coll_sig;
  // in-process rank group (hgnn_ctx_create_local): the exchange and the
  // all-reduces rendezvous on the host and copy device-to-device
  hgnn_b200::LocalGroup* group = nullptr;
  cudaEvent_t ev_pub = nullptr, ev_consumed = nullptr;  // exposed buffer ready / peers' reads done
  const float* xpub = nullptr;                          // buffer this rank exposes to its peers
  int num_sms = 148;

  // configuration
  int64_t H = 0, M = 0, K = 0;
  int mode = HGNN_MODE_NONE;
  bool configured = false, graph_ready = false, params_ready = false, forward_done = false;

  // graph
  int64_t nl = 0, nh = 0, rows = 0, ne = 0, max_buffer_rows = 0;
  hgnn_b200::DevBuf<int32_t> src, dst, twin, slot_of;
  // Slot order: receiver-sorted, and for R > 1 the segments of the boundary
  // rows (rows packed by the halo exchange) first, so the overlapped forward
  // can finish them, start the exchange and run the interior edges meanwhile.
  // Row i's in-edges are slots [seg_beg[i], seg_end[i]) in in-CSR order.
  hgnn_b200::DevBuf<int32_t> seg_beg, seg_end, rows_bnd, rows_int;
  int64_t ne_bnd = 0, n_rows_bnd = 0, n_rows_int = 0;
  int halo_overlap = 1;   // option "halo_overlap": exchange on `side` overlapped with the interior edges
  int halo_sm_reserve = 0;  // option "halo_sm_reserve": SMs the interior edge launches leave to pack / NCCL
  int sm_reserve = 0;       // the reserve in force for the launch being issued
  cudaStream_t side = nullptr;
  cudaEvent_t ev_bnd = nullptr, ev_halo = nullptr;
  hgnn_b200::DevBuf<float> inv;
  hgnn_b200::DevBuf<int64_t> gid;
  // halo
  std::vector<int32_t> h_nbr, h_send_off, h_recv_off;
  std::vector<int64_t> h_recv_base;
  hgnn_b200::DevBuf<int32_t> send_rows, recv_rows, sync_local, sync_off, sync_slots, acc_rows, acc_off;
  hgnn_b200::DevBuf<int64_t> pos_na2a, pos_a2a_send, pos_a2a_recv, acc_pos_na2a, acc_pos_a2a;
  int64_t n_send = 0, n_recv = 0, n_sync = 0, n_acc = 0;
  hgnn_b200::DevBuf<float> sendbuf, recvbuf;

  // parameters (fp32) and gradients (fp64), MP layers
  int64_t n_edge_par = 0, n_node_par = 0, n_mp_par = 0;
  hgnn_b200::DevBuf<float> par, par_t;
  hgnn_b200::DevBuf<float> chunks;                 // tcgen05 B operands, [W_hi | W_lo]^T chunks per MLP
  std::vector<int64_t> chunk_off;       // per (layer, edge / node / factorised edge): mp_chunk_plan
  hgnn_b200::DevBuf<double> grads;
  int fwd_impl = 1;                     // 0 = SIMT, 1 = tcgen05 (H in {32, 64})
  int bwd_impl = 1;                     // 0 = SIMT, 1 = tcgen05 (H = 64)
  hgnn_b200::DevBuf<float> bchunks;                // backward chunk sequence per MLP
  std::vector<int64_t> bchunk_off;
  hgnn_b200::DevBuf<float> tc_scratch;
  hgnn_b200::DevBuf<unsigned long long> prof;      // optional backward-kernel wait profile
  bool prof_on = false;

  // factorised edge MLP (kEdgeFact, edge_fact.cuh): receiver-segment tiles of
  // the fused edge kernel ([0, n_tiles_bnd) cover the boundary slots), rows
  // with an empty segment (zeroed aggregate), node projections per layer
  int edge_fact = 1;              // option "edge_factorized" (default on: measured faster at C3)
  int adj_presum = 0;             // option "adjoint_presum": node-level adjoint with precomputed segment sums (measured slower, off)
  int tma_gather = 0;             // option "tma_gather": fused edge forward input rows by TMA tile::gather4 (H = 64; measured slower, off)
  bool fact_ok = false;           // every receiver segment fits one 128-slot tile
  hgnn_b200::DevBuf<int32_t> tiles, rows_empty;
  int64_t n_tiles = 0, n_tiles_bnd = 0, n_rows_empty = 0;
  std::vector<std::unique_ptr<hgnn_b200::DevBuf<float>>> ps;  // P_m = x_m [W0_s | W0_d], rows x 2H
  std::vector<uint8_t> ps_ready;                              // P_m computed by this forward
  hgnn_b200::DevBuf<float> fact_part;                         // node-level dW0_s / dW0_d partials
  int fact_blocks = 0;

  // memory plan (option "memory_lean": -1 auto = when the standard plan does
  // not fit the device, 0 off, 1 on). Lean: the dead last-layer e' is not
  // stored, the edge adjoint of layer m overwrites e_m (after the backward
  // kernel's reads of that row), one node-projection buffer recomputed per
  // layer, the node-update x adjoint overwrites dx in place, x_M lives in the
  // (then idle) dY buffer, and the bench's dx seed is re-synthesised.
  int lean_opt = -1;
  bool lean = false;
  int64_t plan_key[6] = {-1, -1, -1, -1, -1, -1};
  uint64_t synth_seed = 0;
  bool synth_valid = false;

  // activations
  std::vector<std::unique_ptr<hgnn_b200::DevBuf<float>>> xs, es, as;
  hgnn_b200::DevBuf<float> dx, dxn, d_a, de, dsrc, ddst, dx_in;
  hgnn_b200::DevBuf<float> grad_part, scratch;
  hgnn_b200::DevBuf<double> stage;
  int64_t stage_elems = 0;

  // MLP launch geometry
  int grid_edge_f = 0, grid_edge_b = 0, grid_node_f = 0, grid_node_b = 0;
  size_t smem_edge_f = 0, smem_edge_b = 0, smem_node_f = 0, smem_node_b = 0;
  bool wsm_edge_f = false, wsm_edge_b = false, wsm_node_f = false, wsm_node_b = false;

  // model level: encoders, decoder, consistent loss,
  // gradient averaging, Adam. Parameters: full ModelParams::for_each vector.
  hgnn_b200::DevBuf<double> node_inv;                         // [num_local] 1/d per local node (loss weights)
  int64_t fx = 0, fe = 0, fy = 0;
  bool model_configured = false, model_params_ready = false, model_data_ready = false;
  int64_t off_ne = 0, off_ee = 0, off_mp = 0, off_dec = 0, n_ne = 0, n_ee = 0, n_dec = 0, n_full = 0;
  hgnn_b200::DevBuf<double> mparams, mgrads, adam_m, adam_v;  // fp64 master parameters, gradients, Adam moments
  hgnn_b200::DevBuf<float> gen_par;                           // fp32 copy of the full vector (encoders / decoder read it)
  hgnn_b200::DevBuf<float> node_feat, edge_feat, target, y, dy;
  hgnn_b200::DevBuf<float> gen_part, gen_scratch;
  hgnn_b200::DevBuf<double> loss_part, loss_st;               // block partials; [s, n, seed]
  hgnn_b200::DevBuf<int32_t> pt_src;                          // par_t[i] = par[pt_src[i]] (MP block)
  hgnn_b200::DevBuf<uint32_t> ch_map, bch_map;                // chunk refresh maps (bit 31: tf32 lo part)
  // tcgen05 encoders (option "encoder_impl", H = 64): forward / backward chunk
  // sequences of the node and edge encoder MLPs (zero-padded F-feature input
  // segment), refreshed from the fp64 master through enc_map ([fwd | bwd])
  int enc_impl = 1;
  hgnn_b200::DevBuf<float> enc_ch;
  hgnn_b200::DevBuf<uint32_t> enc_map;                        // 0x7fffffff: zero padding
  int64_t enc_off[6] = {0, 0, 0, 0, 0, 0};                    // fwd node, edge, decoder; bwd node, edge, decoder
  hgnn_b200::DevBuf<float> enc_tmp, enc_part;                 // pre-LN output / its adjoint; LN-adjoint partials
  hgnn_b200::DevBuf<int> nonfinite;
  int64_t adam_step = 0;
  double last_loss = 0.0;

  // instrumentation
  bool timing = false;
  std::vector<hgnn_b200::EventPair> ev[HGNN_K_COUNT];
  size_t ev_used[HGNN_K_COUNT] = {};
  int64_t launches = 0;
  int64_t halo_bytes = 0;
};

namespace hgnn_b200::engine {

inline unsigned blocks_for(int64_t n, int threads = kEwThreads) {
  return (unsigned)std::max<int64_t>(1, (n + threads - 1) / threads);
}


struct Timed {
  hgnn_ctx* c;
  int cls;
  Timed(hgnn_ctx* ctx, int k, cudaStream_t s = nullptr) : c(ctx), cls(k), st(s ? s : ctx->stream) {
    if (!c->timing) return;
    auto& v = c->ev[cls];
    if (c->ev_used[cls] == v.size()) {
      EventPair p;
      CUDA_OK(cudaEventCreate(&p.a));
      CUDA_OK(cudaEventCreate(&p.b));
      v.push_back(p);
    }
    CUDA_OK(cudaEventRecord(v[c->ev_used[cls]].a, st));
  }
  ~Timed() { stop(); }
  void stop() {
    if (!c->timing || done) return;
    done = true;
    cudaEventRecord(c->ev[cls][c->ev_used[cls]].b, st);
    c->ev_used[cls] += 1;
  }
  cudaStream_t st;
  bool done = false;
};

// Chunk layouts of one MLP's tcgen05 B operands. emit(pos, src, lo) places
// element `src` of the MLP's for_each parameter block at chunk float `pos`,
// as its tf32 hi part (lo = false) or lo part (lo = true).
// Forward sequence (mlp_tc.cuh): input segments of W0, W1 .. W_{k+1}.
// seg0 / nseg: the input segments (K = H row blocks of W0) the kernel
// multiplies on the tensor cores: all of them, or only the e block (seg0 = 2,
// nseg = 1) for the factorised edge MLP (kEdgeFact).
// out_dim < H (the decoder): W_{k+1} is H x out_dim, its columns >= out_dim
// are zero padding (src -1).
template <class Emit>
void chunk_layout_fwd(int in_dim, int H, int K, int64_t base, Emit&& emit, int seg0 = 0, int nseg = -1,
                      int out_dim = -1) {
  if (nseg < 0) nseg = in_dim / H;
  if (out_dim < 0) out_dim = H;
  for (int l = 0; l < K + 2; ++l) {
    const int64_t w = mlp_w_offset(l, in_dim, H);
    const int n_ch = l == 0 ? nseg : 1;
    for (int ci = 0; ci < n_ch; ++ci, base += 2 * (int64_t)H * H)
      for (int kk = 0; kk < H; ++kk)
        for (int n = 0; n < H; ++n) {
          const int cidx = l == 0 ? seg0 + ci : 0;
          const int r = cidx * H + kk;  // row of W_l (W0 rows >= in_dim: zero padding, src -1)
          int64_t src = (l == 0 && r >= in_dim) ? -1 : w + (int64_t)r * H + n;
          if (l == K + 1 && out_dim < H) src = n < out_dim ? w + (int64_t)kk * out_dim + n : -1;
          emit(base + tc_chunk_index(n, kk, H), src, false);
          emit(base + tc_chunk_index(H + n, kk, H), src, true);
        }
  }
}
// Backward sequence (mlp_tc_bwd.cuh): the forward chunks of the recompute
// (input segments, hidden linears), then W_{k+1}^T, W_k^T .. W_1^T and W_0^T
// per input segment. A transposed chunk stores element (n = input feature,
// k = output feature) = W[n][k].
template <class Emit>
void chunk_layout_bwd(int in_dim, int H, int K, int64_t base, Emit&& emit, int seg0 = 0, int nseg = -1,
                      int out_dim = -1) {
  if (nseg < 0) nseg = in_dim / H;
  if (out_dim < 0) out_dim = H;
  auto chunk = [&](auto src_of) {
    for (int kk = 0; kk < H; ++kk)
      for (int n = 0; n < H; ++n) {
        const int64_t src = src_of(n, kk);
        emit(base + tc_chunk_index(n, kk, H), src, false);
        emit(base + tc_chunk_index(H + n, kk, H), src, true);
      }
    base += 2 * (int64_t)H * H;
  };
  auto W = [&](int l) { return mlp_w_offset(l, in_dim, H); };
  // W0 rows >= in_dim are zero padding (src -1): the encoders' F-feature input
  for (int c = seg0; c < seg0 + nseg; ++c)
    chunk([&](int n, int kk) { return c * H + kk < in_dim ? W(0) + (int64_t)(c * H + kk) * H + n : (int64_t)-1; });
  for (int l = 1; l <= K; ++l) chunk([&](int n, int kk) { return W(l) + (int64_t)kk * H + n; });
  chunk([&](int n, int kk) { return kk < out_dim ? W(K + 1) + (int64_t)n * out_dim + kk : (int64_t)-1; });
  for (int l = K; l >= 1; --l) chunk([&](int n, int kk) { return W(l) + (int64_t)n * H + kk; });
  for (int c = seg0; c < seg0 + nseg; ++c)
    chunk([&](int n, int kk) { return c * H + n < in_dim ? W(0) + (int64_t)(c * H + n) * H + kk : (int64_t)-1; });
}
// The backward sequence of an H = 32 MLP run zero-padded on the 64-wide
// kernel (mlp_tc_bwd.cuh, HL = 32): same order as chunk_layout_bwd, 64 x 64
// chunks whose entries outside the HL x HL blocks are padding (src -1).
template <class Emit>
void chunk_layout_bwd_pad(int in_dim, int HL, int K, int64_t base, Emit&& emit) {
  constexpr int P = 64;
  const int nseg = in_dim / HL;
  auto chunk = [&](auto src_of) {
    for (int kk = 0; kk < P; ++kk)
      for (int n = 0; n < P; ++n) {
        const int64_t src = (n < HL && kk < HL) ? src_of(n, kk) : (int64_t)-1;
        emit(base + tc_chunk_index(n, kk, P), src, false);
        emit(base + tc_chunk_index(P + n, kk, P), src, true);
      }
    base += 2 * (int64_t)P * P;
  };
  auto W = [&](int l) { return mlp_w_offset(l, in_dim, HL); };
  for (int c = 0; c < nseg; ++c) chunk([&](int n, int kk) { return W(0) + (int64_t)(c * HL + kk) * HL + n; });
  for (int l = 1; l <= K; ++l) chunk([&](int n, int kk) { return W(l) + (int64_t)kk * HL + n; });
  for (int l = K + 1; l >= 1; --l) chunk([&](int n, int kk) { return W(l) + (int64_t)n * HL + kk; });
  for (int c = 0; c < nseg; ++c) chunk([&](int n, int kk) { return W(0) + (int64_t)(c * HL + n) * HL + kk; });
}
inline int64_t chunk_floats_fwd(int in_dim, int H, int K, int nseg = -1) {
  return (int64_t)((nseg < 0 ? in_dim / H : nseg) + K + 1) * 2 * H * H;
}
inline int64_t chunk_floats_bwd(int in_dim, int H, int K, int nseg = -1) {
  return (int64_t)(2 * (nseg < 0 ? in_dim / H : nseg) + 2 * K + 1) * 2 * H * H;
}

// Every tcgen05 weight-chunk sequence of the MP block, in buffer order: per
// layer m the edge MLP (3 input segments), the node MLP, and the factorised
// edge MLP (kEdgeFact: e segment only); fwd offsets at [3 m + {0, 1, 2}], the
// backward sequences (H = 64, or H = 32 zero-padded to 64) likewise. emit(fwd?, pos, src, lo) places
// element src of the MP parameter block; the same code serves the host upload
// and the device refresh maps of the Adam step (src -1: zero padding).
template <class Emit>
void mp_chunk_plan(int H, int K, int64_t M, bool with_bwd, Emit&& emit, std::vector<int64_t>& fwd_off,
                   std::vector<int64_t>& bwd_off, int64_t& fwd_total, int64_t& bwd_total) {
  fwd_off.clear();
  bwd_off.clear();
  fwd_total = bwd_total = 0;
  int64_t off = 0;
  for (int64_t m = 0; m < M; ++m) {
    const int64_t off_edge = off, off_node = off + mlp_param_count(3 * H, H, K);
    for (int v = 0; v < 3; ++v) {
      const int in_dim = (v == 1 ? 2 : 3) * H;
      const int seg0 = v == 2 ? 2 : 0, nseg = v == 2 ? 1 : -1;
      const int64_t poff = v == 1 ? off_node : off_edge;
      fwd_off.push_back(fwd_total);
      chunk_layout_fwd(in_dim, H, K, fwd_total, [&](int64_t pos, int64_t src, bool lo) { emit(true, pos, poff + src, lo); },
                       seg0, nseg);
      fwd_total += chunk_floats_fwd(in_dim, H, K, nseg);
      if (with_bwd) {
        bwd_off.push_back(bwd_total);
        auto e = [&](int64_t pos, int64_t src, bool lo) { emit(false, pos, src < 0 ? src : poff + src, lo); };
        if (H == 64) {
          chunk_layout_bwd(in_dim, H, K, bwd_total, e, seg0, nseg);
          bwd_total += chunk_floats_bwd(in_dim, H, K, nseg);
        } else {  // H = 32: zero-padded 64-wide sequence (no factorised variant: an empty slot)
          if (v != 2) chunk_layout_bwd_pad(in_dim, H, K, bwd_total, e);
          if (v != 2) bwd_total += chunk_floats_bwd(in_dim / H * 64, 64, K);
        }
      }
    }
    off = off_node + mlp_param_count(2 * H, H, K);
  }
}

// Buffer views of the memory plan (see hgnn_ctx::lean).
inline float* x_buf(hgnn_ctx* c, int64_t m) {
  return (c->lean && m == c->M) ? c->dsrc.p : c->xs[(size_t)m]->p;
}
inline float* e_buf(hgnn_ctx* c, int64_t m) {  // nullptr: not materialised (lean, m = M)
  return (c->lean && m == c->M) ? nullptr : c->es[(size_t)m]->p;
}
inline const float* de_in_buf(hgnn_ctx* c, int64_t m) {  // adjoint of e_{m+1} (nullptr: zero)
  if (!c->lean) return c->de.p;
  return m + 1 == c->M ? nullptr : c->es[(size_t)m + 1]->p;
}
inline float* de_out_buf(hgnn_ctx* c, int64_t m) { return c->lean ? c->es[(size_t)m]->p : c->de.p; }
inline float* dxn_buf(hgnn_ctx* c) { return c->lean ? c->dx.p : c->dxn.p; }
inline float* proj_buf(hgnn_ctx* c, int64_t m) { return c->ps[c->lean ? 0 : (size_t)m]->p; }

void bind(hgnn_ctx* c);
// in-place sum over ranks of n device doubles on the compute stream (NCCL, or
// the in-process group's host rendezvous in rank order)
void allreduce_sum_f64(hgnn_ctx* c, double* d, int64_t n);
void check_launch(hgnn_ctx* c);
bool tc_eligible(const hgnn_ctx* c);
void ensure_buffers(hgnn_ctx* c);
void require_ready(hgnn_ctx* c);
void run_forward(hgnn_ctx* c);
void run_backward(hgnn_ctx* c);
// fp64 host rows -> fp32 device (n values), and back (synchronous)
void rows_to_device(hgnn_ctx* c, const double* h, int64_t n, float* d);
void rows_to_host(hgnn_ctx* c, const float* d, int64_t n, double* h);
// N_e x cols fp64 host rows in reference edge-id order -> fp32 receiver-sorted slots
void edges_cols_to_device(hgnn_ctx* c, const double* h, int cols, float* d);

}  // namespace hgnn_b200::engine
