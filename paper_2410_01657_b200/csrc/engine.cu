// Device engine of the consistent NMP layer: per-rank context, receiver-sorted
// graph layout, parameter staging, the forward / backward MP stack, NCCL halo
// exchange over NVLink and the C-ABI declared in include/hgnn_b200.h.
//
// Per-rank HBM layout (fp32, row-major, H = hidden width):
//   xs[m]  rows x H     node state entering layer m (m = 0..M; halo rows = 0 for m > 0)
//   es[m]  N_e x H      edge state entering layer m, receiver-sorted slots
//   as[m]  rows x H     synchronised aggregate a* of layer m (backward recompute input)
//   dx, dxn, d_a        node adjoints;  de, dsrc, ddst  edge adjoints (N_e x H)
// Edge slot p = position in the reference in-CSR (graph.cpp:122-136); the
// boundary permutes to / from the reference edge-id order.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "graph_kernels.cuh"
#include "mlp_simt.cuh"
#include "mlp_tc.cuh"
#include "mlp_tc_bwd.cuh"
#include "mlp_generic.cuh"
#include "model_kernels.cuh"

using namespace hgnn_b200;

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

namespace {

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

}  // namespace

struct hgnn_ctx {
  int device = 0;
  int32_t rank = 0, nranks = 1;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  int num_sms = 148;

  // configuration
  int64_t H = 0, M = 0, K = 0;
  int mode = HGNN_MODE_NONE;
  bool configured = false, graph_ready = false, params_ready = false, forward_done = false;

  // graph
  int64_t nl = 0, nh = 0, rows = 0, ne = 0, max_buffer_rows = 0;
  DevBuf<int32_t> src, dst, in_off, twin, slot_of;
  DevBuf<float> inv;
  DevBuf<int64_t> gid;
  // halo
  std::vector<int32_t> h_nbr, h_send_off, h_recv_off;
  std::vector<int64_t> h_recv_base;
  DevBuf<int32_t> send_rows, recv_rows, sync_local, sync_off, sync_slots, acc_rows, acc_off;
  DevBuf<int64_t> pos_na2a, pos_a2a_send, pos_a2a_recv, acc_pos_na2a, acc_pos_a2a;
  int64_t n_send = 0, n_recv = 0, n_sync = 0, n_acc = 0;
  DevBuf<float> sendbuf, recvbuf;

  // parameters (fp32) and gradients (fp64), MP layers
  int64_t n_edge_par = 0, n_node_par = 0, n_mp_par = 0;
  DevBuf<float> par, par_t;
  DevBuf<float> chunks;                 // tcgen05 B operands, [W_hi | W_lo]^T chunks per MLP
  std::vector<int64_t> chunk_off;       // per (layer, edge/node)
  DevBuf<double> grads;
  int fwd_impl = 1;                     // 0 = SIMT, 1 = tcgen05 (H in {32, 64})
  int bwd_impl = 1;                     // 0 = SIMT, 1 = tcgen05 (H = 64)
  DevBuf<float> bchunks;                // backward chunk sequence per MLP
  std::vector<int64_t> bchunk_off;
  DevBuf<float> tc_scratch;
  DevBuf<unsigned long long> prof;      // optional backward-kernel wait profile
  bool prof_on = false;

  // activations
  std::vector<std::unique_ptr<DevBuf<float>>> xs, es, as;
  DevBuf<float> dx, dxn, d_a, de, dsrc, ddst, dx_in;
  DevBuf<float> grad_part, scratch;
  DevBuf<double> stage;
  int64_t stage_elems = 0;

  // MLP launch geometry
  int grid_edge_f = 0, grid_edge_b = 0, grid_node_f = 0, grid_node_b = 0;
  size_t smem_edge_f = 0, smem_edge_b = 0, smem_node_f = 0, smem_node_b = 0;
  bool wsm_edge_f = false, wsm_edge_b = false, wsm_node_f = false, wsm_node_b = false;

  // model level: encoders, decoder, consistent loss,
  // gradient averaging, Adam. Parameters: full ModelParams::for_each vector.
  DevBuf<double> node_inv;                         // [num_local] 1/d per local node (loss weights)
  int64_t fx = 0, fe = 0, fy = 0;
  bool model_configured = false, model_params_ready = false, model_data_ready = false;
  int64_t off_ne = 0, off_ee = 0, off_mp = 0, off_dec = 0, n_ne = 0, n_ee = 0, n_dec = 0, n_full = 0;
  DevBuf<double> mparams, mgrads, adam_m, adam_v;  // fp64 master parameters, gradients, Adam moments
  DevBuf<float> gen_par;                           // fp32 copy of the full vector (encoders / decoder read it)
  DevBuf<float> node_feat, edge_feat, target, y, dy;
  DevBuf<float> gen_part, gen_scratch;
  DevBuf<double> loss_part, loss_st;               // block partials; [s, n, seed]
  DevBuf<int32_t> pt_src;                          // par_t[i] = par[pt_src[i]] (MP block)
  DevBuf<uint32_t> ch_map, bch_map;                // chunk refresh maps (bit 31: tf32 lo part)
  DevBuf<int> nonfinite;
  int64_t adam_step = 0;
  double last_loss = 0.0;

  // instrumentation
  bool timing = false;
  std::vector<EventPair> ev[HGNN_K_COUNT];
  size_t ev_used[HGNN_K_COUNT] = {};
  int64_t launches = 0;
  int64_t halo_bytes = 0;
};

namespace {

void bind(hgnn_ctx* c) {
  if (!c) fail(HGNN_ERR_CONFIG, "null hgnn_ctx");
  CUDA_OK(cudaSetDevice(c->device));
}

inline unsigned blocks_for(int64_t n, int threads = kEwThreads) {
  return (unsigned)std::max<int64_t>(1, (n + threads - 1) / threads);
}

void check_launch(hgnn_ctx* c) {
  c->launches += 1;
  CUDA_OK(cudaGetLastError());
}

struct Timed {
  hgnn_ctx* c;
  int cls;
  Timed(hgnn_ctx* ctx, int k) : c(ctx), cls(k) {
    if (!c->timing) return;
    auto& v = c->ev[cls];
    if (c->ev_used[cls] == v.size()) {
      EventPair p;
      CUDA_OK(cudaEventCreate(&p.a));
      CUDA_OK(cudaEventCreate(&p.b));
      v.push_back(p);
    }
    CUDA_OK(cudaEventRecord(v[c->ev_used[cls]].a, c->stream));
  }
  ~Timed() { stop(); }
  void stop() {
    if (!c->timing || done) return;
    done = true;
    cudaEventRecord(c->ev[cls][c->ev_used[cls]].b, c->stream);
    c->ev_used[cls] += 1;
  }
  bool done = false;
};

// --------------------------------------------------------------------------
// MLP kernel dispatch over the supported hidden widths
// --------------------------------------------------------------------------
template <int H>
struct MlpKernels {
  static void* fwd(int mode, bool wsm) {
    if (mode == kEdgeInput)
      return wsm ? (void*)mlp_forward_kernel<H, kEdgeInput, true> : (void*)mlp_forward_kernel<H, kEdgeInput, false>;
    return wsm ? (void*)mlp_forward_kernel<H, kNodeInput, true> : (void*)mlp_forward_kernel<H, kNodeInput, false>;
  }
  static void* bwd(int mode, bool wsm) {
    if (mode == kEdgeInput)
      return wsm ? (void*)mlp_backward_kernel<H, kEdgeInput, true> : (void*)mlp_backward_kernel<H, kEdgeInput, false>;
    return wsm ? (void*)mlp_backward_kernel<H, kNodeInput, true> : (void*)mlp_backward_kernel<H, kNodeInput, false>;
  }
};

void* mlp_kernel(int64_t H, bool forward, int mode, bool wsm) {
  switch (H) {
    case 8: return forward ? MlpKernels<8>::fwd(mode, wsm) : MlpKernels<8>::bwd(mode, wsm);
    case 16: return forward ? MlpKernels<16>::fwd(mode, wsm) : MlpKernels<16>::bwd(mode, wsm);
    case 32: return forward ? MlpKernels<32>::fwd(mode, wsm) : MlpKernels<32>::bwd(mode, wsm);
    case 64: return forward ? MlpKernels<64>::fwd(mode, wsm) : MlpKernels<64>::bwd(mode, wsm);
    default: fail(HGNN_ERR_CONFIG, "hidden_dim must be one of 8, 16, 32, 64 on this build");
  }
}

// Picks shared-memory residency of the weights and a persistent grid.
void plan_mlp(hgnn_ctx* c, bool forward, int mode, int64_t n_rows, int& grid, size_t& smem, bool& wsm) {
  const int in_dim = (mode == kEdgeInput ? 3 : 2) * (int)c->H;
  const int64_t n_par = mlp_param_count(in_dim, (int)c->H, (int)c->K);
  const size_t cols = (size_t)(forward ? 1 : 2) * (size_t)c->H * kColStride * sizeof(float);
  const size_t with_w = (size_t)((n_par + 3) / 4) * 4 * sizeof(float) + cols;
  int max_optin = 0;
  CUDA_OK(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  wsm = with_w <= (size_t)max_optin;
  smem = wsm ? with_w : cols;
  void* k = mlp_kernel(c->H, forward, mode, wsm);
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kMlpThreads, smem));
  per_sm = std::max(per_sm, 1);
  const int64_t tiles = std::max<int64_t>(1, (n_rows + kMlpThreads - 1) / kMlpThreads);
  grid = (int)std::min<int64_t>(tiles, (int64_t)per_sm * c->num_sms);
}

void launch_mlp(hgnn_ctx* c, bool forward, int mode, const MlpRowArgs& args, const MlpParamsDev& prm) {
  int grid;
  size_t smem;
  bool wsm;
  if (mode == kEdgeInput) {
    grid = forward ? c->grid_edge_f : c->grid_edge_b;
    smem = forward ? c->smem_edge_f : c->smem_edge_b;
    wsm = forward ? c->wsm_edge_f : c->wsm_edge_b;
  } else {
    grid = forward ? c->grid_node_f : c->grid_node_b;
    smem = forward ? c->smem_node_f : c->smem_node_b;
    wsm = forward ? c->wsm_node_f : c->wsm_node_b;
  }
  if (args.n_rows == 0) return;
  void* k = mlp_kernel(c->H, forward, mode, wsm);
  MlpRowArgs a = args;
  MlpParamsDev p = prm;
  void* params[] = {&a, &p};
  CUDA_OK(cudaLaunchKernel(k, dim3(grid), dim3(kMlpThreads), params, smem, c->stream));
  check_launch(c);
}

// --------------------------------------------------------------------------
// tcgen05 weight chunks (host-side layout, mlp_tc.cuh)
// --------------------------------------------------------------------------
float tf32_rna_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

bool tc_eligible(const hgnn_ctx* c) { return c->H == 32 || c->H == 64; }

// Chunks of one processor MLP in MMA order: the input linear split into
// nseg K-chunks of H rows, then one chunk per H x H linear. Each chunk is the
// B operand [W_hi | W_lo]^T (2H x H) in K-major core-matrix order.
// Chunk layouts of one MLP's tcgen05 B operands. emit(pos, src, lo) places
// element `src` of the MLP's for_each parameter block at chunk float `pos`,
// as its tf32 hi part (lo = false) or lo part (lo = true).
// Forward sequence (mlp_tc.cuh): input segments of W0, W1 .. W_{k+1}.
template <class Emit>
void chunk_layout_fwd(int in_dim, int H, int K, int64_t base, Emit&& emit) {
  const int nseg = in_dim / H;
  for (int l = 0; l < K + 2; ++l) {
    const int64_t w = mlp_w_offset(l, in_dim, H);
    const int n_ch = l == 0 ? nseg : 1;
    for (int cidx = 0; cidx < n_ch; ++cidx, base += 2 * (int64_t)H * H)
      for (int kk = 0; kk < H; ++kk)
        for (int n = 0; n < H; ++n) {
          const int64_t src = w + (int64_t)(cidx * H + kk) * H + n;
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
void chunk_layout_bwd(int in_dim, int H, int K, int64_t base, Emit&& emit) {
  const int nseg = in_dim / H;
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
  for (int c = 0; c < nseg; ++c) chunk([&](int n, int kk) { return W(0) + (int64_t)(c * H + kk) * H + n; });
  for (int l = 1; l <= K; ++l) chunk([&](int n, int kk) { return W(l) + (int64_t)kk * H + n; });
  for (int l = K + 1; l >= 1; --l) chunk([&](int n, int kk) { return W(l) + (int64_t)n * H + kk; });
  for (int c = 0; c < nseg; ++c) chunk([&](int n, int kk) { return W(0) + (int64_t)(c * H + n) * H + kk; });
}
int64_t chunk_floats_fwd(int in_dim, int H, int K) { return (int64_t)(in_dim / H + K + 1) * 2 * H * H; }
int64_t chunk_floats_bwd(int in_dim, int H, int K) { return (int64_t)(2 * (in_dim / H) + 2 * K + 1) * 2 * H * H; }

void build_chunks(const float* p, int in_dim, int H, int K, std::vector<float>& out) {
  const int64_t base = (int64_t)out.size();
  out.resize((size_t)(base + chunk_floats_fwd(in_dim, H, K)));
  chunk_layout_fwd(in_dim, H, K, base, [&](int64_t pos, int64_t src, bool lo) {
    const float hi = tf32_rna_host(p[src]);
    out[(size_t)pos] = lo ? tf32_rna_host(p[src] - hi) : hi;
  });
}
void build_bwd_chunks(const float* p, int in_dim, int H, int K, std::vector<float>& out) {
  const int64_t base = (int64_t)out.size();
  out.resize((size_t)(base + chunk_floats_bwd(in_dim, H, K)));
  chunk_layout_bwd(in_dim, H, K, base, [&](int64_t pos, int64_t src, bool lo) {
    const float hi = tf32_rna_host(p[src]);
    out[(size_t)pos] = lo ? tf32_rna_host(p[src] - hi) : hi;
  });
}

// --------------------------------------------------------------------------
// buffers
// --------------------------------------------------------------------------
void ensure_buffers(hgnn_ctx* c) {
  if (!c->configured) fail(HGNN_ERR_UNINITIALIZED, "hgnn_configure has not been called");
  if (!c->graph_ready) fail(HGNN_ERR_UNINITIALIZED, "hgnn_graph_upload has not been called");
  const int64_t H = c->H, M = c->M;
  if (c->xs.size() != (size_t)(M + 1) || (c->xs.size() && c->xs[0]->n != c->rows * H) ||
      (c->es.size() && c->es[0]->n != c->ne * H)) {
    c->xs.clear();
    c->es.clear();
    c->as.clear();
    for (int64_t m = 0; m <= M; ++m) {
      c->xs.emplace_back(new DevBuf<float>());
      c->xs.back()->alloc(c->rows * H);
      c->es.emplace_back(new DevBuf<float>());
      c->es.back()->alloc(std::max<int64_t>(1, c->ne * H));
      if (m < M) {
        c->as.emplace_back(new DevBuf<float>());
        c->as.back()->alloc(c->rows * H);
      }
    }
    c->dx.alloc(c->rows * H);
    c->dx_in.alloc(c->rows * H);
    c->d_a.alloc(c->rows * H);
    c->dxn.alloc(std::max<int64_t>(1, c->nl * H));
    c->de.alloc(std::max<int64_t>(1, c->ne * H));
    c->dsrc.alloc(std::max<int64_t>(1, c->ne * H));
    c->ddst.alloc(std::max<int64_t>(1, c->ne * H));
  }
  plan_mlp(c, true, kEdgeInput, c->ne, c->grid_edge_f, c->smem_edge_f, c->wsm_edge_f);
  plan_mlp(c, false, kEdgeInput, c->ne, c->grid_edge_b, c->smem_edge_b, c->wsm_edge_b);
  plan_mlp(c, true, kNodeInput, c->nl, c->grid_node_f, c->smem_node_f, c->wsm_node_f);
  plan_mlp(c, false, kNodeInput, c->nl, c->grid_node_b, c->smem_node_b, c->wsm_node_b);
  const int64_t max_grid = std::max<int64_t>({c->grid_edge_b, c->grid_node_b, (int64_t)c->num_sms});
  const int64_t max_par = std::max(c->n_edge_par, c->n_node_par);
  c->grad_part.alloc(2 * max_grid * max_par);  // tcgen05 backward keeps two partials per CTA
  const int64_t n_slots = (2 * c->K + 1) * H + c->K;
  c->scratch.alloc(max_grid * n_slots * kMlpThreads);
  if (c->H == 64) c->tc_scratch.alloc((int64_t)c->num_sms * 2 * std::max<int64_t>(c->K, 1) * (16 * 128 * 4 + 128));
  c->stage_elems = std::min<int64_t>(std::max<int64_t>(c->rows, c->ne) * H, int64_t{1} << 24);
  c->stage.alloc(std::max<int64_t>(c->stage_elems, 1));
  // halo buffers
  const int64_t a2a = (int64_t)c->nranks * c->max_buffer_rows;
  c->sendbuf.alloc(std::max<int64_t>({c->n_send, a2a, 1}) * H);
  c->recvbuf.alloc(std::max<int64_t>({c->n_send, a2a, 1}) * H);
}

// --------------------------------------------------------------------------
// boundary transfers (chunked through a device fp64 staging buffer)
// --------------------------------------------------------------------------
void rows_to_device(hgnn_ctx* c, const double* h, int64_t n, float* d) {
  for (int64_t o = 0; o < n; o += c->stage_elems) {
    const int64_t m = std::min(c->stage_elems, n - o);
    CUDA_OK(cudaMemcpyAsync(c->stage.p, h + o, sizeof(double) * (size_t)m, cudaMemcpyHostToDevice, c->stream));
    rows_f64_to_f32_kernel<<<blocks_for(m), kEwThreads, 0, c->stream>>>(c->stage.p, m, d + o);
    check_launch(c);
  }
}
void rows_to_host(hgnn_ctx* c, const float* d, int64_t n, double* h) {
  for (int64_t o = 0; o < n; o += c->stage_elems) {
    const int64_t m = std::min(c->stage_elems, n - o);
    rows_f32_to_f64_kernel<<<blocks_for(m), kEwThreads, 0, c->stream>>>(d + o, m, c->stage.p);
    check_launch(c);
    CUDA_OK(cudaMemcpyAsync(h + o, c->stage.p, sizeof(double) * (size_t)m, cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_OK(cudaStreamSynchronize(c->stream));
}
void edges_to_device(hgnn_ctx* c, const double* h, float* d) {
  const int64_t H = c->H, per = std::max<int64_t>(1, c->stage_elems / H);
  for (int64_t e0 = 0; e0 < c->ne; e0 += per) {
    const int64_t m = std::min(per, c->ne - e0);
    CUDA_OK(cudaMemcpyAsync(c->stage.p, h + e0 * H, sizeof(double) * (size_t)(m * H), cudaMemcpyHostToDevice,
                            c->stream));
    edges_in_kernel<<<blocks_for(m * H), kEwThreads, 0, c->stream>>>(c->stage.p, c->slot_of.p, e0, m, (int)H, d);
    check_launch(c);
  }
}
void edges_to_host(hgnn_ctx* c, const float* d, double* h) {
  const int64_t H = c->H, per = std::max<int64_t>(1, c->stage_elems / H);
  for (int64_t e0 = 0; e0 < c->ne; e0 += per) {
    const int64_t m = std::min(per, c->ne - e0);
    edges_out_kernel<<<blocks_for(m * H), kEwThreads, 0, c->stream>>>(d, c->slot_of.p, e0, m, (int)H, c->stage.p);
    check_launch(c);
    CUDA_OK(cudaMemcpyAsync(h + e0 * H, c->stage.p, sizeof(double) * (size_t)(m * H), cudaMemcpyDeviceToHost,
                            c->stream));
  }
  CUDA_OK(cudaStreamSynchronize(c->stream));
}

// --------------------------------------------------------------------------
// halo exchange (comm.cpp:281-357) over NCCL point-to-point
// --------------------------------------------------------------------------
void halo_exchange(hgnn_ctx* c, float* a) {
  Timed t(c, HGNN_K_HALO);
  const int64_t H = c->H;
  const int R = c->nranks;
  if (c->mode == HGNN_MODE_NA2A) {
    if (c->n_send > 0) {
      gather_rows_kernel<<<blocks_for(c->n_send * H / 4), kEwThreads, 0, c->stream>>>(a, c->send_rows.p, nullptr,
                                                                                     c->n_send, (int)H, c->sendbuf.p);
      check_launch(c);
    }
    if (R > 1 && !c->h_nbr.empty()) {
      NCCL_OK(ncclGroupStart());
      for (size_t n = 0; n < c->h_nbr.size(); ++n) {
        const int64_t cs = c->h_send_off[n + 1] - c->h_send_off[n];
        const int64_t cr = c->h_recv_off[n + 1] - c->h_recv_off[n];
        NCCL_OK(ncclSend(c->sendbuf.p + (int64_t)c->h_send_off[n] * H, (size_t)(cs * H), ncclFloat, c->h_nbr[n],
                         c->comm, c->stream));
        NCCL_OK(ncclRecv(a + c->h_recv_base[n] * H, (size_t)(cr * H), ncclFloat, c->h_nbr[n], c->comm, c->stream));
        c->halo_bytes += cs * H * (int64_t)sizeof(float);
      }
      NCCL_OK(ncclGroupEnd());
    }
  } else if (c->mode == HGNN_MODE_A2A) {
    const int64_t pad = c->max_buffer_rows;
    if (pad == 0 || R == 1) return;
    CUDA_OK(cudaMemsetAsync(c->sendbuf.p, 0, sizeof(float) * (size_t)(R * pad * H), c->stream));
    if (c->n_send > 0) {
      gather_rows_kernel<<<blocks_for(c->n_send * H / 4), kEwThreads, 0, c->stream>>>(
          a, c->send_rows.p, c->pos_a2a_send.p, c->n_send, (int)H, c->sendbuf.p);
      check_launch(c);
    }
    NCCL_OK(ncclGroupStart());
    for (int d = 0; d < R; ++d) {
      NCCL_OK(ncclSend(c->sendbuf.p + (int64_t)d * pad * H, (size_t)(pad * H), ncclFloat, d, c->comm, c->stream));
      NCCL_OK(ncclRecv(c->recvbuf.p + (int64_t)d * pad * H, (size_t)(pad * H), ncclFloat, d, c->comm, c->stream));
    }
    NCCL_OK(ncclGroupEnd());
    c->halo_bytes += (int64_t)R * pad * H * (int64_t)sizeof(float);
    if (c->n_recv > 0) {
      scatter_rows_kernel<<<blocks_for(c->n_recv * H / 4), kEwThreads, 0, c->stream>>>(
          c->recvbuf.p, c->pos_a2a_recv.p, c->recv_rows.p, c->n_recv, (int)H, a);
      check_launch(c);
    }
  }
}

void halo_exchange_adjoint(hgnn_ctx* c, float* d_a) {
  Timed t(c, HGNN_K_HALO);
  const int64_t H = c->H;
  const int R = c->nranks;
  const int64_t* acc_pos = nullptr;
  if (c->mode == HGNN_MODE_NA2A) {
    if (R > 1 && !c->h_nbr.empty()) {
      NCCL_OK(ncclGroupStart());
      for (size_t n = 0; n < c->h_nbr.size(); ++n) {
        const int64_t cs = c->h_send_off[n + 1] - c->h_send_off[n];
        const int64_t cr = c->h_recv_off[n + 1] - c->h_recv_off[n];
        // halo rows of neighbour n are one contiguous block: sent as they lie
        NCCL_OK(ncclSend(d_a + c->h_recv_base[n] * H, (size_t)(cr * H), ncclFloat, c->h_nbr[n], c->comm, c->stream));
        NCCL_OK(ncclRecv(c->recvbuf.p + (int64_t)c->h_send_off[n] * H, (size_t)(cs * H), ncclFloat, c->h_nbr[n],
                         c->comm, c->stream));
        c->halo_bytes += cr * H * (int64_t)sizeof(float);
      }
      NCCL_OK(ncclGroupEnd());
    }
    acc_pos = c->acc_pos_na2a.p;
  } else if (c->mode == HGNN_MODE_A2A) {
    const int64_t pad = c->max_buffer_rows;
    if (pad == 0 || R == 1) return;
    CUDA_OK(cudaMemsetAsync(c->sendbuf.p, 0, sizeof(float) * (size_t)(R * pad * H), c->stream));
    if (c->n_recv > 0) {
      gather_rows_kernel<<<blocks_for(c->n_recv * H / 4), kEwThreads, 0, c->stream>>>(
          d_a, c->recv_rows.p, c->pos_a2a_recv.p, c->n_recv, (int)H, c->sendbuf.p);
      check_launch(c);
    }
    NCCL_OK(ncclGroupStart());
    for (int d = 0; d < R; ++d) {
      NCCL_OK(ncclSend(c->sendbuf.p + (int64_t)d * pad * H, (size_t)(pad * H), ncclFloat, d, c->comm, c->stream));
      NCCL_OK(ncclRecv(c->recvbuf.p + (int64_t)d * pad * H, (size_t)(pad * H), ncclFloat, d, c->comm, c->stream));
    }
    NCCL_OK(ncclGroupEnd());
    c->halo_bytes += (int64_t)R * pad * H * (int64_t)sizeof(float);
    acc_pos = c->acc_pos_a2a.p;
  } else {
    return;
  }
  // the overwritten halo rows contribute nothing upstream (comm.cpp:339-342)
  if (c->nh > 0)
    CUDA_OK(cudaMemsetAsync(d_a + c->nl * H, 0, sizeof(float) * (size_t)(c->nh * H), c->stream));
  if (c->n_acc > 0 && R > 1) {
    adjoint_accumulate_kernel<<<blocks_for(c->n_acc * H / 4), kEwThreads, 0, c->stream>>>(
        d_a, c->recvbuf.p, c->acc_rows.p, c->acc_off.p, acc_pos, c->n_acc, (int)H);
    check_launch(c);
  }
}

// --------------------------------------------------------------------------
// MP stack
// --------------------------------------------------------------------------
MlpParamsDev layer_params(hgnn_ctx* c, int64_t m, bool edge) {
  const int64_t off = m * (c->n_edge_par + c->n_node_par) + (edge ? 0 : c->n_edge_par);
  MlpParamsDev p;
  p.p = c->par.p + off;
  p.wt = c->par_t.p + off;
  p.k = (int)c->K;
  p.in_dim = (int)((edge ? 3 : 2) * c->H);
  return p;
}

bool use_tc(const hgnn_ctx* c) { return c->fwd_impl == 1 && tc_eligible(c); }

template <int H, int MODE>
void launch_tc_typed(hgnn_ctx* c, const TcFwdArgs& args) {
  using Cfg = TcCfg<H>;
  const bool prof = args.prof != nullptr;
  auto k = prof ? mlp_tc_forward_kernel<H, MODE, true> : mlp_tc_forward_kernel<H, MODE, false>;
  static bool attr[2] = {false, false};
  if (!attr[prof]) {
    CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    attr[prof] = true;
  }
  const int64_t pairs = ((args.n_rows + 127) / 128 + 1) / 2;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(pairs, c->num_sms));
  k<<<grid, Cfg::THREADS, Cfg::SMEM, c->stream>>>(args);
  check_launch(c);
}

void launch_tc_forward(hgnn_ctx* c, int mode, int64_t m, int64_t n_rows, const float* x, const float* e,
                       const float* a, float* out) {
  if (n_rows == 0) return;
  const bool edge = mode == kEdgeInput;
  TcFwdArgs args{};
  args.n_rows = n_rows;
  args.src = c->src.p;
  args.dst = c->dst.p;
  args.x = x;
  args.e_in = e;
  args.a = a;
  args.out = out;
  args.chunks = c->chunks.p + c->chunk_off[(size_t)(2 * m + (edge ? 0 : 1))];
  args.params = layer_params(c, m, edge).p;
  args.k = (int)c->K;
  args.prof = c->prof_on ? c->prof.p + 2 * kProfCount + (edge ? 0 : kProfCount) : nullptr;
  if (c->H == 64) {
    if (edge) launch_tc_typed<64, kEdgeInput>(c, args);
    else launch_tc_typed<64, kNodeInput>(c, args);
  } else {
    if (edge) launch_tc_typed<32, kEdgeInput>(c, args);
    else launch_tc_typed<32, kNodeInput>(c, args);
  }
}

bool use_tc_bwd(const hgnn_ctx* c) { return c->bwd_impl == 1 && c->H == 64; }

int tc_bwd_grid(const hgnn_ctx* c, int64_t n_rows) {
  const int64_t pairs = ((n_rows + 127) / 128 + 1) / 2;
  return (int)std::max<int64_t>(1, std::min<int64_t>(pairs, c->num_sms));
}

// Returns the grid used (rows of grad_part written).
int launch_tc_backward(hgnn_ctx* c, int mode, int64_t m, const TcBwdArgs& in) {
  const bool edge = mode == kEdgeInput;
  TcBwdArgs args = in;
  args.chunks = c->bchunks.p + c->bchunk_off[(size_t)(2 * m + (edge ? 0 : 1))];
  args.params = layer_params(c, m, edge).p;
  args.k = (int)c->K;
  args.scratch = c->tc_scratch.p;
  args.prof = c->prof_on ? c->prof.p + (edge ? 0 : kProfCount) : nullptr;
  const int grid = tc_bwd_grid(c, args.n_rows);
  const bool prof = args.prof != nullptr;
  auto k = edge ? (prof ? mlp_tc_backward_kernel<kEdgeInput, true> : mlp_tc_backward_kernel<kEdgeInput, false>)
                : (prof ? mlp_tc_backward_kernel<kNodeInput, true> : mlp_tc_backward_kernel<kNodeInput, false>);
  static bool attr[2][2] = {{false, false}, {false, false}};
  if (!attr[edge][prof]) {
    CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TcBwdCfg::SMEM));
    attr[edge][prof] = true;
  }
  k<<<grid, TcBwdCfg::THREADS, TcBwdCfg::SMEM, c->stream>>>(args);
  check_launch(c);
  return grid;
}

void layer_forward(hgnn_ctx* c, int64_t m) {
  const int64_t H = c->H;
  float* x = c->xs[m]->p;
  float* e = c->es[m]->p;
  float* e2 = c->es[m + 1]->p;
  float* a = c->as[m]->p;
  float* x2 = c->xs[m + 1]->p;
  {  // edge update (model.cpp:233-235)
    Timed t(c, HGNN_K_EDGE_FWD);
    if (use_tc(c)) {
      launch_tc_forward(c, kEdgeInput, m, c->ne, x, e, nullptr, e2);
    } else {
      MlpRowArgs args{};
      args.n_rows = c->ne;
      args.src = c->src.p;
      args.dst = c->dst.p;
      args.x = x;
      args.e_in = e;
      args.out = e2;
      launch_mlp(c, true, kEdgeInput, args, layer_params(c, m, true));
    }
  }
  {  // degree-scaled aggregation (model.cpp:237-240)
    Timed t(c, HGNN_K_AGG);
    aggregate_kernel<<<blocks_for(c->rows * H / 4), kEwThreads, 0, c->stream>>>(e2, c->inv.p, c->in_off.p, c->rows,
                                                                               (int)H, a);
    check_launch(c);
  }
  if (c->mode != HGNN_MODE_NONE) {  // exchange + synchronisation (model.cpp:243-257)
    halo_exchange(c, a);
    if (c->n_sync > 0) {
      Timed t(c, HGNN_K_HALO);
      sync_kernel<<<blocks_for(c->n_sync * H / 4), kEwThreads, 0, c->stream>>>(a, c->sync_local.p, c->sync_off.p,
                                                                              c->sync_slots.p, c->n_sync, (int)H);
      check_launch(c);
    }
  }
  {  // node update on local rows (model.cpp:260-264)
    Timed t(c, HGNN_K_NODE_FWD);
    if (c->nh > 0) CUDA_OK(cudaMemsetAsync(x2 + c->nl * H, 0, sizeof(float) * (size_t)(c->nh * H), c->stream));
    if (use_tc(c)) {
      launch_tc_forward(c, kNodeInput, m, c->nl, x, nullptr, a, x2);
    } else {
      MlpRowArgs args{};
      args.n_rows = c->nl;
      args.x = x;
      args.a = a;
      args.out = x2;
      launch_mlp(c, true, kNodeInput, args, layer_params(c, m, false));
    }
  }
}

void reduce_grads(hgnn_ctx* c, int grid, int64_t n_par, double* out) {
  Timed t(c, HGNN_K_GRAD_REDUCE);
  grad_reduce_kernel<<<blocks_for(n_par), kEwThreads, 0, c->stream>>>(c->grad_part.p, grid, n_par, out);
  check_launch(c);
}

// dx / de hold the layer-output adjoints on entry; on exit dx holds the input
// adjoint (c->dx) and de the edge input adjoint (in place).
void layer_backward(hgnn_ctx* c, int64_t m) {
  const int64_t H = c->H;
  float* x = c->xs[m]->p;
  float* e = c->es[m]->p;
  float* a = c->as[m]->p;
  const int64_t goff = m * (c->n_edge_par + c->n_node_par);
  {  // node update backward (model.cpp:326-340)
    Timed t(c, HGNN_K_NODE_BWD);
    CUDA_OK(cudaMemsetAsync(c->d_a.p, 0, sizeof(float) * (size_t)(c->rows * H), c->stream));
    if (use_tc_bwd(c)) {
      const int grid = tc_bwd_grid(c, c->nl);
      CUDA_OK(cudaMemsetAsync(c->grad_part.p, 0, sizeof(float) * (size_t)(2 * grid * c->n_node_par), c->stream));
      TcBwdArgs args{};
      args.n_rows = c->nl;
      args.x = x;
      args.a = a;
      args.d_out = c->dx.p;
      args.d_a_out = c->d_a.p;
      args.d_x_out = c->dxn.p;
      args.grad_partial = c->grad_part.p;
      if (c->nl > 0) {
        launch_tc_backward(c, kNodeInput, m, args);
        reduce_grads(c, 2 * grid, c->n_node_par, c->grads.p + goff + c->n_edge_par);
      }
    } else {
      CUDA_OK(cudaMemsetAsync(c->grad_part.p, 0, sizeof(float) * (size_t)(c->grid_node_b * c->n_node_par), c->stream));
      MlpRowArgs args{};
      args.n_rows = c->nl;
      args.x = x;
      args.a = a;
      args.d_out = c->dx.p;
      args.d_a_out = c->d_a.p;
      args.d_x_out = c->dxn.p;
      args.grad_partial = c->grad_part.p;
      args.scratch = c->scratch.p;
      args.n_slots = (2 * c->K + 1) * H + c->K;
      launch_mlp(c, false, kNodeInput, args, layer_params(c, m, false));
      if (c->nl > 0) reduce_grads(c, c->grid_node_b, c->n_node_par, c->grads.p + goff + c->n_edge_par);
    }
  }
  if (c->mode != HGNN_MODE_NONE) {  // sync + exchange adjoints (model.cpp:343-351)
    if (c->n_sync > 0) {
      Timed t(c, HGNN_K_HALO);
      sync_adjoint_kernel<<<blocks_for(c->n_sync * H / 4), kEwThreads, 0, c->stream>>>(
          c->d_a.p, c->sync_local.p, c->sync_off.p, c->sync_slots.p, c->n_sync, (int)H);
      check_launch(c);
    }
    halo_exchange_adjoint(c, c->d_a.p);
  }
  {  // aggregation + edge update backward (model.cpp:353-375)
    Timed t(c, HGNN_K_EDGE_BWD);
    if (use_tc_bwd(c)) {
      const int grid = tc_bwd_grid(c, c->ne);
      CUDA_OK(cudaMemsetAsync(c->grad_part.p, 0, sizeof(float) * (size_t)(2 * grid * c->n_edge_par), c->stream));
      TcBwdArgs args{};
      args.n_rows = c->ne;
      args.src = c->src.p;
      args.dst = c->dst.p;
      args.x = x;
      args.e_in = e;
      args.inv_deg = c->inv.p;
      args.d_a = c->d_a.p;
      args.de_io = c->de.p;
      args.d_src = c->dsrc.p;
      args.d_dst = c->ddst.p;
      args.grad_partial = c->grad_part.p;
      if (c->ne > 0) {
        launch_tc_backward(c, kEdgeInput, m, args);
        reduce_grads(c, 2 * grid, c->n_edge_par, c->grads.p + goff);
      }
    } else {
      CUDA_OK(cudaMemsetAsync(c->grad_part.p, 0, sizeof(float) * (size_t)(c->grid_edge_b * c->n_edge_par), c->stream));
      MlpRowArgs args{};
      args.n_rows = c->ne;
      args.src = c->src.p;
      args.dst = c->dst.p;
      args.x = x;
      args.e_in = e;
      args.inv_deg = c->inv.p;
      args.d_a = c->d_a.p;
      args.de_io = c->de.p;
      args.d_src = c->dsrc.p;
      args.d_dst = c->ddst.p;
      args.grad_partial = c->grad_part.p;
      args.scratch = c->scratch.p;
      args.n_slots = (2 * c->K + 1) * H + c->K;
      launch_mlp(c, false, kEdgeInput, args, layer_params(c, m, true));
      if (c->ne > 0) reduce_grads(c, c->grid_edge_b, c->n_edge_par, c->grads.p + goff);
    }
  }
  {  // input-node adjoint (model.cpp:378-386)
    Timed t(c, HGNN_K_DX);
    dx_gather_kernel<<<blocks_for(c->rows * H / 4), kEwThreads, 0, c->stream>>>(
        c->dsrc.p, c->ddst.p, c->dxn.p, c->in_off.p, c->twin.p, c->rows, c->nl, (int)H, c->dx.p);
    check_launch(c);
  }
}

void run_forward(hgnn_ctx* c) {
  for (int64_t m = 0; m < c->M; ++m) layer_forward(c, m);
  c->forward_done = true;
}

void run_backward(hgnn_ctx* c) {
  if (!c->forward_done) fail(HGNN_ERR_UNINITIALIZED, "hgnn_mp_backward called before hgnn_mp_forward");
  if (c->M == 0) return;
  CUDA_OK(cudaMemsetAsync(c->grads.p, 0, sizeof(double) * (size_t)c->n_mp_par, c->stream));
  for (int64_t m = c->M - 1; m >= 0; --m) layer_backward(c, m);
}

void require_ready(hgnn_ctx* c) {
  if (!c->configured) fail(HGNN_ERR_UNINITIALIZED, "hgnn_configure has not been called");
  if (!c->graph_ready) fail(HGNN_ERR_UNINITIALIZED, "hgnn_graph_upload has not been called");
  if (!c->params_ready) fail(HGNN_ERR_UNINITIALIZED, "hgnn_params_upload has not been called");
  if (c->mode != HGNN_MODE_NONE && c->nranks > 1 && !c->comm)
    fail(HGNN_ERR_CONFIG, "nmp_layer: exchange mode requires a rank runtime");
}

}  // namespace


// ==========================================================================
// model level: encoders + MP stack + decoder, consistent loss, gradient
// averaging, Adam (model.cpp:289-307, 390-424, 455-579,
// nn.cpp:331-360)
// ==========================================================================
namespace {

bool gen_supported(int64_t fx, int64_t fe, int64_t fy) { return fx == 3 && fe == 7 && fy == 3; }

template <int IN, int OUT, bool SKIP, bool LN>
void gen_forward(hgnn_ctx* c, int64_t n_rows, const float* in, float* out, int64_t par_off, int64_t n_par) {
  if (n_rows == 0) return;
  GenArgs a{};
  a.n_rows = n_rows;
  a.in = in;
  a.out = out;
  a.params = c->gen_par.p + par_off;
  a.k = (int)c->K;
  a.n_par = n_par;
  auto k = gen_mlp_forward_kernel<IN, OUT, SKIP, LN>;
  const size_t smem = (size_t)n_par * 4;
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t tiles = (n_rows + kGenThreads - 1) / kGenThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 2 * (int64_t)c->num_sms));
  k<<<grid, kGenThreads, smem, c->stream>>>(a);
  check_launch(c);
}

// Backward of one encoder / decoder MLP; parameter gradients (rank-local)
// land in mgrads[par_off, par_off + n_par).
template <int IN, int OUT, bool SKIP, bool LN, bool DIN>
void gen_backward(hgnn_ctx* c, int64_t n_rows, const float* in, const float* d_out, float* d_in, int64_t par_off,
                  int64_t n_par) {
  if (n_rows == 0) {
    CUDA_OK(cudaMemsetAsync(c->mgrads.p + par_off, 0, sizeof(double) * (size_t)n_par, c->stream));
    return;
  }
  const int64_t tiles = (n_rows + kGenThreads - 1) / kGenThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 2 * (int64_t)c->num_sms));  // 2 CTAs / SM
  const int64_t slots = gen_scratch_slots((int)c->K, OUT);
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
  auto k = gen_mlp_backward_kernel<IN, OUT, SKIP, LN, DIN>;
  const size_t smem = gen_backward_smem(IN, OUT);
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<grid, kGenThreads, smem, c->stream>>>(a);
  check_launch(c);
  reduce_partials_kernel<<<blocks_for(n_par), kEwThreads, 0, c->stream>>>(c->gen_part.p, grid, n_par,
                                                                          c->mgrads.p + par_off);
  check_launch(c);
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
    gen_forward<3, 64, true, true>(c, c->rows, c->node_feat.p, c->xs[0]->p, c->off_ne, c->n_ne);
    gen_forward<7, 64, true, true>(c, c->ne, c->edge_feat.p, c->es[0]->p, c->off_ee, c->n_ee);
  }
  // message passing (model.cpp:295-300)
  run_forward(c);
  // decoder on local rows (model.cpp:303-306)
  c->y.alloc(std::max<int64_t>(nl * c->fy, 1));
  c->dy.alloc(std::max<int64_t>(nl * c->fy, 1));
  {
    Timed t(c, HGNN_K_DECODE);
    gen_forward<64, 3, true, false>(c, nl, c->xs[(size_t)c->M]->p, c->y.p, c->off_dec, c->n_dec);
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
  if (c->nranks > 1) NCCL_OK(ncclAllReduce(c->loss_st.p, c->loss_st.p, 2, ncclDouble, ncclSum, c->comm, c->stream));
  loss_seed_kernel<<<1, 32, 0, c->stream>>>(c->loss_st.p, (int)c->fy, c->nranks);
  check_launch(c);
  loss_backward_kernel<<<blocks_for(nl * c->fy), kEwThreads, 0, c->stream>>>(
      c->y.p, c->target.p, c->node_inv.p, c->loss_st.p + 2, nl, (int)c->fy, c->dy.p);
  check_launch(c);
  t_loss.stop();
  {  // decoder backward (model.cpp:402-409): adjoint of x_M on local rows, halo rows 0
    Timed t(c, HGNN_K_DECODE);
    CUDA_OK(cudaMemsetAsync(c->dx.p, 0, sizeof(float) * (size_t)(c->rows * H), c->stream));
    gen_backward<64, 3, true, false, true>(c, nl, c->xs[(size_t)c->M]->p, c->dy.p, c->dx.p, c->off_dec, c->n_dec);
  }
  // message-passing backward (model.cpp:411-415), de_M = 0 (model.cpp:412)
  CUDA_OK(cudaMemsetAsync(c->de.p, 0, sizeof(float) * (size_t)(c->ne * H), c->stream));
  run_backward(c);
  CUDA_OK(cudaMemcpyAsync(c->mgrads.p + c->off_mp, c->grads.p, sizeof(double) * (size_t)c->n_mp_par,
                          cudaMemcpyDeviceToDevice, c->stream));
  {  // encoder backward (model.cpp:417-423)
    Timed t(c, HGNN_K_ENCODE);
    gen_backward<3, 64, true, true, false>(c, c->rows, c->node_feat.p, c->dx.p, nullptr, c->off_ne, c->n_ne);
    gen_backward<7, 64, true, true, false>(c, c->ne, c->edge_feat.p, c->de.p, nullptr, c->off_ee, c->n_ee);
  }
  // average over ranks (model.cpp:516-531)
  if (c->nranks > 1) {
    NCCL_OK(ncclAllReduce(c->mgrads.p, c->mgrads.p, (size_t)c->n_full, ncclDouble, ncclSum, c->comm, c->stream));
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
      if (tc_eligible(c)) {
        const int64_t base = (int64_t)ch.size();
        ch.resize((size_t)(base + chunk_floats_fwd(in_dim, H, K)));
        chunk_layout_fwd(in_dim, H, K, base, [&](int64_t pos, int64_t src, bool lo) {
          ch[(size_t)pos] = (uint32_t)(off + src) | (lo ? 0x80000000u : 0u);
        });
      }
      if (H == 64) {
        const int64_t base = (int64_t)bch.size();
        bch.resize((size_t)(base + chunk_floats_bwd(in_dim, H, K)));
        chunk_layout_bwd(in_dim, H, K, base, [&](int64_t pos, int64_t src, bool lo) {
          bch[(size_t)pos] = (uint32_t)(off + src) | (lo ? 0x80000000u : 0u);
        });
      }
      off += mlp_param_count(in_dim, H, K);
    }
  c->pt_src.upload(pt.data(), (int64_t)pt.size(), c->stream);
  c->ch_map.upload(ch.data(), (int64_t)ch.size(), c->stream);
  c->bch_map.upload(bch.data(), (int64_t)bch.size(), c->stream);
}

}  // namespace

// ==========================================================================
// C-ABI
// ==========================================================================
extern "C" {

int hgnn_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int hgnn_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
    ncclUniqueId id;
    NCCL_OK(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

int hgnn_ctx_create(int device, int32_t rank, int32_t nranks, const uint8_t* uid, hgnn_ctx** out) {
  return guarded([&] {
    if (!out) fail(HGNN_ERR_CONFIG, "hgnn_ctx_create: null output");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(HGNN_ERR_CONFIG, "hgnn_ctx_create: bad rank/nranks");
    int ndev = 0;
    CUDA_OK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) fail(HGNN_ERR_CUDA, "hgnn_ctx_create: no such CUDA device");
    auto c = std::make_unique<hgnn_ctx>();
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    CUDA_OK(cudaSetDevice(device));
    int major = 0;
    CUDA_OK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10) fail(HGNN_ERR_CUDA, "this build targets sm_100a (B200); found compute capability major " +
                                             std::to_string(major));
    CUDA_OK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    if (nranks > 1) {
      if (!uid) fail(HGNN_ERR_CONFIG, "hgnn_ctx_create: nccl unique id required for num_ranks > 1");
      ncclUniqueId id;
      std::memcpy(&id, uid, sizeof(id));
      NCCL_OK(ncclCommInitRank(&c->comm, nranks, id, rank));
    }
    *out = c.release();
  });
}

int hgnn_ctx_destroy(hgnn_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& v : c->ev)
      for (auto& p : v) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
      }
    if (c->comm) ncclCommDestroy(c->comm);
    cudaStreamDestroy(c->stream);
    delete c;
  });
}

void* hgnn_ctx_stream(hgnn_ctx* c) { return c ? (void*)c->stream : nullptr; }

int hgnn_graph_upload(hgnn_ctx* c, const hgnn_graph_desc* g) {
  return guarded([&] {
    bind(c);
    if (!g) fail(HGNN_ERR_CONFIG, "hgnn_graph_upload: null graph");
    if (g->rank != c->rank || g->num_ranks != c->nranks)
      fail(HGNN_ERR_INTEGRITY, "hgnn_graph_upload: graph rank/num_ranks do not match the context");
    const int64_t nl = g->num_local, nh = g->num_halo, ne = g->num_edges, rows = nl + nh;
    if (nl < 0 || nh < 0 || ne < 0 || rows >= INT32_MAX || ne >= INT32_MAX)
      fail(HGNN_ERR_SHAPE, "hgnn_graph_upload: sizes out of range");
    if (ne % 2) fail(HGNN_ERR_INTEGRITY, "directed edges must come in twin pairs (graph.cpp:107-110)");
    // receiver-sorted slots = in-CSR order; twin slots via the e^1 pairing
    std::vector<int32_t> slot_of((size_t)ne), src_s((size_t)ne), dst_s((size_t)ne), twin((size_t)ne);
    std::vector<float> inv_s((size_t)ne);
    if (g->in_offsets[0] != 0 || g->in_offsets[rows] != ne) fail(HGNN_ERR_INTEGRITY, "in_offsets do not span N_e");
    for (int64_t i = 0; i < rows; ++i)
      for (int32_t p = g->in_offsets[i]; p < g->in_offsets[i + 1]; ++p) {
        const int32_t e = g->in_edges[p];
        if (e < 0 || e >= ne || g->edge_dst[e] != i) fail(HGNN_ERR_INTEGRITY, "in-CSR inconsistent with edge_dst");
        slot_of[(size_t)e] = p;
      }
    for (int64_t p = 0; p < ne; ++p) {
      const int32_t e = g->in_edges[p];
      const int32_t s = g->edge_src[e], d = g->edge_dst[e];
      if (s < 0 || s >= nl || d < 0 || d >= nl) fail(HGNN_ERR_INTEGRITY, "edges must not reference halo rows");
      const int32_t t = e ^ 1;
      if (g->edge_src[t] != d || g->edge_dst[t] != s) fail(HGNN_ERR_INTEGRITY, "edge e^1 is not the twin of e");
      src_s[(size_t)p] = s;
      dst_s[(size_t)p] = d;
      inv_s[(size_t)p] = (float)g->edge_inv_degree[e];
      twin[(size_t)p] = slot_of[(size_t)t];
    }
    c->nl = nl;
    c->nh = nh;
    c->rows = rows;
    c->ne = ne;
    c->max_buffer_rows = g->max_buffer_rows;
    c->src.upload(src_s.data(), ne, c->stream);
    c->dst.upload(dst_s.data(), ne, c->stream);
    c->twin.upload(twin.data(), ne, c->stream);
    c->slot_of.upload(slot_of.data(), ne, c->stream);
    c->inv.upload(inv_s.data(), ne, c->stream);
    if (g->node_inv_degree) c->node_inv.upload(g->node_inv_degree, nl, c->stream);
    c->in_off.upload(g->in_offsets, rows + 1, c->stream);
    std::vector<int64_t> gids(g->global_ids, g->global_ids + rows);
    c->gid.upload(gids.data(), rows, c->stream);
    // halo map
    const int nn = g->num_neighbors;
    c->h_nbr.assign(g->neighbors, g->neighbors + nn);
    c->h_send_off.assign(g->send_offsets, g->send_offsets + nn + 1);
    c->h_recv_off.assign(g->recv_offsets, g->recv_offsets + nn + 1);
    c->h_recv_base.assign((size_t)nn, 0);
    c->n_send = nn ? c->h_send_off[(size_t)nn] : 0;
    c->n_recv = nn ? c->h_recv_off[(size_t)nn] : 0;
    if (c->n_recv != nh) fail(HGNN_ERR_INTEGRITY, "recv masks must cover exactly the halo rows");
    for (int n = 0; n < nn; ++n) {
      if (g->neighbors[n] < 0 || g->neighbors[n] >= c->nranks || g->neighbors[n] == c->rank ||
          (n > 0 && g->neighbors[n] <= g->neighbors[n - 1]))
        fail(HGNN_ERR_INTEGRITY, "neighbors must be ascending peer ranks");
      const int64_t base = g->recv_rows[c->h_recv_off[(size_t)n]];
      c->h_recv_base[(size_t)n] = base;
      for (int32_t t = c->h_recv_off[(size_t)n]; t < c->h_recv_off[(size_t)n + 1]; ++t)
        if (g->recv_rows[t] != base + (t - c->h_recv_off[(size_t)n]))
          fail(HGNN_ERR_INTEGRITY, "recv rows of a neighbour must be one consecutive block (graph.cpp:184-201)");
      if (c->h_send_off[(size_t)n + 1] - c->h_send_off[(size_t)n] > g->max_buffer_rows)
        fail(HGNN_ERR_INTEGRITY, "send mask longer than max_buffer_rows");
    }
    c->send_rows.upload(g->send_rows, c->n_send, c->stream);
    c->recv_rows.upload(g->recv_rows, c->n_recv, c->stream);
    // A2A padded positions: peer d's block starts at d * max_buffer_rows
    std::vector<int64_t> a2a_send((size_t)c->n_send), a2a_recv((size_t)c->n_recv);
    for (int n = 0; n < nn; ++n) {
      for (int32_t t = c->h_send_off[(size_t)n]; t < c->h_send_off[(size_t)n + 1]; ++t)
        a2a_send[(size_t)t] = (int64_t)g->neighbors[n] * g->max_buffer_rows + (t - c->h_send_off[(size_t)n]);
      for (int32_t t = c->h_recv_off[(size_t)n]; t < c->h_recv_off[(size_t)n + 1]; ++t)
        a2a_recv[(size_t)t] = (int64_t)g->neighbors[n] * g->max_buffer_rows + (t - c->h_recv_off[(size_t)n]);
    }
    c->pos_a2a_send.upload(a2a_send.data(), c->n_send, c->stream);
    c->pos_a2a_recv.upload(a2a_recv.data(), c->n_recv, c->stream);
    // exchange-adjoint accumulation lists: per local row, positions in
    // ascending neighbour order (comm.cpp:344-356)
    std::vector<std::vector<int32_t>> lists((size_t)nl);
    for (int n = 0; n < nn; ++n)
      for (int32_t t = c->h_send_off[(size_t)n]; t < c->h_send_off[(size_t)n + 1]; ++t) {
        const int32_t r = g->send_rows[t];
        if (r < 0 || r >= nl) fail(HGNN_ERR_INTEGRITY, "send rows must be local rows");
        lists[(size_t)r].push_back(t);
      }
    std::vector<int32_t> acc_rows, acc_off{0};
    std::vector<int64_t> pos_n, pos_a;
    for (int64_t r = 0; r < nl; ++r) {
      if (lists[(size_t)r].empty()) continue;
      acc_rows.push_back((int32_t)r);
      for (int32_t t : lists[(size_t)r]) {
        pos_n.push_back(t);
        pos_a.push_back(a2a_send[(size_t)t]);
      }
      acc_off.push_back((int32_t)pos_n.size());
    }
    c->n_acc = (int64_t)acc_rows.size();
    c->acc_rows.upload(acc_rows.data(), c->n_acc, c->stream);
    c->acc_off.upload(acc_off.data(), (int64_t)acc_off.size(), c->stream);
    c->acc_pos_na2a.upload(pos_n.data(), (int64_t)pos_n.size(), c->stream);
    c->acc_pos_a2a.upload(pos_a.data(), (int64_t)pos_a.size(), c->stream);
    // sync groups
    c->n_sync = g->num_sync_groups;
    c->sync_local.upload(g->sync_local, c->n_sync, c->stream);
    c->sync_off.upload(g->sync_offsets, c->n_sync + 1, c->stream);
    c->sync_slots.upload(g->sync_slots, c->n_sync ? g->sync_offsets[c->n_sync] : 0, c->stream);
    CUDA_OK(cudaStreamSynchronize(c->stream));
    c->graph_ready = true;
    c->forward_done = false;
    c->xs.clear();
    c->es.clear();
    c->as.clear();
  });
}

int hgnn_configure(hgnn_ctx* c, int64_t hidden, int64_t M, int64_t k, int mode) {
  return guarded([&] {
    bind(c);
    if (hidden != 8 && hidden != 16 && hidden != 32 && hidden != 64)
      fail(HGNN_ERR_CONFIG, "hidden_dim must be one of 8, 16, 32, 64 on this build");
    if (M < 0) fail(HGNN_ERR_CONFIG, "GnnConfig: num_mp_layers must be >= 0");
    if (k < 0 || k > 16) fail(HGNN_ERR_CONFIG, "GnnConfig: mlp_hidden_layers must be in [0, 16]");
    if (mode < HGNN_MODE_NONE || mode > HGNN_MODE_NA2A) fail(HGNN_ERR_CONFIG, "unknown exchange mode");
    if (mode != HGNN_MODE_NONE && c->nranks > 1 && !c->comm)
      fail(HGNN_ERR_CONFIG, "nmp_layer: exchange mode requires a rank runtime");
    if (c->H != hidden || c->M != M || c->K != k) {
      c->params_ready = false;
      c->xs.clear();
      c->es.clear();
      c->as.clear();
    }
    c->H = hidden;
    c->M = M;
    c->K = k;
    c->mode = mode;
    c->n_edge_par = mlp_param_count((int)(3 * hidden), (int)hidden, (int)k);
    c->n_node_par = mlp_param_count((int)(2 * hidden), (int)hidden, (int)k);
    c->n_mp_par = M * (c->n_edge_par + c->n_node_par);
    c->configured = true;
    c->forward_done = false;
  });
}

int hgnn_params_upload(hgnn_ctx* c, const double* flat, int64_t count) {
  return guarded([&] {
    bind(c);
    if (!c->configured) fail(HGNN_ERR_UNINITIALIZED, "hgnn_configure has not been called");
    if (count != c->n_mp_par)
      fail(HGNN_ERR_SHAPE, "hgnn_params_upload: expected " + std::to_string(c->n_mp_par) + " values, got " +
                               std::to_string(count));
    std::vector<float> p((size_t)count), pt((size_t)count);
    for (int64_t i = 0; i < count; ++i) p[(size_t)i] = (float)flat[i];
    // transposed copy of every weight (out x in) for the adjoint products
    const int H = (int)c->H, K = (int)c->K;
    int64_t off = 0;
    for (int64_t m = 0; m < c->M; ++m)
      for (int which = 0; which < 2; ++which) {
        const int in_dim = (which == 0 ? 3 : 2) * H;
        for (int l = 0; l < K + 2; ++l) {
          const int rin = l == 0 ? in_dim : H;
          const int64_t wo = off + mlp_w_offset(l, in_dim, H), bo = off + mlp_b_offset(l, in_dim, H);
          for (int i = 0; i < rin; ++i)
            for (int j = 0; j < H; ++j) pt[(size_t)(wo + (int64_t)j * rin + i)] = p[(size_t)(wo + (int64_t)i * H + j)];
          for (int j = 0; j < H; ++j) pt[(size_t)(bo + j)] = p[(size_t)(bo + j)];
        }
        off += mlp_param_count(in_dim, H, K);
      }
    c->par.upload(p.data(), count, c->stream);
    c->par_t.upload(pt.data(), count, c->stream);
    if (tc_eligible(c)) {
      std::vector<float> ch;
      c->chunk_off.clear();
      int64_t poff = 0;
      for (int64_t m = 0; m < c->M; ++m)
        for (int which = 0; which < 2; ++which) {
          const int in_dim = (which == 0 ? 3 : 2) * H;
          c->chunk_off.push_back((int64_t)ch.size());
          build_chunks(p.data() + poff, in_dim, H, K, ch);
          poff += mlp_param_count(in_dim, H, K);
        }
      c->chunks.upload(ch.data(), (int64_t)ch.size(), c->stream);
    }
    if (H == 64) {
      std::vector<float> ch;
      c->bchunk_off.clear();
      int64_t poff = 0;
      for (int64_t m = 0; m < c->M; ++m)
        for (int which = 0; which < 2; ++which) {
          const int in_dim = (which == 0 ? 3 : 2) * H;
          c->bchunk_off.push_back((int64_t)ch.size());
          build_bwd_chunks(p.data() + poff, in_dim, H, K, ch);
          poff += mlp_param_count(in_dim, H, K);
        }
      c->bchunks.upload(ch.data(), (int64_t)ch.size(), c->stream);
    }
    c->grads.alloc(std::max<int64_t>(count, 1));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    c->params_ready = true;
  });
}

int hgnn_mp_forward(hgnn_ctx* c, const double* x0, const double* e0, double* x_out, double* e_out) {
  return guarded([&] {
    bind(c);
    require_ready(c);
    if (!x0 || !e0) fail(HGNN_ERR_SHAPE, "hgnn_mp_forward: null input");
    ensure_buffers(c);
    rows_to_device(c, x0, c->rows * c->H, c->xs[0]->p);
    edges_to_device(c, e0, c->es[0]->p);
    run_forward(c);
    if (x_out) rows_to_host(c, c->xs[(size_t)c->M]->p, c->rows * c->H, x_out);
    if (e_out) edges_to_host(c, c->es[(size_t)c->M]->p, e_out);
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
}

int hgnn_mp_backward(hgnn_ctx* c, const double* dx, const double* de, double* dx0, double* de0, double* grads) {
  return guarded([&] {
    bind(c);
    require_ready(c);
    if (!dx) fail(HGNN_ERR_SHAPE, "hgnn_mp_backward: null output adjoint");
    ensure_buffers(c);
    rows_to_device(c, dx, c->rows * c->H, c->dx.p);
    if (de) edges_to_device(c, de, c->de.p);
    else CUDA_OK(cudaMemsetAsync(c->de.p, 0, sizeof(float) * (size_t)(c->ne * c->H), c->stream));
    run_backward(c);
    if (dx0) rows_to_host(c, c->dx.p, c->rows * c->H, dx0);
    if (de0) edges_to_host(c, c->de.p, de0);
    if (grads) {
      CUDA_OK(cudaMemcpyAsync(grads, c->grads.p, sizeof(double) * (size_t)c->n_mp_par, cudaMemcpyDeviceToHost,
                              c->stream));
    }
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
}

int hgnn_get_trace(hgnn_ctx* c, int layer, int which, double* out) {
  return guarded([&] {
    bind(c);
    if (!c->forward_done) fail(HGNN_ERR_UNINITIALIZED, "no forward trace available");
    if (layer < 0 || layer >= c->M) fail(HGNN_ERR_SHAPE, "trace layer out of range");
    switch (which) {
      case HGNN_TRACE_X_IN: rows_to_host(c, c->xs[(size_t)layer]->p, c->rows * c->H, out); break;
      case HGNN_TRACE_E_IN: edges_to_host(c, c->es[(size_t)layer]->p, out); break;
      case HGNN_TRACE_A_SYNC: rows_to_host(c, c->as[(size_t)layer]->p, c->rows * c->H, out); break;
      case HGNN_TRACE_X_OUT: rows_to_host(c, c->xs[(size_t)layer + 1]->p, c->rows * c->H, out); break;
      case HGNN_TRACE_E_OUT: edges_to_host(c, c->es[(size_t)layer + 1]->p, out); break;
      default: fail(HGNN_ERR_CONFIG, "unknown trace selector");
    }
  });
}

int hgnn_synthetic_inputs(hgnn_ctx* c, uint64_t seed) {
  return guarded([&] {
    bind(c);
    require_ready(c);
    ensure_buffers(c);
    const int64_t H = c->H;
    synth_rows_kernel<<<blocks_for(c->rows * H), kEwThreads, 0, c->stream>>>(c->gid.p, c->rows, c->nl, (int)H, seed,
                                                                            1.0f, c->xs[0]->p);
    check_launch(c);
    if (c->ne > 0) {
      synth_edges_kernel<<<blocks_for(c->ne * H), kEwThreads, 0, c->stream>>>(c->gid.p, c->src.p, c->dst.p, c->ne,
                                                                             (int)H, seed ^ 0x5bd1e995ull, c->es[0]->p);
      check_launch(c);
    }
    synth_rows_kernel<<<blocks_for(c->rows * H), kEwThreads, 0, c->stream>>>(c->gid.p, c->rows, c->nl, (int)H,
                                                                            seed ^ 0xc2b2ae35ull, 1e-3f, c->dx_in.p);
    check_launch(c);
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
}

int hgnn_set_inputs(hgnn_ctx* c, const double* x0, const double* e0, const double* dx) {
  return guarded([&] {
    bind(c);
    require_ready(c);
    ensure_buffers(c);
    rows_to_device(c, x0, c->rows * c->H, c->xs[0]->p);
    edges_to_device(c, e0, c->es[0]->p);
    rows_to_device(c, dx, c->rows * c->H, c->dx_in.p);
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
}

int hgnn_mp_step_device(hgnn_ctx* c) {
  return guarded([&] {
    bind(c);
    require_ready(c);
    ensure_buffers(c);
    run_forward(c);
    CUDA_OK(cudaMemcpyAsync(c->dx.p, c->dx_in.p, sizeof(float) * (size_t)(c->rows * c->H), cudaMemcpyDeviceToDevice,
                            c->stream));
    CUDA_OK(cudaMemsetAsync(c->de.p, 0, sizeof(float) * (size_t)(c->ne * c->H), c->stream));
    run_backward(c);
  });
}

int hgnn_get_grads(hgnn_ctx* c, double* out) {
  return guarded([&] {
    bind(c);
    if (!c->params_ready) fail(HGNN_ERR_UNINITIALIZED, "no parameters");
    CUDA_OK(cudaMemcpyAsync(out, c->grads.p, sizeof(double) * (size_t)c->n_mp_par, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
}

int hgnn_set_option(hgnn_ctx* c, const char* key, int64_t value) {
  return guarded([&] {
    bind(c);
    const std::string k = key ? key : "";
    if (k == "mlp_forward_impl") {
      if (value != 0 && value != 1) fail(HGNN_ERR_CONFIG, "mlp_forward_impl: 0 (simt) or 1 (tcgen05)");
      c->fwd_impl = (int)value;
    } else if (k == "bwd_profile") {
      c->prof.alloc(4 * kProfCount);
      CUDA_OK(cudaMemsetAsync(c->prof.p, 0, sizeof(unsigned long long) * 4 * kProfCount, c->stream));
      c->prof_on = value != 0;
    } else if (k == "mlp_backward_impl") {
      if (value != 0 && value != 1) fail(HGNN_ERR_CONFIG, "mlp_backward_impl: 0 (simt) or 1 (tcgen05)");
      c->bwd_impl = (int)value;
    } else {
      fail(HGNN_ERR_CONFIG, "unknown option '" + k + "'");
    }
  });
}

int hgnn_kernel_timing(hgnn_ctx* c, int enable) {
  return guarded([&] {
    bind(c);
    CUDA_OK(cudaStreamSynchronize(c->stream));
    c->timing = enable != 0;
    for (auto& u : c->ev_used) u = 0;
  });
}

int hgnn_kernel_time(hgnn_ctx* c, int cls, double* total_ms, int64_t* launches) {
  return guarded([&] {
    bind(c);
    if (cls < 0 || cls >= HGNN_K_COUNT) fail(HGNN_ERR_CONFIG, "unknown kernel class");
    CUDA_OK(cudaStreamSynchronize(c->stream));
    double t = 0.0;
    for (size_t i = 0; i < c->ev_used[cls]; ++i) {
      float ms = 0.f;
      CUDA_OK(cudaEventElapsedTime(&ms, c->ev[cls][i].a, c->ev[cls][i].b));
      t += ms;
    }
    *total_ms = t;
    *launches = (int64_t)c->ev_used[cls];
  });
}

int hgnn_debug_profile(hgnn_ctx* c, uint64_t* out64) {
  return guarded([&] {
    bind(c);
    if (!c->prof.p) fail(HGNN_ERR_UNINITIALIZED, "bwd_profile not enabled");
    CUDA_OK(cudaMemcpy(out64, c->prof.p, sizeof(unsigned long long) * 4 * kProfCount, cudaMemcpyDeviceToHost));
  });
}

int64_t hgnn_launch_count(hgnn_ctx* c, int reset) {
  if (!c) return -1;
  const int64_t n = c->launches;
  if (reset) c->launches = 0;
  return n;
}

int64_t hgnn_halo_bytes(hgnn_ctx* c, int reset) {
  if (!c) return -1;
  const int64_t n = c->halo_bytes;
  if (reset) c->halo_bytes = 0;
  return n;
}

// ---- model level ----------------------------------------
int hgnn_model_configure(hgnn_ctx* c, int64_t in_node_dim, int64_t in_edge_dim, int64_t out_dim) {
  return guarded([&] {
    bind(c);
    if (!c->configured) fail(HGNN_ERR_UNINITIALIZED, "hgnn_configure has not been called");
    if (c->H != kGenH) fail(HGNN_ERR_CONFIG, "model level: hidden width 64 only");
    if (!gen_supported(in_node_dim, in_edge_dim, out_dim))
      fail(HGNN_ERR_CONFIG, "model level: feature widths (F_x, F_e, F_y) = (3, 7, 3) supported");
    c->fx = in_node_dim;
    c->fe = in_edge_dim;
    c->fy = out_dim;
    const int K = (int)c->K;
    c->n_ne = gen_param_count((int)c->fx, kGenH, K, true, true);
    c->n_ee = gen_param_count((int)c->fe, kGenH, K, true, true);
    c->n_dec = gen_param_count(kGenH, (int)c->fy, K, true, false);
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
    const int64_t per = std::max<int64_t>(1, c->stage_elems / c->fe);
    for (int64_t e0 = 0; e0 < c->ne; e0 += per) {  // reference edge-id order -> receiver-sorted slots
      const int64_t m = std::min(per, c->ne - e0);
      CUDA_OK(cudaMemcpyAsync(c->stage.p, edge_features + e0 * c->fe, sizeof(double) * (size_t)(m * c->fe),
                              cudaMemcpyHostToDevice, c->stream));
      edges_in_kernel<<<blocks_for(m * c->fe), kEwThreads, 0, c->stream>>>(c->stage.p, c->slot_of.p, e0, m,
                                                                          (int)c->fe, c->edge_feat.p);
      check_launch(c);
    }
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
    c->adam_step += 1;
    const double bc1 = 1.0 - std::pow(beta1, (double)c->adam_step);
    const double bc2 = 1.0 - std::pow(beta2, (double)c->adam_step);
    Timed t(c, HGNN_K_LOSS_ADAM);
    CUDA_OK(cudaMemsetAsync(c->nonfinite.p, 0, sizeof(int), c->stream));
    adam_kernel<<<blocks_for(c->n_full), kEwThreads, 0, c->stream>>>(c->mparams.p, c->mgrads.p, c->adam_m.p,
                                                                     c->adam_v.p, c->n_full, lr, beta1, beta2, eps,
                                                                     bc1, bc2, c->nonfinite.p);
    check_launch(c);
    int bad = 0;
    CUDA_OK(cudaMemcpyAsync(&bad, c->nonfinite.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    if (bad) fail(HGNN_ERR_OPTIMIZER, "adam_step: non-finite gradient");
    model_refresh_params(c);
    t.stop();
    CUDA_OK(cudaStreamSynchronize(c->stream));
    if (loss) *loss = c->last_loss;
  });
}

}  // extern "C"
