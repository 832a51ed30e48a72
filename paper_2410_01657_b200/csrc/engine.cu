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
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include "edge_fact.cuh"
#include "engine_ctx.hpp"
#include "graph_kernels.cuh"
#include "mlp_simt.cuh"
#include "mlp_tc.cuh"
#include "mlp_tc_bwd.cuh"

using namespace hgnn_b200;
using namespace hgnn_b200::engine;


namespace hgnn_b200::engine {

void bind(hgnn_ctx* c) {
  if (!c) fail(HGNN_ERR_CONFIG, "null hgnn_ctx");
  CUDA_OK(cudaSetDevice(c->device));
}


// Waits for the stream with a deadline; on expiry aborts the communicator so
// the stuck NCCL kernels end, and raises CollectiveError (instead of hanging).
void nccl_wait_or_abort(hgnn_ctx* c, cudaStream_t st, const char* what) {
  cudaEvent_t ev;
  CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_OK(cudaEventRecord(ev, st));
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t q;
  while ((q = cudaEventQuery(ev)) == cudaErrorNotReady) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(c->coll_timeout_ms)) {
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      c->comm_aborted = true;
      cudaEventDestroy(ev);
      fail(HGNN_ERR_COLLECTIVE, std::string("collective aborted: ") + what + " did not complete within " +
                                    std::to_string(c->coll_timeout_ms) + " ms (a rank is missing or out of sequence)");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  cudaEventDestroy(ev);
  if (q != cudaSuccess) CUDA_OK(q);
}

// Debug guard (option "collective_check"): before every collective each rank
// all-gathers (kind, mode, count, sequence number); any difference raises
// CollectiveError on every rank — the reference's poisoning of mismatched
// collective sequences (comm.cpp:184-188) — and a rank that never arrives
// times out into ncclCommAbort.
void nccl_check_sequence(hgnn_ctx* c, int kind, int64_t count) {
  if (!c->coll_check || !c->comm) {
    if (c->comm_aborted) fail(HGNN_ERR_COLLECTIVE, "collective aborted: the communicator was aborted");
    return;
  }
  const int R = c->nranks;
  c->coll_sig.alloc(4 * (int64_t)(R + 1));
  const int32_t mine[4] = {kind, c->mode, (int32_t)count, (int32_t)c->coll_seq++};
  CUDA_OK(cudaMemcpyAsync(c->coll_sig.p, mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream));
  NCCL_OK(ncclAllGather(c->coll_sig.p, c->coll_sig.p + 4, 4, ncclInt32, c->comm, c->stream));
  nccl_wait_or_abort(c, c->stream, "collective sequence check");
  std::vector<int32_t> all((size_t)(4 * R));
  CUDA_OK(cudaMemcpy(all.data(), c->coll_sig.p + 4, sizeof(int32_t) * all.size(), cudaMemcpyDeviceToHost));
  for (int r = 0; r < R; ++r)
    for (int q = 0; q < 4; ++q)
      if (all[(size_t)(4 * r + q)] != all[(size_t)q])
        fail(HGNN_ERR_COLLECTIVE, "collective aborted: mismatched collective sequence (rank " + std::to_string(r) +
                                      " posted kind " + std::to_string(all[(size_t)(4 * r)]) + " mode " +
                                      std::to_string(all[(size_t)(4 * r + 1)]) + " #" +
                                      std::to_string(all[(size_t)(4 * r + 3)]) + ", rank 0 kind " +
                                      std::to_string(all[0]) + " mode " + std::to_string(all[1]) + " #" +
                                      std::to_string(all[3]) + ")");
}

void allreduce_sum_f64(hgnn_ctx* c, double* d, int64_t n) {
  if (c->nranks <= 1 || n <= 0) return;
  if (c->comm || c->comm_aborted) {
    nccl_check_sequence(c, kCollAllReduce, n);
    NCCL_OK(ncclAllReduce(d, d, (size_t)n, ncclDouble, ncclSum, c->comm, c->stream));
  } else if (c->group) {
    std::vector<double> h((size_t)n);
    CUDA_OK(cudaMemcpyAsync(h.data(), d, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    c->group->allreduce_sum(c->rank, h);
    CUDA_OK(cudaMemcpyAsync(d, h.data(), sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
  } else {
    fail(HGNN_ERR_CONFIG, "all_reduce_sum: no rank runtime");
  }
}

void check_launch(hgnn_ctx* c) {
  c->launches += 1;
  CUDA_OK(cudaGetLastError());
}


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

// --------------------------------------------------------------------------
// buffers
// --------------------------------------------------------------------------
bool use_fact(const hgnn_ctx* c);
bool use_tc_bwd(const hgnn_ctx* c);

// Activation / adjoint buffers of the MP stack under the standard or the
// memory-lean plan (hgnn_ctx::lean). Per rank, node = rows x H, edge = N_e x H
// fp32 tensors:
//   standard  x_0..M, a*_0..M-1, dx, dx_seed, d_a, dx_node     (2M + 5) node
//             e_0..M, de, dY (or d_src + d_dst)                 (M + 3 or 4) edge
//             node projections per layer (factorised)          2M node
//   lean      x_0..M-1 (x_M in dY), a*, dx (= dx_node), d_a    (2M + 2) node
//             e_0..M-1 (de_m over e_m), dY                      (M + 1) edge, 2 node
void ensure_buffers(hgnn_ctx* c) {
  if (!c->configured) fail(HGNN_ERR_UNINITIALIZED, "hgnn_configure has not been called");
  if (!c->graph_ready) fail(HGNN_ERR_UNINITIALIZED, "hgnn_graph_upload has not been called");
  const int64_t H = c->H, M = c->M;
  const int64_t node = c->rows * H * 4, edge = std::max<int64_t>(1, c->ne * H) * 4;
  const bool lean_ok = c->fact_ok && H == 64 && c->bwd_impl == 1 && c->fwd_impl == 1 && M > 0;
  auto release = [&] {
    c->xs.clear();
    c->es.clear();
    c->as.clear();
    c->ps.clear();
    c->dx.release();
    c->dx_in.release();
    c->d_a.release();
    c->dxn.release();
    c->de.release();
    c->dsrc.release();
    c->ddst.release();
    for (auto& v : c->plan_key) v = -1;
  };
  bool lean = c->lean_opt == 1;
  if (c->lean_opt == 1 && !lean_ok)
    fail(HGNN_ERR_CONFIG, "memory_lean needs the tcgen05 forward / backward at H = 64 (factorised edge path)");
  if (c->lean_opt == -1 && lean_ok) {
    const int64_t fact_ps = (c->edge_fact && c->fact_ok && H == 64) ? 2 * M * node : 0;
    const int64_t standard = (2 * M + 5) * node + (M + (c->edge_fact ? 3 : 4)) * edge + fact_ps;
    const bool same = c->plan_key[0] == H && c->plan_key[1] == M && c->plan_key[2] == c->rows &&
                      c->plan_key[3] == c->ne;
    if (!same) {  // (re)plan against the free device memory
      release();
      size_t free_b = 0, total_b = 0;
      CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
      lean = (double)standard > 0.94 * (double)free_b;
    } else {
      lean = c->plan_key[4] == 1;
    }
  }
  if (lean) c->edge_fact = 1;  // the lean plan has no per-edge d_x_dst / d_x_src tensors
  const bool fact = c->edge_fact && c->fact_ok && H == 64;
  const int64_t key[6] = {H, M, c->rows, c->ne, lean ? 1 : 0, fact ? 1 : 0};
  if (!std::equal(key, key + 6, c->plan_key)) {
    release();
    std::copy(key, key + 6, c->plan_key);
    c->lean = lean;
    c->forward_done = false;
    for (int64_t m = 0; m <= M; ++m) {
      if (!(lean && m == M)) {
        c->xs.emplace_back(new DevBuf<float>());
        c->xs.back()->alloc(c->rows * H);
        c->es.emplace_back(new DevBuf<float>());
        c->es.back()->alloc(std::max<int64_t>(1, c->ne * H));
      }
      if (m < M) {
        c->as.emplace_back(new DevBuf<float>());
        c->as.back()->alloc(c->rows * H);
      }
    }
    c->dx.alloc(c->rows * H);
    c->d_a.alloc(c->rows * H);
    c->dsrc.alloc(std::max<int64_t>({1, c->ne * H, lean ? c->rows * H : 0}));
    if (!lean) {
      c->dx_in.alloc(c->rows * H);
      c->dxn.alloc(std::max<int64_t>(1, c->nl * H));
      c->de.alloc(std::max<int64_t>(1, c->ne * H));
    }
    if (!(fact && c->bwd_impl == 1)) c->ddst.alloc(std::max<int64_t>(1, c->ne * H));
    for (int64_t m = 0; m < (lean ? 1 : M); ++m) {
      c->ps.emplace_back(new DevBuf<float>());
      if (fact) c->ps.back()->alloc(c->rows * 2 * H);
    }
    c->synth_valid = false;
  }
  if (c->ddst.n == 0 && !(use_fact(c) && use_tc_bwd(c))) c->ddst.alloc(std::max<int64_t>(1, c->ne * H));
  plan_mlp(c, true, kEdgeInput, c->ne, c->grid_edge_f, c->smem_edge_f, c->wsm_edge_f);
  plan_mlp(c, false, kEdgeInput, c->ne, c->grid_edge_b, c->smem_edge_b, c->wsm_edge_b);
  plan_mlp(c, true, kNodeInput, c->nl, c->grid_node_f, c->smem_node_f, c->wsm_node_f);
  plan_mlp(c, false, kNodeInput, c->nl, c->grid_node_b, c->smem_node_b, c->wsm_node_b);
  const int64_t max_grid = std::max<int64_t>({c->grid_edge_b, c->grid_node_b, (int64_t)c->num_sms});
  const int64_t max_par = std::max(c->n_edge_par, c->n_node_par);
  // tcgen05 backward: two partials per CTA; the overlapped edge backward runs two launches
  c->grad_part.alloc(2 * (max_grid + c->num_sms) * max_par);
  const int64_t n_slots = (2 * c->K + 1) * H + c->K;
  c->scratch.alloc(max_grid * n_slots * kMlpThreads);
  if (tc_eligible(c)) c->tc_scratch.alloc((int64_t)c->num_sms * 2 * std::max<int64_t>(c->K, 1) * (16 * 128 * 4 + 128));
  if (c->ps_ready.size() != (size_t)M) c->ps_ready.assign((size_t)M, 0);
  c->fact_blocks = (int)std::min<int64_t>(std::max<int64_t>(1, (c->rows + kFactRows - 1) / kFactRows),
                                          (int64_t)c->num_sms * 2);  // 112 KB shared memory: two per SM
  if (c->edge_fact && c->fact_ok && H == 64) c->fact_part.alloc((int64_t)c->fact_blocks * 2 * H * H);
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
void edges_cols_to_device(hgnn_ctx* c, const double* h, int cols, float* d) {
  const int64_t per = std::max<int64_t>(1, c->stage_elems / cols);
  for (int64_t e0 = 0; e0 < c->ne; e0 += per) {
    const int64_t m = std::min(per, c->ne - e0);
    CUDA_OK(cudaMemcpyAsync(c->stage.p, h + e0 * cols, sizeof(double) * (size_t)(m * cols), cudaMemcpyHostToDevice,
                            c->stream));
    edges_in_kernel<<<blocks_for(m * cols), kEwThreads, 0, c->stream>>>(c->stage.p, c->slot_of.p, e0, m, cols, d);
    check_launch(c);
  }
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
// ---- in-process rank group (LocalGroup): the same exchange, with the NCCL
// transfers replaced by device-to-device copies between the ranks' buffers.
// Phase 1: every rank exposes a buffer (event ev_pub) and meets its peers;
// each then pulls what the peers expose for it; phase 2: every rank records
// ev_consumed after its pulls, meets its peers again, and orders its stream
// after the peers' pulls before it may overwrite the exposed buffer.
int nbr_index(const hgnn_ctx* p, int32_t r) {
  for (size_t n = 0; n < p->h_nbr.size(); ++n)
    if (p->h_nbr[n] == r) return (int)n;
  return -1;
}

template <class Pull>
void local_exchange(hgnn_ctx* c, int kind, const float* exposed, cudaStream_t st, Pull&& pull) {
  LocalGroup& G = *c->group;
  c->xpub = exposed;
  CUDA_OK(cudaEventRecord(c->ev_pub, st));
  const CollSig sig{kind, c->mode, c->H};
  G.barrier(c->rank, sig);
  try {
    pull(G);
    CUDA_OK(cudaEventRecord(c->ev_consumed, st));
  } catch (const Error& e) {
    G.abort(std::string("rank ") + std::to_string(c->rank) + ": " + e.what());
    throw;
  }
  G.barrier(c->rank, CollSig{kCollDone, c->mode, c->H});
  for (int32_t r = 0; r < G.R; ++r)
    if (r != c->rank) CUDA_OK(cudaStreamWaitEvent(st, G.ctx[(size_t)r]->ev_consumed, 0));
}

void copy_from_peer(hgnn_ctx* c, float* dst, const hgnn_ctx* p, const float* src, int64_t n_floats,
                    cudaStream_t st) {
  if (n_floats <= 0) return;
  CUDA_OK(cudaStreamWaitEvent(st, p->ev_pub, 0));
  CUDA_OK(cudaMemcpyPeerAsync(dst, c->device, src, p->device, sizeof(float) * (size_t)n_floats, st));
}

void local_halo_exchange(hgnn_ctx* c, float* a, cudaStream_t st) {
  const int64_t H = c->H;
  const int R = c->nranks;
  if (c->mode == HGNN_MODE_NA2A) {
    if (c->n_send > 0) {
      gather_rows_kernel<<<blocks_for(c->n_send * H / 4), kEwThreads, 0, st>>>(a, c->send_rows.p, nullptr,
                                                                                     c->n_send, (int)H, c->sendbuf.p);
      check_launch(c);
    }
    local_exchange(c, kCollHaloFwd, c->sendbuf.p, st, [&](LocalGroup& G) {
      for (size_t n = 0; n < c->h_nbr.size(); ++n) {  // pull neighbour n's send block for this rank
        const hgnn_ctx* p = G.ctx[(size_t)c->h_nbr[n]];
        const int j = nbr_index(p, c->rank);
        const int64_t cr = c->h_recv_off[n + 1] - c->h_recv_off[n];
        if (j < 0 || p->h_send_off[(size_t)j + 1] - p->h_send_off[(size_t)j] != cr)
          fail(HGNN_ERR_COLLECTIVE, "halo_exchange: send / receive masks of ranks " + std::to_string(p->rank) +
                                        " and " + std::to_string(c->rank) + " do not pair");
        copy_from_peer(c, a + c->h_recv_base[n] * H, p, p->xpub + (int64_t)p->h_send_off[(size_t)j] * H, cr * H, st);
        c->halo_bytes += cr * H * (int64_t)sizeof(float);
      }
    });
  } else if (c->mode == HGNN_MODE_A2A) {
    const int64_t pad = c->max_buffer_rows;
    if (pad == 0 || R == 1) return;
    CUDA_OK(cudaMemsetAsync(c->sendbuf.p, 0, sizeof(float) * (size_t)(R * pad * H), st));
    if (c->n_send > 0) {
      gather_rows_kernel<<<blocks_for(c->n_send * H / 4), kEwThreads, 0, st>>>(
          a, c->send_rows.p, c->pos_a2a_send.p, c->n_send, (int)H, c->sendbuf.p);
      check_launch(c);
    }
    local_exchange(c, kCollHaloFwd, c->sendbuf.p, st, [&](LocalGroup& G) {
      for (int d = 0; d < R; ++d) {  // padded block of every rank (itself included), comm.cpp:297-298
        const hgnn_ctx* p = G.ctx[(size_t)d];
        if (p->max_buffer_rows != pad) fail(HGNN_ERR_COLLECTIVE, "all_to_all (A2A): buffers must be padded to one common size");
        copy_from_peer(c, c->recvbuf.p + (int64_t)d * pad * H, p, p->xpub + (int64_t)c->rank * pad * H, pad * H, st);
      }
      c->halo_bytes += (int64_t)R * pad * H * (int64_t)sizeof(float);
    });
    if (c->n_recv > 0) {
      scatter_rows_kernel<<<blocks_for(c->n_recv * H / 4), kEwThreads, 0, st>>>(
          c->recvbuf.p, c->pos_a2a_recv.p, c->recv_rows.p, c->n_recv, (int)H, a);
      check_launch(c);
    }
  }
}

// Adjoint (comm.cpp:317-357): rank c pulls, for each neighbour p, p's halo
// adjoint block of the rows c sent it into recvbuf at c's send offsets.
void local_halo_exchange_adjoint(hgnn_ctx* c, float* d_a, cudaStream_t st) {
  const int64_t H = c->H;
  const int R = c->nranks;
  if (c->mode == HGNN_MODE_NA2A) {
    local_exchange(c, kCollHaloAdj, d_a, st, [&](LocalGroup& G) {
      for (size_t n = 0; n < c->h_nbr.size(); ++n) {
        const hgnn_ctx* p = G.ctx[(size_t)c->h_nbr[n]];
        const int j = nbr_index(p, c->rank);
        const int64_t cs = c->h_send_off[n + 1] - c->h_send_off[n];
        if (j < 0 || p->h_recv_off[(size_t)j + 1] - p->h_recv_off[(size_t)j] != cs)
          fail(HGNN_ERR_COLLECTIVE, "halo_exchange_adjoint: masks of ranks " + std::to_string(p->rank) + " and " +
                                        std::to_string(c->rank) + " do not pair");
        copy_from_peer(c, c->recvbuf.p + (int64_t)c->h_send_off[n] * H, p, p->xpub + p->h_recv_base[(size_t)j] * H,
                       cs * H, st);
        c->halo_bytes += cs * H * (int64_t)sizeof(float);
      }
    });
  } else if (c->mode == HGNN_MODE_A2A) {
    const int64_t pad = c->max_buffer_rows;
    if (pad == 0 || R == 1) return;
    CUDA_OK(cudaMemsetAsync(c->sendbuf.p, 0, sizeof(float) * (size_t)(R * pad * H), st));
    if (c->n_recv > 0) {
      gather_rows_kernel<<<blocks_for(c->n_recv * H / 4), kEwThreads, 0, st>>>(
          d_a, c->recv_rows.p, c->pos_a2a_recv.p, c->n_recv, (int)H, c->sendbuf.p);
      check_launch(c);
    }
    local_exchange(c, kCollHaloAdj, c->sendbuf.p, st, [&](LocalGroup& G) {
      for (int d = 0; d < R; ++d) {
        const hgnn_ctx* p = G.ctx[(size_t)d];
        copy_from_peer(c, c->recvbuf.p + (int64_t)d * pad * H, p, p->xpub + (int64_t)c->rank * pad * H, pad * H, st);
      }
      c->halo_bytes += (int64_t)R * pad * H * (int64_t)sizeof(float);
    });
  }
}

void halo_exchange(hgnn_ctx* c, float* a, cudaStream_t st) {
  if (c->group) {
    Timed t(c, HGNN_K_HALO, st);
    local_halo_exchange(c, a, st);
    return;
  }
  if (c->nranks > 1) nccl_check_sequence(c, kCollHaloFwd, c->H);
  Timed t(c, HGNN_K_HALO, st);
  const int64_t H = c->H;
  const int R = c->nranks;
  if (c->mode == HGNN_MODE_NA2A) {
    if (c->n_send > 0) {
      gather_rows_kernel<<<blocks_for(c->n_send * H / 4), kEwThreads, 0, st>>>(a, c->send_rows.p, nullptr,
                                                                                     c->n_send, (int)H, c->sendbuf.p);
      check_launch(c);
    }
    if (R > 1 && !c->h_nbr.empty()) {
      NCCL_OK(ncclGroupStart());
      for (size_t n = 0; n < c->h_nbr.size(); ++n) {
        const int64_t cs = c->h_send_off[n + 1] - c->h_send_off[n];
        const int64_t cr = c->h_recv_off[n + 1] - c->h_recv_off[n];
        NCCL_OK(ncclSend(c->sendbuf.p + (int64_t)c->h_send_off[n] * H, (size_t)(cs * H), ncclFloat, c->h_nbr[n],
                         c->comm, st));
        NCCL_OK(ncclRecv(a + c->h_recv_base[n] * H, (size_t)(cr * H), ncclFloat, c->h_nbr[n], c->comm, st));
        c->halo_bytes += cs * H * (int64_t)sizeof(float);
      }
      NCCL_OK(ncclGroupEnd());
    }
  } else if (c->mode == HGNN_MODE_A2A) {
    const int64_t pad = c->max_buffer_rows;
    if (pad == 0 || R == 1) return;
    CUDA_OK(cudaMemsetAsync(c->sendbuf.p, 0, sizeof(float) * (size_t)(R * pad * H), st));
    if (c->n_send > 0) {
      gather_rows_kernel<<<blocks_for(c->n_send * H / 4), kEwThreads, 0, st>>>(
          a, c->send_rows.p, c->pos_a2a_send.p, c->n_send, (int)H, c->sendbuf.p);
      check_launch(c);
    }
    NCCL_OK(ncclGroupStart());
    for (int d = 0; d < R; ++d) {
      NCCL_OK(ncclSend(c->sendbuf.p + (int64_t)d * pad * H, (size_t)(pad * H), ncclFloat, d, c->comm, st));
      NCCL_OK(ncclRecv(c->recvbuf.p + (int64_t)d * pad * H, (size_t)(pad * H), ncclFloat, d, c->comm, st));
    }
    NCCL_OK(ncclGroupEnd());
    c->halo_bytes += (int64_t)R * pad * H * (int64_t)sizeof(float);
    if (c->n_recv > 0) {
      scatter_rows_kernel<<<blocks_for(c->n_recv * H / 4), kEwThreads, 0, st>>>(
          c->recvbuf.p, c->pos_a2a_recv.p, c->recv_rows.p, c->n_recv, (int)H, a);
      check_launch(c);
    }
  }
}

void halo_exchange_adjoint(hgnn_ctx* c, float* d_a, cudaStream_t st) {
  if (!c->group && c->nranks > 1 && c->mode != HGNN_MODE_NONE) nccl_check_sequence(c, kCollHaloAdj, c->H);
  Timed t(c, HGNN_K_HALO, st);
  const int64_t H = c->H;
  const int R = c->nranks;
  const int64_t* acc_pos = nullptr;
  if (c->group) {
    if (c->mode == HGNN_MODE_NONE || (c->mode == HGNN_MODE_A2A && (c->max_buffer_rows == 0 || R == 1))) return;
    local_halo_exchange_adjoint(c, d_a, st);
    acc_pos = c->mode == HGNN_MODE_NA2A ? c->acc_pos_na2a.p : c->acc_pos_a2a.p;
  } else if (c->mode == HGNN_MODE_NA2A) {
    if (R > 1 && !c->h_nbr.empty()) {
      NCCL_OK(ncclGroupStart());
      for (size_t n = 0; n < c->h_nbr.size(); ++n) {
        const int64_t cs = c->h_send_off[n + 1] - c->h_send_off[n];
        const int64_t cr = c->h_recv_off[n + 1] - c->h_recv_off[n];
        // halo rows of neighbour n are one contiguous block: sent as they lie
        NCCL_OK(ncclSend(d_a + c->h_recv_base[n] * H, (size_t)(cr * H), ncclFloat, c->h_nbr[n], c->comm, st));
        NCCL_OK(ncclRecv(c->recvbuf.p + (int64_t)c->h_send_off[n] * H, (size_t)(cs * H), ncclFloat, c->h_nbr[n],
                         c->comm, st));
        c->halo_bytes += cr * H * (int64_t)sizeof(float);
      }
      NCCL_OK(ncclGroupEnd());
    }
    acc_pos = c->acc_pos_na2a.p;
  } else if (c->mode == HGNN_MODE_A2A) {
    const int64_t pad = c->max_buffer_rows;
    if (pad == 0 || R == 1) return;
    CUDA_OK(cudaMemsetAsync(c->sendbuf.p, 0, sizeof(float) * (size_t)(R * pad * H), st));
    if (c->n_recv > 0) {
      gather_rows_kernel<<<blocks_for(c->n_recv * H / 4), kEwThreads, 0, st>>>(
          d_a, c->recv_rows.p, c->pos_a2a_recv.p, c->n_recv, (int)H, c->sendbuf.p);
      check_launch(c);
    }
    NCCL_OK(ncclGroupStart());
    for (int d = 0; d < R; ++d) {
      NCCL_OK(ncclSend(c->sendbuf.p + (int64_t)d * pad * H, (size_t)(pad * H), ncclFloat, d, c->comm, st));
      NCCL_OK(ncclRecv(c->recvbuf.p + (int64_t)d * pad * H, (size_t)(pad * H), ncclFloat, d, c->comm, st));
    }
    NCCL_OK(ncclGroupEnd());
    c->halo_bytes += (int64_t)R * pad * H * (int64_t)sizeof(float);
    acc_pos = c->acc_pos_a2a.p;
  } else {
    return;
  }
  // the overwritten halo rows contribute nothing upstream (comm.cpp:339-342)
  if (c->nh > 0)
    CUDA_OK(cudaMemsetAsync(d_a + c->nl * H, 0, sizeof(float) * (size_t)(c->nh * H), st));
  if (c->n_acc > 0 && R > 1) {
    adjoint_accumulate_kernel<<<blocks_for(c->n_acc * H / 4), kEwThreads, 0, st>>>(
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
  // per launch: the attribute belongs to the current device (cheap host call)
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
  const int64_t pairs = ((args.n_rows + 127) / 128 + 1) / 2;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(pairs, c->num_sms - c->sm_reserve));
  k<<<grid, Cfg::THREADS, Cfg::SMEM, c->stream>>>(args);
  check_launch(c);
}

// Edge mode: slots [s0, s0 + n_rows).
void launch_tc_forward(hgnn_ctx* c, int mode, int64_t m, int64_t n_rows, const float* x, const float* e,
                       const float* a, float* out, int64_t s0 = 0) {
  if (n_rows == 0) return;
  const bool edge = mode == kEdgeInput;
  TcFwdArgs args{};
  args.n_rows = n_rows;
  args.src = c->src.p + s0;
  args.dst = c->dst.p + s0;
  args.x = x;
  args.e_in = e ? e + s0 * c->H : nullptr;
  args.a = a;
  args.out = out + s0 * c->H;
  args.chunks = c->chunks.p + c->chunk_off[(size_t)(3 * m + (edge ? 0 : 1))];
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

bool use_fact(const hgnn_ctx* c) { return c->edge_fact && c->fact_ok && c->H == 64; }
bool use_fused_fwd(const hgnn_ctx* c) { return use_tc(c) && c->fact_ok; }

// P_m = x_m [W0_s | W0_d] on the local rows (edges never reference halo rows)
void edge_proj(hgnn_ctx* c, int64_t m, const float* x) {
  Timed t(c, HGNN_K_EDGE_PROJ);
  if (c->nl == 0) return;
  const float* w0 = layer_params(c, m, true).p;
  constexpr size_t smem = edge_proj_smem<64>();
  CUDA_OK(cudaFuncSetAttribute(edge_proj_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned grid = (unsigned)std::min<int64_t>((c->nl + kFactRows - 1) / kFactRows, (int64_t)c->num_sms * 4);
  edge_proj_kernel<64><<<grid, kFactThreads, smem, c->stream>>>(x, w0, c->nl, proj_buf(c, m));
  check_launch(c);
  if (c->lean) std::fill(c->ps_ready.begin(), c->ps_ready.end(), 0);  // one shared buffer
  c->ps_ready[(size_t)m] = 1;
}

// 2-D fp32 tensor map over a rows x H row-major buffer for TMA tile::gather4
// (box 32 floats x 1 row, 128-byte swizzle). The driver entry point comes
// from the runtime (no libcuda link dependency).
CUtensorMap row_tensor_map(const float* base, int64_t rows, int H) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) fail(HGNN_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CUtensorMap m{};
  const cuuint64_t dims[2] = {(cuuint64_t)H, (cuuint64_t)std::max<int64_t>(rows, 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)H * sizeof(float)};
  const cuuint32_t box[2] = {32, 1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(HGNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

template <int MODE>
void launch_fused_tma(hgnn_ctx* c, const TcFwdArgs& args) {
  using Cfg = TcCfg<64>;
  auto k = mlp_tc_forward_tma_kernel<64, MODE>;
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM_TMA));
  const CUtensorMap tx = row_tensor_map(args.x, c->rows, 64), te = row_tensor_map(args.e_in, c->ne, 64);
  const int64_t pairs = (args.n_tiles + 1) / 2;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(pairs, c->num_sms - c->sm_reserve));
  k<<<grid, Cfg::THREADS, Cfg::SMEM_TMA, c->stream>>>(args, tx, te);
  check_launch(c);
}

// The fused edge update (kEdgeFact / kEdgeFused): tiles [t0, t1) of the
// segment table; writes e' and the aggregate of every receiver in those tiles.
template <int H, int MODE>
void launch_fused_typed(hgnn_ctx* c, const TcFwdArgs& args) {
  auto k = mlp_tc_forward_kernel<H, MODE, false>;
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TcCfg<H>::SMEM_FACT));
  const int64_t pairs = (args.n_tiles + 1) / 2;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(pairs, c->num_sms - c->sm_reserve));
  k<<<grid, TcCfg<H>::THREADS, TcCfg<H>::SMEM_FACT, c->stream>>>(args);
  check_launch(c);
}
// The fused edge update: tiles [t0, t1) of the receiver-segment table; writes
// e' (e2) and the aggregate of every receiver in those tiles. kEdgeFact when
// the input linear is factorised through the nodes, else kEdgeFused.
void launch_fused_forward(hgnn_ctx* c, int64_t m, int64_t t0, int64_t t1, const float* x, const float* e, float* e2,
                          float* a) {
  if (t1 <= t0) return;
  const bool fact = use_fact(c);
  TcFwdArgs args{};
  args.n_tiles = t1 - t0;
  args.tiles = c->tiles.p + t0;
  args.src = c->src.p;
  args.dst = c->dst.p;
  args.inv = c->inv.p;
  args.x = x;
  args.e_in = e;
  args.out = e2;
  args.agg = a;
  args.proj = fact ? proj_buf(c, m) : nullptr;
  args.chunks = c->chunks.p + c->chunk_off[(size_t)(3 * m + (fact ? 2 : 0))];
  args.params = layer_params(c, m, true).p;
  args.k = (int)c->K;
  if (c->H == 64 && c->tma_gather) {
    if (fact) launch_fused_tma<kEdgeFact>(c, args);
    else launch_fused_tma<kEdgeFused>(c, args);
  } else if (c->H == 64) {
    if (fact) launch_fused_typed<64, kEdgeFact>(c, args);
    else launch_fused_typed<64, kEdgeFused>(c, args);
  } else {
    launch_fused_typed<32, kEdgeFused>(c, args);
  }
}
void zero_empty_rows(hgnn_ctx* c, float* a) {
  if (c->n_rows_empty == 0) return;
  zero_rows_kernel<<<blocks_for(c->n_rows_empty * c->H / 4), kEwThreads, 0, c->stream>>>(c->rows_empty.p,
                                                                                       c->n_rows_empty, (int)c->H, a);
  check_launch(c);
}

// H = 32 runs zero-padded on the 64-wide backward kernel (HL = 32)
bool use_tc_bwd(const hgnn_ctx* c) { return c->bwd_impl == 1 && tc_eligible(c); }
bool use_fact_bwd(const hgnn_ctx* c) { return use_tc_bwd(c) && use_fact(c); }

int tc_bwd_grid(const hgnn_ctx* c, int64_t n_rows) {
  const int64_t pairs = ((n_rows + 127) / 128 + 1) / 2;
  return (int)std::max<int64_t>(1, std::min<int64_t>(pairs, c->num_sms - c->sm_reserve));
}

// Returns the grid used (rows of grad_part written).
int launch_tc_backward(hgnn_ctx* c, int mode, int64_t m, const TcBwdArgs& in) {
  const bool edge = mode != kNodeInput;
  TcBwdArgs args = in;
  args.chunks = c->bchunks.p + c->bchunk_off[(size_t)(3 * m + (mode == kEdgeFact ? 2 : (edge ? 0 : 1)))];
  args.params = layer_params(c, m, edge).p;
  args.k = (int)c->K;
  args.scratch = c->tc_scratch.p;
  args.prof = c->prof_on ? c->prof.p + (edge ? 0 : kProfCount) : nullptr;
  const int grid = tc_bwd_grid(c, args.n_rows);
  const bool prof = args.prof != nullptr;
  if (c->H == 32) {  // zero-padded H = 32 instance
    auto k32 = edge ? mlp_tc_backward_kernel<kEdgeInput, false, 32> : mlp_tc_backward_kernel<kNodeInput, false, 32>;
    CUDA_OK(cudaFuncSetAttribute(k32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TcBwdCfg::SMEM));
    k32<<<grid, TcBwdCfg::THREADS, TcBwdCfg::SMEM, c->stream>>>(args);
    check_launch(c);
    return grid;
  }
  auto k = mode == kEdgeFact
               ? (prof ? mlp_tc_backward_kernel<kEdgeFact, true> : mlp_tc_backward_kernel<kEdgeFact, false>)
               : edge ? (prof ? mlp_tc_backward_kernel<kEdgeInput, true> : mlp_tc_backward_kernel<kEdgeInput, false>)
                      : (prof ? mlp_tc_backward_kernel<kNodeInput, true> : mlp_tc_backward_kernel<kNodeInput, false>);
  CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TcBwdCfg::SMEM));
  k<<<grid, TcBwdCfg::THREADS, TcBwdCfg::SMEM, c->stream>>>(args);
  check_launch(c);
  return grid;
}

// node update on local rows (model.cpp:260-264)
void node_forward(hgnn_ctx* c, int64_t m, const float* x, const float* a, float* x2) {
  const int64_t H = c->H;
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


void sync_aggregates(hgnn_ctx* c, float* a) {
  if (c->n_sync == 0) return;
  Timed t(c, HGNN_K_HALO);
  sync_kernel<<<blocks_for(c->n_sync * c->H / 4), kEwThreads, 0, c->stream>>>(a, c->sync_local.p, c->sync_off.p,
                                                                              c->sync_slots.p, c->n_sync, (int)c->H);
  check_launch(c);
}

bool can_overlap(const hgnn_ctx* c) {
  return c->halo_overlap && c->mode != HGNN_MODE_NONE && c->nranks > 1 && (c->comm || c->group);
}

// Edge update as ONE fused kernel (gather -> tcgen05 MLP -> e' + segmented
// 1/d aggregate), after the node projections when the input linear is
// factorised; with an exchange, the boundary tiles first and the exchange on
// the side stream while the interior tiles run.
void layer_forward_fused(hgnn_ctx* c, int64_t m, float* x, float* e, float* e2, float* a, float* x2) {
  if (use_fact(c)) edge_proj(c, m, x);
  zero_empty_rows(c, a);  // empty segments (halo rows: before the receive overwrites them)
  if (can_overlap(c) && c->n_tiles_bnd > 0) {
    {
      Timed t(c, HGNN_K_EDGE_FWD);
      launch_fused_forward(c, m, 0, c->n_tiles_bnd, x, e, e2, a);
    }
    CUDA_OK(cudaEventRecord(c->ev_bnd, c->stream));
    CUDA_OK(cudaStreamWaitEvent(c->side, c->ev_bnd, 0));
    halo_exchange(c, a, c->side);
    CUDA_OK(cudaEventRecord(c->ev_halo, c->side));
    {
      Timed t(c, HGNN_K_EDGE_FWD);
      c->sm_reserve = c->halo_sm_reserve;
      launch_fused_forward(c, m, c->n_tiles_bnd, c->n_tiles, x, e, e2, a);
      c->sm_reserve = 0;
    }
    CUDA_OK(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
    sync_aggregates(c, a);
  } else {
    {
      Timed t(c, HGNN_K_EDGE_FWD);
      launch_fused_forward(c, m, 0, c->n_tiles, x, e, e2, a);
    }
    if (c->mode != HGNN_MODE_NONE) {
      halo_exchange(c, a, c->stream);
      sync_aggregates(c, a);
    }
  }
  node_forward(c, m, x, a, x2);
}

void layer_forward(hgnn_ctx* c, int64_t m) {
  const int64_t H = c->H;
  float* x = x_buf(c, m);
  float* e = e_buf(c, m);
  float* e2 = e_buf(c, m + 1);  // nullptr: the dead last-layer e' (lean plan, fused path only)
  float* a = c->as[m]->p;
  float* x2 = x_buf(c, m + 1);
  if (use_fused_fwd(c)) {
    layer_forward_fused(c, m, x, e, e2, a, x2);
    return;
  }
  if (c->halo_overlap && c->mode != HGNN_MODE_NONE && c->nranks > 1 && (c->comm || c->group) && c->n_rows_bnd > 0 &&
      use_tc(c)) {
    // Overlapped schedule, same results: boundary-row edges + aggregates,
    // then the exchange on the side stream while the interior edges run on
    // all but halo_sm_reserve SMs (left to the pack and NCCL kernels).
    {
      Timed t(c, HGNN_K_EDGE_FWD);
      launch_tc_forward(c, kEdgeInput, m, c->ne_bnd, x, e, nullptr, e2, 0);
    }
    {
      Timed t(c, HGNN_K_AGG);
      aggregate_kernel<<<blocks_for(c->n_rows_bnd * H / 4), kEwThreads, 0, c->stream>>>(
          e2, c->inv.p, c->seg_beg.p, c->seg_end.p, c->rows_bnd.p, c->n_rows_bnd, (int)H, a);
      check_launch(c);
    }
    CUDA_OK(cudaEventRecord(c->ev_bnd, c->stream));
    CUDA_OK(cudaStreamWaitEvent(c->side, c->ev_bnd, 0));
    halo_exchange(c, a, c->side);
    CUDA_OK(cudaEventRecord(c->ev_halo, c->side));
    {
      Timed t(c, HGNN_K_EDGE_FWD);
      c->sm_reserve = c->halo_sm_reserve;
      launch_tc_forward(c, kEdgeInput, m, c->ne - c->ne_bnd, x, e, nullptr, e2, c->ne_bnd);
      c->sm_reserve = 0;
    }
    if (c->n_rows_int > 0) {
      Timed t(c, HGNN_K_AGG);
      aggregate_kernel<<<blocks_for(c->n_rows_int * H / 4), kEwThreads, 0, c->stream>>>(
          e2, c->inv.p, c->seg_beg.p, c->seg_end.p, c->rows_int.p, c->n_rows_int, (int)H, a);
      check_launch(c);
    }
    CUDA_OK(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
    if (c->n_sync > 0) {
      Timed t(c, HGNN_K_HALO);
      sync_kernel<<<blocks_for(c->n_sync * H / 4), kEwThreads, 0, c->stream>>>(a, c->sync_local.p, c->sync_off.p,
                                                                              c->sync_slots.p, c->n_sync, (int)H);
      check_launch(c);
    }
    node_forward(c, m, x, a, x2);
    return;
  }
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
    aggregate_kernel<<<blocks_for(c->rows * H / 4), kEwThreads, 0, c->stream>>>(
        e2, c->inv.p, c->seg_beg.p, c->seg_end.p, nullptr, c->rows, (int)H, a);
    check_launch(c);
  }
  if (c->mode != HGNN_MODE_NONE) {  // exchange + synchronisation (model.cpp:243-257)
    halo_exchange(c, a, c->stream);
    if (c->n_sync > 0) {
      Timed t(c, HGNN_K_HALO);
      sync_kernel<<<blocks_for(c->n_sync * H / 4), kEwThreads, 0, c->stream>>>(a, c->sync_local.p, c->sync_off.p,
                                                                              c->sync_slots.p, c->n_sync, (int)H);
      check_launch(c);
    }
  }
  node_forward(c, m, x, a, x2);
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
  float* x = x_buf(c, m);
  float* e = e_buf(c, m);
  const float* de_in = de_in_buf(c, m);
  float* de_out = de_out_buf(c, m);
  float* dxn = dxn_buf(c);
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
      args.d_x_out = dxn;
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
      args.d_x_out = dxn;
      args.grad_partial = c->grad_part.p;
      args.scratch = c->scratch.p;
      args.n_slots = (2 * c->K + 1) * H + c->K;
      launch_mlp(c, false, kNodeInput, args, layer_params(c, m, false));
      if (c->nl > 0) reduce_grads(c, c->grid_node_b, c->n_node_par, c->grads.p + goff + c->n_edge_par);
    }
  }
  const bool fact = use_fact_bwd(c);
  const int emode = fact ? kEdgeFact : kEdgeInput;
  if (fact && !c->ps_ready[(size_t)m]) edge_proj(c, m, x);  // forward ran without the node projections
  if (c->halo_overlap && c->mode != HGNN_MODE_NONE && c->nranks > 1 && (c->comm || c->group) && c->n_rows_bnd > 0 &&
      use_tc_bwd(c)) {
    // Overlapped schedule: sync adjoint, then the adjoint exchange on the side
    // stream while the interior edges (receivers whose d_a the exchange does
    // not touch) run their backward; the boundary edges follow the exchange.
    if (c->n_sync > 0) {
      Timed t(c, HGNN_K_HALO);
      sync_adjoint_kernel<<<blocks_for(c->n_sync * H / 4), kEwThreads, 0, c->stream>>>(
          c->d_a.p, c->sync_local.p, c->sync_off.p, c->sync_slots.p, c->n_sync, (int)H);
      check_launch(c);
    }
    CUDA_OK(cudaEventRecord(c->ev_bnd, c->stream));
    CUDA_OK(cudaStreamWaitEvent(c->side, c->ev_bnd, 0));
    halo_exchange_adjoint(c, c->d_a.p, c->side);
    CUDA_OK(cudaEventRecord(c->ev_halo, c->side));
    const int64_t n_int = c->ne - c->ne_bnd;
    c->sm_reserve = c->halo_sm_reserve;
    const int g1 = n_int > 0 ? tc_bwd_grid(c, n_int) : 0;
    c->sm_reserve = 0;
    const int g2 = c->ne_bnd > 0 ? tc_bwd_grid(c, c->ne_bnd) : 0;
    auto edge_args = [&](int64_t s0, int64_t n, float* part) {
      TcBwdArgs args{};
      args.n_rows = n;
      args.src = c->src.p + s0;
      args.dst = c->dst.p + s0;
      args.x = x;
      args.e_in = e + s0 * H;
      args.inv_deg = c->inv.p + s0;
      args.d_a = c->d_a.p;
      args.de_in = de_in ? de_in + s0 * H : nullptr;
      args.de_io = de_out + s0 * H;
      args.d_src = c->dsrc.p + s0 * H;
      args.d_dst = c->ddst.p + s0 * H;
      args.proj = fact ? proj_buf(c, m) : nullptr;
      args.dy_out = c->dsrc.p + s0 * H;  // kEdgeFact: dY
      args.grad_partial = part;
      return args;
    };
    {
      Timed t(c, HGNN_K_EDGE_BWD);
      CUDA_OK(cudaMemsetAsync(c->grad_part.p, 0, sizeof(float) * (size_t)(2 * (g1 + g2) * c->n_edge_par),
                              c->stream));
      if (n_int > 0) {
        c->sm_reserve = c->halo_sm_reserve;
        launch_tc_backward(c, emode, m, edge_args(c->ne_bnd, n_int, c->grad_part.p));
        c->sm_reserve = 0;
      }
    }
    CUDA_OK(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
    {
      Timed t(c, HGNN_K_EDGE_BWD);
      if (c->ne_bnd > 0)
        launch_tc_backward(c, emode, m, edge_args(0, c->ne_bnd, c->grad_part.p + 2 * g1 * c->n_edge_par));
      reduce_grads(c, 2 * (g1 + g2), c->n_edge_par, c->grads.p + goff);
    }
  } else {
  if (c->mode != HGNN_MODE_NONE) {  // sync + exchange adjoints (model.cpp:343-351)
    if (c->n_sync > 0) {
      Timed t(c, HGNN_K_HALO);
      sync_adjoint_kernel<<<blocks_for(c->n_sync * H / 4), kEwThreads, 0, c->stream>>>(
          c->d_a.p, c->sync_local.p, c->sync_off.p, c->sync_slots.p, c->n_sync, (int)H);
      check_launch(c);
    }
    halo_exchange_adjoint(c, c->d_a.p, c->stream);
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
      args.de_in = de_in;
      args.de_io = de_out;
      args.d_src = c->dsrc.p;
      args.d_dst = c->ddst.p;
      args.proj = fact ? proj_buf(c, m) : nullptr;
      args.dy_out = c->dsrc.p;  // kEdgeFact: dY
      args.grad_partial = c->grad_part.p;
      if (c->ne > 0) {
        launch_tc_backward(c, emode, m, args);
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
      args.de_io = c->de.p;  // SIMT path: standard plan only (in place)
      args.d_src = c->dsrc.p;
      args.d_dst = c->ddst.p;
      args.grad_partial = c->grad_part.p;
      args.scratch = c->scratch.p;
      args.n_slots = (2 * c->K + 1) * H + c->K;
      launch_mlp(c, false, kEdgeInput, args, layer_params(c, m, true));
      if (c->ne > 0) reduce_grads(c, c->grid_edge_b, c->n_edge_par, c->grads.p + goff);
    }
  }
  }  // serial schedule
  if (fact) {  // input-node adjoint through the node-level sums of dY (edge_fact.cuh), + dW0_s / dW0_d
    Timed t(c, HGNN_K_DX);
    const float* w0 = layer_params(c, m, true).p;
    constexpr size_t smem = edge_input_adjoint_smem<64>();
    if (c->adj_presum) {  // segment sums at full occupancy into the (now dead) node projection of layer m
      float* S = proj_buf(c, m);
      seg_sum_kernel<64><<<blocks_for(c->rows * 2 * H / 4), kEwThreads, 0, c->stream>>>(
          c->dsrc.p, c->seg_beg.p, c->seg_end.p, c->twin.p, c->rows, S);
      check_launch(c);
      if (c->lean) std::fill(c->ps_ready.begin(), c->ps_ready.end(), 0);
      else c->ps_ready[(size_t)m] = 0;  // a repeated backward recomputes P_m
      CUDA_OK(cudaFuncSetAttribute(edge_input_adjoint_kernel<64, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      edge_input_adjoint_kernel<64, true><<<c->fact_blocks, kFactThreads, smem, c->stream>>>(
          c->dsrc.p, x, dxn, w0, c->seg_beg.p, c->seg_end.p, c->twin.p, c->rows, c->nl, c->dx.p, c->fact_part.p, S);
    } else {
      CUDA_OK(cudaFuncSetAttribute(edge_input_adjoint_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
      edge_input_adjoint_kernel<64><<<c->fact_blocks, kFactThreads, smem, c->stream>>>(
          c->dsrc.p, x, dxn, w0, c->seg_beg.p, c->seg_end.p, c->twin.p, c->rows, c->nl, c->dx.p, c->fact_part.p);
    }
    check_launch(c);
    const int64_t nw = 2 * H * H;  // W0 rows 0 .. 2H-1 (x_src, x_dst blocks) of the edge MLP
    grad_reduce_add_kernel<<<blocks_for(nw), kEwThreads, 0, c->stream>>>(c->fact_part.p, c->fact_blocks, nw,
                                                                         c->grads.p + goff);
    check_launch(c);
  } else {  // input-node adjoint (model.cpp:378-386)
    Timed t(c, HGNN_K_DX);
    dx_gather_kernel<<<blocks_for(c->rows * H / 4), kEwThreads, 0, c->stream>>>(
        c->dsrc.p, c->ddst.p, dxn, c->seg_beg.p, c->seg_end.p, c->twin.p, c->rows, c->nl, (int)H, c->dx.p);
    check_launch(c);
  }
}

void run_forward(hgnn_ctx* c) {
  c->ps_ready.assign((size_t)c->M, 0);
  for (int64_t m = 0; m < c->M; ++m) layer_forward(c, m);
  c->forward_done = true;
}

void run_backward(hgnn_ctx* c) {
  if (!c->forward_done) fail(HGNN_ERR_UNINITIALIZED, "hgnn_mp_backward called before hgnn_mp_forward");
  if (c->M == 0) return;
  CUDA_OK(cudaMemsetAsync(c->grads.p, 0, sizeof(double) * (size_t)c->n_mp_par, c->stream));
  for (int64_t m = c->M - 1; m >= 0; --m) layer_backward(c, m);
  if (c->lean) c->forward_done = false;  // de_m overwrote e_m, dY overwrote x_M
}

void require_ready(hgnn_ctx* c) {
  if (!c->configured) fail(HGNN_ERR_UNINITIALIZED, "hgnn_configure has not been called");
  if (!c->graph_ready) fail(HGNN_ERR_UNINITIALIZED, "hgnn_graph_upload has not been called");
  if (!c->params_ready) fail(HGNN_ERR_UNINITIALIZED, "hgnn_params_upload has not been called");
  if (c->mode != HGNN_MODE_NONE && c->nranks > 1 && !c->comm && !c->group)
    fail(HGNN_ERR_CONFIG, "nmp_layer: exchange mode requires a rank runtime");
}

}  // namespace hgnn_b200::engine

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

int hgnn_local_group_create(int32_t num_ranks, hgnn_local_group** out) {
  return guarded([&] {
    if (!out) fail(HGNN_ERR_CONFIG, "hgnn_local_group_create: null output");
    if (num_ranks < 1) fail(HGNN_ERR_CONFIG, "RankRuntime: need at least one rank");
    *out = reinterpret_cast<hgnn_local_group*>(new LocalGroup(num_ranks));
  });
}

int hgnn_local_group_destroy(hgnn_local_group* g) {
  return guarded([&] { delete reinterpret_cast<LocalGroup*>(g); });
}

int hgnn_local_group_set_timeout(hgnn_local_group* g, int64_t timeout_ms) {
  return guarded([&] {
    if (!g || timeout_ms <= 0) fail(HGNN_ERR_CONFIG, "hgnn_local_group_set_timeout: bad arguments");
    reinterpret_cast<LocalGroup*>(g)->timeout_ms = timeout_ms;
  });
}

int hgnn_ctx_create_local(int device, int32_t rank, hgnn_local_group* group, hgnn_ctx** out) {
  return guarded([&] {
    if (!group) fail(HGNN_ERR_CONFIG, "hgnn_ctx_create_local: null group");
    LocalGroup* G = reinterpret_cast<LocalGroup*>(group);
    if (rank < 0 || rank >= G->R) fail(HGNN_ERR_CONFIG, "hgnn_ctx_create_local: bad rank");
    hgnn_ctx* c = nullptr;
    const int rc = hgnn_ctx_create(device, 0, 1, nullptr, &c);  // a single-rank context, then joined to the group
    if (rc != HGNN_OK) fail(rc, hgnn_last_error());
    c->rank = rank;
    c->nranks = G->R;
    c->group = G;
    try {
      CUDA_OK(cudaEventCreateWithFlags(&c->ev_pub, cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&c->ev_consumed, cudaEventDisableTiming));
      G->attach(rank, c);
    } catch (...) {
      c->group = nullptr;
      hgnn_ctx_destroy(c);
      throw;
    }
    *out = c;
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
    CUDA_OK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_bnd, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
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
    if (c->group) c->group->retire(c->rank);
    if (c->ev_pub) cudaEventDestroy(c->ev_pub);
    if (c->ev_consumed) cudaEventDestroy(c->ev_consumed);
    if (c->ev_bnd) cudaEventDestroy(c->ev_bnd);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    if (c->side) cudaStreamDestroy(c->side);
    cudaStreamDestroy(c->stream);
    delete c;
  });
}

void* hgnn_ctx_stream(hgnn_ctx* c) { return c ? (void*)c->stream : nullptr; }

int hgnn_graph_upload(hgnn_ctx* c, const hgnn_graph_desc* g) {
  return guarded([&] {
    bind(c);
    if (!g) fail(HGNN_ERR_CONFIG, "hgnn_graph_upload: null graph");
    // num_ranks == 0: not known to the caller (a loaded HGNNGRB1 file, or the
    // reference-side GraphDesc); the context carries the rank count.
    if (g->rank != c->rank || (g->num_ranks != 0 && g->num_ranks != c->nranks))
      fail(HGNN_ERR_INTEGRITY, "hgnn_graph_upload: graph rank/num_ranks do not match the context");
    const int64_t nl = g->num_local, nh = g->num_halo, ne = g->num_edges, rows = nl + nh;
    if (nl < 0 || nh < 0 || ne < 0 || rows >= INT32_MAX || ne >= INT32_MAX)
      fail(HGNN_ERR_SHAPE, "hgnn_graph_upload: sizes out of range");
    if (ne % 2) fail(HGNN_ERR_INTEGRITY, "directed edges must come in twin pairs (graph.cpp:107-110)");
    // Slots: receiver segments in in-CSR order (each segment keeps the
    // reference's in-edge order, so every per-row sum is unchanged); with
    // R > 1 the boundary rows' segments (rows the exchange packs) come first.
    // Twin slots via the e^1 pairing.
    if (g->in_offsets[0] != 0 || g->in_offsets[rows] != ne) fail(HGNN_ERR_INTEGRITY, "in_offsets do not span N_e");
    const int nn0 = g->num_neighbors;
    const int64_t n_send0 = nn0 > 0 ? g->send_offsets[nn0] : 0;
    std::vector<uint8_t> bnd((size_t)rows, 0);
    for (int64_t i = nl; i < rows; ++i) bnd[(size_t)i] = 1;  // halo rows: no in-edges, zeroed before the receive
    for (int64_t t = 0; t < n_send0; ++t) {
      const int32_t r = g->send_rows[t];
      if (r < 0 || r >= nl) fail(HGNN_ERR_INTEGRITY, "send rows must be local rows");
      bnd[(size_t)r] = 1;
    }
    const bool split = c->nranks > 1 && n_send0 > 0;
    std::vector<int32_t> new_of_old((size_t)ne), seg_b((size_t)rows), seg_e((size_t)rows), rb, ri;
    int32_t next = 0;
    auto place = [&](int64_t i) {
      seg_b[(size_t)i] = next;
      for (int32_t p = g->in_offsets[i]; p < g->in_offsets[i + 1]; ++p) new_of_old[(size_t)p] = next++;
      seg_e[(size_t)i] = next;
    };
    for (int64_t i = 0; i < rows; ++i)
      if (!split || bnd[(size_t)i]) {
        place(i);
        rb.push_back((int32_t)i);
      }
    const int64_t ne_bnd = split ? next : ne;
    if (split)
      for (int64_t i = 0; i < rows; ++i)
        if (!bnd[(size_t)i]) {
          place(i);
          ri.push_back((int32_t)i);
        }
    std::vector<int32_t> slot_of((size_t)ne), src_s((size_t)ne), dst_s((size_t)ne), twin((size_t)ne);
    std::vector<float> inv_s((size_t)ne);
    for (int64_t i = 0; i < rows; ++i)
      for (int32_t p = g->in_offsets[i]; p < g->in_offsets[i + 1]; ++p) {
        const int32_t e = g->in_edges[p];
        if (e < 0 || e >= ne || g->edge_dst[e] != i) fail(HGNN_ERR_INTEGRITY, "in-CSR inconsistent with edge_dst");
        slot_of[(size_t)e] = new_of_old[(size_t)p];
      }
    for (int64_t p = 0; p < ne; ++p) {
      const int32_t e = g->in_edges[p];
      const int32_t s = g->edge_src[e], d = g->edge_dst[e];
      if (s < 0 || s >= nl || d < 0 || d >= nl) fail(HGNN_ERR_INTEGRITY, "edges must not reference halo rows");
      const int32_t t = e ^ 1;
      if (g->edge_src[t] != d || g->edge_dst[t] != s) fail(HGNN_ERR_INTEGRITY, "edge e^1 is not the twin of e");
      const size_t q = (size_t)new_of_old[(size_t)p];
      src_s[q] = s;
      dst_s[q] = d;
      inv_s[q] = (float)g->edge_inv_degree[e];
      twin[q] = slot_of[(size_t)t];
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
    else c->node_inv.release();
    c->model_data_ready = false;  // features / targets were sized for the previous graph
    c->seg_beg.upload(seg_b.data(), rows, c->stream);
    c->seg_end.upload(seg_e.data(), rows, c->stream);
    c->ne_bnd = ne_bnd;
    c->n_rows_bnd = split ? (int64_t)rb.size() : 0;
    c->n_rows_int = split ? (int64_t)ri.size() : 0;
    c->rows_bnd.upload(rb.data(), c->n_rows_bnd, c->stream);
    c->rows_int.upload(ri.data(), c->n_rows_int, c->stream);
    {  // fused edge kernel tiles: runs of whole receiver segments, <= 128 slots,
       // in slot order, cut at the boundary / interior split
      std::vector<int32_t> tl{0}, empty;
      int32_t cur = 0;  // slots in the open tile
      bool ok = true;
      auto add_rows = [&](const std::vector<int32_t>& order) {
        for (int32_t i : order) {
          const int32_t len = seg_e[(size_t)i] - seg_b[(size_t)i];
          if (len == 0) {
            empty.push_back(i);
            continue;
          }
          if (len > 128) ok = false;
          if (cur + len > 128 && cur > 0) {
            tl.push_back(seg_b[(size_t)i]);
            cur = 0;
          }
          cur += len;
        }
        if (cur > 0) {
          tl.push_back(tl.back() + cur);
          cur = 0;
        }
      };
      std::vector<int32_t> all_rows;
      if (!split) {
        all_rows.resize((size_t)rows);
        for (int64_t i = 0; i < rows; ++i) all_rows[(size_t)i] = (int32_t)i;
      }
      add_rows(split ? rb : all_rows);
      c->n_tiles_bnd = split ? (int64_t)tl.size() - 1 : 0;
      if (split) add_rows(ri);
      c->fact_ok = ok && tl.back() == ne;
      c->n_tiles = (int64_t)tl.size() - 1;
      c->tiles.upload(tl.data(), (int64_t)tl.size(), c->stream);
      c->n_rows_empty = (int64_t)empty.size();
      c->rows_empty.upload(empty.data(), c->n_rows_empty, c->stream);
    }
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
      // an empty receive block has no base row (and its first index may be nh)
      const bool empty_recv = c->h_recv_off[(size_t)n + 1] == c->h_recv_off[(size_t)n];
      const int64_t base = empty_recv ? nl : g->recv_rows[c->h_recv_off[(size_t)n]];
      c->h_recv_base[(size_t)n] = base;
      if (!empty_recv && (base < nl || base + (c->h_recv_off[(size_t)n + 1] - c->h_recv_off[(size_t)n]) > rows))
        fail(HGNN_ERR_INTEGRITY, "recv rows must be halo rows [num_local, rows)");
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
    // sync groups: sync_kernel writes each group's local row in place and
    // reads its slots, so a slot must be -1 (the row itself) or a halo row
    // (never written by the sync), and each local row may own one group
    {
      std::vector<uint8_t> owned((size_t)nl, 0);
      for (int64_t q = 0; q < g->num_sync_groups; ++q) {
        const int32_t li = g->sync_local[q];
        if (li < 0 || li >= nl || owned[(size_t)li]) fail(HGNN_ERR_INTEGRITY, "sync group local rows must be distinct local rows");
        owned[(size_t)li] = 1;
        if (g->sync_offsets[q + 1] < g->sync_offsets[q]) fail(HGNN_ERR_INTEGRITY, "sync offsets must be ascending");
        for (int32_t t = g->sync_offsets[q]; t < g->sync_offsets[q + 1]; ++t) {
          const int32_t sl = g->sync_slots[t];
          if (sl != -1 && (sl < nl || sl >= rows)) fail(HGNN_ERR_INTEGRITY, "sync slots must be -1 or halo rows");
        }
      }
    }
    c->n_sync = g->num_sync_groups;
    c->sync_local.upload(g->sync_local, c->n_sync, c->stream);
    c->sync_off.upload(g->sync_offsets, c->n_sync + 1, c->stream);
    c->sync_slots.upload(g->sync_slots, c->n_sync ? g->sync_offsets[c->n_sync] : 0, c->stream);
    CUDA_OK(cudaStreamSynchronize(c->stream));
    c->graph_ready = true;
    c->forward_done = false;
    for (auto& v : c->plan_key) v = -1;  // buffers re-planned by the next ensure_buffers
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
    if (mode != HGNN_MODE_NONE && c->nranks > 1 && !c->comm && !c->group)
      fail(HGNN_ERR_CONFIG, "nmp_layer: exchange mode requires a rank runtime");
    if (c->H != hidden || c->M != M || c->K != k) {
      // every size derived from (H, M, k) is stale: the MP parameters and the
      // model level's layout (off_mp, n_full, ...) must be set up again
      c->params_ready = false;
      c->model_configured = c->model_params_ready = c->model_data_ready = false;
      for (auto& v : c->plan_key) v = -1;
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
      std::vector<float> ch, bch;
      int64_t nf = 0, nb = 0;
      const bool with_bwd = true;  // H = 32: zero-padded 64-wide backward chunks
      mp_chunk_plan(H, K, c->M, with_bwd, [](bool, int64_t, int64_t, bool) {}, c->chunk_off, c->bchunk_off, nf, nb);
      ch.resize((size_t)nf);
      bch.resize((size_t)nb);
      mp_chunk_plan(
          H, K, c->M, with_bwd,
          [&](bool fwd, int64_t pos, int64_t src, bool lo) {
            const float w = src < 0 ? 0.f : p[(size_t)src];  // src -1: zero padding
            const float hi = tf32_rna_host(w);
            (fwd ? ch : bch)[(size_t)pos] = lo ? tf32_rna_host(w - hi) : hi;
          },
          c->chunk_off, c->bchunk_off, nf, nb);
      c->chunks.upload(ch.data(), nf, c->stream);
      c->bchunks.upload(bch.data(), nb, c->stream);
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
    if (e_out && c->lean) fail(HGNN_ERR_SIZE, "hgnn_mp_forward: e_out is not materialised under the memory-lean plan");
    rows_to_device(c, x0, c->rows * c->H, c->xs[0]->p);
    edges_to_device(c, e0, c->es[0]->p);
    run_forward(c);
    if (x_out) rows_to_host(c, x_buf(c, c->M), c->rows * c->H, x_out);
    if (e_out) edges_to_host(c, e_buf(c, c->M), e_out);
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
}

int hgnn_mp_backward(hgnn_ctx* c, const double* dx, const double* de, double* dx0, double* de0, double* grads) {
  return guarded([&] {
    bind(c);
    require_ready(c);
    if (!dx) fail(HGNN_ERR_SHAPE, "hgnn_mp_backward: null output adjoint");
    ensure_buffers(c);
    if (de && c->lean) fail(HGNN_ERR_SIZE, "hgnn_mp_backward: de (adjoint of e_M) needs the standard memory plan");
    rows_to_device(c, dx, c->rows * c->H, c->dx.p);
    if (!c->lean) {
      if (de) edges_to_device(c, de, c->de.p);
      else CUDA_OK(cudaMemsetAsync(c->de.p, 0, sizeof(float) * (size_t)(c->ne * c->H), c->stream));
    }
    run_backward(c);
    if (dx0) rows_to_host(c, c->dx.p, c->rows * c->H, dx0);
    if (de0) edges_to_host(c, de_out_buf(c, 0), de0);
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
      case HGNN_TRACE_X_IN: rows_to_host(c, x_buf(c, layer), c->rows * c->H, out); break;
      case HGNN_TRACE_E_IN: edges_to_host(c, e_buf(c, layer), out); break;
      case HGNN_TRACE_A_SYNC: rows_to_host(c, c->as[(size_t)layer]->p, c->rows * c->H, out); break;
      case HGNN_TRACE_X_OUT: rows_to_host(c, x_buf(c, layer + 1), c->rows * c->H, out); break;
      case HGNN_TRACE_E_OUT:
        if (!e_buf(c, layer + 1)) fail(HGNN_ERR_SIZE, "e_out of the last layer is not stored (memory-lean plan)");
        edges_to_host(c, e_buf(c, layer + 1), out);
        break;
      default: fail(HGNN_ERR_CONFIG, "unknown trace selector");
    }
  });
}

}  // extern "C"

namespace hgnn_b200::engine {
// Seeded device inputs keyed by global id; what the lean plan's backward
// consumes (e_0 storage, the dx seed) is re-created by step_device.
void synth_edges_in(hgnn_ctx* c) {
  if (c->ne == 0) return;
  synth_edges_kernel<<<blocks_for(c->ne * c->H), kEwThreads, 0, c->stream>>>(
      c->gid.p, c->src.p, c->dst.p, c->ne, (int)c->H, c->synth_seed ^ 0x5bd1e995ull, c->es[0]->p);
  check_launch(c);
}
void synth_dx_seed(hgnn_ctx* c, float* dst) {
  synth_rows_kernel<<<blocks_for(c->rows * c->H), kEwThreads, 0, c->stream>>>(
      c->gid.p, c->rows, c->nl, (int)c->H, c->synth_seed ^ 0xc2b2ae35ull, 1e-3f, dst);
  check_launch(c);
}
}  // namespace hgnn_b200::engine

extern "C" {

int hgnn_synthetic_inputs(hgnn_ctx* c, uint64_t seed) {
  return guarded([&] {
    bind(c);
    require_ready(c);
    ensure_buffers(c);
    const int64_t H = c->H;
    c->synth_seed = seed;
    synth_rows_kernel<<<blocks_for(c->rows * H), kEwThreads, 0, c->stream>>>(c->gid.p, c->rows, c->nl, (int)H, seed,
                                                                            1.0f, c->xs[0]->p);
    check_launch(c);
    synth_edges_in(c);
    if (!c->lean) synth_dx_seed(c, c->dx_in.p);
    c->synth_valid = true;
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
}

int hgnn_set_inputs(hgnn_ctx* c, const double* x0, const double* e0, const double* dx) {
  return guarded([&] {
    bind(c);
    require_ready(c);
    ensure_buffers(c);
    if (c->lean) fail(HGNN_ERR_SIZE, "hgnn_set_inputs needs the standard memory plan (use hgnn_synthetic_inputs)");
    rows_to_device(c, x0, c->rows * c->H, c->xs[0]->p);
    edges_to_device(c, e0, c->es[0]->p);
    rows_to_device(c, dx, c->rows * c->H, c->dx_in.p);
    c->synth_valid = false;
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
}

int hgnn_mp_step_device(hgnn_ctx* c) {
  return guarded([&] {
    bind(c);
    require_ready(c);
    ensure_buffers(c);
    if (c->lean) {  // the previous backward wrote de_0 over e_0: re-create the inputs
      if (!c->synth_valid) fail(HGNN_ERR_UNINITIALIZED, "memory-lean step_device needs hgnn_synthetic_inputs");
      synth_edges_in(c);
      run_forward(c);
      synth_dx_seed(c, c->dx.p);
      run_backward(c);
      return;
    }
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
    } else if (k == "halo_overlap") {
      if (value != 0 && value != 1) fail(HGNN_ERR_CONFIG, "halo_overlap: 0 (serial) or 1 (exchange overlapped)");
      c->halo_overlap = (int)value;
    } else if (k == "halo_sm_reserve") {
      if (value < 0 || value > 32) fail(HGNN_ERR_CONFIG, "halo_sm_reserve: 0..32 SMs");
      c->halo_sm_reserve = (int)value;
    } else if (k == "edge_factorized") {
      if (value != 0 && value != 1) fail(HGNN_ERR_CONFIG, "edge_factorized: 0 (3-segment edge kernels) or 1");
      c->edge_fact = (int)value;  // buffers follow at the next ensure_buffers (plan key)
    } else if (k == "memory_lean") {
      if (value < -1 || value > 1) fail(HGNN_ERR_CONFIG, "memory_lean: -1 (auto), 0 or 1");
      c->lean_opt = (int)value;
      for (auto& v : c->plan_key) v = -1;  // re-plan at the next call
    } else if (k == "collective_check") {
      if (value != 0 && value != 1) fail(HGNN_ERR_CONFIG, "collective_check: 0 or 1");
      c->coll_check = (int)value;
    } else if (k == "collective_timeout_ms") {
      if (value <= 0) fail(HGNN_ERR_CONFIG, "collective_timeout_ms must be positive");
      c->coll_timeout_ms = value;
      if (c->group) c->group->timeout_ms = value;
    } else if (k == "adjoint_presum") {
      if (value != 0 && value != 1) fail(HGNN_ERR_CONFIG, "adjoint_presum: 0 or 1");
      c->adj_presum = (int)value;
    } else if (k == "tma_gather") {
      if (value != 0 && value != 1) fail(HGNN_ERR_CONFIG, "tma_gather: 0 (per-thread row loads) or 1 (TMA gather4)");
      c->tma_gather = (int)value;
    } else if (k == "encoder_impl") {
      if (value != 0 && value != 1) fail(HGNN_ERR_CONFIG, "encoder_impl: 0 (simt) or 1 (tcgen05, H = 64)");
      c->enc_impl = (int)value;
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

}  // extern "C"
