// integration/hgnn_b200_backend.hpp — reference-side C++ binding of the
// B200 C-ABI (include/hgnn_b200.h).
//
// This header is meant to be compiled INSIDE the reference tree (it includes
// the reference's own hgnn/*.hpp). It is the code a maintainer adds to route
// the MP-layer loop of gnn_forward / gnn_backward through the GPU:
//
//   model.cpp:295-300  for m: nmp_layer_forward(...)   -> MpStack::forward
//   model.cpp:411-415  for m: nmp_layer_backward(...)  -> MpStack::backward
//
// Everything crossing the boundary is a plain pointer into the reference's own
// containers (Tensor2D row-major double, std::vector<int32_t>), so no copies
// are made on the host beyond flattening the per-neighbour halo masks and the
// sync groups into CSR arrays. Status codes are rethrown as the matching
// hgnn::Error subclass (error.hpp), so callers keep their exception handling.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "hgnn/error.hpp"
#include "hgnn/graph.hpp"
#include "hgnn/model.hpp"
#include "hgnn_b200.h"

namespace hgnn::b200 {

// Status code -> reference exception type (include/hgnn_b200.h status table).
inline void check(int status, const char* where) {
  if (status == HGNN_OK) return;
  const std::string msg = std::string(where) + ": " + hgnn_last_error();
  switch (status) {
    case HGNN_ERR_SHAPE: throw ShapeError(msg);
    case HGNN_ERR_CONFIG: throw ConfigError(msg);
    case HGNN_ERR_PARTITION: throw PartitionError(msg);
    case HGNN_ERR_COLLECTIVE: throw CollectiveError(msg);
    case HGNN_ERR_INTEGRITY: throw IntegrityError(msg);
    case HGNN_ERR_UNINITIALIZED: throw UninitializedError(msg);
    case HGNN_ERR_SIZE: throw SizeError(msg);
    case HGNN_ERR_OPTIMIZER: throw OptimizerError(msg);
    case HGNN_ERR_IO: throw IoError(msg);
    default: throw Error(msg);  // device / NCCL / internal failures
  }
}

inline int mode_code(ExchangeMode m) {
  switch (m) {
    case ExchangeMode::None: return HGNN_MODE_NONE;
    case ExchangeMode::AllToAll: return HGNN_MODE_A2A;
    case ExchangeMode::NeighborAllToAll: return HGNN_MODE_NA2A;
  }
  return HGNN_MODE_NONE;
}

// One rank's ReducedGraph + HaloMap as an hgnn_graph_desc (graph.hpp:16-65).
// Owns only the flattened halo / sync arrays; the rest points into `g`.
class GraphDesc {
 public:
  GraphDesc(const ReducedGraph& g, const HaloMap& h) {
    send_off_.push_back(0);
    recv_off_.push_back(0);
    for (size_t n = 0; n < h.neighbors.size(); ++n) {
      send_rows_.insert(send_rows_.end(), h.send_masks[n].begin(), h.send_masks[n].end());
      recv_rows_.insert(recv_rows_.end(), h.recv_masks[n].begin(), h.recv_masks[n].end());
      send_off_.push_back(static_cast<int32_t>(send_rows_.size()));
      recv_off_.push_back(static_cast<int32_t>(recv_rows_.size()));
    }
    sync_off_.push_back(0);
    for (const auto& s : h.sync_groups) {
      sync_local_.push_back(s.local_node);
      sync_slots_.insert(sync_slots_.end(), s.slots.begin(), s.slots.end());
      sync_off_.push_back(static_cast<int32_t>(sync_slots_.size()));
    }
    d_.rank = g.rank;
    d_.num_ranks = 0;  // informational; the context carries the rank count
    d_.num_local = g.num_local;
    d_.num_halo = g.num_halo;
    d_.num_edges = g.num_edges();
    d_.global_ids = g.global_ids.data();
    d_.positions = g.positions.data();
    d_.edge_src = g.edge_src.data();
    d_.edge_dst = g.edge_dst.data();
    d_.node_degree = g.node_degree.data();
    d_.edge_degree = g.edge_degree.data();
    d_.node_inv_degree = g.node_inv_degree.data();
    d_.edge_inv_degree = g.edge_inv_degree.data();
    d_.in_offsets = g.in_offsets.data();
    d_.in_edges = g.in_edges.data();
    d_.out_offsets = g.out_offsets.data();
    d_.out_edges = g.out_edges.data();
    d_.num_neighbors = static_cast<int32_t>(h.neighbors.size());
    d_.neighbors = h.neighbors.data();
    d_.send_offsets = send_off_.data();
    d_.send_rows = send_rows_.data();
    d_.recv_offsets = recv_off_.data();
    d_.recv_rows = recv_rows_.data();
    d_.halo_to_local = h.halo_to_local.data();
    d_.num_sync_groups = static_cast<int64_t>(h.sync_groups.size());
    d_.sync_local = sync_local_.data();
    d_.sync_offsets = sync_off_.data();
    d_.sync_slots = sync_slots_.data();
    d_.max_buffer_rows = h.max_buffer_rows;
  }
  const hgnn_graph_desc* get() const { return &d_; }

 private:
  hgnn_graph_desc d_{};
  std::vector<int32_t> send_off_, send_rows_, recv_off_, recv_rows_, sync_local_, sync_off_, sync_slots_;
};

// The M message-passing layers of one rank on one GPU (one per RankComm body,
// comm.cpp:74-89). Collective across ranks when mode != None: every rank calls
// forward / backward in the same order, exactly as with RankComm.
class MpStack {
 public:
  // nccl_uid: 128 bytes from hgnn_nccl_unique_id() on rank 0, broadcast by the
  // caller (nullptr when num_ranks == 1).
  MpStack(int device, int32_t rank, int32_t num_ranks, const uint8_t* nccl_uid) {
    check(hgnn_ctx_create(device, rank, num_ranks, nccl_uid, &ctx_), "hgnn_ctx_create");
  }
  ~MpStack() {
    if (ctx_) hgnn_ctx_destroy(ctx_);
  }
  MpStack(const MpStack&) = delete;
  MpStack& operator=(const MpStack&) = delete;

  void upload_graph(const ReducedGraph& g, const HaloMap& h) {
    GraphDesc d(g, h);
    check(hgnn_graph_upload(ctx_, d.get()), "hgnn_graph_upload");
    rows_ = g.rows();
    edges_ = g.num_edges();
  }

  // GnnConfig (model.hpp:19-27): hidden, M, k and the exchange mode.
  void configure(const GnnConfig& c) {
    check(hgnn_configure(ctx_, c.hidden_dim, c.num_mp_layers, c.mlp_hidden_layers, mode_code(c.mode)),
          "hgnn_configure");
    hidden_ = c.hidden_dim;
    layers_ = c.num_mp_layers;
  }

  // MP-layer block of ModelParams::for_each (model.cpp:124-135), in order.
  void upload_params(const ModelParams& p) {
    std::vector<double> flat;
    p.for_each([&](const std::string& name, const Tensor2D& t) {
      if (name.rfind("layer", 0) == 0) flat.insert(flat.end(), t.data(), t.data() + t.size());
    });
    check(hgnn_params_upload(ctx_, flat.data(), static_cast<int64_t>(flat.size())), "hgnn_params_upload");
  }

  // gnn_forward's layer loop (model.cpp:295-300): encoder outputs in, layer
  // M-1 outputs (x, e) out. Layer traces stay on the device for backward.
  std::pair<Tensor2D, Tensor2D> forward(const Tensor2D& x0, const Tensor2D& e0) {
    shape(x0, rows_, "x0");
    shape(e0, edges_, "e0");
    Tensor2D x(rows_, hidden_), e(edges_, hidden_);
    check(hgnn_mp_forward(ctx_, x0.data(), e0.data(), x.data(), e.data()), "hgnn_mp_forward");
    return {std::move(x), std::move(e)};
  }

  // gnn_backward's layer loop (model.cpp:411-415): adjoints of the last
  // layer's outputs in (de may be null = zeros, model.cpp:412), adjoints of the
  // encoder outputs out; the MP-layer gradients are written into `grads`
  // (rank-local, before the AllReduce average of model.cpp:520-527).
  std::pair<Tensor2D, Tensor2D> backward(const Tensor2D& dx, const Tensor2D* de, ModelGrads& grads) {
    shape(dx, rows_, "dx");
    if (de) shape(*de, edges_, "de");
    Tensor2D dx0(rows_, hidden_), de0(edges_, hidden_);
    std::vector<double> flat;
    grads.for_each([&](const std::string& name, Tensor2D& t) {
      if (name.rfind("layer", 0) == 0) flat.resize(flat.size() + static_cast<size_t>(t.size()));
    });
    check(hgnn_mp_backward(ctx_, dx.data(), de ? de->data() : nullptr, dx0.data(), de0.data(), flat.data()),
          "hgnn_mp_backward");
    size_t off = 0;
    grads.for_each([&](const std::string& name, Tensor2D& t) {
      if (name.rfind("layer", 0) != 0) return;
      for (int64_t i = 0; i < t.size(); ++i) t.data()[i] += flat[off + static_cast<size_t>(i)];
      off += static_cast<size_t>(t.size());
    });
    return {std::move(dx0), std::move(de0)};
  }

  // NmpLayerTrace::a_sync of layer m (read by test_model.cpp:119-127).
  Tensor2D a_sync(int layer) const {
    Tensor2D a(rows_, hidden_);
    check(hgnn_get_trace(ctx_, layer, HGNN_TRACE_A_SYNC, a.data()), "hgnn_get_trace");
    return a;
  }

 private:
  void shape(const Tensor2D& t, int64_t rows, const char* what) const {
    if (t.rows() != rows || t.cols() != hidden_)
      throw ShapeError(std::string("MpStack: ") + what + " has shape " + std::to_string(t.rows()) + "x" +
                       std::to_string(t.cols()) + ", expected " + std::to_string(rows) + "x" +
                       std::to_string(hidden_));
  }

  hgnn_ctx* ctx_ = nullptr;
  int64_t rows_ = 0, edges_ = 0, hidden_ = 0, layers_ = 0;
};

}  // namespace hgnn::b200
