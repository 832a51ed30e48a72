// integration/binding_gpu_check.cpp — the reference's own gnn_forward /
// gnn_backward (model.cpp:278-430, compiled in place into oracle/_ref) against
// the SAME computation with the MP-layer loops routed through the binding
// (hgnn_b200_backend.hpp), wired exactly as INTEGRATION.md §2 shows:
//
//   encode (reference) -> MpStack::forward -> decode (reference)
//   decoder adjoint (reference) -> MpStack::backward -> encoder adjoints (reference)
//
// Checks, per the reference's metrics (fixtures.hpp:56-70, harness.cpp:201-212):
// decoder output and every a_sync trace within 5e-5, every gradient tensor
// within 2e-4, each normalised by the tensor's max |reference|; and that
// backward before forward throws UninitializedError (model.cpp:281-285).
//
// Test infrastructure: built here by oracle/Makefile (needs the reference
// headers), run on a B200 by tests/test_gpu_binding.py.
#include <cmath>
#include <cstdio>
#include <map>
#include <string>

#include "hgnn/harness.hpp"
#include "hgnn/mesh.hpp"
#include "hgnn/nn.hpp"
#include "hgnn_b200_backend.hpp"

namespace {

int failures = 0;

double rel(const hgnn::Tensor2D& a, const hgnn::Tensor2D& b) {
  double mag = 0.0, dev = 0.0;
  for (int64_t i = 0; i < b.size(); ++i) {
    mag = std::fmax(mag, std::fabs(b.data()[i]));
    dev = std::fmax(dev, std::fabs(a.data()[i] - b.data()[i]));
  }
  return dev / (mag > 0 ? mag : 1.0);
}

void expect_close(const hgnn::Tensor2D& a, const hgnn::Tensor2D& b, double tol, const std::string& what) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) {
    std::printf("FAIL %s: shape\n", what.c_str());
    ++failures;
    return;
  }
  const double r = rel(a, b);
  if (!(r < tol)) {
    std::printf("FAIL %s: rel %.3e >= %.1e\n", what.c_str(), r, tol);
    ++failures;
  }
}

void run_case(int64_t E, int64_t p, int64_t H, int64_t M, int64_t k) {
  using namespace hgnn;
  MeshConfig mc;
  mc.elements_per_axis = E;
  mc.poly_order = p;
  const Mesh mesh = build_box_mesh(mc);
  DistributedGraph dg = build_distributed_graph(mesh, verify_partition(mesh, 1));
  attach_tgv_features(dg, mc);
  const ReducedGraph& g = dg.graphs[0];
  const HaloMap& h = dg.halos[0];

  GnnConfig cfg;
  cfg.hidden_dim = H;
  cfg.num_mp_layers = M;
  cfg.mlp_hidden_layers = k;
  cfg.mode = ExchangeMode::None;  // one rank: comm may be null (model.hpp:92-95)
  const ModelParams params = init_params(cfg, 7);
  const std::string tag = "E" + std::to_string(E) + "p" + std::to_string(p) + "H" + std::to_string(H) + "M" +
                          std::to_string(M) + "k" + std::to_string(k);

  // The reference, end to end.
  ForwardTrace tr;
  const Tensor2D y_ref = gnn_forward(params, g, h, nullptr, &tr);
  Tensor2D d_out(y_ref.rows(), y_ref.cols());
  for (int64_t i = 0; i < d_out.size(); ++i) d_out.data()[i] = std::sin(0.37 * static_cast<double>(i)) + 0.1;
  ModelGrads g_ref = gnn_backward(params, g, h, nullptr, tr, d_out);

  // The same step with the MP layers on the GPU through the binding.
  b200::MpStack gpu(/*device=*/0, /*rank=*/0, /*num_ranks=*/1, nullptr);
  gpu.upload_graph(g, h);
  gpu.configure(cfg);
  gpu.upload_params(params);
  {
    const Tensor2D dx_probe(g.rows(), H);
    bool thrown = false;
    try {
      ModelGrads tmp = make_grads(params);
      gpu.backward(dx_probe, nullptr, tmp);
    } catch (const UninitializedError&) {
      thrown = true;
    }
    if (!thrown) {
      std::printf("FAIL %s: backward before forward did not throw UninitializedError\n", tag.c_str());
      ++failures;
    }
  }
  auto [x0, e0] = encode(params, g.node_features, g.edge_features);
  auto [x, e] = gpu.forward(x0, e0);
  const Tensor2D y = decode(params, x);  // R = 1: every row is local
  expect_close(y, y_ref, 5e-5, tag + " y");
  for (int64_t m = 0; m < M; ++m)
    expect_close(gpu.a_sync(static_cast<int>(m)), tr.layers[static_cast<size_t>(m)].a_sync, 5e-5,
                 tag + " a_sync[" + std::to_string(m) + "]");

  ModelGrads grads = make_grads(params);
  const Tensor2D dx = mlp_backward(params.node_decoder, x, d_out, grads.node_decoder);
  auto [dx0, de0] = gpu.backward(dx, nullptr, grads);
  mlp_backward(params.node_encoder, g.node_features, dx0, grads.node_encoder);
  mlp_backward(params.edge_encoder, g.edge_features, de0, grads.edge_encoder);

  std::map<std::string, const Tensor2D*> ref;
  g_ref.for_each([&](const std::string& name, Tensor2D& t) { ref[name] = &t; });
  int n = 0;
  grads.for_each([&](const std::string& name, Tensor2D& t) {
    ++n;
    expect_close(t, *ref.at(name), 2e-4, tag + " grad " + name);
  });
  std::printf("%s: %d gradient tensors compared\n", tag.c_str(), n);
}

}  // namespace

int main() {
  if (hgnn_device_count() == 0) {
    std::printf("binding_gpu_check: no GPU\n");
    return 2;
  }
  try {
    run_case(2, 3, 64, 2, 2);  // tensor-core kernels (H = 64)
    run_case(3, 2, 32, 2, 5);  // SIMT kernels (H = 32)
  } catch (const std::exception& ex) {
    std::printf("FAIL exception: %s\n", ex.what());
    ++failures;
  }
  std::printf(failures ? "binding_gpu_check: %d failure(s)\n" : "binding_gpu_check: OK\n", failures);
  return failures ? 1 : 0;
}
