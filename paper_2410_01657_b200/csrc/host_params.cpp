// Seeded parameter initialisation in the reference layout (host, C++).
//
// init_params (model.cpp:105-122) draws, from one mt19937_64 stream, the node
// encoder, edge encoder, (edge_update, node_update) per MP layer and the
// decoder; make_mlp (nn.cpp:76-97) draws W then b per linear (Glorot-uniform,
// bias with the same bound, nn.cpp:65-72), then the skip projection. The
// uniform mapping is Rng::uniform (rng.hpp:17-20). The output vector is in
// ModelParams::for_each order (model.cpp:124-135, nn.cpp:38-46); bit-exact.
#include <cmath>
#include <random>
#include <vector>

#include "common.hpp"

namespace hgnn_b200 {
namespace {

struct Spec {
  int64_t in, out, hidden, k;
  bool skip, out_ln;
};

int64_t spec_count(const Spec& s) {
  int64_t n = s.in * s.hidden + s.hidden + s.k * (s.hidden * s.hidden + s.hidden) + s.hidden * s.out + s.out;
  if (s.skip) n += s.in * s.out;
  if (s.out_ln) n += 2 * s.out;
  return n;
}

std::vector<Spec> model_specs(int64_t H, int64_t M, int64_t k, int64_t in_node, int64_t in_edge, int64_t out_dim) {
  if (H < 1) fail(HGNN_ERR_CONFIG, "GnnConfig: hidden_dim must be >= 1");
  if (M < 0) fail(HGNN_ERR_CONFIG, "GnnConfig: num_mp_layers must be >= 0");
  if (k < 0) fail(HGNN_ERR_CONFIG, "GnnConfig: mlp_hidden_layers must be >= 0");
  if (in_node < 1 || in_edge < 1 || out_dim < 1) fail(HGNN_ERR_CONFIG, "GnnConfig: feature dimensions must be >= 1");
  std::vector<Spec> v;
  v.push_back({in_node, H, H, k, true, true});  // encoder_spec (model.cpp:70-80)
  v.push_back({in_edge, H, H, k, true, true});
  for (int64_t m = 0; m < M; ++m) {
    v.push_back({3 * H, H, H, k, false, false});  // processor_spec (model.cpp:82-90)
    v.push_back({2 * H, H, H, k, false, false});
  }
  v.push_back({H, out_dim, H, k, true, false});  // decoder_spec (model.cpp:92-101)
  return v;
}

struct Rng {
  std::mt19937_64 gen;
  explicit Rng(uint64_t seed) : gen(seed) {}
  double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + uniform() * (hi - lo); }
};

}  // namespace
}  // namespace hgnn_b200

using namespace hgnn_b200;

extern "C" {

int64_t hgnn_param_count(int64_t H, int64_t M, int64_t k, int64_t in_node, int64_t in_edge, int64_t out_dim) {
  int64_t n = -1;
  guarded([&] {
    n = 0;
    for (const Spec& s : model_specs(H, M, k, in_node, in_edge, out_dim)) n += spec_count(s);
  });
  return n;
}

int hgnn_mp_param_range(int64_t H, int64_t M, int64_t k, int64_t in_node, int64_t in_edge, int64_t* offset,
                        int64_t* count) {
  return guarded([&] {
    const auto specs = model_specs(H, M, k, in_node, in_edge, 1);
    *offset = spec_count(specs[0]) + spec_count(specs[1]);
    *count = 0;
    for (int64_t m = 0; m < 2 * M; ++m) *count += spec_count(specs[static_cast<size_t>(2 + m)]);
  });
}

int hgnn_init_params(int64_t H, int64_t M, int64_t k, int64_t in_node, int64_t in_edge, int64_t out_dim, uint64_t seed,
                     double* flat) {
  return guarded([&] {
    if (!flat) fail(HGNN_ERR_CONFIG, "hgnn_init_params: null output");
    Rng rng(seed);
    double* o = flat;
    auto draw = [&](int64_t rows, int64_t cols, double bound) {
      for (int64_t i = 0; i < rows * cols; ++i) *o++ = rng.uniform(-bound, bound);
    };
    for (const Spec& s : model_specs(H, M, k, in_node, in_edge, out_dim)) {
      auto linear = [&](int64_t in, int64_t out) {
        const double a = std::sqrt(6.0 / static_cast<double>(in + out));
        draw(in, out, a);  // weight (in x out)
        draw(1, out, a);   // bias, same bound
      };
      linear(s.in, s.hidden);
      for (int64_t j = 0; j < s.k; ++j) linear(s.hidden, s.hidden);
      linear(s.hidden, s.out);
      if (s.skip) draw(s.in, s.out, std::sqrt(6.0 / static_cast<double>(s.in + s.out)));
      if (s.out_ln) {
        for (int64_t j = 0; j < s.out; ++j) *o++ = 1.0;  // ln_g
        for (int64_t j = 0; j < s.out; ++j) *o++ = 0.0;  // ln_b
      }
    }
  });
}

}  // extern "C"
