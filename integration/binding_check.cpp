// integration/binding_check.cpp — compiles the reference-side binding
// (hgnn_b200_backend.hpp) against the reference's own headers and checks the
// host half of the boundary without a GPU:
//   1. GraphDesc built from the REFERENCE's ReducedGraph/HaloMap (graph.cpp
//      builder, linked from oracle/_ref) equals, array for array, the
//      descriptor of our own host builder (hgnn_graph_build / hgnn_graph_view);
//   2. status codes surface as the matching hgnn::Error subclasses;
//   3. MpStack on a machine without a GPU fails loudly (hgnn::Error), never
//      silently on the CPU.
// Built and run by tests/test_integration_binding.py (CPU suite).
#include <cstdio>
#include <cstring>
#include <typeinfo>

#include "hgnn/mesh.hpp"
#include "hgnn_b200_backend.hpp"

namespace {

int failures = 0;

template <class T>
bool same(const T* a, const T* b, int64_t n) {
  if (n == 0) return true;
  if (!a || !b) return false;
  return std::memcmp(a, b, sizeof(T) * static_cast<size_t>(n)) == 0;
}

void expect(bool ok, const char* what) {
  if (!ok) {
    std::printf("FAIL %s\n", what);
    ++failures;
  }
}

template <class E>
void expect_throw(int status, const char* what) {
  try {
    hgnn::b200::check(status, what);
    std::printf("FAIL %s: no exception\n", what);
    ++failures;
  } catch (const E&) {
  } catch (const std::exception& ex) {
    std::printf("FAIL %s: wrong exception %s\n", what, typeid(ex).name());
    ++failures;
  }
}

}  // namespace

int main() {
  using namespace hgnn;
  const int64_t E = 4, p = 3, R = 4;
  MeshConfig mc;
  mc.elements_per_axis = E;
  mc.poly_order = p;
  const Mesh mesh = build_box_mesh(mc);
  const PartitionMap part = partition_mesh(mesh, R, PartitionStrategy::Block);
  const DistributedGraph dg = build_distributed_graph(mesh, part);

  for (int32_t r = 0; r < R; ++r) {
    const ReducedGraph& g = dg.graphs[static_cast<size_t>(r)];
    const HaloMap& h = dg.halos[static_cast<size_t>(r)];
    b200::GraphDesc ref(g, h);
    const hgnn_graph_desc& a = *ref.get();

    hgnn_host_graph* ours = nullptr;
    b200::check(hgnn_graph_build(E, p, R, HGNN_PART_BLOCK, nullptr, r, &ours), "hgnn_graph_build");
    hgnn_graph_desc b{};
    b200::check(hgnn_graph_view(ours, &b), "hgnn_graph_view");

    const int64_t rows = a.num_local + a.num_halo, ne = a.num_edges;
    expect(a.num_local == b.num_local && a.num_halo == b.num_halo && ne == b.num_edges, "sizes");
    expect(same(a.global_ids, b.global_ids, rows), "global_ids");
    expect(same(a.edge_src, b.edge_src, ne) && same(a.edge_dst, b.edge_dst, ne), "edges");
    expect(same(a.edge_inv_degree, b.edge_inv_degree, ne), "edge_inv_degree");
    expect(same(a.in_offsets, b.in_offsets, rows + 1) && same(a.in_edges, b.in_edges, ne), "in-CSR");
    expect(a.num_neighbors == b.num_neighbors && same(a.neighbors, b.neighbors, a.num_neighbors), "neighbors");
    expect(same(a.send_offsets, b.send_offsets, a.num_neighbors + 1) &&
               same(a.send_rows, b.send_rows, a.send_offsets[a.num_neighbors]),
           "send masks");
    expect(same(a.recv_offsets, b.recv_offsets, a.num_neighbors + 1) &&
               same(a.recv_rows, b.recv_rows, a.recv_offsets[a.num_neighbors]),
           "recv masks");
    expect(a.num_sync_groups == b.num_sync_groups && same(a.sync_local, b.sync_local, a.num_sync_groups) &&
               same(a.sync_offsets, b.sync_offsets, a.num_sync_groups + 1) &&
               same(a.sync_slots, b.sync_slots, a.sync_offsets[a.num_sync_groups]),
           "sync groups");
    expect(a.max_buffer_rows == b.max_buffer_rows, "max_buffer_rows");
    hgnn_graph_free(ours);
  }

  expect_throw<ShapeError>(HGNN_ERR_SHAPE, "shape");
  expect_throw<ConfigError>(HGNN_ERR_CONFIG, "config");
  expect_throw<PartitionError>(HGNN_ERR_PARTITION, "partition");
  expect_throw<CollectiveError>(HGNN_ERR_COLLECTIVE, "collective");
  expect_throw<UninitializedError>(HGNN_ERR_UNINITIALIZED, "uninitialized");
  expect_throw<OptimizerError>(HGNN_ERR_OPTIMIZER, "optimizer");
  expect_throw<IoError>(HGNN_ERR_IO, "io");
  expect_throw<Error>(HGNN_ERR_CUDA, "cuda");
  try {  // a bad partition request reaches the caller as PartitionError
    hgnn_host_graph* g = nullptr;
    b200::check(hgnn_graph_build(3, 2, 7, HGNN_PART_BLOCK, nullptr, 0, &g), "hgnn_graph_build");
    std::printf("FAIL infeasible partition accepted\n");
    ++failures;
  } catch (const PartitionError&) {
  }

  if (hgnn_device_count() == 0) {  // CPU machine: the device path must refuse loudly
    try {
      b200::MpStack s(0, 0, 1, nullptr);
      std::printf("FAIL MpStack constructed without a GPU\n");
      ++failures;
    } catch (const Error&) {
    }
  }
  std::printf(failures ? "binding_check: %d failure(s)\n" : "binding_check: OK\n", failures);
  return failures ? 1 : 0;
}
