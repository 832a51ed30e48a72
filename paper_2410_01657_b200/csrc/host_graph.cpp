// Analytic per-rank graph builder (host, C++).
//
// Produces exactly the ReducedGraph + HaloMap the reference builds with
// build_box_mesh -> partition_mesh -> build_distributed_graph
// (mesh.cpp:106-226, graph.cpp:40-265), but for ONE rank and without the
// global hash maps: on a structured GLL box every ownership question has a
// closed form in lattice coordinates, so each rank builds only its own
// sub-graph in O(local elements). Bit-exactness (node numbering, edge order,
// halo order, sync slots, degrees, CSR) is pinned against the reference in
// tests/test_graph_builder.py.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

#include "common.hpp"

namespace hgnn_b200 {

namespace {

thread_local std::string g_last_error;

// legendre + gll_points (mesh.cpp:23-69). Same arithmetic so the lattice
// positions are bitwise those of the reference.
void legendre(int64_t p, double x, double& value, double& deriv) {
  double p0 = 1.0, p1 = x;
  if (p == 0) {
    value = 1.0;
    deriv = 0.0;
    return;
  }
  for (int64_t n = 1; n < p; ++n) {
    const double p2 = ((2.0 * n + 1.0) * x * p1 - n * p0) / (n + 1.0);
    p0 = p1;
    p1 = p2;
  }
  value = p1;
  deriv = p * (p0 - x * p1) / (1.0 - x * x);
}

std::vector<double> gll_points(int64_t p) {
  std::vector<double> x(static_cast<size_t>(p + 1), 0.0);
  x.front() = -1.0;
  x.back() = 1.0;
  for (int64_t i = 1; i <= (p - 1) / 2; ++i) {
    double xi = -std::cos(M_PI * static_cast<double>(i) / static_cast<double>(p));
    for (int it = 0; it < 100; ++it) {
      double v, d;
      legendre(p, xi, v, d);
      const double dd = (2.0 * xi * d - static_cast<double>(p * (p + 1)) * v) / (1.0 - xi * xi);
      const double step = d / dd;
      xi -= step;
      if (std::abs(step) < 1e-14) break;
    }
    x[static_cast<size_t>(i)] = xi;
    x[static_cast<size_t>(p - i)] = -xi;
  }
  if (p % 2 == 0) x[static_cast<size_t>(p / 2)] = 0.0;
  return x;
}

}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

// balanced_factors (mesh.cpp:154-176): spread-minimising (a,b,c), ties to the
// lexicographically largest triple.
std::array<int64_t, 3> balanced_factors(int64_t R, int64_t E) {
  std::array<int64_t, 3> best{0, 0, 0};
  int64_t best_spread = -1;
  for (int64_t a = 1; a <= R; ++a) {
    if (R % a != 0 || E % a != 0) continue;
    const int64_t bc = R / a;
    for (int64_t b = 1; b <= bc; ++b) {
      if (bc % b != 0 || E % b != 0) continue;
      const int64_t c = bc / b;
      if (E % c != 0) continue;
      const int64_t spread = std::max({a, b, c}) - std::min({a, b, c});
      const std::array<int64_t, 3> cand{a, b, c};
      if (best_spread < 0 || spread < best_spread || (spread == best_spread && cand > best)) {
        best = cand;
        best_spread = spread;
      }
    }
  }
  if (best_spread < 0)
    fail(HGNN_ERR_PARTITION, "block partition: no factorization of R=" + std::to_string(R) +
                                 " with every factor dividing E=" + std::to_string(E));
  return best;
}

struct HostGraph {
  hgnn_graph_desc view{};
  std::vector<int64_t> global_ids;
  std::vector<double> positions;
  std::vector<int32_t> edge_src, edge_dst, node_degree, edge_degree;
  std::vector<double> node_inv, edge_inv;
  std::vector<int32_t> in_off, in_edges, out_off, out_edges;
  std::vector<int32_t> nbr, send_off, send_rows, recv_off, recv_rows, halo_to_local;
  std::vector<int32_t> sync_local, sync_off, sync_slots;
};

namespace {

// Block-partition geometry in lattice coordinates. Rank r owns the element box
// [b_a*per_a, (b_a+1)*per_a) per axis (mesh.cpp:207-217), i.e. the closed
// lattice interval [b_a*P_a, (b_a+1)*P_a] with P_a = per_a*p.
struct Geometry {
  int64_t E, p, R;
  std::array<int64_t, 3> f, per, span;  // factors, elements per block, lattice span P_a
  int64_t n1d;

  // Blocks along axis a whose closed lattice interval contains coordinate g,
  // ascending (one, or two on an interior block face).
  int candidates(int a, int64_t g, int64_t out[2]) const {
    int64_t b = std::min(g / span[a], f[a] - 1);
    if (g == b * span[a] && b > 0) {
      out[0] = b - 1;
      out[1] = b;
      return 2;
    }
    out[0] = b;
    return 1;
  }
  int32_t rank_of(int64_t bx, int64_t by, int64_t bz) const {
    return static_cast<int32_t>(bx + by * f[0] + bz * f[0] * f[1]);
  }
  // Owner ranks of a lattice point, ascending rank order (graph.cpp:504-518
  // builds the same list by scanning ranks in order).
  int owners(const int64_t g[3], int32_t out[8]) const {
    int64_t c[3][2];
    int n[3];
    for (int a = 0; a < 3; ++a) n[a] = candidates(a, g[a], c[a]);
    int k = 0;
    for (int iz = 0; iz < n[2]; ++iz)
      for (int iy = 0; iy < n[1]; ++iy)
        for (int ix = 0; ix < n[0]; ++ix) out[k++] = rank_of(c[0][ix], c[1][iy], c[2][iz]);
    return k;
  }
};

void finalize_view(HostGraph& hg) {
  hgnn_graph_desc& v = hg.view;
  v.global_ids = hg.global_ids.data();
  v.positions = hg.positions.data();
  v.edge_src = hg.edge_src.data();
  v.edge_dst = hg.edge_dst.data();
  v.node_degree = hg.node_degree.data();
  v.edge_degree = hg.edge_degree.data();
  v.node_inv_degree = hg.node_inv.data();
  v.edge_inv_degree = hg.edge_inv.data();
  v.in_offsets = hg.in_off.data();
  v.in_edges = hg.in_edges.data();
  v.out_offsets = hg.out_off.data();
  v.out_edges = hg.out_edges.data();
  v.num_neighbors = static_cast<int32_t>(hg.nbr.size());
  v.neighbors = hg.nbr.data();
  v.send_offsets = hg.send_off.data();
  v.send_rows = hg.send_rows.data();
  v.recv_offsets = hg.recv_off.data();
  v.recv_rows = hg.recv_rows.data();
  v.halo_to_local = hg.halo_to_local.data();
  v.num_sync_groups = static_cast<int64_t>(hg.sync_local.size());
  v.sync_local = hg.sync_local.data();
  v.sync_offsets = hg.sync_off.data();
  v.sync_slots = hg.sync_slots.data();
}

// In/out CSR by counting sort, ascending edge id per node (graph.cpp:122-136).
void build_csr(HostGraph& hg, int64_t rows) {
  const int64_t ne = static_cast<int64_t>(hg.edge_src.size());
  auto csr = [&](const std::vector<int32_t>& key, std::vector<int32_t>& off, std::vector<int32_t>& ids) {
    off.assign(static_cast<size_t>(rows + 1), 0);
    for (int64_t e = 0; e < ne; ++e) off[static_cast<size_t>(key[static_cast<size_t>(e)]) + 1]++;
    for (int64_t i = 0; i < rows; ++i) off[static_cast<size_t>(i + 1)] += off[static_cast<size_t>(i)];
    ids.resize(static_cast<size_t>(ne));
    std::vector<int32_t> cur(off.begin(), off.end() - 1);
    for (int64_t e = 0; e < ne; ++e) ids[static_cast<size_t>(cur[static_cast<size_t>(key[static_cast<size_t>(e)])]++)] = static_cast<int32_t>(e);
  };
  csr(hg.edge_dst, hg.in_off, hg.in_edges);
  csr(hg.edge_src, hg.out_off, hg.out_edges);
}

// dmin / dmax: MeshConfig::domain_min / domain_max (mesh.hpp, default the unit cube)
std::unique_ptr<HostGraph> build(int64_t E, int64_t p, int64_t R, int strategy, const int64_t* factors,
                                 int32_t rank, const double* dmin, const double* dmax) {
  if (E < 1) fail(HGNN_ERR_CONFIG, "MeshConfig: elements_per_axis must be >= 1");
  if (p < 1) fail(HGNN_ERR_CONFIG, "MeshConfig: poly_order must be >= 1");
  for (int a = 0; a < 3; ++a)  // MeshConfig::validate (mesh.cpp:12-14)
    if (!(dmax[a] > dmin[a])) fail(HGNN_ERR_CONFIG, "MeshConfig: domain_max must exceed domain_min on every axis");
  if (R < 1) fail(HGNN_ERR_PARTITION, "partition: rank count must be >= 1");
  if (rank < 0 || rank >= R) fail(HGNN_ERR_PARTITION, "assemble_rank_graph: rank out of range");
  const int64_t n1d = E * p + 1;
  if (n1d * n1d * n1d > (int64_t{1} << 62)) fail(HGNN_ERR_SIZE, "mesh too large");

  Geometry geo;
  geo.E = E;
  geo.p = p;
  geo.R = R;
  geo.n1d = n1d;
  if (strategy == HGNN_PART_VERIFY) strategy = R == 1 ? HGNN_PART_SLAB : HGNN_PART_BLOCK;
  if (strategy == HGNN_PART_SLAB) {
    if (E % R != 0)
      fail(HGNN_ERR_PARTITION, "slab partition: R=" + std::to_string(R) +
                                   " must divide elements_per_axis E=" + std::to_string(E) +
                                   " (R <= E along the split axis)");
    geo.f = {R, 1, 1};
  } else if (strategy == HGNN_PART_BLOCK) {
    if (factors) {
      if (factors[0] * factors[1] * factors[2] != R)
        fail(HGNN_ERR_PARTITION, "block partition: factors do not multiply to R=" + std::to_string(R));
      for (int a = 0; a < 3; ++a)
        if (factors[a] < 1 || E % factors[a] != 0)
          fail(HGNN_ERR_PARTITION, "block partition: factor " + std::to_string(factors[a]) +
                                       " does not divide elements_per_axis E=" + std::to_string(E));
      geo.f = {factors[0], factors[1], factors[2]};
    } else {
      geo.f = balanced_factors(R, E);
    }
  } else {
    fail(HGNN_ERR_CONFIG, "unknown partition strategy");
  }
  for (int a = 0; a < 3; ++a) {
    geo.per[a] = E / geo.f[a];
    geo.span[a] = geo.per[a] * p;
  }
  const int64_t bx = rank % geo.f[0];
  const int64_t by = (rank / geo.f[0]) % geo.f[1];
  const int64_t bz = rank / (geo.f[0] * geo.f[1]);
  const std::array<int64_t, 3> b{bx, by, bz};
  const std::array<int64_t, 3> lo{bx * geo.span[0], by * geo.span[1], bz * geo.span[2]};  // lattice origin
  const std::array<int64_t, 3> nb{geo.span[0] + 1, geo.span[1] + 1, geo.span[2] + 1};    // lattice box
  const int64_t q = p + 1;
  const int64_t box_points = nb[0] * nb[1] * nb[2];
  auto box_index = [&](int64_t gx, int64_t gy, int64_t gz) {
    return (gx - lo[0]) + nb[0] * ((gy - lo[1]) + nb[1] * (gz - lo[2]));
  };

  auto hg = std::make_unique<HostGraph>();
  hg->view.rank = rank;
  hg->view.num_ranks = static_cast<int32_t>(R);

  // ---- local nodes: first occurrence in ascending element order, lattice
  //      order inside the element (graph.cpp:66-92; element order is
  //      x-fastest, mesh.cpp:122-125).
  std::vector<int32_t> local_of(static_cast<size_t>(box_points), -1);
  std::vector<int64_t> local_box;  // box index per local node
  local_box.reserve(static_cast<size_t>(box_points));
  for (int64_t ez = b[2] * geo.per[2]; ez < (b[2] + 1) * geo.per[2]; ++ez)
    for (int64_t ey = b[1] * geo.per[1]; ey < (b[1] + 1) * geo.per[1]; ++ey)
      for (int64_t ex = b[0] * geo.per[0]; ex < (b[0] + 1) * geo.per[0]; ++ex)
        for (int64_t k = 0; k < q; ++k)
          for (int64_t j = 0; j < q; ++j)
            for (int64_t i = 0; i < q; ++i) {
              const int64_t bi = box_index(ex * p + i, ey * p + j, ez * p + k);
              if (local_of[static_cast<size_t>(bi)] < 0) {
                local_of[static_cast<size_t>(bi)] = static_cast<int32_t>(local_box.size());
                local_box.push_back(bi);
              }
            }
  const int64_t nl = static_cast<int64_t>(local_box.size());
  if (nl > INT32_MAX / 2) fail(HGNN_ERR_SIZE, "rank graph exceeds int32 indexing");
  auto coords = [&](int64_t bi, int64_t g[3]) {
    g[0] = lo[0] + bi % nb[0];
    g[1] = lo[1] + (bi / nb[0]) % nb[1];
    g[2] = lo[2] + bi / (nb[0] * nb[1]);
  };
  auto gid_of = [&](const int64_t g[3]) { return g[0] + g[1] * n1d + g[2] * n1d * n1d; };

  hg->global_ids.resize(static_cast<size_t>(nl));
  for (int64_t i = 0; i < nl; ++i) {
    int64_t g[3];
    coords(local_box[static_cast<size_t>(i)], g);
    hg->global_ids[static_cast<size_t>(i)] = gid_of(g);
  }

  // ---- directed edges: per element, element_edges order (graph.cpp:18-34),
  //      first occurrence of each unordered pair kept (graph.cpp:94-115).
  {
    std::vector<uint8_t> seen(static_cast<size_t>(box_points), 0);  // bit a: edge along axis a from this point
    const int64_t edge_cap = 3 * nl * 2;
    hg->edge_src.reserve(static_cast<size_t>(edge_cap));
    hg->edge_dst.reserve(static_cast<size_t>(edge_cap));
    const int64_t step[3] = {1, nb[0], nb[0] * nb[1]};
    for (int64_t ez = b[2] * geo.per[2]; ez < (b[2] + 1) * geo.per[2]; ++ez)
      for (int64_t ey = b[1] * geo.per[1]; ey < (b[1] + 1) * geo.per[1]; ++ey)
        for (int64_t ex = b[0] * geo.per[0]; ex < (b[0] + 1) * geo.per[0]; ++ex)
          for (int64_t k = 0; k < q; ++k)
            for (int64_t j = 0; j < q; ++j)
              for (int64_t i = 0; i < q; ++i) {
                const int64_t bi = box_index(ex * p + i, ey * p + j, ez * p + k);
                const bool has[3] = {i + 1 < q, j + 1 < q, k + 1 < q};
                for (int a = 0; a < 3; ++a) {
                  if (!has[a]) continue;
                  uint8_t& s = seen[static_cast<size_t>(bi)];
                  if (s & (1u << a)) continue;
                  s = static_cast<uint8_t>(s | (1u << a));
                  const int32_t u = local_of[static_cast<size_t>(bi)];
                  const int32_t v = local_of[static_cast<size_t>(bi + step[a])];
                  hg->edge_src.push_back(u);
                  hg->edge_dst.push_back(v);
                  hg->edge_src.push_back(v);
                  hg->edge_dst.push_back(u);
                }
              }
  }
  const int64_t ne = static_cast<int64_t>(hg->edge_src.size());

  // ---- ownership, degrees and shared lists (graph.cpp:527-539).
  hg->node_degree.assign(static_cast<size_t>(nl), 1);
  hg->node_inv.assign(static_cast<size_t>(nl), 1.0);
  std::vector<std::vector<std::pair<int64_t, int32_t>>> shared(static_cast<size_t>(R));
  std::vector<uint8_t> multi(static_cast<size_t>(nl), 0);
  for (int64_t i = 0; i < nl; ++i) {
    int64_t g[3];
    coords(local_box[static_cast<size_t>(i)], g);
    int32_t own[8];
    const int n = geo.owners(g, own);
    if (n < 2) continue;
    multi[static_cast<size_t>(i)] = 1;
    hg->node_degree[static_cast<size_t>(i)] = n;
    hg->node_inv[static_cast<size_t>(i)] = 1.0 / static_cast<double>(n);
    for (int t = 0; t < n; ++t)
      if (own[t] != rank) shared[static_cast<size_t>(own[t])].emplace_back(hg->global_ids[static_cast<size_t>(i)], static_cast<int32_t>(i));
  }

  // ---- halo rows ordered by (source rank, gid) (graph.cpp:541-561).
  int64_t next_row = nl;
  hg->send_off.push_back(0);
  hg->recv_off.push_back(0);
  std::vector<int64_t> nbr_base(static_cast<size_t>(R), -1);
  for (int64_t s = 0; s < R; ++s) {
    auto& list = shared[static_cast<size_t>(s)];
    if (list.empty()) continue;
    std::sort(list.begin(), list.end());
    hg->nbr.push_back(static_cast<int32_t>(s));
    nbr_base[static_cast<size_t>(s)] = next_row;
    for (const auto& [gid, local] : list) {
      hg->send_rows.push_back(local);
      hg->recv_rows.push_back(static_cast<int32_t>(next_row));
      hg->halo_to_local.push_back(local);
      hg->global_ids.push_back(gid);
      ++next_row;
    }
    hg->send_off.push_back(static_cast<int32_t>(hg->send_rows.size()));
    hg->recv_off.push_back(static_cast<int32_t>(hg->recv_rows.size()));
  }
  const int64_t nh = next_row - nl;
  const int64_t rows = nl + nh;

  // ---- positions (lattice_position, mesh.cpp:86-104) incl. mirrored halo rows.
  {
    const std::vector<double> gll = gll_points(p);
    hg->positions.resize(static_cast<size_t>(rows * 3));
    for (int64_t i = 0; i < nl; ++i) {
      int64_t g[3];
      coords(local_box[static_cast<size_t>(i)], g);
      for (int a = 0; a < 3; ++a) {
        int64_t elem = g[a] / p, loc = g[a] % p;
        if (elem == E) {
          elem = E - 1;
          loc = p;
        }
        const double h = (dmax[a] - dmin[a]) / static_cast<double>(E);
        hg->positions[static_cast<size_t>(i * 3 + a)] =
            dmin[a] + static_cast<double>(elem) * h + 0.5 * (gll[static_cast<size_t>(loc)] + 1.0) * h;
      }
    }
    for (int64_t hr = 0; hr < nh; ++hr) {
      const int32_t l = hg->halo_to_local[static_cast<size_t>(hr)];
      for (int a = 0; a < 3; ++a)
        hg->positions[static_cast<size_t>((nl + hr) * 3 + a)] = hg->positions[static_cast<size_t>(l * 3 + a)];
    }
  }

  // ---- sync groups: ascending owner rank, own slot = -1 (graph.cpp:573-587).
  hg->sync_off.push_back(0);
  for (int64_t i = 0; i < nl; ++i) {
    if (!multi[static_cast<size_t>(i)]) continue;
    int64_t g[3];
    coords(local_box[static_cast<size_t>(i)], g);
    int32_t own[8];
    const int n = geo.owners(g, own);
    const int64_t gid = hg->global_ids[static_cast<size_t>(i)];
    hg->sync_local.push_back(static_cast<int32_t>(i));
    for (int t = 0; t < n; ++t) {
      if (own[t] == rank) {
        hg->sync_slots.push_back(-1);
        continue;
      }
      const auto& list = shared[static_cast<size_t>(own[t])];
      const auto it = std::lower_bound(list.begin(), list.end(), std::make_pair(gid, INT32_MIN));
      hg->sync_slots.push_back(static_cast<int32_t>(nbr_base[static_cast<size_t>(own[t])] + (it - list.begin())));
    }
    hg->sync_off.push_back(static_cast<int32_t>(hg->sync_slots.size()));
  }

  // ---- edge degrees (graph.cpp:590-612): ranks owning an element that holds
  //      both endpoints. Along the edge axis the element is unique; along the
  //      other axes the closed-interval rule applies.
  hg->edge_degree.assign(static_cast<size_t>(ne), 1);
  hg->edge_inv.assign(static_cast<size_t>(ne), 1.0);
  for (int64_t e = 0; e < ne; e += 2) {
    int64_t ga[3], gb[3];
    coords(local_box[static_cast<size_t>(hg->edge_src[static_cast<size_t>(e)])], ga);
    coords(local_box[static_cast<size_t>(hg->edge_dst[static_cast<size_t>(e)])], gb);
    int d = 1;
    for (int a = 0; a < 3; ++a) {
      if (ga[a] != gb[a]) continue;  // edge axis: exactly one owning block
      int64_t c[2];
      d *= geo.candidates(a, ga[a], c);
    }
    hg->edge_degree[static_cast<size_t>(e)] = d;
    hg->edge_degree[static_cast<size_t>(e + 1)] = d;
    hg->edge_inv[static_cast<size_t>(e)] = 1.0 / static_cast<double>(d);
    hg->edge_inv[static_cast<size_t>(e + 1)] = 1.0 / static_cast<double>(d);
  }

  // ---- CSR by counting sort (graph.cpp:122-136).
  build_csr(*hg, rows);

  // ---- global max send-mask length (graph.cpp:616-621): the largest
  //      lattice-box intersection between two distinct ranks.
  int64_t max_rows = 0;
  for (int64_t r1 = 0; r1 < R; ++r1)
    for (int64_t r2 = 0; r2 < R; ++r2) {
      if (r1 == r2) continue;
      const int64_t c1[3] = {r1 % geo.f[0], (r1 / geo.f[0]) % geo.f[1], r1 / (geo.f[0] * geo.f[1])};
      const int64_t c2[3] = {r2 % geo.f[0], (r2 / geo.f[0]) % geo.f[1], r2 / (geo.f[0] * geo.f[1])};
      int64_t cnt = 1;
      for (int a = 0; a < 3; ++a) {
        const int64_t dlt = std::llabs(c1[a] - c2[a]);
        cnt *= dlt == 0 ? geo.span[a] + 1 : (dlt == 1 ? 1 : 0);
      }
      max_rows = std::max(max_rows, cnt);
    }

  hg->view.num_local = nl;
  hg->view.num_halo = nh;
  hg->view.num_edges = ne;
  hg->view.max_buffer_rows = max_rows;
  finalize_view(*hg);
  return hg;
}

// ---- HGNNGRB1 per-rank graph files (io.cpp:200-309). Little-endian:
//   "HGNNGRB1", i64 rank, num_local, num_halo, num_edges, F_x = 3, F_e = 7,
//   vec<i64> global_ids, vec<f64> positions (rows*3), vec<i32> edge_src,
//   edge_dst, node_degree, edge_degree, i64 n_nbr, n_nbr x {i32 neighbor,
//   vec<i32> send_mask, vec<i32> recv_mask}, vec<i32> halo_to_local,
//   i64 max_buffer_rows, i64 n_groups, n_groups x {i32 local, vec<i32> slots};
// vec<T> = i64 length + raw elements (io.cpp:47-74).
constexpr char kGraphMagic[8] = {'H', 'G', 'N', 'N', 'G', 'R', 'B', '1'};

struct FileWriter {
  std::FILE* f;
  std::string path;
  void raw(const void* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f) != n) fail(HGNN_ERR_IO, "cannot write " + path);
  }
  template <class T>
  void pod(T v) { raw(&v, sizeof(T)); }
  template <class T>
  void vec(const T* p, int64_t n) {
    pod<int64_t>(n);
    raw(p, sizeof(T) * static_cast<size_t>(n));
  }
};

struct FileReader {
  std::FILE* f;
  std::string path;
  int64_t left;  // bytes not yet consumed
  void raw(void* p, size_t n) {
    if (static_cast<int64_t>(n) > left || (n && std::fread(p, 1, n, f) != n))
      fail(HGNN_ERR_IO, path + ": truncated graph file");
    left -= static_cast<int64_t>(n);
  }
  template <class T>
  T pod() {
    T v{};
    raw(&v, sizeof(T));
    return v;
  }
  template <class T>
  std::vector<T> vec() {
    const int64_t n = pod<int64_t>();
    if (n < 0 || n > left / static_cast<int64_t>(sizeof(T))) fail(HGNN_ERR_IO, path + ": bad vector length");
    std::vector<T> v(static_cast<size_t>(n));
    raw(v.data(), sizeof(T) * v.size());
    return v;
  }
};

struct File {
  std::FILE* f;
  ~File() {
    if (f) std::fclose(f);
  }
};

void save_binary(const hgnn_graph_desc& g, const std::string& path) {
  File file{std::fopen(path.c_str(), "wb")};
  if (!file.f) fail(HGNN_ERR_IO, "cannot write " + path);
  FileWriter w{file.f, path};
  const int64_t rows = g.num_local + g.num_halo, ne = g.num_edges;
  w.raw(kGraphMagic, 8);
  w.pod<int64_t>(g.rank);
  w.pod<int64_t>(g.num_local);
  w.pod<int64_t>(g.num_halo);
  w.pod<int64_t>(ne);
  w.pod<int64_t>(3);  // F_x
  w.pod<int64_t>(7);  // F_e
  w.vec(g.global_ids, rows);
  w.vec(g.positions, rows * 3);
  w.vec(g.edge_src, ne);
  w.vec(g.edge_dst, ne);
  w.vec(g.node_degree, g.num_local);
  w.vec(g.edge_degree, ne);
  w.pod<int64_t>(g.num_neighbors);
  for (int32_t n = 0; n < g.num_neighbors; ++n) {
    w.pod<int32_t>(g.neighbors[n]);
    w.vec(g.send_rows + g.send_offsets[n], g.send_offsets[n + 1] - g.send_offsets[n]);
    w.vec(g.recv_rows + g.recv_offsets[n], g.recv_offsets[n + 1] - g.recv_offsets[n]);
  }
  w.vec(g.halo_to_local, g.num_halo);
  w.pod<int64_t>(g.max_buffer_rows);
  w.pod<int64_t>(g.num_sync_groups);
  for (int64_t t = 0; t < g.num_sync_groups; ++t) {
    w.pod<int32_t>(g.sync_local[t]);
    w.vec(g.sync_slots + g.sync_offsets[t], g.sync_offsets[t + 1] - g.sync_offsets[t]);
  }
  if (std::fflush(file.f) != 0) fail(HGNN_ERR_IO, "cannot write " + path);
}

void check_index(const std::vector<int32_t>& v, int64_t lo, int64_t hi, const std::string& what) {
  for (int32_t x : v)
    if (x < lo || x >= hi) fail(HGNN_ERR_IO, what + " index out of range");
}

std::unique_ptr<HostGraph> load_binary(const std::string& path) {
  File file{std::fopen(path.c_str(), "rb")};
  if (!file.f) fail(HGNN_ERR_IO, "cannot open " + path);
  std::fseek(file.f, 0, SEEK_END);
  const int64_t size = std::ftell(file.f);
  std::fseek(file.f, 0, SEEK_SET);
  FileReader in{file.f, path, size};
  char magic[8] = {};
  if (size < 8) fail(HGNN_ERR_IO, path + ": not an HGNNGRB1 graph file");
  in.raw(magic, 8);
  if (std::memcmp(magic, kGraphMagic, 8) != 0)
    fail(HGNN_ERR_IO, path + ": not an HGNNGRB1 graph file (JSON graph dumps are not supported)");
  auto hg = std::make_unique<HostGraph>();
  const int64_t rank = in.pod<int64_t>(), nl = in.pod<int64_t>(), nh = in.pod<int64_t>(), ne = in.pod<int64_t>();
  in.pod<int64_t>();  // F_x
  in.pod<int64_t>();  // F_e
  if (rank < 0 || nl < 0 || nh < 0 || ne < 0 || nl + nh >= (int64_t{1} << 31) || ne >= (int64_t{1} << 31))
    fail(HGNN_ERR_IO, path + ": bad header");
  const int64_t rows = nl + nh;
  hg->global_ids = in.vec<int64_t>();
  hg->positions = in.vec<double>();
  if (static_cast<int64_t>(hg->positions.size()) != rows * 3) fail(HGNN_ERR_IO, path + ": bad positions");
  hg->edge_src = in.vec<int32_t>();
  hg->edge_dst = in.vec<int32_t>();
  if (static_cast<int64_t>(hg->edge_src.size()) != ne || static_cast<int64_t>(hg->edge_dst.size()) != ne)
    fail(HGNN_ERR_IO, path + ": bad adjacency");
  hg->node_degree = in.vec<int32_t>();
  hg->edge_degree = in.vec<int32_t>();
  const int64_t n_nbr = in.pod<int64_t>();
  if (n_nbr < 0 || n_nbr > in.left / 20) fail(HGNN_ERR_IO, path + ": bad neighbour count");
  hg->send_off.push_back(0);
  hg->recv_off.push_back(0);
  for (int64_t n = 0; n < n_nbr; ++n) {
    hg->nbr.push_back(in.pod<int32_t>());
    const auto sm = in.vec<int32_t>(), rm = in.vec<int32_t>();
    hg->send_rows.insert(hg->send_rows.end(), sm.begin(), sm.end());
    hg->recv_rows.insert(hg->recv_rows.end(), rm.begin(), rm.end());
    hg->send_off.push_back(static_cast<int32_t>(hg->send_rows.size()));
    hg->recv_off.push_back(static_cast<int32_t>(hg->recv_rows.size()));
  }
  hg->halo_to_local = in.vec<int32_t>();
  const int64_t max_rows = in.pod<int64_t>();
  const int64_t n_groups = in.pod<int64_t>();
  if (n_groups < 0 || n_groups > in.left / 12) fail(HGNN_ERR_IO, path + ": bad sync-group count");
  hg->sync_off.push_back(0);
  for (int64_t t = 0; t < n_groups; ++t) {
    hg->sync_local.push_back(in.pod<int32_t>());
    const auto sl = in.vec<int32_t>();
    hg->sync_slots.insert(hg->sync_slots.end(), sl.begin(), sl.end());
    hg->sync_off.push_back(static_cast<int32_t>(hg->sync_slots.size()));
  }
  // The reference's checks (io.cpp:300-305), then the ones the device path
  // relies on: every index the kernels dereference is in range.
  if (static_cast<int64_t>(hg->global_ids.size()) != rows) fail(HGNN_ERR_IO, path + ": global_ids length mismatch");
  if (static_cast<int64_t>(hg->node_degree.size()) != nl) fail(HGNN_ERR_IO, path + ": node_degree length mismatch");
  if (static_cast<int64_t>(hg->edge_degree.size()) != ne) fail(HGNN_ERR_IO, path + ": edge_degree length mismatch");
  if (static_cast<int64_t>(hg->halo_to_local.size()) != nh) fail(HGNN_ERR_IO, path + ": halo_to_local length mismatch");
  check_index(hg->edge_src, 0, rows, path + ": edge_src");
  check_index(hg->edge_dst, 0, rows, path + ": edge_dst");
  check_index(hg->send_rows, 0, nl, path + ": send mask");
  check_index(hg->recv_rows, nl, rows, path + ": recv mask");
  check_index(hg->sync_local, 0, nl, path + ": sync group");
  for (int32_t x : hg->sync_slots)  // -1 = the local row itself, else a halo row (graph.cpp:203-228)
    if (x != -1 && (x < nl || x >= rows)) fail(HGNN_ERR_IO, path + ": sync slot index out of range");
  for (int32_t d : hg->node_degree)
    if (d < 1) fail(HGNN_ERR_IO, path + ": node_degree must be >= 1");
  for (int32_t d : hg->edge_degree)
    if (d < 1) fail(HGNN_ERR_IO, path + ": edge_degree must be >= 1");
  // finalize_loaded_graph (io.cpp:152-161): reciprocal degrees + CSR.
  hg->node_inv.resize(hg->node_degree.size());
  for (size_t i = 0; i < hg->node_degree.size(); ++i) hg->node_inv[i] = 1.0 / static_cast<double>(hg->node_degree[i]);
  hg->edge_inv.resize(hg->edge_degree.size());
  for (size_t i = 0; i < hg->edge_degree.size(); ++i) hg->edge_inv[i] = 1.0 / static_cast<double>(hg->edge_degree[i]);
  build_csr(*hg, rows);
  hg->view.rank = static_cast<int32_t>(rank);
  hg->view.num_ranks = 0;  // not stored in the file; the context carries the rank count
  hg->view.num_local = nl;
  hg->view.num_halo = nh;
  hg->view.num_edges = ne;
  hg->view.max_buffer_rows = max_rows;
  finalize_view(*hg);
  return hg;
}

}  // namespace
}  // namespace hgnn_b200

using namespace hgnn_b200;

struct hgnn_host_graph {
  std::unique_ptr<HostGraph> g;
};

extern "C" {

const char* hgnn_last_error(void) { return g_last_error.c_str(); }

int hgnn_graph_build_domain(int64_t E, int64_t p, int64_t R, int strategy, const int64_t* factors, int32_t rank,
                            const double* domain_min, const double* domain_max, hgnn_host_graph** out) {
  return guarded([&] {
    if (!out) fail(HGNN_ERR_CONFIG, "hgnn_graph_build: null output handle");
    static const double unit_min[3] = {0.0, 0.0, 0.0}, unit_max[3] = {1.0, 1.0, 1.0};
    auto h = std::make_unique<hgnn_host_graph>();
    h->g = build(E, p, R, strategy, factors, rank, domain_min ? domain_min : unit_min,
                 domain_max ? domain_max : unit_max);
    *out = h.release();
  });
}

int hgnn_graph_build(int64_t E, int64_t p, int64_t R, int strategy, const int64_t* factors, int32_t rank,
                     hgnn_host_graph** out) {
  return hgnn_graph_build_domain(E, p, R, strategy, factors, rank, nullptr, nullptr, out);
}

void hgnn_graph_free(hgnn_host_graph* g) { delete g; }

int hgnn_graph_view(const hgnn_host_graph* g, hgnn_graph_desc* out) {
  return guarded([&] {
    if (!g || !out) fail(HGNN_ERR_CONFIG, "hgnn_graph_view: null argument");
    *out = g->g->view;
  });
}

int hgnn_graph_save_binary(const hgnn_graph_desc* g, const char* path) {
  return guarded([&] {
    if (!g || !path) fail(HGNN_ERR_CONFIG, "hgnn_graph_save_binary: null argument");
    save_binary(*g, path);
  });
}

int hgnn_graph_load_binary(const char* path, hgnn_host_graph** out) {
  return guarded([&] {
    if (!path || !out) fail(HGNN_ERR_CONFIG, "hgnn_graph_load_binary: null argument");
    auto h = std::make_unique<hgnn_host_graph>();
    h->g = load_binary(path);
    *out = h.release();
  });
}

int hgnn_balanced_factors(int64_t R, int64_t E, int64_t out[3]) {
  return guarded([&] {
    const auto f = balanced_factors(R, E);
    out[0] = f[0];
    out[1] = f[1];
    out[2] = f[2];
  });
}

}  // extern "C"
