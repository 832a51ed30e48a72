/* oracle/hgnn_oracle.c — TEST INFRASTRUCTURE ONLY (see hgnn_oracle.h).
 *
 * fp64 restatement of the reference hot path. Floating-point operation order
 * follows the cited reference loops exactly; build with -ffp-contract=off.
 * Row-at-a-time processing is equivalent to the reference's 16,384-row chunks
 * (nn.cpp:14) because every accumulation (matmul_tn_acc, colsum_acc) adds
 * rows in ascending order directly into its destination element.
 */
#include "hgnn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define LN_EPS 1e-12 /* kLayerNormEps, nn.hpp:65 */

int64_t or_mlp_param_count(int64_t in_dim, int64_t H, int64_t k) {
  return in_dim * H + H + k * (H * H + H) + H * H + H; /* nn.cpp:28-36, no skip / LN */
}

/* Parameter views: w0,b0,w1,b1,...,w_{k+1},b_{k+1} (nn.cpp:38-46). */
typedef struct {
  const double* w[64];
  const double* b[64];
} mlp_view;

static void view_params(const double* p, int64_t in_dim, int64_t H, int64_t k, mlp_view* v) {
  int64_t off = 0;
  for (int64_t l = 0; l < k + 2; ++l) {
    const int64_t rows = l == 0 ? in_dim : H;
    v->w[l] = p + off;
    off += rows * H;
    v->b[l] = p + off;
    off += H;
  }
}

/* matmul_nn row (kernels.cpp:15-26) + add_bias (kernels.cpp:52-57). */
static void linear_row(const double* x, const double* w, const double* b, int64_t kdim, int64_t m, double* y) {
  for (int64_t j = 0; j < m; ++j) y[j] = 0.0;
  for (int64_t t = 0; t < kdim; ++t) {
    const double av = x[t];
    const double* bt = w + t * m;
    for (int64_t j = 0; j < m; ++j) y[j] += av * bt[j];
  }
  for (int64_t j = 0; j < m; ++j) y[j] += b[j];
}

/* Parameter-free LN0 row (kernels.cpp:81-94 with gamma=1, beta=0) returning inv_std. */
static void ln0_row(const double* x, double* y, int64_t m) {
  double mean = 0.0;
  for (int64_t j = 0; j < m; ++j) mean += x[j];
  mean /= (double)m;
  double var = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double d = x[j] - mean;
    var += d * d;
  }
  var /= (double)m;
  const double inv_std = 1.0 / sqrt(var + LN_EPS);
  for (int64_t j = 0; j < m; ++j) y[j] = 1.0 * ((x[j] - mean) * inv_std) + 0.0;
}

/* layernorm_backward_row (kernels.cpp:97-124) with gamma = 1. */
static void ln0_backward_row(const double* x, const double* dy, double* dx, int64_t m) {
  double mean = 0.0;
  for (int64_t j = 0; j < m; ++j) mean += x[j];
  mean /= (double)m;
  double var = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double d = x[j] - mean;
    var += d * d;
  }
  var /= (double)m;
  const double inv_std = 1.0 / sqrt(var + LN_EPS);
  double g_mean = 0.0, gx_mean = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double xhat = (x[j] - mean) * inv_std;
    const double g = 1.0 * dy[j];
    g_mean += g;
    gx_mean += g * xhat;
  }
  g_mean /= (double)m;
  gx_mean /= (double)m;
  for (int64_t j = 0; j < m; ++j) {
    const double xhat = (x[j] - mean) * inv_std;
    dx[j] = (1.0 * dy[j] - g_mean - xhat * gx_mean) * inv_std;
  }
}

/* One row of chunk_forward (nn.cpp:136-188) for a processor MLP; keeps the
 * residual stream hidden[0..k] and pre-LN / normed values when asked. */
static void mlp_row_forward(const mlp_view* v, int64_t in_dim, int64_t H, int64_t k, const double* in,
                            double* out, double* hidden, double* pre, double* normed, double* scratch) {
  double* h = hidden ? hidden : scratch;            /* hidden[0] */
  double* u = scratch + H;
  double* t = scratch + 2 * H;
  linear_row(in, v->w[0], v->b[0], in_dim, H, h);
  for (int64_t j = 0; j < k; ++j) {
    double* hn = hidden ? hidden + (j + 1) * H : scratch + 3 * H;
    double* uj = pre ? pre + j * H : u;
    double* tj = normed ? normed + j * H : t;
    linear_row(h, v->w[1 + j], v->b[1 + j], H, H, uj);
    ln0_row(uj, tj, H);
    for (int64_t c = 0; c < H; ++c) hn[c] = tj[c] > 0.0 ? tj[c] : expm1(tj[c]); /* elu, kernels.cpp:63-66 */
    for (int64_t c = 0; c < H; ++c) hn[c] += h[c];                              /* add_inplace, nn.cpp:164 */
    if (!hidden) memcpy(scratch, hn, sizeof(double) * (size_t)H);
    h = hidden ? hn : scratch;
  }
  linear_row(h, v->w[k + 1], v->b[k + 1], H, H, out);
}

void or_mlp_forward(const double* params, int64_t in_dim, int64_t H, int64_t k, int64_t rows, const double* in,
                    double* out) {
  mlp_view v;
  view_params(params, in_dim, H, k, &v);
  double* scratch = (double*)malloc(sizeof(double) * (size_t)(4 * H));
  for (int64_t r = 0; r < rows; ++r)
    mlp_row_forward(&v, in_dim, H, k, in + r * in_dim, out + r * H, NULL, NULL, NULL, scratch);
  free(scratch);
}

/* grads layout equals params layout. */
void or_mlp_backward(const double* params, int64_t in_dim, int64_t H, int64_t k, int64_t rows, const double* in,
                     const double* d_out, double* d_in, double* grads) {
  mlp_view v, gv;
  view_params(params, in_dim, H, k, &v);
  view_params(grads, in_dim, H, k, &gv);
  double* hidden = (double*)malloc(sizeof(double) * (size_t)((k + 1) * H));
  double* pre = (double*)malloc(sizeof(double) * (size_t)((k + 1) * H));
  double* normed = (double*)malloc(sizeof(double) * (size_t)((k + 1) * H));
  double* scratch = (double*)malloc(sizeof(double) * (size_t)(8 * H + 2 * in_dim));
  double* y = scratch;
  double* d_h = scratch + H;
  double* d_t = scratch + 2 * H;
  double* d_u = scratch + 3 * H;
  double* d_prev = scratch + 4 * H;
  double* fwd_scratch = scratch + 5 * H; /* 4H not needed: hidden/pre/normed given */
  double* d_in_proj = scratch + 8 * H;
  for (int64_t r = 0; r < rows; ++r) {
    const double* x = in + r * in_dim;
    const double* dy = d_out + r * H;
    double* dxr = d_in + r * in_dim;
    mlp_row_forward(&v, in_dim, H, k, x, y, hidden, pre, normed, fwd_scratch); /* nn.cpp:226-227 */
    /* output projection (nn.cpp:241-245): matmul_tn_acc, colsum_acc, matmul_nt */
    double* gw = (double*)gv.w[k + 1];
    double* gb = (double*)gv.b[k + 1];
    const double* hk = hidden + k * H;
    for (int64_t i = 0; i < H; ++i)
      for (int64_t j = 0; j < H; ++j) gw[i * H + j] += hk[i] * dy[j];
    for (int64_t j = 0; j < H; ++j) gb[j] += dy[j];
    for (int64_t i = 0; i < H; ++i) {
      const double* wj = v.w[k + 1] + i * H;
      double s = 0.0;
      for (int64_t t = 0; t < H; ++t) s += dy[t] * wj[t];
      d_h[i] = s;
    }
    for (int64_t c = 0; c < in_dim; ++c) dxr[c] = 0.0; /* no skip projection (nn.cpp:252-254) */
    /* hidden blocks in reverse (nn.cpp:259-274) */
    for (int64_t j = k - 1; j >= 0; --j) {
      const double* nj = normed + j * H;
      for (int64_t c = 0; c < H; ++c) d_t[c] = 0.0;
      for (int64_t c = 0; c < H; ++c) d_t[c] += d_h[c] * (nj[c] > 0.0 ? 1.0 : exp(nj[c])); /* kernels.cpp:68-71 */
      ln0_backward_row(pre + j * H, d_t, d_u, H);
      double* gwj = (double*)gv.w[1 + j];
      double* gbj = (double*)gv.b[1 + j];
      const double* hj = hidden + j * H;
      for (int64_t i = 0; i < H; ++i)
        for (int64_t c = 0; c < H; ++c) gwj[i * H + c] += hj[i] * d_u[c];
      for (int64_t c = 0; c < H; ++c) gbj[c] += d_u[c];
      for (int64_t i = 0; i < H; ++i) {
        const double* wi = v.w[1 + j] + i * H;
        double s = 0.0;
        for (int64_t t = 0; t < H; ++t) s += d_u[t] * wi[t];
        d_prev[i] = s;
      }
      for (int64_t c = 0; c < H; ++c) d_prev[c] += d_h[c];
      memcpy(d_h, d_prev, sizeof(double) * (size_t)H);
    }
    /* input projection (nn.cpp:277-281) */
    double* gw0 = (double*)gv.w[0];
    double* gb0 = (double*)gv.b[0];
    for (int64_t i = 0; i < in_dim; ++i)
      for (int64_t c = 0; c < H; ++c) gw0[i * H + c] += x[i] * d_h[c];
    for (int64_t c = 0; c < H; ++c) gb0[c] += d_h[c];
    for (int64_t i = 0; i < in_dim; ++i) {
      const double* wi = v.w[0] + i * H;
      double s = 0.0;
      for (int64_t t = 0; t < H; ++t) s += d_h[t] * wi[t];
      d_in_proj[i] = s;
    }
    for (int64_t i = 0; i < in_dim; ++i) dxr[i] += d_in_proj[i];
  }
  free(hidden);
  free(pre);
  free(normed);
  free(scratch);
}

/* ------------------------------------------------------------------------- */
/* halo exchange (comm.cpp:281-357) on R in-process ranks                     */
/* ------------------------------------------------------------------------- */

/* index of rank `r` in the neighbour list of `g` (-1 if absent) */
static int nbr_index(const or_rank_graph* g, int r) {
  for (int n = 0; n < g->num_nbr; ++n)
    if (g->nbr[n] == r) return n;
  return -1;
}

void or_halo_exchange(int R, const or_rank_graph* g, int64_t width, double* const* values) {
  /* pack every rank's send buffers first (comm.cpp:287-296) */
  double** packed = (double**)calloc((size_t)R, sizeof(double*));
  for (int r = 0; r < R; ++r) {
    const int64_t ns = g[r].send_off[g[r].num_nbr];
    packed[r] = (double*)malloc(sizeof(double) * (size_t)(ns * width + 1));
    for (int64_t t = 0; t < ns; ++t)
      memcpy(packed[r] + t * width, values[r] + (int64_t)g[r].send_rows[t] * width, sizeof(double) * (size_t)width);
  }
  /* unpack into recv rows (comm.cpp:302-314) */
  for (int r = 0; r < R; ++r) {
    for (int n = 0; n < g[r].num_nbr; ++n) {
      const int s = g[r].nbr[n];
      const int back = nbr_index(&g[s], r);
      const double* buf = packed[s] + (int64_t)g[s].send_off[back] * width;
      for (int64_t t = g[r].recv_off[n]; t < g[r].recv_off[n + 1]; ++t)
        memcpy(values[r] + (int64_t)g[r].recv_rows[t] * width, buf + (t - g[r].recv_off[n]) * width,
               sizeof(double) * (size_t)width);
    }
  }
  for (int r = 0; r < R; ++r) free(packed[r]);
  free(packed);
}

void or_halo_exchange_adjoint(int R, const or_rank_graph* g, int64_t width, double* const* adj) {
  /* halo rows travel back to their owners (comm.cpp:323-337) */
  double** packed = (double**)calloc((size_t)R, sizeof(double*));
  for (int r = 0; r < R; ++r) {
    const int64_t nr = g[r].recv_off[g[r].num_nbr];
    packed[r] = (double*)malloc(sizeof(double) * (size_t)(nr * width + 1));
    for (int64_t t = 0; t < nr; ++t)
      memcpy(packed[r] + t * width, adj[r] + (int64_t)g[r].recv_rows[t] * width, sizeof(double) * (size_t)width);
  }
  for (int r = 0; r < R; ++r) {
    /* zero the halo rows (comm.cpp:340-342) */
    const int64_t nr = g[r].recv_off[g[r].num_nbr];
    for (int64_t t = 0; t < nr; ++t) memset(adj[r] + (int64_t)g[r].recv_rows[t] * width, 0, sizeof(double) * (size_t)width);
    /* accumulate in ascending neighbour order (comm.cpp:344-356) */
    for (int n = 0; n < g[r].num_nbr; ++n) {
      const int s = g[r].nbr[n];
      const int back = nbr_index(&g[s], r);
      const double* buf = packed[s] + (int64_t)g[s].recv_off[back] * width;
      for (int64_t t = g[r].send_off[n]; t < g[r].send_off[n + 1]; ++t) {
        double* dst = adj[r] + (int64_t)g[r].send_rows[t] * width;
        const double* src = buf + (t - g[r].send_off[n]) * width;
        for (int64_t c = 0; c < width; ++c) dst[c] += src[c];
      }
    }
  }
  for (int r = 0; r < R; ++r) free(packed[r]);
  free(packed);
}

int64_t or_exchange_bytes(int R, int mode, const or_rank_graph* g, int rank, int64_t width,
                          int64_t max_buffer_rows) {
  if (mode == OR_MODE_A2A) return (int64_t)R * max_buffer_rows * width * 8; /* comm.cpp:285-298 */
  (void)R;
  return (int64_t)g[rank].send_off[g[rank].num_nbr] * width * 8;
}

/* ------------------------------------------------------------------------- */
/* consistent NMP layer                                                      */
/* ------------------------------------------------------------------------- */

void or_nmp_layer_forward(int R, int mode, const or_rank_graph* g, const double* layer_params, int64_t H,
                          int64_t k, const double* const* x, const double* const* e, double* const* x_out,
                          double* const* e_out, double* const* a_pre, double* const* a_sync) {
  const double* edge_p = layer_params;
  const double* node_p = layer_params + or_mlp_param_count(3 * H, H, k);
  double** a = (double**)calloc((size_t)R, sizeof(double*));
  for (int r = 0; r < R; ++r) {
    const or_rank_graph* gr = &g[r];
    const int64_t rows = gr->num_local + gr->num_halo;
    /* edge update (model.cpp:233-235) with edge_concat_filler (model.cpp:184-195) */
    double* cat = (double*)malloc(sizeof(double) * (size_t)(gr->num_edges * 3 * H + 1));
    for (int64_t ed = 0; ed < gr->num_edges; ++ed) {
      memcpy(cat + ed * 3 * H, x[r] + (int64_t)gr->edge_src[ed] * H, sizeof(double) * (size_t)H);
      memcpy(cat + ed * 3 * H + H, x[r] + (int64_t)gr->edge_dst[ed] * H, sizeof(double) * (size_t)H);
      memcpy(cat + ed * 3 * H + 2 * H, e[r] + ed * H, sizeof(double) * (size_t)H);
    }
    or_mlp_forward(edge_p, 3 * H, H, k, gr->num_edges, cat, e_out[r]);
    free(cat);
    /* degree-scaled aggregation: scatter_rows_csr (kernels.cpp:174-186) */
    a[r] = (double*)malloc(sizeof(double) * (size_t)(rows * H + 1));
    for (int64_t i = 0; i < rows; ++i) {
      double* oi = a[r] + i * H;
      for (int64_t c = 0; c < H; ++c) oi[c] = 0.0;
      for (int32_t t = gr->in_off[i]; t < gr->in_off[i + 1]; ++t) {
        const int64_t ed = gr->in_edges[t];
        const double s = gr->edge_inv[ed];
        const double* re = e_out[r] + ed * H;
        for (int64_t c = 0; c < H; ++c) oi[c] += s * re[c];
      }
    }
  }
  /* halo exchange + synchronization (model.cpp:243-257) */
  if (mode != OR_MODE_NONE) or_halo_exchange(R, g, H, a);
  for (int r = 0; r < R; ++r) {
    const or_rank_graph* gr = &g[r];
    const int64_t rows = gr->num_local + gr->num_halo;
    if (a_pre) memcpy(a_pre[r], a[r], sizeof(double) * (size_t)(rows * H));
    memcpy(a_sync[r], a[r], sizeof(double) * (size_t)(rows * H));
    if (mode != OR_MODE_NONE) {
      for (int64_t grp = 0; grp < gr->num_sync; ++grp) {
        double* out = a_sync[r] + (int64_t)gr->sync_local[grp] * H;
        for (int64_t c = 0; c < H; ++c) out[c] = 0.0;
        for (int32_t s = gr->sync_off[grp]; s < gr->sync_off[grp + 1]; ++s) {
          const int32_t slot = gr->sync_slots[s];
          const double* src = slot < 0 ? a[r] + (int64_t)gr->sync_local[grp] * H : a[r] + (int64_t)slot * H;
          for (int64_t c = 0; c < H; ++c) out[c] += src[c];
        }
      }
    }
    /* node update on local rows (model.cpp:260-264), node_concat_filler (model.cpp:198-207) */
    double* cat = (double*)malloc(sizeof(double) * (size_t)(gr->num_local * 2 * H + 1));
    for (int64_t i = 0; i < gr->num_local; ++i) {
      memcpy(cat + i * 2 * H, a_sync[r] + i * H, sizeof(double) * (size_t)H);
      memcpy(cat + i * 2 * H + H, x[r] + i * H, sizeof(double) * (size_t)H);
    }
    memset(x_out[r], 0, sizeof(double) * (size_t)(rows * H));
    or_mlp_forward(node_p, 2 * H, H, k, gr->num_local, cat, x_out[r]);
    free(cat);
    free(a[r]);
  }
  free(a);
}

void or_nmp_layer_backward(int R, int mode, const or_rank_graph* g, const double* layer_params, int64_t H,
                           int64_t k, const double* const* x_in, const double* const* e_in,
                           const double* const* a_sync, double* const* dx, double* const* de,
                           double* const* grads) {
  const int64_t n_edge_p = or_mlp_param_count(3 * H, H, k);
  const double* edge_p = layer_params;
  const double* node_p = layer_params + n_edge_p;
  double** d_a = (double**)calloc((size_t)R, sizeof(double*));
  double** dx_node = (double**)calloc((size_t)R, sizeof(double*));
  for (int r = 0; r < R; ++r) {
    const or_rank_graph* gr = &g[r];
    const int64_t rows = gr->num_local + gr->num_halo;
    const int64_t nl = gr->num_local;
    /* node update backward (model.cpp:326-340) */
    double* cat = (double*)malloc(sizeof(double) * (size_t)(nl * 2 * H + 1));
    double* dcat = (double*)malloc(sizeof(double) * (size_t)(nl * 2 * H + 1));
    for (int64_t i = 0; i < nl; ++i) {
      memcpy(cat + i * 2 * H, a_sync[r] + i * H, sizeof(double) * (size_t)H);
      memcpy(cat + i * 2 * H + H, x_in[r] + i * H, sizeof(double) * (size_t)H);
    }
    or_mlp_backward(node_p, 2 * H, H, k, nl, cat, dx[r], dcat, grads[r] + n_edge_p);
    d_a[r] = (double*)calloc((size_t)(rows * H + 1), sizeof(double));
    dx_node[r] = (double*)malloc(sizeof(double) * (size_t)(nl * H + 1));
    for (int64_t i = 0; i < nl; ++i) {
      memcpy(d_a[r] + i * H, dcat + i * 2 * H, sizeof(double) * (size_t)H);
      memcpy(dx_node[r] + i * H, dcat + i * 2 * H + H, sizeof(double) * (size_t)H);
    }
    free(cat);
    free(dcat);
    /* synchronization adjoint (model.cpp:345-349) */
    if (mode != OR_MODE_NONE) {
      for (int64_t grp = 0; grp < gr->num_sync; ++grp) {
        const double* v = d_a[r] + (int64_t)gr->sync_local[grp] * H;
        for (int32_t s = gr->sync_off[grp]; s < gr->sync_off[grp + 1]; ++s)
          if (gr->sync_slots[s] >= 0) memcpy(d_a[r] + (int64_t)gr->sync_slots[s] * H, v, sizeof(double) * (size_t)H);
      }
    }
  }
  if (mode != OR_MODE_NONE) or_halo_exchange_adjoint(R, g, H, d_a); /* model.cpp:350 */
  for (int r = 0; r < R; ++r) {
    const or_rank_graph* gr = &g[r];
    const int64_t rows = gr->num_local + gr->num_halo;
    const int64_t ne = gr->num_edges;
    /* aggregation backward (model.cpp:354-360) */
    for (int64_t ed = 0; ed < ne; ++ed) {
      const double s = gr->edge_inv[ed];
      const double* src = d_a[r] + (int64_t)gr->edge_dst[ed] * H;
      double* dst = de[r] + ed * H;
      for (int64_t c = 0; c < H; ++c) dst[c] += s * src[c];
    }
    /* edge update backward (model.cpp:363-375) */
    double* cat = (double*)malloc(sizeof(double) * (size_t)(ne * 3 * H + 1));
    double* dcat = (double*)malloc(sizeof(double) * (size_t)(ne * 3 * H + 1));
    for (int64_t ed = 0; ed < ne; ++ed) {
      memcpy(cat + ed * 3 * H, x_in[r] + (int64_t)gr->edge_src[ed] * H, sizeof(double) * (size_t)H);
      memcpy(cat + ed * 3 * H + H, x_in[r] + (int64_t)gr->edge_dst[ed] * H, sizeof(double) * (size_t)H);
      memcpy(cat + ed * 3 * H + 2 * H, e_in[r] + ed * H, sizeof(double) * (size_t)H);
    }
    or_mlp_backward(edge_p, 3 * H, H, k, ne, cat, de[r], dcat, grads[r]);
    free(cat);
    for (int64_t ed = 0; ed < ne; ++ed) memcpy(de[r] + ed * H, dcat + ed * 3 * H + 2 * H, sizeof(double) * (size_t)H);
    /* input-node adjoint (model.cpp:378-386) */
    double* dx_prev = (double*)malloc(sizeof(double) * (size_t)(rows * H + 1));
    for (int64_t i = 0; i < rows; ++i) {
      double* oi = dx_prev + i * H;
      double tmp[4096];
      double* dd = H <= 4096 ? tmp : (double*)malloc(sizeof(double) * (size_t)H);
      for (int64_t c = 0; c < H; ++c) oi[c] = 0.0;
      for (int32_t t = gr->out_off[i]; t < gr->out_off[i + 1]; ++t) { /* scatter_rows_csr, scale=null */
        const double* re = dcat + (int64_t)gr->out_edges[t] * 3 * H;
        for (int64_t c = 0; c < H; ++c) oi[c] += 1.0 * re[c];
      }
      for (int64_t c = 0; c < H; ++c) dd[c] = 0.0;
      for (int32_t t = gr->in_off[i]; t < gr->in_off[i + 1]; ++t) {
        const double* re = dcat + (int64_t)gr->in_edges[t] * 3 * H + H;
        for (int64_t c = 0; c < H; ++c) dd[c] += 1.0 * re[c];
      }
      for (int64_t c = 0; c < H; ++c) oi[c] += dd[c];
      if (i < gr->num_local)
        for (int64_t c = 0; c < H; ++c) oi[c] += dx_node[r][i * H + c];
      if (dd != tmp) free(dd);
    }
    memcpy(dx[r], dx_prev, sizeof(double) * (size_t)(rows * H));
    free(dx_prev);
    free(dcat);
    free(d_a[r]);
    free(dx_node[r]);
  }
  free(d_a);
  free(dx_node);
}
