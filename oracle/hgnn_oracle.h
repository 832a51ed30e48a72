/* oracle/hgnn_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, fp64 restatement of the reference's consistent neural message-
 * passing layer (arXiv 2410.01657; /root/reference/proj). Every function cites
 * the reference file:line it follows and reproduces its floating-point
 * operation order (compiled with -ffp-contract=off), so its results are
 * bitwise equal to the reference built in place (oracle/_ref). Parity is
 * pinned by tests/test_oracle.py against that build and against the golden
 * fixtures in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product path never does.
 */
#ifndef HGNN_ORACLE_H
#define HGNN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One rank's ReducedGraph + HaloMap (graph.hpp:16-65) as flat arrays.
 * send/recv/sync lists are CSR-flattened over neighbours / groups. */
typedef struct {
  int64_t num_local, num_halo, num_edges;
  const int32_t *edge_src, *edge_dst;          /* [num_edges] */
  const double *edge_inv;                      /* [num_edges] 1/d  (graph.cpp:231-255) */
  const int32_t *in_off, *in_edges;            /* CSR by receiver (graph.cpp:122-136) */
  const int32_t *out_off, *out_edges;          /* CSR by sender */
  int32_t num_nbr;
  const int32_t *nbr;                          /* ascending ranks */
  const int32_t *send_off, *send_rows;         /* [num_nbr+1], local rows, ascending gid */
  const int32_t *recv_off, *recv_rows;         /* [num_nbr+1], halo rows */
  int64_t num_sync;
  const int32_t *sync_local, *sync_off, *sync_slots; /* slots: -1 = own, else halo row */
} or_rank_graph;

enum { OR_MODE_NONE = 0, OR_MODE_A2A = 1, OR_MODE_NA2A = 2 }; /* comm.hpp:17 */

/* Processor-MLP parameter count: in->H, k x (H->H), H->H (nn.cpp:28-36). */
int64_t or_mlp_param_count(int64_t in_dim, int64_t H, int64_t k);

/* mlp_forward_rows for a processor MLP (nn.cpp:136-202; model.cpp:82-90).
 * params: w0,b0,...,w_{k+1},b_{k+1} flat in MlpParams::for_each order. */
void or_mlp_forward(const double* params, int64_t in_dim, int64_t H, int64_t k, int64_t rows,
                    const double* in, double* out);

/* mlp_backward_rows (nn.cpp:204-285): writes d_in, accumulates into grads. */
void or_mlp_backward(const double* params, int64_t in_dim, int64_t H, int64_t k, int64_t rows,
                     const double* in, const double* d_out, double* d_in, double* grads);

/* nmp_layer_forward (model.cpp:220-272) for R ranks in lock step.
 * layer_params = edge_update tensors then node_update tensors (model.cpp:131-132).
 * a_pre (nullable) receives the pre-exchange aggregate. */
void or_nmp_layer_forward(int R, int mode, const or_rank_graph* g, const double* layer_params, int64_t H,
                          int64_t k, const double* const* x, const double* const* e, double* const* x_out,
                          double* const* e_out, double* const* a_pre, double* const* a_sync);

/* nmp_layer_backward (model.cpp:318-387). dx (rows x H) and de (N_e x H) hold the
 * output adjoints on entry and the input adjoints on exit; grads accumulate. */
void or_nmp_layer_backward(int R, int mode, const or_rank_graph* g, const double* layer_params, int64_t H,
                           int64_t k, const double* const* x_in, const double* const* e_in,
                           const double* const* a_sync, double* const* dx, double* const* de,
                           double* const* grads);

/* halo_exchange / halo_exchange_adjoint (comm.cpp:281-357) on R ranks. */
void or_halo_exchange(int R, const or_rank_graph* g, int64_t width, double* const* values);
void or_halo_exchange_adjoint(int R, const or_rank_graph* g, int64_t width, double* const* adj);

/* Bytes one rank transmits in one exchange call (comm.cpp:127-153 accounting). */
int64_t or_exchange_bytes(int R, int mode, const or_rank_graph* g, int rank, int64_t width,
                          int64_t max_buffer_rows);

#ifdef __cplusplus
}
#endif
#endif
