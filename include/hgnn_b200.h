/* include/hgnn_b200.h — C-ABI of the B200-native consistent NMP layer.
 *
 * Drop-in boundary for the reference's hot path (arXiv 2410.01657 reference,
 * /root/reference/proj). Plain C: opaque handles, plain pointers and sizes,
 * int status codes. No torch / CUDA types in any signature. Host arrays use the
 * reference's own layouts (row-major double Tensor2D, int32 index vectors), so
 * a C++ caller holding hgnn::ReducedGraph / HaloMap / ModelParams can bind it
 * without conversion beyond pointer extraction.
 *
 * Every entry point cites the reference interface it replaces.
 */
#ifndef HGNN_B200_H
#define HGNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per hgnn::Error subclass (error.hpp:8-72) ---------- */
enum {
  HGNN_OK = 0,
  HGNN_ERR_SHAPE = 1,          /* ShapeError */
  HGNN_ERR_CONFIG = 2,         /* ConfigError */
  HGNN_ERR_PARTITION = 3,      /* PartitionError */
  HGNN_ERR_COLLECTIVE = 4,     /* CollectiveError */
  HGNN_ERR_INTEGRITY = 5,      /* IntegrityError */
  HGNN_ERR_UNINITIALIZED = 6,  /* UninitializedError */
  HGNN_ERR_SIZE = 7,           /* SizeError */
  HGNN_ERR_OPTIMIZER = 8,      /* OptimizerError */
  HGNN_ERR_IO = 9,             /* IoError */
  HGNN_ERR_CUDA = 20,          /* device fault / missing GPU */
  HGNN_ERR_NCCL = 21,          /* NCCL failure */
  HGNN_ERR_INTERNAL = 22
};

/* ExchangeMode (comm.hpp:17), same numeric order. */
enum { HGNN_MODE_NONE = 0, HGNN_MODE_A2A = 1, HGNN_MODE_NA2A = 2 };

/* PartitionStrategy (mesh.hpp:53) plus the harness's verify_partition rule
 * (harness.cpp:42-45: slab at R=1, balanced block otherwise). */
enum { HGNN_PART_SLAB = 0, HGNN_PART_BLOCK = 1, HGNN_PART_VERIFY = 2 };

/* Message of the last failing call on this host thread. */
const char* hgnn_last_error(void);

/* ========================================================================== */
/* Host graph description: one rank's ReducedGraph + HaloMap                  */
/* (graph.hpp:16-65), flattened. Lists over neighbours / sync groups are CSR. */
/* ========================================================================== */
typedef struct {
  int32_t rank, num_ranks; /* num_ranks 0 = unknown (the context's count is used) */
  int64_t num_local, num_halo, num_edges;
  const int64_t* global_ids;        /* [rows]        graph.hpp:22 */
  const double* positions;          /* [rows*3]      (nullable for upload) */
  const int32_t* edge_src;          /* [num_edges]   reference edge-id order */
  const int32_t* edge_dst;          /* [num_edges] */
  const int32_t* node_degree;       /* [num_local]   (nullable for upload) */
  const int32_t* edge_degree;       /* [num_edges]   (nullable for upload) */
  const double* node_inv_degree;    /* [num_local]   (nullable for upload) */
  const double* edge_inv_degree;    /* [num_edges] */
  const int32_t* in_offsets;        /* [rows+1]      graph.cpp:122-136 */
  const int32_t* in_edges;          /* [num_edges] */
  const int32_t* out_offsets;       /* [rows+1]      (nullable for upload) */
  const int32_t* out_edges;         /* [num_edges]   (nullable for upload) */
  int32_t num_neighbors;
  const int32_t* neighbors;         /* [num_neighbors] ascending */
  const int32_t* send_offsets;      /* [num_neighbors+1] */
  const int32_t* send_rows;         /* local rows, ascending gid per neighbour */
  const int32_t* recv_offsets;      /* [num_neighbors+1] */
  const int32_t* recv_rows;         /* halo rows (consecutive per neighbour) */
  const int32_t* halo_to_local;     /* [num_halo]    (nullable for upload) */
  int64_t num_sync_groups;
  const int32_t* sync_local;        /* [num_sync_groups] */
  const int32_t* sync_offsets;      /* [num_sync_groups+1] */
  const int32_t* sync_slots;        /* -1 = own aggregate, else halo row */
  int64_t max_buffer_rows;          /* global max send-mask length (A2A pad) */
} hgnn_graph_desc;

/* ---- host graph builder (replaces build_box_mesh + partition_mesh +        */
/*      build_distributed_graph for ONE rank: mesh.cpp:106-226,               */
/*      graph.cpp:40-265). Bit-exact to the reference; analytic, O(rank).     */
typedef struct hgnn_host_graph hgnn_host_graph;

/* factors: (Rx,Ry,Rz) for HGNN_PART_BLOCK, or NULL for balanced_factors. */
int hgnn_graph_build(int64_t elements_per_axis, int64_t poly_order, int64_t num_ranks, int strategy,
                     const int64_t* factors, int32_t rank, hgnn_host_graph** out);
/* Same on the box [domain_min, domain_max] (MeshConfig::domain_min / domain_max,
 * mesh.hpp; NULL = the unit cube). HGNN_ERR_CONFIG unless max > min per axis. */
int hgnn_graph_build_domain(int64_t elements_per_axis, int64_t poly_order, int64_t num_ranks, int strategy,
                            const int64_t* factors, int32_t rank, const double* domain_min,
                            const double* domain_max, hgnn_host_graph** out);
void hgnn_graph_free(hgnn_host_graph* g);
/* Zero-copy view of the built arrays (valid until hgnn_graph_free). */
int hgnn_graph_view(const hgnn_host_graph* g, hgnn_graph_desc* out);
/* Per-rank HGNNGRB1 graph files, byte-compatible with the reference's
 * save_graph_binary / load_graph (io.cpp:200-309; replaces both for the binary
 * format). The loader recomputes the reciprocal degrees and the CSR exactly
 * as finalize_loaded_graph (io.cpp:152-161) and range-checks every index the
 * device path dereferences; a loaded graph has num_ranks = 0 (not stored).
 * Errors: HGNN_ERR_IO (missing/truncated/corrupt file, JSON dumps). */
int hgnn_graph_save_binary(const hgnn_graph_desc* g, const char* path);
int hgnn_graph_load_binary(const char* path, hgnn_host_graph** out);
/* balanced_factors (mesh.cpp:154-176) */
int hgnn_balanced_factors(int64_t num_ranks, int64_t elements_per_axis, int64_t out[3]);

/* ---- parameters (model.cpp:105-169, nn.cpp:55-97) ------------------------ */
/* Full-model parameter count and seeded init, ModelParams::for_each order. */
int64_t hgnn_param_count(int64_t hidden, int64_t num_mp_layers, int64_t mlp_hidden_layers,
                         int64_t in_node_dim, int64_t in_edge_dim, int64_t out_dim);
int hgnn_init_params(int64_t hidden, int64_t num_mp_layers, int64_t mlp_hidden_layers, int64_t in_node_dim,
                     int64_t in_edge_dim, int64_t out_dim, uint64_t seed, double* flat);
/* Offset / length of the MP-layer block (layer{0..M-1}.{edge,node}_update.*)
 * inside the full for_each vector. */
int hgnn_mp_param_range(int64_t hidden, int64_t num_mp_layers, int64_t mlp_hidden_layers, int64_t in_node_dim,
                        int64_t in_edge_dim, int64_t* offset, int64_t* count);

/* ========================================================================== */
/* Device engine: one context per rank / GPU (replaces the per-rank body of   */
/* RankRuntime::run, comm.cpp:58-93, for the MP stack).                       */
/* ========================================================================== */
typedef struct hgnn_ctx hgnn_ctx;

/* Number of visible CUDA devices (0 when no driver / GPU is present). */
int hgnn_device_count(void);

/* NCCL unique id (128 bytes) created on rank 0 and broadcast by the caller. */
int hgnn_nccl_unique_id(uint8_t out[128]);

/* device: CUDA ordinal; uid may be NULL when num_ranks == 1. */
int hgnn_ctx_create(int device, int32_t rank, int32_t num_ranks, const uint8_t* nccl_uid, hgnn_ctx** out);

/* In-process rank group: the reference's RankRuntime (comm.cpp:35-93) — R
 * ranks driven by R host threads of one process, each with its own context,
 * on one GPU or several. Exchanges and all-reduces rendezvous on the host with
 * the reference's rule (same collective, same order on every rank; a mismatch
 * poisons the group and every rank gets HGNN_ERR_COLLECTIVE, comm.cpp:168-208)
 * and move data with device-to-device copies; a rank that does not arrive
 * within the timeout (default 120 s) fails its peers instead of hanging them. */
typedef struct hgnn_local_group hgnn_local_group;
int hgnn_local_group_create(int32_t num_ranks, hgnn_local_group** out);
int hgnn_local_group_destroy(hgnn_local_group* group); /* after every member context is destroyed */
int hgnn_local_group_set_timeout(hgnn_local_group* group, int64_t timeout_ms);
int hgnn_ctx_create_local(int device, int32_t rank, hgnn_local_group* group, hgnn_ctx** out);
int hgnn_ctx_destroy(hgnn_ctx* ctx);
/* cudaStream_t of the compute stream, as an opaque pointer (for event timing). */
void* hgnn_ctx_stream(hgnn_ctx* ctx);

/* Upload one rank's graph (ReducedGraph + HaloMap). Edges are re-ordered on the
 * device by receiver (the in-CSR order); the permutation is applied at the
 * boundary so host tensors stay in reference edge-id order. */
int hgnn_graph_upload(hgnn_ctx* ctx, const hgnn_graph_desc* graph);

/* GnnConfig (model.hpp:19-27) fields the MP stack needs; mode = ExchangeMode. */
int hgnn_configure(hgnn_ctx* ctx, int64_t hidden, int64_t num_mp_layers, int64_t mlp_hidden_layers, int mode);

/* MP-layer parameters, for_each order of layer{m}.edge_update.* then
 * layer{m}.node_update.* (model.cpp:130-133), fp64 host. */
int hgnn_params_upload(hgnn_ctx* ctx, const double* mp_params, int64_t count);

/* gnn_forward's layer loop (model.cpp:295-300) = M x nmp_layer_forward
 * (model.cpp:220-272). x0: rows x H, e0: N_e x H (edge-id order), fp64 host.
 * x_out / e_out (nullable) receive layer M-1's outputs. Traces for the
 * backward pass stay on the device. Collective over all ranks when mode != None. */
int hgnn_mp_forward(hgnn_ctx* ctx, const double* x0, const double* e0, double* x_out, double* e_out);

/* gnn_backward's layer loop (model.cpp:411-415) = M x nmp_layer_backward
 * (model.cpp:318-387). dx: rows x H adjoint of the last layer's x output; de
 * (nullable = zeros, model.cpp:412) its e output. Outputs (each nullable):
 * dx0 (rows x H), de0 (N_e x H), mp_grads (same layout as hgnn_params_upload;
 * rank-local, not averaged). */
int hgnn_mp_backward(hgnn_ctx* ctx, const double* dx, const double* de, double* dx0, double* de0,
                     double* mp_grads);

/* Layer trace (NmpLayerTrace, model.hpp:78-87 plus outputs) to host fp64. */
enum { HGNN_TRACE_X_IN = 0, HGNN_TRACE_E_IN = 1, HGNN_TRACE_A_SYNC = 2, HGNN_TRACE_X_OUT = 3, HGNN_TRACE_E_OUT = 4 };
int hgnn_get_trace(hgnn_ctx* ctx, int layer, int which, double* out);

/* ---- device-resident step (bench `value`: inputs already in HBM) --------- */
/* Fill x0 / e0 / dx_M on the device with seeded values that depend only on
 * global ids (so coincident rows agree bitwise across ranks). */
int hgnn_synthetic_inputs(hgnn_ctx* ctx, uint64_t seed);
/* Stage host fp64 inputs once into the device input buffers. */
int hgnn_set_inputs(hgnn_ctx* ctx, const double* x0, const double* e0, const double* dx);
/* One full MP-stack forward + backward on the staged device inputs. */
int hgnn_mp_step_device(hgnn_ctx* ctx);
/* Device gradients -> host (fp64), same layout as hgnn_params_upload. */
int hgnn_get_grads(hgnn_ctx* ctx, double* mp_grads);

/* ========================================================================== */
/* Model level: node / edge encoders and the decoder on  */
/* the device around the MP stack, the consistent loss, rank-averaged          */
/* gradients and Adam — compute_gradients / train_step (model.cpp:556-579).   */
/* Hidden width 32 or 64, feature widths (F_x, F_e, F_y) = (3, 7, 3).        */
/* ========================================================================== */
/* After hgnn_configure: feature widths (GnnConfig in_node_dim, in_edge_dim, out_dim). */
int hgnn_model_configure(hgnn_ctx* ctx, int64_t in_node_dim, int64_t in_edge_dim, int64_t out_dim);
/* Length of the full ModelParams::for_each vector (model.cpp:124-135), -1 before configure. */
int64_t hgnn_model_param_count(hgnn_ctx* ctx);
/* Full parameter vector, fp64, for_each order; resets the Adam state. */
int hgnn_model_params_upload(hgnn_ctx* ctx, const double* params, int64_t count);
int hgnn_model_params_download(hgnn_ctx* ctx, double* params);
/* node_features: rows x F_x (ReducedGraph::node_features), edge_features:
 * N_e x F_e in edge-id order (init_edge_features), target: num_local x F_y or
 * NULL for the autoencoding target (model.cpp:605-607). Needs node_inv_degree
 * in the uploaded graph (consistent-loss weights). */
int hgnn_model_set_data(hgnn_ctx* ctx, const double* node_features, const double* edge_features, const double* target);
/* compute_gradients (model.cpp:556-567): loss (all ranks), gradients averaged
 * over ranks in for_each order (nullable), decoder output y (num_local x F_y,
 * nullable). Collective over all ranks. */
int hgnn_compute_gradients(hgnn_ctx* ctx, double* loss, double* grads, double* y);
/* train_step (model.cpp:569-579): compute_gradients + bias-corrected Adam
 * (nn.cpp:331-360) on fp64 master parameters; returns the loss before the update. */
int hgnn_train_step(hgnn_ctx* ctx, double lr, double beta1, double beta2, double eps, double* loss);

/* ---- options --------------------------------------------------------------- */
/* "edge_factorized":  1 = (default; tcgen05 paths, H = 64) the edge MLP's input linear is
 *                     split through the nodes, P = x [W0_s | W0_d] once per node and
 *                     only e W0_e per edge; the forward edge kernel also forms the
 *                     aggregate (one fused kernel, no aggregate launch) and the
 *                     backward's x adjoints / W0_s, W0_d gradients are node-level
 *                     sums (no per-edge d_x_src / d_x_dst tensors). 0 = the
 *                     3-segment edge kernels + aggregate + dx gather.
 * "mlp_forward_impl": 1 = tcgen05 tensor-core MLP forward (default, H in {32,64}),
 *                     0 = SIMT fp32 kernels.
 * "mlp_backward_impl": 1 = tcgen05 tensor-core MLP backward (default, H in {32, 64};
 *                      H = 32 runs zero-padded on the 64-wide kernel), 0 = SIMT fp32.
 * "adjoint_presum":    1 = the factorised path's node-level input adjoint reads segment
 *                      sums precomputed by a separate kernel; 0 = (default) in-kernel.
 * "tma_gather":        1 = the fused edge forward's input rows gathered by TMA
 *                      tile::gather4 into SMEM (H = 64); 0 = (default, measured
 *                      faster) per-thread 256-bit row loads into registers.
 * "encoder_impl":      1 = (default, H = 64 with both MLP impls 1) node / edge
 *                      encoders on the tcgen05 MLP kernels (zero-padded F-feature
 *                      input, skip + output LayerNorm in the epilogue); 0 = SIMT.
 * "memory_lean":       -1 = (default) auto, 0 = standard plan, 1 = lean plan.
 * "collective_check", "collective_timeout_ms": debug collective-sequence guard. 
 * "halo_overlap":      1 = (default; R > 1, exchange mode set, tcgen05 path) forward:
 *                      boundary-row edges + aggregates first, then the exchange on
 *                      a side stream while the interior edges run; backward: the
 *                      adjoint exchange on the side stream during the interior
 *                      edges' backward. 0 = the serial schedule. Same results
 *                      (outputs and adjoints bitwise; weight gradients regrouped).
 * "halo_sm_reserve":   SMs the overlapped interior launches leave free for the
 *                      pack / NCCL kernels (0..32). */
int hgnn_set_option(hgnn_ctx* ctx, const char* key, int64_t value);

/* ---- instrumentation ------------------------------------------------------ */
/* When enabled, every launch of the listed kernel classes is bracketed by CUDA
 * events on its stream; totals are read back with hgnn_kernel_time. */
enum {
  HGNN_K_EDGE_FWD = 0, HGNN_K_EDGE_BWD = 1, HGNN_K_NODE_FWD = 2, HGNN_K_NODE_BWD = 3,
  HGNN_K_AGG = 4, HGNN_K_DX = 5, HGNN_K_HALO = 6, HGNN_K_GRAD_REDUCE = 7,
  HGNN_K_ENCODE = 8, HGNN_K_DECODE = 9, HGNN_K_LOSS_ADAM = 10,
  HGNN_K_EDGE_PROJ = 11, /* node-level projections P = x [W0_s | W0_d] of the factorised edge MLP */
  HGNN_K_COUNT = 12
};
int hgnn_kernel_timing(hgnn_ctx* ctx, int enable);
int hgnn_kernel_time(hgnn_ctx* ctx, int kernel_class, double* total_ms, int64_t* launches);
/* Cycle counters of the tensor-core kernels (after hgnn_set_option(ctx,
 * "bwd_profile", 1); debugging aid, summed over CTAs):
 *   [0..16)  backward, edge MLP  (kProf* in mlp_tc_bwd.cuh)
 *   [16..32) backward, node MLP
 *   [32..48) forward, edge MLP   (kFwdProf* in mlp_tc.cuh)
 *   [48..64) forward, node MLP */
int hgnn_debug_profile(hgnn_ctx* ctx, uint64_t* out64);
/* Own-kernel launches issued since the last reset (for gpu_launches). */
int64_t hgnn_launch_count(hgnn_ctx* ctx, int reset);
/* Bytes handed to NCCL by this rank since the last reset (CommCounters analogue). */
int64_t hgnn_halo_bytes(hgnn_ctx* ctx, int reset);

#ifdef __cplusplus
}
#endif
#endif /* HGNN_B200_H */
