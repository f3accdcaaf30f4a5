/*
 * mrf_cuda.h -- C-ABI of the B200 (sm_100a) ISGMR / TRWP min-sum message
 * passing library (libmrf_cuda.so).
 *
 * This is the drop-in boundary for the reference library's hot path
 * (/root/reference/proj, namespace mp). The reference exposes C++ templates
 * with no FFI; every entry point below replaces one of them (cited per
 * function) for Real = float, with the reference's tensor layouts extended by
 * a leading batch dimension B:
 *
 *   unary          [B][N][L]    f32   (UnaryVolume::values, potentials.hpp:88-105)
 *   pairwise       [L][L]       f32   V(a,b) = pairwise[a*L+b], shared by the batch
 *                                     (PairwiseFunction::table, potentials.hpp:27-35)
 *   weight planes  [B][R/2][N]  f32   plane[r>>1][(r&1)?cur:prev] (potentials.hpp:131-138)
 *   rho planes     [B][R/2][N]  f32   same indexing (potentials.hpp:152-155)
 *   messages       [B][R][N][L] f32   (IsgmrEngine::m_, isgmr.hpp:36-39)
 *   p              [B][K][E][L] u8    byte ((k*E + dir_offset(r) + e)*L + l) per image
 *   q              [B][K][E]    u8    (IndexStore, index_store.hpp:35-46)
 *   cost           [B][N][L]    f32   (CostOutput::cost, inference.hpp:16-23)
 *   labels         [B][N]       u16   (CostOutput::labels_map)
 *
 * N = H*W, R = connectivity (4 or 8; 16 accepted), E = sum_r |E^r| edges.
 *
 * Conventions
 *  - Every function returns MRF_OK (0) or an error code; mrf_last_error()
 *    returns a thread-local message for the last failure on this thread.
 *    Invalid arguments (the reference's std::invalid_argument cases: K < 1,
 *    L > 256, bad rho, size mismatches) return MRF_EINVAL.
 *  - All tensor pointers are caller-owned DEVICE pointers on the current
 *    device. Execution is stream-ordered on `stream`; nothing blocks the host
 *    except mrf_check_finite_f32 (it returns a verdict).
 *  - Workspace is caller-owned device memory sized by the *_workspace_bytes
 *    queries; it needs no initialisation.
 *  - Results are bit-identical to the reference CPU implementation for
 *    messages, cost, labels, p and q (FP32, no FMA contraction, lowest index
 *    wins ties). Gradients match within 1e-5 (normwise and elementwise) and
 *    are bit-identical run to run.
 *  - p and q buffers are read as aligned 32-bit words: their allocations must
 *    extend to the next multiple of 4 bytes past the last index byte (any
 *    cudaMalloc allocation does; a sub-buffer needs up to 3 bytes of slack).
 */
#ifndef MRF_CUDA_H
#define MRF_CUDA_H

#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MRF_OK 0
#define MRF_EINVAL 1
#define MRF_ECUDA 2
#define MRF_ENOMEM 3

#define MRF_ENGINE_ISGMR 0
#define MRF_ENGINE_TRWP 1

/* Thread-local description of the last error returned on this thread. */
const char* mrf_last_error(void);
/* Library ABI version (major*10000 + minor*100 + patch): 20000 = 2.0.0, the
 * layout with mrf_problem_f32::assume_finite / diag_gap. */
#define MRF_VERSION 20000
int mrf_version(void);

/* ---------------------------------------------------------------- topology */

typedef struct mrf_topology_s* mrf_topology_t;

/* Replaces mp::GridTopology(GridGraph(H, W), DirectionSet::build(connectivity))
 * (grid.hpp:73-96, src/grid.cpp:96-114, :13-26). Same direction order,
 * scanline order and dense per-direction edge numbering. */
int mrf_topology_create(int height, int width, int connectivity, mrf_topology_t* out);
int mrf_topology_destroy(mrf_topology_t topo);
/* num_dirs(), total_edges(), edge_count(r), dir_offset(r) (grid.hpp:79-86).
 * edge_count / dir_offset may be NULL, else arrays of num_dirs entries. */
int mrf_topology_info(mrf_topology_t topo, int* num_dirs, int64_t* total_edges, int64_t* edge_count,
                      int64_t* dir_offset);
/* Host copy of edge_index(r, node) for all r, node: [R][N], -1 at heads. */
int mrf_topology_edge_index(mrf_topology_t topo, int32_t* out);
/* Host copy of scanlines(r): first node and node count of each, in order.
 * *count receives the number of scanlines; at most `cap` entries are written. */
int mrf_topology_scanlines(mrf_topology_t topo, int r, int32_t* first, int32_t* length, int32_t* count, int cap);

/* ---------------------------------------------------------------- problem */

typedef struct {
  int batch;                 /* B >= 1 images sharing one topology and one V */
  int height, width, labels; /* H, W, L (1 <= L <= 256) */
  const float* unary;        /* [B][N][L] */
  const float* pairwise;     /* [L][L] */
  float weight;              /* constant edge weight, used when weight_planes == NULL */
  const float* weight_planes;/* [B][R/2][N] or NULL */
  float rho;                 /* TRWP uniform tree coefficient (0,1], used when rho_planes == NULL */
  const float* rho_planes;   /* [B][R/2][N] or NULL */
  /* 0 (default): the forward entry points scan `unary` for non-finite values
   * and return MRF_EINVAL (the reference engines throw, isgmr.hpp:32-35,
   * trwp.hpp:33-36); this synchronises `stream` once per call. 1: the caller
   * guarantees finite unaries (no scan). */
  int assume_finite;
  /* NULL (default), or device float [B] initialised by the caller (e.g. to
   * +inf): diagnostic mode. Every forward sweep then also tracks the smallest
   * (second best - best) gap of the min-plus argmins and of the
   * reparametrisation argmin (IsgmrEngine/TrwpEngine::min_argmin_gap,
   * isgmr.hpp:64-68,109-115,125-129, trwp.hpp:57-59) and min-accumulates it
   * into diag_gap[b]. Diagnostic sweeps run the dense min-plus kernel (every
   * (mu, l) candidate): same messages and indices, much slower. */
  float* diag_gap;
} mrf_problem_f32;

typedef struct {
  float* cost;      /* [B][N][L] or NULL */
  uint16_t* labels; /* [B][N] or NULL */
  float* messages;  /* [B][R][N][L], required: final messages */
  uint8_t* p;       /* [B][K][E][L], required */
  uint8_t* q;       /* [B][K][E], required */
} mrf_forward_out;

typedef struct {
  float* unary;         /* [B][N][L]  d/d theta (GradientSet::unary) */
  float* pairwise;      /* [B][L][L]  d/d V per image (GradientSet::pairwise) */
  float* weight_planes; /* [B][R/2][N] d/d w planes (GradientSet::edge_weights); may be NULL */
} mrf_grads_f32;

/* Scans the unary volume for non-finite values (the reference engines reject
 * them, isgmr.hpp:33-35). Synchronises `stream`. */
int mrf_check_finite_f32(const float* data, size_t count, int* all_finite, cudaStream_t stream);

/* ---------------------------------------------------------------- forward */

size_t mrf_forward_workspace_bytes(mrf_topology_t topo, const mrf_problem_f32* prob, int engine, int iterations);

/* Replaces mp::isgmr_forward<float>(topo, pots, K, threads) (isgmr.hpp:145-152):
 * K iterations of Alg. 1 (all directions and scanlines of an iteration in one
 * launch, m <- mhat published by a buffer swap), then aggregate (inference.hpp:40-57). */
int mrf_isgmr_forward_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int iterations,
                          const mrf_forward_out* out, void* workspace, size_t workspace_bytes,
                          cudaStream_t stream);
/* Replaces mp::trwp_forward<float>(topo, pots, rho, K, threads) (trwp.hpp:148-156):
 * directions strictly sequential, in place. */
int mrf_trwp_forward_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int iterations,
                         const mrf_forward_out* out, void* workspace, size_t workspace_bytes,
                         cudaStream_t stream);

/* Engine API: one IsgmrEngine::step() (isgmr.hpp:49-56). Reads published
 * messages m_in, writes the swept buffer m_out (the new published messages)
 * and iteration k's indices into p/q (capacity K_cap iterations). m_out must
 * hold zeros on scanline-head rows (e.g. a zero-filled buffer or an earlier
 * message buffer of the same engine). */
int mrf_isgmr_step_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int k, int K_cap, const float* m_in,
                       float* m_out, uint8_t* p, uint8_t* q, cudaStream_t stream);
/* One TrwpEngine::step() (trwp.hpp:47-61), in place on `messages`. */
int mrf_trwp_step_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int k, int K_cap, float* messages,
                      uint8_t* p, uint8_t* q, cudaStream_t stream);
/* IsgmrEngine/TrwpEngine::aggregate() == aggregate_costs (inference.hpp:40-57). */
int mrf_aggregate_f32(mrf_topology_t topo, const mrf_problem_f32* prob, const float* messages, float* cost,
                      uint16_t* labels, cudaStream_t stream);

/* --------------------------------------------------------------- backward */

size_t mrf_backward_workspace_bytes(mrf_topology_t topo, const mrf_problem_f32* prob, int engine, int iterations);

/* Replaces mp::isgmr_backward<float>(topo, pots, indices, grad_cost, threads)
 * (autodiff.hpp:63-126). grad_cost is [B][N][L]. */
int mrf_isgmr_backward_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int iterations, const uint8_t* p,
                           const uint8_t* q, const float* grad_cost, const mrf_grads_f32* grads, void* workspace,
                           size_t workspace_bytes, cudaStream_t stream);
/* Replaces mp::trwp_backward<float>(topo, pots, rho, indices, grad_cost, threads)
 * (autodiff.hpp:133-197). */
int mrf_trwp_backward_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int iterations, const uint8_t* p,
                          const uint8_t* q, const float* grad_cost, const mrf_grads_f32* grads, void* workspace,
                          size_t workspace_bytes, cudaStream_t stream);

/* Shared-parameter gradient pack for data parallelism: out[0:L*L] = sum over
 * the batch of grads->pairwise (fixed image order), out[L*L] = sum of all
 * weight-plane gradients (GradientSet::edge_weight_total, autodiff.hpp:24-28)
 * when weight_planes != NULL, else 0. out is device [L*L + 1]. */
int mrf_pack_shared_grads_f32(const mrf_problem_f32* prob, int num_dirs, const mrf_grads_f32* grads, float* out,
                              cudaStream_t stream);

/* One NCCL all-reduce (sum, float) of `count` floats in place, on `stream`,
 * over `nccl_comm` (an ncclComm_t created by the caller). libnccl.so.2 is
 * resolved at run time. Multi-GPU data parallelism needs exactly one such call
 * per training step, over the buffer mrf_pack_shared_grads_f32 produced. */
int mrf_allreduce_grads_f32(void* nccl_comm, float* buffer, size_t count, cudaStream_t stream);

/* Communicator helpers for callers without their own NCCL binding (bench.py,
 * paper_1910_10892_b200/dist.py): mrf_nccl_unique_id writes rank 0's 128-byte
 * ncclUniqueId (broadcast it to the other ranks out of band), every rank then
 * calls mrf_nccl_comm_init(&comm, nranks, id, rank) on its own device;
 * mrf_nccl_comm_destroy frees it. */
int mrf_nccl_unique_id(void* out, size_t bytes);
int mrf_nccl_comm_init(void** comm, int nranks, const void* unique_id, int rank);
int mrf_nccl_comm_destroy(void* comm);

/* ------------------------------------------------- readout and evaluation */

/* Replaces mp::soft_head_forward<float> + mp::soft_head_backward<float>
 * (softhead.hpp:22-74) for a batch, fused in one pass over the cost volume:
 * per node confidence = softmax(-c), disparity d = sum_l l f_l, loss[b] =
 * mean_i |d_i - target_i| (device float [B], accumulated in double), and
 * grad_cost = d loss / d c = sign(d - t)/N * (-f (l - d)) (zero on exact
 * ties). cost [B][N][L], target [B][N]; confidence [B][N][L], disparity
 * [B][N] and grad_cost [B][N][L] may be NULL. Stream-ordered. */
int mrf_soft_head_f32(int batch, int nodes, int labels, const float* cost, const float* target, float* confidence,
                      float* disparity, float* grad_cost, float* loss, cudaStream_t stream);

/* Replaces mp::energy<float, uint16_t> (potentials.hpp:175-199): unaries plus
 * every undirected edge once (the even direction of each family), in double,
 * for each image of the batch. labels [B][N] (device), energy: host double
 * [B]. Synchronises `stream`; MRF_EINVAL when a label is out of range (the
 * reference's std::out_of_range). */
int mrf_energy_f32(mrf_topology_t topo, const mrf_problem_f32* prob, const uint16_t* labels, double* energy,
                   cudaStream_t stream);

/* Replaces mp::sgm_forward<float>(topo, pots, variant, threads)
 * (baselines.hpp:31-98). variant 0 = SgmVariant::standard (the message keeps
 * the unary; cost = sum_r m^r), 1 = SgmVariant::revised (== one ISGMR
 * iteration, test_baselines.cpp:58-68). messages [B][R][N][L] (required),
 * cost [B][N][L] and labels [B][N] (may be NULL). Stream-ordered. */
int mrf_sgm_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int variant, float* messages, float* cost,
                uint16_t* labels, cudaStream_t stream);

/* Iterated SGM (mp::SgmIterative::step, baselines.hpp:108-161): after a
 * mrf_sgm_f32 round, the next round's unary volume from that round's
 * messages: next(i, l) = sum_r m^r(i, l) - min_l' sum_r m^r(i, l') (r
 * ascending). messages [B][R][N][L], next_unary [B][N][L] (device, must not
 * alias messages). Stream-ordered. */
int mrf_sgm_next_unary_f32(mrf_topology_t topo, const mrf_problem_f32* prob, const float* messages, float* next_unary,
                           cudaStream_t stream);

/* ---------------------------------------------------------- instrumentation */

/* Kernel classes for the launch profiler. */
#define MRF_KCLASS_FWD_SWEEP 0
#define MRF_KCLASS_BWD_SWEEP 1
#define MRF_KCLASS_AGGREGATE 2
#define MRF_KCLASS_AUX 3
#define MRF_KCLASS_COUNT 4

/* Not part of the reference surface. When enabled (on != 0; clears previous
 * records), every kernel launch of this library is bracketed by CUDA events
 * recorded on its own stream. mrf_profiler_read synchronises those events and
 * returns the summed device time and launch count of one kernel class. */
int mrf_profiler_enable(int on);
int mrf_profiler_read(int kernel_class, double* total_ms, int64_t* launches);
/* Number of kernel launches this library has made since it was loaded
 * (including the launches a sweep makes for strategies that do not own it and
 * exit at once). */
int mrf_launch_count(int64_t* total);

#ifdef __cplusplus
}
#endif
#endif /* MRF_CUDA_H */
