/* TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, single-threaded, FP32 without contraction) of the
 * reference's ISGMR / TRWP message passing and its index-driven backward. It is
 * the checker the GPU parity tests compare against; it is pinned bit-for-bit
 * against the reference library itself (oracle/_ref, tests/test_oracle.py).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it. The product library never links or calls it.
 */
#ifndef MRF_ORACLE_H
#define MRF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_topo orc_topo;

orc_topo* orc_topo_create(int H, int W, int connectivity);
void orc_topo_free(orc_topo* t);
int64_t orc_total_edges(const orc_topo* t);
int orc_num_dirs(const orc_topo* t);
/* Same dump contract as ref_topology (oracle/ref_capi.cpp). */
void orc_topo_dump(const orc_topo* t, int64_t* edge_count, int64_t* dir_offset, int32_t* edge_index,
                   int32_t* nlines, int32_t* line_first, int32_t* line_len, int cap);

typedef struct {
  int H, W, L;
  const float* unary;      /* [N][L] label fastest */
  const float* pairwise;   /* [L][L], V(a,b) = pairwise[a*L+b] */
  float w_const;           /* used when w_planes == NULL */
  const float* w_planes;   /* [R/2][N] or NULL */
  float rho_const;         /* TRWP only */
  const float* rho_planes; /* [R/2][N] or NULL */
} orc_problem;

int orc_isgmr_forward(const orc_topo* t, const orc_problem* pr, int K, float* cost, uint16_t* labels,
                      float* messages, uint8_t* p, uint8_t* q);
int orc_trwp_forward(const orc_topo* t, const orc_problem* pr, int K, float* cost, uint16_t* labels,
                     float* messages, uint8_t* p, uint8_t* q);
int orc_isgmr_backward(const orc_topo* t, const orc_problem* pr, int K, const uint8_t* p, const uint8_t* q,
                       const float* grad_cost, float* g_unary, float* g_pairwise, float* g_wplanes);
int orc_trwp_backward(const orc_topo* t, const orc_problem* pr, int K, const uint8_t* p, const uint8_t* q,
                      const float* grad_cost, float* g_unary, float* g_pairwise, float* g_wplanes);
/* Soft readout head: loss, disparity [N] and d loss / d cost [N][L]. */
float orc_soft_head(int N, int L, const float* cost, const float* target, float* disparity, float* grad_cost);

#ifdef __cplusplus
}
#endif
#endif
