/* TEST INFRASTRUCTURE ONLY -- see mrf_oracle.h.
 *
 * Plain-C restatement of the reference path. Every float operation is written
 * in the reference's order, one rounding per operation (built with
 * -ffp-contract=off, no -march): that is what makes the recorded argmin
 * indices comparable bit-for-bit. Citations are to /root/reference/proj.
 */
#include "mrf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Direction order E,W,S,N,SE,NW,SW,NE,... with opposite = r^1
 * (src/grid.cpp:17-26). */
static const int kSteps[16][2] = {{0, 1},  {0, -1},  {1, 0},  {-1, 0}, {1, 1},  {-1, -1}, {1, -1}, {-1, 1},
                                  {1, 2},  {-1, -2}, {1, -2}, {-1, 2}, {2, 1},  {-2, -1}, {2, -1}, {-2, 1}};

struct orc_topo {
  int H, W, R, N;
  int nl[16];          /* scanlines per direction */
  int32_t* first[16];  /* first node of each scanline */
  int32_t* len[16];    /* node count of each scanline */
  int64_t ecount[16], doff[16], total;
  int32_t* eidx;       /* [R][N], -1 at heads */
};

static int floor_div(int x, int a) { return x >= 0 ? x / a : -((-x + a - 1) / a); }
static int pos_mod(int x, int m) { return ((x % m) + m) % m; }

/* Scanline enumeration (src/grid.cpp:37-94): first-node candidates for the
 * canonical step (a,b) = (|dh|,|dw|) -- rows/columns, "wide" lines entering
 * from row 0 shifted left by (H-1)*b, or "narrow" lines interpolated from the
 * shifted tree index -- advanced along (a,b) until in bounds, then mirrored
 * for negative step components. */
static void enumerate(orc_topo* t, int r) {
  const int H = t->H, W = t->W, sh = kSteps[r][0], sw = kSteps[r][1];
  const int a = abs(sh), b = abs(sw);
  int ncand;
  if (a == 0) ncand = H;
  else if (b == 0) ncand = W;
  else if (a <= b) ncand = W + (H - 1) * b;
  else ncand = (W - 1) * a + (H - 1) + 1;
  t->first[r] = (int32_t*)malloc(sizeof(int32_t) * (size_t)ncand);
  t->len[r] = (int32_t*)malloc(sizeof(int32_t) * (size_t)ncand);
  int n = 0;
  for (int c = 0; c < ncand; ++c) {
    int ph, pw;
    if (a == 0) { ph = c; pw = 0; }
    else if (b == 0) { ph = 0; pw = c; }
    else if (a <= b) { ph = 0; pw = c - (H - 1) * b; }
    else {
      const int ts = c - (H - 1);
      ph = pos_mod(a - pos_mod(ts, a), a);
      pw = -floor_div(-ts, a); /* ceil(ts / a) */
    }
    while (ph < H && !(ph >= 0 && pw >= 0 && pw < W)) { ph += a; pw += b; }
    if (ph >= H) continue;
    int cnt = 0, h = ph, w = pw;
    while (h >= 0 && h < H && w >= 0 && w < W) { ++cnt; h += a; w += b; }
    const int mh = sh < 0 ? H - 1 - ph : ph;
    const int mw = sw < 0 ? W - 1 - pw : pw;
    t->first[r][n] = mh * W + mw;
    t->len[r][n] = cnt;
    ++n;
  }
  t->nl[r] = n;
}

orc_topo* orc_topo_create(int H, int W, int conn) {
  if (H < 1 || W < 1 || (conn != 4 && conn != 8 && conn != 16)) return NULL;
  orc_topo* t = (orc_topo*)calloc(1, sizeof(orc_topo));
  t->H = H; t->W = W; t->R = conn; t->N = H * W;
  t->eidx = (int32_t*)malloc(sizeof(int32_t) * (size_t)conn * t->N);
  /* Dense edge numbering: scanline order, then position (src/grid.cpp:96-114). */
  for (int r = 0; r < conn; ++r) {
    enumerate(t, r);
    int32_t* ei = t->eidx + (size_t)r * t->N;
    for (int i = 0; i < t->N; ++i) ei[i] = -1;
    const int step = kSteps[r][0] * W + kSteps[r][1];
    int32_t e = 0;
    for (int s = 0; s < t->nl[r]; ++s)
      for (int j = 1; j < t->len[r][s]; ++j) ei[t->first[r][s] + j * step] = e++;
    t->ecount[r] = e;
    t->doff[r] = t->total;
    t->total += e;
  }
  return t;
}

void orc_topo_free(orc_topo* t) {
  if (!t) return;
  for (int r = 0; r < t->R; ++r) { free(t->first[r]); free(t->len[r]); }
  free(t->eidx);
  free(t);
}

int64_t orc_total_edges(const orc_topo* t) { return t->total; }
int orc_num_dirs(const orc_topo* t) { return t->R; }

void orc_topo_dump(const orc_topo* t, int64_t* edge_count, int64_t* dir_offset, int32_t* edge_index,
                   int32_t* nlines, int32_t* line_first, int32_t* line_len, int cap) {
  for (int r = 0; r < t->R; ++r) {
    edge_count[r] = t->ecount[r];
    dir_offset[r] = t->doff[r];
    memcpy(edge_index + (size_t)r * t->N, t->eidx + (size_t)r * t->N, sizeof(int32_t) * t->N);
    nlines[r] = t->nl[r];
    for (int s = 0; s < t->nl[r] && s < cap; ++s) {
      line_first[(size_t)r * cap + s] = t->first[r][s];
      line_len[(size_t)r * cap + s] = t->len[r][s];
    }
  }
}

/* ---- shared helpers ------------------------------------------------------ */

/* Edge weight of (prev,cur) along r: constant, or planes[r>>1][(r&1)?cur:prev]
 * (include/mp/potentials.hpp:131-138); rho uses the same indexing (:152-155). */
static float plane_val(const float* planes, float c, int N, int r, int prev, int cur) {
  if (!planes) return c;
  return planes[(size_t)(r >> 1) * N + ((r & 1) ? cur : prev)];
}

/* V'(mu,l): canonical undirected orientation -- V(mu,l) on even directions,
 * V(l,mu) on odd ones (include/mp/isgmr.hpp:94-96). */
static float vprime(const float* V, int L, int r, int mu, int l) {
  return (r & 1) ? V[(size_t)l * L + mu] : V[(size_t)mu * L + l];
}

/* Min-plus + argmin into p, then reparametrization with argmin into q
 * (isgmr.hpp:98-131, identical in trwp.hpp:100-133). Strict '<' scans keep
 * the lowest index on ties. */
static void minplus_reparam(const float* base, const float* V, int L, int r, float w, float* out,
                            uint8_t* prow, uint8_t* qcell) {
  for (int l = 0; l < L; ++l) {
    float best = INFINITY;
    int arg = 0;
    for (int mu = 0; mu < L; ++mu) {
      const float wv = w * vprime(V, L, r, mu, l);
      const float v = base[mu] + wv;
      if (v < best) { best = v; arg = mu; }
    }
    prow[l] = (uint8_t)arg;
    out[l] = best;
  }
  int ls = 0;
  float lo = out[0];
  for (int l = 1; l < L; ++l)
    if (out[l] < lo) { lo = out[l]; ls = l; }
  *qcell = (uint8_t)ls;
  for (int l = 0; l < L; ++l) out[l] = out[l] - lo;
}

/* c = theta, c += m^r for r = 0..R-1 in order; labels = first argmin
 * (include/mp/inference.hpp:25-57). */
static void aggregate(int N, int L, int R, const float* unary, const float* m, float* cost, uint16_t* labels) {
  const size_t NL = (size_t)N * L;
  float* c = cost ? cost : (float*)malloc(sizeof(float) * NL);
  memcpy(c, unary, sizeof(float) * NL);
  for (int r = 0; r < R; ++r)
    for (size_t i = 0; i < NL; ++i) c[i] = c[i] + m[(size_t)r * NL + i];
  if (labels)
    for (int i = 0; i < N; ++i) {
      const float* row = c + (size_t)i * L;
      int best = 0;
      for (int l = 1; l < L; ++l)
        if (row[l] < row[best]) best = l;
      labels[i] = (uint16_t)best;
    }
  if (!cost) free(c);
}

static int check_problem(const orc_problem* pr, int K) {
  if (K < 1 || pr->L < 1 || pr->L > 256) return 1;
  const size_t NL = (size_t)pr->H * pr->W * pr->L;
  for (size_t i = 0; i < NL; ++i)
    if (!isfinite(pr->unary[i])) return 1;
  return 0;
}

/* ---- ISGMR forward (include/mp/isgmr.hpp:26-152) ------------------------- */

int orc_isgmr_forward(const orc_topo* t, const orc_problem* pr, int K, float* cost, uint16_t* labels,
                      float* messages, uint8_t* p, uint8_t* q) {
  if (check_problem(pr, K)) return 1;
  const int N = t->N, L = pr->L, R = t->R;
  const size_t NL = (size_t)N * L, E = (size_t)t->total;
  float* m = (float*)calloc((size_t)R * NL, sizeof(float));
  float* mh = (float*)calloc((size_t)R * NL, sizeof(float));
  float* base = (float*)malloc(sizeof(float) * L);
  for (int k = 0; k < K; ++k) {
    for (int r = 0; r < R; ++r) {
      const int opp = r ^ 1, step = kSteps[r][0] * t->W + kSteps[r][1];
      float* mr = mh + (size_t)r * NL;
      for (int s = 0; s < t->nl[r]; ++s)
        for (int j = 1; j < t->len[r][s]; ++j) {
          const int prev = t->first[r][s] + (j - 1) * step, cur = prev + step;
          /* base = (theta + mhat^r) + m^d for d ascending, d not in {r, r-} (:82-88) */
          for (int mu = 0; mu < L; ++mu) base[mu] = pr->unary[(size_t)prev * L + mu] + mr[(size_t)prev * L + mu];
          for (int d = 0; d < R; ++d) {
            if (d == r || d == opp) continue;
            const float* md = m + (size_t)d * NL + (size_t)prev * L;
            for (int mu = 0; mu < L; ++mu) base[mu] = base[mu] + md[mu];
          }
          const float w = plane_val(pr->w_planes, pr->w_const, N, r, prev, cur);
          const size_t flat = (size_t)k * E + (size_t)t->doff[r] + (size_t)t->eidx[(size_t)r * N + cur];
          minplus_reparam(base, pr->pairwise, L, r, w, mr + (size_t)cur * L, p + flat * L, q + flat);
        }
    }
    memcpy(m, mh, sizeof(float) * (size_t)R * NL); /* publish after all directions (:55) */
  }
  aggregate(N, L, R, pr->unary, m, cost, labels);
  if (messages) memcpy(messages, m, sizeof(float) * (size_t)R * NL);
  free(m); free(mh); free(base);
  return 0;
}

/* ---- TRWP forward (include/mp/trwp.hpp:25-156) --------------------------- */

int orc_trwp_forward(const orc_topo* t, const orc_problem* pr, int K, float* cost, uint16_t* labels,
                     float* messages, uint8_t* p, uint8_t* q) {
  if (check_problem(pr, K)) return 1;
  const int N = t->N, L = pr->L, R = t->R;
  const size_t NL = (size_t)N * L, E = (size_t)t->total;
  float* m = (float*)calloc((size_t)R * NL, sizeof(float));
  float* base = (float*)malloc(sizeof(float) * L);
  for (int k = 0; k < K; ++k)
    for (int r = 0; r < R; ++r) { /* directions strictly sequential, in place (:50) */
      const int opp = r ^ 1, step = kSteps[r][0] * t->W + kSteps[r][1];
      float* mr = m + (size_t)r * NL;
      for (int s = 0; s < t->nl[r]; ++s)
        for (int j = 1; j < t->len[r][s]; ++j) {
          const int prev = t->first[r][s] + (j - 1) * step, cur = prev + step;
          const float rho = plane_val(pr->rho_planes, pr->rho_const, N, r, prev, cur);
          /* s = theta + sum_{d=0..R-1} m^d; base = rho*s - m^{r-} (:84-90) */
          for (int mu = 0; mu < L; ++mu) base[mu] = pr->unary[(size_t)prev * L + mu];
          for (int d = 0; d < R; ++d) {
            const float* md = m + (size_t)d * NL + (size_t)prev * L;
            for (int mu = 0; mu < L; ++mu) base[mu] = base[mu] + md[mu];
          }
          const float* mo = m + (size_t)opp * NL + (size_t)prev * L;
          for (int mu = 0; mu < L; ++mu) {
            const float sc = rho * base[mu];
            base[mu] = sc - mo[mu];
          }
          const float w = plane_val(pr->w_planes, pr->w_const, N, r, prev, cur);
          const size_t flat = (size_t)k * E + (size_t)t->doff[r] + (size_t)t->eidx[(size_t)r * N + cur];
          minplus_reparam(base, pr->pairwise, L, r, w, mr + (size_t)cur * L, p + flat * L, q + flat);
        }
    }
  aggregate(N, L, R, pr->unary, m, cost, labels);
  if (messages) memcpy(messages, m, sizeof(float) * (size_t)R * NL);
  free(m); free(base);
  return 0;
}

/* ---- backward (include/mp/autodiff.hpp:33-197) --------------------------- */

/* Reparametrization backward: row[q] -= sum(row) (:48-53). */
static void reparam_bwd(float* row, int L, int q) {
  float s = 0.0f;
  for (int l = 0; l < L; ++l) s = s + row[l];
  row[q] = row[q] - s;
}

static int backward(int trwp, const orc_topo* t, const orc_problem* pr, int K, const uint8_t* p,
                    const uint8_t* q, const float* gc, float* gu, float* gv, float* gw) {
  if (K < 1 || pr->L < 1 || pr->L > 256) return 1;
  const int N = t->N, L = pr->L, R = t->R;
  const size_t NL = (size_t)N * L, E = (size_t)t->total, LL = (size_t)L * L;
  /* make_gradients: dtheta <- dc, dV <- 0, dw planes <- 0 (:33-44) */
  memcpy(gu, gc, sizeof(float) * NL);
  memset(gv, 0, sizeof(float) * LL);
  memset(gw, 0, sizeof(float) * (size_t)(R / 2) * N);
  float* gm = (float*)malloc(sizeof(float) * (size_t)R * NL);
  for (int r = 0; r < R; ++r) memcpy(gm + (size_t)r * NL, gc, sizeof(float) * NL);
  float* gnext = trwp ? NULL : (float*)calloc((size_t)R * NL, sizeof(float));
  float* vp = (float*)malloc(sizeof(float) * LL);
  for (int k = K - 1; k >= 0; --k) {
    for (int ri = 0; ri < R; ++ri) {
      const int r = trwp ? R - 1 - ri : ri; /* TRWP replays directions in reverse (:147) */
      const int opp = r ^ 1, fam = r >> 1, step = kSteps[r][0] * t->W + kSteps[r][1];
      float* gr = gm + (size_t)r * NL;
      for (int s = 0; s < t->nl[r]; ++s) {
        memset(vp, 0, sizeof(float) * LL); /* per-scanline dV partial (:81,:86) */
        for (int j = t->len[r][s] - 1; j >= 1; --j) {
          const int prev = t->first[r][s] + (j - 1) * step, cur = prev + step;
          const size_t flat = (size_t)k * E + (size_t)t->doff[r] + (size_t)t->eidx[(size_t)r * N + cur];
          const float w = plane_val(pr->w_planes, pr->w_const, N, r, prev, cur);
          const float rho = trwp ? plane_val(pr->rho_planes, pr->rho_const, N, r, prev, cur) : 1.0f;
          const int wnode = (r & 1) ? cur : prev;
          const uint8_t* pr_ = p + flat * L;
          float* row = gr + (size_t)cur * L;
          reparam_bwd(row, L, q[flat]);
          for (int l = 0; l < L; ++l) {
            const float g = row[l];
            if (g == 0.0f) continue;
            const int mu = pr_[l];
            const size_t pm = (size_t)prev * L + mu;
            if (!trwp) {
              /* (:104-109) */
              gu[pm] = gu[pm] + g;
              gr[pm] = gr[pm] + g;
              for (int d = 0; d < R; ++d) {
                if (d == r || d == opp) continue;
                gnext[(size_t)d * NL + pm] = gnext[(size_t)d * NL + pm] + g;
              }
            } else {
              /* (:174-177) */
              const float rg = rho * g;
              gu[pm] = gu[pm] + rg;
              for (int d = 0; d < R; ++d) gm[(size_t)d * NL + pm] = gm[(size_t)d * NL + pm] + rg;
              gm[(size_t)opp * NL + pm] = gm[(size_t)opp * NL + pm] - g;
            }
            const float vval = vprime(pr->pairwise, L, r, mu, l);
            const float gvv = g * vval;
            gw[(size_t)fam * N + wnode] = gw[(size_t)fam * N + wnode] + gvv;
            const size_t vi = (r & 1) ? (size_t)l * L + mu : (size_t)mu * L + l;
            const float gww = g * w;
            vp[vi] = vp[vi] + gww;
          }
        }
        /* partials reduced in scanline order (:119-120) */
        for (size_t i = 0; i < LL; ++i) gv[i] = gv[i] + vp[i];
      }
      if (trwp) memset(gr, 0, sizeof(float) * NL); /* plane r consumed (:190-193) */
    }
    if (!trwp) { /* swap and clear (:122-123) */
      float* tmp = gm; gm = gnext; gnext = tmp;
      memset(gnext, 0, sizeof(float) * (size_t)R * NL);
    }
  }
  free(gm); free(gnext); free(vp);
  return 0;
}

int orc_isgmr_backward(const orc_topo* t, const orc_problem* pr, int K, const uint8_t* p, const uint8_t* q,
                       const float* grad_cost, float* g_unary, float* g_pairwise, float* g_wplanes) {
  return backward(0, t, pr, K, p, q, grad_cost, g_unary, g_pairwise, g_wplanes);
}

int orc_trwp_backward(const orc_topo* t, const orc_problem* pr, int K, const uint8_t* p, const uint8_t* q,
                      const float* grad_cost, float* g_unary, float* g_pairwise, float* g_wplanes) {
  return backward(1, t, pr, K, p, q, grad_cost, g_unary, g_pairwise, g_wplanes);
}

/* ---- soft readout head (include/mp/softhead.hpp:22-74) ------------------- */

float orc_soft_head(int N, int L, const float* cost, const float* target, float* disparity, float* grad) {
  float total = 0.0f;
  float* f = (float*)malloc(sizeof(float) * L);
  for (int i = 0; i < N; ++i) {
    const float* c = cost + (size_t)i * L;
    float hi = -c[0];
    for (int l = 1; l < L; ++l) hi = fmaxf(hi, -c[l]);
    float sum = 0.0f;
    for (int l = 0; l < L; ++l) { f[l] = expf(-c[l] - hi); sum = sum + f[l]; }
    float d = 0.0f;
    for (int l = 0; l < L; ++l) { f[l] = f[l] / sum; d = d + (float)l * f[l]; }
    if (disparity) disparity[i] = d;
    total = total + fabsf(d - target[i]);
    if (grad) {
      const float diff = d - target[i];
      float* g = grad + (size_t)i * L;
      if (diff == 0.0f) {
        for (int l = 0; l < L; ++l) g[l] = 0.0f;
      } else {
        const float s = (diff > 0.0f ? 1.0f : -1.0f) / (float)N;
        for (int l = 0; l < L; ++l) g[l] = s * (-f[l] * ((float)l - d));
      }
    }
  }
  free(f);
  return total / (float)N;
}
