/*
 * oracle/batchlp_oracle.c -- TEST INFRASTRUCTURE ONLY (never shipped, never
 * timed as the product).
 *
 * A plain-C restatement of the reference's batched PDHG hot path, written
 * from the reference's behaviour (proj/include/batchlp/, cited per function)
 * with every sum in the reference's sequential order and no FMA contraction
 * (built with -ffp-contract=off), so on the same inputs it reproduces the
 * compiled reference (oracle/_ref) bit for bit. It is pinned against that
 * library and against tests/golden/ by tests/test_oracle.py, and serves as
 * the CPU-side parity checker on hosts where oracle/_ref is absent.
 *
 * Layout: column-major dense blocks, one contiguous column per LP, like the
 * reference's DenseColumnBlock (sparse.hpp:46-88).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "batchlp_cuda.h"

typedef struct orc_lp {
  int m, n;
  const int32_t *rp, *ci, *trp, *tci; /* A and its explicit transpose (CSR) */
  const double *cv, *tcv;
  const double *c, *xl, *xu, *rl, *ru;
} orc_lp;

static const double kInf = HUGE_VAL;

/* ---- bounds.hpp:67-102 ----------------------------------------------------*/
static double smin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double smax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double project_box(double v, double lo, double hi) { return smax(smin(v, hi), lo); }
static double project_barrier(double v, double lo, double hi) {
  const int lo_inf = lo == -kInf, hi_inf = hi == kInf;
  if (lo_inf && hi_inf) return 0.0;
  if (lo_inf) return smax(v, 0.0);
  if (hi_inf) return smin(v, 0.0);
  return v;
}
static double project_recession(double v, double lo, double hi) {
  const int lo_inf = lo == -kInf, hi_inf = hi == kInf;
  if (lo_inf && hi_inf) return v;
  if (hi_inf) return smax(v, 0.0);
  if (lo_inf) return smin(v, 0.0);
  return 0.0;
}
static double support_term(double v, double lo, double hi) {
  if (v > 0.0) return hi * v;
  if (v < 0.0) return lo * v;
  return 0.0;
}

/* ---- sparse.hpp:176-183: per-row sum in stored order ---------------------*/
static void csr_apply(int rows, const int32_t* rp, const int32_t* ci, const double* cv,
                      const double* x, double* out) {
  for (int i = 0; i < rows; ++i) {
    double acc = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) acc += cv[p] * x[ci[p]];
    out[i] = acc;
  }
}

void orc_spmm(const orc_lp* lp, int transpose, int width, int active, const double* x,
              double* out) {
  const int rin = transpose ? lp->m : lp->n, rout = transpose ? lp->n : lp->m;
  (void)width;
  for (int j = 0; j < active; ++j) {
    if (transpose)
      csr_apply(rout, lp->trp, lp->tci, lp->tcv, x + (size_t)j * rin, out + (size_t)j * rout);
    else
      csr_apply(rout, lp->rp, lp->ci, lp->cv, x + (size_t)j * rin, out + (size_t)j * rout);
  }
}

/* ---- sparse.hpp:249-319: power iteration from two starts ------------------*/
static double power_iteration_from(const orc_lp* lp, double* v) {
  const int n = lp->n, m = lp->m;
  double* u = (double*)malloc(sizeof(double) * (m ? m : 1));
  double* w = (double*)malloc(sizeof(double) * (n ? n : 1));
  double estimate = 0.0;
  int stagnant = 0;
  for (int iter = 0; iter < 5000; ++iter) {
    csr_apply(m, lp->rp, lp->ci, lp->cv, v, u);
    double unorm = 0.0;
    for (int i = 0; i < m; ++i) unorm += u[i] * u[i];
    unorm = sqrt(unorm);
    if (unorm == 0.0) {
      for (int i = 0; i < n; ++i) v[i] = 0.0;
      v[iter % n] = 1.0;
      estimate = 0.0;
      stagnant = 0;
      continue;
    }
    csr_apply(n, lp->trp, lp->tci, lp->tcv, u, w);
    double wnorm = 0.0;
    for (int i = 0; i < n; ++i) wnorm += w[i] * w[i];
    wnorm = sqrt(wnorm);
    const double prev = estimate;
    estimate = unorm;
    if (prev > 0.0 && fabs(estimate - prev) <= 1e-4 * estimate) {
      if (++stagnant >= 10) break;
    } else {
      stagnant = 0;
    }
    if (wnorm == 0.0) break;
    for (int i = 0; i < n; ++i) v[i] = w[i] / wnorm;
  }
  free(u);
  free(w);
  return estimate;
}

/* returns < 0 for the zero matrix (the reference throws invalid_argument) */
double orc_spectral_norm(const orc_lp* lp) {
  const int n = lp->n;
  if (lp->rp[lp->m] == 0) return -1.0;
  double* v = (double*)malloc(sizeof(double) * n);
  for (int i = 0; i < n; ++i) v[i] = 1.0 / sqrt((double)n);
  const double a = power_iteration_from(lp, v);
  uint64_t state = 0x9e3779b97f4a7c15ull;
  double norm_sq = 0.0;
  for (int i = 0; i < n; ++i) {
    state ^= state << 13;
    state ^= state >> 7;
    state ^= state << 17;
    v[i] = (double)(state >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    norm_sq += v[i] * v[i];
  }
  const double inv = 1.0 / sqrt(norm_sq);
  for (int i = 0; i < n; ++i) v[i] *= inv;
  const double b = power_iteration_from(lp, v);
  free(v);
  return ((a < b) ? b : a) * 1.01;
}

/* ---- problem.hpp:199-236: a batch column's cost and bounds ----------------*/
typedef struct column_view {
  const orc_lp* lp;
  int mode, column;
  const bl_override* ov; /* this column's overrides, list order */
  int n_ov;
} column_view;

static double cv_cost(const column_view* v, int i) {
  double c;
  if (v->mode == BL_SHARED_OBJECTIVE) {
    c = v->lp->c[i];
  } else {
    const int n = v->lp->n;
    c = v->column < n ? (i == v->column ? 1.0 : 0.0) : (i == v->column - n ? -1.0 : 0.0);
  }
  for (int k = 0; k < v->n_ov; ++k)
    if (v->ov[k].kind == BL_OVERRIDE_OBJECTIVE && v->ov[k].variable == i) c = v->ov[k].value;
  return c;
}
static double cv_lower(const column_view* v, int i) {
  double x = v->lp->xl[i];
  for (int k = 0; k < v->n_ov; ++k)
    if (v->ov[k].kind == BL_OVERRIDE_LOWER && v->ov[k].variable == i) x = v->ov[k].value;
  return x;
}
static double cv_upper(const column_view* v, int i) {
  double x = v->lp->xu[i];
  for (int k = 0; k < v->n_ov; ++k)
    if (v->ov[k].kind == BL_OVERRIDE_UPPER && v->ov[k].variable == i) x = v->ov[k].value;
  return x;
}

/* ---- solver.hpp:250-334: residual metric, restart rule, weight ------------*/
static int m_residual(double dx2, double dy2, double cross, double eta, double w,
                      double* out) {
  const double msq = (w / eta) * dx2 + (1.0 / (eta * w)) * dy2 + 2.0 * cross;
  if (msq < 0.0) {
    const double scale = (w / eta) * dx2 + (1.0 / (eta * w)) * dy2 + 2.0 * fabs(cross);
    if (msq < -1e-12 * smax(1.0, scale)) return BL_ERR_DOMAIN;
    *out = 0.0;
    return BL_OK;
  }
  *out = sqrt(msq);
  return BL_OK;
}

static int restart_reason(double r, double ra, double rp, int64_t ik, int64_t tk,
                          const bl_config* c) {
  if (r <= c->beta_sufficient * ra) return BL_RESTART_SUFFICIENT;
  if (r <= c->beta_necessary * ra && r > rp) return BL_RESTART_NECESSARY;
  if ((double)ik > c->beta_artificial * (double)tk) return BL_RESTART_ARTIFICIAL;
  return -1;
}

static double smoothed_weight(double w, double dxn, double dyn, double theta) {
  if (!(dxn > 0.0) || !(dyn > 0.0) || !isfinite(dxn) || !isfinite(dyn)) return w;
  const double d = dyn / dxn;
  if (!isfinite(d) || d <= 0.0) return w;
  const double log_w = log(w);
  const double proposed = theta * log(d) + (1.0 - theta) * log_w;
  const double cap = log(4.0);
  if (proposed > log_w + cap) return exp(log_w + cap);
  if (proposed < log_w - cap) return exp(log_w - cap);
  return exp(proposed);
}

/* ---- solver.hpp:358-416 ---------------------------------------------------*/
typedef struct report {
  double objective, bound_support, row_support, base_bound_support;
  double gap, primal, dual, score;
  int gap_ok, primal_ok, dual_ok;
} report;

static report evaluate_optimality(const column_view* v, const double* xt, const double* yt,
                                  const double* axt, const double* at_yt, double* red,
                                  double eps, double eps_dual, int robust) {
  const orc_lp* p = v->lp;
  report r;
  memset(&r, 0, sizeof(r));
  double obj = 0.0, c_sq = 0.0, dres_sq = 0.0, sup_r = 0.0, bsup = 0.0;
  for (int i = 0; i < p->n; ++i) {
    const double c = cv_cost(v, i);
    obj += c * xt[i];
    c_sq += c * c;
    const double lo = cv_lower(v, i), hi = cv_upper(v, i);
    const double g = -c - at_yt[i];
    const double rr = project_barrier(g, lo, hi);
    red[i] = rr;
    const double viol = c + at_yt[i] + rr;
    dres_sq += viol * viol;
    if (robust) {
      if (g > 0.0 && hi != kInf) sup_r += hi * g;
      else if (g < 0.0 && lo != -kInf) sup_r += lo * g;
    } else {
      sup_r += support_term(rr, lo, hi);
    }
    bsup += support_term(rr, p->xl[i], p->xu[i]);
  }
  double sup_y = 0.0, pres_sq = 0.0, ax_sq = 0.0;
  for (int i = 0; i < p->m; ++i) {
    const double lo = p->rl[i], hi = p->ru[i];
    sup_y += support_term(yt[i], lo, hi);
    const double viol = axt[i] - project_box(axt[i], lo, hi);
    pres_sq += viol * viol;
    ax_sq += axt[i] * axt[i];
  }
  r.objective = obj;
  r.bound_support = sup_r;
  r.row_support = sup_y;
  r.base_bound_support = bsup;
  r.primal = sqrt(pres_sq);
  r.dual = sqrt(dres_sq);
  const double supports = sup_r + sup_y;
  const double gap = obj + supports;
  const double gap_scale = 1.0 + fabs(obj) + fabs(supports);
  r.gap = isfinite(gap) ? fabs(gap) : kInf;
  r.gap_ok = isfinite(gap) && fabs(gap) <= eps * gap_scale;
  const double primal_scale = 1.0 + sqrt(ax_sq);
  r.primal_ok = r.primal <= eps * primal_scale;
  const double dual_scale = 1.0 + sqrt(c_sq);
  r.dual_ok = r.dual <= eps_dual * dual_scale;
  double score = r.gap / gap_scale;
  if (score < r.primal / primal_scale) score = r.primal / primal_scale;
  if (score < r.dual / dual_scale) score = r.dual / dual_scale;
  r.score = score;
  return r;
}

/* ---- solver.hpp:433-527; returns 0 none, 1 primal, 2 dual -----------------*/
static int infeasibility_probe(const column_view* v, const double* x, const double* y,
                               const double* xt, const double* yt, const double* aty,
                               const double* ax, const double* axt, const double* red,
                               double eps, double* ws_n1, double* ws_n2, double* ws_m,
                               int64_t* products) {
  const orc_lp* p = v->lp;
  const int n = p->n, m = p->m;
  double* dy = ws_m;
  double* dr = ws_n1;
  for (int i = 0; i < m; ++i) dy[i] = project_barrier(yt[i] - y[i], p->rl[i], p->ru[i]);
  for (int i = 0; i < n; ++i) {
    const double lo = cv_lower(v, i), hi = cv_upper(v, i);
    const double cur = project_barrier(-cv_cost(v, i) - aty[i], lo, hi);
    dr[i] = project_barrier(red[i] - cur, lo, hi);
  }
  double sup = 0.0, scale = 0.0;
  for (int i = 0; i < m; ++i) {
    const double t = support_term(dy[i], p->rl[i], p->ru[i]);
    sup += t;
    scale += fabs(t);
  }
  for (int i = 0; i < n; ++i) {
    const double t = support_term(dr[i], cv_lower(v, i), cv_upper(v, i));
    sup += t;
    scale += fabs(t);
  }
  if (sup < -1e-9 * smax(1.0, scale)) {
    double* atdy = ws_n2;
    csr_apply(n, p->trp, p->tci, p->tcv, dy, atdy);
    ++*products;
    double res = 0.0;
    for (int i = 0; i < n; ++i) {
      const double q = atdy[i] + dr[i];
      res += q * q;
    }
    if (sqrt(res) <= eps * fabs(sup)) return 1;
  }
  double desc = 0.0, dscale = 0.0;
  for (int i = 0; i < n; ++i) {
    const double t = cv_cost(v, i) * (xt[i] - x[i]);
    desc += t;
    dscale += fabs(t);
  }
  if (desc < -1e-9 * smax(1.0, dscale)) {
    double var_sq = 0.0, row_sq = 0.0;
    for (int i = 0; i < n; ++i) {
      const double d = xt[i] - x[i];
      const double q = d - project_recession(d, cv_lower(v, i), cv_upper(v, i));
      var_sq += q * q;
    }
    for (int i = 0; i < m; ++i) {
      const double d = axt[i] - ax[i];
      const double q = d - project_recession(d, p->rl[i], p->ru[i]);
      row_sq += q * q;
    }
    const double budget = eps * fabs(desc);
    if (sqrt(var_sq) <= budget && sqrt(row_sq) <= budget) return 2;
  }
  return 0;
}

/* ---- batch_solver.hpp:78-355 ----------------------------------------------*/
typedef struct best_cand {
  double score;
  report rep;
  double fixed_point;
  int has;
} best_cand;

static void swap_d(double* a, int s, int t) { double q = a[s]; a[s] = a[t]; a[t] = q; }
static void swap_i(int* a, int s, int t) { int q = a[s]; a[s] = a[t]; a[t] = q; }
static void swap_col(double* M, int rows, int s, int t) {
  if (s == t) return;
  double* a = M + (size_t)s * rows;
  double* b = M + (size_t)t * rows;
  for (int i = 0; i < rows; ++i) { double q = a[i]; a[i] = b[i]; b[i] = q; }
}
static int cmp_ov(const void* a, const void* b) {
  const bl_override* x = (const bl_override*)a;
  const bl_override* y = (const bl_override*)b;
  if (x->column != y->column) return x->column < y->column ? -1 : 1;
  return x->reserved < y->reserved ? -1 : (x->reserved > y->reserved); /* stable */
}

static void fill_result(bl_column_result* r, int status, const report* rep, double fp,
                        int64_t it, int restarts, int kind) {
  memset(r, 0, sizeof(*r));
  r->status = status;
  r->objective = rep->objective;
  r->gap = rep->gap;
  r->primal = rep->primal;
  r->dual = rep->dual;
  r->fixed_point = fp;
  r->iterations = it;
  r->restarts = restarts;
  r->bound_support = rep->bound_support;
  r->row_support = rep->row_support;
  r->base_bound_support = rep->base_bound_support;
  r->has_solution = 1;
  r->vectors_exist = 1;
  r->certificate_kind = kind;
  r->has_certificate = kind != 0;
}

/* x_out/y_out/r_out (column-major, may be NULL) receive the returned
 * vectors. Returns a bl_code. */
int orc_solve_batch(const orc_lp* lp, int width, int mode, const bl_override* ov_in,
                    int n_ov, const bl_config* cfg, const int32_t* presets, int n_presets,
                    const double* w0, bl_summary* sum, bl_column_result* res,
                    double* x_out, double* y_out, double* r_out) {
  const int n = lp->n, m = lp->m;
  memset(sum, 0, sizeof(*sum));
  sum->trajectory_hash = 1469598103934665603ull;
  if (width == 0) return BL_OK;
  int* frozen = (int*)calloc((size_t)width, sizeof(int));
  for (int k = 0; k < n_presets; ++k) {
    if (presets[k] < 0 || presets[k] >= width) { free(frozen); return BL_ERR_OUT_OF_RANGE; }
    if (frozen[presets[k]]) { free(frozen); return BL_ERR_INVALID_ARGUMENT; }
    frozen[presets[k]] = 1;
  }
  /* overrides sorted by column, stable (problem.hpp:168-176) */
  bl_override* ov = (bl_override*)malloc(sizeof(bl_override) * (n_ov ? n_ov : 1));
  memcpy(ov, ov_in, sizeof(bl_override) * n_ov);
  for (int k = 0; k < n_ov; ++k) ov[k].reserved = k;
  qsort(ov, n_ov, sizeof(bl_override), cmp_ov);
  int* off = (int*)calloc((size_t)width + 1, sizeof(int));
  for (int k = 0; k < n_ov; ++k) ++off[ov[k].column + 1];
  for (int j = 0; j < width; ++j) off[j + 1] += off[j];

  const size_t W = (size_t)width;
  double *X = calloc(W * n, 8), *Y = calloc(W * m, 8), *AX = calloc(W * m, 8);
  double *aX = calloc(W * n, 8), *aY = calloc(W * m, 8), *aAX = calloc(W * m, 8);
  double *XT = calloc(W * n, 8), *YT = calloc(W * m, 8), *AXT = calloc(W * m, 8);
  double *ATY = calloc(W * n, 8), *ATYT = calloc(W * n, 8);
  double *wts = malloc(W * 8), *resid = calloc(W, 8), *anc = calloc(W, 8);
  double *red = calloc((size_t)n + 1, 8), *wn1 = calloc((size_t)n + 1, 8);
  double *wn2 = calloc((size_t)n + 1, 8), *wm = calloc((size_t)m + 1, 8);
  int* slot = malloc(W * sizeof(int));
  best_cand* best = calloc(W, sizeof(best_cand));
  /* best vectors, per slot (swapped along like BestCandidate) */
  double *bX = calloc(W * n, 8), *bY = calloc(W * m, 8), *bR = calloc(W * n, 8);
  int rc = BL_OK;

  for (int j = 0; j < width; ++j) {
    wts[j] = w0 ? w0[j] : cfg->w_init;
    slot[j] = j;
    best[j].score = kInf;
    best[j].fixed_point = kInf;
    best[j].rep.gap = best[j].rep.primal = best[j].rep.dual = kInf;
  }
  double eta = cfg->eta;
  if (!(eta > 0.0)) eta = 0.998 / (lp->rp[m] == 0 ? 1.0 : orc_spectral_norm(lp));
  const double eps_dual = cfg->eps_dual < 0.0 ? cfg->eps_opt : cfg->eps_dual;
  sum->eta = eta;

  for (int j = 0; j < width; ++j) {
    column_view v = {lp, mode, j, ov + off[j], off[j + 1] - off[j]};
    for (int i = 0; i < n; ++i)
      X[(size_t)j * n + i] = project_box(0.0, cv_lower(&v, i), cv_upper(&v, i));
  }
  for (int j = 0; j < width; ++j)
    csr_apply(m, lp->rp, lp->ci, lp->cv, X + (size_t)j * n, AX + (size_t)j * m);
  sum->sparse_products = 1;

  int active = width;
#define SWAP_SLOTS(s, t)                                      \
  do {                                                        \
    if ((s) != (t)) {                                         \
      swap_col(X, n, s, t); swap_col(Y, m, s, t);             \
      swap_col(AX, m, s, t); swap_col(aX, n, s, t);           \
      swap_col(aY, m, s, t); swap_col(aAX, m, s, t);          \
      swap_d(wts, s, t); swap_d(resid, s, t); swap_d(anc, s, t); \
      swap_i(slot, s, t);                                     \
      { best_cand q = best[s]; best[s] = best[t]; best[t] = q; } \
      swap_col(bX, n, s, t); swap_col(bY, m, s, t); swap_col(bR, n, s, t); \
    }                                                         \
  } while (0)
  for (int s = active - 1; s >= 0; --s)
    if (frozen[slot[s]]) { --active; SWAP_SLOTS(s, active); }
  memcpy(aX, X, W * n * 8);
  memcpy(aY, Y, W * m * 8);
  memcpy(aAX, AX, W * m * 8);

  double mean_anchor = 0.0, mean_prev = 0.0;
  int64_t inner_k = 0, total_k = 0;
  int restarts = 0;
  while (active > 0) {
    for (int j = 0; j < active; ++j)
      csr_apply(n, lp->trp, lp->tci, lp->tcv, Y + (size_t)j * m, ATY + (size_t)j * n);
    ++sum->sparse_products;
    for (int j = 0; j < active; ++j) {
      const int o = slot[j];
      column_view v = {lp, mode, o, ov + off[o], off[o + 1] - off[o]};
      const double tau = eta / wts[j];
      const double* x = X + (size_t)j * n;
      const double* aty = ATY + (size_t)j * n;
      double* xt = XT + (size_t)j * n;
      for (int i = 0; i < n; ++i)
        xt[i] = project_box(x[i] - tau * (cv_cost(&v, i) + aty[i]), cv_lower(&v, i),
                            cv_upper(&v, i));
    }
    for (int j = 0; j < active; ++j)
      csr_apply(m, lp->rp, lp->ci, lp->cv, XT + (size_t)j * n, AXT + (size_t)j * m);
    ++sum->sparse_products;
    for (int j = 0; j < active; ++j) {
      const double sigma = eta * wts[j];
      for (int i = 0; i < m; ++i) {
        const size_t e = (size_t)j * m + i;
        const double vv = 2.0 * AXT[e] - AX[e];
        const double s = Y[e] / sigma + vv;
        YT[e] = sigma * (s - project_box(s, lp->rl[i], lp->ru[i]));
      }
    }
    for (int j = 0; j < active; ++j) {
      double dx2 = 0.0, dy2 = 0.0, cross = 0.0;
      for (int i = 0; i < n; ++i) {
        const double d = XT[(size_t)j * n + i] - X[(size_t)j * n + i];
        dx2 += d * d;
      }
      for (int i = 0; i < m; ++i) {
        const size_t e = (size_t)j * m + i;
        const double d = YT[e] - Y[e];
        dy2 += d * d;
        cross += d * (AXT[e] - AX[e]);
      }
      rc = m_residual(dx2, dy2, cross, eta, wts[j], &resid[j]);
      if (rc != BL_OK) goto out;
    }
    double rsum = 0.0;
    int rcount;
    if (cfg->average_over_all_columns) {
      for (int j = 0; j < width; ++j) rsum += resid[j];
      rcount = width;
    } else {
      for (int j = 0; j < active; ++j) rsum += resid[j];
      rcount = active;
    }
    const double mean = rsum / rcount;
    if (inner_k == 0) {
      mean_anchor = mean;
      for (int j = 0; j < active; ++j) anc[j] = resid[j];
    }
    const int at_cap = total_k >= cfg->max_iterations;
    if (total_k % cfg->termination_check_period == 0 || at_cap) {
      for (int j = 0; j < active; ++j)
        csr_apply(n, lp->trp, lp->tci, lp->tcv, YT + (size_t)j * m, ATYT + (size_t)j * n);
      ++sum->sparse_products;
      int finished = 0;
      for (int j = 0; j < active; ++j) {
        const int o = slot[j];
        column_view v = {lp, mode, o, ov + off[o], off[o + 1] - off[o]};
        const double* xt = XT + (size_t)j * n;
        const double* yt = YT + (size_t)j * m;
        report rep = evaluate_optimality(&v, xt, yt, AXT + (size_t)j * m,
                                         ATYT + (size_t)j * n, red, cfg->eps_opt, eps_dual,
                                         cfg->robust_bound_contribution);
        int status = -1, kind = 0;
        if (rep.gap_ok && rep.primal_ok && rep.dual_ok) {
          status = BL_OPTIMAL;
        } else {
          kind = infeasibility_probe(&v, X + (size_t)j * n, Y + (size_t)j * m, xt, yt,
                                     ATY + (size_t)j * n, AX + (size_t)j * m,
                                     AXT + (size_t)j * m, red, cfg->eps_infeas, wn1, wn2, wm,
                                     &sum->sparse_products);
          if (kind == 1) status = BL_PRIMAL_INFEASIBLE;
          else if (kind == 2) status = BL_DUAL_INFEASIBLE;
        }
        if (status >= 0) {
          fill_result(&res[o], status, &rep, resid[j], total_k, restarts, kind);
          if (x_out) memcpy(x_out + (size_t)o * n, xt, 8 * (size_t)n);
          if (y_out) memcpy(y_out + (size_t)o * m, yt, 8 * (size_t)m);
          if (r_out) memcpy(r_out + (size_t)o * n, red, 8 * (size_t)n);
          frozen[o] = 1;
          ++finished;
          continue;
        }
        if (!(rep.score >= best[j].score)) {
          best[j].score = rep.score;
          best[j].rep = rep;
          best[j].fixed_point = resid[j];
          best[j].has = 1;
          memcpy(bX + (size_t)j * n, xt, 8 * (size_t)n);
          memcpy(bY + (size_t)j * m, yt, 8 * (size_t)m);
          memcpy(bR + (size_t)j * n, red, 8 * (size_t)n);
        }
      }
      if (finished) {
        for (int s = active - 1; s >= 0; --s)
          if (frozen[slot[s]]) { --active; SWAP_SLOTS(s, active); }
        if (active == 0) break;
      }
    }
    if (at_cap) {
      for (int j = 0; j < active; ++j) {
        const int o = slot[j];
        fill_result(&res[o], BL_ITERATION_LIMIT, &best[j].rep, best[j].fixed_point, total_k,
                    restarts, 0);
        res[o].has_solution = res[o].vectors_exist = best[j].has;
        if (!best[j].has) res[o].objective = 0.0;
        if (best[j].has) {
          if (x_out) memcpy(x_out + (size_t)o * n, bX + (size_t)j * n, 8 * (size_t)n);
          if (y_out) memcpy(y_out + (size_t)o * m, bY + (size_t)j * m, 8 * (size_t)m);
          if (r_out) memcpy(r_out + (size_t)o * n, bR + (size_t)j * n, 8 * (size_t)n);
        } else {
          res[o].bound_support = res[o].row_support = res[o].base_bound_support = 0.0;
        }
        frozen[o] = 1;
      }
      active = 0;
      break;
    }
    if (inner_k >= 1) {
      const int reason = restart_reason(mean, mean_anchor, mean_prev, inner_k, total_k, cfg);
      if (reason >= 0) {
        sum->restart_log_size += 1;
        for (int j = 0; j < active; ++j) {
          if (resid[j] <= anc[j]) {
            double dx = 0.0, dy = 0.0;
            for (int i = 0; i < n; ++i) {
              const double d = X[(size_t)j * n + i] - aX[(size_t)j * n + i];
              dx += d * d;
            }
            for (int i = 0; i < m; ++i) {
              const double d = Y[(size_t)j * m + i] - aY[(size_t)j * m + i];
              dy += d * d;
            }
            wts[j] = smoothed_weight(wts[j], sqrt(dx), sqrt(dy), cfg->theta);
          }
          memcpy(aX + (size_t)j * n, X + (size_t)j * n, 8 * (size_t)n);
          memcpy(aY + (size_t)j * m, Y + (size_t)j * m, 8 * (size_t)m);
          memcpy(aAX + (size_t)j * m, AX + (size_t)j * m, 8 * (size_t)m);
        }
        inner_k = 0;
        ++restarts;
        continue;
      }
    }
    {
      const double alpha = (double)(inner_k + 1) / (double)(inner_k + 2);
      for (int j = 0; j < active; ++j) {
        /* Halpern on post-compaction slots with the slot's XT/YT/AXT, which
         * are NOT swapped by compaction (batch_solver.hpp:143-156,326-335) */
        for (int i = 0; i < n; ++i) {
          const size_t e = (size_t)j * n + i;
          X[e] = alpha * (2.0 * XT[e] - X[e]) + (1.0 - alpha) * aX[e];
        }
        for (int i = 0; i < m; ++i) {
          const size_t e = (size_t)j * m + i;
          Y[e] = alpha * (2.0 * YT[e] - Y[e]) + (1.0 - alpha) * aY[e];
          AX[e] = alpha * (2.0 * AXT[e] - AX[e]) + (1.0 - alpha) * aAX[e];
        }
      }
    }
    mean_prev = mean;
    ++inner_k;
    ++total_k;
    if (cfg->trace_iterates) {
      uint64_t h = sum->trajectory_hash;
      const unsigned char* b = (const unsigned char*)X;
      for (size_t k = 0; k < (size_t)n * 8; ++k) { h ^= b[k]; h *= 1099511628211ull; }
      b = (const unsigned char*)Y;
      for (size_t k = 0; k < (size_t)m * 8; ++k) { h ^= b[k]; h *= 1099511628211ull; }
      sum->trajectory_hash = h;
    }
  }
  sum->iterations = total_k;
  sum->restarts = restarts;
  for (int j = 0; j < width; ++j)
    if (!frozen[j]) rc = BL_ERR_LOGIC;
out:
#undef SWAP_SLOTS
  free(frozen); free(ov); free(off);
  free(X); free(Y); free(AX); free(aX); free(aY); free(aAX);
  free(XT); free(YT); free(AXT); free(ATY); free(ATYT);
  free(wts); free(resid); free(anc); free(red); free(wn1); free(wn2); free(wm);
  free(slot); free(best); free(bX); free(bY); free(bR);
  return rc;
}
